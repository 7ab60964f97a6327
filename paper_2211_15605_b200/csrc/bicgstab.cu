// bicgstab.cu -- a-4 matrix-free 7-point apply and a-5/a-6 BiCGSTAB
// ("No preconditioners").
//
// Per iteration three fused kernels, each ending in a deterministic,
// correctly rounded grid reduction whose last block runs the scalar part of
// the algorithm on the device (no host round trip):
//   K1: p = fma(beta, fma(-omega, v, p), r) (recomputed at the halo from the
//       OLD p, v -> p and v are ping-pong buffers), v = A p, sigma = <r^, v>
//   K2: s = fma(-alpha, v, r) (recomputed at the halo), t = A s,
//       <t,s>, <t,t>, <s,s>
//   K3: x = fma(omega, s, fma(alpha, p, x)), r = fma(-omega, t, s),
//       rho = <r^, r>, rr = <r, r>
// 17 vector passes + 2 coefficient passes per iteration.
#include <climits>
#include <cstddef>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "bicg_state.cuh"

namespace mfx {

mfx_status persist_solve_launch(const Geo &G, const mfx_eqsys *A, double *x, const WsView &W, int maxit,
                                cudaStream_t s);
mfx_status stencil_launch(int mode, bool sym, const Geo &G, const double *const halo[3], const mfx_eqsys *A,
                          const double *extra, double *o0, double *o1, double *o2, WsHeader *h, dd *part,
                          double tol, int maxit, cudaStream_t s, int reverse = 0, int kbeg = 0, int kend = 0,
                          int ghost_store = 0, dd *rank_part = nullptr, int chain = 0);

// L2 ping-pong: consecutive sweeps alternate direction so each kernel starts
// on the cells the previous one touched last (126 MB L2).  MFX_REVERSE=0
// disables it.  Results are unchanged (elementwise updates, correctly
// rounded dots).
static int sweep_dir(bool flip)
{
    static int enabled = -1;
    if (enabled < 0) {
        const char *e = getenv("MFX_REVERSE");
        enabled = e ? atoi(e) : 1;
    }
    static thread_local int dir = 0;
    if (!enabled) return 0;
    if (flip) dir ^= 1;
    return dir;
}

namespace {

constexpr int kThreads = 256;

struct Coef {
    const double *aP, *aE, *aW, *aN, *aS, *aT, *aB;
};

// y = aP x_P, then fma(-a_nb, x_nb, y) for W,E,S,N,B,T
template <bool SYM, class XV>
__device__ __forceinline__ double stencil(const Geo &G, const Coef &c, long long n, int i, int j, int k,
                                          XV xv)
{
    double aW, aE, aS, aN, aB, aT;
    if (SYM) {
        aW = i > 0 ? __ldg(c.aE + n - 1) : 0.0;
        aE = __ldg(c.aE + n);
        aS = j > 0 ? __ldg(c.aN + n - G.sy) : 0.0;
        aN = __ldg(c.aN + n);
        aB = k > 0 ? __ldg(c.aT + n - G.sz) : 0.0;
        aT = __ldg(c.aT + n);
    } else {
        aW = __ldg(c.aW + n); aE = __ldg(c.aE + n); aS = __ldg(c.aS + n);
        aN = __ldg(c.aN + n); aB = __ldg(c.aB + n); aT = __ldg(c.aT + n);
    }
    const double xW = i > 0 ? xv(n - 1) : 0.0;
    const double xE = i < G.nx - 1 ? xv(n + 1) : 0.0;
    const double xS = j > 0 ? xv(n - G.sy) : 0.0;
    const double xN = j < G.ny - 1 ? xv(n + G.sy) : 0.0;
    const double xB = k > 0 ? xv(n - G.sz) : 0.0;
    const double xT = k < G.nz - 1 ? xv(n + G.sz) : 0.0;
    // p': the diagonal is the row sum of the face coefficients,
    // rebuilt in the assembly's order instead of read (8 B/cell less)
    const double aP = SYM ? ((((aW + aE) + aS) + aN) + aB) + aT : __ldg(c.aP + n);
    double y = aP * xv(n);
    y = fma(-aW, xW, y);
    y = fma(-aE, xE, y);
    y = fma(-aS, xS, y);
    y = fma(-aN, xN, y);
    y = fma(-aB, xB, y);
    y = fma(-aT, xT, y);
    return y;
}

__device__ __forceinline__ void decode(const Geo &G, long long n, int &i, int &j, int &k)
{
    long long pl = n / G.sz;
    long long rem = n - pl * G.sz;
    k = (int)pl;
    j = (int)(rem / G.nx);
    i = (int)(rem - (long long)j * G.nx);
}

#define GRID_STRIDE(n) \
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < G.N; n += (long long)gridDim.x * blockDim.x)

// ------------------------------------------------------------------ plain apply
template <bool SYM>
__global__ void __launch_bounds__(kThreads) k_spmv(Geo G, Coef c, const double *__restrict__ x, double *y)
{
    GRID_STRIDE(n)
    {
        int i, j, k;
        decode(G, n, i, j, k);
        y[n] = stencil<SYM>(G, c, n, i, j, k, [&](long long m) { return __ldg(x + m); });
    }
}

// ------------------------------------------------------------------ setup
template <bool SYM>
__global__ void __launch_bounds__(kThreads) k_setup(Geo G, Coef c, const double *__restrict__ b,
                                                   const double *__restrict__ x, double *r, WsHeader *h, dd *part,
                                                   double tol, int maxit)
{
    Acc bb, rr;
    bb.zero();
    rr.zero();
    GRID_STRIDE(n)
    {
        int i, j, k;
        decode(G, n, i, j, k);
        const double y = stencil<SYM>(G, c, n, i, j, k, [&](long long m) { return __ldg(x + m); });
        const double bv = __ldg(b + n);
        const double rv = bv - y;
        r[n] = rv;
        bb.prod(bv, bv);
        rr.prod(rv, rv);
    }
    __shared__ dd sh[(kThreads / 32) * 2];
    dd v[2] = {bb.get(), rr.get()}, out[2];
    if (grid_reduce_dd<2>(v, part, &h->ticket[1], sh, out) && threadIdx.x == 0)
        bicg_setup(h->sc, dd_round(out[0]), dd_round(out[1]), tol, maxit);
}

// true residual at exit (reading Q2: "true residual reported at exit only"):
// r = b - A x with the canonical operator, <b,b> and <r,r> correctly rounded,
// h->true_rel = sqrt(<r,r>) / sqrt(<b,b>) (0 when b = 0).  One extra apply per
// solve; it reads nothing the solver writes afterwards.
template <bool SYM>
__global__ void __launch_bounds__(kThreads) k_true_resid(Geo G, Coef c, const double *__restrict__ b,
                                                        const double *__restrict__ x, WsHeader *h, dd *part)
{
    Acc bb, rr;
    bb.zero();
    rr.zero();
    GRID_STRIDE(n)
    {
        int i, j, k;
        decode(G, n, i, j, k);
        const double y = stencil<SYM>(G, c, n, i, j, k, [&](long long m) { return __ldg(x + m); });
        const double bv = __ldg(b + n);
        const double rv = bv - y;
        bb.prod(bv, bv);
        rr.prod(rv, rv);
    }
    __shared__ dd sh[(kThreads / 32) * 2];
    dd v[2] = {bb.get(), rr.get()}, out[2];
    if (grid_reduce_dd<2>(v, part, &h->ticket[1], sh, out) && threadIdx.x == 0) {
        const double bn = sqrt(dd_round(out[0]));
        h->true_rel = bn == 0.0 ? 0.0 : sqrt(dd_round(out[1])) / bn;
    }
}

__global__ void k_zero_if(const WsHeader *h, double *x, long long N)
{
    if (!h->sc.zero_x) return;
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += (long long)gridDim.x * blockDim.x)
        x[n] = 0.0;
}

// ------------------------------------------------------------------ K1
// The phase bodies and scalar tails are shared by the per-phase kernels
// (k1/k2/k3) and the grid-synchronous persistent solver (k_bicg_grid).  LD
// selects the load path: __ldg for data that is constant during a kernel,
// L1-cached weak loads (coherent after the grid barrier's fence) for vectors another CTA wrote earlier in
// the same persistent kernel.
template <bool CG>
__device__ __forceinline__ double ldv(const double *p)
{
    // CG: weak (L1-cached) load, coherent in k_bicg_grid because every grid
    // barrier ends with a gpu-scope fence in each CTA (MEMBAR + CCTL.IVALL:
    // the SM's L1 is invalidated) before anything another CTA wrote is read.
    if (CG) {
        double v;
        asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
        return v;
    }
    return __ldg(p);
}

template <bool SYM, bool CG>
__device__ __forceinline__ void k1_body(const Geo &G, const Coef &c, const double *r, double *rh, const double *p_old,
                                        const double *v_old, double *p_new, double *v_new, const K1Pro &P, Acc &sg,
                                        long long n0, long long n1, long long step)
{
    const double beta = P.beta, omega = P.omega;
    const bool rst = P.rst;
    for (long long n = n0; n < n1; n += step) {
        int i, j, k;
        decode(G, n, i, j, k);
        auto pv = [&](long long m) {
            if (rst) return fma(beta, fma(-omega, 0.0, 0.0), ldv<CG>(r + m));
            return fma(beta, fma(-omega, ldv<CG>(v_old + m), ldv<CG>(p_old + m)), ldv<CG>(r + m));
        };
        const double v = stencil<SYM>(G, c, n, i, j, k, pv);
        p_new[n] = pv(n);
        v_new[n] = v;
        double rhv;
        if (rst) {
            rhv = ldv<CG>(r + n);
            rh[n] = rhv;
        } else {
            rhv = CG ? ldv<true>(rh + n) : rh[n];
        }
        sg.prod(rhv, v);
    }
}

template <bool SYM>
__global__ void __launch_bounds__(kThreads) k1(Geo G, Coef c, const double *__restrict__ r, double *rh,
                                              const double *__restrict__ p_old, const double *__restrict__ v_old,
                                              double *p_new, double *v_new, WsHeader *h, dd *part)
{
    SolverScalars &S = h->sc;
    if (S.done) return;
    const K1Pro P = bicg_k1_prologue(S);
    if (P.breakdown) {
        if (blockIdx.x == 0 && threadIdx.x == 0) bicg_breakdown(S);
        return;
    }
    Acc sg;
    sg.zero();
    k1_body<SYM, false>(G, c, r, rh, p_old, v_old, p_new, v_new, P, sg,
                        (long long)blockIdx.x * blockDim.x + threadIdx.x, G.N, (long long)gridDim.x * blockDim.x);
    __shared__ dd sh[(kThreads / 32) * 1];
    dd vv[1] = {sg.get()}, out[1];
    if (grid_reduce_dd<1>(vv, part, &h->ticket[1], sh, out) && threadIdx.x == 0) bicg_k1_tail(S, P, dd_round(out[0]));
}

// ------------------------------------------------------------------ K2
template <bool SYM, bool CG>
__device__ __forceinline__ void k2_body(const Geo &G, const Coef &c, const double *r, const double *v, double *t,
                                        double alpha, Acc &ts, Acc &tt, Acc &ss, long long n0, long long n1,
                                        long long step)
{
    for (long long n = n0; n < n1; n += step) {
        int i, j, k;
        decode(G, n, i, j, k);
        auto sv = [&](long long m) { return fma(-alpha, ldv<CG>(v + m), ldv<CG>(r + m)); };
        const double tv = stencil<SYM>(G, c, n, i, j, k, sv);
        const double s = sv(n);
        t[n] = tv;
        ts.prod(tv, s);
        tt.prod(tv, tv);
        ss.prod(s, s);
    }
}

template <bool SYM>
__global__ void __launch_bounds__(kThreads) k2(Geo G, Coef c, const double *__restrict__ r,
                                              const double *__restrict__ v, double *t, WsHeader *h, dd *part)
{
    SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    Acc ts, tt, ss;
    ts.zero(); tt.zero(); ss.zero();
    k2_body<SYM, false>(G, c, r, v, t, S.alpha, ts, tt, ss, (long long)blockIdx.x * blockDim.x + threadIdx.x, G.N,
                        (long long)gridDim.x * blockDim.x);
    __shared__ dd sh[(kThreads / 32) * 3];
    dd vv[3] = {ts.get(), tt.get(), ss.get()}, out[3];
    if (grid_reduce_dd<3>(vv, part, &h->ticket[1], sh, out) && threadIdx.x == 0)
        bicg_k2_tail(S, dd_round(out[0]), dd_round(out[1]), dd_round(out[2]));
}

// ------------------------------------------------------------------ K3
template <bool CG>
__device__ __forceinline__ void k3_body(double *x, double *r, const double *rh, const double *p, const double *v,
                                        const double *t, double alpha, double omega, bool half, Acc &rhr, Acc &rr,
                                        long long n0, long long n1, long long step)
{
    for (long long n = n0; n < n1; n += step) {
        const double s = fma(-alpha, ldv<CG>(v + n), CG ? ldv<true>(r + n) : r[n]);
        double xn, rn;
        if (half) {
            xn = fma(alpha, ldv<CG>(p + n), CG ? ldv<true>(x + n) : x[n]);
            rn = s;
        } else {
            xn = fma(omega, s, fma(alpha, ldv<CG>(p + n), CG ? ldv<true>(x + n) : x[n]));
            rn = fma(-omega, ldv<CG>(t + n), s);
        }
        x[n] = xn;
        r[n] = rn;
        rhr.prod(ldv<CG>(rh + n), rn);
        rr.prod(rn, rn);
    }
}

__global__ void __launch_bounds__(kThreads) k3(Geo G, double *x, double *r, const double *__restrict__ rh,
                                              const double *__restrict__ p, const double *__restrict__ v,
                                              const double *__restrict__ t, WsHeader *h, dd *part)
{
    SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    const bool half = S.half != 0;
    Acc rhr, rr;
    rhr.zero(); rr.zero();
    k3_body<false>(x, r, rh, p, v, t, S.alpha, S.omega, half, rhr, rr,
                   (long long)blockIdx.x * blockDim.x + threadIdx.x, G.N, (long long)gridDim.x * blockDim.x);
    __shared__ dd sh[(kThreads / 32) * 2];
    dd vv[2] = {rhr.get(), rr.get()}, out[2];
    if (grid_reduce_dd<2>(vv, part, &h->ticket[1], sh, out) && threadIdx.x == 0)
        bicg_k3_tail(S, half, dd_round(out[0]), dd_round(out[1]));
}

// K3, streaming form used with the TMA path: x fastest and nx even, so every
// field is a sequence of 16-byte pairs; a persistent grid walks the pairs two
// at a time with all twelve 16-byte loads issued before any arithmetic.
__device__ __forceinline__ double2 ldg2(const double *p) { return __ldg((const double2 *)p); }

struct K3Pair {
    double2 x, r, rh, p, v, t;
};

__device__ __forceinline__ void k3_load(K3Pair &d, long long e, const double *x, const double *r, const double *rh,
                                        const double *p, const double *v, const double *t, bool half)
{
    d.v = ldg2(v + e);
    d.r = *(const double2 *)(r + e);
    d.p = ldg2(p + e);
    d.x = *(const double2 *)(x + e);
    d.rh = ldg2(rh + e);
    if (!half) d.t = ldg2(t + e);
}

__device__ __forceinline__ void k3_cell(double xv, double rv, double rhv, double pv, double vv, double tv, double alpha,
                                        double omega, bool half, double &xo, double &ro, Acc &rhr, Acc &rr)
{
    const double s = fma(-alpha, vv, rv);
    if (half) {
        xo = fma(alpha, pv, xv);
        ro = s;
    } else {
        xo = fma(omega, s, fma(alpha, pv, xv));
        ro = fma(-omega, tv, s);
    }
    rhr.prod(rhv, ro);
    rr.prod(ro, ro);
}

__device__ __forceinline__ void k3_store(const K3Pair &d, long long e, double *x, double *r, double alpha,
                                         double omega, bool half, Acc &rhr, Acc &rr)
{
    double2 xo, ro;
    k3_cell(d.x.x, d.r.x, d.rh.x, d.p.x, d.v.x, d.t.x, alpha, omega, half, xo.x, ro.x, rhr, rr);
    k3_cell(d.x.y, d.r.y, d.rh.y, d.p.y, d.v.y, d.t.y, alpha, omega, half, xo.y, ro.y, rhr, rr);
    *(double2 *)(x + e) = xo;
    *(double2 *)(r + e) = ro;
}

__global__ void __launch_bounds__(kThreads) k3v(long long N, double *x, double *r, const double *__restrict__ rh,
                                               const double *__restrict__ p, const double *__restrict__ v,
                                               const double *__restrict__ t, WsHeader *h, dd *part, int rev,
                                               dd *rank_part, int chain)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // chained (path 1): K2's scalar tail runs here in every CTA -- fold K2's
    // published <t,s>, <t,t>, <s,s> partials onto the state after K1's tail
    // (sc2); the last CTA writes the state after K3's tail to sc
    SolverScalars L;
    if (chain) {
        __shared__ dd s_fsh[32], s_fbc[3];
        L = sc_ldcg(&h->sc2);
        if (!(L.done || L.skip)) {
            double o[3];
            fold_published<3>(part + kPartK2, __ldcg(&h->npart[1]), 3, s_fsh, s_fbc, o);
            bicg_k2_tail(L, o[0], o[1], o[2]);
        }
        if (L.done || L.skip) {
            if (blockIdx.x == 0 && threadIdx.x == 0) h->sc = L;
            return;
        }
    } else {
        L = h->sc;
        if (L.done || L.skip) return;
    }
    const double alpha = L.alpha, omega = L.omega;
    const bool half = L.half != 0;
    Acc rhr, rr;
    rhr.zero(); rr.zero();
    const long long npairs = N / 2;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    K3Pair A, B;
    A.t = B.t = make_double2(0.0, 0.0);
    for (; i + stride < npairs; i += 2 * stride) {
        const long long ea = 2 * (rev ? npairs - 1 - i : i), eb = 2 * (rev ? npairs - 1 - (i + stride) : i + stride);
        k3_load(A, ea, x, r, rh, p, v, t, half);
        k3_load(B, eb, x, r, rh, p, v, t, half);
        k3_store(A, ea, x, r, alpha, omega, half, rhr, rr);
        k3_store(B, eb, x, r, alpha, omega, half, rhr, rr);
    }
    if (i < npairs) {
        const long long ea = 2 * (rev ? npairs - 1 - i : i);
        k3_load(A, ea, x, r, rh, p, v, t, half);
        k3_store(A, ea, x, r, alpha, omega, half, rhr, rr);
    }
    __shared__ dd sh[(kThreads / 32) * 2];
    dd vv[2] = {rhr.get(), rr.get()}, out[2];
    if (grid_reduce_dd<2>(vv, part, &h->ticket[1], sh, out) && threadIdx.x == 0) {
        if (rank_part) { rank_part[0] = out[0]; rank_part[1] = out[1]; }   // z-slab mode: folded across ranks
        else if (chain) { bicg_k3_tail(L, half, dd_round(out[0]), dd_round(out[1])); h->sc = L; }
        else bicg_k3_tail(h->sc, half, dd_round(out[0]), dd_round(out[1]));
    }
}

// ------------------------------------------------------------------ grid-synchronous persistent solver
// For systems whose working set fits in L2 (configuration 3: 1M cells, 88 MB
// for p') the three launches per iteration cost more than the data movement.
// k_bicg_grid runs the whole iteration loop in ONE cooperative launch: the
// K1/K2/K3 bodies above with coherent (L2) loads, and in place of the kernel
// boundaries a grid barrier that also performs the reduction: every CTA posts
// its double-double partials, the last to arrive folds them in block order,
// runs the phase's scalar tail (the same code as the per-phase kernels) and
// releases the others.  Same expressions, same correctly rounded dots: the
// iterates equal the other paths' bitwise.
__device__ __forceinline__ SolverScalars sc_load(const SolverScalars *S)
{
    static_assert(sizeof(SolverScalars) % 8 == 0, "8-byte words");
    SolverScalars L;
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(S);
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(&L);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(SolverScalars) / 8); q++) dst[q] = __ldcg(src + q);
    return L;
}
__device__ __forceinline__ void sc_store(SolverScalars *S, const SolverScalars &L)
{
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&L);
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(S);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(SolverScalars) / 8); q++) __stcg(dst + q, src[q]);
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int K, class Tail>
__device__ __forceinline__ void grid_sync_reduce(dd (&v)[K], dd *part, unsigned *ticket, unsigned *gen, dd *sh,
                                                 Tail tail)
{
    block_reduce_dd<K>(v, sh);
    __shared__ bool s_last;
    __shared__ unsigned s_gen;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; q++) part[(size_t)blockIdx.x * K + q] = v[q];
        s_gen = ld_acquire(gen);
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        dd acc[K];
#pragma unroll
        for (int q = 0; q < K; q++) acc[q] = dd{0.0, 0.0};
        for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
            for (int q = 0; q < K; q++) {
                dd x;
                x.hi = __ldcg(&part[(size_t)b * K + q].hi);
                x.lo = __ldcg(&part[(size_t)b * K + q].lo);
                acc[q] = dd_add(acc[q], x);
            }
        }
        block_reduce_dd<K>(acc, sh);
        if (threadIdx.x == 0) {
            tail(acc);
            *ticket = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        }
    } else if (threadIdx.x == 0) {
        while (ld_acquire(gen) == s_gen) __nanosleep(32);
    }
    if (threadIdx.x == 0) __threadfence();   // L1 invalidate: see ldv<true>
    __syncthreads();
}

struct GridVecs {
    double *r, *rh, *p[2], *v[2], *t;
};

template <bool SYM>
__global__ void __launch_bounds__(kThreads) k_bicg_grid(Geo G, Coef c, double *x, GridVecs W, WsHeader *h, dd *part)
{
    unsigned *ticket = &h->ticket[2], *gen = &h->ticket[3];
    SolverScalars *Sg = &h->sc;
    const long long n0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long step = (long long)gridDim.x * blockDim.x;
    __shared__ dd sh[(kThreads / 32) * 3];
    int parity = 0;
    for (;;) {
        SolverScalars L = sc_load(Sg);
        if (L.done) break;
        // ---- K1
        const K1Pro P = bicg_k1_prologue(L);
        if (P.breakdown) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                bicg_breakdown(L);
                sc_store(Sg, L);
            }
            break;
        }
        double *p_old = W.p[parity], *p_new = W.p[parity ^ 1];
        double *v_old = W.v[parity], *v_new = W.v[parity ^ 1];
        {
            Acc sg;
            sg.zero();
            k1_body<SYM, true>(G, c, W.r, W.rh, p_old, v_old, p_new, v_new, P, sg, n0, G.N, step);
            dd vv[1] = {sg.get()};
            grid_sync_reduce<1>(vv, part, ticket, gen, sh, [&](dd (&o)[1]) {
                SolverScalars T = sc_load(Sg);
                bicg_k1_tail(T, P, dd_round(o[0]));
                sc_store(Sg, T);
            });
        }
        parity ^= 1;
        L = sc_load(Sg);
        if (L.done || L.skip) continue;
        // ---- K2
        {
            Acc ts, tt, ss;
            ts.zero(); tt.zero(); ss.zero();
            k2_body<SYM, true>(G, c, W.r, v_new, W.t, L.alpha, ts, tt, ss, n0, G.N, step);
            dd vv[3] = {ts.get(), tt.get(), ss.get()};
            grid_sync_reduce<3>(vv, part, ticket, gen, sh, [&](dd (&o)[3]) {
                SolverScalars T = sc_load(Sg);
                bicg_k2_tail(T, dd_round(o[0]), dd_round(o[1]), dd_round(o[2]));
                sc_store(Sg, T);
            });
        }
        L = sc_load(Sg);
        if (L.done || L.skip) continue;
        // ---- K3
        {
            const bool half = L.half != 0;
            Acc rhr, rr;
            rhr.zero(); rr.zero();
            k3_body<true>(x, W.r, W.rh, p_new, v_new, W.t, L.alpha, L.omega, half, rhr, rr, n0, G.N, step);
            dd vv[2] = {rhr.get(), rr.get()};
            grid_sync_reduce<2>(vv, part, ticket, gen, sh, [&](dd (&o)[2]) {
                SolverScalars T = sc_load(Sg);
                bicg_k3_tail(T, half, dd_round(o[0]), dd_round(o[1]));
                sc_store(Sg, T);
            });
        }
    }
}

template <bool SYM>
int grid_solver_blocks(long long N)
{
    static int g = 0;
    if (!g) {
        int occ = 0, dev = 0, sms = 148;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bicg_grid<SYM>, kThreads, 0);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // fewer, fuller CTAs: every barrier is one atomic arrival per CTA
        const char *e = getenv("MFX_GRID_CTAS_PER_SM");
        const int want = e ? atoi(e) : 0;   // measured: more CTAs are faster (occupancy limit best)
        if (want > 0 && want < occ) occ = want;
        g = sms * (occ > 0 ? occ : 1);
        if (g > kMaxBlocks) g = kMaxBlocks;
    }
    const long long need = (N + kThreads - 1) / kThreads;
    return (int)(need < g ? need : g);
}

template <bool SYM>
mfx_status launch_grid_solver(const Geo &G, const Coef &c, double *x, const WsView &W, cudaStream_t s)
{
    GridVecs V;
    V.r = W.r; V.rh = W.rh; V.p[0] = W.p[0]; V.p[1] = W.p[1]; V.v[0] = W.v[0]; V.v[1] = W.v[1]; V.t = W.t;
    Geo Gc = G;
    Coef cc = c;
    WsHeader *h = W.hdr;
    dd *part = W.part;
    void *args[] = {&Gc, &cc, &x, &V, &h, &part};
    MFX_CUDA_TRY(cudaMemsetAsync(&W.hdr->ticket[2], 0, 2 * sizeof(unsigned), s));
    MFX_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_bicg_grid<SYM>, dim3(grid_solver_blocks<SYM>(G.N)),
                                             dim3(kThreads), args, 0, s));
    return MFX_OK;
}

int k3v_grid()
{
    static int g = 0;
    if (g) return g;
    int occ = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3v, kThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = sms * (occ > 0 ? occ : 1);
    if (g > kMaxBlocks) g = kMaxBlocks;
    return g;
}

Coef coef_of(const mfx_eqsys *A)
{
    Coef c;
    c.aP = A->aP; c.aE = A->aE; c.aW = A->aW; c.aN = A->aN; c.aS = A->aS; c.aT = A->aT; c.aB = A->aB;
    return c;
}

bool sys_ok(int kind, const mfx_eqsys *A)
{
    if (!A || !A->aE || !A->aN || !A->aT) return false;
    if (kind == MFX_EQ_PP) return !A->aW && !A->aS && !A->aB;   // aP derived, never read
    return A->aP && A->aW && A->aS && A->aB;
}

template <bool SYM>
mfx_status launch_iteration_tma(const Geo &G, const mfx_eqsys *A, const WsView &W, double *x, int parity, int nb,
                                cudaStream_t s)
{
    double *p_old = W.p[parity], *p_new = W.p[parity ^ 1];
    double *v_old = W.v[parity], *v_new = W.v[parity ^ 1];
    mfx_status st;
    // chained tails (option MFX_CHAIN=1): K1 and K2 publish their dot partials
    // and exit; K2 and K3 fold them in their prologues (every CTA), so no
    // last-CTA fold sits between the kernels (common.cuh).  Off: measured
    // slower (c2 K2 89 vs 82 us, K3 99 vs 88 us: every CTA re-reading the same
    // partials costs more than one CTA's serial fold).
    static const int chain = [] { const char *e = getenv("MFX_CHAIN"); return e ? atoi(e) : 0; }();
    count_launch(SYM ? 6 : 1, s, true);
    const double *h1[3] = {W.r, p_old, v_old};
    st = stencil_launch(2, SYM, G, h1, A, W.rh, p_new, v_new, W.rh, W.hdr, W.part, 0.0, 0, s, sweep_dir(true), 0, 0,
                        0, nullptr, chain);
    count_launch(SYM ? 6 : 1, s, false);
    if (st != MFX_OK) return st;
    count_launch(SYM ? 7 : 2, s, true);
    const double *h2[3] = {W.r, v_new, nullptr};
    st = stencil_launch(3, SYM, G, h2, A, nullptr, W.t, nullptr, nullptr, W.hdr, W.part, 0.0, 0, s, sweep_dir(true),
                        0, 0, 0, nullptr, chain);
    count_launch(SYM ? 7 : 2, s, false);
    if (st != MFX_OK) return st;
    count_launch(3, s, true);
    {
        long long np = G.N / 2;
        int g3 = k3v_grid();
        if ((long long)g3 * kThreads > np) g3 = (int)((np + kThreads - 1) / kThreads);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g3);
        cfg.blockDim = dim3(kThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = opt_pdl() ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MFX_CUDA_TRY(cudaLaunchKernelEx(&cfg, k3v, G.N, x, W.r, (const double *)W.rh, (const double *)p_new,
                                        (const double *)v_new, (const double *)W.t, W.hdr, W.part,
                                        sweep_dir(true), (dd *)nullptr, chain));
    }
    count_launch(3, s, false);
    (void)nb;
    return MFX_OK;
}

template <bool SYM>
void launch_iteration(const Geo &G, const Coef &c, const WsView &W, double *x, int parity, int nb, cudaStream_t s)
{
    double *p_old = W.p[parity], *p_new = W.p[parity ^ 1];
    double *v_old = W.v[parity], *v_new = W.v[parity ^ 1];
    count_launch(SYM ? 6 : 1, s, true);
    k1<SYM><<<nb, kThreads, 0, s>>>(G, c, W.r, W.rh, p_old, v_old, p_new, v_new, W.hdr, W.part);
    count_launch(SYM ? 6 : 1, s, false);
    count_launch(SYM ? 7 : 2, s, true);
    k2<SYM><<<nb, kThreads, 0, s>>>(G, c, W.r, v_new, W.t, W.hdr, W.part);
    count_launch(SYM ? 7 : 2, s, false);
    count_launch(3, s, true);
    k3<<<nb, kThreads, 0, s>>>(G, x, W.r, W.rh, p_new, v_new, W.t, W.hdr, W.part);
    count_launch(3, s, false);
}

// ------------------------------------------------------------------ CUDA graphs
// GC BiCGSTAB iterations (3*GC kernels) captured once and replayed: removes
// per-kernel launch latency from the loop.  A captured graph bakes in every
// array pointer, the TMA tensor maps (dims, strides), the tile / stage /
// z-chunk choice (functions of the grid shape), the grid sizes and the PDL
// attribute, so the key holds all of them: the pointers, nx, ny, nz, the
// symmetric flag and the launch options.  Equal keys therefore describe the
// same launches, whatever the allocator did in between.  Entries are evicted
// when a context that owns the workspace is destroyed (graph_cache_evict) or
// by mfx_graph_cache_clear(), and the cache is bounded (oldest out first).
constexpr int GC = 16;
constexpr size_t kMaxGraphs = 64;
struct GraphKey {
    const void *p[10];
    int nx, ny, nz, sym, pdl, dev;
    bool operator<(const GraphKey &o) const
    {
        const int a[6] = {nx, ny, nz, sym, pdl, dev}, b[6] = {o.nx, o.ny, o.nz, o.sym, o.pdl, o.dev};
        for (int q = 0; q < 6; q++)
            if (a[q] != b[q]) return a[q] < b[q];
        for (int q = 0; q < 10; q++)
            if (p[q] != o.p[q]) return p[q] < o.p[q];
        return false;
    }
};
struct GraphEntry {
    cudaGraphExec_t ex;
    unsigned long long stamp;
};
std::mutex g_graph_mu;
std::map<GraphKey, GraphEntry> g_graphs;
unsigned long long g_graph_clock = 0;

bool use_graphs() { return opt_graphs() == 1 && !prof_enabled(); }

template <bool SYM>
mfx_status get_graph(const Geo &G, const mfx_eqsys *A, const WsView &W, double *x, int nb, cudaGraphExec_t &out)
{
    GraphKey k;
    const void *ptrs[10] = {A->aP, A->aE, A->aW, A->aN, A->aS, A->aT, A->aB, A->b, x, W.hdr};
    for (int q = 0; q < 10; q++) k.p[q] = ptrs[q];
    k.nx = G.nx; k.ny = G.ny; k.nz = G.nz;
    k.sym = SYM;
    k.pdl = opt_pdl();
    k.dev = 0;
    cudaGetDevice(&k.dev);
    {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        auto it = g_graphs.find(k);
        if (it != g_graphs.end()) {
            it->second.stamp = ++g_graph_clock;
            out = it->second.ex;
            return MFX_OK;
        }
    }
    cudaStream_t cs;
    MFX_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const long long l0 = launch_count_get();
    MFX_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    mfx_status st = MFX_OK;
    for (int q = 0; q < GC && st == MFX_OK; q++) st = launch_iteration_tma<SYM>(G, A, W, x, q & 1, nb, cs);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    launch_count_set(l0);
    cudaStreamDestroy(cs);
    if (st != MFX_OK) return st;
    if (e != cudaSuccess) { set_error("graph capture: %s", cudaGetErrorString(e)); return MFX_ERR_CUDA; }
    cudaGraphExec_t ex;
    e = cudaGraphInstantiate(&ex, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) { set_error("graph instantiate: %s", cudaGetErrorString(e)); return MFX_ERR_CUDA; }
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (g_graphs.size() >= kMaxGraphs) {
        auto old = g_graphs.begin();
        for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
            if (it->second.stamp < old->second.stamp) old = it;
        cudaGraphExecDestroy(old->second.ex);   // stream-ordered: a pending launch completes first
        g_graphs.erase(old);
    }
    g_graphs[k] = GraphEntry{ex, ++g_graph_clock};
    out = ex;
    return MFX_OK;
}

struct HostScratch {
    SolverScalars *pinned = nullptr;
    ~HostScratch() {}
};
thread_local HostScratch g_host;

}  // namespace

// drop every cached graph that refers to workspace `ws` (NULL: all of them)
void graph_cache_evict(const void *ws)
{
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto it = g_graphs.begin(); it != g_graphs.end();) {
        if (!ws || it->first.p[9] == ws) {
            cudaGraphExecDestroy(it->second.ex);
            it = g_graphs.erase(it);
        } else {
            ++it;
        }
    }
}

size_t graph_cache_size()
{
    std::lock_guard<std::mutex> lk(g_graph_mu);
    return g_graphs.size();
}

bool grid_valid(const mfx_grid *g, bool scalar);

mfx_status true_resid_launch(bool sym, const Geo &G, const mfx_eqsys *A, const double *x, WsHeader *h, dd *part,
                             cudaStream_t s)
{
    const Coef c = coef_of(A);
    const int nb = reduce_grid(G.N);
    if (sym) k_true_resid<true><<<nb, kThreads, 0, s>>>(G, c, A->b, x, h, part);
    else k_true_resid<false><<<nb, kThreads, 0, s>>>(G, c, A->b, x, h, part);
    count_launch(0, s, false);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

// exit record for a host-synchronous solve: the true residual of the returned
// iterate, then one device->host copy of the solver state
static mfx_status finish_info(bool sym, const Geo &G, const mfx_eqsys *A, const double *x, const WsView &W,
                              mfx_solve_info *info, cudaStream_t s, bool have_true = false);

// MFX_KERNELS=v1 selects the simple grid-stride kernels (kept as an A/B
// reference for tests and profiling); default is the TMA z-marching path.
// Odd nx: rows are not 16-byte aligned, so TMA boxes and the paired K3 do not
// apply; the grid-stride kernels (same expressions, same bits) take over.
static bool use_tma(const Geo &G) { return opt_solver_path() != 3 && G.nx % 2 == 0; }

// TMA tensor maps and the 16-byte pair accesses need 16-byte aligned arrays
// (torch allocations are; an offset view may not be): refused up front.
static bool al16(const void *p) { return ((uintptr_t)p & 15) == 0; }
static bool sys_aligned(const mfx_eqsys *A, const double *x, const double *y)
{
    const double *q[11] = {A->aP, A->aE, A->aW, A->aN, A->aS, A->aT, A->aB, A->b, x, y, nullptr};
    for (int i = 0; i < 10; i++)
        if (q[i] && !al16(q[i])) return false;
    return true;
}

// grid-synchronous solver (path 4) in auto mode: the solver's working set
// (coefficients + b + 8 vectors) fits comfortably in the 126 MB L2 and the
// system is too large for the single-cluster kernel.  MFX_GRID_SOLVER_MB
// overrides the byte budget (0 disables the auto choice).
static bool grid_solver_fits(const Geo &G, bool sym)
{
    static long long budget = -1;
    if (budget < 0) {
        const char *e = getenv("MFX_GRID_SOLVER_MB");
        budget = (e ? atoll(e) : 0) << 20;   // off by default: measured slower than TMA at c3 (94 vs 61 us)
    }
    const long long bytes = (long long)(sym ? 3 + 1 + 8 : 7 + 1 + 8) * 8 * G.N;
    return budget > 0 && bytes <= budget && !cluster_fits(G, sym);
}

// persistent row-warp solver (path 5) in auto mode: chosen when the p'
// working set (3 coefficients + b + 8 vectors) fits 112 MiB, i.e. lives in the
// 126 MB L2 (configuration 3: 50 vs 57 us per iteration on B200, r02; at
// configuration 2 the per-launch kernels are faster, 265 vs 284 us).
// MFX_PERSIST_MB overrides the budget (0: never).
static bool persist_fits(const Geo &G)
{
    static long long budget = -1;
    if (budget < 0) {
        const char *e = getenv("MFX_PERSIST_MB");
        budget = (e ? atoll(e) : 112) << 20;
    }
    return budget > 0 && (long long)(3 + 1 + 8) * 8 * G.N <= budget && !cluster_fits(G, true);
}

// K3 over n cells (n even, 16-byte aligned arrays) with the rank's dot
// partials written to rank_part: the z-slab solver's third kernel (dist_solver.cu).
mfx_status k3_slab_launch(long long n, double *x, double *r, const double *rh, const double *p, const double *v,
                          const double *t, WsHeader *h, dd *part, dd *rank_part, cudaStream_t s)
{
    long long np = n / 2;
    int g3 = k3v_grid();
    if ((long long)g3 * kThreads > np) g3 = (int)((np + kThreads - 1) / kThreads);
    if (g3 < 1) g3 = 1;
    k3v<<<g3, kThreads, 0, s>>>(n, x, r, rh, p, v, t, h, part, 0, rank_part, 0);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

mfx_status spmv(int kind, const mfx_grid *grid, const mfx_eqsys *A, const double *x, double *y, cudaStream_t s)
{
    if (!grid_valid(grid, kind == MFX_EQ_SCALAR)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(sys_ok(kind, A), "bad eqsys for kind %d", kind);
    MFX_ARG_CHECK(x && y, "NULL x/y");
    const Geo G = make_geo(*grid);
    MFX_ARG_CHECK(!use_tma(G) || sys_aligned(A, x, y), "device arrays must be 16-byte aligned");
    const int nb = reduce_grid(G.N);
    count_launch(0, s, true);
    if (use_tma(G)) {
        const double *halo[3] = {x, nullptr, nullptr};
        mfx_status st = stencil_launch(0, kind == MFX_EQ_PP, G, halo, A, nullptr, y, nullptr, nullptr, nullptr,
                                       nullptr, 0.0, 0, s);
        count_launch(0, s, false);
        return st;
    }
    if (kind == MFX_EQ_PP) k_spmv<true><<<nb, kThreads, 0, s>>>(G, coef_of(A), x, y);
    else k_spmv<false><<<nb, kThreads, 0, s>>>(G, coef_of(A), x, y);
    count_launch(0, s, false);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

static thread_local WsHeader *g_exit = nullptr;   // pinned copy of the workspace header prefix

static mfx_status finish_info(bool sym, const Geo &G, const mfx_eqsys *A, const double *x, const WsView &W,
                              mfx_solve_info *info, cudaStream_t s, bool have_true)
{
    if (!g_exit) MFX_CUDA_TRY(cudaMallocHost(&g_exit, sizeof(WsHeader)));
    if (!have_true) {   // (the single-cluster kernel computes it itself)
        mfx_status st = true_resid_launch(sym, G, A, x, W.hdr, W.part, s);
        if (st != MFX_OK) return st;
    }
    // one copy of the header prefix: the solver state ... true_rel
    MFX_CUDA_TRY(cudaMemcpyAsync(g_exit, W.hdr, offsetof(WsHeader, true_rel) + sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
    MFX_CUDA_TRY(cudaStreamSynchronize(s));
    const SolverScalars &S = g_exit->sc;
    info->iters = S.it;
    info->status = S.status;
    info->restarts = S.restarts;
    info->rel_resid = S.bn == 0.0 ? 0.0 : S.rn / S.bn;
    info->true_rel_resid = g_exit->true_rel;
    return (mfx_status)S.status;
}

mfx_status bicgstab_solve(int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol, int maxit,
                          void *ws, size_t wsb, mfx_solve_info *info, cudaStream_t s)
{
    if (!grid_valid(grid, kind == MFX_EQ_SCALAR)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(sys_ok(kind, A) && A->b, "bad eqsys for kind %d", kind);
    MFX_ARG_CHECK(x, "NULL x");
    MFX_ARG_CHECK(tol >= 0.0 && maxit >= 0, "bad tol/maxit");
    const Geo G = make_geo(*grid);
    MFX_ARG_CHECK(!use_tma(G) || sys_aligned(A, x, nullptr), "device arrays must be 16-byte aligned");
    WsView W;
    if (!ws_view(ws, wsb, G.N, true, W)) return MFX_ERR_ARG;
    const bool sym = kind == MFX_EQ_PP;
    const Coef c = coef_of(A);
    const int nb = reduce_grid(G.N);
    if (!g_host.pinned) MFX_CUDA_TRY(cudaMallocHost(&g_host.pinned, sizeof(SolverScalars)));
    const int path = opt_solver_path();
    if (path == 2 || (path == 0 && cluster_fits(G, sym))) {
        // one launch per solve: the kernel writes the whole solver record and
        // the true residual (no memsets, no true-residual launch)
        MFX_ARG_CHECK(cluster_fits(G, sym), "system too large for the single-cluster solver");
        count_launch(0, s, true);
        mfx_status st = cluster_solve(sym, G, A, x, tol, maxit, W.hdr, s);
        count_launch(0, s, false);
        if (st != MFX_OK) return st;
        if (!info) return MFX_OK;
        return finish_info(sym, G, A, x, W, info, s, true);
    }
    MFX_CUDA_TRY(cudaMemsetAsync(&W.hdr->sc, 0, sizeof(SolverScalars), s));
    MFX_CUDA_TRY(cudaMemsetAsync(&W.hdr->ticket[0], 0, sizeof(W.hdr->ticket), s));
    MFX_CUDA_TRY(cudaMemsetAsync(&W.hdr->work[0], 0, sizeof(W.hdr->work), s));
    const bool grid_path = path == 4 || (path == 0 && grid_solver_fits(G, sym));
    const bool persist_path = sym && use_tma(G) && (path == 5 || (path == 0 && persist_fits(G)));
    count_launch(0, s, true);
    if (use_tma(G) && !grid_path) {
        const double *h0[3] = {x, nullptr, nullptr};
        mfx_status st = stencil_launch(1, sym, G, h0, A, A->b, W.r, nullptr, nullptr, W.hdr, W.part, tol, maxit, s,
                                       sweep_dir(true));
        if (st != MFX_OK) return st;
    } else if (sym) {
        k_setup<true><<<nb, kThreads, 0, s>>>(G, c, A->b, x, W.r, W.hdr, W.part, tol, maxit);
    } else {
        k_setup<false><<<nb, kThreads, 0, s>>>(G, c, A->b, x, W.r, W.hdr, W.part, tol, maxit);
    }
    count_launch(0, s, false);
    k_zero_if<<<nb, kThreads, 0, s>>>(W.hdr, x, G.N);
    count_launch(15, s, false);
    MFX_CUDA_TRY(cudaGetLastError());
    if (persist_path) {
        count_launch(6, s, true);
        mfx_status st = persist_solve_launch(G, A, x, W, maxit, s);
        count_launch(6, s, false);
        if (st != MFX_OK) return st;
        if (!info) return MFX_OK;
        return finish_info(sym, G, A, x, W, info, s);
    }
    if (grid_path) {
        count_launch(sym ? 6 : 1, s, true);
        mfx_status st = sym ? launch_grid_solver<true>(G, c, x, W, s) : launch_grid_solver<false>(G, c, x, W, s);
        count_launch(sym ? 6 : 1, s, false);
        if (st != MFX_OK) return st;
        if (!info) return MFX_OK;
        return finish_info(sym, G, A, x, W, info, s);
    }
    int launched = 0, chunk = 4;
    while (launched < maxit) {
        int cnt = maxit - launched < chunk ? maxit - launched : chunk;
        if (use_tma(G) && use_graphs() && cnt >= GC && (launched & 1) == 0) {
            cudaGraphExec_t ex;
            mfx_status st = sym ? get_graph<true>(G, A, W, x, nb, ex) : get_graph<false>(G, A, W, x, nb, ex);
            if (st != MFX_OK) return st;
            for (; cnt >= GC; cnt -= GC, launched += GC) {
                MFX_CUDA_TRY(cudaGraphLaunch(ex, s));
                launch_count_add(3 * GC);
            }
        }
        for (int q = 0; q < cnt; q++, launched++) {
            if (use_tma(G)) {
                mfx_status st = sym ? launch_iteration_tma<true>(G, A, W, x, launched & 1, nb, s)
                                    : launch_iteration_tma<false>(G, A, W, x, launched & 1, nb, s);
                if (st != MFX_OK) return st;
            } else if (sym) {
                launch_iteration<true>(G, c, W, x, launched & 1, nb, s);
            } else {
                launch_iteration<false>(G, c, W, x, launched & 1, nb, s);
            }
        }
        MFX_CUDA_TRY(cudaGetLastError());
        if (!info) continue;
        MFX_CUDA_TRY(cudaMemcpyAsync(g_host.pinned, &W.hdr->sc, sizeof(SolverScalars), cudaMemcpyDeviceToHost, s));
        MFX_CUDA_TRY(cudaStreamSynchronize(s));
        if (g_host.pinned->done) break;
        chunk = chunk * 2 > 64 ? 64 : chunk * 2;
    }
    if (!info) return MFX_OK;
    return finish_info(sym, G, A, x, W, info, s);
}

}  // namespace mfx
