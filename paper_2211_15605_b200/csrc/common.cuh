// common.cuh -- shared device helpers of libmfx (CUDA path only; the oracle
// never includes this).  Compiled with --fmad=false: no FMA contraction,
// fma() appears only where DESIGN.md §3 writes it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mfx.h"

namespace mfx {

// ------------------------------------------------------------------ errors
void set_error(const char *fmt, ...);
#define MFX_CUDA_TRY(expr)                                                               \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            ::mfx::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
            return MFX_ERR_CUDA;                                                         \
        }                                                                                \
    } while (0)
#define MFX_ARG_CHECK(cond, ...)                \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            ::mfx::set_error(__VA_ARGS__);                                               \
            return MFX_ERR_ARG;                                                          \
        }                                                                                \
    } while (0)

// ------------------------------------------------------------------ geometry
struct Geo {
    int nx, ny, nz;
    long long N;
    long long sy, sz;            // strides (elements)
    double dx, dy, dz;
    double A[3], h[3], V;        // A_x = dy*dz, A_y = dx*dz, A_z = dx*dy, V = (dx*dy)*dz
    int bc_zlo, bc_zhi;
    double w_in, phi_in, phi_out;
};

inline Geo make_geo(const mfx_grid &g)
{
    Geo G;
    G.nx = g.nx; G.ny = g.ny; G.nz = g.nz;
    G.N = (long long)g.nx * g.ny * g.nz;
    G.sy = g.nx; G.sz = (long long)g.nx * g.ny;
    G.dx = g.dx; G.dy = g.dy; G.dz = g.dz;
    G.A[0] = g.dy * g.dz; G.A[1] = g.dx * g.dz; G.A[2] = g.dx * g.dy;
    G.h[0] = g.dx; G.h[1] = g.dy; G.h[2] = g.dz;
    G.V = (g.dx * g.dy) * g.dz;
    G.bc_zlo = g.bc_zlo; G.bc_zhi = g.bc_zhi;
    G.w_in = g.w_in; G.phi_in = g.phi_in; G.phi_out = g.phi_out;
    return G;
}

// ------------------------------------------------------------------ double-double
// Correctly rounded reductions: per-thread compensated
// accumulation of exact products, then an accurate double-double tree.
struct dd { double hi, lo; };

constexpr int kMaxBlocks = 2048;
constexpr int kMaxDots = 4;
constexpr int kPartCap = kMaxBlocks * kMaxDots * 8;   // dd slots of the partials buffer (warp partials)


__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e)
{
    s = a + b;
    double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void fast_two_sum(double a, double b, double &s, double &e)
{
    s = a + b;
    e = b - (s - a);
}
// AccurateDWPlusDW (Joldes, Muller, Popescu 2017, Alg. 6): rel. error <= 3u^2.
__device__ __forceinline__ dd dd_add(dd x, dd y)
{
    double sh, sl, th, tl, vh, vl, zh, zl;
    two_sum(x.hi, y.hi, sh, sl);
    two_sum(x.lo, y.lo, th, tl);
    double c = sl + th;
    fast_two_sum(sh, c, vh, vl);
    double w = tl + vl;
    fast_two_sum(vh, w, zh, zl);
    return dd{zh, zl};
}

// Dekker's double-double add ("sloppy"): TwoSum of the heads, tails added
// plainly.  Error <= ~u^2 (|x| + |y|) per add -- the same O(u^2 * sum|partials|)
// class as the per-thread accumulation -- at half the dependent-add depth of
// dd_add.  Used where a reduction tree sits on a latency-critical path.
__device__ __forceinline__ dd dd_add_fast(dd x, dd y)
{
    double s, e;
    two_sum(x.hi, y.hi, s, e);
    const double c = (x.lo + y.lo) + e;
    dd r;
    fast_two_sum(s, c, r.hi, r.lo);
    return r;
}

// Lazy double-double add for reduction trees: TwoSum of the heads, the tails
// and the TwoSum error added plainly, no renormalisation.  The heads' chain is
// one add per tree level (the tails follow off the critical path), so a level
// costs a shuffle and two dependent adds instead of the ~9-add chain of
// dd_add_fast.  The error stays in the same O(depth u^2 sum|partials|) class:
// every head error is captured exactly, the tails (each <= u |head|) are
// summed with relative error u.
__device__ __forceinline__ dd dd_add_lazy(dd x, dd y)
{
    double s, e;
    two_sum(x.hi, y.hi, s, e);
    return dd{s, (x.lo + y.lo) + e};
}

// Per-thread accumulator: s + c with s the running TwoSum head.
struct Acc {
    double s, c;
    __device__ __forceinline__ void zero() { s = 0.0; c = 0.0; }
    __device__ __forceinline__ void prod(double a, double b)
    {
        double ph = a * b;
        double pl = fma(a, b, -ph);
        double t, e;
        two_sum(s, ph, t, e);
        s = t;
        c = c + (e + pl);
    }
    __device__ __forceinline__ void add(double x)
    {
        double t, e;
        two_sum(s, x, t, e);
        s = t;
        c = c + e;
    }
    __device__ __forceinline__ dd get() const
    {
        dd r;
        two_sum(s, c, r.hi, r.lo);
        return r;
    }
};

__device__ __forceinline__ dd shfl_dd(dd v, int off)
{
    dd r;
    r.hi = __shfl_xor_sync(0xffffffffu, v.hi, off);
    r.lo = __shfl_xor_sync(0xffffffffu, v.lo, off);
    return r;
}

// Block reduction of K double-doubles in a fixed order; result valid in
// thread 0.  `sh` needs (blockDim/32) + K dd slots.  All threads must call.
// Per value: a lane butterfly, then one warp's butterfly over the warp
// partials, with Dekker's double-double add (error ~u^2 (|x| + |y|) per add:
// the O(depth u^2 sum|terms|) class of DESIGN.md §3.1).  The K values are
// reduced one after another: interleaving the K chains inside the dot
// kernels' tails measured slower (K = 3: 9.5 vs 6.4 us for the K2 tail on
// B200, register pressure), and so was the earlier linear fold of the warp
// partials by one thread.
__device__ __forceinline__ void butterfly_dd1(dd &x)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const dd y = shfl_dd(x, off);
        x = (lane & off) ? dd_add_fast(y, x) : dd_add_fast(x, y);
    }
}

// butterfly over the lanes of a warp with Dekker's double-double add, the K
// chains interleaved level by level; every lane ends with the same bits
template <int K, int W>
__device__ __forceinline__ void butterfly_k(dd (&x)[K])
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        dd y[K];
#pragma unroll
        for (int q = 0; q < K; q++) y[q] = shfl_dd(x[q], off);
#pragma unroll
        for (int q = 0; q < K; q++) x[q] = (lane & off) ? dd_add_fast(y[q], x[q]) : dd_add_fast(x[q], y[q]);
    }
}

// the same butterfly with lazy adds (every lane ends with the same bits)
template <int K, int W>
__device__ __forceinline__ void butterfly_lazy(dd (&x)[K])
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        dd y[K];
#pragma unroll
        for (int q = 0; q < K; q++) y[q] = shfl_dd(x[q], off);
#pragma unroll
        for (int q = 0; q < K; q++) x[q] = (lane & off) ? dd_add_lazy(y[q], x[q]) : dd_add_lazy(x[q], y[q]);
    }
}

template <int K>
__device__ __forceinline__ void block_reduce_dd(dd (&v)[K], dd *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < K; q++) {
        dd x = v[q];
        butterfly_dd1(x);
        __syncthreads();   // the previous value's readers of sh are done
        if (lane == 0) sh[wid] = x;
        __syncthreads();
        if (wid == 0) {
            x = lane < nw ? sh[lane] : dd{0.0, 0.0};
            butterfly_dd1(x);
            v[q] = x;
        }
    }
    __syncthreads();
}

// Block reduction with lazy trees, the K values interleaved: a lane butterfly
// per warp, then warp 0 folds the warp partials; the result is valid in warp
// 0 (every lane of it when blockDim <= 512).  All threads must call.
// (B200: the K-serial block_reduce_dd costs ~1k cycles per value in the K2 /
// persistent tails; this is one pass for all K.)
template <int K>
__device__ __forceinline__ void block_reduce_lazy(dd (&v)[K])
{
    __shared__ dd s_w[3][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    butterfly_lazy<K, 32>(v);
    __syncthreads();   // readers of the previous call's slots are done
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < K; q++) s_w[q][wid] = v[q];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < K; q++) v[q] = lane < nw ? s_w[q][lane] : dd{0.0, 0.0};
        if (nw <= 16) butterfly_lazy<K, 16>(v);
        else butterfly_lazy<K, 32>(v);
    }
}

// every thread folds its share of n published partials part[b * stride + q]
// (thread-strided: one L2 round trip for n <= blockDim), then the block tree;
// the result is valid in warp 0.  All threads must call.  (A one-warp fold
// is slower: ~10 L2 round trips per lane at n ~ 300.)
template <int K>
__device__ __forceinline__ void block_fold_partials(const dd *part, unsigned n, int stride, dd (&f)[K])
{
#pragma unroll
    for (int q = 0; q < K; q++) f[q] = dd{0.0, 0.0};
    for (unsigned b = threadIdx.x; b < n; b += blockDim.x) {
#pragma unroll
        for (int q = 0; q < K; q++) {
            dd x;
            x.hi = __ldcg(&part[(size_t)b * stride + q].hi);
            x.lo = __ldcg(&part[(size_t)b * stride + q].lo);
            f[q] = dd_add_lazy(f[q], x);
        }
    }
    block_reduce_lazy<K>(f);
}

// Deterministic grid reduction: each block writes K partials to part[blk*K+q];
// the last block to finish (ticket) folds them with all its threads and returns
// true in every thread of that block, with out[q] valid in thread 0.
// (Publishing warp partials instead, to keep one block reduction off the
// tail, measured slower: the last block's fold over 9x more partials costs more.)
template <int K>
__device__ __forceinline__ bool grid_reduce_dd(dd (&v)[K], dd *part, unsigned int *ticket, dd *sh,
                                               dd (&out)[K])
{
    (void)sh;
    block_reduce_lazy<K>(v);
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; q++) part[(size_t)blockIdx.x * K + q] = v[q];
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    dd f[K];
    block_fold_partials<K>(part, gridDim.x, K, f);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; q++) out[q] = f[q];
        *ticket = 0u;   // reset for the next launch (stream-ordered)
    }
    return true;
}

__device__ __forceinline__ double dd_round(dd x) { return (x.hi + x.lo) + 0.0; }

// ------------------------------------------------------------------ workspace
struct SolverScalars {
    double rho, rho_prev, alpha, omega;
    double sigma, ss, ts, tt, rr;
    double bn, rn, rhn, tol;
    int it, maxit, status, done;
    int restarted, restarts, restart_mode, skip;
    int half, zero_x, pad0, pad1;
};

struct WsHeader {
    SolverScalars sc;
    unsigned long long bad_nonfinite;   // first offending cell (ULLONG_MAX = none)
    unsigned long long bad_zerodiag;
    unsigned int ticket[4];
    double resid[4];
    unsigned long long bad_parcel;      // first parcel outside the domain (ULLONG_MAX = none)
    double true_rel;                    // ||b - A x|| / ||b|| of the last solve's exit iterate (0 if b = 0)
    unsigned int work[2];               // dynamic unit counters of the z-marching kernels (reset by their last CTA)
    double pad[3];
    // chained tails (bicgstab.cu, path 1): K1 and K2 publish block partials
    // without a last-CTA fold; the next kernel's CTAs fold them in their
    // prologue.  sc2 = the state after K1's tail (written by K2, read by K3);
    // npart = how many partials K1 / K2 published.
    SolverScalars sc2;
    unsigned int npart[2];
};

// offsets of the chained partials in the workspace's partials buffer
constexpr int kPartK1 = 0, kPartK2 = 8192;

// every thread gets the same fold of n published partials part[b * stride + q]
// (thread-strided, then the block tree of block_reduce_dd): the prologue of a
// chained kernel.  `bc` is K dd of shared memory.
template <int K>
__device__ __forceinline__ void fold_published(const dd *part, unsigned n, int stride, dd *sh, dd *bc,
                                               double (&out)[K])
{
    dd f[K];
#pragma unroll
    for (int q = 0; q < K; q++) f[q] = dd{0.0, 0.0};
    for (unsigned b = threadIdx.x; b < n; b += blockDim.x) {
#pragma unroll
        for (int q = 0; q < K; q++) {
            dd x;
            x.hi = __ldcg(&part[(size_t)b * stride + q].hi);
            x.lo = __ldcg(&part[(size_t)b * stride + q].lo);
            f[q] = dd_add(f[q], x);
        }
    }
    block_reduce_dd<K>(f, sh);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < K; q++) bc[q] = f[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < K; q++) out[q] = dd_round(bc[q]);
}

__device__ __forceinline__ SolverScalars sc_ldcg(const SolverScalars *S)
{
    SolverScalars L;
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(S);
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(&L);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(SolverScalars) / 8); q++) dst[q] = __ldcg(src + q);
    return L;
}

// publish this block's K partials (no ticket): the chained kernels' epilogue
template <int K>
__device__ __forceinline__ void publish_partials(dd (&v)[K], dd *part, unsigned *npart, dd *sh)
{
    block_reduce_dd<K>(v, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; q++) part[(size_t)blockIdx.x * K + q] = v[q];
        if (blockIdx.x == 0) *npart = gridDim.x;
    }
}


struct WsView {
    WsHeader *hdr;
    dd *part;                 // kPartCap
    double *r, *rh, *p[2], *v[2], *t;
};

size_t ws_header_bytes();
size_t ws_total_bytes(long long N);
bool ws_view(void *ws, size_t bytes, long long N, bool need_vectors, WsView &out);

// launch accounting / profiling
void count_launch(int id, cudaStream_t s, bool start);
bool prof_enabled();
int opt_solver_path();   // 0 auto, 1 TMA, 2 cluster, 3 v1
int opt_graphs();
int opt_pdl();
int opt_asm_tma();
mfx_status assemble_mom_tma(int kind, const Geo &G, const mfx_params *pr, const mfx_state *st, mfx_eqsys *out,
                            double *resid2, WsHeader *hdr, dd *part, cudaStream_t s);
bool cluster_fits(const Geo &G, bool sym);
mfx_status cluster_solve(bool sym, const Geo &G, const mfx_eqsys *A, double *x, double tol, int maxit,
                         WsHeader *h, cudaStream_t s);
long long launch_count_get();
size_t pic_sort_scratch_bytes(long long N, long long m);
mfx_status pic_sort(const mfx_grid *grid, const mfx_pic_params *pp, const mfx_parcels *in, double *const out[7],
                    unsigned int *orig_out, unsigned int *start_out, void *scratch, size_t scratch_bytes,
                    cudaStream_t s);
mfx_status pic_deposit_binned(int drag, const mfx_grid *grid, const mfx_params *pr, const mfx_pic_params *pp,
                              const mfx_parcels *pc, const unsigned int *orig, const unsigned int *start,
                              const double *eps_in, const double *u, const double *v, const double *w,
                              double *const outs[4], double *Kout, double *vals, void *ws, size_t wsb,
                              cudaStream_t s);
mfx_status pic_deposit_eps(const mfx_grid *grid, const mfx_pic_params *pp, const mfx_parcels *pc, double *eps,
                           void *ws, size_t wsb, cudaStream_t s);
mfx_status pic_drag(const mfx_grid *grid, const mfx_params *pr, const mfx_pic_params *pp, const mfx_parcels *pc,
                    const double *eps, const double *u, const double *v, const double *w, double *beta,
                    double *sbu, double *sbv, double *sbw, double *Kout, void *ws, size_t wsb, cudaStream_t s);
void launch_count_set(long long v);
void launch_count_add(long long v);
int reduce_grid(long long N);
mfx_status true_resid_launch(bool sym, const Geo &G, const mfx_eqsys *A, const double *x, WsHeader *h, dd *part,
                             cudaStream_t s);

}  // namespace mfx
