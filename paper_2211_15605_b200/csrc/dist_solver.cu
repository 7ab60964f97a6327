// dist_solver.cu -- domain-decomposed (z-slab) BiCGSTAB across the ranks of a
// context: the comparator of BASELINE.json configuration 5 ("domain-
// decomposed allreduce-dot baseline"; the MPI strategy of PAPER.md:87 and
// Fig. 2a) and the building block of a multi-GPU pressure solve.
//
// Rank r owns global planes [k0_r, k1_r), k0_r = nz*r/R.  Every iteration
// exchanges one halo plane per stencil apply with the z-neighbours and
// all-gathers the double-double dot partials of every rank, which each rank
// folds in rank order -> the scalars are correctly rounded
// and identical on every rank, and the iterates equal the single-GPU solve
// bitwise.  Kernels are plain grid-stride slab kernels; the per-iteration
// sequence is
//   p-update | halo(p) | v = A p, <r^,v> | allgather | fold: alpha
//   s-update | halo(s) | t = A s, <t,s>,<t,t>,<s,s> | allgather | fold: omega
//   x, r update, <r^,r>, <r,r> | allgather | fold: rho, stop test
// The scalar state machine of §3.6 runs in the single-block fold kernels.
#include <cstring>

#include "common.cuh"
#include "bicg_state.cuh"

namespace mfx {

namespace {

constexpr int kT = 256;

struct DSlab {
    int nx, ny, nz, k0, npl;
    long long plane, nloc;
};

struct DCoef {
    const double *aP, *aE, *aW, *aN, *aS, *aT, *aB;
};

// y = A X at local cell n of the slab (DESIGN.md §3.2 order); planes k0-1 and
// k1 come from the halo copies hb / ha, the B coefficient of the first plane
// (symmetric storage) from czb.
template <bool SYM>
__device__ __forceinline__ double apply_slab(const DSlab &D, const DCoef &c, const double *czb, const double *X,
                                             const double *hb, const double *ha, long long n)
{
    const int kl = (int)(n / D.plane);
    const long long o = n - (long long)kl * D.plane;
    const int iy = (int)(o / D.nx), ix = (int)(o - (long long)iy * D.nx);
    const int k = D.k0 + kl;
    const double xc = X[n];
    const double xW = ix > 0 ? X[n - 1] : 0.0;
    const double xE = ix < D.nx - 1 ? X[n + 1] : 0.0;
    const double xS = iy > 0 ? X[n - D.nx] : 0.0;
    const double xN = iy < D.ny - 1 ? X[n + D.nx] : 0.0;
    double xB = 0.0, xT = 0.0;
    if (k > 0) xB = kl > 0 ? X[n - D.plane] : hb[o];
    if (k < D.nz - 1) xT = kl < D.npl - 1 ? X[n + D.plane] : ha[o];
    double aP, aW, aE, aS, aN, aB, aT;
    if (SYM) {
        aW = ix > 0 ? c.aE[n - 1] : 0.0;
        aE = c.aE[n];
        aS = iy > 0 ? c.aN[n - D.nx] : 0.0;
        aN = c.aN[n];
        aB = 0.0;
        if (k > 0) aB = kl > 0 ? c.aT[n - D.plane] : czb[o];
        aT = c.aT[n];
        aP = ((((aW + aE) + aS) + aN) + aB) + aT;   // p' diagonal = row sum
    } else {
        aP = c.aP[n];
        aW = c.aW[n]; aE = c.aE[n]; aS = c.aS[n]; aN = c.aN[n]; aB = c.aB[n]; aT = c.aT[n];
    }
    double y = aP * xc;
    y = fma(-aW, xW, y);
    y = fma(-aE, xE, y);
    y = fma(-aS, xS, y);
    y = fma(-aN, xN, y);
    y = fma(-aB, xB, y);
    y = fma(-aT, xT, y);
    return y;
}

#define SLAB_LOOP(n) for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < D.nloc; n += (long long)gridDim.x * blockDim.x)

// rank-local double-double partials of K dots -> rank_part[K] (not rounded)
template <int K>
__device__ __forceinline__ void rank_partials(Acc (&acc)[K], dd *part, unsigned int *ticket, dd *rank_part)
{
    __shared__ dd sh[(kT / 32) * K];
    dd v[K], out[K];
#pragma unroll
    for (int q = 0; q < K; q++) v[q] = acc[q].get();
    if (grid_reduce_dd<K>(v, part, ticket, sh, out) && threadIdx.x == 0)
        for (int q = 0; q < K; q++) rank_part[q] = out[q];
}

// fold the R rank partials of value q in rank order (single thread)
__device__ __forceinline__ double fold_ranks(const dd *all, int R, int K, int q)
{
    dd acc = dd{0.0, 0.0};
    for (int r = 0; r < R; r++) acc = dd_add(acc, all[r * K + q]);
    return dd_round(acc);
}

// ------------------------------------------------------------------ kernels
template <bool SYM>
__global__ void __launch_bounds__(kT) dk_setup(DSlab D, DCoef c, const double *czb, const double *b, const double *x,
                                               const double *hb, const double *ha, double *r, WsHeader *h, dd *part,
                                               dd *rank_part)
{
    Acc acc[2];
    acc[0].zero(); acc[1].zero();
    SLAB_LOOP(n) {
        const double y = apply_slab<SYM>(D, c, czb, x, hb, ha, n);
        const double bv = b[n];
        const double rv = bv - y;
        r[n] = rv;
        acc[0].prod(bv, bv);
        acc[1].prod(rv, rv);
    }
    rank_partials<2>(acc, part, &h->ticket[1], rank_part);
}

__global__ void dk_fold_setup(WsHeader *h, const dd *all, int R, double tol, int maxit)
{
    if (threadIdx.x != 0) return;
    bicg_setup(h->sc, fold_ranks(all, R, 2, 0), fold_ranks(all, R, 2, 1), tol, maxit);
}

__global__ void dk_zero_if(DSlab D, const WsHeader *h, double *x)
{
    if (!h->sc.zero_x) return;
    SLAB_LOOP(n) x[n] = 0.0;
}

__global__ void __launch_bounds__(kT) dk_p(DSlab D, const double *r, double *rh, double *p, const double *v,
                                           WsHeader *h)
{
    SolverScalars &S = h->sc;
    if (S.done) return;
    const K1Pro d = bicg_k1_prologue(S);
    if (d.breakdown) {
        if (blockIdx.x == 0 && threadIdx.x == 0) bicg_breakdown(S);
        return;
    }
    SLAB_LOOP(n) {
        if (d.rst) {
            p[n] = fma(d.beta, fma(-d.omega, 0.0, 0.0), r[n]);
            rh[n] = r[n];
        } else {
            p[n] = fma(d.beta, fma(-d.omega, v[n], p[n]), r[n]);
        }
    }
}

template <bool SYM>
__global__ void __launch_bounds__(kT) dk_apply_v(DSlab D, DCoef c, const double *czb, const double *p,
                                                 const double *hb, const double *ha, const double *rh, double *v,
                                                 WsHeader *h, dd *part, dd *rank_part)
{
    if (h->sc.done) return;
    Acc acc[1];
    acc[0].zero();
    SLAB_LOOP(n) {
        const double vv = apply_slab<SYM>(D, c, czb, p, hb, ha, n);
        v[n] = vv;
        acc[0].prod(rh[n], vv);
    }
    rank_partials<1>(acc, part, &h->ticket[1], rank_part);
}

__global__ void dk_fold_sigma(WsHeader *h, const dd *all, int R)
{
    if (threadIdx.x != 0) return;
    SolverScalars &S = h->sc;
    if (S.done) return;
    const K1Pro d = bicg_k1_prologue(S);
    bicg_k1_tail(S, d, fold_ranks(all, R, 1, 0));
}

__global__ void __launch_bounds__(kT) dk_s(DSlab D, const double *r, const double *v, double *s, const WsHeader *h)
{
    const SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    const double alpha = S.alpha;
    SLAB_LOOP(n) s[n] = fma(-alpha, v[n], r[n]);
}

template <bool SYM>
__global__ void __launch_bounds__(kT) dk_apply_t(DSlab D, DCoef c, const double *czb, const double *s,
                                                 const double *hb, const double *ha, double *t, WsHeader *h,
                                                 dd *part, dd *rank_part)
{
    const SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    Acc acc[3];
    acc[0].zero(); acc[1].zero(); acc[2].zero();
    SLAB_LOOP(n) {
        const double tv = apply_slab<SYM>(D, c, czb, s, hb, ha, n);
        const double sv = s[n];
        t[n] = tv;
        acc[0].prod(tv, sv);
        acc[1].prod(tv, tv);
        acc[2].prod(sv, sv);
    }
    rank_partials<3>(acc, part, &h->ticket[1], rank_part);
}

__global__ void dk_fold_t(WsHeader *h, const dd *all, int R)
{
    if (threadIdx.x != 0) return;
    SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    bicg_k2_tail(S, fold_ranks(all, R, 3, 0), fold_ranks(all, R, 3, 1), fold_ranks(all, R, 3, 2));
}

__global__ void __launch_bounds__(kT) dk_k3(DSlab D, double *x, double *r, const double *rh, const double *p,
                                            const double *s, const double *t, WsHeader *h, dd *part, dd *rank_part)
{
    const SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    const double alpha = S.alpha, omega = S.omega;
    const bool half = S.half != 0;
    Acc acc[2];
    acc[0].zero(); acc[1].zero();
    SLAB_LOOP(n) {
        const double sv = s[n];
        double xn, rn;
        if (half) {
            xn = fma(alpha, p[n], x[n]);
            rn = sv;
        } else {
            xn = fma(omega, sv, fma(alpha, p[n], x[n]));
            rn = fma(-omega, t[n], sv);
        }
        x[n] = xn;
        r[n] = rn;
        acc[0].prod(rh[n], rn);
        acc[1].prod(rn, rn);
    }
    rank_partials<2>(acc, part, &h->ticket[1], rank_part);
}

__global__ void dk_fold_r(WsHeader *h, const dd *all, int R)
{
    if (threadIdx.x != 0) return;
    SolverScalars &S = h->sc;
    if (S.done || S.skip) return;
    const bool half = S.half != 0;
    bicg_k3_tail(S, half, half ? 0.0 : fold_ranks(all, R, 2, 0), half ? 0.0 : fold_ranks(all, R, 2, 1));
}

int dgrid(long long n)
{
    long long b = (n + kT - 1) / kT;
    if (b > 148 * 4) b = 148 * 4;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

void dist_slab(int nz, int rank, int nranks, int *k0, int *k1)
{
    *k0 = (int)((long long)nz * rank / nranks);
    *k1 = (int)((long long)nz * (rank + 1) / nranks);
}

// Transport hooks implemented in simple.cu (NCCL or the in-process group).
mfx_status ctx_halo_exchange(mfx_ctx *c, const double *slab, int npl, long long plane, double *hb, double *ha,
                             cudaStream_t s);
mfx_status ctx_allgather_dd(mfx_ctx *c, const dd *mine, int K, dd *all, cudaStream_t s);
int ctx_rank(const mfx_ctx *c);
int ctx_nranks(const mfx_ctx *c);
bool ctx_capturable(const mfx_ctx *c);
void *ctx_dist_scratch(mfx_ctx *c, size_t bytes);

mfx_status stencil_launch(int mode, bool sym, const Geo &G, const double *const halo[3], const mfx_eqsys *A,
                          const double *extra, double *o0, double *o1, double *o2, WsHeader *h, dd *part,
                          double tol, int maxit, cudaStream_t s, int reverse = 0, int kbeg = 0, int kend = 0,
                          int ghost_store = 0, dd *rank_part = nullptr, int chain = 0);
mfx_status k3_slab_launch(long long n, double *x, double *r, const double *rh, const double *p, const double *v,
                          const double *t, WsHeader *h, dd *part, dd *rank_part, cudaStream_t s);

// p' (symmetric, even nx) slab solve on the fused TMA row-warp kernels of the
// single-GPU path (stencil_tma.cu, slab mode).  Every vector lives in an
// EXTENDED slab of npl + 2 planes: local plane 0 = global k0 - 1 and plane
// npl + 1 = global k1 hold the neighbours' ghost copies (zero beyond the
// domain ends, which is the boundary rule of §3.2).  K1 recomputes p on the
// ghost planes from the ghost r, p_old, v_old (and stores it, so p_old's
// ghosts stay current without an exchange); K2 recomputes s there from the
// ghost r, v.  So per iteration only v (after K1) and r (after K3) cross to
// the neighbours, next to the three all-gathers of dot partials:
//   K1 | allgather <r^,v>, halo(v) | fold: alpha
//   K2 | allgather <t,s>,<t,t>,<s,s> | fold: omega
//   K3 | allgather <r^,r>,<r,r>, halo(r) | fold: rho, stop test
static mfx_status dist_solve_tma(mfx_ctx *ctx, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol,
                                 int maxit, mfx_solve_info *info, cudaStream_t s)
{
    const int R = ctx_nranks(ctx), rank = ctx_rank(ctx);
    int k0, k1;
    dist_slab(grid->nz, rank, R, &k0, &k1);
    const int npl = k1 - k0, ne = npl + 2;
    const long long plane = (long long)grid->nx * grid->ny;
    DSlab D;
    D.nx = grid->nx; D.ny = grid->ny; D.nz = grid->nz; D.k0 = k0; D.npl = npl;
    D.plane = plane;
    D.nloc = plane * npl;
    auto r256 = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t hdr = r256(sizeof(WsHeader)), partb = r256(sizeof(dd) * kPartCap);
    const size_t rpb = r256(sizeof(dd) * 4), apb = r256(sizeof(dd) * 4 * 64);
    const size_t eb = r256(sizeof(double) * (size_t)(plane * ne));
    constexpr int NV = 12;   // r rh p0 p1 v0 v1 t | x b | cx cy cz
    const size_t total = hdr + partb + rpb + apb + NV * eb;
    char *w = (char *)ctx_dist_scratch(ctx, total);
    if (!w) return MFX_ERR_CUDA;
    WsHeader *h = (WsHeader *)w;
    dd *part = (dd *)(w + hdr);
    dd *rank_part = (dd *)(w + hdr + partb);
    // one rank: the fold kernels read the rank's own partials (no gather copy)
    dd *all = R == 1 ? rank_part : (dd *)(w + hdr + partb + rpb);
    char *vb = w + hdr + partb + rpb + apb;
    auto E = [&](int q) { return (double *)(vb + (size_t)q * eb); };
    double *r = E(0), *rh = E(1), *P[2] = {E(2), E(3)}, *V[2] = {E(4), E(5)}, *t = E(6);
    double *xe = E(7), *be = E(8), *cxe = E(9), *cye = E(10), *cze = E(11);
    const size_t slab_b = sizeof(double) * (size_t)D.nloc;
    MFX_CUDA_TRY(cudaMemsetAsync(w, 0, hdr, s));
    MFX_CUDA_TRY(cudaMemsetAsync(vb, 0, NV * eb, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(xe + plane, x, slab_b, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(be + plane, A->b, slab_b, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(cxe + plane, A->aE, slab_b, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(cye + plane, A->aN, slab_b, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(cze + plane, A->aT, slab_b, cudaMemcpyDeviceToDevice, s));
    mfx_grid ge = *grid;
    ge.nz = ne;
    const Geo G = make_geo(ge);
    mfx_eqsys Ae;
    memset(&Ae, 0, sizeof(Ae));
    Ae.aE = cxe; Ae.aN = cye; Ae.aT = cze; Ae.b = be;
    mfx_status st;
#define XCHG(vecp) do { if ((st = ctx_halo_exchange(ctx, (vecp) + plane, npl, plane, (vecp), (vecp) + (size_t)(npl + 1) * plane, s)) != MFX_OK) return st; } while (0)
#define GATHER(K) do { if (R > 1 && (st = ctx_allgather_dd(ctx, rank_part, K, all, s)) != MFX_OK) return st; } while (0)
#define TRY(expr) do { if ((st = (expr)) != MFX_OK) return st; } while (0)
    XCHG(cze);   // c_z of plane k0 - 1: the B coefficient of the first own plane
    XCHG(xe);
    {
        const double *h0[3] = {xe, nullptr, nullptr};
        TRY(stencil_launch(1, true, G, h0, &Ae, be, r, nullptr, nullptr, h, part, tol, maxit, s, 0, 1, npl + 1, 0,
                           rank_part));
    }
    GATHER(2);
    dk_fold_setup<<<1, 32, 0, s>>>(h, all, R, tol, maxit);
    dk_zero_if<<<dgrid(D.nloc), kT, 0, s>>>(D, h, xe + plane);
    MFX_CUDA_TRY(cudaGetLastError());
    XCHG(r);
    launch_count_add(3);
    static thread_local SolverScalars *pin = nullptr;
    if (!pin) MFX_CUDA_TRY(cudaMallocHost(&pin, sizeof(SolverScalars)));
    auto iteration = [&](int par, cudaStream_t st_) -> mfx_status {
        double *p_old = P[par], *p_new = P[par ^ 1], *v_old = V[par], *v_new = V[par ^ 1];
        const double *h1[3] = {r, p_old, v_old};
        cudaStream_t s = st_;
        TRY(stencil_launch(2, true, G, h1, &Ae, rh, p_new, v_new, rh, h, part, 0.0, 0, s, 0, 1, npl + 1, 1,
                           rank_part));
        GATHER(1);
        XCHG(v_new);
        dk_fold_sigma<<<1, 32, 0, s>>>(h, all, R);
        const double *h2[3] = {r, v_new, nullptr};
        TRY(stencil_launch(3, true, G, h2, &Ae, nullptr, t, nullptr, nullptr, h, part, 0.0, 0, s, 0, 1, npl + 1, 0,
                           rank_part));
        GATHER(3);
        dk_fold_t<<<1, 32, 0, s>>>(h, all, R);
        TRY(k3_slab_launch(D.nloc, xe + plane, r + plane, rh + plane, p_new + plane, v_new + plane, t + plane, h,
                           part, rank_part, s));
        GATHER(2);
        XCHG(r);
        dk_fold_r<<<1, 32, 0, s>>>(h, all, R);
        MFX_CUDA_TRY(cudaGetLastError());
        return MFX_OK;
    };
    // NCCL (or a single rank): the iteration sequence is captured once per solve
    // into a CUDA graph of DG iterations and replayed (the in-process transport
    // synchronises host threads, so it launches directly)
    constexpr int DG = 16;
    cudaGraphExec_t gex = nullptr;
    if (ctx_capturable(ctx) && maxit >= DG) {
        cudaStream_t cs;
        MFX_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        MFX_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        mfx_status cst = MFX_OK;
        for (int q = 0; q < DG && cst == MFX_OK; q++) cst = iteration(q & 1, cs);
        cudaGraph_t gr = nullptr;
        cudaError_t e = cudaStreamEndCapture(cs, &gr);
        cudaStreamDestroy(cs);
        if (cst != MFX_OK) { if (gr) cudaGraphDestroy(gr); return cst; }
        if (e != cudaSuccess) { set_error("dist graph capture: %s", cudaGetErrorString(e)); return MFX_ERR_CUDA; }
        e = cudaGraphInstantiate(&gex, gr, 0);
        cudaGraphDestroy(gr);
        if (e != cudaSuccess) { set_error("dist graph instantiate: %s", cudaGetErrorString(e)); return MFX_ERR_CUDA; }
    }
    int launched = 0, chunk = 4;
    mfx_status lst = MFX_OK;
    while (launched < maxit && lst == MFX_OK) {
        int cnt = maxit - launched < chunk ? maxit - launched : chunk;
        if (gex && (launched & 1) == 0)
            for (; cnt >= DG; cnt -= DG, launched += DG) {
                if (cudaGraphLaunch(gex, s) != cudaSuccess) { lst = MFX_ERR_CUDA; break; }
                launch_count_add(6 * DG);
            }
        for (int q = 0; q < cnt && lst == MFX_OK; q++, launched++) {
            lst = iteration(launched & 1, s);
            launch_count_add(6);
        }
        if (lst != MFX_OK) break;
        MFX_CUDA_TRY(cudaMemcpyAsync(pin, &h->sc, sizeof(SolverScalars), cudaMemcpyDeviceToHost, s));
        MFX_CUDA_TRY(cudaStreamSynchronize(s));
        if (pin->done) break;
        chunk = chunk * 2 > 64 ? 64 : chunk * 2;
    }
    if (gex) cudaGraphExecDestroy(gex);
    if (lst != MFX_OK) {
        if (lst == MFX_ERR_CUDA) set_error("dist solve: %s", cudaGetErrorString(cudaGetLastError()));
        return lst;
    }
#undef XCHG
#undef GATHER
#undef TRY
    MFX_CUDA_TRY(cudaMemcpyAsync(x, xe + plane, slab_b, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(pin, &h->sc, sizeof(SolverScalars), cudaMemcpyDeviceToHost, s));
    MFX_CUDA_TRY(cudaStreamSynchronize(s));
    if (info) {
        info->iters = pin->it;
        info->status = pin->status;
        info->restarts = pin->restarts;
        info->rel_resid = pin->bn == 0.0 ? 0.0 : pin->rn / pin->bn;
        info->true_rel_resid = -1.0;
    }
    return (mfx_status)pin->status;
}

mfx_status dist_solve(mfx_ctx *ctx, int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol,
                      int maxit, mfx_solve_info *info, cudaStream_t s)
{
    if (kind == MFX_EQ_PP && grid->nx % 2 == 0 && opt_solver_path() != 3 && A->aE && A->aN && A->aT && A->b &&
        !A->aW && !A->aS && !A->aB && grid->nz >= ctx_nranks(ctx) && !((uintptr_t)x & 15))
        return dist_solve_tma(ctx, grid, A, x, tol, maxit, info, s);
    MFX_ARG_CHECK(ctx && grid && A && x, "NULL argument");
    const bool sym = kind == MFX_EQ_PP;
    MFX_ARG_CHECK(A->aE && A->aN && A->aT && A->b && (sym ? (!A->aW && !A->aS && !A->aB)
                                                          : (A->aP && A->aW && A->aS && A->aB)),
                  "bad slab eqsys for kind %d", kind);
    const int R = ctx_nranks(ctx), rank = ctx_rank(ctx);
    MFX_ARG_CHECK(grid->nz >= R, "dist solve: nz (%d) must be >= number of ranks (%d)", grid->nz, R);
    int k0, k1;
    dist_slab(grid->nz, rank, R, &k0, &k1);
    DSlab D;
    D.nx = grid->nx; D.ny = grid->ny; D.nz = grid->nz; D.k0 = k0; D.npl = k1 - k0;
    D.plane = (long long)grid->nx * grid->ny;
    D.nloc = D.plane * D.npl;
    // scratch: header | block partials | rank part | all parts | r rh p v s t | hb ha czb
    auto r256 = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t hdr = r256(sizeof(WsHeader)), partb = r256(sizeof(dd) * kPartCap);
    const size_t rpb = r256(sizeof(dd) * 4), apb = r256(sizeof(dd) * 4 * 64);
    const size_t vb = r256(sizeof(double) * D.nloc), pb = r256(sizeof(double) * D.plane);
    const size_t total = hdr + partb + rpb + apb + 6 * vb + 3 * pb;
    char *w = (char *)ctx_dist_scratch(ctx, total);
    if (!w) return MFX_ERR_CUDA;
    WsHeader *h = (WsHeader *)w;
    dd *part = (dd *)(w + hdr);
    dd *rank_part = (dd *)(w + hdr + partb);
    dd *all = (dd *)(w + hdr + partb + rpb);
    double *vec = (double *)(w + hdr + partb + rpb + apb);
    double *r = vec, *rh = (double *)((char *)vec + vb), *p = (double *)((char *)vec + 2 * vb);
    double *v = (double *)((char *)vec + 3 * vb), *sv = (double *)((char *)vec + 4 * vb);
    double *t = (double *)((char *)vec + 5 * vb);
    double *hb = (double *)((char *)vec + 6 * vb), *ha = (double *)((char *)hb + pb), *czb = (double *)((char *)hb + 2 * pb);
    MFX_CUDA_TRY(cudaMemsetAsync(w, 0, hdr, s));
    MFX_CUDA_TRY(cudaMemsetAsync(czb, 0, pb, s));
    MFX_CUDA_TRY(cudaMemsetAsync(hb, 0, 2 * pb, s));
    DCoef c = {A->aP, A->aE, A->aW, A->aN, A->aS, A->aT, A->aB};
    const int nb = dgrid(D.nloc);
    mfx_status st;
#define XCHG(vecp) do { if ((st = ctx_halo_exchange(ctx, vecp, D.npl, D.plane, hb, ha, s)) != MFX_OK) return st; } while (0)
#define GATHER(K) do { if ((st = ctx_allgather_dd(ctx, rank_part, K, all, s)) != MFX_OK) return st; } while (0)
    if (sym) {   // cz of plane k0-1 (B coefficient of the first own plane)
        XCHG(A->aT);
        MFX_CUDA_TRY(cudaMemcpyAsync(czb, hb, pb, cudaMemcpyDeviceToDevice, s));
    }
    XCHG(x);
    if (sym) dk_setup<true><<<nb, kT, 0, s>>>(D, c, czb, A->b, x, hb, ha, r, h, part, rank_part);
    else dk_setup<false><<<nb, kT, 0, s>>>(D, c, czb, A->b, x, hb, ha, r, h, part, rank_part);
    GATHER(2);
    dk_fold_setup<<<1, 32, 0, s>>>(h, all, R, tol, maxit);
    dk_zero_if<<<nb, kT, 0, s>>>(D, h, x);
    MFX_CUDA_TRY(cudaGetLastError());
    static thread_local SolverScalars *pin = nullptr;
    if (!pin) MFX_CUDA_TRY(cudaMallocHost(&pin, sizeof(SolverScalars)));
    int launched = 0, chunk = 4;
    while (launched < maxit) {
        const int cnt = maxit - launched < chunk ? maxit - launched : chunk;
        for (int q = 0; q < cnt; q++, launched++) {
            dk_p<<<nb, kT, 0, s>>>(D, r, rh, p, v, h);
            XCHG(p);
            if (sym) dk_apply_v<true><<<nb, kT, 0, s>>>(D, c, czb, p, hb, ha, rh, v, h, part, rank_part);
            else dk_apply_v<false><<<nb, kT, 0, s>>>(D, c, czb, p, hb, ha, rh, v, h, part, rank_part);
            GATHER(1);
            dk_fold_sigma<<<1, 32, 0, s>>>(h, all, R);
            dk_s<<<nb, kT, 0, s>>>(D, r, v, sv, h);
            XCHG(sv);
            if (sym) dk_apply_t<true><<<nb, kT, 0, s>>>(D, c, czb, sv, hb, ha, t, h, part, rank_part);
            else dk_apply_t<false><<<nb, kT, 0, s>>>(D, c, czb, sv, hb, ha, t, h, part, rank_part);
            GATHER(3);
            dk_fold_t<<<1, 32, 0, s>>>(h, all, R);
            dk_k3<<<nb, kT, 0, s>>>(D, x, r, rh, p, sv, t, h, part, rank_part);
            GATHER(2);
            dk_fold_r<<<1, 32, 0, s>>>(h, all, R);
            launch_count_add(13);
        }
        MFX_CUDA_TRY(cudaGetLastError());
        MFX_CUDA_TRY(cudaMemcpyAsync(pin, &h->sc, sizeof(SolverScalars), cudaMemcpyDeviceToHost, s));
        MFX_CUDA_TRY(cudaStreamSynchronize(s));
        if (pin->done) break;
        chunk = chunk * 2 > 64 ? 64 : chunk * 2;
    }
#undef XCHG
#undef GATHER
    MFX_CUDA_TRY(cudaMemcpyAsync(pin, &h->sc, sizeof(SolverScalars), cudaMemcpyDeviceToHost, s));
    MFX_CUDA_TRY(cudaStreamSynchronize(s));
    if (info) {
        info->iters = pin->it;
        info->status = pin->status;
        info->restarts = pin->restarts;
        info->rel_resid = pin->bn == 0.0 ? 0.0 : pin->rn / pin->bn;
        info->true_rel_resid = -1.0;   // not computed per slab (mfx_simple_iter computes it on P0)
    }
    return (mfx_status)pin->status;
}

}  // namespace mfx
