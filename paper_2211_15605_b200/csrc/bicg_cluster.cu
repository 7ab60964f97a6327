// bicg_cluster.cu -- a-6 for small systems (BASELINE.json configuration 1,
// 16x16x32): the whole unpreconditioned BiCGSTAB solve in
// ONE launch of one thread-block cluster of CL CTAs (16 SMs, the
// non-portable maximum on B200; 8 where a 16-CTA cluster cannot be placed).
//
// The grid is split into CL z-slabs; CTA `rank` keeps its slab of every
// coefficient and vector in shared memory for the whole solve.  Nothing in the
// iteration loop uses barrier.cluster: every cross-CTA transfer is a PUSH --
// st.async remote stores into the consumer CTA's shared memory that complete
// a transaction count on the consumer's own mbarrier -- so a consumer waits
// exactly for the bytes it needs, and no CTA reads remote memory inside the
// loop (the setup reads x0's and cz's halo planes once, after a full cluster
// barrier):
//   * z halos: the thread that updates a cell of a slab's first/last plane
//     (p in the K1 update, s in the K2 update) also stores it into the
//     neighbour's halo plane (one mbarrier per halo vector);
//   * reductions: lane butterfly per warp, one warp folds the CTA's warp
//     partials, and its first CL lanes store the CTA partial into slot `rank`
//     of every CTA (double-buffered slots, one mbarrier per buffer); each CTA
//     then folds the CL partials in rank order, so all CTAs take identical
//     scalar decisions (correctly rounded dots, §3.1).
// Reuse of a buffer is safe without a barrier because a CTA can only push into
// a buffer's next use after every CTA has pushed the intervening transfer,
// i.e. after every CTA has consumed this one (program order: consume, then
// push the next).  For the same reason each mbarrier is armed (expect_tx) for
// its next phase right after the consumer's wait, before any producer can
// push that phase.  At exit the kernel also computes the true residual of the
// returned iterate (x's halos pushed like p's, one more reduction) and writes
// the whole solver record, so a solve is one launch.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace mfx {

namespace {

#ifndef MFX_CL_CT
#define MFX_CL_CT 256
#endif
constexpr int CT = MFX_CL_CT;   // threads per CTA (B200, c1: 256 -> 6.4 us per iteration, 512 -> 7.2 us)
constexpr int NW = CT / 32;

struct ClArgs {
    int nx, ny, nz;
    const double *aP, *aE, *aW, *aN, *aS, *aT, *aB, *b;
    double *x;
    double tol;
    int maxit;
    int M;                 // smem stride: max cells owned by one CTA
    WsHeader *h;
    long long *trace;      // optional: clock64 stamps of CTA 0 per phase (MFX_CLUSTER_TRACE)
};

// Cluster-wide correctly rounded reduction of K double-doubles (push model,
// see the file comment); every thread of every CTA gets the same out[].
// Default: warp 0 folds the CTA's warp partials and pushes one CTA partial
// per value (NS = CL slots).  MFX_CL_WPUSH: every warp pushes its own
// partial (NS = CL x NW slots), skipping the CTA barrier and fold before the
// push at the price of a longer final fold.
#ifdef MFX_CL_WPUSH
constexpr int kWpush = 1;
#else
constexpr int kWpush = 0;
#endif
template <int CL>
struct ClusterRed {
    static constexpr int NS = kWpush ? CL * NW : CL;
    dd (*wpart)[NW];       // [3][NW] this CTA's warp partials
    dd (*red)[3][NS];      // [2][3][NS] pushed partials
    uint64_t *mb;          // [2] one mbarrier per buffer
    uint32_t dst;          // lane j < CL: address of this CTA's (warp's) slot red[0][0][.] in CTA j
    uint32_t bar0, bar1;   // lane j < CL: CTA j's mbarriers
    double (*bc)[3];       // [2][3] folded results (double-buffered: no barrier before the next write)
    uint32_t ph0 = 0, ph1 = 0;   // (scalars, not arrays indexed by buf: no local memory)
    int buf = 0;
    template <int K>
    __device__ __forceinline__ void run(dd (&v)[K], double (&out)[K])
    {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        butterfly_lazy<K, 32>(v);
        // always 3 slots (zeros beyond K): every use of a buffer carries the
        // same byte count, so its mbarrier is re-armed right after each use
        if (kWpush) {
            if (lane < CL)
#pragma unroll
                for (int q = 0; q < 3; q++)
                    push_f64x2(dst + (uint32_t)((buf * 3 + q) * NS * 16), q < K ? v[q].hi : 0.0, q < K ? v[q].lo : 0.0,
                               buf ? bar1 : bar0);
        } else {
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < K; q++) wpart[q][wid] = v[q];
            __syncthreads();
            if (wid == 0) {
                dd y[K];
#pragma unroll
                for (int q = 0; q < K; q++) y[q] = wpart[q][lane & (NW - 1)];
                butterfly_lazy<K, NW>(y);
                if (lane < CL)
#pragma unroll
                    for (int q = 0; q < 3; q++)
                        push_f64x2(dst + (uint32_t)((buf * 3 + q) * NS * 16), q < K ? y[q].hi : 0.0,
                                   q < K ? y[q].lo : 0.0, buf ? bar1 : bar0);
            }
        }
        if (buf) { mbar_wait_cluster(&mb[1], ph1); ph1 ^= 1u; }
        else { mbar_wait_cluster(&mb[0], ph0); ph0 ^= 1u; }
        // arm the buffer's next use now: no CTA can push into it before this
        // CTA has pushed the next reduction (so the arm precedes every push)
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&mb[buf], (uint32_t)(NS * 3 * 16));
        // one warp folds the pushed partials, the others wait at the CTA
        // barrier (16 warps folding redundantly contend for the fp64 pipe:
        // measured slower)
        if (wid == 0) {
            dd y[K];
            if (NS <= 32) {
#pragma unroll
                for (int q = 0; q < K; q++) y[q] = red[buf][q][lane & (NS - 1)];
                butterfly_lazy<K, (NS <= 32 ? NS : 32)>(y);
            } else {
#pragma unroll
                for (int q = 0; q < K; q++) {
                    y[q] = red[buf][q][lane];
#pragma unroll
                    for (int j = 32; j < NS; j += 32) y[q] = dd_add_lazy(y[q], red[buf][q][lane + j]);
                }
                butterfly_lazy<K, 32>(y);
            }
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < K; q++) bc[buf][q] = dd_round(y[q]);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < K; q++) out[q] = bc[buf][q];
        buf ^= 1;
    }
};

template <bool SYM, int CL>
__global__ void __launch_bounds__(CT) k_bicg_cluster(ClArgs a)
{
    const int rank = (int)cl_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int NA = SYM ? 3 : 7;
    extern __shared__ __align__(16) double smd[];
    const int M = a.M;
    double *C = smd;                     // NA arrays: SYM {cx, cy, cz} (aP derived); else {aP, aW, aE, aS, aN, aB, aT}
    double *b = C + NA * M;
    double *x = b + M, *r = x + M, *rh = r + M, *p = rh + M, *v = p + M, *s = v + M, *t = s + M;
    __shared__ int k0s[CL + 1];
    __shared__ __align__(16) dd wpart[3][NW];     // this CTA's warp partials
    __shared__ __align__(16) dd red[2][3][ClusterRed<CL>::NS];   // pushed partials, double-buffered
    __shared__ double bcast[2][3];                // folded results
    __shared__ __align__(8) uint64_t mb_red[2], mb_halo[2];   // reductions; halo planes of p / s
    const int nx = a.nx, ny = a.ny, nz = a.nz, plane = nx * ny;
    if (tid <= CL) k0s[tid] = (int)((long long)nz * tid / CL);
    if (tid == 0) {
        mbar_init(&mb_red[0], 1); mbar_init(&mb_red[1], 1);
        mbar_init(&mb_halo[0], 1); mbar_init(&mb_halo[1], 1);
        // first phases armed before any CTA can push (the setup cluster barrier)
        mbar_arrive_expect_tx(&mb_red[0], (uint32_t)(ClusterRed<CL>::NS * 3 * 16));
        mbar_arrive_expect_tx(&mb_red[1], (uint32_t)(ClusterRed<CL>::NS * 3 * 16));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int k0 = k0s[rank], k1 = k0s[rank + 1];
    const int npl = k1 - k0, nc = npl * plane;
    const long long g0 = (long long)k0 * plane;
    // owners of the halo planes k0-1 and k1 (ranks with at least one plane)
    int rb = -1, ra = -1;
    if (k0 >= 1 && npl > 0)
        for (int q = 0; q < CL; q++)
            if (k0s[q] <= k0 - 1 && k0 - 1 < k0s[q + 1]) rb = q;
    if (k1 < nz && npl > 0)
        for (int q = 0; q < CL; q++)
            if (k0s[q] <= k1 && k1 < k0s[q + 1]) ra = q;
    const int lb = rb >= 0 ? (k0 - 1 - k0s[rb]) * plane : 0;   // offset of plane k0-1 in rb's slab
    const int la = ra >= 0 ? (k1 - k0s[ra]) * plane : 0;       // offset of plane k1 in ra's slab
    // halo bytes this CTA receives per halo transfer
    const uint32_t halo_bytes = (uint32_t)(((rb >= 0) + (ra >= 0)) * plane * 8);

    for (int i = tid; i < nc; i += CT) {
        if (SYM) {
            C[0 * M + i] = a.aE[g0 + i];
            C[1 * M + i] = a.aN[g0 + i];
            C[2 * M + i] = a.aT[g0 + i];
        } else {
            C[0 * M + i] = a.aP[g0 + i];
            C[1 * M + i] = a.aW[g0 + i];
            C[2 * M + i] = a.aE[g0 + i];
            C[3 * M + i] = a.aS[g0 + i];
            C[4 * M + i] = a.aN[g0 + i];
            C[5 * M + i] = a.aB[g0 + i];
            C[6 * M + i] = a.aT[g0 + i];
        }
        b[i] = a.b[g0 + i];
        x[i] = a.x[g0 + i];
    }
    // halo planes: [vector 0 = p (and x at setup) | 1 = s][below | above]
    double *hal = t + M;
    double *czb = hal + 4 * plane;                        // cz of plane k0-1 (SYM)
    int *cf = (int *)(czb + plane);                       // per-cell neighbour flags | in-plane offset << 8
    for (int i = tid; i < nc; i += CT) {
        const int kl = i / plane, o = i - kl * plane;
        const int iy = o / nx, ix = o - iy * nx;
        const int k = k0 + kl;
        int f = 0;
        if (ix > 0) f |= 1;
        if (ix < nx - 1) f |= 2;
        if (iy > 0) f |= 4;
        if (iy < ny - 1) f |= 8;
        if (k > 0) f |= 16;
        if (k < nz - 1) f |= 32;
        if (kl > 0) f |= 64;
        if (kl < npl - 1) f |= 128;
        cf[i] = f | (o << 8);
    }
    // remote addresses: the neighbour below receives my first plane into its
    // "above" halo, the neighbour above my last plane into its "below" halo
    const uint32_t hal_u = smem_u32(hal);
    // (halo vector h's planes sit 2 h planes apart, its mbarrier 8 h bytes apart)
    uint32_t dst_b = 0, dst_a = 0, bar_b = 0, bar_a = 0;
    if (rb >= 0) {
        dst_b = mapa_u32(hal_u + (uint32_t)(plane * 8), rb);
        bar_b = mapa_u32(smem_u32(&mb_halo[0]), rb);
    }
    if (ra >= 0) {
        dst_a = mapa_u32(hal_u, ra);
        bar_a = mapa_u32(smem_u32(&mb_halo[0]), ra);
    }
    uint32_t red_dst = 0, red_bar[2] = {0, 0};   // lane j < CL of the folding warp pushes to CTA j
    if (lane < CL) {
        red_dst = mapa_u32(smem_u32(&red[0][0][kWpush ? rank * NW + (tid >> 5) : rank]), lane);
        red_bar[0] = mapa_u32(smem_u32(&mb_red[0]), lane);
        red_bar[1] = mapa_u32(smem_u32(&mb_red[1]), lane);
    }
    uint32_t ph_halo0 = 0, ph_halo1 = 0;

    ClusterRed<CL> R{wpart, red, mb_red, red_dst, red_bar[0], red_bar[1], bcast};

    // y = A X at own cell i (DESIGN.md §3.2 order W,E,S,N,B,T); X's z halo in hb / ha
    auto apply = [&](const double *X, const double *hb, const double *ha, int i) -> double {
        const int f = cf[i], o = f >> 8;
        const double xc = X[i];
        const double xW = (f & 1) ? X[i - 1] : 0.0;
        const double xE = (f & 2) ? X[i + 1] : 0.0;
        const double xS = (f & 4) ? X[i - nx] : 0.0;
        const double xN = (f & 8) ? X[i + nx] : 0.0;
        double xB = 0.0, xT = 0.0;
        if (f & 16) xB = (f & 64) ? X[i - plane] : hb[o];
        if (f & 32) xT = (f & 128) ? X[i + plane] : ha[o];
        double aP, aW, aE, aS, aN, aB, aT;
        if (SYM) {
            const double *cx = C, *cy = C + M, *cz = C + 2 * M;
            aW = (f & 1) ? cx[i - 1] : 0.0;
            aE = cx[i];
            aS = (f & 4) ? cy[i - nx] : 0.0;
            aN = cy[i];
            aB = 0.0;
            if (f & 16) aB = (f & 64) ? cz[i - plane] : czb[o];
            aT = cz[i];
            aP = ((((aW + aE) + aS) + aN) + aB) + aT;   // p' diagonal = row sum
        } else {
            aP = C[i];
            aW = C[1 * M + i]; aE = C[2 * M + i]; aS = C[3 * M + i];
            aN = C[4 * M + i]; aB = C[5 * M + i]; aT = C[6 * M + i];
        }
        double y = aP * xc;
        y = fma(-aW, xW, y);
        y = fma(-aE, xE, y);
        y = fma(-aS, xS, y);
        y = fma(-aN, xN, y);
        y = fma(-aB, xB, y);
        y = fma(-aT, xT, y);
        return y;
    };
    // a slab-boundary value of halo vector h goes to the neighbours' halo planes
    auto push_halo = [&](int h, int i, double val) {
        const int kl = i / plane, o = i - kl * plane;
#ifdef MFX_CL_PULL
        return;
#endif
        const uint32_t ho = (uint32_t)(h * 2 * plane * 8 + o * 8);
        if (kl == 0 && rb >= 0) push_f64(dst_b + ho, val, bar_b + 8u * h);
        if (kl == npl - 1 && ra >= 0) push_f64(dst_a + ho, val, bar_a + 8u * h);
    };
    // halo mbarriers: armed for their first phase before the setup barrier and
    // re-armed right after each wait (a neighbour pushes the next phase only
    // after the following reduction, which waits for this CTA)
    if (tid == 0 && halo_bytes) {
        mbar_arrive_expect_tx(&mb_halo[0], halo_bytes);
        mbar_arrive_expect_tx(&mb_halo[1], halo_bytes);
    }
    auto arm_halo = [&](int) {};
    auto wait_halo = [&](int h) {
        __syncthreads();   // in-slab neighbours
#ifdef MFX_CL_PULL
        {
            cluster_sync_full();
            const double *X = h ? s : p;
            const double *xb = rb >= 0 ? (const double *)__cluster_map_shared_rank((void *)X, rb) : nullptr;
            const double *xa = ra >= 0 ? (const double *)__cluster_map_shared_rank((void *)X, ra) : nullptr;
            for (int o = tid; o < plane; o += CT) {
                if (rb >= 0) hal[2 * h * plane + o] = xb[lb + o];
                if (ra >= 0) hal[(2 * h + 1) * plane + o] = xa[la + o];
            }
            cluster_sync_full();
            return;
        }
#endif
        if (halo_bytes) {
            if (h) { mbar_wait_cluster(&mb_halo[1], ph_halo1); ph_halo1 ^= 1u; }
            else { mbar_wait_cluster(&mb_halo[0], ph_halo0); ph_halo0 ^= 1u; }
            if (tid == 0) mbar_arrive_expect_tx(&mb_halo[h], halo_bytes);
        }
    };

    const double tol = a.tol;
    const int maxit = a.maxit;
    int tix = 0;
    auto stamp = [&]() {
        if (a.trace && rank == 0 && tid == 0 && tix < 512) a.trace[tix++] = clock64();
    };
    int status = MFX_NOT_CONVERGED, iters = 0, restarts = 0;
    double bn, rr, rn;

    // ---- setup: r = b - A x0 (x0 and cz halos read once over DSMEM after a full barrier)
    cluster_sync_full();   // x0, coefficients and mbarriers of every CTA initialised
    {
        const double *xr_b = rb >= 0 ? (const double *)__cluster_map_shared_rank((void *)x, rb) : nullptr;
        const double *xr_a = ra >= 0 ? (const double *)__cluster_map_shared_rank((void *)x, ra) : nullptr;
        const double *cz_b = (SYM && rb >= 0) ? (const double *)__cluster_map_shared_rank((void *)(C + 2 * M), rb)
                                              : nullptr;
        for (int o = tid; o < plane; o += CT) {
            if (rb >= 0) hal[o] = xr_b[lb + o];
            if (ra >= 0) hal[plane + o] = xr_a[la + o];
            if (SYM) czb[o] = rb >= 0 ? cz_b[lb + o] : 0.0;
        }
    }
    __syncthreads();   // halo planes and cz below filled before any thread applies A
    // (no second cluster barrier: a neighbour pushes p into these halo planes only
    // after the setup reduction, which waits for this CTA's push, issued after its reads)
    {
        Acc bb, ra_;
        bb.zero(); ra_.zero();
        for (int i = tid; i < nc; i += CT) {
            const double y = apply(x, hal, hal + plane, i);
            const double rv = b[i] - y;
            r[i] = rv;
            bb.prod(b[i], b[i]);
            ra_.prod(rv, rv);
        }
        dd vv[2] = {bb.get(), ra_.get()};
        double out[2];
        R.template run<2>(vv, out);
        bn = sqrt(out[0]);
        rr = out[1];
        rn = sqrt(rr);
    }
    if (bn == 0.0) {
        for (int i = tid; i < nc; i += CT) x[i] = 0.0;
        status = MFX_OK; rn = 0.0;
    } else if (rn <= tol * bn) {
        status = MFX_OK;
    } else {
        for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
        double rhn = rn, rho = rr, rho_prev = 1.0, alpha = 1.0, omega = 1.0, aw = 1.0;   // aw = alpha / omega
        bool restarted = false;
        int it;
        for (it = 1; it <= maxit; it++) {
            if (fabs(rho) <= (1e-14 * rhn) * rn) {
                if (restarted) { status = MFX_ERR_BREAKDOWN; iters = it - 1; break; }
                for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
                rhn = rn; rho = rr; rho_prev = alpha = omega = aw = 1.0; restarted = true; restarts++;
            }
            stamp();
            const double beta = (rho / rho_prev) * aw;
            arm_halo(0);
            for (int i = tid; i < nc; i += CT) {
                const double pv = fma(beta, fma(-omega, v[i], p[i]), r[i]);
                p[i] = pv;
                push_halo(0, i, pv);
            }
            stamp();
            wait_halo(0);   // p of this slab and of the neighbours' boundary planes
            stamp();
            Acc sg;
            sg.zero();
            for (int i = tid; i < nc; i += CT) {
                const double vv = apply(p, hal, hal + plane, i);
                v[i] = vv;
                sg.prod(rh[i], vv);
            }
            double sigma;
            stamp();
            {
                dd vv[1] = {sg.get()};
                double out[1];
                R.template run<1>(vv, out);
                sigma = out[0];
            }
            stamp();
            if (sigma == 0.0) {
                if (restarted) { status = MFX_ERR_BREAKDOWN; iters = it; break; }
                for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
                rhn = rn; rho = rr; rho_prev = alpha = omega = aw = 1.0; restarted = true; restarts++;
                continue;
            }
            alpha = rho / sigma;
            arm_halo(1);
            for (int i = tid; i < nc; i += CT) {
                const double sv = fma(-alpha, v[i], r[i]);
                s[i] = sv;
                push_halo(1, i, sv);
            }
            wait_halo(1);
            Acc ts, tt, ss;
            ts.zero(); tt.zero(); ss.zero();
            for (int i = tid; i < nc; i += CT) {
                const double tv = apply(s, hal + 2 * plane, hal + 3 * plane, i);
                t[i] = tv;
                ts.prod(tv, s[i]);
                tt.prod(tv, tv);
                ss.prod(s[i], s[i]);
            }
            double tsv, ttv, ssv;
            stamp();
            {
                dd vv[3] = {ts.get(), tt.get(), ss.get()};
                double out[3];
                R.template run<3>(vv, out);
                tsv = out[0]; ttv = out[1]; ssv = out[2];
            }
            stamp();
            if (sqrt(ssv) <= tol * bn) {
                for (int i = tid; i < nc; i += CT) { x[i] = fma(alpha, p[i], x[i]); r[i] = s[i]; }
                rn = sqrt(ssv);
                status = MFX_OK; iters = it;
                break;
            }
            const double om = ttv == 0.0 ? 0.0 : tsv / ttv;
            if (ttv == 0.0 || om == 0.0) {
                if (restarted) { status = MFX_ERR_BREAKDOWN; iters = it; break; }
                for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
                rhn = rn; rho = rr; rho_prev = alpha = omega = aw = 1.0; restarted = true; restarts++;
                continue;
            }
            omega = om;
            aw = alpha / omega;   // beta's second quotient, off the critical path after the next reduction
            Acc rhr, rra;
            rhr.zero(); rra.zero();
            for (int i = tid; i < nc; i += CT) {
                const double xn = fma(omega, s[i], fma(alpha, p[i], x[i]));
                const double rv = fma(-omega, t[i], s[i]);
                x[i] = xn;
                r[i] = rv;
                rhr.prod(rh[i], rv);
                rra.prod(rv, rv);
            }
            rho_prev = rho;
            stamp();
            {
                dd vv[2] = {rhr.get(), rra.get()};
                double out[2];
                R.template run<2>(vv, out);
                rho = out[0]; rr = out[1];
            }
            rn = sqrt(rr);
            if (rn <= tol * bn) { status = MFX_OK; iters = it; break; }
        }
        if (it > maxit) { status = MFX_NOT_CONVERGED; iters = maxit; }
    }
    // true residual of the returned iterate (mfx_solve_info.true_rel_resid,
    // the k_true_resid definition: sqrt(dot(r, r)) / sqrt(dot(b, b)) with
    // r = b - A x, correctly rounded dots): x's boundary planes travel like
    // p's (halo 0 is armed for its next phase), one more reduction; saves the
    // separate launch per solve
    double true_rel = 0.0;
    if (bn != 0.0) {
        for (int i = tid; i < nc; i += CT) push_halo(0, i, x[i]);
        wait_halo(0);
        Acc rt;
        rt.zero();
        for (int i = tid; i < nc; i += CT) {
            const double rv = b[i] - apply(x, hal, hal + plane, i);
            rt.prod(rv, rv);
        }
        dd vv[1] = {rt.get()};
        double out[1];
        R.template run<1>(vv, out);
        true_rel = sqrt(out[0]) / bn;
    }
    for (int i = tid; i < nc; i += CT) a.x[g0 + i] = x[i];
    if (rank == 0 && tid == 0) {
        SolverScalars S = SolverScalars{};   // the whole record (the host path skips its memset)
        S.it = iters; S.status = status; S.restarts = restarts; S.rn = rn; S.bn = bn; S.done = 1;
        S.tol = tol; S.maxit = maxit;
        a.h->sc = S;
        a.h->true_rel = true_rel;
    }
    // every push into this CTA's shared memory has completed (each was waited
    // for); keep it alive until every CTA is done as well
    cluster_sync_full();
}

// cluster size: 16 where the device can place a 16-CTA cluster of this
// kernel, else 8 (portable); MFX_CLUSTER=8 forces the portable size
int g_cl = 0;

template <bool SYM, int CL>
bool cluster_can_launch(size_t smem)
{
    auto kfn = k_bicg_cluster<SYM, CL>;
    if (CL > 8 && cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL); cfg.blockDim = dim3(CT); cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kfn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return n >= 1;
}

}  // namespace

int cluster_size()
{
    if (g_cl == 0) {
        const char *e = getenv("MFX_CLUSTER");
        int want = e ? atoi(e) : 16;
        if (want != 8) want = cluster_can_launch<true, 16>(200 * 1024) && cluster_can_launch<false, 16>(200 * 1024)
                              ? 16 : 8;
        g_cl = want;
    }
    return g_cl;
}
void cluster_size_set(int cl) { g_cl = cl; }

long long *&cluster_trace_ptr()
{
    static long long *p = nullptr;
    return p;
}

// dynamic smem: (NA + 8) arrays of M cells + 5 planes (four halo planes, cz below) + M flags
size_t cluster_smem(const Geo &G, bool sym)
{
    const long long plane = (long long)G.nx * G.ny;
    const int CL = cluster_size();
    const long long M = plane * ((G.nz + CL - 1) / CL);
    return (size_t)(((sym ? 11 : 15) * M + 5 * plane) * sizeof(double) + M * sizeof(int));
}

bool cluster_fits(const Geo &G, bool sym) { return cluster_smem(G, sym) <= 200 * 1024; }

template <bool SYM, int CL>
static mfx_status cluster_launch(const ClArgs &a, size_t smem, cudaStream_t s)
{
    auto kfn = k_bicg_cluster<SYM, CL>;
    if (CL > 8) MFX_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    MFX_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL); cfg.blockDim = dim3(CT); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cfg.attrs = at; cfg.numAttrs = 1;
    MFX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kfn, a));
    return MFX_OK;
}

mfx_status cluster_solve(bool sym, const Geo &G, const mfx_eqsys *A, double *x, double tol, int maxit,
                         WsHeader *h, cudaStream_t s)
{
    ClArgs a;
    a.nx = G.nx; a.ny = G.ny; a.nz = G.nz;
    a.aP = A->aP; a.aE = A->aE; a.aW = A->aW; a.aN = A->aN; a.aS = A->aS; a.aT = A->aT; a.aB = A->aB; a.b = A->b;
    a.x = x; a.tol = tol; a.maxit = maxit; a.h = h;
    a.trace = nullptr;
    if (getenv("MFX_CLUSTER_TRACE")) {
        static long long *tr = nullptr;
        if (!tr) cudaMalloc(&tr, 512 * sizeof(long long));
        cudaMemsetAsync(tr, 0, 512 * sizeof(long long), s);
        a.trace = tr;
        cluster_trace_ptr() = tr;
    }
    const int CL = cluster_size();
    a.M = G.nx * G.ny * ((G.nz + CL - 1) / CL);
    const size_t smem = cluster_smem(G, sym);
    mfx_status st;
    if (CL == 16) st = sym ? cluster_launch<true, 16>(a, smem, s) : cluster_launch<false, 16>(a, smem, s);
    else st = sym ? cluster_launch<true, 8>(a, smem, s) : cluster_launch<false, 8>(a, smem, s);
    if (st != MFX_OK) return st;
    MFX_CUDA_TRY(cudaGetLastError());
    if (a.trace) {   // debug: per-phase cycle deltas of CTA 0 for the first iterations
        long long hh[512];
        cudaMemcpyAsync(hh, a.trace, sizeof(hh), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "cluster trace (CL %d, cycles): p-update halo-wait apply1 red1 s+halo+apply2 red3 k3 red2\n",
                CL);
        for (int it = 0; it < 8 && hh[it * 8 + 7] != 0; it++) {
            fprintf(stderr, "  it %d:", it + 1);
            for (int q = 1; q < 8; q++) fprintf(stderr, " %lld", hh[it * 8 + q] - hh[it * 8 + q - 1]);
            if (hh[(it + 1) * 8] != 0) fprintf(stderr, " | total %lld", hh[(it + 1) * 8] - hh[it * 8]);
            fprintf(stderr, "\n");
        }
    }
    return MFX_OK;
}

}  // namespace mfx
