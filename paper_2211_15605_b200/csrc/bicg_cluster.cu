// bicg_cluster.cu -- a-6 for small systems (BASELINE.json configuration 1,
// 16x16x32): the whole unpreconditioned BiCGSTAB solve in
// ONE launch of one thread-block cluster of 8 CTAs (8 SMs).
//
// The grid is split into 8 z-slabs; CTA `rank` keeps its slab of every
// coefficient and vector in shared memory for the whole solve, reads the z
// halo planes of its neighbours through distributed shared memory
// (map_shared_rank), and replaces the grid-wide reductions of the large-N
// kernels by cluster barriers: each CTA publishes its double-double partial,
// barrier.cluster, and every CTA folds the 8 partials in rank order, so all
// CTAs take identical scalar decisions (correctly rounded dots, §3.1).
// Five cluster barriers per iteration; no kernel launches inside the loop.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mfx {

namespace {

constexpr int CL = 8;     // CTAs per cluster (portable maximum)
constexpr int CT = 256;   // threads per CTA

// Cluster barrier for shared-memory exchange.  cg::cluster_group::sync()
// (barrier.cluster.arrive.release) compiles to MEMBAR.ALL.GPU on sm_100a;
// everything exchanged here lives in shared memory, so a CTA barrier (which
// drains this CTA's pending shared stores) followed by a relaxed cluster
// arrive / wait orders the writes before any remote DSMEM read.
__device__ __forceinline__ void cluster_barrier()
{
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

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

// Cluster-wide correctly rounded reduction of K double-doubles: each warp
// publishes its butterfly partial; after barrier.cluster the 64 partials
// (8 CTAs x 8 warps) of each value are gathered in parallel into local
// shared memory and folded by one warp in a fixed order, so every CTA gets
// the identical result.  Publication slots alternate between two buffers
// (the barrier of reduction j+1 orders all remote reads of reduction j
// before any CTA overwrites its slots in reduction j+2).
struct ClusterRed {
    dd (*pub)[3][8];       // [2][3][8] this CTA's per-warp partials
    dd (*tmp)[64];         // [3][64] gathered partials
    dd *bc;                // [3] folded results
    template <int K>
    __device__ void run(cg::cluster_group &cl, int &buf, dd (&v)[K], double (&out)[K])
    {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        dd x[K];
#pragma unroll
        for (int q = 0; q < K; q++) x[q] = v[q];
        // the K butterflies advance level by level (independent chains interleave)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            dd y[K];
#pragma unroll
            for (int q = 0; q < K; q++) y[q] = shfl_dd(x[q], off);
#pragma unroll
            for (int q = 0; q < K; q++) x[q] = (lane & off) ? dd_add_fast(y[q], x[q]) : dd_add_fast(x[q], y[q]);
        }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < K; q++) pub[buf][q][wid] = x[q];
        cluster_barrier();
        if (threadIdx.x < 64 * K) {
            const int q = threadIdx.x >> 6, idx = threadIdx.x & 63;
            tmp[q][idx] = *cl.map_shared_rank(&pub[buf][q][idx & 7], idx >> 3);
        }
        __syncthreads();
        if (wid == 0) {
#pragma unroll
            for (int q = 0; q < K; q++) x[q] = dd_add_fast(tmp[q][lane], tmp[q][lane + 32]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                dd y[K];
#pragma unroll
                for (int q = 0; q < K; q++) y[q] = shfl_dd(x[q], off);
#pragma unroll
                for (int q = 0; q < K; q++) x[q] = (lane & off) ? dd_add_fast(y[q], x[q]) : dd_add_fast(x[q], y[q]);
            }
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < K; q++) bc[q] = x[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < K; q++) out[q] = dd_round(bc[q]);
        buf ^= 1;
    }
};

template <bool SYM>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(CT) k_bicg_cluster(ClArgs a)
{
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x;
    constexpr int NA = SYM ? 3 : 7;
    extern __shared__ __align__(16) double smd[];
    const int M = a.M;
    double *C = smd;                     // NA arrays: SYM {cx, cy, cz} (aP derived); else {aP, aW, aE, aS, aN, aB, aT}
    double *b = C + NA * M;
    double *x = b + M, *r = x + M, *rh = r + M, *p = rh + M, *v = p + M, *s = v + M, *t = s + M;
    __shared__ int k0s[CL + 1];
    __shared__ dd pub[2][3][8];
    __shared__ dd tmp[3][64];
    __shared__ dd bc[3];
    const int nx = a.nx, ny = a.ny, nz = a.nz, plane = nx * ny;
    if (tid <= CL) k0s[tid] = (int)((long long)nz * tid / CL);
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
    ClusterRed R{pub, tmp, bc};
    int buf = 0;   // parity of the publication slots, shared by all reductions
    double *hb = t + M, *ha = hb + plane;                 // local copies of the z-halo planes
    double *czb = ha + plane;                             // cz of plane k0-1 (SYM)
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

    // y = A X at own cell i (DESIGN.md §3.2 order W,E,S,N,B,T); X read with its z halo
    auto apply = [&](const double *X, int i) -> double {
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
    auto reduce1 = [&](Acc &a0, double &o0) {
        dd vv[1] = {a0.get()};
        double out[1];
        R.run<1>(cl, buf, vv, out);
        o0 = out[0];
    };
    auto reduce2 = [&](Acc &a0, Acc &a1, double &o0, double &o1) {
        dd vv[2] = {a0.get(), a1.get()};
        double out[2];
        R.run<2>(cl, buf, vv, out);
        o0 = out[0]; o1 = out[1];
    };
    // after a cluster barrier: copy the neighbours' boundary planes of X locally
    auto fetch_halo = [&](const double *X) {
        for (int o = tid; o < plane; o += CT) {
            if (rb >= 0) hb[o] = cl.map_shared_rank(X, rb)[lb + o];
            if (ra >= 0) ha[o] = cl.map_shared_rank(X, ra)[la + o];
        }
        __syncthreads();
    };

    const double tol = a.tol;
    const int maxit = a.maxit;
    int tix = 0;
    auto stamp = [&]() {
        if (a.trace && rank == 0 && tid == 0 && tix < 512) a.trace[tix++] = clock64();
    };
    int status = MFX_NOT_CONVERGED, iters = 0, restarts = 0;
    double bn, rr, rn;

    // ---- setup: r = b - A x0
    cluster_barrier();   // x0 and coefficients of every slab loaded
    if (SYM)
        for (int o = tid; o < plane; o += CT) czb[o] = rb >= 0 ? cl.map_shared_rank(C + 2 * M, rb)[lb + o] : 0.0;
    fetch_halo(x);
    {
        Acc bb, ra_;
        bb.zero(); ra_.zero();
        for (int i = tid; i < nc; i += CT) {
            const double y = apply(x, i);
            const double rv = b[i] - y;
            r[i] = rv;
            bb.prod(b[i], b[i]);
            ra_.prod(rv, rv);
        }
        double bbv;
        reduce2(bb, ra_, bbv, rr);
        bn = sqrt(bbv);
        rn = sqrt(rr);
    }
    if (bn == 0.0) {
        for (int i = tid; i < nc; i += CT) x[i] = 0.0;
        status = MFX_OK; rn = 0.0;
    } else if (rn <= tol * bn) {
        status = MFX_OK;
    } else {
        for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
        double rhn = rn, rho = rr, rho_prev = 1.0, alpha = 1.0, omega = 1.0;
        bool restarted = false;
        int it;
        for (it = 1; it <= maxit; it++) {
            if (fabs(rho) <= (1e-14 * rhn) * rn) {
                if (restarted) { status = MFX_ERR_BREAKDOWN; iters = it - 1; break; }
                for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
                rhn = rn; rho = rr; rho_prev = alpha = omega = 1.0; restarted = true; restarts++;
            }
            stamp();
            const double beta = (rho / rho_prev) * (alpha / omega);
            for (int i = tid; i < nc; i += CT) p[i] = fma(beta, fma(-omega, v[i], p[i]), r[i]);
            stamp();
            cluster_barrier();   // p of every slab visible
            stamp();
            fetch_halo(p);
            stamp();
            Acc sg;
            sg.zero();
            for (int i = tid; i < nc; i += CT) {
                const double vv = apply(p, i);
                v[i] = vv;
                sg.prod(rh[i], vv);
            }
            double sigma;
            stamp();
            reduce1(sg, sigma);
            stamp();
            if (sigma == 0.0) {
                if (restarted) { status = MFX_ERR_BREAKDOWN; iters = it; break; }
                for (int i = tid; i < nc; i += CT) { rh[i] = r[i]; p[i] = 0.0; v[i] = 0.0; }
                rhn = rn; rho = rr; rho_prev = alpha = omega = 1.0; restarted = true; restarts++;
                continue;
            }
            alpha = rho / sigma;
            for (int i = tid; i < nc; i += CT) s[i] = fma(-alpha, v[i], r[i]);
            cluster_barrier();   // s of every slab visible
            fetch_halo(s);
            stamp();
            Acc ts, tt, ss;
            ts.zero(); tt.zero(); ss.zero();
            for (int i = tid; i < nc; i += CT) {
                const double tv = apply(s, i);
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
                R.run<3>(cl, buf, vv, out);
                tsv = out[0]; ttv = out[1]; ssv = out[2];
            }
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
                rhn = rn; rho = rr; rho_prev = alpha = omega = 1.0; restarted = true; restarts++;
                continue;
            }
            omega = om;
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
            reduce2(rhr, rra, rho, rr);
            stamp();
            rn = sqrt(rr);
            if (rn <= tol * bn) { status = MFX_OK; iters = it; break; }
        }
        if (it > maxit) { status = MFX_NOT_CONVERGED; iters = maxit; }
    }
    for (int i = tid; i < nc; i += CT) a.x[g0 + i] = x[i];
    if (rank == 0 && tid == 0) {
        SolverScalars &S = a.h->sc;
        S.it = iters; S.status = status; S.restarts = restarts; S.rn = rn; S.bn = bn; S.done = 1;
        S.tol = tol; S.maxit = maxit;
    }
    cluster_barrier();   // keep every CTA's shared memory alive until all remote reads are done
}

}  // namespace

long long *&cluster_trace_ptr()
{
    static long long *p = nullptr;
    return p;
}

// dynamic smem: (NA + 8) arrays of M cells + 3 planes (two halo copies, cz below)
size_t cluster_smem(const Geo &G, bool sym)
{
    const long long plane = (long long)G.nx * G.ny;
    const long long M = plane * ((G.nz + CL - 1) / CL);
    return (size_t)(((sym ? 11 : 15) * M + 3 * plane) * sizeof(double) + M * sizeof(int));
}

bool cluster_fits(const Geo &G, bool sym) { return cluster_smem(G, sym) <= 200 * 1024; }

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
    a.M = G.nx * G.ny * ((G.nz + CL - 1) / CL);
    const size_t smem = cluster_smem(G, sym);
    if (sym) {
        MFX_CUDA_TRY(cudaFuncSetAttribute(k_bicg_cluster<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_bicg_cluster<true><<<CL, CT, smem, s>>>(a);
    } else {
        MFX_CUDA_TRY(cudaFuncSetAttribute(k_bicg_cluster<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_bicg_cluster<false><<<CL, CT, smem, s>>>(a);
    }
    MFX_CUDA_TRY(cudaGetLastError());
    if (a.trace) {   // debug: per-phase cycle deltas of CTA 0 for the first iterations
        long long h[512];
        cudaMemcpyAsync(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "cluster trace (cycles): p-update bar halo apply1 red1 s+bar+halo+apply2 red3 k3 red2\n");
        for (int it = 0; it < 8 && h[it * 10 + 9] != 0; it++) {
            fprintf(stderr, "  it %d:", it + 1);
            for (int q = 1; q < 10; q++) fprintf(stderr, " %lld", h[it * 10 + q] - h[it * 10 + q - 1]);
            if (h[(it + 1) * 10] != 0) fprintf(stderr, " | total %lld", h[(it + 1) * 10] - h[it * 10]);
            fprintf(stderr, "\n");
        }
    }
    return MFX_OK;
}

}  // namespace mfx
