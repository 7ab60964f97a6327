// stencil_tma.cu -- the bandwidth-critical 7-point kernels of BiCGSTAB
// (setup r = b - A x0, K1, K2, plain apply) as persistent TMA z-marching
// kernels for sm_100a.
//
// Layout: fields are nx*ny*nz fp64, x fastest, described to the TMA unit as
// 3-D tensors (16-byte row stride: nx even).  A CTA owns an x-y tile of
// TX x TY cells and marches along z; every plane of every input array is
// fetched by ONE cp.async.bulk.tensor per array into a ring of S shared-
// memory stages (mbarrier complete_tx), S-2 planes ahead of the compute.
// Arrays read with a stencil halo are fetched as (TX+4) x (TY+2) boxes whose
// out-of-domain part the TMA zero-fills, which is exactly the boundary rule
// of DESIGN.md §3.2 (x_nb = 0 outside the domain).
//
// Per plane:  step 1  value on the halo'd plane (x for the apply,
//                     p = fma(beta, fma(-omega, v, p), r) for K1,
//                     s = fma(-alpha, v, r) for K2) -> P ring (4 planes:
//                     one barrier per plane suffices)
//             sync; thread 0 refills the stage freed two planes ago
//             step 2  y = A P at the plane below, canonical order
//                     W,E,S,N,B,T, fused epilogue + correctly rounded dots.
// Work is split into (z-chunk, tile) units dealt round-robin over a persistent
// grid (148 x CTAs/SM) so neighbouring tiles march in lockstep (L2 reuse of
// the halo rows) and every SM streams about the same number of planes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tma.cuh"
#include "bicg_state.cuh"

namespace mfx {

enum StencilMode { SM_SPMV = 0, SM_SETUP = 1, SM_K1 = 2, SM_K2 = 3 };

struct TmaMaps {
    CUtensorMap halo[3];   // halo box arrays (x | r,p_old,v_old | r,v)
    CUtensorMap coef[7];   // SYM: cz (cell), -, cx (x-halo box), cy (y-halo box); else aP,aW,aE,aS,aN,aB,aT
    CUtensorMap extra;     // SETUP: b ; K1: r^
};

struct StencilArgs {
    int nx, ny, nz;
    int tiles_x, tiles_y;
    int Lz;                                // z-chunk length
    int reverse;                           // walk the units last-to-first (L2 ping-pong)
    long long units;                       // tiles * ceil(nz / Lz) work units
    double *out0, *out1, *out2;            // SPMV: y | SETUP: r | K1: p_new, v_new, r^ | K2: t
    WsHeader *h;
    dd *part;
    double tol;
    int maxit;
    // z-slab mode (dist_solver.cu): outputs planes [kbeg, kend) of an extended
    // slab whose planes kbeg-1 and kend hold the neighbours' ghost copies; the
    // rank's dot partials go to rank_part (folded across ranks by the caller)
    // instead of the scalar tail; K1 with ghost_store also writes p on the two
    // ghost planes (the next iteration's p_old there, bitwise the neighbour's).
    int kbeg, kend, ghost_store;
    dd *rank_part;
    unsigned long long *trace;             // optional (MFX_RW_TRACE): per-CTA %globaltimer stamps
    unsigned int *work;                    // dynamic units: grab counter (NULL: static round-robin)
    int chain;                             // K1/K2: chained tails (common.cuh: publish partials; K2 folds K1's)
};

// per-CTA %globaltimer traces (MFX_RW_TRACE / MFX_PERSIST_TRACE) are compiled
// only with -DMFX_TRACE (a variant build: MFX_EXTRA_NVCC_FLAGS=-DMFX_TRACE);
// in the default build they cost registers in the persistent kernel
#ifdef MFX_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif

__device__ __forceinline__ void ktrace(const StencilArgs &a, int slot)
{
    if (kTrace && a.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[blockIdx.x * 4 + slot] = t;
    }
}

namespace {

constexpr int r128(int b) { return (b + 127) & ~127; }

int env_int(const char *name, int dflt)
{
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}


template <int CPT>
__device__ __forceinline__ void store_cells(double *dst, const double (&v)[CPT])
{
    if (CPT == 2) *(double2 *)dst = make_double2(v[0], v[CPT - 1]);
    else dst[0] = v[0];
}

template <int MODE, bool SYM, int TX, int TY, int CPT_>
struct Cfg {
    static constexpr int NT = TX * TY / CPT_;               // consumer threads (one per owned cell or pair)
    static constexpr int HX = TX + 4, HY = TY + 2;        // halo box: x in [x0-2, x0+TX+2), y in [y0-1, y0+TY+1)
    static constexpr int CPT = CPT_;                        // owned cells per consumer thread (1 or 2)
    static constexpr int NW = NT / 32;                      // consumer warps; the producer is warp NW
    static_assert(CPT == 1 || CPT == 2, "1 or 2 cells per thread");
    static_assert(NT % 32 == 0 && NT <= 512, "consumer threads");
    static constexpr int NH = MODE == SM_K1 ? 3 : (MODE == SM_K2 ? 2 : 1);
    static constexpr int NCELLC = SYM ? 1 : 7;             // coefficient arrays with the cell box (SYM: cz; aP derived)
    static constexpr int NE = (MODE == SM_SETUP || MODE == SM_K1) ? 1 : 0;
    static constexpr int HALO_TX = HX * HY * 8, CELL_TX = TX * TY * 8;
    static constexpr int XW_TX = HX * TY * 8, YS_TX = TX * (TY + 1) * 8;
    static constexpr int HALO_B = r128(HALO_TX), CELL_B = r128(CELL_TX), XW_B = r128(XW_TX), YS_B = r128(YS_TX);
    static constexpr int STAGE_TX = NH * HALO_TX + NCELLC * CELL_TX + (SYM ? XW_TX + YS_TX : 0) + NE * CELL_TX;
    static constexpr int STAGE_B = NH * HALO_B + NCELLC * CELL_B + (SYM ? XW_B + YS_B : 0) + NE * CELL_B;
    static constexpr int PBUF_B = r128(HX * HY * 8);
    // stage offsets
    static constexpr int OFF_HALO = 0;
    static constexpr int OFF_CELL = NH * HALO_B;
    static constexpr int OFF_XW = OFF_CELL + NCELLC * CELL_B;
    static constexpr int OFF_YS = OFF_XW + (SYM ? XW_B : 0);
    static constexpr int OFF_EXTRA = OFF_YS + (SYM ? YS_B : 0);
    static constexpr int NDOT = MODE == SM_SPMV ? 0 : (MODE == SM_SETUP ? 2 : (MODE == SM_K1 ? 1 : 3));
};

template <class C>
__host__ __device__ constexpr size_t smem_bytes(int S)
{
    return (size_t)S * C::STAGE_B + 4 * (size_t)C::PBUF_B + 24 * (size_t)S;   // + full, empty, meta
}

// plane-stream cursor.  Units are (z-chunk, tile) pairs in chunk-major order,
// dealt round-robin to the persistent CTAs (unit u -> CTA u % G), so at any
// time all CTAs work on the same slab of ~G/ntiles chunks: a tile's y/x halo
// rows and its chunk-boundary planes are fetched by the neighbouring CTAs at
// the same moment and hit in L2.  A unit streams planes k0-1 .. k1
// (virtual, i.e. zero, outside [0, nz)) and outputs planes k0 .. k1-1.
struct Cursor {
    int u, units;
    int G, ntiles, Lz, tiles_x, TX, TY, rev, kbeg, kend;
    int x0, y0, k, k0, k1;
    bool valid, pending;
    unsigned int *work;   // dynamic units: the producer grabs them, consumers read them from the stage
    __device__ void start(int nz)
    {
        if (u >= units) { valid = false; return; }
        const int uu = rev ? units - 1 - u : u;
        const int chunk = uu / ntiles;
        const int tile = uu - chunk * ntiles;
        const int ty = tile / tiles_x;
        x0 = (tile - ty * tiles_x) * TX;
        y0 = ty * TY;
        k0 = kbeg + chunk * Lz;
        k1 = k0 + Lz < kend ? k0 + Lz : kend;
        k = k0 - 1;
        valid = true;
    }
    // producer: dyn -> units come from the counter; consumer: dyn -> from the stage (set_unit)
    __device__ void init(int u0, const StencilArgs &a, int nt, int tX, int tY, bool producer = true)
    {
        units = (int)a.units; G = gridDim.x; ntiles = nt; Lz = a.Lz; tiles_x = a.tiles_x; TX = tX; TY = tY;
        rev = a.reverse; kbeg = a.kbeg; kend = a.kend; work = a.work;
        pending = false;
        if (work && !producer) { pending = true; valid = true; return; }
        u = work ? (int)atomicAdd(work, 1u) : u0;
        start(a.nz);
    }
    __device__ void set_unit(int uu, int nz) { u = uu; pending = false; start(nz); }
    __device__ void advance(int nz, bool producer = true)
    {
        k++;
        if (k > k1) {
            if (!work) { u += G; start(nz); }
            else if (producer) { u = (int)atomicAdd(work, 1u); start(nz); }
            else pending = true;
        }
    }
    __device__ bool is_virtual(int nz) const { return k < 0 || k >= nz; }
    __device__ bool produces() const { return k >= k0 + 1; }
};

// dynamic units: every issued stage carries its unit id (meta[s]); after the
// last unit the producer posts one stage with id -1 and no data
__device__ __forceinline__ void post_end(uint64_t *full, uint64_t *empty, int *meta, int S, int q)
{
    const int s = q % S;
    if (q >= S) mbar_wait(&empty[s], (uint32_t)(((q / S) - 1) & 1));
    meta[s] = -1;
    mbar_arrive(&full[s]);
}

template <int MODE, bool SYM, int TX, int TY, int CPT_, int S, int STRIDE = Cfg<MODE, SYM, TX, TY, CPT_>::STAGE_B>
__device__ __forceinline__ void issue(const TmaMaps &M, const Cursor &c, int nz, uint8_t *stages, uint64_t *full,
                                      int q, int *meta = nullptr)
{
    using C = Cfg<MODE, SYM, TX, TY, CPT_>;
    static_assert(STRIDE >= C::STAGE_B, "stage slot too small");
    const int s = q % S;
    uint64_t *bar = &full[s];
    if (meta) meta[s] = c.u;   // read by the consumers after the full barrier (release by the arrive below)
    if (c.is_virtual(nz)) {
        mbar_arrive(bar);
        return;
    }
    uint8_t *st = stages + (size_t)s * STRIDE;
    const int x0 = c.x0, y0 = c.y0, k = c.k;
    mbar_arrive_expect_tx(bar, C::STAGE_TX);
#pragma unroll
    for (int a = 0; a < C::NH; a++) tma_load_3d(st + C::OFF_HALO + a * C::HALO_B, &M.halo[a], x0 - 2, y0 - 1, k, bar);
#pragma unroll
    for (int a = 0; a < C::NCELLC; a++) tma_load_3d(st + C::OFF_CELL + a * C::CELL_B, &M.coef[a], x0, y0, k, bar);
    if (SYM) {
        tma_load_3d(st + C::OFF_XW, &M.coef[2], x0 - 2, y0, k, bar);
        tma_load_3d(st + C::OFF_YS, &M.coef[3], x0, y0 - 1, k, bar);
    }
    if (C::NE) tma_load_3d(st + C::OFF_EXTRA, &M.extra, x0, y0, k, bar);
}

template <int MODE, bool SYM, int TX, int TY, int CPT_, int S>
__global__ void __launch_bounds__(Cfg<MODE, SYM, TX, TY, CPT_>::NT + 32) k_stencil(const __grid_constant__ TmaMaps M, StencilArgs a)
{
    // warps 0-7: consumers (one owned cell per thread); warp 8: TMA producer
    using C = Cfg<MODE, SYM, TX, TY, CPT_>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *stages = smem;
    double *pbuf = (double *)(smem + (size_t)S * C::STAGE_B);
    uint64_t *full = (uint64_t *)(smem + (size_t)S * C::STAGE_B + 4 * C::PBUF_B);
    uint64_t *empty = full + S;
    int *meta = (int *)(empty + S);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    // Programmatic dependent launch: let the next kernel in the stream start its
    // launch and prologue while this grid drains; everything below the wait
    // reads data the previous kernel produced.
    pdl_trigger();
    const int ntiles = a.tiles_x * a.tiles_y;
    if (tid == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    pdl_wait();

    // ---- scalar prologue (uniform across the grid)
    double beta = 0.0, omega = 0.0, alpha = 0.0;
    bool rst = false;
    K1Pro P1;
    P1.rst = false;
    if (MODE == SM_K2 && a.chain) {
        // chained: K1's scalar tail runs here, in every CTA (identical bits):
        // fold K1's published <r^, v> partials, apply it to the state K1 read
        __shared__ dd s_fsh[32], s_fbc[3];
        SolverScalars L = sc_ldcg(&a.h->sc);
        if (!L.done) {
            const K1Pro P = bicg_k1_prologue(L);
            double sg[1];
            fold_published<1>(a.part + kPartK1, __ldcg(&a.h->npart[0]), 1, s_fsh, s_fbc, sg);
            bicg_k1_tail(L, P, sg[0]);
        }
        if (blockIdx.x == 0 && tid == 0) a.h->sc2 = L;   // read by K3
        if (L.done || L.skip) return;
        alpha = L.alpha;
    } else if (MODE == SM_K1 || MODE == SM_K2) {
        SolverScalars &Sc = a.h->sc;
        if (Sc.done) return;
        if (MODE == SM_K2 && Sc.skip) return;
        if (MODE == SM_K1) {
            P1 = bicg_k1_prologue(Sc);           // DESIGN.md §3.6 restart / breakdown decision
            if (P1.breakdown) {
                if (blockIdx.x == 0 && tid == 0) bicg_breakdown(Sc);
                return;
            }
            rst = P1.rst;
            beta = P1.beta;
            omega = P1.omega;
        } else {
            alpha = Sc.alpha;
        }
    }

    constexpr int ND = C::NDOT > 0 ? C::NDOT : 1;
    Acc acc[ND][C::CPT];   // one accumulator per dot and owned cell: independent TwoSum chains
#pragma unroll
    for (int d = 0; d < ND; d++)
#pragma unroll
        for (int m = 0; m < C::CPT; m++) acc[d][m].zero();

    if (warp == C::NW) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < C::NH; q++) prefetch_map(&M.halo[q]);
            Cursor prod;
            prod.init(blockIdx.x, a, ntiles, TX, TY);
            int q = 0;
            for (; prod.valid; q++) {
                if (q >= S) mbar_wait(&empty[q % S], (uint32_t)(((q / S) - 1) & 1));
                issue<MODE, SYM, TX, TY, CPT_, S>(M, prod, a.nz, stages, full, q, a.work ? meta : nullptr);
                prod.advance(a.nz);
            }
            if (a.work) post_end(full, empty, meta, S, q);
        }
    } else {
        // ------------------------------------------------ consumer warps
        // CPT = 1: thread owns cell (tid % TX, tid / TX); CPT = 2: the x-adjacent
        // pair (2 (tid % (TX/2)), tid / (TX/2)), read and written as double2.
        constexpr int CPT = C::CPT;
        constexpr int RW = TX / CPT;                 // threads per tile row
        Cursor cons;
        cons.init(blockIdx.x, a, ntiles, TX, TY, false);
        double czq1[CPT], czq0[CPT];                 // cz at planes q-1 (aT of output) and q-2 (aB)
#pragma unroll
        for (int m = 0; m < CPT; m++) { czq1[m] = 0.0; czq0[m] = 0.0; }
        // SYM: what step 2 of plane q-1 needs from that plane's stage -- c_x at
        // x-1..x+CPT, c_y at y-1 and y, the extra field (b | r^ or r) -- is
        // copied to registers at the end of iteration q-1, so the stage is
        // released one plane earlier (prefetch depth S-1 instead of S-2).
        double kxw[CPT + 1], kys[CPT], kyn[CPT], kex[CPT];
#pragma unroll
        for (int m = 0; m < CPT; m++) { kxw[m] = 0.0; kys[m] = 0.0; kyn[m] = 0.0; kex[m] = 0.0; }
        kxw[CPT] = 0.0;
        // non-SYM: the seven coefficients of the owned cells, carried the same way
        double kc[7][CPT];
#pragma unroll
        for (int c7 = 0; c7 < 7; c7++)
#pragma unroll
            for (int m = 0; m < CPT; m++) kc[c7][m] = 0.0;
        const int cx0 = (tid % RW) * CPT, cy = tid / RW;
        const int ci = cy * TX + cx0;                // cell-box index of the first owned cell
        const int hc = (cy + 1) * C::HX + (cx0 + 2); // halo-box index of the first owned cell
        for (int q = 0; cons.valid; q++) {
            const int s = q % S;
            mbar_wait(&full[s], (uint32_t)((q / S) & 1));
            if (cons.pending) {   // dynamic units: the stage names the unit (or the end)
                const int um = meta[s];
                if (um < 0) break;
                cons.set_unit(um, a.nz);
            }
            const bool virt = cons.is_virtual(a.nz);
            const bool produce = cons.produces();
            const int kout = cons.k - 1;
            const int x0 = cons.x0, y0 = cons.y0;
            const uint8_t *st = stages + (size_t)s * C::STAGE_B;
            double *P = pbuf + (size_t)(q & 3) * (C::PBUF_B / 8);

            // step 1: value on the halo'd plane, PPI pairs of x-adjacent cells per
            // item.  PPI = 2 when one pair per thread would need a second, mostly
            // idle pass over the plane (K2 at 64x8 tiles, 2 cells per thread: 340
            // pairs for 256 threads); all loads of an item are issued first.
            constexpr int NPAIR = C::HX * C::HY / 2;
            constexpr int PPI = (NPAIR > C::NT && NPAIR % 2 == 0) ? 2 : 1;
            for (int it = tid; it < NPAIR / PPI; it += C::NT) {
                double2 val[PPI];
                if (!virt) {
                    const double2 *h0 = (const double2 *)(st + C::OFF_HALO);
                    double2 rv[PPI], pv[PPI], vv[PPI];
#pragma unroll
                    for (int u = 0; u < PPI; u++) {
                        const int pi = it * PPI + u;
                        rv[u] = h0[pi];
                        if (MODE == SM_K1) {
                            pv[u] = ((const double2 *)(st + C::OFF_HALO + C::HALO_B))[pi];
                            vv[u] = ((const double2 *)(st + C::OFF_HALO + 2 * C::HALO_B))[pi];
                        } else if (MODE == SM_K2) {
                            vv[u] = ((const double2 *)(st + C::OFF_HALO + C::HALO_B))[pi];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < PPI; u++) {
                        if (MODE == SM_SPMV || MODE == SM_SETUP) {
                            val[u] = rv[u];
                        } else if (MODE == SM_K1) {
                            if (rst) {
                                val[u].x = fma(beta, fma(-omega, 0.0, 0.0), rv[u].x);
                                val[u].y = fma(beta, fma(-omega, 0.0, 0.0), rv[u].y);
                            } else {
                                val[u].x = fma(beta, fma(-omega, vv[u].x, pv[u].x), rv[u].x);
                                val[u].y = fma(beta, fma(-omega, vv[u].y, pv[u].y), rv[u].y);
                            }
                        } else {
                            val[u].x = fma(-alpha, vv[u].x, rv[u].x);
                            val[u].y = fma(-alpha, vv[u].y, rv[u].y);
                        }
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < PPI; u++) val[u] = make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < PPI; u++) ((double2 *)P)[it * PPI + u] = val[u];
            }
            double czcur[CPT];
            if (CPT == 2 && SYM && !virt) {
                const double2 z2 = *(const double2 *)((const double *)(st + C::OFF_CELL) + ci);
                czcur[0] = z2.x; czcur[CPT - 1] = z2.y;
            } else {
#pragma unroll
                for (int m = 0; m < CPT; m++)
                    czcur[m] = (SYM && !virt) ? ((const double *)(st + C::OFF_CELL))[ci + m] : 0.0;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(C::NT) : "memory");

            // step 2: output plane kout = k(q) - 1 (stage of plane q-1)
            if (produce) {
                const uint8_t *so = stages + (size_t)((q + S - 1) % S) * C::STAGE_B;
                const double *Pc = pbuf + (size_t)((q + 3) & 3) * (C::PBUF_B / 8);   // plane q-1
                const double *Pb = pbuf + (size_t)((q + 2) & 3) * (C::PBUF_B / 8);   // plane q-2
                const double *Pt = P;                                                // plane q
                const int gx = x0 + cx0, gy = y0 + cy;
                const bool active = gx < a.nx && gy < a.ny;   // nx even: a pair is all in or all out
                double aP[CPT], aW[CPT], aE[CPT], aS[CPT], aN[CPT], aB[CPT], aT[CPT];
                double xc[CPT], xW[CPT], xE[CPT], xS[CPT], xN[CPT], xB[CPT], xT[CPT];
                if (CPT == 2) {
                    const double2 c2 = *(const double2 *)&Pc[hc];
                    const double2 s2 = *(const double2 *)&Pc[hc - C::HX];
                    const double2 n2 = *(const double2 *)&Pc[hc + C::HX];
                    const double2 b2 = *(const double2 *)&Pb[hc];
                    const double2 t2 = *(const double2 *)&Pt[hc];
                    xc[0] = c2.x; xc[CPT - 1] = c2.y;
                    xW[0] = Pc[hc - 1]; xW[CPT - 1] = c2.x;
                    xE[0] = c2.y; xE[CPT - 1] = Pc[hc + 2];
                    xS[0] = s2.x; xS[CPT - 1] = s2.y;
                    xN[0] = n2.x; xN[CPT - 1] = n2.y;
                    xB[0] = b2.x; xB[CPT - 1] = b2.y;
                    xT[0] = t2.x; xT[CPT - 1] = t2.y;
                } else {
                    xc[0] = Pc[hc]; xW[0] = Pc[hc - 1]; xE[0] = Pc[hc + 1];
                    xS[0] = Pc[hc - C::HX]; xN[0] = Pc[hc + C::HX]; xB[0] = Pb[hc]; xT[0] = Pt[hc];
                }
                if (CPT == 2) {
                    if (SYM) {
                        aW[0] = kxw[0]; aE[0] = kxw[1];
                        aW[CPT - 1] = kxw[1]; aE[CPT - 1] = kxw[CPT];
                        aS[0] = kys[0]; aS[CPT - 1] = kys[CPT - 1];
                        aN[0] = kyn[0]; aN[CPT - 1] = kyn[CPT - 1];
                        aB[0] = czq0[0]; aB[CPT - 1] = czq0[CPT - 1];
                        aT[0] = czq1[0]; aT[CPT - 1] = czq1[CPT - 1];
                    } else {
#pragma unroll
                        for (int m = 0; m < CPT; m++) {
                            aP[m] = kc[0][m]; aW[m] = kc[1][m]; aE[m] = kc[2][m]; aS[m] = kc[3][m];
                            aN[m] = kc[4][m]; aB[m] = kc[5][m]; aT[m] = kc[6][m];
                        }
                    }
                } else
#pragma unroll
                for (int m = 0; m < CPT; m++) {
                    if (SYM) {
                        aW[m] = kxw[m];
                        aE[m] = kxw[m + 1];
                        aS[m] = kys[m];
                        aN[m] = kyn[m];
                        aB[m] = czq0[m];
                        aT[m] = czq1[m];
                    } else {
                        aP[m] = kc[0][m]; aW[m] = kc[1][m]; aE[m] = kc[2][m]; aS[m] = kc[3][m];
                        aN[m] = kc[4][m]; aB[m] = kc[5][m]; aT[m] = kc[6][m];
                    }
                }
                // p': the diagonal is the row sum of the face coefficients (DESIGN.md
                // §3.4), rebuilt in the assembly's order instead of streamed (8 B/cell)
                if (SYM)
#pragma unroll
                    for (int m = 0; m < CPT; m++) aP[m] = ((((aW[m] + aE[m]) + aS[m]) + aN[m]) + aB[m]) + aT[m];
                double y[CPT];
#pragma unroll
                for (int m = 0; m < CPT; m++) {
                    double t = aP[m] * xc[m];
                    t = fma(-aW[m], xW[m], t);
                    t = fma(-aE[m], xE[m], t);
                    t = fma(-aS[m], xS[m], t);
                    t = fma(-aN[m], xN[m], t);
                    t = fma(-aB[m], xB[m], t);
                    t = fma(-aT[m], xT[m], t);
                    y[m] = t;
                }
                if (active) {
                    const long long n = (long long)gx + (long long)a.nx * ((long long)gy + (long long)a.ny * kout);
                    if (MODE == SM_SPMV) {
                        store_cells<CPT>(a.out0 + n, y);
                    } else if (MODE == SM_SETUP) {
                        const double *bb = (const double *)(so + C::OFF_EXTRA) + ci;
                        double rv[CPT];
#pragma unroll
                        for (int m = 0; m < CPT; m++) {
                            const double bm = kex[m];
                            rv[m] = bm - y[m];
                            acc[0][m].prod(bm, bm);
                            acc[ND > 1 ? 1 : 0][m].prod(rv[m], rv[m]);
                        }
                        store_cells<CPT>(a.out0 + n, rv);
                    } else if (MODE == SM_K1) {
                        store_cells<CPT>(a.out0 + n, xc);   // p_new
                        store_cells<CPT>(a.out1 + n, y);    // v_new
                        double rhv[CPT];
#pragma unroll
                        for (int m = 0; m < CPT; m++)
                            rhv[m] = kex[m];                                           // r^ (or r on a restart)
                        if (rst) store_cells<CPT>(a.out2 + n, rhv);
#pragma unroll
                        for (int m = 0; m < CPT; m++) acc[0][m].prod(rhv[m], y[m]);
                    } else {
                        store_cells<CPT>(a.out0 + n, y);    // t
#pragma unroll
                        for (int m = 0; m < CPT; m++) {
                            acc[0][m].prod(y[m], xc[m]);
                            acc[ND > 1 ? 1 : 0][m].prod(y[m], y[m]);
                            acc[ND > 2 ? 2 : 0][m].prod(xc[m], xc[m]);
                        }
                    }
                }
            }
            // plane q's step-2 inputs -> registers (SYM: c_x at x-1..x+CPT, c_y at y-1
            // and y; else the seven coefficients of the owned cells; both: the
            // extra field b | r^ (r on a restart)), then the stage goes back to the
            // producer: nothing of stage q is read after this point, so the ring
            // prefetches S-1 planes ahead instead of S-2
            if (!virt) {
                if (SYM) {
                    const double *xw = (const double *)(st + C::OFF_XW);
                    const double *ys = (const double *)(st + C::OFF_YS);
#pragma unroll
                    for (int m = 0; m <= CPT; m++) kxw[m] = xw[cy * C::HX + cx0 + m + 1];
#pragma unroll
                    for (int m = 0; m < CPT; m++) {
                        kys[m] = ys[cy * TX + cx0 + m];
                        kyn[m] = ys[(cy + 1) * TX + cx0 + m];
                    }
                } else {
                    const double *cell = (const double *)(st + C::OFF_CELL);
#pragma unroll
                    for (int c7 = 0; c7 < 7; c7++)
#pragma unroll
                        for (int m = 0; m < CPT; m++) kc[c7][m] = cell[c7 * (C::CELL_B / 8) + ci + m];
                }
#pragma unroll
                for (int m = 0; m < CPT; m++) {
                    if (MODE == SM_SETUP) kex[m] = ((const double *)(st + C::OFF_EXTRA))[ci + m];
                    if (MODE == SM_K1)
                        kex[m] = rst ? ((const double *)(st + C::OFF_HALO))[hc + m]
                                     : ((const double *)(st + C::OFF_EXTRA))[ci + m];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
            for (int m = 0; m < CPT; m++) { czq0[m] = czq1[m]; czq1[m] = czcur[m]; }
            cons.advance(a.nz, false);
        }
    }

    if constexpr (C::NDOT > 0) {
        __shared__ dd sh[(C::NW + 1) * ND];
        dd v[ND], out[ND];
#pragma unroll
        for (int d = 0; d < ND; d++) {
            v[d] = acc[d][0].get();
#pragma unroll
            for (int m = 1; m < C::CPT; m++) v[d] = dd_add(v[d], acc[d][m].get());
        }
        if ((MODE == SM_K1 || MODE == SM_K2) && a.chain) {   // the next kernel folds them
            publish_partials<ND>(v, a.part + (MODE == SM_K1 ? kPartK1 : kPartK2), &a.h->npart[MODE == SM_K1 ? 0 : 1],
                                 sh);
            return;
        }
        if (!grid_reduce_dd<ND>(v, a.part, &a.h->ticket[1], sh, out) || tid != 0) return;
        if (a.work) *a.work = 0u;   // every CTA has passed the ticket: all units were taken
        if (a.rank_part) {
#pragma unroll
            for (int d = 0; d < ND; d++) a.rank_part[d] = out[d];
            return;
        }
        SolverScalars &Sc = a.h->sc;
        if (MODE == SM_SETUP) bicg_setup(Sc, dd_round(out[0]), dd_round(out[1]), a.tol, a.maxit);
        else if (MODE == SM_K1) bicg_k1_tail(Sc, P1, dd_round(out[0]));
        else if (MODE == SM_K2) bicg_k2_tail(Sc, dd_round(out[0]), dd_round(out[1]), dd_round(out[2]));
    }
}

// ------------------------------------------------------------------ row-warp kernels
// Symmetric (p') systems, DESIGN.md §7 "row-warp": the tile is (32 CPT) x 8
// cells and consumer warp w owns tile row w (lane l: cells 2l, 2l+1 for
// CPT = 2).  Everything step 2 needs from the halo'd plane -- the value
// (x | p | s) on rows y-1, y, y+1 and the two x-edge cells -- the warp
// computes itself from the staged halo arrays; W/E neighbours inside the row
// travel by shuffles and z neighbours stay in registers (planes q-2, q-1, q).
// Warps therefore never wait on each other (no P ring, no per-plane named
// barrier) and a warp hands its stage back as soon as its loads are in
// registers.  The expressions and their order are those of k_stencil, so the
// bits are the same (tested against the oracle on every p' path).
// TMA producer of a row-warp pass (lane 0 of the producer warp)
template <int MODE, int CPT, int S, int STRIDE>
__device__ __forceinline__ void rw_produce(const TmaMaps &M, const StencilArgs &a, uint8_t *stages, uint64_t *full,
                                           uint64_t *empty, int &q, int *meta = nullptr)
{
    constexpr int TX = 32 * CPT, TY = 8;
    Cursor prod;
    prod.init(blockIdx.x, a, a.tiles_x * a.tiles_y, TX, TY);
    for (; prod.valid; q++) {
        if (q >= S) mbar_wait(&empty[q % S], (uint32_t)(((q / S) - 1) & 1));
        issue<MODE, true, TX, TY, CPT, S, STRIDE>(M, prod, a.nz, stages, full, q, a.work ? meta : nullptr);
        prod.advance(a.nz);
    }
    if (a.work) post_end(full, empty, meta, S, q++);
}

// consumer warps of a row-warp pass (MODE) over this CTA's units; q is the
// ring position shared with rw_produce, carried across passes of a persistent
// kernel; stage slots are STRIDE bytes apart.  acc[d][m]: dot d, owned cell m.
template <int MODE, int CPT, int S, int STRIDE, bool ONEACC = false>
__device__ __forceinline__ void rw_consume(const StencilArgs &a, double alpha, double beta, double omega, bool rst,
                                           Acc (&acc)[3][CPT], const uint8_t *stages, uint64_t *full,
                                           uint64_t *empty, int &q, const int *meta = nullptr)
{
    constexpr int TX = 32 * CPT, TY = 8;
    using C = Cfg<MODE, true, TX, TY, CPT>;
    constexpr int ND = C::NDOT > 0 ? C::NDOT : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Cursor cons;
    cons.init(blockIdx.x, a, a.tiles_x * a.tiles_y, TX, TY, false);
    const int cx0 = lane * CPT;
    const int hc = (warp + 1) * C::HX + cx0 + 2;                    // halo-box index of the first owned cell
    const int he = lane == 31 ? (warp + 1) * C::HX + TX + 2          // right edge cell x0 + TX
                              : (warp + 1) * C::HX + 1;              // left edge cell x0 - 1 (used by lane 0)
    const int ci = warp * TX + cx0;
    // register pipeline: values of planes q-2 (B), q-1 (centre row + S/N rows + edge), q (T)
    double vB[CPT], vC[CPT], vS[CPT], vN[CPT], vE = 0.0;
    double kxw[CPT + 1], kys[CPT], kyn[CPT], kex[CPT], czp[CPT], czpp[CPT];
#pragma unroll
    for (int m = 0; m < CPT; m++) {
        vB[m] = vC[m] = vS[m] = vN[m] = 0.0;
        kys[m] = kyn[m] = kex[m] = czp[m] = czpp[m] = 0.0;
    }
#pragma unroll
    for (int m = 0; m <= CPT; m++) kxw[m] = 0.0;

    // value of the step-1 field at halo index i (CPT consecutive cells from i)
    auto value = [&](const uint8_t *st, int i, double (&out)[CPT]) {
        const double *h0 = (const double *)(st + C::OFF_HALO);
        const double *h1 = (const double *)(st + C::OFF_HALO + C::HALO_B);
        const double *h2 = (const double *)(st + C::OFF_HALO + 2 * C::HALO_B);
        double rv[CPT], pv[CPT], vv[CPT];
        if (CPT == 2) {
            const double2 r2 = *(const double2 *)(h0 + i);
            rv[0] = r2.x; rv[CPT - 1] = r2.y;
            if (MODE == SM_K1) {
                const double2 p2 = *(const double2 *)(h1 + i), v2 = *(const double2 *)(h2 + i);
                pv[0] = p2.x; pv[CPT - 1] = p2.y; vv[0] = v2.x; vv[CPT - 1] = v2.y;
            } else if (MODE == SM_K2) {
                const double2 v2 = *(const double2 *)(h1 + i);
                vv[0] = v2.x; vv[CPT - 1] = v2.y;
            }
        } else {
            rv[0] = h0[i];
            if (MODE == SM_K1) { pv[0] = h1[i]; vv[0] = h2[i]; }
            else if (MODE == SM_K2) vv[0] = h1[i];
        }
#pragma unroll
        for (int m = 0; m < CPT; m++) {
            if (MODE == SM_SPMV || MODE == SM_SETUP) out[m] = rv[m];
            else if (MODE == SM_K1) out[m] = rst ? fma(beta, fma(-omega, 0.0, 0.0), rv[m])
                                                 : fma(beta, fma(-omega, vv[m], pv[m]), rv[m]);
            else out[m] = fma(-alpha, vv[m], rv[m]);
        }
    };
    auto value1 = [&](const uint8_t *st, int i) -> double {
        const double r = ((const double *)(st + C::OFF_HALO))[i];
        if (MODE == SM_K1) {
            const double p = ((const double *)(st + C::OFF_HALO + C::HALO_B))[i];
            const double v = ((const double *)(st + C::OFF_HALO + 2 * C::HALO_B))[i];
            return rst ? fma(beta, fma(-omega, 0.0, 0.0), r) : fma(beta, fma(-omega, v, p), r);
        }
        if (MODE == SM_K2) return fma(-alpha, ((const double *)(st + C::OFF_HALO + C::HALO_B))[i], r);
        return r;
    };

    for (; cons.valid; q++) {
        const int s = q % S;
        mbar_wait(&full[s], (uint32_t)((q / S) & 1));
        if (cons.pending) {   // dynamic units: the stage names the unit (or the end)
            const int um = meta[s];
            if (um < 0) { q++; break; }
            cons.set_unit(um, a.nz);
        }
        const bool virt = cons.is_virtual(a.nz);
        const bool produce = cons.produces();
        const int kout = cons.k - 1;
        const uint8_t *st = stages + (size_t)s * STRIDE;
        // ---- centre row of plane q (T of the output plane, B of the next)
        double tC[CPT];
        if (!virt) value(st, hc, tC);
        else
#pragma unroll
            for (int m = 0; m < CPT; m++) tC[m] = 0.0;
        if (MODE == SM_K1 && a.ghost_store && !virt && (cons.k == a.kbeg - 1 || cons.k == a.kend)) {
            const int gx = cons.x0 + cx0, gy = cons.y0 + warp;
            if (gx < a.nx && gy < a.ny)
                store_cells<CPT>(a.out0 + (long long)gx + (long long)a.nx * ((long long)gy + (long long)a.ny * cons.k),
                                 tC);
        }
        // ---- step 2: output plane q-1
        if (produce) {
            double xc[CPT], xW[CPT], xE[CPT], xS[CPT], xN[CPT], xB[CPT], xT[CPT];
            const double left = __shfl_up_sync(0xffffffffu, vC[CPT - 1], 1);
            const double right = __shfl_down_sync(0xffffffffu, vC[0], 1);
#pragma unroll
            for (int m = 0; m < CPT; m++) {
                xc[m] = vC[m];
                xW[m] = m > 0 ? vC[m - 1] : (lane == 0 ? vE : left);
                xE[m] = m < CPT - 1 ? vC[m + 1] : (lane == 31 ? vE : right);
                xS[m] = vS[m]; xN[m] = vN[m]; xB[m] = vB[m]; xT[m] = tC[m];
            }
            double y[CPT];
#pragma unroll
            for (int m = 0; m < CPT; m++) {
                const double aW = kxw[m], aE = kxw[m + 1], aS = kys[m], aN = kyn[m], aB = czpp[m], aT = czp[m];
                const double aP = ((((aW + aE) + aS) + aN) + aB) + aT;
                double t = aP * xc[m];
                t = fma(-aW, xW[m], t);
                t = fma(-aE, xE[m], t);
                t = fma(-aS, xS[m], t);
                t = fma(-aN, xN[m], t);
                t = fma(-aB, xB[m], t);
                t = fma(-aT, xT[m], t);
                y[m] = t;
            }
            const int gx = cons.x0 + cx0, gy = cons.y0 + warp;
            if (gx < a.nx && gy < a.ny) {
                const long long n = (long long)gx + (long long)a.nx * ((long long)gy + (long long)a.ny * kout);
                if (MODE == SM_SPMV) {
                    store_cells<CPT>(a.out0 + n, y);
                } else if (MODE == SM_SETUP) {
                    double rv[CPT];
#pragma unroll
                    for (int m = 0; m < CPT; m++) {
                        rv[m] = kex[m] - y[m];
                        acc[0][ONEACC ? 0 : m].prod(kex[m], kex[m]);
                        acc[ND > 1 ? 1 : 0][ONEACC ? 0 : m].prod(rv[m], rv[m]);
                    }
                    store_cells<CPT>(a.out0 + n, rv);
                } else if (MODE == SM_K1) {
                    store_cells<CPT>(a.out0 + n, xc);
                    store_cells<CPT>(a.out1 + n, y);
                    if (rst) store_cells<CPT>(a.out2 + n, kex);
#pragma unroll
                    for (int m = 0; m < CPT; m++) acc[0][ONEACC ? 0 : m].prod(kex[m], y[m]);
                } else {
                    store_cells<CPT>(a.out0 + n, y);
#pragma unroll
                    for (int m = 0; m < CPT; m++) {
                        acc[0][ONEACC ? 0 : m].prod(y[m], xc[m]);
                        acc[ND > 1 ? 1 : 0][ONEACC ? 0 : m].prod(y[m], y[m]);
                        acc[ND > 2 ? 2 : 0][ONEACC ? 0 : m].prod(xc[m], xc[m]);
                    }
                }
            }
        }
        // ---- the rest of plane q -> registers, then the stage goes back to the producer
        double tS[CPT], tN[CPT], tE = 0.0;
        double nkxw[CPT + 1], nkys[CPT], nkyn[CPT], nkex[CPT], ncz[CPT];
        if (!virt) {
            value(st, hc - C::HX, tS);
            value(st, hc + C::HX, tN);
            tE = value1(st, he);
            const double *xw = (const double *)(st + C::OFF_XW);
            const double *ys = (const double *)(st + C::OFF_YS);
            const double *cz = (const double *)(st + C::OFF_CELL);
#pragma unroll
            for (int m = 0; m <= CPT; m++) nkxw[m] = xw[warp * C::HX + cx0 + m + 1];
#pragma unroll
            for (int m = 0; m < CPT; m++) {
                nkys[m] = ys[warp * TX + cx0 + m];
                nkyn[m] = ys[(warp + 1) * TX + cx0 + m];
                ncz[m] = cz[ci + m];
                if (MODE == SM_SETUP) nkex[m] = ((const double *)(st + C::OFF_EXTRA))[ci + m];
                else if (MODE == SM_K1)
                    nkex[m] = rst ? ((const double *)(st + C::OFF_HALO))[hc + m]
                                  : ((const double *)(st + C::OFF_EXTRA))[ci + m];
                else nkex[m] = 0.0;
            }
        } else {
#pragma unroll
            for (int m = 0; m < CPT; m++) tS[m] = tN[m] = nkys[m] = nkyn[m] = nkex[m] = ncz[m] = 0.0;
#pragma unroll
            for (int m = 0; m <= CPT; m++) nkxw[m] = 0.0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);

        // ---- rotate the register pipeline
#pragma unroll
        for (int m = 0; m < CPT; m++) {
            vB[m] = vC[m]; vC[m] = tC[m]; vS[m] = tS[m]; vN[m] = tN[m];
            czpp[m] = czp[m]; czp[m] = ncz[m];
            kys[m] = nkys[m]; kyn[m] = nkyn[m]; kex[m] = nkex[m];
        }
#pragma unroll
        for (int m = 0; m <= CPT; m++) kxw[m] = nkxw[m];
        vE = tE;
        cons.advance(a.nz, false);
    }
}

template <int MODE, int CPT, int S, int MB>
__global__ void __launch_bounds__(8 * 32 + 32, MB) k_stencil_rw(const __grid_constant__ TmaMaps M, StencilArgs a)
{
    constexpr int TX = 32 * CPT, TY = 8;
    using C = Cfg<MODE, true, TX, TY, CPT>;
    static_assert(C::NW == TY, "one consumer warp per tile row");
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *stages = smem;
    uint64_t *full = (uint64_t *)(smem + (size_t)S * C::STAGE_B);
    uint64_t *empty = full + S;
    int *meta = (int *)(empty + S);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    pdl_trigger();
    if (tid == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    ktrace(a, 0);

    double beta = 0.0, omega = 0.0, alpha = 0.0;
    bool rst = false;
    K1Pro P1;
    P1.rst = false;
    if (MODE == SM_K2 && a.chain) {
        // chained: K1's scalar tail runs here, in every CTA (identical bits):
        // fold K1's published <r^, v> partials, apply it to the state K1 read
        __shared__ dd s_fsh[32], s_fbc[3];
        SolverScalars L = sc_ldcg(&a.h->sc);
        if (!L.done) {
            const K1Pro P = bicg_k1_prologue(L);
            double sg[1];
            fold_published<1>(a.part + kPartK1, __ldcg(&a.h->npart[0]), 1, s_fsh, s_fbc, sg);
            bicg_k1_tail(L, P, sg[0]);
        }
        if (blockIdx.x == 0 && tid == 0) a.h->sc2 = L;   // read by K3
        if (L.done || L.skip) return;
        alpha = L.alpha;
    } else if (MODE == SM_K1 || MODE == SM_K2) {
        SolverScalars &Sc = a.h->sc;
        if (Sc.done) return;
        if (MODE == SM_K2 && Sc.skip) return;
        if (MODE == SM_K1) {
            P1 = bicg_k1_prologue(Sc);
            if (P1.breakdown) {
                if (blockIdx.x == 0 && tid == 0) bicg_breakdown(Sc);
                return;
            }
            rst = P1.rst;
            beta = P1.beta;
            omega = P1.omega;
        } else {
            alpha = Sc.alpha;
        }
    }

    constexpr int ND = C::NDOT > 0 ? C::NDOT : 1;
    Acc acc[3][CPT];
#pragma unroll
    for (int d = 0; d < 3; d++)
#pragma unroll
        for (int m = 0; m < CPT; m++) acc[d][m].zero();

    int q = 0;
    if (warp == C::NW) {
        if (lane == 0) {
#pragma unroll
            for (int h = 0; h < C::NH; h++) prefetch_map(&M.halo[h]);
            rw_produce<MODE, CPT, S, C::STAGE_B>(M, a, stages, full, empty, q, meta);
        }
    } else {
        // MB = 3 CTAs per SM: one accumulator per dot (registers)
        rw_consume<MODE, CPT, S, C::STAGE_B, (MB >= 3)>(a, alpha, beta, omega, rst, acc, stages, full, empty, q, meta);
    }

    ktrace(a, 1);
    if constexpr (C::NDOT > 0) {
        __shared__ dd sh[(C::NW + 1) * ND];
        dd v[ND], out[ND];
#pragma unroll
        for (int d = 0; d < ND; d++) {
            v[d] = acc[d][0].get();
#pragma unroll
            for (int m = 1; m < CPT; m++) v[d] = dd_add(v[d], acc[d][m].get());
        }
        if ((MODE == SM_K1 || MODE == SM_K2) && a.chain) {   // the next kernel folds them
            publish_partials<ND>(v, a.part + (MODE == SM_K1 ? kPartK1 : kPartK2), &a.h->npart[MODE == SM_K1 ? 0 : 1],
                                 sh);
            return;
        }
        const bool last = grid_reduce_dd<ND>(v, a.part, &a.h->ticket[1], sh, out);
        ktrace(a, last ? 3 : 2);
        if (!last || tid != 0) return;
        if (a.work) *a.work = 0u;   // every CTA has passed the ticket: all units were taken
        if (a.rank_part) {
#pragma unroll
            for (int d = 0; d < ND; d++) a.rank_part[d] = out[d];
            return;
        }
        SolverScalars &Sc = a.h->sc;
        if (MODE == SM_SETUP) bicg_setup(Sc, dd_round(out[0]), dd_round(out[1]), a.tol, a.maxit);
        else if (MODE == SM_K1) bicg_k1_tail(Sc, P1, dd_round(out[0]));
        else if (MODE == SM_K2) bicg_k2_tail(Sc, dd_round(out[0]), dd_round(out[1]), dd_round(out[2]));
    }
}

// ------------------------------------------------------------------ persistent row-warp solver
// The whole BiCGSTAB loop for a symmetric (p') system in ONE cooperative
// launch (solver path 5; DESIGN.md §7 "persistent"): per iteration the
// row-warp K1 and K2 passes (TMA ring carried across passes) and a K3 pass
// over the CTA's own cells, separated by grid all-reduces.  Every CTA posts its
// double-double partials, one arrival counter orders the phase, and then every
// CTA folds all partials in the same fixed order and runs the scalar step of
// §3.6 itself (identical bits in every CTA), so a phase boundary costs one
// atomic arrival and one wait instead of a kernel drain, a launch and a
// pipeline refill.  Same expressions, correctly rounded dots: the iterates
// equal the other paths' bitwise.
struct PersistArgs {
    TmaMaps M1[2], M2[2];          // K1 / K2 maps for iteration parity 0 / 1 (ping-pong p, v)
    StencilArgs a1[2], a2[2];
    double *x, *r, *rh, *p[2], *v[2], *t;
    WsHeader *h;
    dd *part;                      // 2 x gridDim.x x 3 (double-buffered by phase parity)
    unsigned *arrive;              // monotone arrival counter, zero at launch
    int maxit;
    unsigned long long *trace;     // optional (MFX_PERSIST_TRACE): %globaltimer stamps of CTA 0, 8 per iteration
};

__device__ __forceinline__ void ptrace(const PersistArgs &P, int it, int slot)
{
    if (kTrace && P.trace && threadIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (blockIdx.x == 0) P.trace[it * 16 + slot] = t;
        // every CTA: iteration 5's stamps + SM id (load balance across CTAs)
        if (it == 5) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            P.trace[1024 + blockIdx.x * 16 + slot] = t;
            P.trace[1024 + blockIdx.x * 16 + 15] = sm;
        }
    }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// all-reduce of K double-doubles over the grid; out valid in thread 0
template <int K, int CPT>
__device__ __forceinline__ void grid_allreduce(const Acc (&acc)[3][CPT], dd *part, unsigned *arrive, unsigned &phase,
                                               dd *sh, dd (&out)[K], const PersistArgs &P, int it, int slot)
{
    dd v[K];
#pragma unroll
    for (int d = 0; d < K; d++) {
        v[d] = acc[d][0].get();
#pragma unroll
        for (int m = 1; m < CPT; m++) v[d] = dd_add(v[d], acc[d][m].get());
    }
    // this thread's generic stores vs the next passes' TMA (async-proxy) reads; K2's
    // output t is read back only by generic loads (K3), so it needs none
    if (K != 3) asm volatile("fence.proxy.async.global;" ::: "memory");
    (void)sh;
    block_reduce_lazy<K>(v);   // (syncs the CTA: every store precedes the arrival)
    dd *pb = part + (size_t)(phase & 1) * gridDim.x * 3;
    ptrace(P, it, slot);        // every warp of the CTA done with the pass
    if (threadIdx.x == 0) {
#pragma unroll
        for (int d = 0; d < K; d++) pb[(size_t)blockIdx.x * 3 + d] = v[d];
        __threadfence();
        atomicAdd(arrive, 1u);
        const unsigned target = (phase + 1) * gridDim.x;
        if (ld_acquire_u32(arrive) < target) {
            unsigned long long t0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            while (ld_acquire_u32(arrive) < target) {
                __nanosleep(40);   // back off: ~300 spinning CTAs on one L2 line delay the arrivals
                unsigned long long t1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                if (t1 - t0 > 20000000000ull) __trap();   // 20 s: a CTA is missing (never expected)
            }
        }
    }
    phase++;
    ptrace(P, it, slot + 1);    // released
    __syncthreads();
    block_fold_partials<K>(pb, gridDim.x, 3, out);   // out valid in thread 0
}

// Cluster-hierarchical all-reduce (CLP > 1 CTAs per cluster; DESIGN.md §7
// "persistent"): per value a lane butterfly, warp 0 folds the CTA's warp
// partials and pushes the CTA partial into the cluster leader's shared memory
// (st.async + the leader's mbarrier); the leader folds its CLP partials,
// publishes one partial per cluster and is the only CTA to arrive on the
// global counter and spin; after the release it folds the NC cluster
// partials in cluster order and pushes the result into every member's shared
// memory (st.async + the member's mbarrier).  Every CTA gets the same bits.
// Buffer reuse needs no barrier: a member pushes reduction j+1 only after it
// received result j, which the leader sends after consuming partials j; a
// leader publishes j+2 into the global double buffer only after release j+1,
// i.e. after every leader has read the partials of j.
struct ClRed {
    dd (*wsh)[16];          // [3][16] warp partials (slots >= NW stay zero)
    dd (*lred)[3][16];      // [2][3][CLP] leader: pushed CTA partials
    dd (*res)[3];           // [2][3] result (pushed by the leader; written locally in the leader)
    uint64_t *mb;           // [4]: leader receive [0..1], member receive [2..3]
    uint32_t dst_l;         // warp 0 lane 0: address of lred[0][0][rank] in the leader
    uint32_t bar_l;         // ... and of the leader's mb[0]
    uint32_t dst_m, bar_m;  // leader lane j < CLP: res[0][0] and mb[2] of member j
    uint32_t ph = 0;        // per-buffer phase bits: bit b = leader receive b, bit 2+b = member receive b
};

template <int K, int CPT, int CLP>
__device__ __forceinline__ void cluster_allreduce(const Acc (&acc)[3][CPT], dd *cpart, unsigned *arrive,
                                                  unsigned &phase, ClRed &R, dd (&out)[K], const PersistArgs &P,
                                                  int it, int slot)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = (int)cl_rank();
    const int b = (int)(phase & 1);
    if (tid == 0) {
        if (rank == 0) mbar_arrive_expect_tx(&R.mb[b], (uint32_t)(CLP * K * 16));
        else mbar_arrive_expect_tx(&R.mb[2 + b], (uint32_t)(K * 16));
    }
    dd v[K];
#pragma unroll
    for (int d = 0; d < K; d++) {
        v[d] = acc[d][0].get();
#pragma unroll
        for (int m = 1; m < CPT; m++) v[d] = dd_add(v[d], acc[d][m].get());
    }
    if (K != 3) asm volatile("fence.proxy.async.global;" ::: "memory");
    butterfly_k<K, 32>(v);
    if (lane == 0)
#pragma unroll
        for (int d = 0; d < K; d++) R.wsh[d][warp] = v[d];
    __syncthreads();   // every store of the pass precedes the CTA's partial
    ptrace(P, it, slot);
    if (warp == 0) {
        dd y[K];
#pragma unroll
        for (int d = 0; d < K; d++) y[d] = R.wsh[d][lane & 15];
        butterfly_k<K, 16>(y);
        if (lane == 0) {
            __threadfence();   // this CTA's global stores before the leader's publication
#pragma unroll
            for (int d = 0; d < K; d++) push_f64x2(R.dst_l + (uint32_t)((b * 3 + d) * 16 * 16), y[d].hi, y[d].lo, R.bar_l + 8u * b);
        }
    }
    if (rank == 0) {
        if (warp == 0) {
            mbar_wait_cluster(&R.mb[b], (R.ph >> b) & 1u);
            dd y[K];
#pragma unroll
            for (int d = 0; d < K; d++) y[d] = R.lred[b][d][lane & (CLP - 1)];
            butterfly_k<K, CLP>(y);
            const int nc = gridDim.x / CLP, me = blockIdx.x / CLP;
            dd *pb = cpart + (size_t)b * nc * 3;
            if (lane == 0) {
#pragma unroll
                for (int d = 0; d < K; d++) pb[(size_t)me * 3 + d] = y[d];
                __threadfence();
                atomicAdd(arrive, 1u);
                const unsigned target = (phase + 1) * (unsigned)nc;
                if (ld_acquire_u32(arrive) < target) {
                    unsigned long long t0;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                    while (ld_acquire_u32(arrive) < target) {
                        __nanosleep(20);
                        unsigned long long t1;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                        if (t1 - t0 > 20000000000ull) __trap();   // 20 s: a cluster is missing (never expected)
                    }
                }
            }
            __syncwarp();
            ptrace(P, it, slot + 1);
            dd f[K];
#pragma unroll
            for (int d = 0; d < K; d++) f[d] = dd{0.0, 0.0};
            for (int c = lane; c < nc; c += 32) {
#pragma unroll
                for (int d = 0; d < K; d++) {
                    dd x;
                    x.hi = __ldcg(&pb[(size_t)c * 3 + d].hi);
                    x.lo = __ldcg(&pb[(size_t)c * 3 + d].lo);
                    f[d] = dd_add(f[d], x);
                }
            }
            butterfly_k<K, 32>(f);
            if (lane == 0)
#pragma unroll
                for (int d = 0; d < K; d++) R.res[b][d] = f[d];
            if (lane >= 1 && lane < CLP)
#pragma unroll
                for (int d = 0; d < K; d++)
                    push_f64x2(R.dst_m + (uint32_t)((b * 3 + d) * 16), f[d].hi, f[d].lo, R.bar_m + 8u * b);
        }
        R.ph ^= 1u << b;
        __syncthreads();
    } else {
        mbar_wait_cluster(&R.mb[2 + b], (R.ph >> (2 + b)) & 1u);
        R.ph ^= 1u << (2 + b);
        ptrace(P, it, slot + 1);
    }
    phase++;
#pragma unroll
    for (int d = 0; d < K; d++) out[d] = R.res[b][d];
}

template <int CPT, int S, int CLP>
__global__ void __launch_bounds__(8 * 32 + 32, 2) k_bicg_rw(const __grid_constant__ PersistArgs P)
{
    constexpr int TX = 32 * CPT, TY = 8;
    using C1 = Cfg<SM_K1, true, TX, TY, CPT>;
    using C2 = Cfg<SM_K2, true, TX, TY, CPT>;
    constexpr int STRIDE = C1::STAGE_B > C2::STAGE_B ? C1::STAGE_B : C2::STAGE_B;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *stages = smem;
    uint64_t *full = (uint64_t *)(smem + (size_t)S * STRIDE);
    uint64_t *empty = full + S;
    __shared__ SolverScalars Ls;
    __shared__ dd sh[(C1::NW + 1) * 3];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // cluster all-reduce state (CLP > 1)
    constexpr int CLS = CLP > 1 ? CLP : 1;
    __shared__ __align__(16) dd c_wsh[3][16];
    __shared__ __align__(16) dd c_lred[2][3][16];
    __shared__ __align__(16) dd c_res[2][3];
    __shared__ __align__(8) uint64_t c_mb[4];
    ClRed R;
    if constexpr (CLP > 1) {
        static_assert(CLP <= 16 && (CLP & (CLP - 1)) == 0, "cluster size: a power of two <= 16");
        static_assert(C1::NW + 1 <= 16, "warp partial slots");
        if (tid < 3 * 16) c_wsh[tid / 16][tid % 16] = dd{0.0, 0.0};
        if (tid == 0)
            for (int q = 0; q < 4; q++) mbar_init(&c_mb[q], 1);
        const uint32_t rank = cl_rank();
        R.wsh = c_wsh; R.lred = c_lred; R.res = c_res; R.mb = c_mb;
        R.dst_l = mapa_u32(smem_u32(&c_lred[0][0][rank]), 0);
        R.bar_l = mapa_u32(smem_u32(&c_mb[0]), 0);
        R.dst_m = mapa_u32(smem_u32(&c_res[0][0]), (uint32_t)(lane % CLS));
        R.bar_m = mapa_u32(smem_u32(&c_mb[2]), (uint32_t)(lane % CLS));
    }
    if (tid == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C1::NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        Ls = P.h->sc;
    }
    __syncthreads();
    if constexpr (CLP > 1) cluster_sync_full();   // every member's mbarriers initialised before any push
    const bool producer = warp == C1::NW;
    int q = 0;
    unsigned phase = 0;
    const long long units = P.a1[0].units;
    const int ntiles = P.a1[0].tiles_x * P.a1[0].tiles_y;
    Acc acc[3][CPT];
    for (int it = 0; it <= P.maxit; it++) {
        if (Ls.done) break;
        const K1Pro P1 = bicg_k1_prologue(Ls);
        if (P1.breakdown) {
            __syncthreads();
            if (tid == 0) bicg_breakdown(Ls);
            break;
        }
        const int par = it & 1;
        dd out[3];
        ptrace(P, it, 0);
        // ---- K1: p = r + beta (p - omega v) on the halo'd planes, v = A p, <r^, v>
#pragma unroll
        for (int d = 0; d < 3; d++)
#pragma unroll
            for (int m = 0; m < CPT; m++) acc[d][m].zero();
        if (producer) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                rw_produce<SM_K1, CPT, S, STRIDE>(P.M1[par], P.a1[par], stages, full, empty, q);
            }
        } else {
            rw_consume<SM_K1, CPT, S, STRIDE>(P.a1[par], 0.0, P1.beta, P1.omega, P1.rst, acc, stages, full, empty, q);
        }
        ptrace(P, it, 1);
        if constexpr (CLP > 1) cluster_allreduce<1, CPT, CLS>(acc, P.part, P.arrive, phase, R, (dd(&)[1])out, P, it, 2);
        else grid_allreduce<1, CPT>(acc, P.part, P.arrive, phase, sh, (dd(&)[1])out, P, it, 2);
        ptrace(P, it, 4);
        if (tid == 0) bicg_k1_tail(Ls, P1, dd_round(out[0]));
        __syncthreads();
        if (Ls.done || Ls.skip) continue;
        // ---- K2: s = r - alpha v, t = A s, <t,s>, <t,t>, <s,s>
        const double alpha = Ls.alpha;
#pragma unroll
        for (int d = 0; d < 3; d++)
#pragma unroll
            for (int m = 0; m < CPT; m++) acc[d][m].zero();
        if (producer) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                rw_produce<SM_K2, CPT, S, STRIDE>(P.M2[par], P.a2[par], stages, full, empty, q);
            }
        } else {
            rw_consume<SM_K2, CPT, S, STRIDE>(P.a2[par], alpha, 0.0, 0.0, false, acc, stages, full, empty, q);
        }
        ptrace(P, it, 5);
        if constexpr (CLP > 1) cluster_allreduce<3, CPT, CLS>(acc, P.part, P.arrive, phase, R, out, P, it, 6);
        else grid_allreduce<3, CPT>(acc, P.part, P.arrive, phase, sh, out, P, it, 6);
        ptrace(P, it, 8);
        if (tid == 0) bicg_k2_tail(Ls, dd_round(out[0]), dd_round(out[1]), dd_round(out[2]));
        __syncthreads();
        if (Ls.done || Ls.skip) continue;
        // ---- K3 over this CTA's own cells (the units of K1/K2, so every value it
        // reads was written by this CTA): x, r update, <r^, r>, <r, r>
        const bool half = Ls.half != 0;
        const double al = Ls.alpha, om = Ls.omega;
#pragma unroll
        for (int d = 0; d < 3; d++)
#pragma unroll
            for (int m = 0; m < CPT; m++) acc[d][m].zero();
        if (!producer) {
            const StencilArgs &a = P.a1[par];
            const double *pn = P.p[par ^ 1], *vn = P.v[par ^ 1];
            for (long long u = blockIdx.x; u < units; u += gridDim.x) {
                const int chunk = (int)(u / ntiles), tile = (int)(u - (long long)chunk * ntiles);
                const int ty = tile / a.tiles_x;
                const int gx = (tile - ty * a.tiles_x) * TX + lane * CPT, gy = ty * TY + warp;
                if (gx >= a.nx || gy >= a.ny) continue;
                const int k0 = a.kbeg + chunk * a.Lz, k1 = k0 + a.Lz < a.kend ? k0 + a.Lz : a.kend;
                const long long pl = (long long)a.nx * a.ny;
                const long long e0 = (long long)gx + (long long)a.nx * gy;
                // KU planes per step, every load of the step issued before any use
#ifndef MFX_PK3_KU
#define MFX_PK3_KU 1
#endif
                constexpr int KU = MFX_PK3_KU;
                for (int kb = k0; kb < k1; kb += KU) {
                    double xv[KU][CPT], rv[KU][CPT], rhv[KU][CPT], pv[KU][CPT], vv[KU][CPT], tv[KU][CPT];
#pragma unroll
                    for (int j = 0; j < KU; j++) {
                        if (kb + j >= k1) continue;
                        const long long e = e0 + pl * (kb + j);
                        if (CPT == 2) {
                            auto ld2 = [&](const double *b_, double (&o)[CPT]) {
                                const double2 w = __ldcg((const double2 *)(b_ + e));
                                o[0] = w.x; o[CPT - 1] = w.y;
                            };
                            ld2(P.x, xv[j]); ld2(P.r, rv[j]); ld2(P.rh, rhv[j]); ld2(pn, pv[j]); ld2(vn, vv[j]);
                            if (!half) ld2(P.t, tv[j]);
                            else tv[j][0] = tv[j][CPT - 1] = 0.0;
                        } else {
                            xv[j][0] = __ldcg(P.x + e); rv[j][0] = __ldcg(P.r + e); rhv[j][0] = __ldcg(P.rh + e);
                            pv[j][0] = __ldcg(pn + e); vv[j][0] = __ldcg(vn + e); tv[j][0] = half ? 0.0 : __ldcg(P.t + e);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < KU; j++) {
                        if (kb + j >= k1) continue;
                        const long long e = e0 + pl * (kb + j);
#pragma unroll
                        for (int m = 0; m < CPT; m++) {
                            const double sv = fma(-al, vv[j][m], rv[j][m]);
                            double xo, ro;
                            if (half) {
                                xo = fma(al, pv[j][m], xv[j][m]);
                                ro = sv;
                            } else {
                                xo = fma(om, sv, fma(al, pv[j][m], xv[j][m]));
                                ro = fma(-om, tv[j][m], sv);
                            }
                            xv[j][m] = xo;
                            rv[j][m] = ro;
                            acc[0][m].prod(rhv[j][m], ro);
                            acc[1][m].prod(ro, ro);
                        }
                        store_cells<CPT>(P.x + e, xv[j]);
                        store_cells<CPT>(P.r + e, rv[j]);
                    }
                }
            }
        }
        ptrace(P, it, 9);
        if constexpr (CLP > 1) cluster_allreduce<2, CPT, CLS>(acc, P.part, P.arrive, phase, R, (dd(&)[2])out, P, it, 10);
        else grid_allreduce<2, CPT>(acc, P.part, P.arrive, phase, sh, (dd(&)[2])out, P, it, 10);
        ptrace(P, it, 12);
        if (tid == 0) bicg_k3_tail(Ls, half, dd_round(out[0]), dd_round(out[1]));
        __syncthreads();
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) P.h->sc = Ls;
    if constexpr (CLP > 1) cluster_sync_full();   // no CTA exits while a push into it may be in flight
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encode()
{
    if (g_encode) return true;
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return false;
    }
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    return true;
}

bool make_map(CUtensorMap *m, const double *ptr, int nx, int ny, int nz, int bx, int by)
{
    if (!ptr) { memset(m, 0, sizeof(*m)); return true; }
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t strides[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)ptr, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) for box %dx%d", (int)r, bx, by);
        return false;
    }
    return true;
}

// z-chunk length: minimise rounds * (Lz + 2) (the +2 boundary planes of a
// chunk are L2 hits, counted as full planes to stay conservative);
// MFX_LZ overrides for tuning.
int choose_lz(long long ntiles, int nz, int grid)
{
    static int env = -2;
    if (env == -2) {
        const char *e = getenv("MFX_LZ");
        env = e ? atoi(e) : -1;
    }
    if (env > 0) return env < nz ? env : nz;
    int best = nz;
    double best_cost = 1e300;
    for (int lz = 4; lz <= nz; lz++) {
        const long long units = ntiles * ((nz + lz - 1) / lz);
        const long long rounds = (units + grid - 1) / grid;
        const double cost = (double)rounds * (lz + 2);
        if (cost < best_cost - 1e-9) { best_cost = cost; best = lz; }
    }
    return best;
}

template <int MODE, bool SYM, int TX, int TY, int CPT_, int S, bool RW = false, int MB = 2>
struct Launcher {
    using C = Cfg<MODE, SYM, TX, TY, CPT_>;
    static constexpr void (*kern)(const TmaMaps, StencilArgs) =
        RW ? k_stencil_rw<MODE, CPT_, S, MB> : k_stencil<MODE, SYM, TX, TY, CPT_, S>;
    static constexpr size_t smem() { return RW ? (size_t)S * C::STAGE_B + 24 * (size_t)S : smem_bytes<C>(S); }
    static int grid_size()
    {
        static int g = 0;
        if (g) return g;
        const size_t sm = smem();
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT + 32, sm);
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g = sms * (occ > 0 ? occ : 1);
        if (g > kMaxBlocks) g = kMaxBlocks;
        return g;
    }
    static mfx_status run(const Geo &G, const double *const halo[3], const double *const coef[7], const double *extra,
                          const StencilArgs &args0, cudaStream_t s)
    {
        if (!get_encode()) return MFX_ERR_CUDA;
        TmaMaps M;
        memset(&M, 0, sizeof(M));
        for (int q = 0; q < C::NH; q++)
            if (!make_map(&M.halo[q], halo[q], G.nx, G.ny, G.nz, C::HX, C::HY)) return MFX_ERR_CUDA;
        for (int q = 0; q < C::NCELLC; q++)
            if (!make_map(&M.coef[q], coef[q], G.nx, G.ny, G.nz, TX, TY)) return MFX_ERR_CUDA;
        if (SYM) {
            if (!make_map(&M.coef[2], coef[2], G.nx, G.ny, G.nz, C::HX, TY)) return MFX_ERR_CUDA;
            if (!make_map(&M.coef[3], coef[3], G.nx, G.ny, G.nz, TX, TY + 1)) return MFX_ERR_CUDA;
        }
        if (C::NE && !make_map(&M.extra, extra, G.nx, G.ny, G.nz, TX, TY)) return MFX_ERR_CUDA;
        StencilArgs a = args0;
        a.nx = G.nx; a.ny = G.ny; a.nz = G.nz;
        a.tiles_x = (G.nx + TX - 1) / TX;
        a.tiles_y = (G.ny + TY - 1) / TY;
        int grid = grid_size();
        const long long ntiles = (long long)a.tiles_x * a.tiles_y;
        if (a.kend <= a.kbeg) { a.kbeg = 0; a.kend = G.nz; }
        // dynamic units (MFX_DYN=1; off: measured no gain at c2, finer units cost halo planes)
        // (the dot kernels only: their last CTA resets the counter)
        static const int dyn = env_int("MFX_DYN", 0);
        a.work = (dyn && C::NDOT > 0 && a.h) ? &a.h->work[0] : nullptr;
        const int nout = a.kend - a.kbeg;
        a.Lz = choose_lz(ntiles, nout, grid);
        a.units = ntiles * ((nout + a.Lz - 1) / a.Lz);
        if (grid > a.units) grid = (int)a.units;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(C::NT + 32);
        cfg.dynamicSmemBytes = smem();
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = opt_pdl() ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static const int tr = env_int("MFX_RW_TRACE", 0);
        static int traced = 0;
        if (kTrace && RW && tr && traced < 40) {
            MFX_CUDA_TRY(cudaMalloc(&a.trace, (size_t)grid * 4 * sizeof(unsigned long long)));
            MFX_CUDA_TRY(cudaMemsetAsync(a.trace, 0, (size_t)grid * 4 * sizeof(unsigned long long), s));
        }
        MFX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, M, a));
        if (a.trace) {
            traced++;
            std::vector<unsigned long long> h((size_t)grid * 4);
            MFX_CUDA_TRY(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, s));
            MFX_CUDA_TRY(cudaStreamSynchronize(s));
            cudaFree(a.trace);
            unsigned long long t0 = ~0ull, tend = 0, tlast = 0, tpass_max = 0;
            double pass_sum = 0, pass_min = 1e30, pass_max = 0;
            for (int b = 0; b < grid; b++) {
                const unsigned long long *c = &h[(size_t)b * 4];
                if (c[0] < t0) t0 = c[0];
                if (c[1] > tpass_max) tpass_max = c[1];
                const double d = 1e-3 * (double)(c[1] - c[0]);
                pass_sum += d; if (d < pass_min) pass_min = d; if (d > pass_max) pass_max = d;
                if (c[2] > tend) tend = c[2];
                if (c[3]) tlast = c[3];
            }
            if (traced > 3)
                fprintf(stderr, "rw trace mode %d: first start -> last pass end %.2f us; pass per CTA min %.2f mean %.2f "
                        "max %.2f us; last pass end -> last CTA folded %.2f us\n", MODE, 1e-3 * (double)(tpass_max - t0),
                        pass_min, pass_sum / grid, pass_max, tlast ? 1e-3 * (double)(tlast - tpass_max) : -1.0);
        }
        return MFX_OK;
    }
};

// MFX_TILE=32x8 / 64x4 and MFX_STAGES=3/4/6 override the defaults (tuning).

template <int MODE, bool SYM, int TX, int TY, int CPT_>
mfx_status run_tile(const Geo &G, const double *const halo[3], const double *const coef[7], const double *extra,
                    const StencilArgs &a, cudaStream_t s)
{
    static const int st = env_int("MFX_STAGES", 0);
    const int S = st ? st : ((TX * TY == 512 || (MODE == SM_K1 && !SYM)) ? 3 : 4);
    if (S == 3) return Launcher<MODE, SYM, TX, TY, CPT_, 3>::run(G, halo, coef, extra, a, s);
    if (S == 6) return Launcher<MODE, SYM, TX, TY, CPT_, 6>::run(G, halo, coef, extra, a, s);
    return Launcher<MODE, SYM, TX, TY, CPT_, 4>::run(G, halo, coef, extra, a, s);
}

// row-warp kernels (SYM only): MFX_RW = bit mask over modes (1 << MODE) that use
// them; MFX_RW_STAGES overrides their ring depth.
template <int MODE>
mfx_status run_rw(const Geo &G, const double *const halo[3], const double *const coef[7], const double *extra,
                  const StencilArgs &a, cudaStream_t s)
{
    static const int st = env_int("MFX_RW_STAGES", 0);
    static const int mb = env_int("MFX_RW_MB", 2);
    if (G.nx <= 32) {
        if ((st ? st : 4) == 3) return Launcher<MODE, true, 32, 8, 1, 3, true>::run(G, halo, coef, extra, a, s);
        return Launcher<MODE, true, 32, 8, 1, 4, true>::run(G, halo, coef, extra, a, s);
    }
    if (mb == 1) {   // one CTA per SM with a deep ring (prefetch depth S - 1)
        constexpr bool BIG = Cfg<MODE, true, 64, 8, 2>::STAGE_B > 25000;
        if (BIG) return Launcher<MODE, true, 64, 8, 2, 6, true, 1>::run(G, halo, coef, extra, a, s);
        return Launcher<MODE, true, 64, 8, 2, 8, true, 1>::run(G, halo, coef, extra, a, s);
    }
    if (mb == 3) {   // three CTAs per SM: stages must fit 227 KB / 3
        constexpr bool BIG = Cfg<MODE, true, 64, 8, 2>::STAGE_B > 25000;
        if (BIG || st == 2) return Launcher<MODE, true, 64, 8, 2, 2, true, 3>::run(G, halo, coef, extra, a, s);
        return Launcher<MODE, true, 64, 8, 2, 3, true, 3>::run(G, halo, coef, extra, a, s);
    }
    const int S = st ? st : 4;
    if (S == 3) return Launcher<MODE, true, 64, 8, 2, 3, true>::run(G, halo, coef, extra, a, s);
    return Launcher<MODE, true, 64, 8, 2, 4, true>::run(G, halo, coef, extra, a, s);
}

// default: the row-warp kernel for p' K2 only (B200, r02: K2 82 vs 84-86 us at
// c2, 23 vs 27 us at c3; the row-warp K1, apply and setup are not faster)
int rw_mask()
{
    static const int m = env_int("MFX_RW", 1 << SM_K2);
    return m;
}

template <int MODE, bool SYM>
mfx_status run_mode(const Geo &G, const double *const halo[3], const double *const coef[7], const double *extra,
                    const StencilArgs &a, cudaStream_t s)
{
    // tiles: 64x4 (one cell per thread) or 64x8 / 32x16 (x-adjacent pairs)
    if (SYM && ((rw_mask() >> MODE & 1) || a.rank_part)) return run_rw<MODE>(G, halo, coef, extra, a, s);
    static const int tile = env_int("MFX_TILE", 0);   // 1: 64x4, 2: 64x8 pairs, 3: 32x16 pairs, 4: 32x8, 5: 64x8
    int t = tile;
    // measured at c2 (profiles/r01s7_tile_sweep.log): p' K1 is fastest at 64x4,
    // everything else (p' K2, the 7-coefficient kernels) at 64x8 pairs
    if (!t) t = G.nx <= 32 ? (SYM ? 3 : 4) : ((MODE == SM_K1 && SYM) ? 1 : 2);
    if (t == 2) return run_tile<MODE, SYM, 64, 8, 2>(G, halo, coef, extra, a, s);
    if (t == 3) return run_tile<MODE, SYM, 32, 16, 2>(G, halo, coef, extra, a, s);
    if (t == 4) return run_tile<MODE, SYM, 32, 8, 1>(G, halo, coef, extra, a, s);
    if (t == 5) return run_tile<MODE, SYM, 64, 8, 1>(G, halo, coef, extra, a, s);
    return run_tile<MODE, SYM, 64, 4, 1>(G, halo, coef, extra, a, s);
}

template <int CPT, int S, int CLP>
struct PersistLauncher {
    static constexpr int TX = 32 * CPT, TY = 8;
    using C1 = Cfg<SM_K1, true, TX, TY, CPT>;
    using C2 = Cfg<SM_K2, true, TX, TY, CPT>;
    static constexpr int STRIDE = C1::STAGE_B > C2::STAGE_B ? C1::STAGE_B : C2::STAGE_B;
    static constexpr size_t smem() { return (size_t)S * STRIDE + 16 * (size_t)S; }
    // co-resident grid: SMs x CTAs per SM, or (CLP > 1) the clusters the
    // device can hold at once x CLP (0: a cluster of CLP cannot be placed)
    static int grid_size()
    {
        static int g = -1;
        if (g >= 0) return g;
        auto kfn = k_bicg_rw<CPT, S, CLP>;
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem());
        if (CLP > 1) {
            if (CLP > 8) cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CLP; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(CLP); cfg.blockDim = dim3(C1::NT + 32); cfg.dynamicSmemBytes = smem();
            cfg.attrs = at; cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, kfn, &cfg) != cudaSuccess) { cudaGetLastError(); nc = 0; }
            // the leaders' fold reads one partial per cluster per lane pass; keep it to <= 64 clusters
            if (nc > 64) nc = 64;
            g = nc * CLP;
            return g;
        }
        int occ = 0, dev = 0, sms = 148;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, C1::NT + 32, smem());
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g = sms * (occ > 0 ? occ : 1);
        if (g > kMaxBlocks / 2) g = kMaxBlocks / 2;
        return g;
    }
    static mfx_status run(const Geo &G, const mfx_eqsys *A, double *x, const WsView &W, int maxit, cudaStream_t s)
    {
        PersistArgs P;
        memset(&P, 0, sizeof(P));
        StencilArgs a;
        memset(&a, 0, sizeof(a));
        a.nx = G.nx; a.ny = G.ny; a.nz = G.nz;
        a.tiles_x = (G.nx + TX - 1) / TX;
        a.tiles_y = (G.ny + TY - 1) / TY;
        int grid = grid_size();
        const long long ntiles = (long long)a.tiles_x * a.tiles_y;
        a.kbeg = 0; a.kend = G.nz;
        a.Lz = choose_lz(ntiles, G.nz, grid);
        a.units = ntiles * ((G.nz + a.Lz - 1) / a.Lz);
        if (grid > a.units) grid = CLP > 1 ? (int)((a.units + CLP - 1) / CLP) * CLP : (int)a.units;
        a.h = W.hdr; a.part = W.part;
        for (int par = 0; par < 2; par++) {
            const double *h1[3] = {W.r, W.p[par], W.v[par]};
            const double *h2[2] = {W.r, W.v[par ^ 1]};
            for (int q = 0; q < 3; q++)
                if (!make_map(&P.M1[par].halo[q], h1[q], G.nx, G.ny, G.nz, C1::HX, C1::HY)) return MFX_ERR_CUDA;
            for (int q = 0; q < 2; q++)
                if (!make_map(&P.M2[par].halo[q], h2[q], G.nx, G.ny, G.nz, C2::HX, C2::HY)) return MFX_ERR_CUDA;
            TmaMaps *Ms[2] = {&P.M1[par], &P.M2[par]};
            for (TmaMaps *M : Ms) {
                if (!make_map(&M->coef[0], A->aT, G.nx, G.ny, G.nz, TX, TY) ||
                    !make_map(&M->coef[2], A->aE, G.nx, G.ny, G.nz, C1::HX, TY) ||
                    !make_map(&M->coef[3], A->aN, G.nx, G.ny, G.nz, TX, TY + 1))
                    return MFX_ERR_CUDA;
            }
            if (!make_map(&P.M1[par].extra, W.rh, G.nx, G.ny, G.nz, TX, TY)) return MFX_ERR_CUDA;
            P.a1[par] = a;
            P.a1[par].out0 = W.p[par ^ 1]; P.a1[par].out1 = W.v[par ^ 1]; P.a1[par].out2 = W.rh;
            P.a2[par] = a;
            P.a2[par].out0 = W.t;
        }
        P.x = x; P.r = W.r; P.rh = W.rh; P.t = W.t;
        P.p[0] = W.p[0]; P.p[1] = W.p[1]; P.v[0] = W.v[0]; P.v[1] = W.v[1];
        P.h = W.hdr; P.part = W.part; P.arrive = &W.hdr->ticket[2]; P.maxit = maxit;
        MFX_CUDA_TRY(cudaMemsetAsync(&W.hdr->ticket[2], 0, sizeof(unsigned), s));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(C1::NT + 32);
        cfg.dynamicSmemBytes = smem();
        cfg.stream = s;
        // co-residency: a cooperative launch for the flat grid; for clusters the
        // grid never exceeds what cudaOccupancyMaxActiveClusters reports
        cudaLaunchAttribute attr[1];
        if (CLP > 1) {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = CLP; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        } else {
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
        }
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static const int tr = env_int("MFX_PERSIST_TRACE", 0);
        const size_t trn = 1024 + (size_t)grid * 16;
        if (kTrace && tr) {
            MFX_CUDA_TRY(cudaMalloc(&P.trace, trn * sizeof(unsigned long long)));
            MFX_CUDA_TRY(cudaMemsetAsync(P.trace, 0, trn * sizeof(unsigned long long), s));
        }
        MFX_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_bicg_rw<CPT, S, CLP>, P));
        if (kTrace && tr) {
            static unsigned long long h[1024 + 16 * 2048];
            MFX_CUDA_TRY(cudaMemcpyAsync(h, P.trace, trn * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
            MFX_CUDA_TRY(cudaStreamSynchronize(s));
            cudaFree(P.trace);
            // slots: 0 K1 start | 1 warp0 K1 end, 2 CTA K1 end, 3 released, 4 folded | 5..8 K2 | 9..12 K3
            const char *nm[12] = {"K1 warp0", "K1 CTA tail", "K1 barrier", "K1 fold", "K2 warp0", "K2 CTA tail",
                                  "K2 barrier", "K2 fold", "K3 warp0", "K3 CTA tail", "K3 barrier", "K3 fold"};
            double acc[12] = {0};
            int n = 0;
            for (int it = 2; it < 63 && h[it * 16 + 12] && h[(it + 1) * 16]; it++, n++)
                for (int k = 0; k < 12; k++) acc[k] += 1e-3 * (double)(h[it * 16 + k + 1] - h[it * 16 + k]);
            if (n) {
                fprintf(stderr, "persist trace (CTA 0, %d iters, us; grid %d units %lld Lz %d):", n, grid, a.units, a.Lz);
                for (int k = 0; k < 12; k++) fprintf(stderr, " %s %.2f", nm[k], acc[k] / n);
                fprintf(stderr, "\n");
            }
            const unsigned long long *c = h + 1024;
            const int ps[3][3] = {{0, 2, 3}, {4, 6, 7}, {8, 10, 11}};   // pass start, CTA end, released
            for (int k = 0; k < 3; k++) {
                double mn = 1e30, mx = 0, sum = 0;
                unsigned long long amin = ~0ull, amax = 0;
                int slow = 0;
                for (int b = 0; b < grid; b++) {
                    const double d = 1e-3 * (double)(c[b * 16 + ps[k][1]] - c[b * 16 + ps[k][0]]);
                    if (d < mn) mn = d;
                    if (d > mx) { mx = d; slow = b; }
                    sum += d;
                    const unsigned long long ar = c[b * 16 + ps[k][1]];
                    if (ar < amin) amin = ar;
                    if (ar > amax) amax = ar;
                }
                fprintf(stderr, "  iter 5 K%d (pass start -> CTA done) over %d CTAs: min %.2f mean %.2f max %.2f us "
                        "(slowest CTA %d, SM %llu); arrival spread %.2f us\n", k + 1, grid, mn, sum / grid, mx, slow,
                        c[slow * 16 + 15], 1e-3 * (double)(amax - amin));
            }

        }
        return MFX_OK;
    }
};

}  // namespace

// solver path 5: the whole p' BiCGSTAB loop in one cooperative launch (after
// the setup kernel); symmetric systems, even nx, 16-byte aligned arrays.
mfx_status persist_solve_launch(const Geo &G, const mfx_eqsys *A, double *x, const WsView &W, int maxit,
                                cudaStream_t s)
{
    if (!get_encode()) return MFX_ERR_CUDA;
    // MFX_PERSIST_CL: CTAs per cluster of the hierarchical all-reduce (8 or 16;
    // default 1 = the flat grid all-reduce: B200, c3 51.6 us per iteration vs
    // 55.2 with clusters of 8 and 60.2 with 16 -- the two DSMEM hops cost more
    // than the shorter global fold saves)
    static const int clp = env_int("MFX_PERSIST_CL", 1);
    if (G.nx <= 32) {
        if (clp == 16 && PersistLauncher<1, 3, 16>::grid_size() > 0) return PersistLauncher<1, 3, 16>::run(G, A, x, W, maxit, s);
        if (clp >= 8 && PersistLauncher<1, 3, 8>::grid_size() > 0) return PersistLauncher<1, 3, 8>::run(G, A, x, W, maxit, s);
        return PersistLauncher<1, 3, 1>::run(G, A, x, W, maxit, s);
    }
    if (clp == 16 && PersistLauncher<2, 3, 16>::grid_size() > 0) return PersistLauncher<2, 3, 16>::run(G, A, x, W, maxit, s);
    if (clp >= 8 && PersistLauncher<2, 3, 8>::grid_size() > 0) return PersistLauncher<2, 3, 8>::run(G, A, x, W, maxit, s);
    return PersistLauncher<2, 3, 1>::run(G, A, x, W, maxit, s);
}



// coefficient order for the maps: SYM -> {cz, -, cx, cy}; else {aP, aW, aE, aS, aN, aB, aT}
mfx_status stencil_launch(int mode, bool sym, const Geo &G, const double *const halo[3],
                          const mfx_eqsys *A, const double *extra, double *o0, double *o1, double *o2,
                          WsHeader *h, dd *part, double tol, int maxit, cudaStream_t s, int reverse, int kbeg,
                          int kend, int ghost_store, dd *rank_part, int chain)
{
    const double *coef[7];
    if (sym) {
        coef[0] = A->aT; coef[1] = nullptr; coef[2] = A->aE; coef[3] = A->aN;
        coef[4] = coef[5] = coef[6] = nullptr;
    } else {
        coef[0] = A->aP; coef[1] = A->aW; coef[2] = A->aE; coef[3] = A->aS;
        coef[4] = A->aN; coef[5] = A->aB; coef[6] = A->aT;
    }
    StencilArgs a;
    memset(&a, 0, sizeof(a));
    a.out0 = o0; a.out1 = o1; a.out2 = o2; a.h = h; a.part = part; a.tol = tol; a.maxit = maxit;
    a.reverse = reverse;
    a.kbeg = kbeg; a.kend = kend; a.ghost_store = ghost_store; a.rank_part = rank_part;
    a.chain = chain && !rank_part && (mode == SM_K1 || mode == SM_K2);
    MFX_ARG_CHECK(!rank_part || sym, "slab mode: symmetric systems only");
    switch (mode * 2 + (sym ? 1 : 0)) {
    case SM_SPMV * 2 + 0: return run_mode<SM_SPMV, false>(G, halo, coef, extra, a, s);
    case SM_SPMV * 2 + 1: return run_mode<SM_SPMV, true>(G, halo, coef, extra, a, s);
    case SM_SETUP * 2 + 0: return run_mode<SM_SETUP, false>(G, halo, coef, extra, a, s);
    case SM_SETUP * 2 + 1: return run_mode<SM_SETUP, true>(G, halo, coef, extra, a, s);
    case SM_K1 * 2 + 0: return run_mode<SM_K1, false>(G, halo, coef, extra, a, s);
    case SM_K1 * 2 + 1: return run_mode<SM_K1, true>(G, halo, coef, extra, a, s);
    case SM_K2 * 2 + 0: return run_mode<SM_K2, false>(G, halo, coef, extra, a, s);
    case SM_K2 * 2 + 1: return run_mode<SM_K2, true>(G, halo, coef, extra, a, s);
    }
    set_error("bad stencil mode");
    return MFX_ERR_ARG;
}

bool tma_make_map(CUtensorMap *m, const double *ptr, int nx, int ny, int nz, int bx, int by)
{
    return get_encode() && make_map(m, ptr, nx, ny, nz, bx, by);
}

}  // namespace mfx
