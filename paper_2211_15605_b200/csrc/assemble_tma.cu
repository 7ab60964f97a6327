// assemble_tma.cu -- a-1 momentum assembly (Eq. 2,
// P:53) as a persistent TMA z-marching kernel for sm_100a.
//
// The row of a u/v/w face reads a 3x3x3 neighbourhood of four fields (eps and
// the three staggered velocities: face averages, transverse mass fluxes, the
// four-cell edge eps, the residual neighbours) and the P / E values of five
// pointwise fields (eps_old, c_old, p, beta, S_c).  A CTA owns a TX x TY tile
// of rows and marches along z: one producer warp streams each plane of the
// four stencil fields as (TX+4) x (TY+2) TMA boxes into an S-stage ring
// (full/empty mbarriers; out-of-domain parts zero-filled and never used -- the
// boundary rules select constants there), so every stencil value is read from
// HBM once and from shared memory 27 times; the pointwise fields are loaded
// straight from global memory (coalesced, issued before the stage wait).  The
// arithmetic is the grid-stride kernel's (assemble.cu), expression for
// expression, so both produce identical bits.  Work units are (z-chunk, tile)
// pairs dealt round-robin to a persistent grid, as in stencil_tma.cu.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tma.cuh"
#include "mom_row.cuh"

namespace mfx {

struct AsmMomArgs {
    MomRowPar R;                       // row constants (mom_row.cuh)
    int nx, ny, nz;
    int upwind;                        // face_eps_upwind
    int tiles_x, tiles_y, Lz;
    long long units;
    int bc_zlo, bc_zhi;
    double w_in, A[3], V;
    double rho, urf, gc, rVdt, Dc[3];
    const double *eps0, *uold, *p, *beta, *S;
    const unsigned char *blocked;      // NULL or N flags (BLOCKED cells)
    double *aP, *aE, *aW, *aN, *aS, *aT, *aB, *b, *d;
    double *resid2;
    WsHeader *hdr;
    dd *part;
};

struct AsmMomMaps {
    CUtensorMap f[4];   // eps, u, v, w
};

namespace {

constexpr int ATX = 32, ATY = 8;                 // tile: one row per consumer thread
constexpr int ANT = ATX * ATY;                   // 256 consumer threads
constexpr int ANW = ANT / 32;
constexpr int AHX = ATX + 4, AHY = ATY + 2;      // box x in [x0-2, x0+TX+2), y in [y0-1, y0+TY+1)
constexpr int ABOX = AHX * AHY;                  // doubles per field per plane
constexpr int ABOX_B = (ABOX * 8 + 127) & ~127;
constexpr int ASTAGE_B = 4 * ABOX_B;
constexpr int ASTAGE_TX = 4 * ABOX * 8;
constexpr int AS = 6;                            // stages: planes k-1, k, k+1 resident + 3 ahead

struct ACursor {
    int u, units, G, ntiles, Lz, tiles_x;
    int x0, y0, k, k0, k1;
    bool valid;
    __device__ void start(int nz)
    {
        if (u >= units) { valid = false; return; }
        const int chunk = u / ntiles;
        const int tile = u - chunk * ntiles;
        const int ty = tile / tiles_x;
        x0 = (tile - ty * tiles_x) * ATX;
        y0 = ty * ATY;
        k0 = chunk * Lz;
        k1 = k0 + Lz < nz ? k0 + Lz : nz;
        k = k0 - 1;
        valid = true;
    }
    __device__ void init(int u0, int nunits, int g, int nt, int lz, int tx, int nz)
    {
        u = u0; units = nunits; G = g; ntiles = nt; Lz = lz; tiles_x = tx;
        start(nz);
    }
    // a unit streams planes k0-1 .. k1 (virtual = not loaded outside [0, nz))
    __device__ void advance(int nz)
    {
        k++;
        if (k > k1) { u += G; start(nz); }
    }
};

// mom_row inputs read from the staged planes where the row uses them (the
// 3x3x3 neighbourhood of eps, u, v, w) plus the pointwise values in registers
template <int C>
struct SmemRowIn {
    static constexpr int T1 = C == 0 ? 1 : 0, T2 = C == 2 ? 1 : 2;
    int P[3];
    int type;
    bool m_wall, e_ident;
    bool nb_wall_[2][2];   // neighbour row (P + s e_t, E + s e_t) touches a BLOCKED cell (§3.10)
    double e0P, e0E, bP, bE, SP, SE, pP, pEv, uoP;
    const double *pl[3];   // planes k-1, k, k+1
    int hc, e[3], ext[3];
    __device__ double F(int f, int dx, int dy, int dz) const
    {
        return pl[dz + 1][f * (ABOX_B / 8) + hc + dy * AHX + dx];
    }
    __device__ double at(int f, const int o[3]) const { return F(f, o[0], o[1], o[2]); }
    __device__ void off(int ti, int sg, int o[3]) const
    {
        o[0] = o[1] = o[2] = 0;
        o[ti == 0 ? T1 : T2] = sg ? 1 : -1;
    }
    __device__ double epsP() const { return F(0, 0, 0, 0); }
    __device__ double epsE() const { return F(0, e[0], e[1], e[2]); }
    __device__ double epsPt(int ti, int sg) const { int o[3]; off(ti, sg, o); return at(0, o); }
    __device__ double epsEt(int ti, int sg) const
    {
        int o[3]; off(ti, sg, o);
        return F(0, e[0] + o[0], e[1] + o[1], e[2] + o[2]);
    }
    // velocity on the +t face of Q (s>0: Q = P, R = E; s<0: Q = P-e_t, R = E-e_t)
    __device__ double vP(int ti, int sg) const
    {
        const int t = ti == 0 ? T1 : T2;
        int o[3]; off(ti, sg, o);
        return sg ? F(1 + t, 0, 0, 0) : at(1 + t, o);
    }
    __device__ double vE(int ti, int sg) const
    {
        const int t = ti == 0 ? T1 : T2;
        int o[3]; off(ti, sg, o);
        return sg ? F(1 + t, e[0], e[1], e[2]) : F(1 + t, e[0] + o[0], e[1] + o[1], e[2] + o[2]);
    }
    __device__ double umP() const { return F(1 + C, 0, 0, 0); }
    __device__ double umE() const { return F(1 + C, e[0], e[1], e[2]); }
    __device__ double umM() const
    {
        int o[3] = {0, 0, 0};
        o[C] = -1;
        return at(1 + C, o);
    }
    __device__ double unb(int s6) const
    {
        int o[3] = {0, 0, 0};
        o[s6 / 2] = (s6 & 1) ? 1 : -1;
        const int qa = P[s6 / 2] + o[s6 / 2];
        return (qa >= 0 && qa < ext[s6 / 2]) ? at(1 + C, o) : 0.0;
    }
    __device__ bool nb_wall(int ti, int sg) const { return nb_wall_[ti][sg]; }
};

// §3.10: cell q is BLOCKED (outside the domain: not blocked); the flags are
// one byte per cell, read through the read-only path (L1/L2), not staged
__device__ __forceinline__ bool blk_tma(const AsmMomArgs &a, int i, int j, int k)
{
    if (i < 0 || j < 0 || k < 0 || i >= a.nx || j >= a.ny || k >= a.nz) return false;
    return __ldg(a.blocked + ((long long)i + (long long)a.nx * ((long long)j + (long long)a.ny * k))) != 0;
}

// BL: the grid has BLOCKED cells (the row rules of DESIGN.md §3.10, the same
// decisions as the grid-stride kernel's row_type / m_wall / e_ident / nb_wall)
template <int C, bool BL>
__global__ void __launch_bounds__(ANT + 32, 2) k_asm_mom_tma(const __grid_constant__ AsmMomMaps M, AsmMomArgs a)
{
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = (uint64_t *)(smem + (size_t)AS * ASTAGE_B);
    uint64_t *empty = full + AS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = a.tiles_x * a.tiles_y;
    if (tid == 0) {
        for (int s = 0; s < AS; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ANW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    Acc num, den;
    num.zero();
    den.zero();

    if (warp == ANW) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
            for (int f = 0; f < 4; f++) prefetch_map(&M.f[f]);
            ACursor c;
            c.init(blockIdx.x, (int)a.units, gridDim.x, ntiles, a.Lz, a.tiles_x, a.nz);
            for (int q = 0; c.valid; q++) {
                const int s = q % AS;
                if (q >= AS) mbar_wait(&empty[s], (uint32_t)(((q / AS) - 1) & 1));
                if (c.k < 0 || c.k >= a.nz) {
                    mbar_arrive(&full[s]);
                } else {
                    uint8_t *st = smem + (size_t)s * ASTAGE_B;
                    mbar_arrive_expect_tx(&full[s], ASTAGE_TX);
#pragma unroll
                    for (int f = 0; f < 4; f++) tma_load_3d(st + f * ABOX_B, &M.f[f], c.x0 - 2, c.y0 - 1, c.k, &full[s]);
                }
                c.advance(a.nz);
            }
        }
    } else {
        // ------------------------------------------------ consumer warps: one row (cell) per thread
        const int tx = tid % ATX, ty = tid / ATX;
        const int hc = (ty + 1) * AHX + (tx + 2);                  // box index of P
        const int ext[3] = {a.nx, a.ny, a.nz};
        const long long sz = (long long)a.nx * a.ny;
        ACursor c;
        c.init(blockIdx.x, (int)a.units, gridDim.x, ntiles, a.Lz, a.tiles_x, a.nz);
        int q = 0;   // sequence number of plane c.k (k0 - 1) of the current unit
        while (c.valid) {
            const int k0 = c.k0, k1 = c.k1, x0 = c.x0, y0 = c.y0;
            const int nplanes = k1 - k0 + 2;
            // planes k0-1 and k0 must be resident before the first row
            mbar_wait(&full[q % AS], (uint32_t)((q / AS) & 1));
            mbar_wait(&full[(q + 1) % AS], (uint32_t)(((q + 1) / AS) & 1));
            const int P0 = x0 + tx, P1 = y0 + ty;
            const bool mine = P0 < a.nx && P1 < a.ny;
            for (int k = k0; k < k1; k++) {
                const int qk = q + (k - k0) + 1;                     // sequence of plane k
                const int P[3] = {P0, P1, k};
                const long long n = (long long)P0 + (long long)a.nx * ((long long)P1 + (long long)a.ny * k);
                int type = 0;                                        // kInterior / kIdentity / kOutlet
                if (P[C] >= ext[C] - 1) type = (C == 2 && a.bc_zhi == MFX_BC_OUTLET) ? 2 : 1;
                if (BL && mine) {
                    // a blocked P, or an internal wall face (E = P + e_C blocked): identity row
                    int E[3] = {P[0], P[1], P[2]};
                    E[C] += 1;
                    if (blk_tma(a, P[0], P[1], P[2]) || (type == 0 && blk_tma(a, E[0], E[1], E[2]))) type = 1;
                }
                // pointwise fields at P and E (global, issued before the stage wait)
                const int oE = type == 0 ? 1 : 0;
                const long long nE = n + (type == 0 ? (C == 0 ? 1 : (C == 1 ? (long long)a.nx : sz)) : 0);
                double e0P = 0, e0E = 0, bP = 0, bE = 0, SP = 0, SE = 0, pP = 0, pEv = 0, uoP = 0;
                if (mine && type != 1) {
                    e0P = __ldg(a.eps0 + n); e0E = __ldg(a.eps0 + nE);
                    bP = __ldg(a.beta + n); bE = __ldg(a.beta + nE);
                    SP = __ldg(a.S + n); SE = __ldg(a.S + nE);
                    pP = __ldg(a.p + n); pEv = __ldg(a.p + nE);
                    uoP = __ldg(a.uold + n);
                }
                // plane k+1 resident (planes k-1, k already are)
                mbar_wait(&full[(qk + 1) % AS], (uint32_t)(((qk + 1) / AS) & 1));
                const double *pl[3] = {(const double *)(smem + (size_t)((qk - 1) % AS) * ASTAGE_B),
                                       (const double *)(smem + (size_t)(qk % AS) * ASTAGE_B),
                                       (const double *)(smem + (size_t)((qk + 1) % AS) * ASTAGE_B)};
                if (mine) {
                    if (type == 1) {
                        a.aP[n] = 1.0;
                        a.aE[n] = 0.0; a.aW[n] = 0.0; a.aN[n] = 0.0; a.aS[n] = 0.0; a.aT[n] = 0.0; a.aB[n] = 0.0;
                        a.b[n] = 0.0;
                        a.d[n] = 0.0;
                    } else {
                        SmemRowIn<C> in;
                        in.P[0] = P[0]; in.P[1] = P[1]; in.P[2] = P[2];
                        in.type = type;
                        in.e[0] = in.e[1] = in.e[2] = 0;
                        in.e[C] = oE;                                // E = P + e (E = P on the outlet row)
                        in.ext[0] = ext[0]; in.ext[1] = ext[1]; in.ext[2] = ext[2];
                        in.pl[0] = pl[0]; in.pl[1] = pl[1]; in.pl[2] = pl[2];
                        in.hc = hc;
                        in.e0P = e0P; in.e0E = e0E; in.bP = bP; in.bE = bE; in.SP = SP; in.SE = SE;
                        in.pP = pP; in.pEv = pEv; in.uoP = uoP;
                        in.m_wall = false;
                        // E is an identity row iff it is the last face along C and that face is a wall
                        in.e_ident = type != 2 && (P[C] + 1 >= ext[C] - 1) && !(C == 2 && a.bc_zhi == MFX_BC_OUTLET);
                        in.nb_wall_[0][0] = in.nb_wall_[0][1] = in.nb_wall_[1][0] = in.nb_wall_[1][1] = false;
                        if (BL) {
                            int E[3] = {P[0], P[1], P[2]};
                            E[C] += oE;
                            int Pm[3] = {P[0], P[1], P[2]};
                            Pm[C] -= 1;
                            in.m_wall = P[C] >= 1 && blk_tma(a, Pm[0], Pm[1], Pm[2]);
                            if (type != 2) {
                                // row_type(E): E itself blocked, or its own +e_C face a wall (§3.10)
                                int EE[3] = {E[0], E[1], E[2]};
                                EE[C] += 1;
                                const bool eb = blk_tma(a, E[0], E[1], E[2]);
                                in.e_ident = eb || (E[C] < ext[C] - 1 ? blk_tma(a, EE[0], EE[1], EE[2])
                                                                       : !(C == 2 && a.bc_zhi == MFX_BC_OUTLET));
                            }
#pragma unroll
                            for (int ti = 0; ti < 2; ti++) {
                                const int t = ti == 0 ? SmemRowIn<C>::T1 : SmemRowIn<C>::T2;
#pragma unroll
                                for (int sg = 0; sg < 2; sg++) {
                                    const int sgn = sg ? 1 : -1;
                                    int Pt[3] = {P[0], P[1], P[2]}, Et[3] = {E[0], E[1], E[2]};
                                    Pt[t] += sgn;
                                    Et[t] += sgn;
                                    const int pt = P[t] + sgn;
                                    in.nb_wall_[ti][sg] = pt >= 0 && pt < ext[t] &&
                                                          (blk_tma(a, Pt[0], Pt[1], Pt[2]) || blk_tma(a, Et[0], Et[1], Et[2]));
                                }
                            }
                        }
                        MomRowOut ro;
                        mom_row<C>(a.R, in, ro);
                        a.aW[n] = ro.st6[0]; a.aE[n] = ro.st6[1];
                        a.aS[n] = ro.st6[2]; a.aN[n] = ro.st6[3];
                        a.aB[n] = ro.st6[4]; a.aT[n] = ro.st6[5];
                        a.aP[n] = ro.aPr;
                        a.b[n] = ro.bR;
                        a.d[n] = ro.d;
                        const bool nonfin = !isfinite(ro.aPr) || !isfinite(ro.bR) || !isfinite(ro.d);
                        if (nonfin || ro.aPr == 0.0) {
                            if (nonfin) atomicMin(&a.hdr->bad_nonfinite, (unsigned long long)n);
                            else atomicMin(&a.hdr->bad_zerodiag, (unsigned long long)n);
                        }
                        num.add(ro.res);
                        den.add(ro.den);
                    }
                }
                // plane k-1 is no longer needed by this CTA
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[(qk - 1) % AS]);
            }
            // release planes k1-1 and k1 (sequence q + nplanes - 2, q + nplanes - 1)
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[(q + nplanes - 2) % AS]);
                mbar_arrive(&empty[(q + nplanes - 1) % AS]);
            }
            q += nplanes;
            c.u += c.G;
            c.start(a.nz);
        }
    }
    __shared__ dd sh[((ANT + 32) / 32) * 2];
    dd v[2] = {num.get(), den.get()}, out[2];
    if (grid_reduce_dd<2>(v, a.part, &a.hdr->ticket[0], sh, out) && threadIdx.x == 0 && a.resid2) {
        a.resid2[0] = dd_round(out[0]);
        a.resid2[1] = dd_round(out[1]);
    }
}

int asm_choose_lz(long long ntiles, int nz, int grid)
{
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

template <int C, bool BL>
int asm_grid()
{
    static int g = 0;
    if (g) return g;
    const size_t sm = (size_t)AS * ASTAGE_B + 16 * AS;
    cudaFuncSetAttribute(k_asm_mom_tma<C, BL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int occ = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_asm_mom_tma<C, BL>, ANT + 32, sm);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = sms * (occ > 0 ? occ : 1);
    return g;
}

template <int C, bool BL>
mfx_status launch_c(const AsmMomMaps &M, AsmMomArgs &a, cudaStream_t s)
{
    const int grid = asm_grid<C, BL>();
    const long long ntiles = (long long)a.tiles_x * a.tiles_y;
    a.Lz = asm_choose_lz(ntiles, a.nz, grid);
    a.units = ntiles * ((a.nz + a.Lz - 1) / a.Lz);
    const int g = (int)(a.units < grid ? a.units : grid);
    const size_t sm = (size_t)AS * ASTAGE_B + 16 * AS;
    k_asm_mom_tma<C, BL><<<g, ANT + 32, sm, s>>>(M, a);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

}  // namespace

// Called by assemble_eq (assemble.cu) for kinds U/V/W after argument checks.
mfx_status assemble_mom_tma(int kind, const Geo &G, const mfx_params *pr, const mfx_state *st, mfx_eqsys *out,
                            double *resid2, WsHeader *hdr, dd *part, cudaStream_t s)
{
    AsmMomMaps M;
    const double *f4[4] = {st->eps, st->u, st->v, st->w};
    for (int f = 0; f < 4; f++)
        if (!tma_make_map(&M.f[f], f4[f], G.nx, G.ny, G.nz, AHX, AHY)) return MFX_ERR_CUDA;
    AsmMomArgs a;
    memset(&a, 0, sizeof(a));
    a.nx = G.nx; a.ny = G.ny; a.nz = G.nz;
    a.upwind = pr->face_eps_upwind;
    a.R.ext[0] = G.nx; a.R.ext[1] = G.ny; a.R.ext[2] = G.nz;
    a.R.bc_zlo = G.bc_zlo; a.R.bc_zhi = G.bc_zhi; a.R.upwind = pr->face_eps_upwind;
    a.R.w_in = G.w_in; a.R.V = G.V;
    a.R.rho = pr->rho; a.R.urf = pr->urf_mom; a.R.gc = pr->g[kind]; a.R.rVdt = (pr->rho * G.V) / pr->dt;
    for (int t = 0; t < 3; t++) { a.R.A[t] = G.A[t]; a.R.Dc[t] = (pr->mu * G.A[t]) / G.h[t]; }
    a.tiles_x = (G.nx + ATX - 1) / ATX;
    a.tiles_y = (G.ny + ATY - 1) / ATY;
    a.bc_zlo = G.bc_zlo; a.bc_zhi = G.bc_zhi;
    a.w_in = G.w_in;
    for (int t = 0; t < 3; t++) { a.A[t] = G.A[t]; a.Dc[t] = (pr->mu * G.A[t]) / G.h[t]; }
    a.V = G.V;
    a.rho = pr->rho;
    a.urf = pr->urf_mom;
    a.gc = pr->g[kind];
    a.rVdt = (pr->rho * G.V) / pr->dt;
    a.eps0 = st->eps_old;
    a.uold = kind == 0 ? st->u_old : (kind == 1 ? st->v_old : st->w_old);
    a.S = kind == 0 ? st->sbeta_u : (kind == 1 ? st->sbeta_v : st->sbeta_w);
    a.p = st->p; a.beta = st->beta;
    a.aP = out->aP; a.aE = out->aE; a.aW = out->aW; a.aN = out->aN; a.aS = out->aS; a.aT = out->aT;
    a.aB = out->aB; a.b = out->b; a.d = out->d;
    a.resid2 = resid2; a.hdr = hdr; a.part = part;
    a.blocked = st->blocked;
    if (a.blocked) {
        if (kind == 0) return launch_c<0, true>(M, a, s);
        if (kind == 1) return launch_c<1, true>(M, a, s);
        return launch_c<2, true>(M, a, s);
    }
    if (kind == 0) return launch_c<0, false>(M, a, s);
    if (kind == 1) return launch_c<1, false>(M, a, s);
    return launch_c<2, false>(M, a, s);
}

}  // namespace mfx
