// pic.cu -- particle -> grid coupling on the PIC device (NEXT-2; DESIGN.md
// §3.9; "F is the interpolated force from the parcel location to
// the corresponding fluid cell", PAPER.md:97 explicit vs implicit refresh at
// the head of every SIMPLE iteration, PAPER.md:131 interpolation of eps_p).
//
// Two deposits produce the hot path's inputs:
//   k_pic_eps   parcel solid volume -> cell accumulators (trilinear weights),
//               then k_pic_eps_final: eps_g = max(1 - acc / V, eps_min);
//   k_pic_drag  per parcel: trilinear eps_g and staggered-lattice u_g at the
//               parcel, slip, Syamlal-O'Brien K; deposit W (K / V) into beta
//               and W ((K u_p) / V) into beta*u_s (no pass over the grid after).
//
// One thread per parcel, grid-stride over a fixed grid; the 8 node updates go
// to global memory as fp64 reductions (RED.ADD.F64, resolved in L2).  The
// fields the parcels touch (the bed) sit in L2 after the first parcels, so
// the gathers and the reductions are L2 traffic; HBM sees the parcel stream
// (56 B / parcel), the output fields and the zero fill.  Summation order
// inside a cell is the order the reductions arrive in: parity with the oracle
// (parcel-ascending order) is to the tolerance DESIGN.md §3.9 derives, not
// bitwise; per-parcel values (weights, interpolants) use the oracle's exact
// expression order and differ only through pow() (CUDA's vs libm's ulps).
#include <climits>
#include <cstring>

#include "common.cuh"

namespace mfx {

namespace {

constexpr int kPicThreads = 256;
constexpr double kPi = 3.14159265358979323846;

struct PicGeo {
    int n[3];
    double h[3], L[3];
    double V, Vs, eps_min;
    int bc_zlo;
    double w_in;
    long long N;
};

// stencil along one axis from the lattice coordinate xi (= x/h - 0.5 for cell
// centres, x/h - 1 for the face lattice)
__device__ __forceinline__ void pic_axis_xi(double xi, int n, bool face, int nd[2], double w[2])
{
    const double fl = floor(xi);
    const double f = xi - fl;
    int i0 = (int)fl, i1 = i0 + 1;
    const int lo = face ? -1 : 0;
    i0 = i0 < lo ? lo : (i0 > n - 1 ? n - 1 : i0);
    i1 = i1 < lo ? lo : (i1 > n - 1 ? n - 1 : i1);
    nd[0] = i0; nd[1] = i1;
    w[0] = 1.0 - f; w[1] = f;
}

__device__ __forceinline__ double pic_xi(double x, double h, bool face) { return face ? x / h - 1.0 : x / h - 0.5; }

__device__ __forceinline__ void pic_axis(double x, double h, int n, bool face, int nd[2], double w[2])
{
    pic_axis_xi(pic_xi(x, h, face), n, face, nd, w);
}

__device__ __forceinline__ long long pic_lin(const PicGeo &G, int i, int j, int k)
{
    return (long long)i + (long long)G.n[0] * ((long long)j + (long long)G.n[1] * k);
}

__device__ __forceinline__ bool parcel_ok(const PicGeo &G, double x, double y, double z, double om)
{
    return x >= 0.0 && x <= G.L[0] && y >= 0.0 && y <= G.L[1] && z >= 0.0 && z <= G.L[2] && om >= 0.0;
}

// trilinear value of field f on the lattice whose face axis is FA (-1: cell
// centres), from Q[a] = x_a / h_a (one IEEE quotient per axis shared by the
// four lattices: x/h - 0.5 and x/h - 1 are exactly pic_xi's expressions)
template <int FA>
__device__ __forceinline__ double pic_interp(const PicGeo &G, const double *__restrict__ f, const double Q[3])
{
    int nd[3][2];
    double w[3][2];
#pragma unroll
    for (int a = 0; a < 3; a++) pic_axis_xi(a == FA ? Q[a] - 1.0 : Q[a] - 0.5, G.n[a], a == FA, nd[a], w[a]);
    double v8[8];
#pragma unroll
    for (int kk = 0; kk < 2; kk++)
#pragma unroll
        for (int jj = 0; jj < 2; jj++)
#pragma unroll
            for (int ii = 0; ii < 2; ii++) {
                int q[3] = {nd[0][ii], nd[1][jj], nd[2][kk]};
                double v;
                if (FA >= 0 && q[FA] == -1) {
                    v = (FA == 2 && G.bc_zlo == MFX_BC_INLET) ? G.w_in : 0.0;
                } else {
                    v = __ldg(f + pic_lin(G, q[0], q[1], q[2]));
                }
                v8[(kk * 2 + jj) * 2 + ii] = v;
            }
    double val = 0.0;
#pragma unroll
    for (int kk = 0; kk < 2; kk++)
#pragma unroll
        for (int jj = 0; jj < 2; jj++)
#pragma unroll
            for (int ii = 0; ii < 2; ii++) {
                const double W = (w[0][ii] * w[1][jj]) * w[2][kk];
                val = val + W * v8[(kk * 2 + jj) * 2 + ii];
            }
    return val;
}

struct PicEpsArgs {
    PicGeo G;
    const double *x, *y, *z, *om;
    long long m;
    double *acc;
    WsHeader *hdr;
};

__global__ void __launch_bounds__(kPicThreads) k_pic_eps(PicEpsArgs a)
{
    const PicGeo &G = a.G;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < a.m;
         p += (long long)gridDim.x * blockDim.x) {
        const double X[3] = {__ldg(a.x + p), __ldg(a.y + p), __ldg(a.z + p)};
        const double om = __ldg(a.om + p);
        if (!parcel_ok(G, X[0], X[1], X[2], om)) {
            atomicMin(&a.hdr->bad_parcel, (unsigned long long)p);
            continue;
        }
        const double vol = om * G.Vs;
        int nd[3][2];
        double w[3][2];
#pragma unroll
        for (int ax = 0; ax < 3; ax++) pic_axis(X[ax], G.h[ax], G.n[ax], false, nd[ax], w[ax]);
#pragma unroll
        for (int kk = 0; kk < 2; kk++)
#pragma unroll
            for (int jj = 0; jj < 2; jj++)
#pragma unroll
                for (int ii = 0; ii < 2; ii++) {
                    const double W = (w[0][ii] * w[1][jj]) * w[2][kk];
                    atomicAdd(a.acc + pic_lin(G, nd[0][ii], nd[1][jj], nd[2][kk]), W * vol);
                }
    }
}

__global__ void __launch_bounds__(kPicThreads) k_pic_eps_final(double *eps, long long N, double V, double eps_min)
{
    if ((uintptr_t)eps & 15) {   // offset view: plain 8-byte accesses
        for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (long long)gridDim.x * blockDim.x) {
            const double e = 1.0 - eps[q] / V;
            eps[q] = e < eps_min ? eps_min : e;
        }
        return;
    }
    const long long n2 = N / 2;
    double2 *e2 = reinterpret_cast<double2 *>(eps);
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n2;
         q += (long long)gridDim.x * blockDim.x) {
        double2 a = e2[q];
        double e0 = 1.0 - a.x / V, e1 = 1.0 - a.y / V;
        a.x = e0 < eps_min ? eps_min : e0;
        a.y = e1 < eps_min ? eps_min : e1;
        e2[q] = a;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (N & 1)) {
        const double e = 1.0 - eps[N - 1] / V;
        eps[N - 1] = e < eps_min ? eps_min : e;
    }
}

struct PicDragArgs {
    PicGeo G;
    double rho, mu, dp;
    const double *x, *y, *z, *up, *vp, *wp, *om;
    long long m;
    const double *eps, *u, *v, *w;
    double *beta, *sb[3], *Kout;
    WsHeader *hdr;
};

// x^y for x > 0, CORRECTLY ROUNDED (DESIGN.md §3.9 reading; the contract of
// the dots, §3.1): evaluated in double-double and rounded once.
//   ln x:   y0 = log(x) (binary64, any faithful value), then one Newton step
//           L = y0 + (x e^{-y0} - 1) in double-double, error ~ (y0 - ln x)^2 / 2
//           + the double-double rounding, far below 2^-100 relative;
//   exp z:  z = k ln2 + r (ln2 in double-double), r' = r / 32, expm1(r') by its
//           Taylor series to r'^12 (|r'| < 0.011), five expm1 doublings
//           e^{2a} - 1 = (e^a - 1)(e^a - 1 + 2) (relative error kept), 2^k (1 + .).
// The final fast_two_sum leaves hi = RN(hi + lo): the correctly rounded power
// unless x^y lies within ~2^-100 relative of a rounding boundary.  The closure
// needs two powers of one eps: ln is computed once (dd_ln) for both.
__device__ __forceinline__ dd dd_norm(double a, double b)
{
    dd r;
    r.hi = a + b;
    r.lo = b - (r.hi - a);
    return r;
}
__device__ __forceinline__ dd dd_mul(dd a, dd b)
{
    const double p = a.hi * b.hi;
    double e = fma(a.hi, b.hi, -p);
    e = e + (a.hi * b.lo + a.lo * b.hi);
    return dd_norm(p, e);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b)
{
    const double p = a.hi * b;
    double e = fma(a.hi, b, -p);
    e = e + a.lo * b;
    return dd_norm(p, e);
}
__device__ __forceinline__ dd dd_div_d(dd a, double b)
{
    const double q1 = a.hi / b;
    const double rem = fma(-q1, b, a.hi) + a.lo;   // a - q1 b, exact head
    return dd_norm(q1, rem / b);
}
__device__ __forceinline__ dd dd_add_d(dd a, double b)
{
    double s, e;
    two_sum(a.hi, b, s, e);
    return dd_norm(s, e + a.lo);
}
__device__ dd dd_exp(dd z)
{
    const double LN2_HI = 0x1.62e42fefa39efp-1, LN2_LO = 0x1.abc9e3b39803fp-56;
    const double k = rint(z.hi * 0x1.71547652b82fep+0);
    // r = z - k ln2 (k ln2_hi exact as a product pair)
    const double p = k * LN2_HI;
    const double pe = fma(k, LN2_HI, -p);
    dd r = dd_add(z, dd{-p, -pe});
    r = dd_add(r, dd{-k * LN2_LO, -fma(k, LN2_LO, -(k * LN2_LO))});
    r.hi = r.hi * 0x1p-5;
    r.lo = r.lo * 0x1p-5;
    // expm1(r) = r (1 + r/2 (1 + r/3 (1 + ... r/12)))
    dd t = dd{1.0, 0.0};
#pragma unroll 1
    for (int n = 12; n >= 2; n--) t = dd_add_d(dd_div_d(dd_mul(r, t), (double)n), 1.0);
    dd em1 = dd_mul(r, t);
#pragma unroll 1
    for (int q = 0; q < 5; q++) em1 = dd_mul(em1, dd_add_d(em1, 2.0));
    dd e = dd_add_d(em1, 1.0);
    const int ki = (int)k;
    return dd{ldexp(e.hi, ki), ldexp(e.lo, ki)};
}
__device__ dd dd_ln(double x)
{
    const double y0 = log(x);
    const dd E = dd_exp(dd{-y0, 0.0});
    const dd xe = dd_mul_d(E, x);                  // x e^{-y0} ~ 1
    return dd_add_d(dd_add_d(xe, -1.0), y0);
}
// correctly rounded x^y from ln x in double-double (x == 1 gives L = 0 -> 1 exactly)
__device__ __forceinline__ double dd_pow_from_ln(dd L, double y)
{
    const dd P = dd_exp(dd_mul_d(L, y));
    return dd_norm(P.hi, P.lo).hi;
}

// DESIGN.md §3.9 (SPEC.md:285-289 closure, written without the eps_s that cancels)
__device__ __forceinline__ double drag_coef(double rho, double mu, double dp, double Vs, double eg, double slip,
                                            double om)
{
    double Re = ((rho * dp) * slip) / mu;
    Re = Re < 1e-12 ? 1e-12 : Re;
    const dd L = dd_ln(eg);
    const double A = dd_pow_from_ln(L, 4.14);
    const double B = eg <= 0.85 ? 0.8 * dd_pow_from_ln(L, 1.28) : dd_pow_from_ln(L, 2.65);
    const double q = 0.06 * Re;
    const double Vr = 0.5 * ((A - q) + sqrt((q * q + (0.12 * Re) * (2.0 * B - A)) + A * A));
    double Cd = 0.63 + 4.8 / sqrt(Re / Vr);
    Cd = Cd * Cd;
    return (om * Vs) * ((((0.75 * Cd) * eg) * rho) * slip) / ((Vr * Vr) * dp);
}

__global__ void __launch_bounds__(kPicThreads) k_pic_drag(PicDragArgs a)
{
    const PicGeo &G = a.G;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < a.m;
         p += (long long)gridDim.x * blockDim.x) {
        const double X[3] = {__ldg(a.x + p), __ldg(a.y + p), __ldg(a.z + p)};
        const double om = __ldg(a.om + p);
        const double up[3] = {__ldg(a.up + p), __ldg(a.vp + p), __ldg(a.wp + p)};
        if (!parcel_ok(G, X[0], X[1], X[2], om)) {
            atomicMin(&a.hdr->bad_parcel, (unsigned long long)p);
            continue;
        }
        const double Q[3] = {X[0] / G.h[0], X[1] / G.h[1], X[2] / G.h[2]};
        const double eg = pic_interp<-1>(G, a.eps, Q);
        const double ug0 = pic_interp<0>(G, a.u, Q);
        const double ug1 = pic_interp<1>(G, a.v, Q);
        const double ug2 = pic_interp<2>(G, a.w, Q);
        const double sx = ug0 - up[0], sy = ug1 - up[1], sz = ug2 - up[2];
        const double slip = sqrt((sx * sx + sy * sy) + sz * sz);
        const double K = drag_coef(a.rho, a.mu, a.dp, G.Vs, eg, slip, om);
        if (a.Kout) a.Kout[p] = K;
        const double KV = K / G.V;
        double KuV[3];
#pragma unroll
        for (int c = 0; c < 3; c++) KuV[c] = (K * up[c]) / G.V;
        int nd[3][2];
        double w[3][2];
#pragma unroll
        for (int ax = 0; ax < 3; ax++) pic_axis(X[ax], G.h[ax], G.n[ax], false, nd[ax], w[ax]);
#pragma unroll
        for (int kk = 0; kk < 2; kk++)
#pragma unroll
            for (int jj = 0; jj < 2; jj++)
#pragma unroll
                for (int ii = 0; ii < 2; ii++) {
                    const double W = (w[0][ii] * w[1][jj]) * w[2][kk];
                    const long long n = pic_lin(G, nd[0][ii], nd[1][jj], nd[2][kk]);
                    atomicAdd(a.beta + n, W * KV);
#pragma unroll
                    for (int c = 0; c < 3; c++) atomicAdd(a.sb[c] + n, W * KuV[c]);
                }
    }
}

bool pic_geo(const mfx_grid *g, const mfx_pic_params *pp, PicGeo &G)
{
    if (!g || !pp) { set_error("NULL grid / pic params"); return false; }
    if (g->nx < 2 || g->ny < 2 || g->nz < 2) { set_error("grid extents must be >= 2"); return false; }
    if (!(g->dx > 0 && g->dy > 0 && g->dz > 0)) { set_error("spacing must be positive"); return false; }
    if (!(pp->d_p > 0.0)) { set_error("d_p must be positive"); return false; }
    G.n[0] = g->nx; G.n[1] = g->ny; G.n[2] = g->nz;
    G.h[0] = g->dx; G.h[1] = g->dy; G.h[2] = g->dz;
    G.L[0] = g->nx * g->dx; G.L[1] = g->ny * g->dy; G.L[2] = g->nz * g->dz;
    G.V = (g->dx * g->dy) * g->dz;
    G.Vs = (((kPi / 6.0) * pp->d_p) * pp->d_p) * pp->d_p;
    G.eps_min = pp->eps_min;
    G.bc_zlo = g->bc_zlo;
    G.w_in = g->w_in;
    G.N = (long long)g->nx * g->ny * g->nz;
    return true;
}

int pic_grid(long long m)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long need = (m + kPicThreads - 1) / kPicThreads;
    const long long cap = (long long)sms * 8;
    return (int)(need < 1 ? 1 : (need < cap ? need : cap));
}

// ------------------------------------------------------------------ parcel binning
// Deterministic counting sort of the parcels by their BASE cell, i.e. the
// clamped lower corner (floor(x/h - 0.5) per axis) of their trilinear stencil
// (parcels move once per time step, the coupling runs every SIMPLE
// iteration).  Inside a bin the parcels keep ascending original index, so the
// binned order is unique.  Steps: bin + count (atomics), exclusive scan,
// scatter of the original indices (atomic slots), per-bin insertion sort of
// the indices, gather of the seven parcel arrays.
__device__ __forceinline__ unsigned int parcel_bin(const PicGeo &G, double x, double y, double z)
{
    int q[3];
    const double X[3] = {x, y, z};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        int i = (int)floor(X[a] / G.h[a] - 0.5);
        q[a] = i < 0 ? 0 : (i > G.n[a] - 1 ? G.n[a] - 1 : i);
    }
    return (unsigned int)((long long)q[0] + (long long)G.n[0] * ((long long)q[1] + (long long)G.n[1] * q[2]));
}

__global__ void __launch_bounds__(kPicThreads) k_pic_count(PicGeo G, const double *x, const double *y,
                                                           const double *z, long long m, unsigned int *cnt,
                                                           unsigned int *bin_of)
{
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (long long)gridDim.x * blockDim.x) {
        const unsigned int c = parcel_bin(G, __ldg(x + p), __ldg(y + p), __ldg(z + p));
        bin_of[p] = c;
        atomicAdd(cnt + c, 1u);
    }
}

// exclusive scan, levels of 2048-element tiles
constexpr int kScanT = 1024, kScanTile = 2 * kScanT;

__device__ __forceinline__ unsigned int block_exclusive_scan(unsigned int v, unsigned int *sh, unsigned int &total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) sh[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned int w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        sh[lane] = w;   // inclusive warp sums
    }
    __syncthreads();
    total = sh[(blockDim.x >> 5) - 1];
    const unsigned int before = wid ? sh[wid - 1] : 0u;
    __syncthreads();
    return before + incl - v;
}

__global__ void __launch_bounds__(kScanT) k_scan_tiles(unsigned int *a, long long n, unsigned int *tile_sum)
{
    __shared__ unsigned int sh[32];
    const long long base = (long long)blockIdx.x * kScanTile + 2 * threadIdx.x;
    const unsigned int v0 = base < n ? a[base] : 0u, v1 = base + 1 < n ? a[base + 1] : 0u;
    unsigned int total;
    const unsigned int ex = block_exclusive_scan(v0 + v1, sh, total);
    if (base < n) a[base] = ex;
    if (base + 1 < n) a[base + 1] = ex + v0;
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanT) k_scan_add(unsigned int *a, long long n, const unsigned int *tile_off)
{
    const long long base = (long long)blockIdx.x * kScanTile + 2 * threadIdx.x;
    const unsigned int off = tile_off[blockIdx.x];
    if (base < n) a[base] += off;
    if (base + 1 < n) a[base + 1] += off;
}

mfx_status exclusive_scan(unsigned int *a, long long n, unsigned int *scratch, cudaStream_t s)
{
    const long long tiles = (n + kScanTile - 1) / kScanTile;
    k_scan_tiles<<<(unsigned)tiles, kScanT, 0, s>>>(a, n, scratch);
    if (tiles > 1) {
        MFX_ARG_CHECK(tiles <= (long long)kScanTile * kScanTile, "scan too long");
        mfx_status st = exclusive_scan(scratch, tiles, scratch + ((tiles + 255) & ~255LL), s);
        if (st != MFX_OK) return st;
        k_scan_add<<<(unsigned)tiles, kScanT, 0, s>>>(a, n, scratch);
    }
    launch_count_add(tiles > 1 ? 2 : 1);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

__global__ void __launch_bounds__(kPicThreads) k_pic_slot(long long m, const unsigned int *bin_of,
                                                          const unsigned int *start, unsigned int *fill,
                                                          unsigned int *orig)
{
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (long long)gridDim.x * blockDim.x) {
        const unsigned int c = bin_of[p];
        orig[start[c] + atomicAdd(fill + c, 1u)] = (unsigned int)p;
    }
}

// one thread per bin: ascending original index inside the bin (insertion sort)
__global__ void __launch_bounds__(kPicThreads) k_pic_binsort(long long nbins, const unsigned int *start,
                                                             const unsigned int *cnt, unsigned int *orig)
{
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += (long long)gridDim.x * blockDim.x) {
        const unsigned int lo = start[b], len = cnt[b];
        for (unsigned int i = 1; i < len; i++) {
            const unsigned int v = orig[lo + i];
            unsigned int j = i;
            while (j > 0 && orig[lo + j - 1] > v) { orig[lo + j] = orig[lo + j - 1]; j--; }
            orig[lo + j] = v;
        }
    }
}

struct GatherArgs {
    const double *in[7];
    double *out[7];
    long long m;
    const unsigned int *orig;
};

__global__ void __launch_bounds__(kPicThreads) k_pic_gather_parcels(GatherArgs a)
{
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < a.m; q += (long long)gridDim.x * blockDim.x) {
        const unsigned int p = a.orig[q];
#pragma unroll
        for (int f = 0; f < 7; f++) a.out[f][q] = __ldg(a.in[f] + p);
    }
}

__global__ void k_pic_bin_end(unsigned int *start, long long nbins, unsigned int m)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) start[nbins] = m;
}

// ------------------------------------------------------------------ gather deposits on binned parcels
// Node c receives, in ascending original parcel index, W * value from every
// parcel whose stencil contains c -- exactly the sequence of additions the
// parcel-ordered definition makes to that node, so the sums
// are bitwise those of the oracle.  Contributors sit in the bins c - {0,1}^3;
// the (<= 8) bin lists are merged by original index.
template <int NV>
struct NodeGather {
    const PicGeo *G;
    const double *xi[3];     // cell-centre lattice coordinates per binned parcel (k_pic_vals)
    const double *val[NV];
    const unsigned int *orig, *start;
    __device__ void run(long long c, double (&acc)[NV]) const
    {
        const int ci = (int)(c % G->n[0]);
        const int cj = (int)((c / G->n[0]) % G->n[1]);
        const int ck = (int)(c / ((long long)G->n[0] * G->n[1]));
        unsigned int cur[8], end[8];
        int nb = 0;
#pragma unroll
        for (int dk = 1; dk >= 0; dk--)
#pragma unroll
            for (int dj = 1; dj >= 0; dj--)
#pragma unroll
                for (int di = 1; di >= 0; di--) {
                    const int bi = ci - di, bj = cj - dj, bk = ck - dk;
                    cur[nb] = 0u; end[nb] = 0u;
                    if (bi >= 0 && bj >= 0 && bk >= 0) {
                        const long long b = (long long)bi + (long long)G->n[0] * ((long long)bj + (long long)G->n[1] * bk);
                        cur[nb] = __ldg(start + b);
                        end[nb] = __ldg(start + b + 1);
                    }
                    nb++;
                }
#pragma unroll
        for (int v = 0; v < NV; v++) acc[v] = 0.0;
        for (;;) {
            int best = -1;
            unsigned int bo = 0xffffffffu;
#pragma unroll
            for (int q = 0; q < 8; q++)
                if (cur[q] < end[q]) {
                    const unsigned int o = __ldg(orig + cur[q]);
                    if (o < bo) { bo = o; best = q; }
                }
            if (best < 0) break;
            const unsigned int pos = cur[best]++;
            const double X[3] = {__ldg(xi[0] + pos), __ldg(xi[1] + pos), __ldg(xi[2] + pos)};
            // invalid parcels carry value 0 (latched by the value pass); a NaN position
            // would still turn W * 0 into NaN, so those are skipped here
            if (X[0] != X[0] || X[1] != X[1] || X[2] != X[2]) continue;
            int nd[3][2];
            double w[3][2];
#pragma unroll
            for (int ax = 0; ax < 3; ax++) pic_axis_xi(X[ax], G->n[ax], false, nd[ax], w[ax]);
            double vv[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) vv[v] = __ldg(val[v] + pos);
#pragma unroll
            for (int kk = 0; kk < 2; kk++)
#pragma unroll
                for (int jj = 0; jj < 2; jj++)
#pragma unroll
                    for (int ii = 0; ii < 2; ii++)
                        if (nd[0][ii] == ci && nd[1][jj] == cj && nd[2][kk] == ck) {
                            const double W = (w[0][ii] * w[1][jj]) * w[2][kk];
#pragma unroll
                            for (int v = 0; v < NV; v++) acc[v] += W * vv[v];
                        }
        }
    }
};

struct PicValsArgs {
    PicGeo G;
    double rho, mu, dp;
    const double *x, *y, *z, *up, *vp, *wp, *om;
    long long m;
    const double *eps, *u, *v, *w;
    double *vals;           // [4][m]: K/V, (K u)/V, (K v)/V, (K w)/V   or [1][m]: omega Vs (eps mode)
    double *xi;             // [3][m]: cell-centre lattice coordinates x/h - 0.5 (the gathers' stencils)
    double *Kout;
    const unsigned int *orig;
    WsHeader *hdr;
    int drag;
};

// per-parcel values in binned order (invalid parcels contribute 0 and are latched by original index)
__global__ void __launch_bounds__(kPicThreads) k_pic_vals(PicValsArgs a)
{
    const PicGeo &G = a.G;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < a.m; p += (long long)gridDim.x * blockDim.x) {
        const double X[3] = {__ldg(a.x + p), __ldg(a.y + p), __ldg(a.z + p)};
        const double om = __ldg(a.om + p);
        const double Q[3] = {X[0] / G.h[0], X[1] / G.h[1], X[2] / G.h[2]};
#pragma unroll
        for (int ax = 0; ax < 3; ax++) a.xi[ax * a.m + p] = Q[ax] - 0.5;     // = pic_xi(X, h, false)
        if (!parcel_ok(G, X[0], X[1], X[2], om)) {
            atomicMin(&a.hdr->bad_parcel, (unsigned long long)a.orig[p]);
            for (int v = 0; v < (a.drag ? 4 : 1); v++) a.vals[v * a.m + p] = 0.0;
            if (a.Kout) a.Kout[p] = 0.0;
            continue;
        }
        if (!a.drag) {
            a.vals[p] = om * G.Vs;
            continue;
        }
        const double up[3] = {__ldg(a.up + p), __ldg(a.vp + p), __ldg(a.wp + p)};
        const double eg = pic_interp<-1>(G, a.eps, Q);
        const double ug0 = pic_interp<0>(G, a.u, Q);
        const double ug1 = pic_interp<1>(G, a.v, Q);
        const double ug2 = pic_interp<2>(G, a.w, Q);
        const double sx = ug0 - up[0], sy = ug1 - up[1], sz = ug2 - up[2];
        const double slip = sqrt((sx * sx + sy * sy) + sz * sz);
        const double K = drag_coef(a.rho, a.mu, a.dp, G.Vs, eg, slip, om);
        if (a.Kout) a.Kout[p] = K;
        a.vals[p] = K / G.V;
#pragma unroll
        for (int c = 0; c < 3; c++) a.vals[(c + 1) * a.m + p] = (K * up[c]) / G.V;
    }
}

struct NodeArgs1 {
    PicGeo G;
    NodeGather<1> ng;
    double *eps;
};
__global__ void __launch_bounds__(kPicThreads) k_node_eps(NodeArgs1 a)
{
    NodeGather<1> ng = a.ng;
    ng.G = &a.G;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < a.G.N; c += (long long)gridDim.x * blockDim.x) {
        double acc[1];
        ng.run(c, acc);
        const double e = 1.0 - acc[0] / a.G.V;
        a.eps[c] = e < a.G.eps_min ? a.G.eps_min : e;
    }
}

struct NodeArgs4 {
    PicGeo G;
    NodeGather<4> ng;
    double *out[4];
};
__global__ void __launch_bounds__(kPicThreads) k_node_drag(NodeArgs4 a)
{
    NodeGather<4> ng = a.ng;
    ng.G = &a.G;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < a.G.N; c += (long long)gridDim.x * blockDim.x) {
        double acc[4];
        ng.run(c, acc);
#pragma unroll
        for (int v = 0; v < 4; v++) a.out[v][c] = acc[v];
    }
}

}  // namespace

mfx_status pic_deposit_eps(const mfx_grid *grid, const mfx_pic_params *pp, const mfx_parcels *pc, double *eps,
                           void *ws, size_t wsb, cudaStream_t s)
{
    PicGeo G;
    if (!pic_geo(grid, pp, G)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(pc && eps, "NULL parcels / eps");
    MFX_ARG_CHECK(pc->n >= 0, "negative parcel count");
    MFX_ARG_CHECK(pc->n == 0 || (pc->x && pc->y && pc->z && pc->omega), "NULL parcel array");
    MFX_ARG_CHECK(ws && wsb >= ws_header_bytes(), "bad workspace");
    MFX_CUDA_TRY(cudaMemsetAsync(eps, 0, sizeof(double) * G.N, s));
    if (pc->n > 0) {
        PicEpsArgs a;
        a.G = G;
        a.x = pc->x; a.y = pc->y; a.z = pc->z; a.om = pc->omega;
        a.m = pc->n;
        a.acc = eps;
        a.hdr = (WsHeader *)ws;
        count_launch(10, s, true);
        k_pic_eps<<<pic_grid(pc->n), kPicThreads, 0, s>>>(a);
        count_launch(10, s, false);
        MFX_CUDA_TRY(cudaGetLastError());
    }
    k_pic_eps_final<<<reduce_grid(G.N / 2 + 1), kPicThreads, 0, s>>>(eps, G.N, G.V, G.eps_min);
    launch_count_add(1);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

mfx_status pic_drag(const mfx_grid *grid, const mfx_params *pr, const mfx_pic_params *pp, const mfx_parcels *pc,
                    const double *eps, const double *u, const double *v, const double *w, double *beta,
                    double *sbu, double *sbv, double *sbw, double *Kout, void *ws, size_t wsb, cudaStream_t s)
{
    PicGeo G;
    if (!pic_geo(grid, pp, G)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(pr && pc, "NULL params / parcels");
    MFX_ARG_CHECK(pr->mu > 0.0, "mu must be positive");
    MFX_ARG_CHECK(eps && u && v && w && beta && sbu && sbv && sbw, "NULL field");
    MFX_ARG_CHECK(pc->n >= 0, "negative parcel count");
    MFX_ARG_CHECK(pc->n == 0 || (pc->x && pc->y && pc->z && pc->u && pc->v && pc->w && pc->omega),
                  "NULL parcel array");
    MFX_ARG_CHECK(ws && wsb >= ws_header_bytes(), "bad workspace");
    double *outs[4] = {beta, sbu, sbv, sbw};
    for (int q = 0; q < 4; q++) MFX_CUDA_TRY(cudaMemsetAsync(outs[q], 0, sizeof(double) * G.N, s));
    if (pc->n == 0) return MFX_OK;
    PicDragArgs a;
    a.G = G;
    a.rho = pr->rho; a.mu = pr->mu; a.dp = pp->d_p;
    a.x = pc->x; a.y = pc->y; a.z = pc->z; a.up = pc->u; a.vp = pc->v; a.wp = pc->w; a.om = pc->omega;
    a.m = pc->n;
    a.eps = eps; a.u = u; a.v = v; a.w = w;
    a.beta = beta; a.sb[0] = sbu; a.sb[1] = sbv; a.sb[2] = sbw; a.Kout = Kout;
    a.hdr = (WsHeader *)ws;
    count_launch(11, s, true);
    k_pic_drag<<<pic_grid(pc->n), kPicThreads, 0, s>>>(a);
    count_launch(11, s, false);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

size_t pic_sort_scratch_bytes(long long N, long long m)
{
    const long long tiles = (N + 1 + kScanTile - 1) / kScanTile;
    const long long scan = ((tiles + 255) & ~255LL) + ((tiles / kScanTile + 1 + 255) & ~255LL) + 256;
    return sizeof(unsigned int) * (size_t)(2 * ((N + 64) & ~63LL) + ((m + 63) & ~63LL) + ((m + 63) & ~63LL) + scan);
}

// scratch layout: cnt[N+1] (becomes bin starts), fill[N+1], bin_of[m], orig[m], scan scratch
mfx_status pic_sort(const mfx_grid *grid, const mfx_pic_params *pp, const mfx_parcels *in, double *const out[7],
                    unsigned int *orig_out, unsigned int *start_out, void *scratch, size_t scratch_bytes,
                    cudaStream_t s)
{
    PicGeo G;
    if (!pic_geo(grid, pp, G)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(in && out, "NULL parcels / out");
    MFX_ARG_CHECK(in->n >= 0, "negative parcel count");
    const long long m = in->n;
    const double *src[7] = {in->x, in->y, in->z, in->u, in->v, in->w, in->omega};
    for (int f = 0; f < 7; f++) {
        MFX_ARG_CHECK(m == 0 || (src[f] && out[f]), "NULL parcel array %d", f);
        MFX_ARG_CHECK(m == 0 || src[f] != out[f], "parcel sort cannot run in place (array %d)", f);
    }
    MFX_ARG_CHECK(G.N < (1LL << 32) - 1 && m < (1LL << 32), "grid / parcel count too large for 32-bit bins");
    MFX_ARG_CHECK(scratch && scratch_bytes >= pic_sort_scratch_bytes(G.N, m), "scratch of %zu bytes, need %zu",
                  scratch_bytes, pic_sort_scratch_bytes(G.N, m));
    const long long NB = (G.N + 64) & ~63LL;
    unsigned int *cnt = (unsigned int *)scratch;
    unsigned int *fill = cnt + NB;
    unsigned int *bin_of = fill + NB;
    unsigned int *orig = bin_of + ((m + 63) & ~63LL);
    unsigned int *scan_scratch = orig + ((m + 63) & ~63LL);
    MFX_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned int) * 2 * NB, s));
    if (m > 0) {
        k_pic_count<<<pic_grid(m), kPicThreads, 0, s>>>(G, in->x, in->y, in->z, m, cnt, bin_of);
        launch_count_add(1);
    }
    mfx_status st = exclusive_scan(cnt, G.N, scan_scratch, s);
    if (st != MFX_OK) return st;
    k_pic_bin_end<<<1, 1, 0, s>>>(cnt, G.N, (unsigned int)m);
    if (m > 0) {
        k_pic_slot<<<pic_grid(m), kPicThreads, 0, s>>>(m, bin_of, cnt, fill, orig);
        // per-bin sort: fill[] now holds the counts again (every slot taken)
        k_pic_binsort<<<reduce_grid(G.N), kPicThreads, 0, s>>>(G.N, cnt, fill, orig);
        GatherArgs ga;
        for (int f = 0; f < 7; f++) { ga.in[f] = src[f]; ga.out[f] = out[f]; }
        ga.m = m;
        ga.orig = orig;
        k_pic_gather_parcels<<<pic_grid(m), kPicThreads, 0, s>>>(ga);
        launch_count_add(4);
        if (orig_out) MFX_CUDA_TRY(cudaMemcpyAsync(orig_out, orig, sizeof(unsigned int) * m, cudaMemcpyDeviceToDevice, s));
    }
    if (start_out)
        MFX_CUDA_TRY(cudaMemcpyAsync(start_out, cnt, sizeof(unsigned int) * (G.N + 1), cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

// deposits on binned parcels (bitwise the parcel-ordered definition)
mfx_status pic_deposit_binned(int drag, const mfx_grid *grid, const mfx_params *pr, const mfx_pic_params *pp,
                              const mfx_parcels *pc, const unsigned int *orig, const unsigned int *start,
                              const double *eps_in, const double *u, const double *v, const double *w,
                              double *const outs[4], double *Kout, double *vals, void *ws, size_t wsb,
                              cudaStream_t s)
{
    PicGeo G;
    if (!pic_geo(grid, pp, G)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(pc && pc->n >= 0 && start && outs && outs[0], "NULL argument");
    MFX_ARG_CHECK(pc->n == 0 || (pc->x && pc->y && pc->z && pc->omega && orig && vals), "NULL parcel array / orig / vals");
    MFX_ARG_CHECK(ws && wsb >= ws_header_bytes(), "bad workspace");
    if (drag) {
        MFX_ARG_CHECK(pr && pr->mu > 0.0, "params / mu");
        MFX_ARG_CHECK(eps_in && u && v && w && outs[1] && outs[2] && outs[3], "NULL field");
        MFX_ARG_CHECK(pc->n == 0 || (pc->u && pc->v && pc->w), "NULL parcel velocity");
    }
    const long long m = pc->n;
    if (m > 0) {
        PicValsArgs a;
        memset(&a, 0, sizeof(a));
        a.G = G;
        if (drag) { a.rho = pr->rho; a.mu = pr->mu; a.dp = pp->d_p; }
        a.x = pc->x; a.y = pc->y; a.z = pc->z; a.up = pc->u; a.vp = pc->v; a.wp = pc->w; a.om = pc->omega;
        a.m = m;
        a.eps = eps_in; a.u = u; a.v = v; a.w = w;
        a.vals = vals; a.Kout = Kout; a.orig = orig; a.hdr = (WsHeader *)ws; a.drag = drag;
        a.xi = vals + (size_t)(drag ? 4 : 1) * (size_t)m;
        count_launch(drag ? 11 : 10, s, true);
        k_pic_vals<<<pic_grid(m), kPicThreads, 0, s>>>(a);
        count_launch(drag ? 11 : 10, s, false);
    }
    const int nb = reduce_grid(G.N);
    if (drag) {
        NodeArgs4 na;
        na.G = G;
        for (int ax = 0; ax < 3; ax++) na.ng.xi[ax] = vals + (size_t)(4 + ax) * (size_t)m;
        for (int q = 0; q < 4; q++) { na.ng.val[q] = vals + (size_t)q * (size_t)m; na.out[q] = outs[q]; }
        na.ng.orig = orig; na.ng.start = start;
        k_node_drag<<<nb, kPicThreads, 0, s>>>(na);
    } else {
        NodeArgs1 na;
        na.G = G;
        for (int ax = 0; ax < 3; ax++) na.ng.xi[ax] = vals + (size_t)(1 + ax) * (size_t)m;
        na.ng.val[0] = vals;
        na.ng.orig = orig; na.ng.start = start;
        na.eps = outs[0];
        k_node_eps<<<nb, kPicThreads, 0, s>>>(na);
    }
    launch_count_add(1);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

}  // namespace mfx
