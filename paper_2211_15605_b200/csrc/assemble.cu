// assemble.cu -- a-1 momentum, a-2 pressure-correction and a-3 scalar
// coefficient assembly (Eq. 1, Eq. 2 P:53,
// P:85) and a-7 the SIMPLE correction.
//
// One thread per row, grid-stride over cells with a fixed grid, so the
// residual sums reduce in a fixed order (correctly rounded).
// Assembly runs once per outer iteration; the BiCGSTAB kernels dominate.
#include <climits>

#include "common.cuh"
#include "mom_row.cuh"

namespace mfx {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double maxp(double f) { return f > 0.0 ? f : 0.0; }

struct Cell {
    int q[3];
};

__device__ __forceinline__ long long lin(const Geo &G, const int q[3])
{
    return (long long)q[0] + (long long)G.nx * ((long long)q[1] + (long long)G.ny * q[2]);
}
__device__ __forceinline__ int extent(const Geo &G, int a) { return a == 0 ? G.nx : (a == 1 ? G.ny : G.nz); }
__device__ __forceinline__ bool in_dom(const Geo &G, const int q[3])
{
    return q[0] >= 0 && q[0] < G.nx && q[1] >= 0 && q[1] < G.ny && q[2] >= 0 && q[2] < G.nz;
}
__device__ __forceinline__ void decode(const Geo &G, long long n, int q[3])
{
    long long pl = n / G.sz;
    long long rem = n - pl * G.sz;
    q[2] = (int)pl;
    q[1] = (int)(rem / G.nx);
    q[0] = (int)(rem - (long long)q[1] * G.nx);
}

__device__ __forceinline__ void latch(WsHeader *h, bool nonfinite, bool zerodiag, long long n)
{
    if (nonfinite) atomicMin(&h->bad_nonfinite, (unsigned long long)n);
    else if (zerodiag) atomicMin(&h->bad_zerodiag, (unsigned long long)n);
}

// ------------------------------------------------------------------ momentum
struct MomArgs {
    Geo G;
    MomRowPar R;                      // row constants (mom_row.cuh)
    int upwind;                       // face_eps_upwind
    double rho, urf, gc, rVdt;
    double Dc[3];
    const double *eps, *eps0, *vel0, *vel1, *vel2, *uold, *p, *beta, *S;
    const unsigned char *blocked;   // NULL or N flags
    double *aP, *aE, *aW, *aN, *aS, *aT, *aB, *b, *d;
    double *resid2;
    WsHeader *hdr;
    dd *part;
};

// §3.10: cell (i, j, k) is BLOCKED (outside the domain: not blocked)
__device__ __forceinline__ bool blk_at(const Geo &G, const unsigned char *bl, int i, int j, int k)
{
    if (!bl || i < 0 || j < 0 || k < 0 || i >= G.nx || j >= G.ny || k >= G.nz) return false;
    return __ldg(bl + ((long long)i + (long long)G.nx * ((long long)j + (long long)G.ny * k))) != 0;
}
__device__ __forceinline__ bool blk_q(const Geo &G, const unsigned char *bl, const int q[3])
{
    return blk_at(G, bl, q[0], q[1], q[2]);
}

template <int C>
__device__ __forceinline__ int row_type(const Geo &G, const int q[3], const unsigned char *bl = nullptr)
{
    if (bl && blk_q(G, bl, q)) return kIdentity;                         // §3.10
    if (q[C] < extent(G, C) - 1) {
        if (bl) {
            int e[3] = {q[0], q[1], q[2]};
            e[C] += 1;
            if (blk_q(G, bl, e)) return kIdentity;                       // internal wall face
        }
        return kInterior;
    }
    if (C == 2 && G.bc_zhi == MFX_BC_OUTLET) return kOutlet;
    return kIdentity;
}

template <int C>
__device__ __forceinline__ const double *vfield(const MomArgs &a, int t)
{
    return t == 0 ? a.vel0 : (t == 1 ? a.vel1 : a.vel2);
}

// component-C velocity on the face Q + e_C/2 (DESIGN.md §3.3 vel_c)
template <int C>
__device__ __forceinline__ double vel_c(const MomArgs &a, const int Q[3])
{
    const Geo &G = a.G;
    if (Q[C] == -1) return (C == 2 && G.bc_zlo == MFX_BC_INLET) ? G.w_in : 0.0;
    if (Q[C] == extent(G, C) - 1 && row_type<C>(G, Q) == kIdentity) return 0.0;
    return __ldg(vfield<C>(a, C) + lin(G, Q));
}

// +t face mass flux of cell X (interior face)
template <int C>
__device__ __forceinline__ double mflux_t(const MomArgs &a, int t, const int X[3])
{
    const Geo &G = a.G;
    int Xt[3] = {X[0], X[1], X[2]};
    Xt[t] += 1;
    double ef = 0.5 * (__ldg(a.eps + lin(G, X)) + __ldg(a.eps + lin(G, Xt)));
    return ((a.rho * ef) * G.A[t]) * __ldg(vfield<C>(a, t) + lin(G, X));
}

// Clamped neighbour index (always a valid cell; values read at clamped
// positions are only used where DESIGN.md §3.3 says the neighbour exists).
__device__ __forceinline__ long long lin_cl(const Geo &G, int i, int j, int k)
{
    i = i < 0 ? 0 : (i >= G.nx ? G.nx - 1 : i);
    j = j < 0 ? 0 : (j >= G.ny ? G.ny - 1 : j);
    k = k < 0 ? 0 : (k >= G.nz ? G.nz - 1 : k);
    return (long long)i + (long long)G.nx * ((long long)j + (long long)G.ny * k);
}

__device__ __forceinline__ void decode32(const Geo &G, long long n, int q[3])
{
    const unsigned int un = (unsigned int)n, sz = (unsigned int)G.sz, nx = (unsigned int)G.nx;
    const unsigned int k = un / sz, rem = un - k * sz, j = rem / nx;
    q[0] = (int)(rem - j * nx);
    q[1] = (int)j;
    q[2] = (int)k;
}

// Momentum row.  Every neighbour value the row can need is
// loaded first, unconditionally, from clamped indices (34 independent loads in
// flight per thread); the boundary rules then only select among them.
template <int C>
__global__ void __launch_bounds__(kThreads, 2) k_assemble_mom(MomArgs a)
{
    const Geo &G = a.G;
    constexpr int T1 = C == 0 ? 1 : 0, T2 = C == 2 ? 1 : 2;   // transverse axes
    Acc num, den;
    num.zero();
    den.zero();
    const double *um = vfield<C>(a, C);
    const double *vt[2] = {vfield<C>(a, T1), vfield<C>(a, T2)};
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < G.N;
         n += (long long)gridDim.x * blockDim.x) {
        int P[3];
        decode32(G, n, P);
        const int type = row_type<C>(G, P, a.blocked);
        if (type == kIdentity) {
            a.aP[n] = 1.0;
            a.aE[n] = 0.0; a.aW[n] = 0.0; a.aN[n] = 0.0; a.aS[n] = 0.0; a.aT[n] = 0.0; a.aB[n] = 0.0;
            a.b[n] = 0.0;
            a.d[n] = 0.0;
            continue;
        }
        int E[3] = {P[0], P[1], P[2]};
        if (type == kInterior) E[C] += 1;
        const long long nE = lin(G, E);
        // ---- gather (every value the row can need, from clamped indices)
        MomRowIn in;
        in.P[0] = P[0]; in.P[1] = P[1]; in.P[2] = P[2];
        in.type = type;
        in.epsP_ = __ldg(a.eps + n);
        in.epsE_ = __ldg(a.eps + nE);
#pragma unroll
        for (int ti = 0; ti < 2; ti++) {
            const int t = ti == 0 ? T1 : T2;
#pragma unroll
            for (int sg = 0; sg < 2; sg++) {
                const int s = sg ? 1 : -1;
                int Pt[3] = {P[0], P[1], P[2]}, Et[3] = {E[0], E[1], E[2]};
                Pt[t] += s;
                Et[t] += s;
                const long long iP = lin_cl(G, Pt[0], Pt[1], Pt[2]), iE = lin_cl(G, Et[0], Et[1], Et[2]);
                in.epsPt_[ti][sg] = __ldg(a.eps + iP);
                in.epsEt_[ti][sg] = __ldg(a.eps + iE);
                // velocity on the +t face of Q (s>0: Q = P, R = E; s<0: Q = P-e_t, R = E-e_t)
                in.vP_[ti][sg] = __ldg(vt[ti] + (s > 0 ? n : iP));
                in.vE_[ti][sg] = __ldg(vt[ti] + (s > 0 ? nE : iE));
                const int pt = P[t] + s;
                in.nb_wall_[ti][sg] = a.blocked && pt >= 0 && pt < extent(G, t) &&
                                     (blk_q(G, a.blocked, Pt) || blk_q(G, a.blocked, Et));   // §3.10
            }
        }
        int Pm[3] = {P[0], P[1], P[2]};
        Pm[C] -= 1;
        in.umP_ = __ldg(um + n);
        in.umE_ = __ldg(um + nE);
        in.umM_ = __ldg(um + lin_cl(G, Pm[0], Pm[1], Pm[2]));
#pragma unroll
        for (int s6 = 0; s6 < 6; s6++) {
            int Q[3] = {P[0], P[1], P[2]};
            Q[s6 / 2] += (s6 & 1) ? 1 : -1;
            in.unb_[s6] = in_dom(G, Q) ? __ldg(um + lin_cl(G, Q[0], Q[1], Q[2])) : 0.0;
        }
        in.e0P = __ldg(a.eps0 + n); in.e0E = __ldg(a.eps0 + nE);
        in.bP = __ldg(a.beta + n); in.bE = __ldg(a.beta + nE);
        in.SP = __ldg(a.S + n); in.SE = __ldg(a.S + nE);
        in.pP = __ldg(a.p + n); in.pEv = __ldg(a.p + nE);
        in.uoP = __ldg(a.uold + n);
        in.m_wall = P[C] >= 1 && blk_q(G, a.blocked, Pm);                    // internal wall face (§3.10)
        in.e_ident = type != kOutlet && row_type<C>(G, E, a.blocked) == kIdentity;

        // ---- row (mom_row.cuh)
        MomRowOut o;
        mom_row<C>(a.R, in, o);
        a.aW[n] = o.st6[0]; a.aE[n] = o.st6[1];
        a.aS[n] = o.st6[2]; a.aN[n] = o.st6[3];
        a.aB[n] = o.st6[4]; a.aT[n] = o.st6[5];
        a.aP[n] = o.aPr;
        a.b[n] = o.bR;
        a.d[n] = o.d;
        const bool nonfin = !isfinite(o.aPr) || !isfinite(o.bR) || !isfinite(o.d);
        if (nonfin || o.aPr == 0.0) latch(a.hdr, nonfin, o.aPr == 0.0, n);
        num.add(o.res);
        den.add(o.den);
    }
    __shared__ dd sh[(kThreads / 32) * 2];
    dd v[2] = {num.get(), den.get()}, out[2];
    if (grid_reduce_dd<2>(v, a.part, &a.hdr->ticket[0], sh, out) && threadIdx.x == 0 && a.resid2) {
        a.resid2[0] = dd_round(out[0]);
        a.resid2[1] = dd_round(out[1]);
    }
}

// ------------------------------------------------------------------ p'
struct PPArgs {
    Geo G;
    int upwind;
    double rho, rVdt;
    const double *eps, *eps0, *us[3], *dv[3];
    const double *um[3];              // snapshot velocities (upwind direction, §3.12)
    const unsigned char *blocked;
    double *aP, *cx, *cy, *cz, *b;
    double *resid2;
    WsHeader *hdr;
    dd *part;
};

// UP: upwinded convective face eps (§3.12); BL: BLOCKED cells (§3.10).  The
// default <false, false> instantiation is the plain row of §3.4.
template <bool UP, bool BL>
__global__ void __launch_bounds__(kThreads) k_assemble_pp(PPArgs a)
{
    // DESIGN.md §3.4; every neighbour value (and flag / snapshot velocity the
    // variant needs) loaded up front from clamped indices
    const Geo &G = a.G;
    Acc cont;
    cont.zero();
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < G.N;
         n += (long long)gridDim.x * blockDim.x) {
        int P[3];
        decode32(G, n, P);
        const double epsP = __ldg(a.eps + n), eps0P = __ldg(a.eps0 + n);
        double eM[3], eP[3], dP[3], dM[3], uP[3], uM[3], vmP[3], vmM[3];
        bool blP[3], blM[3];
        const bool bP = BL ? __ldg(a.blocked + n) != 0 : false;
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            int Qm[3] = {P[0], P[1], P[2]}, Qp[3] = {P[0], P[1], P[2]};
            Qm[ax] -= 1;
            Qp[ax] += 1;
            const long long im = lin_cl(G, Qm[0], Qm[1], Qm[2]), ip = lin_cl(G, Qp[0], Qp[1], Qp[2]);
            eM[ax] = __ldg(a.eps + im);
            eP[ax] = __ldg(a.eps + ip);
            dP[ax] = __ldg(a.dv[ax] + n);
            dM[ax] = __ldg(a.dv[ax] + im);
            uP[ax] = __ldg(a.us[ax] + n);
            uM[ax] = __ldg(a.us[ax] + im);
            vmP[ax] = UP ? __ldg(a.um[ax] + n) : 0.0;
            vmM[ax] = UP ? __ldg(a.um[ax] + im) : 0.0;
            blP[ax] = BL ? (P[ax] < extent(G, ax) - 1 && __ldg(a.blocked + ip) != 0) : false;
            blM[ax] = BL ? (P[ax] >= 1 && __ldg(a.blocked + im) != 0) : false;
        }
        double cm[3], cpl[3], mm[3], mp[3];
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            const int ext = extent(G, ax);
            const bool wall_p = bP || blP[ax];                               // §3.10 internal walls
            const bool wall_m = bP || blM[ax];
            // +a face of P
            if (P[ax] <= ext - 2 && wall_p) {
                cpl[ax] = 0.0;
                mp[ax] = 0.0;
            } else if (P[ax] <= ext - 2) {
                const double ef = UP ? (vmP[ax] >= 0.0 ? epsP : eP[ax]) : 0.5 * (epsP + eP[ax]);
                cpl[ax] = ((a.rho * ef) * G.A[ax]) * dP[ax];
                mp[ax] = ((a.rho * ef) * G.A[ax]) * uP[ax];
            } else if (ax == 2 && G.bc_zhi == MFX_BC_OUTLET && !bP) {
                cpl[ax] = ((a.rho * epsP) * G.A[2]) * dP[ax];
                mp[ax] = ((a.rho * epsP) * G.A[2]) * uP[ax];
            } else {
                cpl[ax] = 0.0;
                mp[ax] = 0.0;
            }
            // -a face of P = +a face of P - e_a (interior by construction)
            if (P[ax] >= 1 && wall_m) {
                cm[ax] = 0.0;
                mm[ax] = 0.0;
            } else if (P[ax] >= 1) {
                const double ef = UP ? (vmM[ax] >= 0.0 ? eM[ax] : epsP) : 0.5 * (eM[ax] + epsP);
                cm[ax] = ((a.rho * ef) * G.A[ax]) * dM[ax];
                mm[ax] = ((a.rho * ef) * G.A[ax]) * uM[ax];
            } else {
                cm[ax] = 0.0;
                mm[ax] = (ax == 2 && G.bc_zlo == MFX_BC_INLET && !bP) ? ((a.rho * epsP) * G.A[2]) * G.w_in : 0.0;
            }
        }
        const double aP = ((((cm[0] + cpl[0]) + cm[1]) + cpl[1]) + cm[2]) + cpl[2];
        double bb = (((mm[0] - mp[0]) + (mm[1] - mp[1])) + (mm[2] - mp[2])) - a.rVdt * (epsP - eps0P);
        if (bP) bb = 0.0;                                                   // empty row: p' stays 0
        a.aP[n] = aP;
        a.cx[n] = cpl[0];
        a.cy[n] = cpl[1];
        a.cz[n] = cpl[2];
        a.b[n] = bb;
        const bool nonfin = !isfinite(aP) || !isfinite(bb);
        const bool zd = aP == 0.0 && !bP;
        if (nonfin || zd) latch(a.hdr, nonfin, zd, n);
        cont.add(fabs(bb));
    }
    __shared__ dd sh[(kThreads / 32) * 1];
    dd v[1] = {cont.get()}, out[1];
    if (grid_reduce_dd<1>(v, a.part, &a.hdr->ticket[0], sh, out) && threadIdx.x == 0 && a.resid2) {
        a.resid2[0] = dd_round(out[0]);
        a.resid2[1] = 0.0;
    }
}

// ------------------------------------------------------------------ scalar
struct ScalArgs {
    Geo G;
    int upwind;
    double rho, urf, rVdt;
    double Dc[3];
    const double *eps, *eps0, *vel[3], *phim, *phi0;
    const unsigned char *blocked;
    double *aP, *aE, *aW, *aN, *aS, *aT, *aB, *b, *d;
    double *resid2;
    WsHeader *hdr;
    dd *part;
};

// BL: BLOCKED cells (§3.10).  Every neighbour value is loaded up front from
// clamped indices; the boundary rules then only select among them.
template <bool BL>
__global__ void __launch_bounds__(kThreads) k_assemble_scalar(ScalArgs a)
{
    const Geo &G = a.G;
    Acc num, den;
    num.zero();
    den.zero();
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < G.N;
         n += (long long)gridDim.x * blockDim.x) {
        int P[3];
        decode32(G, n, P);
        if (BL && __ldg(a.blocked + n) != 0) {
            // BLOCKED cell (§3.10): identity row phi = 0, no residual
            a.aP[n] = 1.0;
            a.aE[n] = 0.0; a.aW[n] = 0.0; a.aN[n] = 0.0; a.aS[n] = 0.0; a.aT[n] = 0.0; a.aB[n] = 0.0;
            a.b[n] = 0.0;
            if (a.d) a.d[n] = 0.0;
            continue;
        }
        // ---- gather
        const double epsP = __ldg(a.eps + n), eps0P = __ldg(a.eps0 + n);
        const double phP = __ldg(a.phim + n), ph0P = __ldg(a.phi0 + n);
        double eM[3], eP[3], vM[3], vPl[3], phM[3], phPl[3];
        bool blM[3], blP[3];
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            int Qm[3] = {P[0], P[1], P[2]}, Qp[3] = {P[0], P[1], P[2]};
            Qm[ax] -= 1;
            Qp[ax] += 1;
            const long long im = lin_cl(G, Qm[0], Qm[1], Qm[2]), ip = lin_cl(G, Qp[0], Qp[1], Qp[2]);
            eM[ax] = __ldg(a.eps + im);
            eP[ax] = __ldg(a.eps + ip);
            vM[ax] = __ldg(a.vel[ax] + im);
            vPl[ax] = __ldg(a.vel[ax] + n);
            phM[ax] = __ldg(a.phim + im);
            phPl[ax] = __ldg(a.phim + ip);
            blM[ax] = BL ? (P[ax] >= 1 && __ldg(a.blocked + im) != 0) : false;
            blP[ax] = BL ? (P[ax] < extent(G, ax) - 1 && __ldg(a.blocked + ip) != 0) : false;
        }
        // ---- row
        double as[6], phib[6];
        bool kept[6], inP[6];
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            const int sm = 2 * ax, sp = 2 * ax + 1;
            as[sm] = 0.0; as[sp] = 0.0; phib[sm] = 0.0; phib[sp] = 0.0;
            kept[sm] = false; kept[sp] = false; inP[sm] = false; inP[sp] = false;
            if (P[ax] >= 1 && blM[ax]) {
                // internal zero-flux wall (§3.10)
            } else if (P[ax] >= 1) {
                const double e = 0.5 * (eM[ax] + epsP);
                const double eu = a.upwind ? (vM[ax] >= 0.0 ? eM[ax] : epsP) : e;
                const double F = ((a.rho * eu) * G.A[ax]) * vM[ax];
                as[sm] = a.Dc[ax] * e + maxp(F);
                kept[sm] = true; inP[sm] = true;
            } else if (ax == 2 && G.bc_zlo == MFX_BC_INLET) {
                const double F = ((a.rho * epsP) * G.A[2]) * G.w_in;
                as[sm] = 2.0 * (a.Dc[2] * epsP) + maxp(F);
                inP[sm] = true;
                phib[sm] = G.phi_in;
            }
            if (P[ax] <= extent(G, ax) - 2 && blP[ax]) {
                // internal zero-flux wall (§3.10)
            } else if (P[ax] <= extent(G, ax) - 2) {
                const double e = 0.5 * (epsP + eP[ax]);
                const double eu = a.upwind ? (vPl[ax] >= 0.0 ? epsP : eP[ax]) : e;
                const double F = ((a.rho * eu) * G.A[ax]) * vPl[ax];
                as[sp] = a.Dc[ax] * e + maxp(-F);
                kept[sp] = true; inP[sp] = true;
            } else if (ax == 2 && G.bc_zhi == MFX_BC_DIRICHLET_TEST) {
                const double F = ((a.rho * epsP) * G.A[2]) * vPl[2];
                as[sp] = 2.0 * (a.Dc[2] * epsP) + maxp(-F);
                inP[sp] = true;
                phib[sp] = G.phi_out;
            }
        }
        const double sum = ((((as[0] + as[1]) + as[2]) + as[3]) + as[4]) + as[5];
        double bcb = 0.0;
#pragma unroll
        for (int s6 = 0; s6 < 6; s6++)
            if (inP[s6] && !kept[s6]) bcb = bcb + as[s6] * phib[s6];
        const double a0 = a.rVdt * eps0P;
        const double aP = sum + a0;
        const double bb = (a0 * ph0P) + bcb;
        const double aPr = aP / a.urf;
        const double bR = bb + (aPr - aP) * phP;
        double st6[6];
#pragma unroll
        for (int s6 = 0; s6 < 6; s6++) st6[s6] = kept[s6] ? as[s6] : 0.0;
        a.aW[n] = st6[0]; a.aE[n] = st6[1];
        a.aS[n] = st6[2]; a.aN[n] = st6[3];
        a.aB[n] = st6[4]; a.aT[n] = st6[5];
        a.aP[n] = aPr;
        a.b[n] = bR;
        if (a.d) a.d[n] = 0.0;
        const bool nonfin = !isfinite(aPr) || !isfinite(bR);
        if (nonfin || aPr == 0.0) latch(a.hdr, nonfin, aPr == 0.0, n);
        double res = bb - aP * phP;
#pragma unroll
        for (int s6 = 0; s6 < 6; s6++) {
            const int ax = s6 / 2;
            const bool plus = s6 & 1;
            const bool inside = plus ? P[ax] < extent(G, ax) - 1 : P[ax] >= 1;
            const double unb = inside ? (plus ? phPl[ax] : phM[ax]) : 0.0;
            res = res + st6[s6] * unb;
        }
        num.add(fabs(res));
        den.add(fabs(aP * phP));
    }
    __shared__ dd sh[(kThreads / 32) * 2];
    dd v[2] = {num.get(), den.get()}, out[2];
    if (grid_reduce_dd<2>(v, a.part, &a.hdr->ticket[0], sh, out) && threadIdx.x == 0 && a.resid2) {
        a.resid2[0] = dd_round(out[0]);
        a.resid2[1] = dd_round(out[1]);
    }
}

// ------------------------------------------------------------------ correction
struct CorrArgs {
    Geo G;
    double urf_p;
    const double *us[3], *dv[3], *pp, *p;
    double *u[3], *pnew;
};

__global__ void __launch_bounds__(kThreads) k_correct(CorrArgs a)
{
    const Geo &G = a.G;
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < G.N;
         n += (long long)gridDim.x * blockDim.x) {
        int P[3];
        decode(G, n, P);
        const double ppP = __ldg(a.pp + n);
#pragma unroll
        for (int ax = 0; ax < 3; ax++) {
            const double vs = __ldg(a.us[ax] + n);
            double out;
            if (P[ax] <= extent(G, ax) - 2) {
                int E[3] = {P[0], P[1], P[2]};
                E[ax] += 1;
                out = vs + __ldg(a.dv[ax] + n) * (ppP - __ldg(a.pp + lin(G, E)));
            } else if (ax == 2 && G.bc_zhi == MFX_BC_OUTLET) {
                out = vs + __ldg(a.dv[ax] + n) * (ppP - 0.0);
            } else {
                out = vs;
            }
            a.u[ax][n] = out;
        }
        a.pnew[n] = __ldg(a.p + n) + a.urf_p * ppP;
    }
}

bool grid_ok(const mfx_grid *g, bool scalar)
{
    if (!g) { set_error("grid is NULL"); return false; }
    if (g->nx < 2 || g->ny < 2 || g->nz < 2) { set_error("grid extents must be >= 2 (got %d %d %d)", g->nx, g->ny, g->nz); return false; }
    if (!(g->dx > 0 && g->dy > 0 && g->dz > 0)) { set_error("spacing must be positive"); return false; }
    if (g->bc_zlo != MFX_BC_WALL && g->bc_zlo != MFX_BC_INLET) { set_error("bc_zlo must be WALL or INLET"); return false; }
    const bool hi_ok = g->bc_zhi == MFX_BC_WALL || g->bc_zhi == MFX_BC_OUTLET ||
                       (scalar && g->bc_zhi == MFX_BC_DIRICHLET_TEST);
    if (!hi_ok) { set_error("bc_zhi %d not allowed for this equation", g->bc_zhi); return false; }
    return true;
}

}  // namespace

bool grid_valid(const mfx_grid *g, bool scalar) { return grid_ok(g, scalar); }

mfx_status assemble_eq(int kind, int sid, const mfx_grid *grid, const mfx_params *pr, const mfx_state *st,
                       const double *const star[6], mfx_eqsys *out, double *resid2, void *ws, size_t wsb,
                       cudaStream_t s)
{
    const bool scalar = kind == MFX_EQ_SCALAR;
    if (!grid_ok(grid, scalar)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(pr && st && out, "NULL params/state/out");
    MFX_ARG_CHECK(kind >= MFX_EQ_U && kind <= MFX_EQ_SCALAR, "bad kind %d", kind);
    const Geo G = make_geo(*grid);
    WsView W;
    if (!ws_view(ws, wsb, G.N, false, W)) return MFX_ERR_ARG;
    const int nb = reduce_grid(G.N);
    const double V = G.V;
    const double rVdt = (pr->rho * V) / pr->dt;
    if (kind <= MFX_EQ_W) {
        MFX_ARG_CHECK(st->eps && st->eps_old && st->u && st->v && st->w && st->u_old && st->v_old && st->w_old &&
                      st->p && st->beta && st->sbeta_u && st->sbeta_v && st->sbeta_w, "NULL state field");
        MFX_ARG_CHECK(out->aP && out->aE && out->aW && out->aN && out->aS && out->aT && out->aB && out->b && out->d,
                      "NULL eqsys array");
        MomArgs a;
        a.G = G;
        a.upwind = pr->face_eps_upwind;
        a.rho = pr->rho;
        a.urf = pr->urf_mom;
        a.gc = pr->g[kind];
        a.rVdt = rVdt;
        for (int t = 0; t < 3; t++) a.Dc[t] = (pr->mu * G.A[t]) / G.h[t];
        a.R.ext[0] = G.nx; a.R.ext[1] = G.ny; a.R.ext[2] = G.nz;
        a.R.bc_zlo = G.bc_zlo; a.R.bc_zhi = G.bc_zhi; a.R.upwind = pr->face_eps_upwind;
        a.R.w_in = G.w_in; a.R.V = G.V;
        a.R.rho = pr->rho; a.R.urf = pr->urf_mom; a.R.gc = pr->g[kind]; a.R.rVdt = rVdt;
        for (int t = 0; t < 3; t++) { a.R.A[t] = G.A[t]; a.R.Dc[t] = a.Dc[t]; }
        a.eps = st->eps; a.eps0 = st->eps_old;
        a.vel0 = st->u; a.vel1 = st->v; a.vel2 = st->w;
        a.uold = kind == 0 ? st->u_old : (kind == 1 ? st->v_old : st->w_old);
        a.S = kind == 0 ? st->sbeta_u : (kind == 1 ? st->sbeta_v : st->sbeta_w);
        a.p = st->p; a.beta = st->beta;
        a.blocked = st->blocked;
        a.aP = out->aP; a.aE = out->aE; a.aW = out->aW; a.aN = out->aN; a.aS = out->aS; a.aT = out->aT;
        a.aB = out->aB; a.b = out->b; a.d = out->d;
        a.resid2 = resid2; a.hdr = W.hdr; a.part = W.part;
        count_launch(4, s, true);
        // odd nx (rows not 16-byte aligned for TMA): grid-stride kernel; BLOCKED
        // cells (§3.10) take either kernel (the same row decisions in both)
        if (opt_asm_tma() && grid->nx % 2 == 0) {
            const mfx_status rc = assemble_mom_tma(kind, G, pr, st, out, resid2, W.hdr, W.part, s);
            count_launch(4, s, false);
            return rc;
        }
        if (kind == 0) k_assemble_mom<0><<<nb, kThreads, 0, s>>>(a);
        else if (kind == 1) k_assemble_mom<1><<<nb, kThreads, 0, s>>>(a);
        else k_assemble_mom<2><<<nb, kThreads, 0, s>>>(a);
        count_launch(4, s, false);
    } else if (kind == MFX_EQ_PP) {
        MFX_ARG_CHECK(star && star[0] && star[1] && star[2] && star[3] && star[4] && star[5], "p' needs star[6]");
        MFX_ARG_CHECK(st->eps && st->eps_old, "NULL eps");
        MFX_ARG_CHECK(out->aP && out->aE && out->aN && out->aT && out->b && !out->aW && !out->aS && !out->aB,
                      "p' eqsys: aP,aE,aN,aT,b required and aW,aS,aB must be NULL");
        PPArgs a;
        a.G = G;
        a.upwind = pr->face_eps_upwind;
        MFX_ARG_CHECK(!a.upwind || (st->u && st->v && st->w), "upwind p' assembly needs the snapshot u, v, w");
        a.um[0] = st->u; a.um[1] = st->v; a.um[2] = st->w;
        a.rho = pr->rho;
        a.rVdt = rVdt;
        a.eps = st->eps; a.eps0 = st->eps_old;
        a.blocked = st->blocked;
        for (int t = 0; t < 3; t++) { a.us[t] = star[t]; a.dv[t] = star[3 + t]; }
        a.aP = out->aP; a.cx = out->aE; a.cy = out->aN; a.cz = out->aT; a.b = out->b;
        a.resid2 = resid2; a.hdr = W.hdr; a.part = W.part;
        count_launch(8, s, true);
        if (a.upwind && a.blocked) k_assemble_pp<true, true><<<nb, kThreads, 0, s>>>(a);
        else if (a.upwind) k_assemble_pp<true, false><<<nb, kThreads, 0, s>>>(a);
        else if (a.blocked) k_assemble_pp<false, true><<<nb, kThreads, 0, s>>>(a);
        else k_assemble_pp<false, false><<<nb, kThreads, 0, s>>>(a);
        count_launch(8, s, false);
    } else {
        MFX_ARG_CHECK(sid >= 0 && sid < 4, "scalar id %d", sid);
        MFX_ARG_CHECK(st->eps && st->eps_old && st->u && st->v && st->w && st->phi[sid] && st->phi_old[sid],
                      "NULL scalar state field");
        MFX_ARG_CHECK(out->aP && out->aE && out->aW && out->aN && out->aS && out->aT && out->aB && out->b,
                      "NULL eqsys array");
        ScalArgs a;
        a.G = G;
        a.upwind = pr->face_eps_upwind;
        a.rho = pr->rho;
        a.urf = pr->urf_phi;
        a.rVdt = rVdt;
        for (int t = 0; t < 3; t++) a.Dc[t] = (pr->gamma_phi[sid] * G.A[t]) / G.h[t];
        a.eps = st->eps; a.eps0 = st->eps_old;
        a.vel[0] = st->u; a.vel[1] = st->v; a.vel[2] = st->w;
        a.phim = st->phi[sid]; a.phi0 = st->phi_old[sid];
        a.blocked = st->blocked;
        a.aP = out->aP; a.aE = out->aE; a.aW = out->aW; a.aN = out->aN; a.aS = out->aS; a.aT = out->aT;
        a.aB = out->aB; a.b = out->b; a.d = out->d;
        a.resid2 = resid2; a.hdr = W.hdr; a.part = W.part;
        count_launch(9, s, true);
        if (a.blocked) k_assemble_scalar<true><<<nb, kThreads, 0, s>>>(a);
        else k_assemble_scalar<false><<<nb, kThreads, 0, s>>>(a);
        count_launch(9, s, false);
    }
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

mfx_status correct(const mfx_grid *grid, const mfx_params *pr, const double *const star[6], const double *pp,
                   const double *p, double *u, double *v, double *w, double *pnew, cudaStream_t s)
{
    if (!grid_ok(grid, false)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(pr && star && pp && p && u && v && w && pnew, "NULL argument");
    for (int q = 0; q < 6; q++) MFX_ARG_CHECK(star[q], "star[%d] NULL", q);
    CorrArgs a;
    a.G = make_geo(*grid);
    a.urf_p = pr->urf_p;
    for (int t = 0; t < 3; t++) { a.us[t] = star[t]; a.dv[t] = star[3 + t]; }
    a.pp = pp; a.p = p;
    a.u[0] = u; a.u[1] = v; a.u[2] = w; a.pnew = pnew;
    const int nb = reduce_grid(a.G.N);
    count_launch(5, s, true);
    k_correct<<<nb, kThreads, 0, s>>>(a);
    count_launch(5, s, false);
    MFX_CUDA_TRY(cudaGetLastError());
    return MFX_OK;
}

}  // namespace mfx
