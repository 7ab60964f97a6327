// mom_row.cuh -- the momentum row of DESIGN.md §3.3 (Eq. 2, P:53;
// BLOCKED cells §3.10, upwinded face eps §3.12) as ONE device function,
// evaluated from already gathered neighbour values.  Used by the grid-stride
// kernel (assemble.cu, values from global memory) and the TMA z-marching
// kernel (assemble_tma.cu, values from shared memory): both produce the same
// bits because they run the same expressions.  CUDA path only.
#pragma once

#include "common.cuh"

namespace mfx {

enum { kInterior = 0, kIdentity = 1, kOutlet = 2 };

struct MomRowPar {
    int ext[3];
    int bc_zlo, bc_zhi, upwind;
    double w_in, A[3], V;
    double rho, urf, gc, rVdt, Dc[3];
};

// Inputs of the row of face (P, E = P + e_C) (E = P on the outlet row), read
// through accessors so that a kernel can fetch them where they are used
// (shared memory) or hand over gathered registers (MomRowIn below).
// [ti][sg]: transverse axis T1/T2, side - / +.  Values at positions outside
// the domain may be anything; the boundary rules never use them.
struct MomRowIn {
    int P[3];
    int type;                                   // kInterior or kOutlet (identity rows never get here)
    double epsP_, epsE_, epsPt_[2][2], epsEt_[2][2];
    double vP_[2][2], vE_[2][2];                // transverse velocity on the +t face of Q / R
    double umP_, umE_, umM_, unb_[6];           // component C at P, E, P - e_C; residual neighbours W..T
    double e0P, e0E, bP, bE, SP, SE, pP, pEv, uoP;
    bool m_wall;                                // face (P - e_C, P) touches a BLOCKED cell
    bool e_ident;                               // row of face (E, E + e_C) is an identity row
    bool nb_wall_[2][2];                        // neighbour row (P + s e_t, E + s e_t) is an internal wall
    __device__ double epsP() const { return epsP_; }
    __device__ double epsE() const { return epsE_; }
    __device__ double epsPt(int ti, int sg) const { return epsPt_[ti][sg]; }
    __device__ double epsEt(int ti, int sg) const { return epsEt_[ti][sg]; }
    __device__ double vP(int ti, int sg) const { return vP_[ti][sg]; }
    __device__ double vE(int ti, int sg) const { return vE_[ti][sg]; }
    __device__ double umP() const { return umP_; }
    __device__ double umE() const { return umE_; }
    __device__ double umM() const { return umM_; }
    __device__ double unb(int s6) const { return unb_[s6]; }
    __device__ bool nb_wall(int ti, int sg) const { return nb_wall_[ti][sg]; }
};

struct MomRowOut {
    double st6[6], aPr, bR, d;
    double res, den;                            // residual terms |res|, |aP u|
};

__device__ __forceinline__ double mom_maxp(double f) { return f > 0.0 ? f : 0.0; }

template <int C, class In>
__device__ __forceinline__ void mom_row(const MomRowPar &a, const In &in, MomRowOut &o)
{
    constexpr int T1 = C == 0 ? 1 : 0, T2 = C == 2 ? 1 : 2;   // transverse axes
    const int *P = in.P;
    double as[6], phib[6];
    bool kept[6], inP[6];
#pragma unroll
    for (int s6 = 0; s6 < 6; s6++) { as[s6] = 0.0; phib[s6] = 0.0; kept[s6] = false; inP[s6] = false; }
    {
        // main axis, minus side: the face at the centre of P
        double vm;
        if (P[C] == 0) vm = (C == 2 && a.bc_zlo == MFX_BC_INLET) ? a.w_in : 0.0;
        else vm = in.m_wall ? 0.0 : in.umM();
        const double Fm = ((a.rho * in.epsP()) * a.A[C]) * (0.5 * (vm + in.umP()));
        const double Dm = a.Dc[C] * in.epsP();
        as[2 * C] = Dm + mom_maxp(Fm);
        inP[2 * C] = true;
        if (P[C] >= 1 && !in.m_wall) kept[2 * C] = true;
        else phib[2 * C] = vm;                                                // B1
        // plus side: the face at the centre of E
        if (in.type == kOutlet) {
            as[2 * C + 1] = 0.0;                                              // B3
        } else {
            const double vE_ = in.e_ident ? 0.0 : in.umE();
            const double Fp = ((a.rho * in.epsE()) * a.A[C]) * (0.5 * (in.umP() + vE_));
            const double Dp = a.Dc[C] * in.epsE();
            as[2 * C + 1] = Dp + mom_maxp(-Fp);
            inP[2 * C + 1] = true;
            if (in.e_ident) phib[2 * C + 1] = 0.0;                            // B1
            else kept[2 * C + 1] = true;
        }
    }
#pragma unroll
    for (int ti = 0; ti < 2; ti++) {
        const int t = ti == 0 ? T1 : T2;
#pragma unroll
        for (int sg = 0; sg < 2; sg++) {
            const int s = sg ? 1 : -1;
            const int side = 2 * t + sg;
            const int pt = P[t] + s;
            const bool nbw = in.nb_wall(ti, sg);
            if (pt >= 0 && pt < a.ext[t] && !nbw) {
                // +t face mass fluxes of Q and R: eps at X and X + e_t
                const double eQ0 = s > 0 ? in.epsP() : in.epsPt(ti, 0), eQ1 = s > 0 ? in.epsPt(ti, 1) : in.epsP();
                const double eR0 = s > 0 ? in.epsE() : in.epsEt(ti, 0), eR1 = s > 0 ? in.epsEt(ti, 1) : in.epsE();
                const double efQ = a.upwind ? (in.vP(ti, sg) >= 0.0 ? eQ0 : eQ1) : 0.5 * (eQ0 + eQ1);
                const double efR = a.upwind ? (in.vE(ti, sg) >= 0.0 ? eR0 : eR1) : 0.5 * (eR0 + eR1);
                const double mQ = ((a.rho * efQ) * a.A[t]) * in.vP(ti, sg);
                const double mR = ((a.rho * efR) * a.A[t]) * in.vE(ti, sg);
                const double F = 0.5 * (mQ + mR);
                const double e4 = 0.25 * (((in.epsP() + in.epsE()) + in.epsPt(ti, sg)) + in.epsEt(ti, sg));
                const double D = a.Dc[t] * e4;
                as[side] = D + mom_maxp(s > 0 ? -F : F);
                inP[side] = true;
                kept[side] = true;
            } else {
                int bc = MFX_BC_WALL;                                          // domain or internal wall
                if (t == 2 && !nbw) bc = s < 0 ? a.bc_zlo : a.bc_zhi;
                if (bc == MFX_BC_OUTLET) continue;                            // B3
                double F = 0.0;
                if (bc == MFX_BC_INLET)
                    F = 0.5 * (((a.rho * in.epsP()) * a.A[2]) * a.w_in + ((a.rho * in.epsE()) * a.A[2]) * a.w_in);
                const double e2 = 0.5 * (in.epsP() + in.epsE());
                const double D = a.Dc[t] * e2;
                as[side] = 2.0 * D + mom_maxp(s > 0 ? -F : F);                // B2, phi_b = 0
                inP[side] = true;
                phib[side] = 0.0;
            }
        }
    }
    const double sum = ((((as[0] + as[1]) + as[2]) + as[3]) + as[4]) + as[5];
    double bcb = 0.0;
#pragma unroll
    for (int s6 = 0; s6 < 6; s6++)
        if (inP[s6] && !kept[s6]) bcb = bcb + as[s6] * phib[s6];
    const double ef = 0.5 * (in.epsP() + in.epsE());
    const double e0f = 0.5 * (in.e0P + in.e0E);
    const double bf = 0.5 * (in.bP + in.bE);
    const double Sf = 0.5 * (in.SP + in.SE);
    const double pE = in.type == kOutlet ? 0.0 : in.pEv;
    const double a0 = a.rVdt * e0f;
    const double aP = (sum + a0) + bf * a.V;
    const double bb = ((((a0 * in.uoP) + (ef * a.A[C]) * (in.pP - pE)) + ((a.rho * ef) * a.gc) * a.V) + Sf * a.V) + bcb;
    o.aPr = aP / a.urf;
    o.bR = bb + (o.aPr - aP) * in.umP();
    o.d = (ef * a.A[C]) / o.aPr;
#pragma unroll
    for (int s6 = 0; s6 < 6; s6++) o.st6[s6] = kept[s6] ? as[s6] : 0.0;
    double res = bb - aP * in.umP();
#pragma unroll
    for (int s6 = 0; s6 < 6; s6++) res = res + o.st6[s6] * in.unb(s6);
    o.res = fabs(res);
    o.den = fabs(aP * in.umP());
}

}  // namespace mfx
