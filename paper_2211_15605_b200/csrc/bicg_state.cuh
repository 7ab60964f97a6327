// bicg_state.cuh -- the scalar part of BiCGSTAB (PAPER.md:111,
// SPEC.md:370-378, readings Q1-Q5) as one set of device functions, shared by
// every solver path that keeps the state machine in device memory: the
// per-phase kernels (bicgstab.cu), the TMA z-marching kernels
// (stencil_tma.cu), the grid-synchronous kernel and the domain-decomposed
// solver (dist_solver.cu).  Each function takes the correctly rounded dot
// products already folded; SC is SolverScalars or a local copy.
#pragma once

#include "common.cuh"

namespace mfx {

// setup: r = b - A x0 has been formed; bb = <b,b>, rr = <r,r> (S:378 b = 0 -> x = 0)
template <class SC>
__device__ __forceinline__ void bicg_setup(SC &s, double bb, double rr, double tol, int maxit)
{
    const double bn = sqrt(bb);
    s.tol = tol; s.maxit = maxit; s.bn = bn; s.rr = rr; s.rn = sqrt(rr);
    s.it = 0; s.status = MFX_NOT_CONVERGED; s.done = 0; s.restarted = 0; s.restarts = 0;
    s.restart_mode = 1;   // r^ = r, p = v = 0, rho = <r^,r> = rr (DESIGN.md §3.6 init)
    s.skip = 0; s.half = 0; s.zero_x = 0;
    s.rho = rr; s.rhn = s.rn; s.rho_prev = 1.0; s.alpha = 1.0; s.omega = 1.0;
    if (bn == 0.0) { s.zero_x = 1; s.done = 1; s.status = MFX_OK; s.rn = 0.0; }
    else if (s.rn <= tol * bn) { s.done = 1; s.status = MFX_OK; }
    else if (maxit <= 0) { s.done = 1; }
}

struct K1Pro {
    double rho, rhn, beta, omega;
    bool rst, newly, breakdown;
};

// K1 prologue: restart / breakdown decision (Q4).  breakdown: second
// breakdown, the solve ends (the caller records MFX_ERR_BREAKDOWN once).
template <class SC>
__device__ __forceinline__ K1Pro bicg_k1_prologue(const SC &S)
{
    K1Pro o;
    double rho = S.rho, rhn = S.rhn, rho_prev = S.rho_prev, alpha = S.alpha, omega = S.omega;
    const double rn = S.rn, rr = S.rr;
    bool rst = S.restart_mode != 0;
    o.newly = false;
    o.breakdown = false;
    if (rst) { rho = rr; rhn = rn; rho_prev = 1.0; alpha = 1.0; omega = 1.0; }
    if (fabs(rho) <= (1e-14 * rhn) * rn) {
        if (S.restarted) {
            o.breakdown = true;
        } else {
            rst = true;
            o.newly = true;
            rho = rr; rhn = rn; rho_prev = 1.0; alpha = 1.0; omega = 1.0;
        }
    }
    o.rho = rho; o.rhn = rhn; o.omega = omega; o.rst = rst;
    o.beta = (rho / rho_prev) * (alpha / omega);
    return o;
}

template <class SC>
__device__ __forceinline__ void bicg_breakdown(SC &S)
{
    S.status = MFX_ERR_BREAKDOWN;
    S.done = 1;
}

// a sigma / t-t / omega breakdown: restart once (the iteration counts), then fail
template <class SC>
__device__ __forceinline__ void bicg_restart_or_fail(SC &S)
{
    if (S.restarted) {
        S.status = MFX_ERR_BREAKDOWN; S.it += 1; S.done = 1;
    } else {
        S.restarted = 1; S.restarts += 1; S.restart_mode = 1; S.skip = 1; S.it += 1;
        if (S.it >= S.maxit) { S.status = MFX_NOT_CONVERGED; S.done = 1; }
    }
}

// after K1: sigma = <r^, v>
template <class SC>
__device__ __forceinline__ void bicg_k1_tail(SC &S, const K1Pro &P, double sigma)
{
    if (P.rst) { S.rho = P.rho; S.rhn = P.rhn; S.rho_prev = 1.0; S.alpha = 1.0; S.omega = 1.0; }
    if (P.newly) { S.restarted = 1; S.restarts += 1; }
    S.restart_mode = 0;
    S.skip = 0;
    S.sigma = sigma;
    if (sigma == 0.0) bicg_restart_or_fail(S);
    else S.alpha = P.rho / sigma;
}

// after K2: <t,s>, <t,t>, <s,s>; half-step exit test on ||s||
template <class SC>
__device__ __forceinline__ void bicg_k2_tail(SC &S, double ts, double tt, double ss)
{
    S.ts = ts; S.tt = tt; S.ss = ss;
    if (sqrt(ss) <= S.tol * S.bn) {
        S.half = 1;
    } else {
        const double om = tt == 0.0 ? 0.0 : ts / tt;
        if (tt == 0.0 || om == 0.0) bicg_restart_or_fail(S);
        else S.omega = om;
    }
}

// after K3: rho = <r^, r>, rr = <r, r> (unused on the half-step exit)
template <class SC>
__device__ __forceinline__ void bicg_k3_tail(SC &S, bool half, double rho, double rr)
{
    S.it += 1;
    if (half) {
        S.rn = sqrt(S.ss);
        S.status = MFX_OK;
        S.done = 1;
        return;
    }
    S.rho_prev = S.rho;
    S.rho = rho;
    S.rr = rr;
    S.rn = sqrt(S.rr);
    if (S.rn <= S.tol * S.bn) { S.status = MFX_OK; S.done = 1; }
    else if (S.it >= S.maxit) { S.status = MFX_NOT_CONVERGED; S.done = 1; }
}

}  // namespace mfx
