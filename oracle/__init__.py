"""CPU fp64 oracle for the SIMPLE + BiCGSTAB hot path -- TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import this package.  The product path
(`paper_2211_15605_b200`) never imports it and shares no code with it; the
only common module is `synth` (seeded input generators, no method arithmetic).

The C source `oracle.c` follows DESIGN.md §3 (the written discrete
definitions), which restates PAPER.md §2.1 Eqs. (1)-(2), §2.2.2 and §3
("No preconditioners") plus the readings listed in DESIGN.md §4.
Pins (tests/test_oracle_*.py) tie it to closed forms, brute force, dense
direct solves and the paper's worked statements.

Parity status per function:
  or_fsum / or_dot / or_sumabs ... pinned (math.fsum, fractions.Fraction)
  or_spmv ........................ pinned (dense matrix brute force)
  or_bicgstab .................... pinned (dense LU, k-eigenvalue count, SPEC examples)
  or_assemble_pp ................. pinned (symmetry, Laplacian closed form, S:367-369,
                                   consistency with Eq. 1 under mesh refinement)
  or_assemble_scalar ............. pinned (geometric recurrence, pure convection,
                                   consistency under mesh refinement)
  or_assemble_mom ................ pinned (quiescent, hydrostatic, inertia-only, dominance;
                                   the general 3-D row with every term active by
                                   consistency with Eq. 2 under mesh refinement)
  or_correct ..................... pinned (continuity identity b(u_corr) = b(u*) - A p')
  or_pic_deposit_eps / or_pic_drag  pinned (partition of unity, node coincidence, symmetry,
                                   trilinear exactness on linear fields, Dalla Valle
                                   single-sphere limit eps_g = 1 -> V_r = 1, Stokes limit,
                                   SPEC.md:290 V_r = A at Re = 0, momentum bookkeeping)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lquadmath", "-lm"])
        os.replace(tmp, _SO)
    return _SO


class OgGrid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("bc_zlo", C.c_int), ("bc_zhi", C.c_int),
                ("w_in", C.c_double), ("phi_in", C.c_double), ("phi_out", C.c_double)]


class OgParams(C.Structure):
    _fields_ = [("rho", C.c_double), ("mu", C.c_double), ("gamma_phi", C.c_double * 4),
                ("g", C.c_double * 3), ("dt", C.c_double), ("urf_mom", C.c_double),
                ("urf_p", C.c_double), ("urf_phi", C.c_double), ("tol", C.c_double),
                ("lin_tol_mom", C.c_double), ("lin_tol_pp", C.c_double), ("lin_tol_phi", C.c_double),
                ("lin_maxit_mom", C.c_int), ("lin_maxit_pp", C.c_int), ("lin_maxit_phi", C.c_int),
                ("face_eps_upwind", C.c_int)]


_DP = C.POINTER(C.c_double)


class OgState(C.Structure):
    _fields_ = [(n, _DP) for n in ("eps", "eps_old", "u", "v", "w", "u_old", "v_old", "w_old",
                                   "p", "beta", "sbeta_u", "sbeta_v", "sbeta_w")] + \
               [("phi", _DP * 4), ("phi_old", _DP * 4), ("blocked", C.c_void_p)]


class OgEqsys(C.Structure):
    _fields_ = [(n, _DP) for n in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d")]


class OgSolveInfo(C.Structure):
    _fields_ = [("iters", C.c_int), ("status", C.c_int), ("restarts", C.c_int),
                ("rel_resid", C.c_double)]


class OgTimeCtrl(C.Structure):
    _fields_ = [("dt", C.c_double), ("dt_min", C.c_double), ("dt_max", C.c_double), ("grow", C.c_double),
                ("shrink", C.c_double), ("grow_threshold", C.c_int), ("max_outer", C.c_int),
                ("time", C.c_double), ("steps", C.c_int), ("rejected", C.c_int)]


class OgParcels(C.Structure):
    _fields_ = [(k, _DP) for k in ("x", "y", "z", "u", "v", "w", "omega")] + [("n", C.c_long)]


class OgPicParams(C.Structure):
    _fields_ = [("d_p", C.c_double), ("eps_min", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.or_fsum.restype = C.c_double
        L.or_fsum.argtypes = [C.c_long, _DP]
        L.or_dot.restype = C.c_double
        L.or_dot.argtypes = [C.c_long, _DP, _DP]
        L.or_sumabs.restype = C.c_double
        L.or_sumabs.argtypes = [C.c_long, _DP]
        L.or_spmv.argtypes = [C.POINTER(OgGrid), C.POINTER(OgEqsys), _DP, _DP]
        L.or_assemble_mom.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams), C.c_int,
                                      C.POINTER(OgState), C.POINTER(OgEqsys), _DP]
        L.or_assemble_pp.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams), C.POINTER(OgState)] + \
            [_DP] * 6 + [C.POINTER(OgEqsys), _DP]
        L.or_assemble_scalar.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams), C.c_int,
                                         C.POINTER(OgState), C.POINTER(OgEqsys), _DP]
        L.or_bicgstab.argtypes = [C.POINTER(OgGrid), C.POINTER(OgEqsys), _DP, C.c_double, C.c_int,
                                  C.POINTER(OgSolveInfo), _DP]
        L.or_correct.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams)] + [_DP] * 12
        L.or_simple_iter.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams), C.c_int,
                                     C.POINTER(OgState), _DP, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_pic_deposit_eps.argtypes = [C.POINTER(OgGrid), C.POINTER(OgPicParams), C.POINTER(OgParcels), _DP]
        L.or_set_mode.argtypes = [C.c_int, C.c_int]
        L.or_max_threads.restype = C.c_int
        L.or_pow_ambiguous.restype = C.c_long
        L.or_pow_ambiguous.argtypes = []
        L.or_pow.restype = C.c_double
        L.or_pow.argtypes = [C.c_double, C.c_double]
        L.or_pic_drag_coef.restype = C.c_double
        L.or_pic_drag_coef.argtypes = [C.POINTER(OgParams), C.POINTER(OgPicParams), C.c_double, C.c_double,
                                       C.c_double]
        L.or_pic_drag.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams), C.POINTER(OgPicParams),
                                  C.POINTER(OgParcels)] + [_DP] * 10
        L.or_adapt_dt.argtypes = [C.POINTER(OgTimeCtrl), C.c_int, C.c_int]
        L.or_time_step.argtypes = [C.POINTER(OgGrid), C.POINTER(OgParams), C.c_int, C.POINTER(OgState),
                                   C.POINTER(OgTimeCtrl), C.POINTER(C.c_int), _DP]
        _lib = L
    return _lib


# ---------------------------------------------------------------- marshalling
def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_DP)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def c_grid(grid) -> OgGrid:
    return OgGrid(grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz, grid.bc_zlo, grid.bc_zhi,
                  grid.w_in, grid.phi_in, grid.phi_out)


def c_params(pr) -> OgParams:
    return OgParams(pr.rho, pr.mu, (C.c_double * 4)(*pr.gamma_phi), (C.c_double * 3)(*pr.g), pr.dt,
                    pr.urf_mom, pr.urf_p, pr.urf_phi, pr.tol, pr.lin_tol_mom, pr.lin_tol_pp,
                    pr.lin_tol_phi, pr.lin_maxit_mom, pr.lin_maxit_pp, pr.lin_maxit_phi,
                    int(getattr(pr, "face_eps_upwind", 0)))


class _State:
    """Keeps numpy arrays alive while the C struct points at them."""

    def __init__(self, st: dict, n: int):
        self.arrays = {k: (_f64(v).copy() if k != "blocked" else v) for k, v in st.items()}
        for k in ("eps", "eps_old", "u", "v", "w", "u_old", "v_old", "w_old", "p", "beta",
                  "sbeta_u", "sbeta_v", "sbeta_w"):
            self.arrays.setdefault(k, np.zeros(n))
        phis = [self.arrays.setdefault(f"phi{s}", np.zeros(n)) for s in range(4)]
        phios = [self.arrays.setdefault(f"phi_old{s}", np.zeros(n)) for s in range(4)]
        a = self.arrays
        blocked = st.get("blocked")
        self.blocked = None if blocked is None else np.ascontiguousarray(blocked, dtype=np.uint8)
        a.pop("blocked", None)
        self.c = OgState(*[_p(a[k]) for k in ("eps", "eps_old", "u", "v", "w", "u_old", "v_old",
                                              "w_old", "p", "beta", "sbeta_u", "sbeta_v", "sbeta_w")],
                         (_DP * 4)(*[_p(x) for x in phis]), (_DP * 4)(*[_p(x) for x in phios]),
                         None if self.blocked is None else self.blocked.ctypes.data)


SYS_KEYS = ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d")
PP_KEYS = ("aP", "aE", "aN", "aT", "b")   # aE/aN/aT hold c_x/c_y/c_z


def _eqsys(d: dict) -> OgEqsys:
    return OgEqsys(*[_p(d.get(k)) for k in SYS_KEYS])


# ---------------------------------------------------------------- API
def fsum(x) -> float:
    x = _f64(x)
    return lib().or_fsum(x.size, _p(x))


def dot(a, b) -> float:
    a, b = _f64(a), _f64(b)
    assert a.size == b.size
    return lib().or_dot(a.size, _p(a), _p(b))


def sumabs(x) -> float:
    x = _f64(x)
    return lib().or_sumabs(x.size, _p(x))


def spmv(grid, sysd: dict, x):
    x = _f64(x)
    y = np.empty(grid.n)
    cg = c_grid(grid)
    lib().or_spmv(C.byref(cg), C.byref(_eqsys(sysd)), _p(x), _p(y))
    return y


def assemble_mom(grid, params, comp: int, state: dict):
    n = grid.n
    S = _State(state, n)
    out = {k: np.zeros(n) for k in SYS_KEYS}
    r2 = np.zeros(2)
    cg, cp = c_grid(grid), c_params(params)
    rc = lib().or_assemble_mom(C.byref(cg), C.byref(cp), comp, C.byref(S.c), C.byref(_eqsys(out)), _p(r2))
    return out, r2, rc


def assemble_scalar(grid, params, sid: int, state: dict):
    n = grid.n
    S = _State(state, n)
    out = {k: np.zeros(n) for k in SYS_KEYS}
    r2 = np.zeros(2)
    cg, cp = c_grid(grid), c_params(params)
    rc = lib().or_assemble_scalar(C.byref(cg), C.byref(cp), sid, C.byref(S.c), C.byref(_eqsys(out)), _p(r2))
    return out, r2, rc


def assemble_pp(grid, params, state: dict, star, dvec):
    n = grid.n
    S = _State(state, n)
    out = {k: np.zeros(n) for k in PP_KEYS}
    cont = np.zeros(1)
    star = [_f64(a) for a in star]
    dvec = [_f64(a) for a in dvec]
    cg, cp = c_grid(grid), c_params(params)
    rc = lib().or_assemble_pp(C.byref(cg), C.byref(cp), C.byref(S.c), *[_p(a) for a in star],
                              *[_p(a) for a in dvec], C.byref(_eqsys(out)), _p(cont))
    return out, float(cont[0]), rc


def bicgstab(grid, sysd: dict, x0, tol: float, maxit: int, trace: bool = False):
    x = _f64(x0).copy()
    info = OgSolveInfo()
    tr = np.zeros((max(maxit, 1), 8)) if trace else None
    cg = c_grid(grid)
    lib().or_bicgstab(C.byref(cg), C.byref(_eqsys(sysd)), _p(x), tol, maxit, C.byref(info),
                      _p(tr) if trace else None)
    res = dict(x=x, iters=info.iters, status=info.status, restarts=info.restarts, rel_resid=info.rel_resid)
    if trace:
        res["trace"] = tr[:max(info.iters, 0)]
    return res


def correct(grid, params, star, dvec, pp, p):
    n = grid.n
    outs = [np.zeros(n) for _ in range(4)]
    args = [_f64(a) for a in (*star, *dvec, pp, p)]
    cg, cp = c_grid(grid), c_params(params)
    lib().or_correct(C.byref(cg), C.byref(cp), *[_p(a) for a in args], *[_p(a) for a in outs])
    return outs  # u, v, w, p


def simple_iter(grid, params, state: dict, n_scalars: int = 0):
    """One SIMPLE outer iteration; returns (new_state, resid[4], iters[8], status[8], rc)."""
    S = _State(state, grid.n)
    resid = np.zeros(4)
    iters = (C.c_int * 8)()
    status = (C.c_int * 8)()
    cg, cp = c_grid(grid), c_params(params)
    rc = lib().or_simple_iter(C.byref(cg), C.byref(cp), n_scalars, C.byref(S.c), _p(resid), iters, status)
    return S.arrays, resid, list(iters), list(status), rc


PARCEL_KEYS = ("x", "y", "z", "u", "v", "w", "omega")


class _Parcels:
    def __init__(self, parcels: dict):
        self.arrays = {k: _f64(parcels[k]) for k in PARCEL_KEYS}
        n = self.arrays["x"].size
        assert all(a.size == n for a in self.arrays.values())
        self.c = OgParcels(*[_p(self.arrays[k]) for k in PARCEL_KEYS], n)


def pic_deposit_eps(grid, pic, parcels: dict):
    """§3.9 D1: gas volume fraction from parcel solid volume.
    pic = object with d_p, eps_min.  Returns (eps_g[N], rc)."""
    P = _Parcels(parcels)
    eps = np.zeros(grid.n)
    cg, cpp = c_grid(grid), OgPicParams(pic.d_p, pic.eps_min)
    rc = lib().or_pic_deposit_eps(C.byref(cg), C.byref(cpp), C.byref(P.c), _p(eps))
    return eps, rc


def set_mode(threads: int = 0, naive: bool = False):
    """Threads for the row loops and the exact sums (<= 0: unchanged; results are
    bit-identical for any count); naive=True: plain sums (timing only)."""
    lib().or_set_mode(int(threads), int(bool(naive)))


def max_threads() -> int:
    return int(lib().or_max_threads())


def pow_(x: float, y: float) -> float:
    """§3.9: correctly rounded x^y (x > 0), quad-precision powq rounded once."""
    return lib().or_pow(x, y)


def pic_drag_coef(params, pic, eg: float, slip: float, omega: float = 1.0) -> float:
    cp, cpp = c_params(params), OgPicParams(pic.d_p, pic.eps_min)
    return lib().or_pic_drag_coef(C.byref(cp), C.byref(cpp), eg, slip, omega)


def pic_drag(grid, params, pic, parcels: dict, eps_g, u, v, w, diag: bool = False):
    """§3.9 D2: per-parcel Syamlal-O'Brien drag deposited to cell-centred beta and
    beta*u_s.  Returns dict(beta, sbeta_u,
    sbeta_v, sbeta_w, sabs[3,N], diag[M,5] = eps_g@p, u_g@p, v_g@p, w_g@p, K; rc)."""
    P = _Parcels(parcels)
    n, m = grid.n, P.c.n
    out = {k: np.zeros(n) for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w")}
    sabs = np.zeros((3, n))
    dg = np.zeros((m, 5)) if diag else None
    fields = [_f64(a) for a in (eps_g, u, v, w)]
    cg, cp, cpp = c_grid(grid), c_params(params), OgPicParams(pic.d_p, pic.eps_min)
    rc = lib().or_pic_drag(C.byref(cg), C.byref(cp), C.byref(cpp), C.byref(P.c), *[_p(a) for a in fields],
                           _p(out["beta"]), _p(out["sbeta_u"]), _p(out["sbeta_v"]), _p(out["sbeta_w"]),
                           _p(dg) if diag else None, _p(sabs))
    out["sabs"] = sabs
    out["rc"] = rc
    if diag:
        out["diag"] = dg
    return out


def time_ctrl(dt=1e-3, dt_min=1e-5, dt_max=5e-4, grow=1.1, shrink=0.5, grow_threshold=3, max_outer=10):
    return OgTimeCtrl(dt, dt_min, dt_max, grow, shrink, grow_threshold, max_outer, 0.0, 0, 0)


def adapt_dt(tc: OgTimeCtrl, outer_iters: int, converged: bool) -> bool:
    """§3.11 controller; updates tc in place, True if accepted."""
    return bool(lib().or_adapt_dt(C.byref(tc), outer_iters, int(converged)))


def time_step(grid, params, state: dict, tc: OgTimeCtrl, n_scalars: int = 0):
    """One accepted time step (§3.11): returns (new_state, outer_iters, resid[4], rc); tc updated."""
    S = _State(state, grid.n)
    resid = np.zeros(4)
    its = C.c_int()
    cg, cp = c_grid(grid), c_params(params)
    rc = lib().or_time_step(C.byref(cg), C.byref(cp), n_scalars, C.byref(S.c), C.byref(tc), C.byref(its),
                            _p(resid))
    out = dict(S.arrays)
    if S.blocked is not None:
        out["blocked"] = S.blocked
    return out, its.value, resid, rc


# ---------------------------------------------------------------- helpers for pins
def dense_matrix(grid, sysd: dict):
    """Dense A (N x N) built by applying the oracle's own 7-point rows to unit vectors."""
    n = grid.n
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        A[:, j] = spmv(grid, sysd, e)
    return A


def digits_matching(ref, other):
    """Eq. (6): -log10 |a - b| / |a|, 16 for exact, clamp to [-5, 16]; NaN where ref == 0."""
    ref = np.asarray(ref, dtype=np.float64)
    other = np.asarray(other, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        d = -np.log10(np.abs(ref - other) / np.abs(ref))
    d = np.where(ref == other, 16.0, d)
    d = np.clip(d, -5.0, 16.0)
    return np.where(ref == 0.0, np.nan, d)
