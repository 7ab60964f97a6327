"""Python binding of libmfx.so (include/mfx.h) -- argument marshalling only.

Every step of the hot path (assembly, 7-point apply, BiCGSTAB, correction,
SIMPLE orchestration, NCCL exchange) runs inside libmfx.so's sm_100a kernels.
torch supplies device memory, streams and the process group used to ship the
NCCL unique id.  There is no CPU fallback: if the library is missing this
module raises ImportError, and every call raises MfxError on a non-OK status.

Names follow include/mfx.h (§2.2.2 notation: U/V/W/P devices,
assignment strings such as "111[1]" and "234[1]5678").
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("MFX_SO_VARIANT") or os.path.join(_HERE, "libmfx.so")   # variant: A/B builds only
if not os.path.exists(_SO):
    raise ImportError(f"{_SO} is not built: run `python paper_2211_15605_b200/build.py` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(_SO, mode=C.RTLD_GLOBAL)

EQ_U, EQ_V, EQ_W, EQ_PP, EQ_SCALAR = 0, 1, 2, 3, 4
BC_WALL, BC_INLET, BC_OUTLET, BC_DIRICHLET_TEST = 0, 1, 2, 3
OK, NOT_CONVERGED, ERR_ARG, ERR_NONFINITE, ERR_ZERO_DIAG, ERR_BREAKDOWN, ERR_CUDA, ERR_NCCL = 0, 1, -1, -2, -3, -4, -5, -6
OP_SEND, OP_RECV, OP_BCAST = 0, 1, 2
BUF_NAMES = ("u", "v", "w", "dx", "dy", "dz", "p", "phi0", "phi1", "phi2", "phi3", "meta", "pp",
             "beta", "sbeta_u", "sbeta_v", "sbeta_w")
PIC_OFF, PIC_EXPLICIT, PIC_IMPLICIT = 0, 1, 2
NBUF = len(BUF_NAMES)


class MfxError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: status {status}: {_lib.mfx_last_error().decode()}")


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("bc_zlo", C.c_int), ("bc_zhi", C.c_int),
                ("w_in", C.c_double), ("phi_in", C.c_double), ("phi_out", C.c_double)]


class Params(C.Structure):
    _fields_ = [("rho", C.c_double), ("mu", C.c_double), ("gamma_phi", C.c_double * 4),
                ("g", C.c_double * 3), ("dt", C.c_double), ("urf_mom", C.c_double),
                ("urf_p", C.c_double), ("urf_phi", C.c_double), ("tol", C.c_double),
                ("lin_tol_mom", C.c_double), ("lin_tol_pp", C.c_double), ("lin_tol_phi", C.c_double),
                ("lin_maxit_mom", C.c_int), ("lin_maxit_pp", C.c_int), ("lin_maxit_phi", C.c_int),
                ("face_eps_upwind", C.c_int), ("packed_state", C.c_int)]


_DP = C.POINTER(C.c_double)
STATE_KEYS = ("eps", "eps_old", "u", "v", "w", "u_old", "v_old", "w_old", "p", "beta",
              "sbeta_u", "sbeta_v", "sbeta_w")
SYS_KEYS = ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d")


class State(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in STATE_KEYS] + [("phi", C.c_void_p * 4), ("phi_old", C.c_void_p * 4),
                                                        ("blocked", C.c_void_p)]


class Eqsys(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in SYS_KEYS]


class SolveInfo(C.Structure):
    _fields_ = [("iters", C.c_int), ("status", C.c_int), ("restarts", C.c_int), ("rel_resid", C.c_double),
                ("true_rel_resid", C.c_double)]


class Resid(C.Structure):
    _fields_ = [("R_u", C.c_double), ("R_v", C.c_double), ("R_w", C.c_double), ("R_cont", C.c_double),
                ("R_phi", C.c_double * 4), ("iters", C.c_int * 8), ("status", C.c_int * 8),
                ("converged", C.c_int), ("rel_resid", C.c_double * 8), ("true_rel_resid", C.c_double * 8)]


class Assignment(C.Structure):
    _fields_ = [("owner", C.c_int * 8), ("n_scalars", C.c_int), ("n_ranks_used", C.c_int), ("n_p", C.c_int),
                ("p_rank", C.c_int * 9)]


class Xfer(C.Structure):
    _fields_ = [("op", C.c_int), ("peer", C.c_int), ("buf", C.c_int), ("slot", C.c_int), ("nslots", C.c_int),
                ("k0", C.c_int), ("k1", C.c_int)]


class Parcels(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("x", "y", "z", "u", "v", "w", "omega")] + [("n", C.c_longlong)]


class PicParams(C.Structure):
    _fields_ = [("d_p", C.c_double), ("eps_min", C.c_double)]


PARCEL_KEYS = ("x", "y", "z", "u", "v", "w", "omega")


class TimeCtrl(C.Structure):
    """mfx_time_ctrl (include/mfx.h): adaptive dt controller state."""
    _fields_ = [("dt", C.c_double), ("dt_min", C.c_double), ("dt_max", C.c_double), ("grow", C.c_double),
                ("shrink", C.c_double), ("grow_threshold", C.c_int), ("max_outer", C.c_int),
                ("time", C.c_double), ("steps", C.c_int), ("rejected", C.c_int)]


def time_ctrl(dt=1e-3, dt_min=1e-5, dt_max=5e-4, grow=1.1, shrink=0.5, grow_threshold=3, max_outer=10) -> TimeCtrl:
    return TimeCtrl(dt, dt_min, dt_max, grow, shrink, grow_threshold, max_outer, 0.0, 0, 0)

_V = C.c_void_p
_sigs = {
    "mfx_last_error": (C.c_char_p, []),
    "mfx_version": (C.c_char_p, []),
    "mfx_workspace_bytes": (C.c_size_t, [C.POINTER(Grid), C.c_int]),
    "mfx_ws_init": (C.c_int, [_V, C.c_size_t, _V]),
    "mfx_ws_check": (C.c_int, [_V, C.c_size_t, _V]),
    "mfx_assemble_eq": (C.c_int, [C.c_int, C.c_int, C.POINTER(Grid), C.POINTER(Params), C.POINTER(State),
                                  C.POINTER(_V), C.POINTER(Eqsys), _V, _V, C.c_size_t, _V]),
    "mfx_pic_deposit_eps": (C.c_int, [C.POINTER(Grid), C.POINTER(PicParams), C.POINTER(Parcels), _V, _V,
                                      C.c_size_t, _V]),
    "mfx_pic_sort_scratch_bytes": (C.c_size_t, [C.POINTER(Grid), C.c_longlong]),
    "mfx_pic_sort": (C.c_int, [C.POINTER(Grid), C.POINTER(PicParams), C.POINTER(Parcels), C.POINTER(_V), _V, _V,
                               _V, C.c_size_t, _V]),
    "mfx_pic_deposit_eps_binned": (C.c_int, [C.POINTER(Grid), C.POINTER(PicParams), C.POINTER(Parcels), _V, _V,
                                             _V, _V, _V, C.c_size_t, _V]),
    "mfx_pic_drag_binned": (C.c_int, [C.POINTER(Grid), C.POINTER(Params), C.POINTER(PicParams), C.POINTER(Parcels),
                                      _V, _V] + [_V] * 10 + [_V, C.c_size_t, _V]),
    "mfx_pic_drag": (C.c_int, [C.POINTER(Grid), C.POINTER(Params), C.POINTER(PicParams), C.POINTER(Parcels)] +
                     [_V] * 9 + [_V, C.c_size_t, _V]),
    "mfx_state_dump": (C.c_int, [C.c_char_p, C.POINTER(Grid), C.POINTER(State), C.c_int, C.POINTER(Parcels),
                                 C.c_double, C.c_double, _V]),
    "mfx_dump_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_int),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "mfx_state_load": (C.c_int, [C.c_char_p, C.POINTER(Grid), C.POINTER(State), C.c_int, C.POINTER(_V),
                                 C.c_longlong, C.POINTER(C.c_longlong), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), _V]),
    "mfx_spmv": (C.c_int, [C.c_int, C.POINTER(Grid), C.POINTER(Eqsys), _V, _V, _V]),
    "mfx_bicgstab_solve": (C.c_int, [C.c_int, C.POINTER(Grid), C.POINTER(Eqsys), _V, C.c_double, C.c_int,
                                     _V, C.c_size_t, C.POINTER(SolveInfo), _V]),
    "mfx_correct": (C.c_int, [C.POINTER(Grid), C.POINTER(Params), C.POINTER(_V), _V, _V, _V, _V, _V, _V, _V]),
    "mfx_parse_assignment": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(Assignment)]),
    "mfx_exchange_plan": (C.c_int, [C.POINTER(Assignment), C.c_int, C.c_int, C.POINTER(Xfer), C.c_int,
                                    C.POINTER(C.c_int), C.c_int]),
    "mfx_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "mfx_ctx_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.POINTER(Grid), C.POINTER(Params),
                                 C.POINTER(_V)]),
    "mfx_ctx_destroy": (None, [_V]),
    "mfx_local_group_create": (C.c_int, [C.c_int, C.POINTER(_V)]),
    "mfx_local_group_destroy": (None, [_V]),
    "mfx_ctx_create_local": (C.c_int, [C.c_char_p, C.c_int, C.c_int, _V, C.POINTER(Grid), C.POINTER(Params),
                                       C.POINTER(_V)]),
    "mfx_exchange_state": (C.c_int, [_V, C.c_int, C.POINTER(_V), _V]),
    "mfx_simple_iter": (C.c_int, [_V, C.POINTER(State), C.POINTER(Resid), _V]),
    "mfx_ctx_phase_times": (C.c_int, [_V, C.POINTER(C.c_double)]),
    "mfx_ctx_buffer": (C.c_void_p, [_V, C.c_int]),
    "mfx_ctx_set_pic": (C.c_int, [_V, C.POINTER(Parcels), C.POINTER(PicParams), C.c_int]),
    "mfx_adapt_dt": (C.c_int, [C.POINTER(TimeCtrl), C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "mfx_time_step": (C.c_int, [_V, C.POINTER(State), C.POINTER(TimeCtrl), C.POINTER(Resid), C.POINTER(C.c_int), _V]),
    "mfx_dist_solve": (C.c_int, [_V, C.c_int, C.POINTER(Grid), C.POINTER(Eqsys), _V, C.c_double, C.c_int,
                                 C.POINTER(SolveInfo), _V]),
    "mfx_dist_slab": (None, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "mfx_prof_enable": (None, [C.c_int]),
    "mfx_prof_reset": (None, []),
    "mfx_prof_read": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "mfx_launch_count": (C.c_longlong, []),
    "mfx_graph_cache_clear": (None, []),
    "mfx_graph_cache_size": (C.c_size_t, []),
    "mfx_set_option": (C.c_int, [C.c_char_p, C.c_int]),
    "mfx_get_option": (C.c_int, [C.c_char_p]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
EXPORTED = tuple(_sigs)


def lib():
    return _lib


def _check(st, where, ok=(OK,)):
    if st not in ok:
        raise MfxError(st, where)
    return st


def version() -> str:
    return _lib.mfx_version().decode()


def last_error() -> str:
    return _lib.mfx_last_error().decode()


# ---------------------------------------------------------------- marshalling helpers
def c_grid(g) -> Grid:
    return Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz, g.bc_zlo, g.bc_zhi, g.w_in,
                getattr(g, "phi_in", 1.0), getattr(g, "phi_out", 0.0))


def c_params(p) -> Params:
    return Params(p.rho, p.mu, (C.c_double * 4)(*p.gamma_phi), (C.c_double * 3)(*p.g), p.dt, p.urf_mom,
                  p.urf_p, p.urf_phi, p.tol, p.lin_tol_mom, p.lin_tol_pp, p.lin_tol_phi,
                  p.lin_maxit_mom, p.lin_maxit_pp, p.lin_maxit_phi, int(getattr(p, "face_eps_upwind", 0)),
                  int(getattr(p, "packed_state", 0)))


def _ptr(t, n=None):
    if t is None:
        return None
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return t.data_ptr()


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def c_state(state: dict, n: int) -> State:
    st = State(*[_ptr(state.get(k), n) for k in STATE_KEYS])
    for s in range(4):
        st.phi[s] = _ptr(state.get(f"phi{s}"), n)
        st.phi_old[s] = _ptr(state.get(f"phi_old{s}"), n)
    b = state.get("blocked")
    if b is not None:
        import torch
        if not (b.is_cuda and b.dtype == torch.uint8 and b.is_contiguous() and b.numel() == n):
            raise ValueError("blocked must be a contiguous uint8 CUDA tensor of N flags")
        st.blocked = b.data_ptr()
    return st


def c_sys(sysd: dict, n: int) -> Eqsys:
    return Eqsys(*[_ptr(sysd.get(k), n) for k in SYS_KEYS])


def new_system(kind: int, n: int, device="cuda"):
    import torch
    keys = ("aP", "aE", "aN", "aT", "b") if kind == EQ_PP else SYS_KEYS
    return {k: torch.empty(n, dtype=torch.float64, device=device) for k in keys}


class Workspace:
    """Device workspace for one equation (reduction scratch + 7 solver vectors)."""

    def __init__(self, grid, kind: int = 0, device="cuda", stream=None):
        import torch
        self.nbytes = int(_lib.mfx_workspace_bytes(C.byref(c_grid(grid)), kind))
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8, device=device)
        off = (-self.buf.data_ptr()) % 256
        self.ptr = self.buf.data_ptr() + off
        _check(_lib.mfx_ws_init(self.ptr, self.nbytes, _stream(stream)), "mfx_ws_init")

    def check(self, stream=None):
        return _check(_lib.mfx_ws_check(self.ptr, self.nbytes, _stream(stream)), "mfx_ws_check")


# ---------------------------------------------------------------- hot-path entry points
def assemble_eq(kind, grid, params, state: dict, ws: Workspace, star=None, out=None, resid2=None,
                scalar_id: int = 0, stream=None):
    """a-1/a-2/a-3. Returns (system dict, resid2 device tensor[2])."""
    import torch
    n = grid.nx * grid.ny * grid.nz
    dev = state["eps"].device
    out = out if out is not None else new_system(kind, n, dev)
    resid2 = resid2 if resid2 is not None else torch.zeros(2, dtype=torch.float64, device=dev)
    cs = c_state(state, n)
    sarr = None
    if star is not None:
        sarr = (C.c_void_p * 6)(*[_ptr(t, n) for t in star])
    _check(_lib.mfx_assemble_eq(kind, scalar_id, C.byref(c_grid(grid)), C.byref(c_params(params)), C.byref(cs),
                                sarr, C.byref(c_sys(out, n)), _ptr(resid2), C.c_void_p(ws.ptr), ws.nbytes,
                                _stream(stream)), "mfx_assemble_eq")
    return out, resid2


def spmv(kind, grid, sysd: dict, x, y=None, stream=None):
    import torch
    n = grid.nx * grid.ny * grid.nz
    y = y if y is not None else torch.empty_like(x)
    _check(_lib.mfx_spmv(kind, C.byref(c_grid(grid)), C.byref(c_sys(sysd, n)), _ptr(x, n), _ptr(y, n),
                         _stream(stream)), "mfx_spmv")
    return y


def bicgstab_solve(kind, grid, sysd: dict, x, tol: float, maxit: int, ws: Workspace, sync: bool = True,
                   stream=None):
    """a-5/a-6; x is updated in place. Returns the info dict (sync) or None."""
    n = grid.nx * grid.ny * grid.nz
    info = SolveInfo()
    st = _lib.mfx_bicgstab_solve(kind, C.byref(c_grid(grid)), C.byref(c_sys(sysd, n)), _ptr(x, n), tol, maxit,
                                 C.c_void_p(ws.ptr), ws.nbytes, C.byref(info) if sync else None, _stream(stream))
    _check(st, "mfx_bicgstab_solve", ok=(OK, NOT_CONVERGED, ERR_BREAKDOWN))
    if not sync:
        return None
    return dict(iters=info.iters, status=info.status, restarts=info.restarts, rel_resid=info.rel_resid,
                true_rel_resid=info.true_rel_resid)


def c_parcels(parcels: dict) -> Parcels:
    n = parcels["x"].numel()
    for k in PARCEL_KEYS:
        t = parcels[k]
        if not (t.dtype.is_floating_point and t.element_size() == 8 and t.is_contiguous() and t.numel() == n):
            raise ValueError(f"parcel array {k!r} must be a contiguous float64 tensor of {n} elements")
    return Parcels(*[_ptr(parcels[k], n) for k in PARCEL_KEYS], n)


def pic_deposit_eps(grid, pic, parcels: dict, ws: Workspace, eps=None, stream=None):
    """NEXT-2: gas volume fraction from the parcels' solid volume.
    pic: object with d_p, eps_min.  Returns eps_g (device, N)."""
    import torch
    n = grid.nx * grid.ny * grid.nz
    eps = eps if eps is not None else torch.empty(n, dtype=torch.float64, device=parcels["x"].device)
    _check(_lib.mfx_pic_deposit_eps(C.byref(c_grid(grid)), C.byref(PicParams(pic.d_p, pic.eps_min)),
                                    C.byref(c_parcels(parcels)), _ptr(eps, n), C.c_void_p(ws.ptr), ws.nbytes,
                                    _stream(stream)), "mfx_pic_deposit_eps")
    return eps


def pic_sort(grid, pic, parcels: dict, out: dict | None = None, scratch=None, stream=None) -> dict:
    """Binned copy of the parcels (mfx_pic_sort, deterministic): returns a dict with
    the seven sorted arrays plus 'orig' (int32 view of the original indices) and
    'bin_start' (N + 1)."""
    import torch
    m = parcels["x"].numel()
    n = grid.nx * grid.ny * grid.nz
    dev = parcels["x"].device
    out = out if out is not None else {k: torch.empty(m, dtype=torch.float64, device=dev) for k in PARCEL_KEYS}
    out.setdefault("orig", torch.empty(m, dtype=torch.int32, device=dev))
    out.setdefault("bin_start", torch.empty(n + 1, dtype=torch.int32, device=dev))
    nb = int(_lib.mfx_pic_sort_scratch_bytes(C.byref(c_grid(grid)), m))
    scratch = scratch if scratch is not None else torch.empty(nb, dtype=torch.uint8, device=dev)
    arr = (C.c_void_p * 7)(*[_ptr(out[k], m) for k in PARCEL_KEYS])
    _check(_lib.mfx_pic_sort(C.byref(c_grid(grid)), C.byref(PicParams(pic.d_p, pic.eps_min)),
                             C.byref(c_parcels(parcels)), arr, C.c_void_p(out["orig"].data_ptr()),
                             C.c_void_p(out["bin_start"].data_ptr()), C.c_void_p(scratch.data_ptr()), scratch.numel(),
                             _stream(stream)), "mfx_pic_sort")
    return out


def pic_deposit_eps_binned(grid, pic, binned: dict, ws: Workspace, eps=None, vals=None, stream=None):
    """Deterministic gather eps deposit on binned parcels (bitwise the definition)."""
    import torch
    n = grid.nx * grid.ny * grid.nz
    m = binned["x"].numel()
    dev = binned["x"].device
    eps = eps if eps is not None else torch.empty(n, dtype=torch.float64, device=dev)
    vals = vals if vals is not None else torch.empty(max(4 * m, 1), dtype=torch.float64, device=dev)
    _check(_lib.mfx_pic_deposit_eps_binned(C.byref(c_grid(grid)), C.byref(PicParams(pic.d_p, pic.eps_min)),
                                           C.byref(c_parcels(binned)), C.c_void_p(binned["orig"].data_ptr()),
                                           C.c_void_p(binned["bin_start"].data_ptr()), _ptr(eps, n),
                                           C.c_void_p(vals.data_ptr()), C.c_void_p(ws.ptr), ws.nbytes,
                                           _stream(stream)), "mfx_pic_deposit_eps_binned")
    return eps


def pic_drag_binned(grid, params, pic, binned: dict, eps, u, v, w, ws: Workspace, out=None, K=None, vals=None,
                    stream=None):
    """Deterministic gather drag deposit on binned parcels (bitwise the definition)."""
    import torch
    n = grid.nx * grid.ny * grid.nz
    m = binned["x"].numel()
    dev = eps.device
    out = out if out is not None else {k: torch.empty(n, dtype=torch.float64, device=dev)
                                       for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w")}
    vals = vals if vals is not None else torch.empty(max(7 * m, 1), dtype=torch.float64, device=dev)
    _check(_lib.mfx_pic_drag_binned(C.byref(c_grid(grid)), C.byref(c_params(params)),
                                    C.byref(PicParams(pic.d_p, pic.eps_min)), C.byref(c_parcels(binned)),
                                    C.c_void_p(binned["orig"].data_ptr()), C.c_void_p(binned["bin_start"].data_ptr()),
                                    _ptr(eps, n), _ptr(u, n), _ptr(v, n), _ptr(w, n),
                                    *[_ptr(out[k], n) for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w")],
                                    _ptr(K, m) if K is not None else None, C.c_void_p(vals.data_ptr()),
                                    C.c_void_p(ws.ptr), ws.nbytes, _stream(stream)), "mfx_pic_drag_binned")
    return out


def pic_drag(grid, params, pic, parcels: dict, eps, u, v, w, ws: Workspace, out=None, K=None, stream=None):
    """NEXT-2: Syamlal-O'Brien drag of every parcel deposited to the
    cell-centred beta and beta*u_s (the mfx_state drag inputs).  Returns dict
    beta, sbeta_u, sbeta_v, sbeta_w (device, N); K (per parcel) if given."""
    import torch
    n = grid.nx * grid.ny * grid.nz
    dev = eps.device
    out = out if out is not None else {k: torch.empty(n, dtype=torch.float64, device=dev)
                                       for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w")}
    m = parcels["x"].numel()
    _check(_lib.mfx_pic_drag(C.byref(c_grid(grid)), C.byref(c_params(params)),
                             C.byref(PicParams(pic.d_p, pic.eps_min)), C.byref(c_parcels(parcels)),
                             _ptr(eps, n), _ptr(u, n), _ptr(v, n), _ptr(w, n),
                             *[_ptr(out[k], n) for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w")],
                             _ptr(K, m) if K is not None else None, C.c_void_p(ws.ptr), ws.nbytes,
                             _stream(stream)), "mfx_pic_drag")
    return out


def state_dump(path: str, grid, state: dict, n_scalars: int = 0, parcels: dict | None = None, time: float = 0.0,
               dt: float = 0.0, stream=None):
    """NEXT-4: MPXD dump of a device state (and parcels) -- mfx_state_dump."""
    n = grid.nx * grid.ny * grid.nz
    cp = C.byref(c_parcels(parcels)) if parcels is not None else None
    _check(_lib.mfx_state_dump(os.fsencode(path), C.byref(c_grid(grid)), C.byref(c_state(state, n)), n_scalars, cp,
                               time, dt, _stream(stream)), "mfx_state_dump")


def dump_info(path: str) -> dict:
    """Header of an MPXD dump (host only, no GPU needed)."""
    dims = (C.c_int * 3)()
    np_, ns = C.c_longlong(), C.c_int()
    t, dt = C.c_double(), C.c_double()
    _check(_lib.mfx_dump_info(os.fsencode(path), dims, C.byref(np_), C.byref(ns), C.byref(t), C.byref(dt)),
           "mfx_dump_info")
    return dict(dims=tuple(dims), n_parcels=np_.value, n_scalars=ns.value, time=t.value, dt=dt.value)


def state_load(path: str, grid, state: dict, n_scalars: int = 0, parcels: dict | None = None, stream=None) -> dict:
    """Loads an MPXD dump into existing device tensors (state, optional parcels
    dict with capacity >= the dump's count).  Returns dump_info-like fields."""
    n = grid.nx * grid.ny * grid.nz
    pout, cap = None, 0
    if parcels is not None:
        cap = parcels["x"].numel()
        pout = (C.c_void_p * 7)(*[_ptr(parcels[k], cap) for k in PARCEL_KEYS])
    np_ = C.c_longlong()
    t, dt = C.c_double(), C.c_double()
    _check(_lib.mfx_state_load(os.fsencode(path), C.byref(c_grid(grid)), C.byref(c_state(state, n)), n_scalars,
                               pout, cap, C.byref(np_), C.byref(t), C.byref(dt), _stream(stream)), "mfx_state_load")
    return dict(n_parcels=np_.value, time=t.value, dt=dt.value)


def adapt_dt(tc: TimeCtrl, outer_iters: int, converged: bool) -> bool:
    """Host-side adaptive dt rule (mfx_adapt_dt); returns True if accepted."""
    acc = C.c_int()
    _check(_lib.mfx_adapt_dt(C.byref(tc), outer_iters, int(converged), C.byref(acc)), "mfx_adapt_dt")
    return bool(acc.value)


def correct(grid, params, star, pp, p, out=None, stream=None):
    """a-7. star = (u*, v*, w*, d_x, d_y, d_z). Returns (u, v, w, p_new)."""
    import torch
    n = grid.nx * grid.ny * grid.nz
    out = out if out is not None else [torch.empty_like(pp) for _ in range(4)]
    sarr = (C.c_void_p * 6)(*[_ptr(t, n) for t in star])
    _check(_lib.mfx_correct(C.byref(c_grid(grid)), C.byref(c_params(params)), sarr, _ptr(pp, n), _ptr(p, n),
                            *[_ptr(t, n) for t in out], _stream(stream)), "mfx_correct")
    return out


# ---------------------------------------------------------------- equation decomposition
def parse_assignment(text: str, nranks: int) -> dict:
    a = Assignment()
    _check(_lib.mfx_parse_assignment(text.encode(), nranks, C.byref(a)), "mfx_parse_assignment")
    return dict(owner=list(a.owner), n_scalars=a.n_scalars, n_ranks_used=a.n_ranks_used, n_p=a.n_p,
                p_rank=list(a.p_rank)[:a.n_p])


def exchange_plan(text: str, nranks: int, rank: int, phase: int, nz: int = 0):
    a = Assignment()
    _check(_lib.mfx_parse_assignment(text.encode(), nranks, C.byref(a)), "mfx_parse_assignment")
    ops = (Xfer * 64)()
    n = C.c_int()
    _check(_lib.mfx_exchange_plan(C.byref(a), rank, phase, ops, 64, C.byref(n), nz), "mfx_exchange_plan")
    return [dict(op=o.op, peer=o.peer, buf=BUF_NAMES[o.buf], slot=o.slot, nslots=o.nslots, k0=o.k0, k1=o.k1)
            for o in ops[:n.value]]


def dist_slab(nz: int, rank: int, nranks: int):
    """Global z-planes [k0, k1) owned by `rank` in the domain-decomposed solver."""
    k0, k1 = C.c_int(), C.c_int()
    _lib.mfx_dist_slab(nz, rank, nranks, C.byref(k0), C.byref(k1))
    return k0.value, k1.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.mfx_nccl_unique_id(buf), "mfx_nccl_unique_id")
    return buf.raw


class LocalGroup:
    """In-process transport for `nranks` thread-ranks (mfx_local_group)."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.ptr = C.c_void_p()
        _check(_lib.mfx_local_group_create(nranks, C.byref(self.ptr)), "mfx_local_group_create")

    def close(self):
        if self.ptr:
            _lib.mfx_local_group_destroy(self.ptr)
            self.ptr = C.c_void_p()


class SimpleContext:
    """Per-rank equation-decomposition context (mfx_ctx).  Transport: NCCL when
    `uid` is given (one process per GPU), the in-process LocalGroup when
    `group` is given (thread-ranks), none for nranks == 1."""

    def __init__(self, assignment: str, grid, params, rank: int = 0, nranks: int = 1, uid: bytes | None = None,
                 group: LocalGroup | None = None):
        self.grid, self.params = grid, params
        self.rank, self.nranks = rank, nranks
        self._g, self._p = c_grid(grid), c_params(params)
        self.ptr = C.c_void_p()
        if group is not None:
            _check(_lib.mfx_ctx_create_local(assignment.encode(), rank, nranks, group.ptr, C.byref(self._g),
                                             C.byref(self._p), C.byref(self.ptr)), "mfx_ctx_create_local")
        else:
            _check(_lib.mfx_ctx_create(assignment.encode(), rank, nranks, uid, C.byref(self._g), C.byref(self._p),
                                       C.byref(self.ptr)), "mfx_ctx_create")
        self.assignment = parse_assignment(assignment, nranks)

    def step(self, state: dict, stream=None) -> dict:
        """a-9: one SIMPLE outer iteration; state tensors updated in place."""
        n = self.grid.nx * self.grid.ny * self.grid.nz
        cs = c_state(state, n)
        r = Resid()
        st = _lib.mfx_simple_iter(self.ptr, C.byref(cs), C.byref(r), _stream(stream))
        _check(st, "mfx_simple_iter", ok=(OK, NOT_CONVERGED, ERR_BREAKDOWN))   # NONFINITE/ZERO_DIAG raise
        return dict(R=[r.R_u, r.R_v, r.R_w, r.R_cont], R_phi=list(r.R_phi), iters=list(r.iters),
                    status=list(r.status), converged=bool(r.converged), rel_resid=list(r.rel_resid),
                    true_rel_resid=list(r.true_rel_resid))

    def time_step(self, state: dict, tc: TimeCtrl, stream=None) -> dict:
        """One accepted time step with adaptive dt (mfx_time_step);
        tc is updated in place."""
        n = self.grid.nx * self.grid.ny * self.grid.nz
        cs = c_state(state, n)
        r = Resid()
        its = C.c_int()
        st = _lib.mfx_time_step(self.ptr, C.byref(cs), C.byref(tc), C.byref(r), C.byref(its), _stream(stream))
        _check(st, "mfx_time_step", ok=(OK, NOT_CONVERGED))
        return dict(status=st, outer_iters=its.value, R=[r.R_u, r.R_v, r.R_w, r.R_cont], converged=bool(r.converged))

    def set_pic(self, parcels: dict | None, pic=None, mode: int = PIC_IMPLICIT):
        """Particle -> fluid coupling in the SIMPLE loop: PIC_IMPLICIT
        refreshes the state's drag fields at the head of every step, PIC_EXPLICIT
        at the next step only.  Rank 0 (the PIC device) passes the parcels (device
        tensors, kept alive here); other ranks pass None."""
        self._pic_keep = parcels
        cp = C.byref(c_parcels(parcels)) if parcels is not None else None
        pp = C.byref(PicParams(pic.d_p, pic.eps_min)) if pic is not None else None
        _check(_lib.mfx_ctx_set_pic(self.ptr, cp, pp, mode), "mfx_ctx_set_pic")

    def buffer(self, which: str):
        """Copy of an internal buffer of the last step: 'u*','v*','w*','dx','dy','dz','pp'."""
        idx = ("u*", "v*", "w*", "dx", "dy", "dz", "pp").index(which)
        ptr = _lib.mfx_ctx_buffer(self.ptr, idx)
        if not ptr:
            return None
        n = self.grid.nx * self.grid.ny * self.grid.nz
        return device_view(ptr, n).clone()

    def dist_solve(self, kind: int, sysd_slab: dict, x_slab, tol: float, maxit: int, stream=None) -> dict:
        """Domain-decomposed BiCGSTAB over the context's ranks (this rank's slab)."""
        k0, k1 = dist_slab(self.grid.nz, self.rank, self.nranks)
        n = self.grid.nx * self.grid.ny * (k1 - k0)
        info = SolveInfo()
        st = _lib.mfx_dist_solve(self.ptr, kind, C.byref(self._g), C.byref(c_sys(sysd_slab, n)), _ptr(x_slab, n),
                                 tol, maxit, C.byref(info), _stream(stream))
        _check(st, "mfx_dist_solve", ok=(OK, NOT_CONVERGED, ERR_BREAKDOWN))
        return dict(iters=info.iters, status=info.status, restarts=info.restarts, rel_resid=info.rel_resid,
                true_rel_resid=info.true_rel_resid)

    def phase_times(self):
        ms = (C.c_double * 6)()
        _check(_lib.mfx_ctx_phase_times(self.ptr, ms), "mfx_ctx_phase_times")
        return dict(zip(("momentum", "gather", "pp", "correct", "bcast", "total"), list(ms)))

    def close(self):
        if self.ptr:
            _lib.mfx_ctx_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DevPtr:
    """Minimal __cuda_array_interface__ holder for a raw fp64 device pointer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def device_view(ptr: int, n: int):
    """torch view (no copy) of n doubles at a libmfx-owned device pointer."""
    import torch
    return torch.as_tensor(_DevPtr(ptr, n), device="cuda")


# ---------------------------------------------------------------- instrumentation
PROF_IDS = ("spmv_setup", "K1_mom", "K2_mom", "K3", "assemble_mom", "correct", "K1_pp", "K2_pp",
            "assemble_pp", "assemble_scalar")


def prof_enable(on: bool = True):
    _lib.mfx_prof_enable(1 if on else 0)


def prof_reset():
    _lib.mfx_prof_reset()


def prof_read():
    counts = (C.c_int * 16)()
    ms = (C.c_double * 16)()
    _check(_lib.mfx_prof_read(counts, ms), "mfx_prof_read")
    return {PROF_IDS[i]: dict(launches=counts[i], ms=ms[i]) for i in range(len(PROF_IDS))}


PATH_AUTO, PATH_TMA, PATH_CLUSTER, PATH_V1, PATH_GRID, PATH_PERSIST = 0, 1, 2, 3, 4, 5


def set_option(key: str, value: int):
    """Process-wide options: "solver_path" (PATH_*), "graphs" (0/1)."""
    _check(_lib.mfx_set_option(key.encode(), int(value)), "mfx_set_option")


def get_option(key: str) -> int:
    return int(_lib.mfx_get_option(key.encode()))


def graph_cache_clear():
    """Release every cached BiCGSTAB CUDA graph (mfx_graph_cache_clear)."""
    _lib.mfx_graph_cache_clear()


def graph_cache_size() -> int:
    return int(_lib.mfx_graph_cache_size())


def launch_count() -> int:
    return int(_lib.mfx_launch_count())
