"""Seeded synthetic inputs shaped like the paper's fluidized bed.

This module is shared by the oracle tests and the CUDA path. It holds NO
arithmetic of the method (no assembly, no solver, no correction): it only draws
the snapshot fields that the hot path consumes as inputs.  The recipe is stated
in DESIGN.md ("Input recipe") and follows SURVEY.md §8(d):

* domain: L_x = L_y = 0.12 m ("longest side aligned along the z
  direction"), cubic cells Δ = 0.12/nx, L_z = Δ·nz, gravity -z, inlet at z=0,
  outlet at z=L_z, no-slip walls on x and y sides;
* gas: ρ = 1.0 kg/m³, μ = 1.8e-5 Pa·s (PAPER.md:155 BFS values), Δt = 5e-4 s
  (PAPER.md:165/171 maximum time step), inlet w = 0.15 m/s;
* bed: ε = 0.42 ±0.02, bubbles (ε = 0.95, tanh edge) filling 15%
  of the bed, freeboard ε = 1, clamp [0.36, 1]; ε⁰ = ε ± 0.005;
* drag: Syamlal–O'Brien β (closure formulas SPEC.md:283–286)
  with d_p = 200 µm, ρ_p = 2000 kg/m³; S_c = β·u_s,c;
* pressure: gauge hydrostatic bed weight (PAPER.md:125 gauge pressure).

Everything is float64 numpy; `np.random.default_rng(seed)` with
seed = 15605 + config_id for the named configs.
"""
from __future__ import annotations

import dataclasses
import numpy as np

# BC codes, identical numbering to include/mfx.h (mfx_bc).
BC_WALL, BC_INLET, BC_OUTLET, BC_DIRICHLET_TEST = 0, 1, 2, 3

CONFIGS = {
    # id: (nx, ny, nz)  -- BASELINE.json "configs"
    1: (16, 16, 32),
    2: (128, 128, 512),
    3: (64, 64, 256),
    4: (256, 256, 512),
}

FIELD_NAMES = ("eps", "eps_old", "u", "v", "w", "u_old", "v_old", "w_old", "p",
               "beta", "sbeta_u", "sbeta_v", "sbeta_w")


@dataclasses.dataclass
class Grid:
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    bc_zlo: int = BC_INLET
    bc_zhi: int = BC_OUTLET
    w_in: float = 0.15
    phi_in: float = 1.0
    phi_out: float = 0.0

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz


@dataclasses.dataclass
class Params:
    rho: float = 1.0
    mu: float = 1.8e-5
    gamma_phi: tuple = (1.8e-5 / 0.7, 1.8e-5 / 0.7, 1.8e-5 / 1.0, 1.8e-5 / 2.0)
    g: tuple = (0.0, 0.0, -9.81)
    dt: float = 5e-4
    urf_mom: float = 0.7
    urf_p: float = 0.7
    urf_phi: float = 1.0
    tol: float = 1e-3
    lin_tol_mom: float = 1e-4
    lin_tol_pp: float = 1e-6
    lin_tol_phi: float = 1e-4
    lin_maxit_mom: int = 20
    lin_maxit_pp: int = 500
    lin_maxit_phi: int = 20
    face_eps_upwind: int = 0      # DESIGN.md §3.12 (0: central face eps, reading Q9)
    packed_state: int = 0         # multi-rank exchange layout only: u, v, w, p in one [u|v|w|p] block


def syamlal_obrien_beta(eps, slip, d_p=200e-6, rho_g=1.0, mu_g=1.8e-5):
    """Syamlal–O'Brien drag coefficient (input generation only)."""
    eps = np.asarray(eps, dtype=np.float64)
    slip = np.abs(np.asarray(slip, dtype=np.float64))
    eps_p = 1.0 - eps
    re = np.maximum(rho_g * d_p * slip / mu_g, 1e-12)
    a = eps ** 4.14
    b = np.where(eps <= 0.85, 0.8 * eps ** 1.28, eps ** 2.65)
    vr = 0.5 * (a - 0.06 * re + np.sqrt((0.06 * re) ** 2 + 0.12 * re * (2.0 * b - a) + a * a))
    cd = (0.63 + 4.8 / np.sqrt(re / vr)) ** 2
    return 0.75 * cd * (eps_p * eps * rho_g * slip) / (vr * vr * d_p)


def make_grid(nx, ny, nz, bc_zlo=BC_INLET, bc_zhi=BC_OUTLET, w_in=0.15) -> Grid:
    if bc_zlo == BC_WALL:
        w_in = 0.0
    h = 0.12 / nx
    return Grid(nx, ny, nz, h, h, h, bc_zlo=bc_zlo, bc_zhi=bc_zhi, w_in=w_in)


def _fill_bed(rng, grid: Grid):
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    h = grid.dx
    lz = h * nz
    h_bed = min(0.12, 0.5 * lz)
    xc = (np.arange(nx) + 0.5) * grid.dx
    yc = (np.arange(ny) + 0.5) * grid.dy
    zc = (np.arange(nz) + 0.5) * grid.dz
    # arrays are indexed [k, j, i] so that ravel() gives n = i + nx*(j + ny*k)
    z3 = np.broadcast_to(zc[:, None, None], (nz, ny, nx))
    in_bed = z3 < h_bed
    eps = np.where(in_bed, 0.42 + rng.uniform(-0.02, 0.02, (nz, ny, nx)), 1.0)
    # bubbles: radius 3-6 mm, eps = 0.95 with a one-cell tanh edge, 15% of bed volume
    bed_vol = 0.12 * 0.12 * h_bed
    target = 0.15 * bed_vol
    vol = 0.0
    nb = 0
    while vol < target and nb < 100000:
        r = rng.uniform(3e-3, 6e-3)
        c = np.array([rng.uniform(0, 0.12), rng.uniform(0, 0.12), rng.uniform(0, h_bed)])
        vol += 4.0 / 3.0 * np.pi * r ** 3
        nb += 1
        lo = np.maximum(((c - r - 2 * h) / h).astype(int), 0)
        hi = np.minimum(((c + r + 2 * h) / h).astype(int) + 1, [nx, ny, nz])
        if np.any(hi <= lo):
            continue
        X = xc[lo[0]:hi[0]][None, None, :]
        Y = yc[lo[1]:hi[1]][None, :, None]
        Z = zc[lo[2]:hi[2]][:, None, None]
        dist = np.sqrt((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2)
        wgt = 0.5 * (1.0 - np.tanh((dist - r) / h))
        sub = eps[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        bub = sub + wgt * (0.95 - sub)
        sub[...] = np.where(in_bed[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]], np.maximum(sub, bub), sub)
    eps = np.clip(eps, 0.36, 1.0)
    return eps, in_bed, zc, lz, h_bed


def make_state(grid: Grid, seed: int, params: Params | None = None, n_scalars: int = 0):
    """Return a dict of float64 arrays (length N each, x fastest) for one snapshot."""
    params = params or Params()
    rng = np.random.default_rng(seed)
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    eps, in_bed, zc, lz, h_bed = _fill_bed(rng, grid)
    eps_old = np.clip(eps + rng.uniform(-0.005, 0.005, eps.shape), 0.36, 1.0)
    sh = (nz, ny, nx)
    u = rng.normal(0.0, 0.02, sh)
    v = rng.normal(0.0, 0.02, sh)
    w = grid.w_in / eps + rng.normal(0.0, 0.02, sh)
    u_old = u + rng.normal(0.0, 1e-3, sh)
    v_old = v + rng.normal(0.0, 1e-3, sh)
    w_old = w + rng.normal(0.0, 1e-3, sh)
    # stored +side wall faces are identity rows with value 0
    for a in (u, u_old):
        a[:, :, nx - 1] = 0.0
    for a in (v, v_old):
        a[:, ny - 1, :] = 0.0
    if grid.bc_zhi == BC_WALL:
        for a in (w, w_old):
            a[nz - 1, :, :] = 0.0
    g0 = 9.81
    z3 = np.broadcast_to(zc[:, None, None], sh)
    p = 0.58 * 2000.0 * g0 * np.maximum(h_bed - z3, 0.0) + params.rho * g0 * (lz - z3)
    us = np.where(in_bed, rng.normal(0.0, 0.05, (3,) + sh), 0.0)
    wc = np.empty(sh)
    wc[0] = 0.5 * (grid.w_in + w[0])
    wc[1:] = 0.5 * (w[:-1] + w[1:])
    beta = syamlal_obrien_beta(eps, wc - us[2], rho_g=params.rho, mu_g=params.mu)
    st = dict(eps=eps, eps_old=eps_old, u=u, v=v, w=w, u_old=u_old, v_old=v_old, w_old=w_old,
              p=p, beta=beta, sbeta_u=beta * us[0], sbeta_v=beta * us[1], sbeta_w=beta * us[2])
    for s in range(n_scalars):
        st[f"phi{s}"] = np.zeros(sh)
        st[f"phi_old{s}"] = np.zeros(sh)
    return {k: np.ascontiguousarray(a, dtype=np.float64).ravel() for k, a in st.items()}


def config_case(config_id: int, n_scalars: int = 0):
    """(grid, params, state) for BASELINE.json config `config_id` (1..4)."""
    nx, ny, nz = CONFIGS[config_id]
    grid = make_grid(nx, ny, nz)
    params = Params()
    return grid, params, make_state(grid, 15605 + config_id, params, n_scalars)


def random_vector(n: int, seed: int, scale: float = 1.0):
    return np.random.default_rng(seed).uniform(-scale, scale, n)


@dataclasses.dataclass
class PicParams:
    """Parcel properties (d_p = 200 um, rho_p = 2000 kg/m3) and the
    gas-fraction floor of the deposit."""
    d_p: float = 200e-6
    rho_p: float = 2000.0
    eps_min: float = 0.35


# parcels in the paper's bed ("total number of parcels present in
# the domain was 2,983,447"); used for the configuration 2 grid
PAPER_PARCELS = 2_983_447

PARCEL_KEYS = ("x", "y", "z", "u", "v", "w", "omega")


def make_parcels(grid: Grid, seed: int, n_parcels: int, eps=None, pic: PicParams | None = None):
    """Seeded parcels (SoA dict of float64 arrays, DESIGN.md §6 recipe): cells
    drawn with probability proportional to the snapshot's solid fraction
    (1 - eps), positions uniform inside the cell, velocities N(0, 0.05) m/s, one
    statistical weight omega for all parcels such that the parcels carry the
    snapshot's total solid volume.  Sorted by nothing: parcel order is random."""
    pic = pic or PicParams()
    rng = np.random.default_rng(seed)
    n = grid.n
    if eps is None:
        eps = make_state(grid, seed)["eps"]
    solid = np.clip(1.0 - np.asarray(eps, dtype=np.float64), 0.0, None)
    if solid.sum() <= 0.0:
        solid = np.ones(n)
    prob = solid / solid.sum()
    cell = rng.choice(n, size=n_parcels, p=prob)
    i = cell % grid.nx
    j = (cell // grid.nx) % grid.ny
    k = cell // (grid.nx * grid.ny)
    x = (i + rng.uniform(0.0, 1.0, n_parcels)) * grid.dx
    y = (j + rng.uniform(0.0, 1.0, n_parcels)) * grid.dy
    z = (k + rng.uniform(0.0, 1.0, n_parcels)) * grid.dz
    vs = np.pi / 6.0 * pic.d_p ** 3
    total_solid = solid.sum() * grid.dx * grid.dy * grid.dz
    omega = np.full(n_parcels, total_solid / (n_parcels * vs))
    vel = rng.normal(0.0, 0.05, (3, n_parcels))
    out = dict(x=x, y=y, z=z, u=vel[0], v=vel[1], w=vel[2], omega=omega)
    return {k: np.ascontiguousarray(out[k], dtype=np.float64) for k in PARCEL_KEYS}


def bfs_blocked(grid: Grid, step_x: int, step_z: int):
    """BLOCKED flags of a backward-facing step (Fig. 8): the
    block fills x < step_x cells, all y, z < step_z cells.  uint8, N."""
    blocked = np.zeros((grid.nz, grid.ny, grid.nx), dtype=np.uint8)
    blocked[:step_z, :, :step_x] = 1
    return blocked.ravel()


def zero_wall_faces(grid: Grid, state: dict, blocked):
    """Staggered velocities (and their old-time values) on faces that touch a
    BLOCKED cell are wall faces: set them to 0 (input hygiene, no method
    arithmetic)."""
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    bl = np.asarray(blocked).reshape(nz, ny, nx).astype(bool)
    for key, ax in (("u", 2), ("v", 1), ("w", 0)):
        wall = bl.copy()
        src = [slice(None)] * 3
        dst = [slice(None)] * 3
        src[ax] = slice(1, None)
        dst[ax] = slice(0, bl.shape[ax] - 1)
        wall[tuple(dst)] |= bl[tuple(src)]
        for k in (key, key + "_old"):
            if k in state:
                a = state[k].reshape(nz, ny, nx)
                a[wall] = 0.0
    return state


def make_bfs_state(grid: Grid, step_x: int, step_z: int, seed: int, params: Params | None = None):
    """Single-phase backward-facing-step snapshot (rho = 1,
    mu = 1.8e-5, inlet along +z): eps = 1, no drag, w = w_in plus small noise
    in the fluid, u, v small noise, hydrostatic gauge pressure; wall faces 0."""
    params = params or Params()
    rng = np.random.default_rng(seed)
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    sh = (nz, ny, nx)
    blocked = bfs_blocked(grid, step_x, step_z)
    u = rng.normal(0.0, 0.01 * max(grid.w_in, 1e-3), sh)
    v = rng.normal(0.0, 0.01 * max(grid.w_in, 1e-3), sh)
    w = grid.w_in + rng.normal(0.0, 0.01 * max(grid.w_in, 1e-3), sh)
    u[:, :, nx - 1] = 0.0
    v[:, ny - 1, :] = 0.0
    if grid.bc_zhi == BC_WALL:
        w[nz - 1] = 0.0
    zc = (np.arange(nz) + 0.5) * grid.dz
    lz = nz * grid.dz
    p = np.broadcast_to((params.rho * 9.81 * (lz - zc))[:, None, None], sh).copy()
    st = dict(eps=np.ones(sh), eps_old=np.ones(sh), u=u, v=v, w=w, u_old=u.copy(), v_old=v.copy(),
              w_old=w.copy(), p=p, beta=np.zeros(sh), sbeta_u=np.zeros(sh), sbeta_v=np.zeros(sh),
              sbeta_w=np.zeros(sh))
    st = {k: np.ascontiguousarray(a, dtype=np.float64).ravel() for k, a in st.items()}
    zero_wall_faces(grid, st, blocked)
    st["blocked"] = blocked
    return st


# PAPER.md:155, Fig. 8: BFS domain 9.8 x 4.9 x 98 cm, block 4.9 x 4.9 x 9.8 cm,
# inlet 1 m/s along +z; the 10,001,880-cell grid = 126 x 63 x 1260.
BFS_CELLS = (126, 63, 1260)


def bfs_case(nx: int = 126, ny: int = 63, nz: int = 1260, seed: int = 15605 + 10):
    """(grid, params, state) of the paper's backward-facing-step workload at
    nx x ny x nz cells (cubic cells, Delta = 9.8 cm / nx), the block occupying
    half of x and the first tenth of z."""
    h = 0.098 / nx
    grid = Grid(nx, ny, nz, h, h, h, bc_zlo=BC_INLET, bc_zhi=BC_OUTLET, w_in=1.0)
    params = Params()
    state = make_bfs_state(grid, nx // 2, nz // 10, seed, params)
    return grid, params, state
