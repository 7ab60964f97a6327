"""Pins of the oracle's BLOCKED cells (NEXT-3 geometry, DESIGN.md §3.10;
PAPER.md:155 "an internal block ... was used to construct the step").

The pin is an exact embedding: a slab of BLOCKED cells along one side of a
grid must act exactly like that side's domain wall.  Every fluid row of the
embedded grid (momentum u, v, w; p'; scalar) equals, bit for bit, the row of
the smaller grid that has a real wall there, and so does a whole SIMPLE
iteration (BiCGSTAB iterates included: the blocked region contributes only
zero rows, and the dot products are correctly rounded).  Fields inside the
block are filled with garbage to show that nothing leaks through a wall.
"""
import numpy as np
import pytest

import synth
from synth import BC_INLET, BC_OUTLET, BC_WALL

NB = 3   # slab thickness (cells)


def small_case(seed=31, n_scalars=1, bc_zlo=BC_INLET):
    g = synth.make_grid(8, 6, 10, bc_zlo=bc_zlo)
    pr = synth.Params(lin_maxit_pp=3000)
    st = synth.make_state(g, seed, pr, n_scalars=n_scalars)
    rng = np.random.default_rng(seed)
    for s in range(n_scalars):
        st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
        st[f"phi{s}"] = st[f"phi_old{s}"].copy()
    return g, pr, st


def embed(g, st, side):
    """Big grid = small grid + NB blocked layers on `side` (x-, x+, y-, y+, z-).
    Returns (G, ST, sl) with sl the fluid-region slice of the [k, j, i] view."""
    nx, ny, nz = g.nx, g.ny, g.nz
    ax = {"x-": 2, "x+": 2, "y-": 1, "y+": 1, "z-": 0}[side]       # axis in [k, j, i] order
    lo = side.endswith("-")
    shape = [nz, ny, nx]
    shape[ax] += NB
    bc_zlo = BC_INLET if side == "z-" else g.bc_zlo                 # the inlet sits under the block
    G = synth.Grid(shape[2], shape[1], shape[0], g.dx, g.dy, g.dz, bc_zlo=bc_zlo, bc_zhi=g.bc_zhi,
                   w_in=0.15 if side == "z-" else g.w_in)
    sl = [slice(None)] * 3
    sl[ax] = slice(NB, None) if lo else slice(0, shape[ax] - NB)
    sl = tuple(sl)
    rng = np.random.default_rng(5)
    blocked = np.ones(shape, dtype=np.uint8)
    blocked[sl] = 0
    ST = {}
    for k, v in st.items():
        big = rng.uniform(3.0, 7.0, shape)                          # garbage inside the block
        big[sl] = v.reshape(nz, ny, nx)
        ST[k] = big
    # staggered velocities on faces touching a blocked cell are wall faces: 0
    bl = blocked.astype(bool)
    for key, a in (("u", 2), ("v", 1), ("w", 0)):
        wall = bl.copy()
        nxt = np.zeros_like(bl)
        idx = [slice(None)] * 3
        idx_src = [slice(None)] * 3
        idx[a] = slice(0, shape[a] - 1)
        idx_src[a] = slice(1, None)
        nxt[tuple(idx)] = bl[tuple(idx_src)]
        wall |= nxt
        for kk in (key, key + "_old"):
            ST[kk][wall] = 0.0
    for k in ST:                      # no scalar inside an obstacle (identity rows phi = 0)
        if k.startswith("phi"):
            ST[k][bl] = 0.0
    ST = {k: np.ascontiguousarray(v).ravel() for k, v in ST.items()}
    ST["blocked"] = blocked.ravel()
    return G, ST, sl


def fluid(G, arr, sl):
    return np.asarray(arr).reshape(G.nz, G.ny, G.nx)[sl].ravel()


SIDES = ["x-", "x+", "y-", "y+", "z-"]


@pytest.mark.parametrize("side", SIDES)
@pytest.mark.parametrize("comp", [0, 1, 2])
def test_blocked_slab_momentum_rows_equal_wall(orc, side, comp):
    bc_zlo = BC_WALL if side == "z-" else BC_INLET
    g, pr, st = small_case(bc_zlo=bc_zlo)
    G, ST, sl = embed(g, st, side)
    ref, r2, rc = orc.assemble_mom(g, pr, comp, st)
    big, R2, RC = orc.assemble_mom(G, pr, comp, ST)
    assert rc == 0 and RC == 0
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d"):
        assert np.array_equal(fluid(G, big[k], sl), ref[k]), (side, comp, k)
    assert np.array_equal(R2, r2)


@pytest.mark.parametrize("side", SIDES)
def test_blocked_slab_pp_and_scalar_rows_equal_wall(orc, side):
    bc_zlo = BC_WALL if side == "z-" else BC_INLET
    g, pr, st = small_case(bc_zlo=bc_zlo)
    G, ST, sl = embed(g, st, side)
    rng = np.random.default_rng(2)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    star = [st["u"], st["v"], st["w"]]
    DV = [rng.uniform(5, 9, G.n) for _ in range(3)]                 # garbage everywhere ...
    STAR = [rng.uniform(5, 9, G.n) for _ in range(3)]
    for a in range(3):                                              # ... but the fluid values
        fluid_view = DV[a].reshape(G.nz, G.ny, G.nx)
        fluid_view[sl] = dv[a].reshape(g.nz, g.ny, g.nx)
        sv = STAR[a].reshape(G.nz, G.ny, G.nx)
        sv[sl] = star[a].reshape(g.nz, g.ny, g.nx)
    ref, cont, rc = orc.assemble_pp(g, pr, st, star, dv)
    big, CONT, RC = orc.assemble_pp(G, pr, ST, STAR, DV)
    assert rc == 0 and RC == 0
    for k in ("aP", "aE", "aN", "aT", "b"):
        assert np.array_equal(fluid(G, big[k], sl), ref[k]), (side, k)
    assert CONT == cont
    blocked = ST["blocked"].astype(bool)
    assert np.all(big["b"][blocked] == 0.0) and np.all(big["aP"][blocked] == 0.0)
    sref, s2, _ = orc.assemble_scalar(g, pr, 0, st)
    sbig, S2, _ = orc.assemble_scalar(G, pr, 0, ST)
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b"):
        assert np.array_equal(fluid(G, sbig[k], sl), sref[k]), (side, k)
    assert np.array_equal(S2, s2)


@pytest.mark.parametrize("side", ["x+", "y-", "z-"])
def test_blocked_slab_simple_iteration_equals_wall(orc, side):
    """Whole SIMPLE iteration (momentum + scalar + p' BiCGSTAB + correction):
    same iteration counts and bitwise-equal fluid fields."""
    bc_zlo = BC_WALL if side == "z-" else BC_INLET
    g, pr, st = small_case(bc_zlo=bc_zlo)
    G, ST, sl = embed(g, st, side)
    ref, R, it, stt, rc = orc.simple_iter(g, pr, st, n_scalars=1)
    big, RB, itb, sttb, rcb = orc.simple_iter(G, pr, ST, n_scalars=1)
    assert it == itb and list(R) == list(RB)
    for k in ("u", "v", "w", "p", "phi0"):
        assert np.array_equal(fluid(G, big[k], sl), ref[k]), (side, k)


def bfs_case(nx=12, ny=6, nz=40, step_x=6, step_z=4, seed=3):
    """Backward-facing step (Fig. 8) in miniature: single phase
    (eps = 1, no drag), inlet along +z on the open half of the bottom, the
    block filling x < step, all y, z < step_z."""
    g = synth.make_grid(nx, ny, nz, bc_zlo=BC_INLET, w_in=1.0)
    pr = synth.Params(lin_tol_mom=1e-10, lin_maxit_mom=200, lin_tol_pp=1e-10, lin_maxit_pp=4000)
    st = synth.make_bfs_state(g, step_x, step_z, seed, pr)
    return g, pr, st


def test_bfs_pp_symmetric_with_empty_block_rows(orc):
    g, pr, st = bfs_case()
    rng = np.random.default_rng(1)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    sysd, cont, rc = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    assert rc == 0
    A = orc.dense_matrix(g, sysd)
    assert np.array_equal(A, A.T)
    blocked = st["blocked"].astype(bool)
    assert np.all(A[blocked] == 0.0) and np.all(A[:, blocked] == 0.0)


def test_bfs_mass_balance(orc):
    """S:149 for the step geometry: iterated SIMPLE drives the global in/out
    mass mismatch below 1e-6 of the inflow (inlet only on the open half)."""
    g, pr, st = bfs_case()
    s = st
    for _ in range(60):
        s, R, it, stt, rc = orc.simple_iter(g, pr, s)
        s = dict(s, blocked=st["blocked"])
        if max(R) < 1e-8:
            break
    nx, ny, nz = g.nx, g.ny, g.nz
    blocked = st["blocked"].reshape(nz, ny, nx).astype(bool)
    a_z = g.dx * g.dy
    m_in = pr.rho * a_z * g.w_in * float((~blocked[0]).sum())
    w = s["w"].reshape(nz, ny, nx)
    m_out = pr.rho * a_z * float(w[nz - 1].sum())
    assert abs(m_out - m_in) <= 1e-6 * m_in
