"""Pins for the oracle's assembly, correction and SIMPLE iteration
(DESIGN.md §3.3-§3.8).

Each test fixes the oracle to something other than itself: closed forms,
exact identities of the discretisation, or the worked examples of
SPEC.md:358-387.  The general rows with every term active are pinned by
consistency with the PDEs under mesh refinement (test_oracle_consistency.py).
"""
import json
import os

import numpy as np
import pytest

import synth
from synth import Grid, Params, BC_WALL, BC_INLET, BC_OUTLET, BC_DIRICHLET_TEST

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
ULP = np.finfo(np.float64).eps


def base_state(g, **kw):
    n = g.n
    st = {k: np.zeros(n) for k in synth.FIELD_NAMES}
    st["eps"] = np.ones(n)
    st["eps_old"] = np.ones(n)
    for k, v in kw.items():
        st[k] = np.broadcast_to(np.asarray(v, dtype=np.float64), (n,)).copy()
    return st


def ijk(g):
    k, j, i = np.meshgrid(np.arange(g.nz), np.arange(g.ny), np.arange(g.nx), indexing="ij")
    return i.ravel(), j.ravel(), k.ravel()


# ----------------------------------------------------------------- p' rows
def test_pp_symmetric_and_diagonal_sum(orc):
    g, pr, st = synth.config_case(1)
    rng = np.random.default_rng(0)
    star = [st["u"], st["v"], st["w"]]
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    s, cont, rc = orc.assemble_pp(g, pr, st, star, dv)
    assert rc == 0
    A = orc.dense_matrix(g, s)
    assert np.array_equal(A, A.T)                      # symmetric by construction
    i, j, k = ijk(g)
    offsum = -(A.sum(axis=1) - np.diag(A))
    outlet = np.where(k == g.nz - 1, s["aT"], 0.0)      # outlet face stays in a_P only
    assert np.allclose(np.diag(A), offsum + outlet, rtol=4 * ULP, atol=0)
    assert cont == pytest.approx(np.abs(s["b"]).sum(), rel=1e-14)


@pytest.mark.parametrize("shape,bc", [((16, 16, 32), (BC_INLET, BC_OUTLET)), ((6, 5, 7), (BC_WALL, BC_OUTLET)),
                                      ((4, 9, 3), (BC_INLET, BC_WALL))])
def test_pp_diagonal_is_ordered_row_sum(orc, shape, bc):
    """a_P = ((((c_W + c_E) + c_S) + c_N) + c_B) + c_T with the
    minus-face coefficients taken from the neighbours' stored c_x, c_y, c_z
    (0 at the minus boundary).  Bitwise: the GPU solver rebuilds a_P this way
    instead of streaming it, so the stored a_P must be exactly this sum."""
    g = synth.make_grid(*shape, bc_zlo=bc[0], bc_zhi=bc[1])
    pr = Params()
    st = synth.make_state(g, 77, pr)
    rng = np.random.default_rng(1)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    s, _, rc = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    assert rc == 0
    sh = (g.nz, g.ny, g.nx)
    cx, cy, cz = (s[k].reshape(sh) for k in ("aE", "aN", "aT"))
    cW = np.zeros(sh); cW[:, :, 1:] = cx[:, :, :-1]
    cS = np.zeros(sh); cS[:, 1:, :] = cy[:, :-1, :]
    cB = np.zeros(sh); cB[1:, :, :] = cz[:-1, :, :]
    rowsum = ((((cW + cx) + cS) + cy) + cB) + cz
    assert np.array_equal(s["aP"].reshape(sh), rowsum)
    assert np.all(cx[:, :, -1] == 0) and np.all(cy[:, -1, :] == 0)      # wall faces
    if bc[1] == BC_WALL:
        assert np.all(cz[-1] == 0)
    else:
        assert np.all(cz[-1] > 0)                                        # outlet face stays in a_P


def test_pp_laplacian_closed_form(orc):
    """eps = 1, uniform d: interior coefficient c = rho A d and A q for a
    quadratic q equals -sum_a 2 c_a h_a^2 exactly (7-point Laplacian of x^2+y^2+z^2)."""
    g = Grid(6, 5, 7, 0.1, 0.2, 0.3, bc_zlo=BC_INLET, bc_zhi=BC_OUTLET)
    pr = Params(rho=1.3)
    st = base_state(g)
    d = [np.full(g.n, 0.01), np.full(g.n, 0.02), np.full(g.n, 0.03)]
    s, _, rc = orc.assemble_pp(g, pr, st, [np.zeros(g.n)] * 3, d)
    assert rc == 0
    A_ = [g.dy * g.dz, g.dx * g.dz, g.dx * g.dy]
    c = [pr.rho * A_[a] * d[a][0] for a in range(3)]
    i, j, k = ijk(g)
    inner = (i > 0) & (i < g.nx - 1) & (j > 0) & (j < g.ny - 1) & (k > 0) & (k < g.nz - 1)
    assert np.allclose(s["aE"][inner], c[0], rtol=2 * ULP)
    assert np.allclose(s["aT"][inner], c[2], rtol=2 * ULP)
    x, y, z = (i + 0.5) * g.dx, (j + 0.5) * g.dy, (k + 0.5) * g.dz
    q = x * x + y * y + z * z
    Aq = orc.spmv(g, s, q)
    h = [g.dx, g.dy, g.dz]
    closed = -sum(2.0 * c[a] * h[a] ** 2 for a in range(3))
    assert np.allclose(Aq[inner], closed, rtol=1e-9)


def test_pp_divergence_free_gives_zero(orc):
    """divergence-free starred field (eps = eps0) -> b = 0 -> p' = 0."""
    g = Grid(5, 4, 6, 0.1, 0.1, 0.1, w_in=0.3)
    pr = Params()
    st = base_state(g)
    ws = np.full(g.n, 0.3)     # uniform plug flow, inlet 0.3, outlet face 0.3
    d = [np.full(g.n, 1e-3)] * 3
    s, cont, rc = orc.assemble_pp(g, pr, st, [np.zeros(g.n), np.zeros(g.n), ws], d)
    assert rc == 0 and cont == 0.0 and np.all(s["b"] == 0.0)
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-6, 100)
    assert res["iters"] == 0 and np.all(res["x"] == 0.0)


def test_pp_two_cell_imbalance(orc):
    """two cells with imbalance -m/+m across one face:
    p'_1 - p'_0 = m / c_f (closed box, all other faces shut)."""
    g = Grid(2, 2, 2, 0.1, 0.1, 0.1, bc_zlo=BC_WALL, bc_zhi=BC_WALL)
    pr = Params()
    st = base_state(g)
    i, j, k = ijk(g)
    U = 0.2
    us = np.where(i == 0, U, 0.0)
    dx = np.where(i == 0, 2e-3, 0.0)
    s, _, rc = orc.assemble_pp(g, pr, st, [us, np.zeros(g.n), np.zeros(g.n)],
                               [dx, np.zeros(g.n), np.zeros(g.n)])
    assert rc == 0
    m = pr.rho * 1.0 * (g.dy * g.dz) * U
    c = pr.rho * 1.0 * (g.dy * g.dz) * 2e-3
    assert np.allclose(s["b"], np.where(i == 0, -m, m), rtol=1e-15)
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-12, 10)
    x = res["x"]
    assert np.allclose(x[i == 1] - x[i == 0], GOLD["pp_two_cell"]["m_over_c"] * m / c, rtol=1e-14)


def test_pp_all_neumann_null_space(orc):
    """with no outlet the p' operator annihilates constants."""
    g = Grid(4, 3, 5, 0.1, 0.1, 0.1, bc_zlo=BC_WALL, bc_zhi=BC_WALL)
    rng = np.random.default_rng(3)
    st = base_state(g, eps=rng.uniform(0.4, 1.0, g.n))
    d = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    s, _, _ = orc.assemble_pp(g, Params(), st, [np.zeros(g.n)] * 3, d)
    r = orc.spmv(g, s, np.full(g.n, 3.0))
    assert np.max(np.abs(r)) <= 16 * ULP * 3.0 * s["aP"].max()


# ----------------------------------------------------------------- momentum rows
def test_mom_quiescent(orc):
    """quiescent field, no gravity, no drag -> u = 0."""
    g = Grid(4, 5, 6, 0.02, 0.02, 0.02, w_in=0.0)
    pr = Params(g=(0.0, 0.0, 0.0))
    rng = np.random.default_rng(1)
    st = base_state(g, eps=rng.uniform(0.4, 1.0, g.n), p=0.0)  # gauge p = 0 = outlet value
    st["eps_old"] = st["eps"].copy()
    for c in range(3):
        s, r2, rc = orc.assemble_mom(g, pr, c, st)
        assert rc == 0 and np.all(s["b"] == 0.0) and r2[0] == 0.0
        res = orc.bicgstab(g, s, np.zeros(g.n), 1e-6, 20)
        assert res["iters"] == 0 and np.all(res["x"] == 0.0)


def test_mom_hydrostatic_balance(orc):
    """p_P - p_T = rho g0 dz, zero velocity, no drag -> b = 0 up to
    rounding (the same eps_f multiplies the pressure and gravity terms)."""
    g = Grid(3, 4, 8, 0.05, 0.05, 0.04, w_in=0.0)
    pr = Params(rho=1.2, g=(0.0, 0.0, -9.81))
    rng = np.random.default_rng(2)
    i, j, k = ijk(g)
    p = pr.rho * 9.81 * g.dz * (g.nz - k)      # ghost-centre p = 0 above the top cell
    st = base_state(g, eps=rng.uniform(0.4, 1.0, g.n), p=p)
    s, _, rc = orc.assemble_mom(g, pr, 2, st)
    assert rc == 0
    ef = 0.5 * (st["eps"] + np.where(k < g.nz - 1, np.roll(st["eps"], -g.nx * g.ny), st["eps"]))
    pres = ef * (g.dx * g.dy) * pr.rho * 9.81 * g.dz
    assert np.all(np.abs(s["b"]) <= 4 * ULP * pres)


@pytest.mark.parametrize("urf", [1.0, 0.7])
def test_mom_inertia_only_closed_form(orc, urf):
    """mu = 0, zero snapshot velocity, uniform p, g = 0: every a_nb = 0 and
    u = urf (rho eps0_f V u0/dt + S_f V) / (rho eps0_f V/dt + beta_f V)."""
    g = Grid(4, 3, 5, 0.02, 0.03, 0.04, w_in=0.0)
    pr = Params(mu=0.0, g=(0.0, 0.0, 0.0), urf_mom=urf)
    rng = np.random.default_rng(4)
    st = base_state(g, eps=rng.uniform(0.4, 1.0, g.n), eps_old=rng.uniform(0.4, 1.0, g.n), p=0.0,
                    beta=rng.uniform(0, 1e4, g.n), u_old=rng.normal(size=g.n), v_old=rng.normal(size=g.n),
                    w_old=rng.normal(size=g.n), sbeta_u=rng.normal(size=g.n) * 100,
                    sbeta_v=rng.normal(size=g.n) * 100, sbeta_w=rng.normal(size=g.n) * 100)
    V = g.dx * g.dy * g.dz
    i, j, k = ijk(g)
    nn = {0: (i, g.nx, 1), 1: (j, g.ny, g.nx), 2: (k, g.nz, g.nx * g.ny)}
    for c, (old, S) in enumerate([("u_old", "sbeta_u"), ("v_old", "sbeta_v"), ("w_old", "sbeta_w")]):
        s, _, rc = orc.assemble_mom(g, pr, c, st)
        assert rc == 0
        for key in ("aE", "aW", "aN", "aS", "aT", "aB"):
            assert np.all(s[key] == 0.0)
        pos, ext, stride = nn[c]
        outlet = c == 2
        Eidx = np.where(pos < ext - 1, np.arange(g.n) + stride, np.arange(g.n))
        avg = lambda f: 0.5 * (st[f] + st[f][Eidx])
        a0 = pr.rho * avg("eps_old") * V / pr.dt
        expect = urf * (a0 * st[old] + avg(S) * V) / (a0 + avg("beta") * V)
        res = orc.bicgstab(g, s, np.zeros(g.n), 1e-15, 500)
        real = (pos < ext - 1) | outlet
        assert np.allclose(res["x"][real], expect[real], rtol=1e-13)
        assert np.all(res["x"][~real] == 0.0)


def test_mom_uniform_plug_flow_coefficients(orc):
    """eps = 1, u = v = 0, w = W uniform: interior w rows have a_B = D_z + rho A_z W,
    a_T = D_z, a_E = a_W = D_x, a_N = a_S = D_y; x/y walls give 2 D (B2, dropped
    off-diagonal); the inlet row adds a_B w_in to b (B1); the outlet row drops a_T (B3)."""
    g = Grid(4, 4, 5, 0.01, 0.02, 0.03, w_in=0.25)
    W = 0.25
    pr = Params(mu=2e-3, g=(0.0, 0.0, 0.0), urf_mom=1.0, dt=1e30)
    st = base_state(g, w=W, p=0.0)
    s, _, rc = orc.assemble_mom(g, pr, 2, st)
    assert rc == 0
    Ax, Ay, Az = g.dy * g.dz, g.dx * g.dz, g.dx * g.dy
    Dx, Dy, Dz = pr.mu * Ax / g.dx, pr.mu * Ay / g.dy, pr.mu * Az / g.dz
    F = pr.rho * Az * W
    i, j, k = ijk(g)
    inner = (i > 0) & (i < g.nx - 1) & (j > 0) & (j < g.ny - 1) & (k > 0) & (k < g.nz - 1)
    r = lambda a, b: np.allclose(a, b, rtol=1e-14)
    assert r(s["aB"][inner], Dz + F) and r(s["aT"][inner], Dz)
    assert r(s["aE"][inner], Dx) and r(s["aW"][inner], Dx)
    assert r(s["aN"][inner], Dy) and r(s["aS"][inner], Dy)
    wall = (i == 0) & (j > 0) & (j < g.ny - 1) & (k > 0) & (k < g.nz - 1)
    assert np.all(s["aW"][wall] == 0.0)
    assert r(s["aP"][wall], 2 * Dx + Dx + 2 * Dy + (Dz + F) + Dz)
    bot = inner | ((k == 0) & (i > 0) & (i < g.nx - 1) & (j > 0) & (j < g.ny - 1))
    bot = bot & (k == 0)
    assert np.all(s["aB"][bot] == 0.0)
    assert r(s["b"][bot], (Dz + F) * g.w_in)
    top = (k == g.nz - 1) & (i > 0) & (i < g.nx - 1) & (j > 0) & (j < g.ny - 1)
    assert np.all(s["aT"][top] == 0.0)
    assert r(s["aP"][top], 2 * Dx + 2 * Dy + Dz + F)


def test_mom_dominance_on_bed_state(orc):
    """a_P - sum a_nb >= rho eps0_f V/dt > 0 on the synthetic bed."""
    g, pr, st = synth.config_case(1)
    pr.urf_mom = 1.0
    V = g.dx * g.dy * g.dz
    for c in range(3):
        s, _, rc = orc.assemble_mom(g, pr, c, st)
        assert rc == 0
        nb = sum(s[k] for k in ("aE", "aW", "aN", "aS", "aT", "aB"))
        assert np.all(s["aP"] - nb >= pr.rho * 0.36 * V / pr.dt * (1 - 1e-12))


# ----------------------------------------------------------------- scalar rows
def test_scalar_geometric_recurrence(orc):
    """Uniform w, eps = 1, dt -> inf, inlet phi_in = 0 (B2), Dirichlet top phi_out = 1
    (B2): phi_k = A + B r^k with r = 1 + F/D; A, B from the two boundary rows."""
    nz = 12
    g = Grid(3, 3, nz, 0.01, 0.01, 0.01, bc_zlo=BC_INLET, bc_zhi=BC_DIRICHLET_TEST, w_in=0.02)
    g.phi_in, g.phi_out = 0.0, 1.0
    W = 0.02
    pr = Params(dt=1e30, urf_phi=1.0)
    pr.gamma_phi = (2e-4, 0, 0, 0)
    st = base_state(g, w=W)
    s, _, rc = orc.assemble_scalar(g, pr, 0, st)
    assert rc == 0
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-14, 400)
    assert res["status"] == 0
    Az = g.dx * g.dy
    D = pr.gamma_phi[0] * Az / g.dz
    F = pr.rho * Az * W
    r = 1.0 + F / D
    # (2D+F)(A+B-phi_in) = B F ;  (D+F) B r^(N-2) (r-1) = 2D (phi_out - A - B r^(N-1))
    M = np.array([[2 * D + F, (2 * D + F) - F],
                  [2 * D, (D + F) * r ** (nz - 2) * (r - 1) + 2 * D * r ** (nz - 1)]])
    A, B = np.linalg.solve(M, [(2 * D + F) * g.phi_in, 2 * D * g.phi_out])
    k = np.arange(g.n) // 9
    assert np.allclose(res["x"], A + B * r ** k, rtol=1e-9, atol=1e-12)


def test_scalar_pure_convection_forward_substitution(orc):
    """Gamma = 0, one time step, uniform w: phi_k = (a0 phi0_k + F phi_{k-1})/(a0 + F),
    phi_{-1} = phi_in; outlet zero-gradient."""
    g = Grid(2, 2, 9, 0.02, 0.02, 0.02, w_in=0.1)
    pr = Params(dt=1e-2, urf_phi=1.0)
    pr.gamma_phi = (0.0, 0, 0, 0)
    rng = np.random.default_rng(5)
    st = base_state(g, w=0.1)
    st["phi_old0"] = rng.uniform(0, 1, g.n)
    st["phi0"] = np.zeros(g.n)
    s, _, rc = orc.assemble_scalar(g, pr, 0, st)
    res = orc.bicgstab(g, s, np.zeros(g.n), 1e-15, 200)
    V = g.dx * g.dy * g.dz
    a0 = pr.rho * V / pr.dt
    F = pr.rho * g.dx * g.dy * 0.1
    expect = np.zeros(g.n)
    for col in range(4):
        prev = g.phi_in
        for kk in range(g.nz):
            n = col + 4 * kk
            prev = (a0 * st["phi_old0"][n] + F * prev) / (a0 + F)
            expect[n] = prev
    assert np.allclose(res["x"], expect, rtol=1e-12)


def test_scalar_uniform_is_exact_solution(orc):
    """phi0 = phi_in = 1 everywhere: phi = 1 satisfies every row for any flow field."""
    g, pr, st = synth.config_case(1)
    st = dict(st)
    st["phi0"] = np.ones(g.n)
    st["phi_old0"] = np.ones(g.n)
    s, r2, rc = orc.assemble_scalar(g, pr, 0, st)
    assert rc == 0
    r = s["b"] - orc.spmv(g, s, np.ones(g.n))
    assert np.max(np.abs(r)) <= 1e-13 * np.max(np.abs(s["b"]))
    assert r2[0] <= 1e-13 * r2[1]


# ----------------------------------------------------------------- correction
def test_correction_continuity_identity(orc):
    """b(u_corr) = b(u*) - A p' pointwise (the zero-divergence invariant)."""
    g, pr, st = synth.config_case(1)
    rng = np.random.default_rng(8)
    star = [st["u"], st["v"], st["w"]]
    d = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    i, j, k = ijk(g)
    d[0][i == g.nx - 1] = 0.0
    d[1][j == g.ny - 1] = 0.0
    s, _, _ = orc.assemble_pp(g, pr, st, star, d)
    pp = rng.normal(size=g.n)
    u, v, w, p = orc.correct(g, pr, star, d, pp, st["p"])
    s2, _, _ = orc.assemble_pp(g, pr, st, [u, v, w], d)
    scale = pr.rho * g.dx * g.dy * 1.0
    assert np.max(np.abs(s2["b"] - (s["b"] - orc.spmv(g, s, pp)))) <= 1e-12 * scale
    assert np.array_equal(p, st["p"] + pr.urf_p * pp)


def test_correction_zero_and_uniform(orc):
    """S:385 p' = 0 leaves fields unchanged; S:387 uniform p' leaves interior
    faces unchanged (outlet faces change under the ghost p' = 0 reading, Q26)."""
    g, pr, st = synth.config_case(1)
    star = [st["u"], st["v"], st["w"]]
    d = [np.full(g.n, 1e-3)] * 3
    u, v, w, p = orc.correct(g, pr, star, d, np.zeros(g.n), st["p"])
    assert np.array_equal(u, star[0]) and np.array_equal(w, star[2]) and np.array_equal(p, st["p"])
    u, v, w, p = orc.correct(g, pr, star, d, np.full(g.n, 2.0), st["p"])
    i, j, k = ijk(g)
    assert np.array_equal(w[k < g.nz - 1], star[2][k < g.nz - 1])
    assert np.allclose(w[k == g.nz - 1], star[2][k == g.nz - 1] + 2e-3, rtol=1e-14)
    assert np.array_equal(u, star[0])


def test_correction_shrinks_imbalance(orc):
    """after the p' solve the corrected field's imbalance is <= lin_tol ||b||."""
    g, pr, st = synth.config_case(1)
    pr.lin_maxit_pp = 5000
    star, dv = [], []
    for c in range(3):
        s, _, _ = orc.assemble_mom(g, pr, c, st)
        x = orc.bicgstab(g, s, [st["u"], st["v"], st["w"]][c], pr.lin_tol_mom, pr.lin_maxit_mom)["x"]
        star.append(x)
        dv.append(s["d"])
    s, cont, _ = orc.assemble_pp(g, pr, st, star, dv)
    res = orc.bicgstab(g, s, np.zeros(g.n), pr.lin_tol_pp, pr.lin_maxit_pp)
    assert res["status"] == 0
    u, v, w, p = orc.correct(g, pr, star, dv, res["x"], st["p"])
    s2, cont2, _ = orc.assemble_pp(g, pr, st, [u, v, w], dv)
    assert np.linalg.norm(s2["b"]) <= 1.5 * pr.lin_tol_pp * np.linalg.norm(s["b"])
    assert cont2 < cont


# ----------------------------------------------------------------- SIMPLE
def test_simple_single_phase_mass_balance(orc):
    """S:149 / S:683: single-phase duct (eps = 1, beta = 0) iterated to convergence:
    |inflow - outflow| / inflow <= 1e-6."""
    g = Grid(6, 6, 10, 0.01, 0.01, 0.01, w_in=0.05)
    pr = Params(dt=1e-2, lin_tol_pp=1e-10, lin_maxit_pp=2000, lin_tol_mom=1e-8, lin_maxit_mom=200)
    st = base_state(g, w=0.05)
    st["w_old"] = st["w"].copy()
    R = None
    for it in range(60):
        st, R, iters, status, rc = orc.simple_iter(g, pr, st)
        assert rc >= 0
        if max(R) < 1e-7:
            break
    assert max(R) < 1e-6
    k = np.arange(g.n) // (g.nx * g.ny)
    Az = g.dx * g.dy
    inflow = pr.rho * Az * g.w_in * g.nx * g.ny
    outflow = pr.rho * Az * st["w"][k == g.nz - 1].sum()
    assert abs(inflow - outflow) / inflow <= 1e-6


def test_simple_deterministic(orc):
    g, pr, st = synth.config_case(1)
    a = orc.simple_iter(g, pr, st)
    b = orc.simple_iter(g, pr, st)
    for key in ("u", "v", "w", "p"):
        assert np.array_equal(a[0][key], b[0][key])
    assert a[2] == b[2]


# ----------------------------------------------------------------- Eq. 6 digits
def test_digits_matching_examples(orc):
    for a, b, dgt in GOLD["digits"]["cases"]:
        assert orc.digits_matching([a], [b])[0] == pytest.approx(dgt, abs=1e-9)
    x = np.random.default_rng(0).uniform(1, 2, 1000)
    assert np.all(orc.digits_matching(x, x) == 16.0)
    gp = GOLD["digits_perturbation"]
    dg = orc.digits_matching(x, x * (1 + gp["rel"]))
    assert np.all(np.floor(dg + 1e-6) == gp["digits"])


def test_pp_transient_term_sign(orc):
    """Eq. (1): with no flow, the discrete continuity imbalance is
    b = -rho V (eps - eps0)/dt (a volume-fraction rise demands net inflow)."""
    g = Grid(3, 4, 5, 0.01, 0.02, 0.03, w_in=0.0)
    pr = Params(rho=1.1, dt=2e-3)
    rng = np.random.default_rng(6)
    st = base_state(g, eps=rng.uniform(0.4, 1.0, g.n), eps_old=rng.uniform(0.4, 1.0, g.n))
    s, cont, _ = orc.assemble_pp(g, pr, st, [np.zeros(g.n)] * 3, [np.full(g.n, 1e-3)] * 3)
    V = g.dx * g.dy * g.dz
    assert np.allclose(s["b"], -pr.rho * V * (st["eps"] - st["eps_old"]) / pr.dt, rtol=1e-14)


@pytest.mark.parametrize("axis", [0, 1])
def test_mom_edge_eps_uses_four_cells(orc, axis):
    """u rows, transverse (y) diffusion: a_N = mu A_y/dy * eps_edge where the edge
    is shared by cells P, E=P+x, P+y, E+y.  If eps varies only along `axis`, the
    four-cell average collapses to the two distinct values on that axis."""
    g = Grid(5, 5, 4, 0.01, 0.01, 0.01, w_in=0.0)
    pr = Params(mu=1e-3, g=(0.0, 0.0, 0.0))
    i, j, k = ijk(g)
    prof = np.array([0.4, 0.55, 0.7, 0.85, 1.0])
    eps = prof[i] if axis == 0 else prof[j]
    st = base_state(g, eps=eps)
    s, _, _ = orc.assemble_mom(g, pr, 0, st)
    Dy = pr.mu * (g.dx * g.dz) / g.dy
    inner = (i < g.nx - 1) & (j < g.ny - 1)
    if axis == 0:
        expect = Dy * 0.5 * (prof[i] + prof[np.minimum(i + 1, 4)])
    else:
        expect = Dy * 0.5 * (prof[j] + prof[np.minimum(j + 1, 4)])
    assert np.allclose(s["aN"][inner], expect[inner], rtol=1e-14)
