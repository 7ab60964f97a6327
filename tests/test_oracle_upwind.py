"""Pins of the upwinded convective face eps (NEXT-3 "upwinded (eps rho)_f",
DESIGN.md §3.12; SURVEY.md Q9's MFiX-style alternative to the central face
average, frozen per outer iteration by the snapshot velocity)."""
import numpy as np

import synth


def ijk(g):
    n = np.arange(g.n)
    return n % g.nx, (n // g.nx) % g.ny, n // (g.nx * g.ny)


def up_params(**kw):
    return synth.Params(face_eps_upwind=1, **kw)


def test_uniform_eps_upwind_equals_central(orc):
    """With a uniform void fraction the upwind and central face values are the
    same number, so every assembled row is bitwise identical."""
    g = synth.make_grid(10, 8, 12)
    st = synth.make_state(g, 4, synth.Params(), n_scalars=1)
    st["eps"][:] = 0.55
    st["phi0"] = np.random.default_rng(1).uniform(0, 1, g.n)
    st["phi_old0"] = st["phi0"].copy()
    pc, pu = synth.Params(), up_params()
    for c in range(3):
        a, ra, _ = orc.assemble_mom(g, pc, c, st)
        b, rb, _ = orc.assemble_mom(g, pu, c, st)
        for k in a:
            assert np.array_equal(a[k], b[k]), (c, k)
        assert np.array_equal(ra, rb)
    rng = np.random.default_rng(2)
    d = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    star = [st["u"], st["v"], st["w"]]
    a, ca, _ = orc.assemble_pp(g, pc, st, star, d)
    b, cb, _ = orc.assemble_pp(g, pu, st, star, d)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    a, _, _ = orc.assemble_scalar(g, pc, 0, st)
    b, _, _ = orc.assemble_scalar(g, pu, 0, st)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_pp_face_takes_upwind_cell(orc):
    """c_x on an interior face is (rho eps_up A_x) d with eps_up the cell the
    snapshot u flows out of; the mass flux uses the same value."""
    g, pr, st = synth.config_case(1)
    pu = up_params()
    rng = np.random.default_rng(3)
    d = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    star = [rng.normal(size=g.n) for _ in range(3)]
    s, _, _ = orc.assemble_pp(g, pu, st, star, d)
    i, j, k = ijk(g)
    A = g.dy * g.dz
    inner = i < g.nx - 1
    n = np.nonzero(inner)[0]
    e_up = np.where(st["u"][n] >= 0.0, st["eps"][n], st["eps"][n + 1])
    assert np.array_equal(s["aE"][n], ((pu.rho * e_up) * A) * d[0][n])
    # both directions occur in the input
    assert (st["u"][n] > 0).any() and (st["u"][n] < 0).any()


def test_upwind_pp_symmetric_and_continuity_identity(orc):
    """One stored value per face keeps A = A^T, and because the p' coefficient
    and the mass flux share eps_up, b(u_corr) = b(u*) - A p' still holds."""
    g, pr, st = synth.config_case(1)
    pu = up_params()
    rng = np.random.default_rng(8)
    star = [st["u"], st["v"], st["w"]]
    d = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    i, j, k = ijk(g)
    d[0][i == g.nx - 1] = 0.0
    d[1][j == g.ny - 1] = 0.0
    s, _, _ = orc.assemble_pp(g, pu, st, star, d)
    pp = rng.normal(size=g.n)
    u, v, w, p = orc.correct(g, pu, star, d, pp, st["p"])
    s2, _, _ = orc.assemble_pp(g, pu, st, [u, v, w], d)
    scale = pu.rho * g.dx * g.dy * 1.0
    assert np.max(np.abs(s2["b"] - (s["b"] - orc.spmv(g, s, pp)))) <= 1e-12 * scale
    gs = synth.make_grid(6, 5, 7)
    sts = synth.make_state(gs, 6, pu)
    ds = [rng.uniform(1e-4, 1e-3, gs.n) for _ in range(3)]
    ss, _, _ = orc.assemble_pp(gs, pu, sts, [sts["u"], sts["v"], sts["w"]], ds)
    Ad = orc.dense_matrix(gs, ss)
    assert np.array_equal(Ad, Ad.T)


def test_upwind_momentum_transverse_flux(orc):
    """Momentum transverse mass flux: the north face of the u-CV averages the
    two cells' +y face fluxes, each with its upwind eps;
    checked on one interior row against the written formula."""
    g = synth.make_grid(8, 6, 10)
    pu = up_params()
    st = synth.make_state(g, 12, pu)
    st["eps"] = np.random.default_rng(5).uniform(0.4, 1.0, g.n)
    out, _, _ = orc.assemble_mom(g, pu, 0, st)
    i0, j0, k0 = 3, 2, 4
    n = i0 + g.nx * (j0 + g.ny * k0)
    nE, nN, nNE = n + 1, n + g.nx, n + 1 + g.nx
    A_y = g.dx * g.dz
    def m(X, Xn):
        e = st["eps"][X] if st["v"][X] >= 0.0 else st["eps"][Xn]
        return ((pu.rho * e) * A_y) * st["v"][X]
    F = 0.5 * (m(n, nN) + m(nE, nNE))
    e4 = 0.25 * (((st["eps"][n] + st["eps"][nE]) + st["eps"][nN]) + st["eps"][nNE])
    D = ((pu.mu * A_y) / g.dy) * e4
    assert out["aN"][n] == D + max(-F, 0.0)
