"""Consistency pins for the general rows with EVERY term active.

The special-case pins of test_oracle_assembly.py fix each term of the
momentum, scalar and p' rows alone; these tests fix them all together against
the equations they discretise.  Smooth manufactured fields (velocities, eps,
eps0, p, beta, S, old values) are sampled at the staggered positions, the
oracle assembles its rows, and the discrete residual of each interior row,
divided by the cell volume, is compared with the continuous residual of the
PDE evaluated analytically (derivatives by central differences of the
manufactured functions, accurate to ~1e-8) at the row's position:

  momentum (Eq. 2; readings Q10-Q12 of DESIGN.md §4):
    rho eps0 (u - u0)/dt + rho eps U.grad u - div(mu eps grad u) + beta u
      + eps dp/dx_c - rho eps g_c - S_c
  scalar (energy / species; reading Q21):
    rho eps0 (phi - phi0)/dt + rho eps U.grad phi - div(Gamma eps grad phi)
  p' (continuity, Eq. 1; SIMPLE pressure correction):
    b / V      -> -[div(rho eps U*) + rho (eps - eps0)/dt]
    (A p')/V   -> -div(rho eps d grad p')       (d = eps A / A_P, a smooth field here)

A consistent discretisation drives the difference to zero as the mesh is
refined (first order: upwind convection; second order: the rest and every
p' term); a dropped term, a wrong sign, a swapped axis or a transposed
operand leaves an O(1) difference that does not shrink.  Each test also
checks that it would catch such a mistake: the residual with one term
removed does not converge.  Spacings differ per axis (dx != dy != dz) so
that an axis mix-up is visible.
"""
import numpy as np
import pytest

from synth import Grid, Params, BC_INLET, BC_OUTLET

TWO_PI = 2.0 * np.pi
L = (1.0, 1.25, 0.8)                       # domain lengths (x, y, z)
FD = 1e-4                                  # central-difference step of the analytic derivatives


def _s(x, y, z, a, b, c, ph):
    return np.sin(a * x / L[0] * TWO_PI + ph) * np.cos(b * y / L[1] * np.pi + 0.3 * ph) * np.cos(c * z / L[2] * np.pi + 0.7)


# manufactured fields: name -> f(x, y, z)
F = {
    "u": lambda x, y, z: 0.30 + 0.20 * _s(x, y, z, 1.0, 1.0, 1.0, 0.1),
    "v": lambda x, y, z: -0.10 + 0.25 * _s(y, z, x, 1.0, 1.0, 1.0, 0.7),
    "w": lambda x, y, z: 0.20 + 0.15 * _s(z, x, y, 1.0, 1.0, 1.0, 1.3),
    "u_old": lambda x, y, z: 0.25 + 0.20 * _s(x, y, z, 1.0, 0.5, 1.0, 0.4),
    "v_old": lambda x, y, z: -0.05 + 0.20 * _s(y, x, z, 1.0, 1.0, 0.5, 0.2),
    "w_old": lambda x, y, z: 0.15 + 0.10 * _s(z, y, x, 0.5, 1.0, 1.0, 0.9),
    "eps": lambda x, y, z: 0.65 + 0.20 * _s(x, z, y, 1.0, 1.0, 1.0, 0.5),
    "eps_old": lambda x, y, z: 0.62 + 0.18 * _s(y, x, z, 1.0, 1.0, 1.0, 1.1),
    "p": lambda x, y, z: 0.10 * _s(x, y, z, 1.0, 1.0, 0.5, 2.0) + 0.05 * z,
    "beta": lambda x, y, z: 2.0 + 0.8 * _s(z, y, x, 1.0, 0.5, 1.0, 0.6),
    "sbeta_u": lambda x, y, z: 0.40 + 0.30 * _s(x, y, z, 0.5, 1.0, 1.0, 1.7),
    "sbeta_v": lambda x, y, z: -0.20 + 0.30 * _s(y, z, x, 1.0, 0.5, 1.0, 0.8),
    "sbeta_w": lambda x, y, z: 0.30 + 0.25 * _s(z, x, y, 1.0, 1.0, 0.5, 0.3),
    "phi0": lambda x, y, z: 0.5 + 0.3 * _s(x, y, z, 1.0, 1.0, 1.0, 0.25),
    "phi_old0": lambda x, y, z: 0.45 + 0.3 * _s(y, z, x, 1.0, 1.0, 1.0, 0.65),
    "d0": lambda x, y, z: 1.0 + 0.3 * _s(x, y, z, 1.0, 1.0, 1.0, 0.15),
    "d1": lambda x, y, z: 0.8 + 0.2 * _s(y, x, z, 1.0, 1.0, 1.0, 0.45),
    "d2": lambda x, y, z: 1.2 + 0.3 * _s(z, y, x, 1.0, 1.0, 1.0, 0.85),
    "pp": lambda x, y, z: 0.2 * _s(x, y, z, 1.0, 1.0, 1.0, 0.55),
}
VEL = ("u", "v", "w")
PR = dict(rho=1.3, mu=0.05, g=(0.3, -0.2, -1.0), dt=0.2, urf_mom=0.7, gamma_phi=(0.04, 0.0, 0.0, 0.0))


def grad(f, X):
    out = []
    for a in range(3):
        e = np.zeros(3)
        e[a] = FD
        out.append((f(*(X + e[:, None])) - f(*(X - e[:, None]))) / (2 * FD))
    return out


def d2(f, X, a):
    e = np.zeros(3)
    e[a] = FD
    return (f(*(X + e[:, None])) - 2.0 * f(*X) + f(*(X - e[:, None]))) / (FD * FD)


def make_case(n):
    nx, ny, nz = n, n, n
    g = Grid(nx, ny, nz, L[0] / nx, L[1] / ny, L[2] / nz, bc_zlo=BC_INLET, bc_zhi=BC_OUTLET, w_in=0.2)
    h = np.array([g.dx, g.dy, g.dz])
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cc = np.stack([(i.ravel() + 0.5) * h[0], (j.ravel() + 0.5) * h[1], (k.ravel() + 0.5) * h[2]])
    st = {}
    for name, f in F.items():
        X = cc.copy()
        for c, vn in enumerate(VEL):
            if name in (vn, vn + "_old"):
                X[c] += 0.5 * h[c]            # staggered: component c on the +c face
        st[name] = f(*X)
    ijk = (i.ravel(), j.ravel(), k.ravel())
    return g, h, cc, st, ijk


def interior(g, ijk, margin=2):
    i, j, k = ijk
    return ((i >= margin) & (i < g.nx - margin) & (j >= margin) & (j < g.ny - margin) &
            (k >= margin) & (k < g.nz - margin))


def row_residual(g, sys, x, offdiag):
    """a_P x_P - sum a_nb x_nb - b (row convention of SURVEY §8c), interior rows."""
    n = g.n
    idx = np.arange(n)
    r = sys["aP"] * x - sys["b"]
    for key, off in offdiag:
        nb = np.clip(idx + off, 0, n - 1)
        r = r - sys[key] * x[nb]
    return r


MOM_NB = [("aW", -1), ("aE", 1), ("aS", "y-"), ("aN", "y+"), ("aB", "z-"), ("aT", "z+")]


def _offs(g):
    m = {"y-": -g.nx, "y+": g.nx, "z-": -g.nx * g.ny, "z+": g.nx * g.ny}
    return [(k, m.get(o, o)) for k, o in MOM_NB]


def mom_terms(c, X):
    """Continuous momentum residual terms for component c at points X (3, m)."""
    pr = PR
    fu = F[VEL[c]]
    U = [F[vn](*X) for vn in VEL]
    eps, eps0 = F["eps"](*X), F["eps_old"](*X)
    gu = grad(fu, X)
    ge = grad(F["eps"], X)
    lap = sum(d2(fu, X, a) for a in range(3))
    return {
        "transient": pr["rho"] * eps0 * (fu(*X) - F[VEL[c] + "_old"](*X)) / pr["dt"],
        "convection": pr["rho"] * eps * sum(U[a] * gu[a] for a in range(3)),
        "diffusion": -pr["mu"] * (sum(ge[a] * gu[a] for a in range(3)) + eps * lap),
        "drag": F["beta"](*X) * fu(*X),
        "pressure": eps * grad(F["p"], X)[c],
        "gravity": -pr["rho"] * eps * pr["g"][c],
        "source": -F["sbeta_" + "uvw"[c]](*X),
    }


def _mom_errors(orc, n, c, drop=None, upwind=0):
    g, h, cc, st, ijk = make_case(n)
    p = Params(rho=PR["rho"], mu=PR["mu"], g=PR["g"], dt=PR["dt"], urf_mom=PR["urf_mom"], face_eps_upwind=upwind)
    sys, _, rc = orc.assemble_mom(g, p, c, st)
    assert rc == 0
    V = g.dx * g.dy * g.dz
    R = row_residual(g, sys, st[VEL[c]], _offs(g)) / V
    m = interior(g, ijk)
    X = cc[:, m].copy()
    X[c] += 0.5 * h[c]
    terms = mom_terms(c, X)
    cont = sum(v for k, v in terms.items() if k != drop)
    scale = max(np.max(np.abs(v)) for v in terms.values())
    return np.max(np.abs(R[m] - cont)), scale, terms


@pytest.mark.parametrize("c", [0, 1, 2])
def test_momentum_row_consistent_with_eq2(orc, c):
    e16, scale, terms = _mom_errors(orc, 16, c)
    e64, _, _ = _mom_errors(orc, 64, c)
    # every term is O(scale): none is negligible, so none can hide
    for k, v in terms.items():
        assert np.max(np.abs(v)) > 0.05 * scale, k
    # first-order convergence (upwind convection; measured ratio 0.30-0.35 for
    # 4x refinement, 0.25 asymptotically), small at the fine grid
    assert e64 < 0.45 * e16, (e16, e64)
    assert e64 < 0.05 * scale, (e64, scale)


@pytest.mark.parametrize("c", [0, 1, 2])
def test_momentum_row_with_upwinded_face_eps_consistent(orc, c):
    """the upwinded (eps rho)_f convective mass fluxes keep the
    row a consistent (first-order) discretisation of Eq. 2."""
    e16, scale, _ = _mom_errors(orc, 16, c, upwind=1)
    e64, _, _ = _mom_errors(orc, 64, c, upwind=1)
    assert e64 < 0.45 * e16, (e16, e64)
    assert e64 < 0.05 * scale, (e64, scale)


@pytest.mark.parametrize("drop", ["transient", "convection", "diffusion", "drag", "pressure", "gravity", "source"])
def test_momentum_consistency_detects_a_missing_term(orc, drop):
    e16, scale, _ = _mom_errors(orc, 16, 2, drop)
    e32, _, _ = _mom_errors(orc, 32, 2, drop)
    assert e32 > 0.5 * e16 and e32 > 0.05 * scale, (drop, e16, e32)


def _scalar_errors(orc, n, drop=None):
    g, h, cc, st, ijk = make_case(n)
    p = Params(rho=PR["rho"], mu=PR["mu"], dt=PR["dt"], gamma_phi=PR["gamma_phi"], urf_phi=1.0)
    sys, _, rc = orc.assemble_scalar(g, p, 0, st)
    assert rc == 0
    V = g.dx * g.dy * g.dz
    R = row_residual(g, sys, st["phi0"], _offs(g)) / V
    m = interior(g, ijk)
    X = cc[:, m]
    fp = F["phi0"]
    eps, eps0 = F["eps"](*X), F["eps_old"](*X)
    gp, ge = grad(fp, X), grad(F["eps"], X)
    U = [F[vn](*X) for vn in VEL]
    G = PR["gamma_phi"][0]
    terms = {
        "transient": PR["rho"] * eps0 * (fp(*X) - F["phi_old0"](*X)) / PR["dt"],
        "convection": PR["rho"] * eps * sum(U[a] * gp[a] for a in range(3)),
        "diffusion": -G * (sum(ge[a] * gp[a] for a in range(3)) + eps * sum(d2(fp, X, a) for a in range(3))),
    }
    cont = sum(v for k, v in terms.items() if k != drop)
    scale = max(np.max(np.abs(v)) for v in terms.values())
    return np.max(np.abs(R[m] - cont)), scale, terms


def test_scalar_row_consistent_with_transport_equation(orc):
    e16, scale, terms = _scalar_errors(orc, 16)
    e64, _, _ = _scalar_errors(orc, 64)
    for k, v in terms.items():
        assert np.max(np.abs(v)) > 0.05 * scale, k
    assert e64 < 0.45 * e16, (e16, e64)
    assert e64 < 0.05 * scale, (e64, scale)
    for drop in terms:
        d16, _, _ = _scalar_errors(orc, 16, drop)
        d32, _, _ = _scalar_errors(orc, 32, drop)
        assert d32 > 0.5 * d16 and d32 > 0.05 * scale, drop


def _pp_errors(orc, n, drop=None):
    """(b error, A p' error, b scale, A p' scale); A p' is compared after
    scaling by n: n (A p')/V -> -sum_a L_a d/dx_a(rho eps d_a dp'/dx_a)."""
    g, h, cc, st, ijk = make_case(n)
    p = Params(rho=PR["rho"], dt=PR["dt"])
    star = [st[vn] for vn in VEL]
    dv = []                                  # d_c on the staggered faces, like the velocities
    for c in range(3):
        X = cc.copy()
        X[c] += 0.5 * h[c]
        dv.append(F["d%d" % c](*X))
    sys, _, rc = orc.assemble_pp(g, p, st, star, dv)
    assert rc == 0
    V = g.dx * g.dy * g.dz
    m = interior(g, ijk)
    X = cc[:, m]
    rho = PR["rho"]
    div = 0.0
    for a in range(3):
        flux = (lambda a: lambda x, y, z: F["eps"](x, y, z) * F[VEL[a]](x, y, z))(a)
        div = div + rho * grad(flux, X)[a]
    transient = rho * (F["eps"](*X) - F["eps_old"](*X)) / PR["dt"]
    b_cont = -(div + (0.0 if drop == "transient" else transient))
    eb = np.max(np.abs(sys["b"][m] / V - b_cont))
    Ap = orc.spmv(g, sys, F["pp"](*cc))
    op = 0.0
    gpp = grad(F["pp"], X)
    for a in range(3):
        q = (lambda a: lambda x, y, z: F["eps"](x, y, z) * F["d%d" % a](x, y, z))(a)
        dterm = rho * (grad(q, X)[a] * gpp[a] + q(*X) * d2(F["pp"], X, a))
        if drop != "axis%d" % a:
            op = op - L[a] * dterm
    ea = np.max(np.abs(n * Ap[m] / V - op))
    return eb, ea, np.max(np.abs(b_cont)), np.max(np.abs(op))


def test_pp_row_consistent_with_continuity(orc):
    eb16, ea16, sb, sa = _pp_errors(orc, 16)
    eb32, ea32, _, _ = _pp_errors(orc, 32)
    # second order: central face eps, centred differences
    assert eb32 < 0.35 * eb16 and eb32 < 0.01 * sb, (eb16, eb32, sb)
    assert ea32 < 0.35 * ea16 and ea32 < 0.01 * sa, (ea16, ea32, sa)
    for drop in ("transient", "axis0", "axis1", "axis2"):
        db16, da16, _, _ = _pp_errors(orc, 16, drop)
        db32, da32, _, _ = _pp_errors(orc, 32, drop)
        d16, d32 = (db16, db32) if drop == "transient" else (da16, da32)
        scale = sb if drop == "transient" else sa
        assert d32 > 0.5 * d16 and d32 > 0.05 * scale, drop
