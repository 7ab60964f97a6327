"""Pins of the oracle's particle -> grid coupling (NEXT-2;
PAPER.md:65, 97, 131).  Each test ties
or_pic_deposit_eps / or_pic_drag to something other than the oracle itself:
partition of unity, node coincidence and symmetry, exact
reproduction of multilinear fields by trilinear weights, the textbook drag of
one sphere (Dalla Valle C_D, Syamlal-O'Brien's eps_g = 1 limit), the Stokes
limit, and momentum bookkeeping."""
import math

import numpy as np
import pytest

import synth


def grid_pow2(nx=8, ny=6, nz=10, bc_zlo=synth.BC_INLET, w_in=0.15):
    # power-of-two spacing: cell centres and faces are exact binary fractions
    return synth.Grid(nx, ny, nz, 0.25, 0.25, 0.25, bc_zlo=bc_zlo, bc_zhi=synth.BC_OUTLET, w_in=w_in)


def parcels(xyz, vel=None, omega=None):
    xyz = np.asarray(xyz, dtype=np.float64).reshape(-1, 3)
    m = xyz.shape[0]
    vel = np.zeros((m, 3)) if vel is None else np.asarray(vel, dtype=np.float64).reshape(-1, 3)
    omega = np.ones(m) if omega is None else np.broadcast_to(np.asarray(omega, dtype=np.float64), (m,)).copy()
    return dict(x=xyz[:, 0].copy(), y=xyz[:, 1].copy(), z=xyz[:, 2].copy(), u=vel[:, 0].copy(),
                v=vel[:, 1].copy(), w=vel[:, 2].copy(), omega=omega)


def vs(pic):
    return math.pi / 6.0 * pic.d_p ** 3


PIC = synth.PicParams(d_p=0.01, eps_min=0.0)     # large particles: O(1) solid fractions on 0.25 m cells


def test_partition_of_unity_random(orc):
    """sum_c eps_s V = sum_p omega Vs (incl. parcels folded at walls)."""
    g = grid_pow2()
    rng = np.random.default_rng(3)
    L = np.array([g.nx * g.dx, g.ny * g.dy, g.nz * g.dz])
    xyz = rng.uniform(0, 1, (500, 3)) * L
    xyz[:20, 0] = rng.uniform(0, 0.5 * g.dx, 20)          # within half a cell of the x- wall
    xyz[20:40, 2] = L[2] - rng.uniform(0, 0.5 * g.dz, 20)  # near the outlet
    xyz[40, :] = 0.0
    xyz[41, :] = L
    om = rng.uniform(0.5, 2.0, 500)
    eps, rc = orc.pic_deposit_eps(g, PIC, parcels(xyz, omega=om))
    assert rc == 0
    V = g.dx * g.dy * g.dz
    lhs = math.fsum((1.0 - eps) * V)
    rhs = math.fsum(om * vs(PIC))
    assert abs(lhs - rhs) <= 1e-13 * rhs


def test_node_coincidence_and_symmetry(orc):
    """SPEC.md:205 a parcel at a cell centre puts its whole volume there;
    SPEC.md:207 two parcels at adjacent centres give equal eps."""
    g = grid_pow2()
    V = g.dx * g.dy * g.dz
    c1 = ((3 + 0.5) * g.dx, (2 + 0.5) * g.dy, (4 + 0.5) * g.dz)
    eps, _ = orc.pic_deposit_eps(g, PIC, parcels([c1]))
    n1 = 3 + g.nx * (2 + g.ny * 4)
    expect = 1.0 - vs(PIC) / V
    assert eps[n1] == expect
    others = np.delete(eps, n1)
    assert np.all(others == 1.0)
    c2 = ((4 + 0.5) * g.dx, c1[1], c1[2])
    eps2, _ = orc.pic_deposit_eps(g, PIC, parcels([c1, c2]))
    assert eps2[n1] == eps2[n1 + 1] == expect


def test_no_parcels(orc):
    g = grid_pow2()
    pc = parcels(np.zeros((0, 3)))
    eps, rc = orc.pic_deposit_eps(g, PIC, pc)
    assert rc == 0 and np.all(eps == 1.0)
    st = synth.make_state(g, 1)
    out = orc.pic_drag(g, synth.Params(), PIC, pc, eps, st["u"], st["v"], st["w"])
    for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w"):
        assert np.all(out[k] == 0.0)


def test_out_of_domain_rejected(orc):
    g = grid_pow2()
    _, rc = orc.pic_deposit_eps(g, PIC, parcels([(-1e-9, 0.1, 0.1)]))
    assert rc == -1


def test_eps_floor(orc):
    g = grid_pow2()
    pic = synth.PicParams(d_p=0.2, eps_min=0.35)   # one huge parcel over-packs its cell
    c = (0.5 * g.dx, 0.5 * g.dy, 0.5 * g.dz)
    eps, _ = orc.pic_deposit_eps(g, pic, parcels([c], omega=5.0))
    assert eps[0] == 0.35


def _trilinear_field(g, face_axis, fn):
    """Field values at the lattice nodes of `face_axis` (-1: cell centres)."""
    k, j, i = np.meshgrid(np.arange(g.nz), np.arange(g.ny), np.arange(g.nx), indexing="ij")
    pos = [(i + 0.5) * g.dx, (j + 0.5) * g.dy, (k + 0.5) * g.dz]
    if face_axis >= 0:
        pos[face_axis] = pos[face_axis] + 0.5 * (g.dx, g.dy, g.dz)[face_axis]
    return fn(*pos).ravel()


def test_trilinear_reproduces_multilinear_fields(orc):
    """Trilinear weights are exact on span{1, x, y, z, xy, xz, yz, xyz}: the
    interpolated eps_g and staggered u, v, w at a parcel equal the function at
    the parcel position (away from the clamped half-cell next to each wall;
    the unstored boundary face (index -1) carries 0 for walls and w_in for the
    inlet, so fields that take those values there stay exact up to the wall)."""
    g = grid_pow2(bc_zlo=synth.BC_INLET, w_in=0.3)
    L = np.array([g.nx * g.dx, g.ny * g.dy, g.nz * g.dz])
    fe = lambda x, y, z: 0.6 + 0.01 * x - 0.02 * y + 0.015 * z + 0.003 * x * y * z
    fu = lambda x, y, z: x * (0.2 + 0.1 * y - 0.05 * z + 0.02 * y * z)          # 0 on the x- wall
    fv = lambda x, y, z: y * (-0.1 + 0.07 * x + 0.03 * z - 0.01 * x * z)        # 0 on the y- wall
    fw = lambda x, y, z: 0.3 + z * (0.05 - 0.02 * x + 0.04 * y + 0.01 * x * y)  # w_in on the inlet
    eps = _trilinear_field(g, -1, fe)
    u = _trilinear_field(g, 0, fu)
    v = _trilinear_field(g, 1, fv)
    w = _trilinear_field(g, 2, fw)
    rng = np.random.default_rng(11)
    m = 300
    h = np.array([g.dx, g.dy, g.dz])
    xyz = 0.5 * h + rng.uniform(0, 1, (m, 3)) * (L - h)       # cell-centred region: no clamping
    out = orc.pic_drag(g, synth.Params(), PIC, parcels(xyz), eps, u, v, w, diag=True)
    d = out["diag"]
    X, Y, Z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    np.testing.assert_allclose(d[:, 0], fe(X, Y, Z), rtol=0, atol=1e-14)
    # u: exact up to the x- wall (node -1 = 0 = fu(0, y, z)); keep y, z off the clamped half-cells
    xyz_u = xyz.copy()
    xyz_u[:, 0] = rng.uniform(0, L[0] - h[0], m)
    du = orc.pic_drag(g, synth.Params(), PIC, parcels(xyz_u), eps, u, v, w, diag=True)["diag"]
    np.testing.assert_allclose(du[:, 1], fu(xyz_u[:, 0], xyz_u[:, 1], xyz_u[:, 2]), rtol=0, atol=1e-14)
    xyz_w = xyz.copy()
    xyz_w[:, 2] = rng.uniform(0, L[2] - h[2], m)
    dw = orc.pic_drag(g, synth.Params(), PIC, parcels(xyz_w), eps, u, v, w, diag=True)["diag"]
    np.testing.assert_allclose(dw[:, 3], fw(xyz_w[:, 0], xyz_w[:, 1], xyz_w[:, 2]), rtol=0, atol=1e-14)
    np.testing.assert_allclose(d[:, 2], fv(X, Y, Z), rtol=0, atol=1e-14)


def test_uniform_field_interpolates_to_itself(orc):
    """a uniform gas field is the interpolated value at any parcel
    (weights sum to 1, clamped nodes included)."""
    g = grid_pow2()
    n = g.nx * g.ny * g.nz
    L = np.array([g.nx * g.dx, g.ny * g.dy, g.nz * g.dz])
    rng = np.random.default_rng(5)
    xyz = rng.uniform(0, 1, (400, 3)) * L
    out = orc.pic_drag(g, synth.Params(), PIC, parcels(xyz), np.full(n, 0.7), np.zeros(n), np.zeros(n),
                       np.zeros(n), diag=True)
    np.testing.assert_allclose(out["diag"][:, 0], 0.7, rtol=2e-16 * 8)


def test_single_sphere_dalla_valle(orc):
    """eps_g = 1: Syamlal-O'Brien's velocity ratio is exactly 1 (A = B = 1,
    SPEC.md:291), so K is the drag of omega isolated spheres with Dalla Valle's
    C_D = (0.63 + 4.8/sqrt(Re))^2: F = C_D (pi d^2/4)(rho slip^2/2) per sphere."""
    pr = synth.Params()
    pic = synth.PicParams(d_p=200e-6)
    for slip in (1e-3, 0.05, 0.36, 2.0, 17.0):
        Re = pr.rho * pic.d_p * slip / pr.mu
        cd = (0.63 + 4.8 / math.sqrt(Re)) ** 2
        force = cd * (math.pi * pic.d_p ** 2 / 4.0) * (0.5 * pr.rho * slip * slip)
        omega = 7.0
        K = orc.pic_drag_coef(pr, pic, 1.0, slip, omega)
        assert K == pytest.approx(omega * force / slip, rel=1e-13)


def test_stokes_limit(orc):
    """Re -> 0, eps_g = 1: F -> (23.04/24) 3 pi mu d slip (Dalla Valle's 4.8^2 / 24
    of the Stokes drag)."""
    pr = synth.Params()
    pic = synth.PicParams(d_p=200e-6)
    slip = 1e-12
    K = orc.pic_drag_coef(pr, pic, 1.0, slip, 1.0)
    assert K / (3.0 * math.pi * pr.mu * pic.d_p) == pytest.approx(23.04 / 24.0, rel=1e-5)


def test_zero_slip_zero_drag(orc):
    pr = synth.Params()
    for eg in (0.4, 0.9, 1.0):
        assert orc.pic_drag_coef(pr, synth.PicParams(), eg, 0.0, 3.0) == 0.0


def test_bed_drag_magnitude(orc):
    """SURVEY.md §8(d) (survey-time evaluation of the closure): beta_d = 3.06e4
    kg/(m3 s) at eps_g = 0.42, slip 0.36 m/s, d_p = 200 um; beta_d = K eps_s / (omega Vs)."""
    pr = synth.Params()
    pic = synth.PicParams(d_p=200e-6)
    K = orc.pic_drag_coef(pr, pic, 0.42, 0.36, 1.0)
    beta_d = K * (1.0 - 0.42) / vs(pic)
    assert beta_d == pytest.approx(3.06e4, rel=5e-3)


def test_momentum_bookkeeping(orc):
    """sum_c beta V = sum_p K_p and sum_c (beta u_s)_c V = sum_p K_p u_p,c."""
    g = synth.make_grid(16, 12, 20)
    st = synth.make_state(g, 9)
    pic = synth.PicParams()
    pc = synth.make_parcels(g, 10, 5000, st["eps"], pic)
    eps, _ = orc.pic_deposit_eps(g, pic, pc)
    out = orc.pic_drag(g, synth.Params(), pic, pc, eps, st["u"], st["v"], st["w"], diag=True)
    V = g.dx * g.dy * g.dz
    K = out["diag"][:, 4]
    assert math.fsum(out["beta"] * V) == pytest.approx(math.fsum(K), rel=1e-13)
    for c, key in enumerate(("u", "v", "w")):
        lhs = math.fsum(out[f"sbeta_{key}"] * V)
        rhs = math.fsum(K * pc[key])
        assert abs(lhs - rhs) <= 1e-13 * math.fsum(np.abs(K * pc[key]))
    assert np.all(out["beta"] >= 0.0)


def _pow_cr_decimal(x: float, y: float) -> float:
    """x^y correctly rounded, independently of the oracle: exact decimal
    conversion of the binary64 arguments, ln/exp at 60 significant digits
    (error ~1e-58 relative), then Python's correctly rounded str -> float."""
    import decimal
    ctx = decimal.Context(prec=60)
    X, Y = decimal.Decimal(x), decimal.Decimal(y)
    if X == 1:
        return 1.0
    return float(ctx.exp(ctx.multiply(Y, ctx.ln(X))))


def test_pow_correctly_rounded(orc):
    """DESIGN.md §3.9 reading: the closure's powers are the correctly rounded
    x^y (the dots' contract, Q17), pinned against a 60-digit decimal
    evaluation: bitwise on the closure's exponents over the eps range of the
    workload, on random exponents, and at the special points; no call is
    reported ambiguous."""
    rng = np.random.default_rng(12)
    xs = np.concatenate([rng.uniform(0.3, 1.0, 3000), rng.uniform(1e-3, 50.0, 500),
                         [0.35, 0.36, 0.42, 0.5, 0.85, 0.95, 0.999999999, 1.0 - 2**-52, 1.0 + 2**-52, 2.0]])
    n0 = orc.lib().or_pow_ambiguous()
    for y in (4.14, 1.28, 2.65):
        for x in xs:
            assert orc.pow_(x, y) == _pow_cr_decimal(float(x), y), (x, y)
        assert orc.pow_(1.0, y) == 1.0
    for x, y in zip(rng.uniform(0.05, 5.0, 500), rng.uniform(-6.0, 6.0, 500)):
        assert orc.pow_(x, y) == _pow_cr_decimal(float(x), float(y)), (x, y)
    assert orc.pow_(2.0, 3.0) == 8.0 and orc.pow_(4.0, 0.5) == 2.0      # exact powers
    assert orc.lib().or_pow_ambiguous() == n0
