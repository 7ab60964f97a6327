"""GPU parity of the particle -> grid coupling (NEXT-2):
libmfx.so's mfx_pic_deposit_eps / mfx_pic_drag through the C ABI against the
oracle (or_pic_deposit_eps / or_pic_drag) on identical seeded parcels.

Per-parcel quantities use the oracle's expression order; K differs only by
pow()'s last-bit behaviour (CUDA vs libm), bounded here by 1e-13 relative.
The per-cell sums arrive in atomic order instead of parcel order, so the gate
is the summation error bound of DESIGN.md §3.9: for a cell with m
contributions of total magnitude S, |gpu - oracle| <= (m - 1) u S + (per-term
error) <= TOL_SUM * S with TOL_SUM = 1e-12 (m <= ~4500 contributions per cell
at u = 1.1e-16; these inputs have <= ~200).  eps_g = 1 - S/V inherits the
same absolute bound on S/V <= 1.
"""
import math

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_SUM = 1e-12
TOL_K = 1e-13


@pytest.fixture(scope="module")
def mfx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15605_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def with_edge_parcels(g, pc, rng):
    """Put some parcels exactly on the domain faces and corners and inside the
    half-cell next to every wall (the clamped / folded weights)."""
    L = (g.nx * g.dx, g.ny * g.dy, g.nz * g.dz)
    m = pc["x"].size
    k = min(64, m // 4)
    idx = rng.choice(m, size=k, replace=False)
    keys = ("x", "y", "z")
    for t, p in enumerate(idx):
        a = t % 3
        pc[keys[a]][p] = (0.0, L[a], rng.uniform(0, 0.5) * (g.dx, g.dy, g.dz)[a],
                          L[a] - rng.uniform(0, 0.5) * (g.dx, g.dy, g.dz)[a])[t % 4]
    pc["x"][idx[0]], pc["y"][idx[0]], pc["z"][idx[0]] = 0.0, 0.0, 0.0
    pc["x"][idx[1]], pc["y"][idx[1]], pc["z"][idx[1]] = L
    return pc


def case(nx, ny, nz, m, seed, sort=False, edges=True):
    g = synth.make_grid(nx, ny, nz)
    st = synth.make_state(g, seed)
    pic = synth.PicParams()
    pc = synth.make_parcels(g, seed + 1, m, st["eps"], pic)
    if edges:
        pc = with_edge_parcels(g, pc, np.random.default_rng(seed + 2))
    if sort:
        cell = (np.minimum((pc["x"] / g.dx).astype(np.int64), g.nx - 1) + g.nx *
                (np.minimum((pc["y"] / g.dy).astype(np.int64), g.ny - 1) + g.ny *
                 np.minimum((pc["z"] / g.dz).astype(np.int64), g.nz - 1)))
        order = np.argsort(cell, kind="stable")
        pc = {k: np.ascontiguousarray(v[order]) for k, v in pc.items()}
    return g, st, pic, pc


def run_both(mfx, orc, g, st, pic, pc):
    pr = synth.Params()
    ws = mfx.Workspace(g)
    dpc = {k: dev(v) for k, v in pc.items()}
    eps_d = mfx.pic_deposit_eps(g, pic, dpc, ws)
    ws.check()
    eps_o, rc = orc.pic_deposit_eps(g, pic, pc)
    assert rc == 0
    # the drag reads the deposited eps (identical input to both sides: the oracle's)
    u, v, w = dev(st["u"]), dev(st["v"]), dev(st["w"])
    K = torch.empty(pc["x"].size, dtype=torch.float64, device="cuda")
    out_d = mfx.pic_drag(g, pr, pic, dpc, dev(eps_o), u, v, w, ws, K=K)
    ws.check()
    out_o = orc.pic_drag(g, pr, pic, pc, eps_o, st["u"], st["v"], st["w"], diag=True)
    assert out_o["rc"] == 0
    return eps_d, eps_o, out_d, out_o, K


def check(eps_d, eps_o, out_d, out_o, K):
    e = host(eps_d)
    assert np.all(np.abs(e - eps_o) <= TOL_SUM), np.abs(e - eps_o).max()
    Ko = out_o["diag"][:, 4]
    Kd = host(K)
    np.testing.assert_allclose(Kd, Ko, rtol=TOL_K, atol=0)
    b = host(out_d["beta"])
    assert np.all(np.abs(b - out_o["beta"]) <= TOL_SUM * out_o["beta"]), np.abs(b - out_o["beta"]).max()
    for c, key in enumerate(("sbeta_u", "sbeta_v", "sbeta_w")):
        s = host(out_d[key])
        assert np.all(np.abs(s - out_o[key]) <= TOL_SUM * out_o["sabs"][c]), key


@pytest.mark.parametrize("shape,m,sort", [((16, 16, 32), 20000, False),    # configuration 1 grid
                                          ((16, 16, 32), 20000, True),
                                          ((22, 14, 37), 50000, False),     # ragged extents
                                          ((64, 64, 64), 300000, True)])
def test_pic_parity(mfx, orc, shape, m, sort):
    g, st, pic, pc = case(*shape, m, 700 + m % 97, sort=sort)
    check(*run_both(mfx, orc, g, st, pic, pc))


def test_pic_bookkeeping(mfx, orc):
    """SPEC.md:306 on the GPU outputs: sum beta V = sum K (GPU's own K)."""
    g, st, pic, pc = case(16, 16, 32, 20000, 5)
    eps_d, eps_o, out_d, out_o, K = run_both(mfx, orc, g, st, pic, pc)
    V = g.dx * g.dy * g.dz
    assert math.fsum(host(out_d["beta"]) * V) == pytest.approx(math.fsum(host(K)), rel=1e-12)
    vs = math.pi / 6.0 * pic.d_p ** 3
    assert math.fsum((1.0 - host(eps_d)) * V) == pytest.approx(math.fsum(pc["omega"] * vs), rel=1e-12)


def test_pic_no_parcels(mfx, orc):
    g = synth.make_grid(16, 16, 32)
    st = synth.make_state(g, 1)
    ws = mfx.Workspace(g)
    empty = {k: torch.zeros(0, dtype=torch.float64, device="cuda") for k in synth.PARCEL_KEYS}
    eps = mfx.pic_deposit_eps(g, synth.PicParams(), empty, ws)
    assert torch.all(eps == 1.0)
    out = mfx.pic_drag(g, synth.Params(), synth.PicParams(), empty, eps, dev(st["u"]), dev(st["v"]),
                       dev(st["w"]), ws)
    for t in out.values():
        assert torch.all(t == 0.0)


def test_pic_out_of_domain_latched(mfx):
    g = synth.make_grid(16, 16, 32)
    pc = synth.make_parcels(g, 3, 1000)
    pc["z"][417] = g.nz * g.dz * 1.5
    ws = mfx.Workspace(g)
    mfx.pic_deposit_eps(g, synth.PicParams(), {k: dev(v) for k, v in pc.items()}, ws)
    with pytest.raises(mfx.MfxError) as ei:
        ws.check()
    assert "parcel 417" in str(ei.value)
    ws.check()   # latch cleared


def test_pic_fullsize_c2(mfx, orc):
    """Configuration 2 grid (128x128x512) with the paper's parcel count
    (2,983,447 parcels), in the launch configuration bench.py
    times: every cell compared."""
    g, st, pic, pc = case(128, 128, 512, synth.PAPER_PARCELS, 15607, sort=False, edges=False)
    check(*run_both(mfx, orc, g, st, pic, pc))
