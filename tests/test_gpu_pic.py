"""GPU parity of the particle -> grid coupling (NEXT-2):
libmfx.so's mfx_pic_deposit_eps / mfx_pic_drag through the C ABI against the
oracle (or_pic_deposit_eps / or_pic_drag) on identical seeded parcels.

Per-parcel quantities use the oracle's expression order, and both sides
evaluate the closure's powers correctly rounded with
independent implementations, so K is bitwise equal.
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
    # same expressions, and both sides round x^y correctly (quad powq in the
    # oracle, double-double log/exp on the GPU, no shared code): bitwise
    assert np.array_equal(Kd, Ko)
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
    pic = synth.PicParams(eps_min=-1.0)      # no floor: partition of unity holds cell by cell
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


# ---------------------------------------------------------------- coupling inside the SIMPLE loop
def coupled_case():
    g = synth.make_grid(16, 12, 20)
    # tight linear tolerances: both sides converge to the discrete solution, so
    # the 1e-16-level differences of the deposits cannot be amplified by the
    # Krylov iteration's path
    pr = synth.Params(lin_tol_mom=1e-13, lin_maxit_mom=400, lin_tol_pp=1e-13, lin_maxit_pp=6000)
    st = synth.make_state(g, 4321, pr)
    pic = synth.PicParams()
    pc = synth.make_parcels(g, 4322, 6000, st["eps"], pic)
    return g, pr, st, pic, pc


def oracle_coupled(orc, g, pr, st, pic, pc, outer, implicit):
    s = {k: v.copy() for k, v in st.items()}
    for it in range(outer):
        if implicit or it == 0:
            d = orc.pic_drag(g, pr, pic, pc, s["eps"], s["u"], s["v"], s["w"])
            for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w"):
                s[k] = d[k]
        s, R, iters, status, rc = orc.simple_iter(g, pr, s)
        s = {k: np.asarray(v).copy() for k, v in s.items()}
    return s


def rel_l2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("mode", ["implicit", "explicit"])
def test_simple_with_pic_coupling_vs_oracle(mfx, orc, mode):
    g, pr, st, pic, pc = coupled_case()
    sd = {k: dev(v) for k, v in st.items()}
    dpc = {k: dev(v) for k, v in pc.items()}
    ctx = mfx.SimpleContext("111[1]", g, pr)
    ctx.set_pic(dpc, pic, mfx.PIC_IMPLICIT if mode == "implicit" else mfx.PIC_EXPLICIT)
    betas = []
    for _ in range(3):
        ctx.step(sd)
        betas.append(host(sd["beta"]).copy())
    ctx.close()
    ref = oracle_coupled(orc, g, pr, st, pic, pc, 3, mode == "implicit")
    # the context refreshes with the binned gather deposit: bitwise the definition,
    # so the whole coupled SIMPLE loop is bitwise the oracle's
    for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w", "u", "v", "w", "p"):
        assert np.array_equal(host(sd[k]), ref[k]), k
    if mode == "explicit":     # refreshed once, then frozen
        assert np.array_equal(betas[0], betas[1]) and np.array_equal(betas[1], betas[2])
    else:                      # refreshed from the new velocities every iteration
        assert not np.array_equal(betas[0], betas[1])


def test_pic_coupling_multirank_consistent(mfx, orc):
    """"234[1]" over 4 thread-ranks with implicit coupling: only rank 0 (the PIC
    device) holds the parcels; its drag fields are broadcast (phase 3),
    so every rank ends with the same bits, and close to the oracle."""
    import threading
    g, pr, st, pic, pc = coupled_case()
    n = 4
    group = mfx.LocalGroup(n)
    res, errs = {}, []
    bar = threading.Barrier(n)

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sd = {k: dev(v) for k, v in st.items()}
                dpc = {k: dev(v) for k, v in pc.items()} if rank == 0 else None
                ctx = mfx.SimpleContext("234[1]", g, pr, rank=rank, nranks=n, group=group)
                ctx.set_pic(dpc, pic if rank == 0 else None, mfx.PIC_IMPLICIT)
                bar.wait()
                for _ in range(2):
                    ctx.step(sd, stream=stream)
                stream.synchronize()
                res[rank] = {k: host(v) for k, v in sd.items()}
                ctx.close()
        except Exception as e:  # pragma: no cover
            errs.append((rank, repr(e)))
            bar.abort()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errs, errs
    for r in range(1, n):
        for k in ("u", "v", "w", "p", "beta", "sbeta_w"):
            assert np.array_equal(res[r][k], res[0][k]), (r, k)
    ref = oracle_coupled(orc, g, pr, st, pic, pc, 2, True)
    for k in ("u", "v", "w", "p", "beta", "sbeta_w"):
        assert np.array_equal(res[0][k], ref[k]), k


def base_cell(g, x, y, z):
    q = []
    for c, h, n in ((x, g.dx, g.nx), (y, g.dy, g.ny), (z, g.dz, g.nz)):
        q.append(np.clip(np.floor(c / h - 0.5).astype(np.int64), 0, n - 1))
    return q[0] + g.nx * (q[1] + g.ny * q[2])


def test_pic_sort_is_deterministic_binning(mfx):
    """mfx_pic_sort: binned[k] = parcels[k][orig], base cells non-decreasing,
    original indices ascending inside a bin, bin_start consistent."""
    g, st, pic, pc = case(22, 14, 37, 50000, 41, sort=False)
    dpc = {k: dev(v) for k, v in pc.items()}
    srt = mfx.pic_sort(g, pic, dpc)
    orig = host(srt["orig"]).astype(np.int64)
    assert np.array_equal(np.sort(orig), np.arange(pc["x"].size))
    for k in synth.PARCEL_KEYS:
        assert np.array_equal(host(srt[k]), pc[k][orig]), k
    bc = base_cell(g, host(srt["x"]), host(srt["y"]), host(srt["z"]))
    assert np.all(np.diff(bc) >= 0)
    same = np.diff(bc) == 0
    assert np.all(np.diff(orig)[same] > 0)                     # ascending original index inside a bin
    start = host(srt["bin_start"]).astype(np.int64)
    assert start[0] == 0 and start[-1] == pc["x"].size
    assert np.array_equal(np.diff(start), np.bincount(bc, minlength=g.n))
    srt2 = mfx.pic_sort(g, pic, dpc)
    for k in list(synth.PARCEL_KEYS) + ["orig", "bin_start"]:
        assert torch.equal(srt[k], srt2[k]), k                # unique order: run-to-run identical


@pytest.mark.parametrize("shape,m", [((16, 16, 32), 20000), ((22, 14, 37), 50000), ((64, 64, 64), 300000)])
def test_binned_deposits_bitwise(mfx, orc, shape, m):
    """The gather deposits on binned parcels reproduce the parcel-ordered
    definition bit for bit (eps, beta, beta*u_s; K with the written pow)."""
    g, st, pic, pc = case(*shape, m, 900 + m % 89, sort=False)
    pr = synth.Params()
    ws = mfx.Workspace(g)
    srt = mfx.pic_sort(g, pic, {k: dev(v) for k, v in pc.items()})
    eps_d = mfx.pic_deposit_eps_binned(g, pic, srt, ws)
    ws.check()
    eps_o, rc = orc.pic_deposit_eps(g, pic, pc)
    assert rc == 0 and np.array_equal(host(eps_d), eps_o)
    K = torch.empty(m, dtype=torch.float64, device="cuda")
    out = mfx.pic_drag_binned(g, pr, pic, srt, dev(eps_o), dev(st["u"]), dev(st["v"]), dev(st["w"]), ws, K=K)
    ws.check()
    ref = orc.pic_drag(g, pr, pic, pc, eps_o, st["u"], st["v"], st["w"], diag=True)
    orig = host(srt["orig"]).astype(np.int64)
    assert np.array_equal(host(K), ref["diag"][orig, 4])
    for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w"):
        assert np.array_equal(host(out[k]), ref[k]), k


def test_binned_out_of_domain_latched_by_original_index(mfx):
    g = synth.make_grid(16, 16, 32)
    pc = synth.make_parcels(g, 3, 1000)
    pc["z"][417] = g.nz * g.dz * 1.5
    ws = mfx.Workspace(g)
    srt = mfx.pic_sort(g, synth.PicParams(), {k: dev(v) for k, v in pc.items()})
    mfx.pic_deposit_eps_binned(g, synth.PicParams(), srt, ws)
    with pytest.raises(mfx.MfxError) as ei:
        ws.check()
    assert "parcel 417" in str(ei.value)


def test_pic_sort_empty_and_large(mfx):
    g = synth.make_grid(128, 128, 512)
    pic = synth.PicParams()
    empty = {k: torch.zeros(0, dtype=torch.float64, device="cuda") for k in synth.PARCEL_KEYS}
    out = mfx.pic_sort(g, pic, empty)
    assert out["x"].numel() == 0 and int(out["bin_start"][-1]) == 0
    st = synth.make_state(g, 3)
    pc = synth.make_parcels(g, 4, 500000, st["eps"], pic)
    srt = mfx.pic_sort(g, pic, {k: dev(v) for k, v in pc.items()})
    bc = base_cell(g, host(srt["x"]), host(srt["y"]), host(srt["z"]))
    assert np.all(np.diff(bc) >= 0) and np.array_equal(np.sort(host(srt["omega"])), np.sort(pc["omega"]))


def test_pic_eps_into_offset_view(mfx, orc):
    """An eps output that is an 8-byte (not 16-byte) aligned view takes the
    plain-access finalize path: same values as the oracle."""
    g, st, pic, pc = case(22, 14, 37, 20000, 41)
    ws = mfx.Workspace(g)
    buf = torch.zeros(g.n + 1, dtype=torch.float64, device="cuda")
    view = buf[1:]
    assert view.data_ptr() % 16 == 8
    mfx.pic_deposit_eps(g, pic, {k: dev(v) for k, v in pc.items()}, ws, eps=view)
    ws.check()
    eps_o, rc = orc.pic_deposit_eps(g, pic, pc)
    assert rc == 0
    assert np.all(np.abs(host(view) - eps_o) <= TOL_SUM)
    assert host(buf)[0] == 0.0
