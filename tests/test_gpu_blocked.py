"""GPU parity with BLOCKED cells (NEXT-3 geometry): the
backward-facing step of PAPER.md:155 (Fig. 8), libmfx through the C ABI vs
the oracle (pinned by the exact slab-embedding tests), bitwise."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mfx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15605_b200 as m
    return m


def dev(st):
    out = {}
    for k, v in st.items():
        out[k] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    return out


SHAPES = [(12, 6, 40), (26, 9, 33), (64, 32, 96)]


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(params=["tma", "gridstride"])
def asm_path(request, mfx):
    """momentum assembly kernel: TMA z-marching (BLOCKED rules read from the
    flag bytes) or grid-stride; both must give the oracle's bits"""
    mfx.set_option("asm_tma", 1 if request.param == "tma" else 0)
    yield request.param
    mfx.set_option("asm_tma", 1)


@pytest.mark.parametrize("shape", SHAPES)
def test_bfs_assembly_bitwise(mfx, orc, shape, asm_path):
    g, pr, st = synth.bfs_case(*shape, seed=11)
    st["phi0"] = np.zeros(g.n)
    st["phi_old0"] = np.where(st["blocked"] == 0, np.random.default_rng(1).uniform(0, 1, g.n), 0.0)
    st["phi0"] = st["phi_old0"].copy()
    sd = dev(st)
    ws = mfx.Workspace(g)
    for comp in range(3):
        ref, r2, rc = orc.assemble_mom(g, pr, comp, st)
        out, res2 = mfx.assemble_eq(comp, g, pr, sd, ws)
        ws.check()
        for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b", "d"):
            assert np.array_equal(host(out[k]), ref[k]), (comp, k)
        assert np.array_equal(host(res2), r2)
    rng = np.random.default_rng(2)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    star = [st["u"], st["v"], st["w"]]
    ref, cont, rc = orc.assemble_pp(g, pr, st, star, dv)
    out, res2 = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=[sd["u"], sd["v"], sd["w"]] + [dev({"a": d})["a"] for d in dv])
    ws.check()      # no zero-diagonal latch for the empty block rows
    for k in ("aP", "aE", "aN", "aT", "b"):
        assert np.array_equal(host(out[k]), ref[k]), k
    assert host(res2)[0] == cont
    sref, s2, _ = orc.assemble_scalar(g, pr, 0, st)
    sout, sres = mfx.assemble_eq(mfx.EQ_SCALAR, g, pr, sd, ws, scalar_id=0)
    for k in ("aP", "aE", "aW", "aN", "aS", "aT", "aB", "b"):
        assert np.array_equal(host(sout[k]), sref[k]), k


@pytest.mark.parametrize("path", ["tma", "cluster", "v1"])
def test_bfs_simple_iteration_bitwise(mfx, orc, path):
    g, pr, st = synth.bfs_case(12, 6, 40, seed=12)
    pr.lin_maxit_pp = 3000
    mfx.set_option("solver_path", {"tma": mfx.PATH_TMA, "cluster": mfx.PATH_CLUSTER, "v1": mfx.PATH_V1}[path])
    try:
        sd = dev(st)
        ctx = mfx.SimpleContext("111[1]", g, pr)
        o = ctx.step(sd)
        ctx.close()
    finally:
        mfx.set_option("solver_path", mfx.PATH_AUTO)
    ref, R, it, stt, rc = orc.simple_iter(g, pr, st)
    assert o["iters"][:4] == it[:4]
    for k in ("u", "v", "w", "p"):
        assert np.array_equal(host(sd[k]), ref[k]), k


def test_bfs_multirank_equals_single(mfx, orc):
    """"234[1]" over 4 thread-ranks on the step geometry: every rank ends with
    the oracle's bits (the flags are a replicated input)."""
    import threading
    g, pr, st = synth.bfs_case(12, 6, 40, seed=13)
    pr.lin_maxit_pp = 3000
    ref, R, it, stt, rc = orc.simple_iter(g, pr, st)
    n = 4
    group = mfx.LocalGroup(n)
    res, errs = {}, []
    bar = threading.Barrier(n)

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sd = dev(st)
                ctx = mfx.SimpleContext("234[1]", g, pr, rank=rank, nranks=n, group=group)
                bar.wait()
                ctx.step(sd, stream=stream)
                stream.synchronize()
                res[rank] = {k: host(sd[k]) for k in ("u", "v", "w", "p")}
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
    for r in range(n):
        for k in ("u", "v", "w", "p"):
            assert np.array_equal(res[r][k], ref[k]), (r, k)


def test_bfs_fullsize_assembly_bitwise(mfx, orc):
    """The paper's 10,001,880-cell BFS grid (126 x 63 x 1260):
    momentum (w) and p' assembly, every cell compared."""
    g, pr, st = synth.bfs_case()
    sd = dev(st)
    ws = mfx.Workspace(g)
    ref, r2, rc = orc.assemble_mom(g, pr, 2, st)
    out, res2 = mfx.assemble_eq(mfx.EQ_W, g, pr, sd, ws)
    for k in ("aP", "aW", "aT", "b", "d"):
        assert np.array_equal(host(out[k]), ref[k]), k
    rng = np.random.default_rng(3)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    ref, cont, rc = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    out, res2 = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws,
                                star=[sd["u"], sd["v"], sd["w"]] + [torch.from_numpy(d).cuda() for d in dv])
    for k in ("aE", "aN", "aT", "b"):
        assert np.array_equal(host(out[k]), ref[k]), k
