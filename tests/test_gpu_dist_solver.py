"""Domain-decomposed (z-slab) BiCGSTAB (mfx_dist_solve): the comparator of
BASELINE configuration 5 and the basis of a multi-GPU pressure solve (P:85,
P:87).  Thread-ranks on the one GPU (in-process transport) each own a
slab; halo planes and double-double dot partials cross ranks every iteration.
Because the dots are correctly rounded, the iterates must equal the CPU
oracle's (and the single-GPU solve's) bitwise for any number of ranks."""
import threading

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


def slab_dict(sysd, g, k0, k1):
    plane = g.nx * g.ny
    return {k: torch.from_numpy(np.ascontiguousarray(v[k0 * plane:k1 * plane])).cuda() for k, v in sysd.items()}


def dist_run(mfx, g, pr, kind, sysd, x0, tol, maxit, R):
    group = mfx.LocalGroup(R)
    res, errors = {}, []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx = mfx.SimpleContext("111[1]", g, pr, rank=rank, nranks=R, group=group)
                k0, k1 = mfx.dist_slab(g.nz, rank, R)
                sl = slab_dict(sysd, g, k0, k1)
                plane = g.nx * g.ny
                x = torch.from_numpy(np.ascontiguousarray(x0[k0 * plane:k1 * plane])).cuda()
                info = ctx.dist_solve(kind, sl, x, tol, maxit, stream=stream)
                stream.synchronize()
                res[rank] = (k0, k1, x.cpu().numpy(), info)
                ctx.close()
        except Exception as e:  # pragma: no cover
            errors.append((rank, repr(e)))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errors, errors
    plane = g.nx * g.ny
    x = np.zeros(g.n)
    for rank, (k0, k1, xs, info) in res.items():
        x[k0 * plane:k1 * plane] = xs
    infos = [res[r][3] for r in range(R)]
    assert all(i == infos[0] for i in infos), infos   # identical decisions on every rank
    return x, infos[0]


def pp_system(orc, g, pr, st, seed=0):
    rng = np.random.default_rng(seed)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    return sysd


@pytest.mark.parametrize("R", [1, 2, 3, 4])
def test_dist_pp_c1_equals_oracle(mfx, orc, R):
    g, pr, st = synth.config_case(1)
    sysd = pp_system(orc, g, pr, st)
    ref = orc.bicgstab(g, sysd, np.zeros(g.n), 1e-6, 2000)
    x, info = dist_run(mfx, g, pr, mfx.EQ_PP, sysd, np.zeros(g.n), 1e-6, 2000, R)
    assert info["iters"] == ref["iters"] and info["status"] == ref["status"]
    assert np.array_equal(x, ref["x"])


@pytest.mark.parametrize("R", [2, 5])
def test_dist_momentum_ragged_equals_oracle(mfx, orc, R):
    g = synth.make_grid(10, 7, 9)
    pr = synth.Params()
    st = synth.make_state(g, 41, pr)
    sysd, _, _ = orc.assemble_mom(g, pr, 2, st)
    ref = orc.bicgstab(g, sysd, st["w"], 1e-10, 300)
    x, info = dist_run(mfx, g, pr, mfx.EQ_W, sysd, st["w"], 1e-10, 300, R)
    assert info["iters"] == ref["iters"]
    assert np.array_equal(x, ref["x"])


def test_dist_pp_tall_many_ranks_not_converged(mfx, orc):
    """maxit reached: the last iterate, identical to the oracle, on 6 ranks."""
    g = synth.make_grid(6, 5, 41)
    pr = synth.Params()
    st = synth.make_state(g, 43, pr)
    sysd = pp_system(orc, g, pr, st, seed=3)
    ref = orc.bicgstab(g, sysd, np.zeros(g.n), 1e-14, 37)
    x, info = dist_run(mfx, g, pr, mfx.EQ_PP, sysd, np.zeros(g.n), 1e-14, 37, 6)
    assert ref["status"] == 1 and info["status"] == 1 and info["iters"] == 37
    assert np.array_equal(x, ref["x"])


@pytest.mark.parametrize("R", [1, 3])
def test_dist_pp_tma_ragged_tiles_equals_oracle(mfx, orc, R):
    """p' on the TMA row-warp slab kernels (nx > 64, ragged x and y tiles, uneven
    slabs): every iterate path -- ghost-plane recompute of p and s, the v and r
    halos, the rank-ordered dd fold -- must reproduce the oracle bitwise."""
    g = synth.make_grid(70, 36, 50)
    pr = synth.Params()
    st = synth.make_state(g, 47, pr)
    sysd = pp_system(orc, g, pr, st, seed=5)
    ref = orc.bicgstab(g, sysd, np.zeros(g.n), 1e-9, 120)
    x, info = dist_run(mfx, g, pr, mfx.EQ_PP, sysd, np.zeros(g.n), 1e-9, 120, R)
    assert info["iters"] == ref["iters"] and info["status"] == ref["status"]
    assert np.array_equal(x, ref["x"])


def test_dist_pp_tma_nonzero_guess_uneven_slabs(mfx, orc):
    """A nonzero initial guess and a tolerance that needs many iterations on 4
    uneven slabs (nz = 23): bitwise against the oracle, status included."""
    g = synth.make_grid(16, 14, 23)
    pr = synth.Params()
    st = synth.make_state(g, 53, pr)
    sysd = pp_system(orc, g, pr, st, seed=9)
    x0 = np.random.default_rng(2).normal(0.0, 1e-3, g.n)
    ref = orc.bicgstab(g, sysd, x0, 1e-12, 400)
    x, info = dist_run(mfx, g, pr, mfx.EQ_PP, sysd, x0, 1e-12, 400, 4)
    assert info["iters"] == ref["iters"] and info["status"] == ref["status"]
    assert np.array_equal(x, ref["x"])
