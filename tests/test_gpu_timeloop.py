"""GPU time loop (NEXT-3): mfx_time_step against the
oracle's or_time_step, bitwise, through growth, rejection and multi-rank."""
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


def dev(st):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in st.items()}


def case():
    g = synth.make_grid(16, 12, 20)
    pr = synth.Params(lin_maxit_pp=2000, tol=5e-2)
    st = synth.make_state(g, 55, pr)
    return g, pr, st


CTRL = dict(dt=1e-4, dt_min=2.5e-5, dt_max=5e-4, grow=1.5, shrink=0.5, grow_threshold=2, max_outer=4)


@pytest.mark.parametrize("tol", [5e-2, 0.0])      # converging (growth) / never converging (rejections)
def test_time_steps_bitwise_vs_oracle(mfx, orc, tol):
    g, pr, st = case()
    pr.tol = tol
    sd = dev(st)
    ctx = mfx.SimpleContext("111[1]", g, pr)
    tg, to = mfx.time_ctrl(**CTRL), orc.time_ctrl(**CTRL)
    s = st
    for _ in range(3):
        out = ctx.time_step(sd, tg)
        s, its, R, rc = orc.time_step(g, pr, s, to)
        assert out["outer_iters"] == its
        assert (tg.dt, tg.time, tg.steps, tg.rejected) == (to.dt, to.time, to.steps, to.rejected)
        for k in ("u", "v", "w", "p", "u_old", "eps_old"):
            assert np.array_equal(sd[k].cpu().numpy(), s[k]), k
    ctx.close()
    if tol == 0.0:
        assert tg.rejected > 0


def test_time_step_multirank_identical(mfx, orc):
    g, pr, st = case()
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
                tc = mfx.time_ctrl(**CTRL)
                bar.wait()
                for _ in range(2):
                    ctx.time_step(sd, tc, stream=stream)
                stream.synchronize()
                res[rank] = ({k: sd[k].cpu().numpy() for k in ("u", "v", "w", "p")}, tc.dt, tc.time)
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
    to = orc.time_ctrl(**CTRL)
    s = st
    for _ in range(2):
        s, its, R, rc = orc.time_step(g, pr, s, to)
    for r in range(n):
        f, dt, t = res[r]
        assert dt == to.dt and t == to.time
        for k in f:
            assert np.array_equal(f[k], s[k]), (r, k)
