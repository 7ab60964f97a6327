"""Multi-rank equation decomposition on the GPU:
thread-ranks sharing the one B200 through libmfx's in-process transport run
mfx_simple_iter concurrently, each on its own stream, with the assignment
strings of the paper.  Every rank must end with exactly the state of the
single-rank "111[1]" iteration and of the CPU oracle."""
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


def make_case(n_scalars):
    g = synth.make_grid(24, 14, 30)
    pr = synth.Params(lin_maxit_pp=1500)
    st = synth.make_state(g, 2468, pr, n_scalars=n_scalars)
    rng = np.random.default_rng(5)
    for s in range(n_scalars):
        st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
        st[f"phi{s}"] = st[f"phi_old{s}"].copy()
    return g, pr, st


def run_ranks(mfx, assignment, nranks, g, pr, st, outer=2):
    group = mfx.LocalGroup(nranks)
    results, errors = {}, []
    barrier = threading.Barrier(nranks)

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
                ctx = mfx.SimpleContext(assignment, g, pr, rank=rank, nranks=nranks, group=group)
                barrier.wait()
                outs = [ctx.step(sd, stream=stream) for _ in range(outer)]
                stream.synchronize()
                results[rank] = ({k: v.cpu().numpy() for k, v in sd.items()}, outs)
                ctx.close()
        except Exception as e:  # pragma: no cover - reported below
            errors.append((rank, repr(e)))
            barrier.abort()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errors, errors
    return results


@pytest.mark.parametrize("assignment,nranks,n_scalars", [
    ("222[1]", 2, 0),
    ("234[1]", 4, 0),
    ("121[2]", 2, 0),
    ("234[1]5678", 8, 4),
    ("111[1]2", 2, 1),
    ("234[1234]", 4, 0),          # Fig. 2b: multi-GPU pressure solve
    ("212[12]1", 2, 1),
    ("234[12345678]5678", 8, 4),  # p' over all 8 ranks + 4 scalars
    ("234[23]", 4, 0),            # p' over a subset of the devices ("a set of devices")
    ("123[32]1", 3, 1),           # ... listed out of order: P0 = rank 2, slab 1 on rank 1
])
def test_multirank_equals_single_rank(mfx, orc, assignment, nranks, n_scalars):
    g, pr, st = make_case(n_scalars)
    single = run_ranks(mfx, "111[1]" + "1" * n_scalars, 1, g, pr, st)
    multi = run_ranks(mfx, assignment, nranks, g, pr, st)
    keys = ("u", "v", "w", "p") + tuple(f"phi{s}" for s in range(n_scalars))
    ref_state, ref_outs = single[0]
    for rank in range(nranks):
        state, outs = multi[rank]
        for k in keys:
            assert np.array_equal(state[k], ref_state[k]), (rank, k)
        for o, r in zip(outs, ref_outs):
            assert o["R"] == r["R"] and o["iters"] == r["iters"], (rank, o, r)
    # and the single-rank GPU iteration equals the oracle's two outer iterations
    s = st
    for _ in range(2):
        s, R, iters, status, rc = orc.simple_iter(g, pr, s, n_scalars=n_scalars)
    for k in keys:
        assert np.array_equal(ref_state[k], s[k]), k


def packed_state_dict(st, n):
    """u, v, w, p as views of one [u|v|w|p] device block (mfx_params.packed_state)."""
    sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
    blk = torch.cat([sd["u"], sd["v"], sd["w"], sd["p"]])
    for i, k in enumerate(("u", "v", "w", "p")):
        sd[k] = blk[i * n:(i + 1) * n]
    return sd, blk


@pytest.mark.parametrize("assignment,nranks", [("234[1]", 4), ("222[1]", 2), ("234[1234]", 4), ("234[42]", 4)])
def test_packed_bcast_equals_grouped(mfx, orc, assignment, nranks):
    """BCAST of one [u|v|w|p] block (packed_state = 1) gives the same bits as the
    four grouped broadcasts; a non-contiguous state is refused."""
    g, pr, st = make_case(0)
    ref = run_ranks(mfx, assignment, nranks, g, pr, st)
    prp = synth.Params(lin_maxit_pp=1500, packed_state=1)
    group = mfx.LocalGroup(nranks)
    results, errors = {}, []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sd, blk = packed_state_dict(st, g.n)
                ctx = mfx.SimpleContext(assignment, g, prp, rank=rank, nranks=nranks, group=group)
                outs = [ctx.step(sd, stream=stream) for _ in range(2)]
                stream.synchronize()
                results[rank] = ({k: v.cpu().numpy() for k, v in sd.items()}, outs)
                ctx.close()
        except Exception as e:  # pragma: no cover
            errors.append((rank, repr(e)))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errors, errors
    for rank in range(nranks):
        for k in ("u", "v", "w", "p"):
            assert np.array_equal(results[rank][0][k], ref[rank][0][k]), (rank, k)
        assert [o["iters"] for o in results[rank][1]] == [o["iters"] for o in ref[rank][1]]


def test_packed_state_requires_contiguous_block(mfx):
    g, pr, st = make_case(0)
    prp = synth.Params(lin_maxit_pp=1500, packed_state=1)
    group = mfx.LocalGroup(2)
    errors = []

    def worker(rank):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}   # separate allocations
            ctx = mfx.SimpleContext("222[1]", g, prp, rank=rank, nranks=2, group=group)
            try:
                ctx.step(sd, stream=stream)
            except Exception as e:
                errors.append((rank, str(e)))
            finally:
                ctx.close()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    group.close()
    assert len(errors) == 2 and all("packed_state" in e for _, e in errors), errors
