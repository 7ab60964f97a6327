"""TEST INFRASTRUCTURE (tests/test_gpu_nccl_loopback.py runs this in its own
process): thread-ranks on one GPU drive libmfx's NCCL transport through the
loopback NCCL stand-in (MFX_NCCL_PATH), so every NCCL branch of simple.cu --
grouped send/recv GATHER, broadcast BCAST (also packed), the PIC broadcast,
the multi-GPU p' halo exchange and all-gathers, a split sub-communicator --
runs on real device buffers.  Each case must reproduce "111[1]" bitwise.
Usage: run_loopback.py <libnccl_loopback.so>"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["MFX_NCCL_PATH"] = sys.argv[1]
os.environ["MFX_DIST_GRAPH"] = "0"   # the stand-in synchronises host threads: no graph capture

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2211_15605_b200 as mfx  # noqa: E402


def make_case(n_scalars, packed=False):
    g = synth.make_grid(24, 14, 30)
    pr = synth.Params(lin_maxit_pp=1500, packed_state=1 if packed else 0)
    st = synth.make_state(g, 2468, pr, n_scalars=n_scalars)
    rng = np.random.default_rng(5)
    for s in range(n_scalars):
        st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
        st[f"phi{s}"] = st[f"phi_old{s}"].copy()
    return g, pr, st


def device_state(st, n, packed):
    sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
    if packed:
        blk = torch.cat([sd["u"], sd["v"], sd["w"], sd["p"]])
        for i, k in enumerate(("u", "v", "w", "p")):
            sd[k] = blk[i * n:(i + 1) * n]
    return sd


def run(assignment, nranks, n_scalars, packed=False, outer=2):
    g, pr, st = make_case(n_scalars, packed)
    uid = mfx.nccl_unique_id() if nranks > 1 else None
    res, errs = {}, []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sd = device_state(st, g.n, packed)
                ctx = mfx.SimpleContext(assignment, g, pr, rank=rank, nranks=nranks, uid=uid)
                outs = [ctx.step(sd, stream=stream) for _ in range(outer)]
                stream.synchronize()
                res[rank] = ({k: v.cpu().numpy() for k, v in sd.items()}, outs)
                ctx.close()
        except Exception as e:  # reported below
            errs.append((rank, repr(e)))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert len(res) == nranks, "a rank did not finish"
    return res


def run_pic(nranks):
    """Implicit PIC coupling: the PIC device (rank 0) refreshes the drag fields
    and broadcasts them (exchange phase 3, with its error record)."""
    g = synth.make_grid(16, 12, 20)
    pr = synth.Params(lin_tol_mom=1e-13, lin_maxit_mom=400, lin_tol_pp=1e-13, lin_maxit_pp=6000)
    st = synth.make_state(g, 4321, pr)
    pic = synth.PicParams()
    pc = synth.make_parcels(g, 4322, 6000, st["eps"], pic)
    asg = "111[1]" if nranks == 1 else "234[1]"
    uid = mfx.nccl_unique_id() if nranks > 1 else None
    res, errs = {}, []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
                dpc = {k: torch.from_numpy(v).cuda() for k, v in pc.items()} if rank == 0 else None
                ctx = mfx.SimpleContext(asg, g, pr, rank=rank, nranks=nranks, uid=uid)
                ctx.set_pic(dpc, pic if rank == 0 else None, mfx.PIC_IMPLICIT)
                for _ in range(2):
                    ctx.step(sd, stream=stream)
                stream.synchronize()
                res[rank] = {k: v.cpu().numpy() for k, v in sd.items()}
                ctx.close()
        except Exception as e:
            errs.append((rank, repr(e)))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert len(res) == nranks
    return res


def main():
    cases = [("222[1]", 2, 0, False), ("234[1]", 4, 0, False), ("234[1]", 4, 0, True),
             ("234[1]5678", 8, 4, True), ("234[1234]", 4, 0, False), ("234[23]", 4, 0, True),
             ("123[32]1", 3, 1, False)]
    refs = {}
    for asg, n, ns, packed in cases:
        if ns not in refs:
            refs[ns] = run("111[1]" + "1" * ns, 1, ns)[0]
        ref_state, ref_outs = refs[ns]
        multi = run(asg, n, ns, packed)
        keys = ("u", "v", "w", "p") + tuple(f"phi{s}" for s in range(ns))
        for rank in range(n):
            state, outs = multi[rank]
            for k in keys:
                assert np.array_equal(state[k], ref_state[k]), (asg, rank, k)
            for o, r in zip(outs, ref_outs):
                assert o["iters"] == r["iters"] and o["R"] == r["R"], (asg, rank, o["iters"], r["iters"])
        print(f"loopback NCCL {asg} on {n} ranks{' packed' if packed else ''}: bitwise = 111[1]", flush=True)
    ref = run_pic(1)[0]
    multi = run_pic(4)
    for rank in range(4):
        for k in ("u", "v", "w", "p", "beta", "sbeta_w"):
            assert np.array_equal(multi[rank][k], ref[k]), ("pic", rank, k)
    print("loopback NCCL 234[1] with implicit PIC coupling (phase-3 broadcast) on 4 ranks: bitwise = 111[1]",
          flush=True)
    print("LOOPBACK OK", flush=True)


if __name__ == "__main__":
    main()
