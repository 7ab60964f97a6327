"""N>1 host logic on CPU: world_size-2 gloo processes run the equation-
decomposed SIMPLE iteration with the schedule libmfx exports
(mfx_parse_assignment + mfx_exchange_plan), the oracle doing
each rank's owned equations and gloo moving the buffers.  The result must be
bitwise identical to the single-process oracle iteration (SPEC.md:457,469:
any assignment gives the same state, payloads are copied, never reduced)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def case(n_scalars):
    import synth
    g = synth.make_grid(10, 6, 9)
    pr = synth.Params(lin_maxit_pp=1000)
    st = synth.make_state(g, 555, pr, n_scalars=n_scalars)
    rng = np.random.default_rng(3)
    for s in range(n_scalars):
        st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
        st[f"phi{s}"] = st[f"phi_old{s}"].copy()
    return g, pr, st


def decomposed_iter(rank, world, assignment, g, pr, st):
    """One outer iteration on `rank`, following libmfx's exchange plan."""
    import oracle
    import paper_2211_15605_b200 as mfx
    a = mfx.parse_assignment(assignment, world)
    owner = a["owner"]
    P = owner[3]
    n = g.n
    bufs = {k: np.zeros(n) for k in ("u", "v", "w", "dx", "dy", "dz")}
    meta = np.zeros((8, 16))
    for c, key in enumerate(("u", "v", "w")):
        if owner[c] != rank:
            continue
        s, r2, rc = oracle.assemble_mom(g, pr, c, st)
        res = oracle.bicgstab(g, s, st[key], pr.lin_tol_mom, pr.lin_maxit_mom)
        bufs[key] = res["x"]
        bufs["d" + "xyz"[c]] = s["d"]
        meta[c, :4] = (r2[0], r2[1], res["iters"], res["status"])
    phinew = {}
    for sc in range(a["n_scalars"]):
        if owner[4 + sc] != rank:
            continue
        s, r2, rc = oracle.assemble_scalar(g, pr, sc, st)
        res = oracle.bicgstab(g, s, st[f"phi{sc}"], pr.lin_tol_phi, pr.lin_maxit_phi)
        phinew[sc] = res["x"]
        meta[4 + sc, :4] = (r2[0], r2[1], res["iters"], res["status"])

    def run(phase, fields):
        plane = g.nx * g.ny
        for op in mfx.exchange_plan(assignment, world, rank, phase, g.nz):
            if op["buf"] != "meta" and op["k1"] > op["k0"]:
                lo, hi = op["k0"] * plane, op["k1"] * plane
                t = torch.from_numpy(fields[op["buf"]][lo:hi].copy())
                if op["op"] == mfx.OP_SEND:
                    dist.send(t, op["peer"])
                else:
                    dist.recv(t, op["peer"])
                    fields[op["buf"]][lo:hi] = t.numpy()
                continue
            if op["buf"] == "meta":
                t = torch.from_numpy(meta[op["slot"]:op["slot"] + op["nslots"]].copy())
            else:
                t = torch.from_numpy(fields[op["buf"]].copy())
            if op["op"] == mfx.OP_SEND:
                dist.send(t, op["peer"])
            elif op["op"] == mfx.OP_RECV:
                dist.recv(t, op["peer"])
            else:
                dist.broadcast(t, op["peer"])
            if op["op"] != mfx.OP_SEND:
                if op["buf"] == "meta":
                    meta[op["slot"]:op["slot"] + op["nslots"]] = t.numpy()
                else:
                    fields[op["buf"]][...] = t.numpy()

    run(0, bufs)
    out = {k: st[k].copy() for k in ("u", "v", "w", "p")}
    for sc in range(a["n_scalars"]):
        out[f"phi{sc}"] = phinew.get(sc, st[f"phi{sc}"].copy())
    if a["n_p"] > 1:
        # multi-GPU p': every rank holds u*, d; solves (serially, same bits as the
        # domain-decomposed solve) and keeps only its slab; PSLAB gathers at P0
        star = [bufs["u"], bufs["v"], bufs["w"]]
        dv = [bufs["dx"], bufs["dy"], bufs["dz"]]
        s, cont, rc = oracle.assemble_pp(g, pr, st, star, dv)
        res = oracle.bicgstab(g, s, np.zeros(n), pr.lin_tol_pp, pr.lin_maxit_pp)
        plane = g.nx * g.ny
        ppf = {"pp": np.zeros(n)}
        if rank in a["p_rank"]:   # slab i of the P list
            k0, k1 = mfx.dist_slab(g.nz, a["p_rank"].index(rank), a["n_p"])
            ppf["pp"][k0 * plane:k1 * plane] = res["x"][k0 * plane:k1 * plane]
        run(2, ppf)
        meta[3, :4] = (cont, 0.0, res["iters"], res["status"])
        if rank == P:
            assert np.array_equal(ppf["pp"], res["x"])      # the slabs tile the field
            u, v, w, p = oracle.correct(g, pr, star, dv, ppf["pp"], st["p"])
            out.update(u=u, v=v, w=w, p=p)
    elif rank == P:
        star = [bufs["u"], bufs["v"], bufs["w"]]
        dv = [bufs["dx"], bufs["dy"], bufs["dz"]]
        s, cont, rc = oracle.assemble_pp(g, pr, st, star, dv)
        res = oracle.bicgstab(g, s, np.zeros(n), pr.lin_tol_pp, pr.lin_maxit_pp)
        u, v, w, p = oracle.correct(g, pr, star, dv, res["x"], st["p"])
        out.update(u=u, v=v, w=w, p=p)
        meta[3, :4] = (cont, 0.0, res["iters"], res["status"])
    run(1, out)
    return out, meta


def worker(rank, world, port, assignment, n_scalars, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, pr, st = case(n_scalars)
        out, meta = decomposed_iter(rank, world, assignment, g, pr, st)
        q.put((rank, {k: v for k, v in out.items()}, meta))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("assignment,n_scalars", [("222[1]", 0), ("121[2]", 0), ("211[1]2", 1), ("112[2]12", 2),
                                                   ("212[12]", 0), ("122[12]2", 1), ("122[21]", 0)])
def test_two_rank_decomposition_bitwise(orc, mfx_built, assignment, n_scalars):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, assignment, n_scalars, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, out, meta = q.get(timeout=600)
        results[rank] = (out, meta)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g, pr, st = case(n_scalars)
    ref, R, iters, status, rc = orc.simple_iter(g, pr, st, n_scalars=n_scalars)
    for rank in range(world):
        out, meta = results[rank]
        for k in ("u", "v", "w", "p") + tuple(f"phi{s}" for s in range(n_scalars)):
            assert np.array_equal(out[k], ref[k]), (rank, k)
        # residual record identical on every rank and equal to the serial one
        Rm = [meta[c, 0] / max(meta[c, 1], 1e-30) for c in range(3)] + [meta[3, 0]]
        assert np.array_equal(np.array(Rm), R)
        assert [int(meta[q_, 2]) for q_ in range(4)] == iters[:4]
