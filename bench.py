#!/usr/bin/env python
"""bench.py -- BiCGSTAB iters/s (and SIMPLE iters/s) of the equation-decomposed
SIMPLE hot path on B200, BASELINE.json metric, configuration 2 grid.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mfx|reference]

A step is one SIMPLE outer iteration (all SURVEY §8(a) rows: u, v, w momentum
assembly + BiCGSTAB, p' assembly + BiCGSTAB, correction, state exchange) on the
128x128x512 fluidized-bed grid (8.4M cells, fp64).  `value` = BiCGSTAB
iterations completed by all equations on all ranks / device time (CUDA events,
max over ranks); `e2e` = the same metric through the C ABI with the snapshot
copied from pinned host memory and u, v, w, p read back inside the timed region.

--impl reference times the CPU oracle (oracle/, OpenMP over this host's cores,
parity mode) on a bounded sample of the same workload: it is the "reference
arm" of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BiCGSTAB iters/s and SIMPLE iters/s per grid; achieved HBM GB/s vs 8 TB/s"
UNIT = "iters/s"
CONFIG_ID = 2

# algorithmic bytes per cell per launch (SURVEY §8(d) byte model)
BYTES_PER_CELL = {
    "K1_mom": 4 * 8 + 2 * 8 + 7 * 8,     # r, p_old, v_old, r^ read; p, v write; 7 coefficients
    "K2_mom": 2 * 8 + 1 * 8 + 7 * 8,     # r, v read; t write; 7 coefficients
    "K1_pp": 4 * 8 + 2 * 8 + 3 * 8,      # symmetric p' storage c_x, c_y, c_z; aP = row sum, not read
    "K2_pp": 2 * 8 + 1 * 8 + 3 * 8,
    "K3": 6 * 8 + 2 * 8,                 # x, p, r, v, t, r^ read; x, r write
    "assemble_mom": 9 * 8 + 9 * 8,       # eps, eps0, u, v, w, c_old, p, beta, S read; 7 coef + b + d write
    "assemble_pp": 8 * 8 + 5 * 8,        # eps, eps0, u*, v*, w*, d_x, d_y, d_z read; aP, c_x, c_y, c_z, b write
    "correct": 8 * 8 + 4 * 8,            # u*, v*, w*, d_x, d_y, d_z, p', p read; u, v, w, p write
    "spmv_setup": None, "assemble_scalar": None,
}
PP_ITER_BPC = BYTES_PER_CELL["K1_pp"] + BYTES_PER_CELL["K2_pp"] + BYTES_PER_CELL["K3"]   # 184


def assignment_for(n):
    """Equation decomposition per GPU count (PAPER.md:95 notation; p' on GPU 1,
    momentum on the others, then energy + species scalars on GPUs 5..8)."""
    fixed = {1: "111[1]", 2: "222[1]", 3: "233[1]", 4: "234[1]"}
    if n in fixed:
        return fixed[n]
    return "234[1]" + "".join(str(5 + s) for s in range(min(n - 4, 4)))


def assignment_multi_p(n):
    """Same equation owners, pressure correction split over every GPU ([12..n])."""
    base = assignment_for(n)
    head, tail = base.split("]")
    return head.split("[")[0] + "[" + "".join(str(i + 1) for i in range(n)) + "]" + tail


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def bench_config(asg, grid, n_scal):
    return {"workload": "c2: one SIMPLE outer iteration per step on 128x128x512 "
                        f"(assignment {asg}): u,v,w momentum assembly+BiCGSTAB "
                        "(tol 1e-4, maxit 20), p' assembly+BiCGSTAB (tol 1e-6, maxit 500), "
                        "correction, state exchange",
            "grid": list(grid), "assignment": asg, "equations": 4 + n_scal,
            "l2": "inputs larger than L2 (13 fields x 64 MiB snapshot + systems >> 126 MB)"}


# ---------------------------------------------------------------- reference arm (oracle)
PAPER_CONTEXT = ("PAPER.md:17/:165: 4 x A100 over NVLink competitive with ~1000 JOULE 2.0 CPU cores "
                 "(25 nodes x 40 cores); context only, not this run")


def cpu_info():
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = None
    try:
        out = subprocess.check_output(["lscpu"], text=True)
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return cores, model


def oracle_pp_system(cid):
    """The oracle-assembled p' system of configuration `cid` (u* = the snapshot
    velocities, d = seeded U(1e-4, 1e-3)); returns (grid, params, sysd, seconds)."""
    import numpy as np
    import oracle
    import synth
    g, pr, st = synth.config_case(cid)
    rng = np.random.default_rng(0)
    dv = [rng.uniform(1e-4, 1e-3, g.n) for _ in range(3)]
    t0 = time.perf_counter()
    sysd, _, _ = oracle.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv)
    return g, pr, st, sysd, time.perf_counter() - t0


def oracle_iter_seconds(g, sysd, k1, k2):
    """Seconds per BiCGSTAB iteration of the oracle, (T(k2) - T(k1)) / (k2 - k1)
    (excludes the setup r = b - A x0); tol 0 so no early exit."""
    import numpy as np
    import oracle
    ts = []
    for k in (k1, k2):
        t0 = time.perf_counter()
        oracle.bicgstab(g, sysd, np.zeros(g.n), 0.0, k)
        ts.append(time.perf_counter() - t0)
    return (ts[1] - ts[0]) / (k2 - k1), ts


def cpu_baseline_measure():
    """The oracle as it stands, on this host's cores (SURVEY §8(d) oracle timing):
    parity mode (exact dots; bit-identical for any thread count) on all cores
    and on one core, naive-dot mode on all cores; p' BiCGSTAB s/iteration at
    c2 (value) and c1, plus the c2 p' and w-momentum assembly.  About 10-30 s."""
    import oracle
    import synth
    cores, model = cpu_info()
    t_all = time.perf_counter()
    res = {"cores": cores, "cpu_model": model, "kind": "oracle", "unit": UNIT}
    oracle.set_mode(cores, False)
    g2, pr2, st2, s2, t_asm_pp = oracle_pp_system(2)
    t0 = time.perf_counter()
    oracle.assemble_mom(g2, pr2, 2, st2)
    t_asm_mom = time.perf_counter() - t0
    par2, _ = oracle_iter_seconds(g2, s2, 1, 3)
    oracle.set_mode(cores, True)
    nai2, _ = oracle_iter_seconds(g2, s2, 1, 3)
    oracle.set_mode(cores, False)
    del st2, s2
    g1, _, _, s1, _ = oracle_pp_system(1)
    par1, _ = oracle_iter_seconds(g1, s1, 10, 110)
    oracle.set_mode(1, False)
    g3, _, _, s3, _ = oracle_pp_system(3)
    one3, _ = oracle_iter_seconds(g3, s3, 1, 3)
    oracle.set_mode(cores, False)
    res.update({
        "value": 1.0 / par2,
        "sample": ("c2 (128x128x512) p' BiCGSTAB on the oracle-assembled system, parity mode "
                   f"(correctly rounded dots), {cores} threads, (T(3) - T(1)) / 2 per iteration"),
        "c2_pp": {"parity_all_cores_s_per_iter": par2, "naive_dots_all_cores_s_per_iter": nai2,
                  "parity_iters_per_s": 1.0 / par2, "naive_iters_per_s": 1.0 / nai2,
                  "assemble_pp_s": t_asm_pp, "assemble_mom_w_s": t_asm_mom},
        "c1_pp": {"parity_all_cores_us_per_iter": 1e6 * par1, "iters_per_s": 1.0 / par1,
                  "note": "8192 cells: below the oracle's parallel threshold, runs on one thread"},
        "c3_pp_one_core": {"parity_s_per_iter": one3, "iters_per_s": 1.0 / one3},
        "paper_context": PAPER_CONTEXT,
        "seconds": time.perf_counter() - t_all,
    })
    return res


def run_reference(args, rank, world):
    """The reference arm of this tier: the CPU oracle on this host's cores, on
    the product arm's workload (the c2 p' BiCGSTAB iteration, BiCGSTAB iters/s).
    One solve of W iterations and one of W + K iterations: the K timed
    iterations are the difference (setup excluded).  Under torchrun only rank 0
    runs it."""
    if rank != 0:
        return
    import oracle
    cores, model = cpu_info()
    oracle.set_mode(cores, False)
    g, pr, st, sysd, _ = oracle_pp_system(CONFIG_ID)
    del st
    w = max(args.warmup, 1)
    per_it, ts = oracle_iter_seconds(g, sysd, w, w + args.steps)
    v = 1.0 / per_it
    sample = (f"c2 p' BiCGSTAB on the oracle-assembled 128x128x512 system, parity mode (correctly rounded "
              f"dots), {cores} threads; step = one iteration: (T(W+K) - T(W)) / K with W = {w}")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per_it,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded fluidized-bed fields, synth/)",
            "config": bench_config("111[1]", (128, 128, 512), 0),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "cpu_model": model, "kind": "oracle",
                             "sample": sample, "paper_context": PAPER_CONTEXT},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- other BASELINE grids
def measure_other_configs(mfx, torch):
    """Side measurements on the other BASELINE.json grids (same kernels, N=1):
    config 1: the p' BiCGSTAB solve (tol 1e-6, maxit 5000) on 16x16x32 (single-
    cluster solver); configs 3 and 4: SIMPLE outer iterations '111[1]' on
    64x64x256 and 256x256x512 (4 equations on one GPU)."""
    import numpy as np
    import synth
    out = {}
    # config 1: p' system from the GPU's own momentum predictors
    g, pr, st = synth.config_case(1)
    pr.lin_maxit_pp = 5000
    sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
    ctx = mfx.SimpleContext("111[1]", g, pr)
    ctx.step({k: v.clone() for k, v in sd.items()})
    star = [ctx.buffer(k) for k in ("u*", "v*", "w*", "dx", "dy", "dz")]
    ws = mfx.Workspace(g)
    sysd, _ = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=star)
    ctx.close()
    times, iters = [], 0
    for rep in range(12):
        x = torch.zeros(g.n, dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        info = mfx.bicgstab_solve(mfx.EQ_PP, g, sysd, x, pr.lin_tol_pp, pr.lin_maxit_pp, ws)
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            times.append(e0.elapsed_time(e1))
        iters = info["iters"]
    ms = float(np.median(times))
    out["c1"] = {"workload": "p' BiCGSTAB solve 16x16x32, tol 1e-6 (single-cluster solver)",
                 "iters": iters, "ms_per_solve": ms, "us_per_iter": 1e3 * ms / iters,
                 "bicgstab_iters_per_s": iters / (ms / 1e3),
                 "solver": f"single cluster of {mfx.get_option('cluster_size')} CTAs (one launch per solve)",
                 "memory_regime": "shared-memory resident: the whole system lives in the cluster's shared memory "
                                  "for the solve (DRAM: one read of the system, one write of x)"}
    out["c2_momentum"] = measure_momentum_c2(mfx, torch)
    for cid, steps in ((3, 5), (4, 3)):
        g, pr, st = synth.config_case(cid)
        sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
        ctx = mfx.SimpleContext("111[1]", g, pr)
        ctx.step(sd)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its = 0
        for _ in range(steps):
            o = ctx.step(sd)
            its += sum(o["iters"][:4])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ph = ctx.phase_times()
        pp_it = max(o["iters"][3], 1)
        out[f"c{cid}"] = {"workload": f"SIMPLE outer iteration 111[1] on {g.nx}x{g.ny}x{g.nz}",
                          "simple_iters_per_s": steps / (ms / 1e3),
                          "bicgstab_iters_per_s": its / (ms / 1e3),
                          "pp_us_per_iter": 1e3 * ph["pp"] / pp_it,
                          "pp_alg_GBps": PP_ITER_BPC * g.n / (1e-3 * ph["pp"] / pp_it) / 1e9,
                          "iters_last": o["iters"][:4],
                          "memory_regime": ("L2-resident reads: p' working set 92 MB < 126 MB L2 (ncu of the "
                                            "persistent solver: 90% L2 hit rate, profiles/r02q_ncu_summary.md); "
                                            "latency-bound" if cid == 3 else
                                            "HBM-streaming: working set >> 126 MB L2")}
        ctx.close()
        del sd
        torch.cuda.empty_cache()
    out["bfs_10M"] = measure_bfs(mfx, torch)
    out["c5_one_gpu"] = measure_scalars_one_gpu(mfx, torch)
    out["pic_coupling"] = measure_pic(mfx, torch)
    return out


def measure_pic(mfx, torch):
    """NEXT-2: the PIC device's coupling deposits on the
    configuration 2 grid with the paper's parcel count, parcels
    in random order and sorted by cell.  Per launch pair: the eps deposit
    (zero fill + k_pic_eps + finalize) and the drag deposit (4 zero fills +
    k_pic_drag).  Unique HBM bytes: parcels 32 / 56 B, fields 16N (eps: zero +
    finalize read/write ~ 24N) / 4 x 8N written + 4 x 8N gathered."""
    import numpy as np
    import synth
    g, pr, st = synth.config_case(CONFIG_ID)
    pic = synth.PicParams()
    pc = synth.make_parcels(g, 15605 + 77, synth.PAPER_PARCELS, st["eps"], pic)
    cell = (np.minimum((pc["x"] / g.dx).astype(np.int64), g.nx - 1) + g.nx *
            (np.minimum((pc["y"] / g.dy).astype(np.int64), g.ny - 1) + g.ny *
             np.minimum((pc["z"] / g.dz).astype(np.int64), g.nz - 1)))
    order = np.argsort(cell, kind="stable")
    ws = mfx.Workspace(g)
    u, v, w = (torch.from_numpy(st[k]).cuda() for k in ("u", "v", "w"))
    eps = torch.empty(g.n, dtype=torch.float64, device="cuda")
    outs = {k: torch.empty(g.n, dtype=torch.float64, device="cuda") for k in ("beta", "sbeta_u", "sbeta_v", "sbeta_w")}
    res = {"workload": f"{synth.PAPER_PARCELS} parcels (PAPER.md:155) on 128x128x512", "parcels": synth.PAPER_PARCELS}
    m = synth.PAPER_PARCELS
    for name, idx in (("random_order", None), ("cell_sorted", order)):
        d = {k: torch.from_numpy(np.ascontiguousarray(a if idx is None else a[idx])).cuda() for k, a in pc.items()}
        t_eps, _ = _ev_ms(torch, lambda: mfx.pic_deposit_eps(g, pic, d, ws, eps=eps), 7)
        t_drag, _ = _ev_ms(torch, lambda: mfx.pic_drag(g, pr, pic, d, eps, u, v, w, ws, out=outs), 7)
        ws.check()
        if idx is None:   # GPU counting sort of the random-order parcels (once per time step)
            srt = {k: torch.empty_like(v) for k, v in d.items()}
            nb = int(mfx.lib().mfx_pic_sort_scratch_bytes(mfx.c_grid(g), m))
            scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
            t_sort, _ = _ev_ms(torch, lambda: mfx.pic_sort(g, pic, d, out=srt, scratch=scratch), 7)
            t_drag_sorted, _ = _ev_ms(torch, lambda: mfx.pic_drag(g, pr, pic, srt, eps, u, v, w, ws, out=outs), 7)
            vals = torch.empty(7 * m, dtype=torch.float64, device="cuda")
            t_gather, _ = _ev_ms(torch, lambda: mfx.pic_drag_binned(g, pr, pic, srt, eps, u, v, w, ws, out=outs,
                                                                    vals=vals), 7)
            t_eps_gather, _ = _ev_ms(torch, lambda: mfx.pic_deposit_eps_binned(g, pic, srt, ws, eps=eps, vals=vals), 7)
            res["gpu_sort"] = {"sort_us": 1e3 * t_sort, "drag_deposit_after_sort_us": 1e3 * t_drag_sorted,
                               "drag_binned_gather_us": 1e3 * t_gather, "eps_binned_gather_us": 1e3 * t_eps_gather,
                               "note": "binned gathers: deterministic, bitwise the parcel-ordered definition"}
            del vals
            del srt, scratch
        res[name] = {"eps_deposit_us": 1e3 * t_eps, "drag_deposit_us": 1e3 * t_drag,
                     "parcels_per_s_drag": m / (t_drag * 1e-3),
                     "atomic_updates_per_s_drag": 32 * m / (t_drag * 1e-3),
                     "drag_unique_GBps": (56 * m + 8 * 8 * g.n) / (t_drag * 1e-3) / 1e9}
        del d
    torch.cuda.empty_cache()
    return res


def _ev_ms(torch, fn, reps):
    """Median device time (CUDA events on the current stream) of fn() over reps."""
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), r


def measure_bfs(mfx, torch):
    """NEXT-3 geometry: the paper's single-phase backward-facing step
    (Fig. 8) at its 10,001,880-cell size (PAPER.md:165,
    126 x 63 x 1260, BLOCKED cells for the step), SIMPLE outer iterations
    '111[1]' (4 equations on one GPU)."""
    import synth
    g, pr, st = synth.bfs_case()
    sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
    ctx = mfx.SimpleContext("111[1]", g, pr)
    ctx.step(sd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps, its = 3, 0
    e0.record()
    for _ in range(steps):
        o = ctx.step(sd)
        its += sum(o["iters"][:4])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ph = ctx.phase_times()
    ctx.close()
    pp_it = max(o["iters"][3], 1)
    res = {"workload": f"BFS single phase, {g.nx}x{g.ny}x{g.nz} = {g.n} cells (block: {g.nx // 2}x{g.ny}x{g.nz // 10}), "
                       "SIMPLE 111[1]",
           "simple_iters_per_s": steps / (ms / 1e3), "ms_per_simple_iter": ms / steps,
           "bicgstab_iters_per_s": its / (ms / 1e3), "iters_last": o["iters"][:4],
           "pp_us_per_iter": 1e3 * ph["pp"] / pp_it,
           "pp_alg_GBps": PP_ITER_BPC * g.n / (1e-3 * ph["pp"] / pp_it) / 1e9,
           "phase_ms_last": ph}
    del sd
    torch.cuda.empty_cache()
    return res


def measure_momentum_c2(mfx, torch):
    """BASELINE.json configs[1] exactly: one momentum equation (w: convection-
    diffusion + implicit drag) assembled and solved on 128x128x512, 1 GPU.
    Per-iteration time by the SURVEY §8(d) procedure: tol = 0 with maxit 2 and
    10, (T10 - T2) / 8, which excludes the setup."""
    import synth
    g, pr, st = synth.config_case(CONFIG_ID)
    sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
    ws = mfx.Workspace(g)
    sysd = mfx.new_system(mfx.EQ_W, g.n)
    asm_ms, _ = _ev_ms(torch, lambda: mfx.assemble_eq(mfx.EQ_W, g, pr, sd, ws, out=sysd), 7)
    x = sd["w"].clone()

    def solve(tol, maxit):
        x.copy_(sd["w"])
        return mfx.bicgstab_solve(mfx.EQ_W, g, sysd, x, tol, maxit, ws)
    solve_ms, info = _ev_ms(torch, lambda: solve(pr.lin_tol_mom, pr.lin_maxit_mom), 7)
    t2, _ = _ev_ms(torch, lambda: solve(0.0, 2), 7)
    t10, _ = _ev_ms(torch, lambda: solve(0.0, 10), 7)
    it_us = 1e3 * (t10 - t2) / 8
    bpc = BYTES_PER_CELL["K1_mom"] + BYTES_PER_CELL["K2_mom"] + BYTES_PER_CELL["K3"]
    res = {"workload": "configs[1]: w-momentum assembly + BiCGSTAB (tol 1e-4, maxit 20, x0 = snapshot) "
                       "on 128x128x512",
           "assemble_us": 1e3 * asm_ms,
           "assemble_alg_GBps": BYTES_PER_CELL["assemble_mom"] * g.n / (asm_ms * 1e-3) / 1e9,
           "solve_iters": info["iters"], "solve_us": 1e3 * solve_ms,
           "assemble_plus_solve_per_s": 1e3 / (asm_ms + solve_ms),
           "bicgstab_iters_per_s": info["iters"] / ((asm_ms + solve_ms) * 1e-3),
           "us_per_iter": it_us, "iter_alg_GBps": bpc * g.n / (it_us * 1e-6) / 1e9}
    del sd, sysd, ws, x
    torch.cuda.empty_cache()
    return res


def measure_scalars_one_gpu(mfx, torch):
    """Configuration 5, strong reading (ii) at N = 1: the fixed 8-equation set
    {u, v, w, p', E, Y1, Y2, Y3} ('111[1]1111') against the 4-equation '111[1]',
    one SIMPLE outer iteration each, on the c3 and c2 grids."""
    import numpy as np
    import synth
    res = {}
    for cid in (3, 2):
        g, pr, st = synth.config_case(cid, n_scalars=4)
        rng = np.random.default_rng(77)
        for s in range(4):
            st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
            st[f"phi{s}"] = st[f"phi_old{s}"].copy()
        base = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
        row = {}
        for asg in ("111[1]", "111[1]1111"):
            ctx = mfx.SimpleContext(asg, g, pr)
            sd = {k: v.clone() for k, v in base.items()}
            ctx.step(sd)
            ms_l, its = [], 0
            for _ in range(3):
                sd = {k: v.clone() for k, v in base.items()}
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                o = ctx.step(sd)
                e1.record()
                torch.cuda.synchronize()
                ms_l.append(e0.elapsed_time(e1))
                its = sum(o["iters"])
            ms = statistics.median(ms_l)
            row[asg] = {"ms_per_simple_iter": ms, "bicgstab_iters": its, "iters": o["iters"],
                        "equation_solves_per_s": (4 if asg == "111[1]" else 8) / (ms * 1e-3)}
            ctx.close()
        res[f"c{cid}"] = row
        del base
        torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- product arm
def run_mfx(args, rank, world, local_rank):
    import numpy as np
    import torch
    import synth
    import paper_2211_15605_b200 as mfx

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    g, pr, st = synth.config_case(CONFIG_ID, n_scalars=4)
    asg = assignment_for(world)
    n_scal = mfx.parse_assignment(asg, world)["n_scalars"]
    if n_scal:
        rng = np.random.default_rng(77)
        for s in range(n_scal):
            st[f"phi_old{s}"] = rng.uniform(0, 1, g.n)
            st[f"phi{s}"] = st[f"phi_old{s}"].copy()
    keep = list(synth.FIELD_NAMES) + [f"phi{s}" for s in range(n_scal)] + [f"phi_old{s}" for s in range(n_scal)]
    host = {k: torch.from_numpy(st[k]).pin_memory() for k in keep}
    sd = {k: v.cuda(non_blocking=True) for k, v in host.items()}
    if world > 1:
        # BCAST as one broadcast of the [u|v|w|p] block (mfx_params.packed_state)
        blk = torch.cat([sd["u"], sd["v"], sd["w"], sd["p"]])
        for i, k in enumerate(("u", "v", "w", "p")):
            sd[k] = blk[i * g.n:(i + 1) * g.n]
        pr.packed_state = 1
    uid = None
    if world > 1:
        obj = [mfx.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = mfx.SimpleContext(asg, g, pr, rank=rank, nranks=world, uid=uid)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier(device_ids=[local_rank])

    def my_iters(out):
        owner = ctx.assignment["owner"]
        return sum(out["iters"][q] for q in range(8) if owner[q] >= 0)

    # ---- warm-up (untimed)
    for _ in range(args.warmup):
        ctx.step(sd)
    # ---- device-timed region: K consecutive SIMPLE outer iterations
    for k in ("u", "v", "w", "p"):
        sd[k].copy_(host[k], non_blocking=True)
    clocks = ClockSampler(local_rank)
    barrier()
    clocks.start()
    l0 = mfx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    outs = []
    for _ in range(args.steps):
        outs.append(ctx.step(sd))
    ev1.record(stream)
    barrier()
    launches = mfx.launch_count() - l0
    clk = clocks.stop()
    t_ms = ev0.elapsed_time(ev1)
    phase = ctx.phase_times()
    xch = phase["gather"] + phase["bcast"]   # this rank's exchange time in the last step (comm stream)
    if dist is not None:
        tt = torch.tensor([t_ms, xch], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, xch = float(tt[0].item()), float(tt[1].item())
    # iterations: every equation counted once (owners are disjoint; identical records on all ranks)
    it_all = sum(outs[i]["iters"][q] for i in range(len(outs)) for q in range(8)
                 if ctx.assignment["owner"][q] >= 0)
    value = it_all / (t_ms / 1e3)
    simple_per_s = args.steps / (t_ms / 1e3)

    # ---- instrumented replay of the same K steps: CUDA events recorded by libmfx
    # on the launching stream around every hot kernel (graphs off while
    # instrumented, so this pass is slightly slower than the timed one)
    for k in ("u", "v", "w", "p"):
        sd[k].copy_(host[k], non_blocking=True)
    barrier()
    mfx.prof_reset()
    mfx.prof_enable(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        ctx.step(sd)
    p1.record(stream)
    barrier()
    mfx.prof_enable(False)
    prof = mfx.prof_read()
    t_prof_ms = p0.elapsed_time(p1)

    # ---- roofline of the dominant kernel
    n = g.n
    peak, peak_kind = load_peaks()
    best = max((k for k in prof if prof[k]["launches"]), key=lambda k: prof[k]["ms"])
    kern = best
    roof = None
    if BYTES_PER_CELL.get(kern) is not None:
        per_launch_ms = prof[kern]["ms"] / prof[kern]["launches"]
        alg = BYTES_PER_CELL[kern] * n
        achieved = alg / (per_launch_ms / 1e3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f)["dram_bytes_per_launch"].get(kern)
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_kind,
                "alg_bytes_per_launch": alg, "avg_launch_us": per_launch_ms * 1e3,
                "traffic": traffic, "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes_read+write per launch)",
                "share_of_step": prof[kern]["ms"] / t_prof_ms,
                "timing": "CUDA events around each launch on its stream, instrumented replay of the timed steps"}
    kern_ms = {k: (prof[k]["ms"] / prof[k]["launches"] if prof[k]["launches"] else None) for k in prof}
    # every kernel class with a byte model: achieved algorithmic GB/s and fraction of the measured peak.
    # Solves that converge inside a launch chunk leave no-op launches behind (they exit at once), so the
    # per-call time divides the total by the iterations actually executed (identical in both passes:
    # the instrumented replay restarts from the same state and the solver is deterministic).
    owner = ctx.assignment["owner"]
    it_pp = sum(o["iters"][3] for o in outs if owner[3] >= 0)
    it_mom = sum(o["iters"][q] for o in outs for q in range(3) if owner[q] >= 0)
    it_sc = sum(o["iters"][q] for o in outs for q in range(4, 8) if owner[q] >= 0)
    eff = {"K1_pp": it_pp, "K2_pp": it_pp, "K1_mom": it_mom + it_sc, "K2_mom": it_mom + it_sc,
           "K3": it_pp + it_mom + it_sc}
    kernels_roof = {}
    for k, v in prof.items():
        if v["launches"] and BYTES_PER_CELL.get(k):
            calls = eff.get(k) or v["launches"]
            us = 1e3 * v["ms"] / calls
            gbs = BYTES_PER_CELL[k] * g.n / (us * 1e-6) / 1e9
            kernels_roof[k] = {"launches": v["launches"], "executed": calls, "avg_us": us,
                               "alg_bytes": BYTES_PER_CELL[k] * g.n, "achieved_GBps": gbs,
                               "frac": gbs / load_peaks()[0], "share_of_step": v["ms"] / t_prof_ms}
    # whole-iteration algorithmic bandwidth of the p' solve (K1 + K2 + K3 per iteration)
    pp_iter_bytes = (BYTES_PER_CELL["K1_pp"] + BYTES_PER_CELL["K2_pp"] + BYTES_PER_CELL["K3"]) * n

    # ---- e2e through the C ABI with host buffers.  Every step copies its inputs
    # (the 13-field snapshot, pinned host memory) to the device and reads u, v,
    # w, p back.  Double-buffered: step i+1's inputs travel on a copy stream
    # while step i computes, and step i's results come back while step i+1
    # computes; the timed region closes after the last read-back.
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d = sum(v.numel() * 8 for v in host.values())
    e2e_steps = max(1, args.steps)
    outbufs = [{k: torch.empty_like(host[k]).pin_memory() for k in ("u", "v", "w", "p")} for _ in range(e2e_steps)]
    d2h = sum(v.numel() * 8 for v in outbufs[0].values())
    bufs = [sd, {k: torch.empty_like(v) for k, v in sd.items()}]
    copy_stream = torch.cuda.Stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    computed = [torch.cuda.Event(), torch.cuda.Event()]

    def upload(i):
        dst = bufs[i % 2]
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(computed[i % 2])        # the step that last used this buffer is done
            for k, v in host.items():
                dst[k].copy_(v, non_blocking=True)
            copied[i % 2].record(copy_stream)

    for ev in computed:
        ev.record(stream)
    e0.record(stream)
    upload(0)
    e2e_iters = 0
    for i in range(e2e_steps):
        if i + 1 < e2e_steps:
            upload(i + 1)
        stream.wait_event(copied[i % 2])
        out = ctx.step(bufs[i % 2])
        computed[i % 2].record(stream)
        e2e_iters += sum(out["iters"][q] for q in range(8) if ctx.assignment["owner"][q] >= 0)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(computed[i % 2])
            for k in outbufs[i]:
                outbufs[i][k].copy_(bufs[i % 2][k], non_blocking=True)
    stream.wait_stream(copy_stream)
    e1.record(stream)
    barrier()
    e_ms = e0.elapsed_time(e1)
    if dist is not None:
        tt = torch.tensor([e_ms, float(e2e_iters)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_ms = float(tt[0].item())
    e2e_value = e2e_iters / (e_ms / 1e3)

    extras = None
    if world == 1 and not args.no_extras:
        extras = measure_other_configs(mfx, torch)
    elif world > 1 and not args.no_extras:
        extras = {}
        try:   # (a) the paper's multi-GPU pressure solve: same owners, p' over [12..N]
            obj = [mfx.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            asg2 = assignment_multi_p(world)
            ctx2 = mfx.SimpleContext(asg2, g, pr, rank=rank, nranks=world, uid=obj[0])
            for k, v in host.items():
                sd[k].copy_(v, non_blocking=True)
            ctx2.step(sd)
            barrier()
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(stream)
            its2 = 0
            for _ in range(args.steps):
                o2 = ctx2.step(sd)
                its2 += sum(o2["iters"][q] for q in range(8) if ctx2.assignment["owner"][q] >= 0)
            m1.record(stream)
            barrier()
            tt = torch.tensor([m0.elapsed_time(m1)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms2 = float(tt.item())
            extras["multi_gpu_pressure"] = {"assignment": asg2, "simple_iters_per_s": args.steps / (ms2 / 1e3),
                                            "bicgstab_iters_per_s": its2 / (ms2 / 1e3),
                                            "pp_phase_ms_last": ctx2.phase_times()["pp"]}
            # (b) domain-decomposed comparator: the p' solve of this step over all N ranks
            #     (halo planes + all-gathered dots every iteration, P:87 / Fig. 2a)
            k0, k1 = mfx.dist_slab(g.nz, rank, world)
            plane = g.nx * g.ny
            ws2 = mfx.Workspace(g)
            star = [ctx2.buffer(k) for k in ("u*", "v*", "w*", "dx", "dy", "dz")]   # every rank holds them
            sysd, _ = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws2, star=star)
            sl = {k: v[k0 * plane:k1 * plane] for k, v in sysd.items()}
            xs = torch.zeros((k1 - k0) * plane, dtype=torch.float64, device="cuda")
            barrier()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            info = ctx2.dist_solve(mfx.EQ_PP, sl, xs, 0.0, 100)
            d1.record(stream)
            barrier()
            tt = torch.tensor([d0.elapsed_time(d1)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            extras["dd_comparator_pp"] = {"ranks": world, "iters": info["iters"],
                                          "us_per_iter": 1e3 * float(tt.item()) / max(info["iters"], 1),
                                          "single_rank_us_per_iter": 1e3 * phase["pp"] / max(outs[-1]["iters"][3], 1)}
            ctx2.close()
        except Exception as e:  # keep the main line
            extras["error"] = repr(e)[:300]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_measure()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
                "scaling": "weak" if world > 4 else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded fluidized-bed fields, synth/)",
                "config": bench_config(asg, (g.nx, g.ny, g.nz), n_scal),
                "simple_iters_per_s": simple_per_s,
                "bicgstab_iters_per_step": it_all / args.steps,
                "iters_last_step": outs[-1]["iters"],
                "phase_ms_last_step": phase,
                "exchange": {"gather_plus_bcast_ms_max_over_ranks": xch,
                             "share_of_step": xch / (t_ms / args.steps),
                             "packed_bcast": world > 1,
                             "note": "north star: state exchange < 10% of the step (4 GPUs)"},
                "kernel_avg_us": {k: (v * 1e3 if v else None) for k, v in kern_ms.items()},
                "pp_iteration": {"alg_bytes": pp_iter_bytes,
                                 "us": 1e3 * phase["pp"] / max(outs[-1]["iters"][3], 1),
                                 "alg_GBps": pp_iter_bytes / (1e-3 * phase["pp"] / max(outs[-1]["iters"][3], 1)) / 1e9},
                "instrumented_ms_per_step": t_prof_ms / args.steps,
                "roofline": roof,
                "kernels": kernels_roof,
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "steps": e2e_steps, "pipelining": "double-buffered: step i+1 inputs H2D and step i "
                                                           "results D2H overlap step i / i+1 compute"},
                "gpu_launches": launches,
                "clocks": clk,
                "other_configs": extras}
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mfx", choices=["mfx", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config 1/3/4 side measurements")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_mfx(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
