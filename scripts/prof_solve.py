"""Small driver for ncu: assemble the c2 (128x128x512) p' (or w-momentum) system
on the GPU and run a fixed number of BiCGSTAB iterations (tol 0)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_2211_15605_b200 as mfx

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="pp", choices=["pp", "w"])
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--path", type=int, default=0, help="solver_path option: 0 auto, 1 tma, 2 cluster, 3 v1")
ap.add_argument("--tol", type=float, default=0.0)
args = ap.parse_args()

mfx.set_option("solver_path", args.path)
g, pr, st = synth.config_case(args.config)
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ws = mfx.Workspace(g)
if args.kind == "pp":
    rng = np.random.default_rng(0)
    dv = [torch.from_numpy(rng.uniform(1e-4, 1e-3, g.n)).cuda() for _ in range(3)]
    sysd, _ = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=[sd["u"], sd["v"], sd["w"]] + dv)
    kind = mfx.EQ_PP
else:
    sysd, _ = mfx.assemble_eq(mfx.EQ_W, g, pr, sd, ws)
    kind = mfx.EQ_W
torch.cuda.synchronize()
N = g.n
BPC = {"K1_pp": 72, "K2_pp": 48, "K3": 64, "K1_mom": 104, "K2_mom": 80, "spmv_setup": None}
for r in range(args.repeat):
    if r == args.repeat - 1:
        mfx.prof_reset()
        mfx.prof_enable(True)
    x = torch.zeros(g.n, dtype=torch.float64, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    info = mfx.bicgstab_solve(kind, g, sysd, x, args.tol, args.iters, ws)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    tag = "instrumented(no graphs)" if r == args.repeat - 1 else ("first(capture)" if r == 0 else "timed")
    print(f"{args.kind} [{tag}] iters={info['iters']} ms={ms:.3f} us/iter={1e3 * ms / max(info['iters'], 1):.1f}",
          flush=True)
mfx.prof_enable(False)
pr_ = mfx.prof_read()
line = []
for k, v in pr_.items():
    if v["launches"]:
        us = 1e3 * v["ms"] / v["launches"]
        bw = f" {BPC[k] * N / (us * 1e-6) / 1e9:.0f}GB/s" if BPC.get(k) else ""
        line.append(f"{k}:{us:.1f}us{bw}")
print("   kernels: " + "  ".join(line), flush=True)
