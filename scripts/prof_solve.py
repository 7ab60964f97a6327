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
args = ap.parse_args()

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
for r in range(args.repeat):
    x = torch.zeros(g.n, dtype=torch.float64, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    info = mfx.bicgstab_solve(kind, g, sysd, x, 0.0, args.iters, ws)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(f"{args.kind} iters={info['iters']} ms={ms:.3f} us/iter={1e3 * ms / max(info['iters'], 1):.1f}")
