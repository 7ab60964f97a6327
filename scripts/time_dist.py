"""Per-iteration time of the z-slab solver (mfx_dist_solve) with one rank
against the single-GPU BiCGSTAB (mfx_bicgstab_solve) on the same c2 p' system
(within 10%), fixed iteration count (tol 0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_2211_15605_b200 as mfx

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g, pr, st = synth.config_case(cfg)
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ws = mfx.Workspace(g)
rng = np.random.default_rng(0)
dv = [torch.from_numpy(rng.uniform(1e-4, 1e-3, g.n)).cuda() for _ in range(3)]
sysd, _ = mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=[sd["u"], sd["v"], sd["w"]] + dv)
torch.cuda.synchronize()


def timed(fn, n=2):
    out = []
    for _ in range(n + 1):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        info = fn()
        ev1.record()
        torch.cuda.synchronize()
        out.append((ev0.elapsed_time(ev1), info))
    return out[1:]


x1 = torch.zeros(g.n, dtype=torch.float64, device="cuda")
def single():
    x1.zero_()
    return mfx.bicgstab_solve(mfx.EQ_PP, g, sysd, x1, 0.0, iters, ws)

ctx = mfx.SimpleContext("111[1]", g, pr)
x2 = torch.zeros(g.n, dtype=torch.float64, device="cuda")
sl = {k: v for k, v in sysd.items() if v is not None}
def dist():
    x2.zero_()
    return ctx.dist_solve(mfx.EQ_PP, sl, x2, 0.0, iters, stream=torch.cuda.current_stream())

for name, fn in (("bicgstab_solve", single), ("dist_solve R=1", dist)):
    for ms, info in timed(fn):
        print(f"c{cfg} {name}: iters {info['iters']} {1e3 * ms / max(info['iters'], 1):.1f} us/iter", flush=True)
print("bitwise equal:", bool(torch.equal(x1, x2)))
ctx.close()
