"""Small end-to-end run for compute-sanitizer: one SIMPLE iteration per solver
path on a ragged grid (assembly, TMA stencils, K3, cluster solver, correction)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2211_15605_b200 as mfx

path = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mfx.set_option("solver_path", path)
mfx.set_option("graphs", 0)
g = synth.make_grid(34, 11, 13)
pr = synth.Params(lin_maxit_pp=40, lin_maxit_mom=6, lin_maxit_phi=6)
st = synth.make_state(g, 99, pr, n_scalars=1)
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ctx = mfx.SimpleContext("111[1]1", g, pr)
out = ctx.step(sd)
torch.cuda.synchronize()
print("path", path, "iters", out["iters"][:5], "R", out["R"])
ctx.close()
