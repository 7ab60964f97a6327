"""Small end-to-end runs for compute-sanitizer.
  <path 1|2|4>: one SIMPLE iteration on a ragged grid with that solver path
                (TMA momentum assembly, p'/scalar assembly, TMA stencils, K3 /
                single-cluster solver / grid-synchronous solver, correction);
  pic:          eps + drag deposits and one SIMPLE iteration with implicit
                particle coupling (PIC kernels, exchange phase 3 path);
  bfs:          one SIMPLE iteration with BLOCKED cells (step geometry);
  odd:          one SIMPLE iteration on an odd-nx grid (grid-stride kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2211_15605_b200 as mfx

mode = sys.argv[1] if len(sys.argv) > 1 else "1"
mfx.set_option("graphs", 0)
pr = synth.Params(lin_maxit_pp=40, lin_maxit_mom=6, lin_maxit_phi=6)
if mode == "bfs":
    g, _, st = synth.bfs_case(12, 6, 20, seed=4)
    asg = "111[1]"
elif mode == "pic":
    g = synth.make_grid(34, 11, 13)
    st = synth.make_state(g, 99, pr)
    asg = "111[1]"
else:
    mfx.set_option("solver_path", 1 if mode == "odd" else int(mode))
    g = synth.make_grid(33 if mode == "odd" else 34, 11, 13)
    st = synth.make_state(g, 99, pr, n_scalars=1)
    asg = "111[1]1"
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ctx = mfx.SimpleContext(asg, g, pr)
if mode == "pic":
    pic = synth.PicParams()
    pc = {k: torch.from_numpy(v).cuda() for k, v in synth.make_parcels(g, 7, 3000, st["eps"], pic).items()}
    ws = mfx.Workspace(g)
    mfx.pic_deposit_eps(g, pic, pc, ws, eps=torch.empty_like(sd["eps"]))
    ws.check()
    ctx.set_pic(pc, pic, mfx.PIC_IMPLICIT)
out = ctx.step(sd)
torch.cuda.synchronize()
print("mode", mode, "iters", out["iters"][:5], "R", out["R"])
ctx.close()
