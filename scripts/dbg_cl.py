import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth, oracle as orc, paper_2211_15605_b200 as mfx
from synth import Params
pr = Params()
for (nx, ny, nz) in ((16, 16, 16), (16, 16, 32), (16, 16, 64), (8, 8, 48), (16, 16, 20)):
    g = synth.make_grid(nx, ny, nz)
    st = synth.make_state(g, 1000 + nx * 7 + nz, pr, n_scalars=1)
    dv = [np.full(g.n, 5e-4)] * 3
    sysd, _, _ = orc.assemble_pp(g, pr, st, [st["u"], st["v"], st["w"]], dv); x0 = np.zeros(g.n); k = mfx.EQ_PP
    for cl in (16, 8):
        mfx.set_option("cluster_size", cl); mfx.set_option("solver_path", mfx.PATH_CLUSTER)
        res = []
        for maxit in (1, 2, 3):
            ref = orc.bicgstab(g, sysd, x0, 1e-30, maxit)
            ws = mfx.Workspace(g)
            x = torch.from_numpy(x0.copy()).cuda()
            info = mfx.bicgstab_solve(k, g, {kk: torch.from_numpy(v).cuda() for kk, v in sysd.items()}, x, 1e-30, maxit, ws)
            res.append(int(np.sum(x.cpu().numpy() != ref["x"])))
        print((nx, ny, nz), "CL", cl, "planes/CTA", -(-nz // cl), "nbad for maxit 1,2,3:", res, flush=True)
