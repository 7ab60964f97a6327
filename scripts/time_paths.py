"""Per-iteration time of the p' / momentum BiCGSTAB on every solver path and
grid (tol 0, k1 and k2 iterations: (T(k2) - T(k1)) / (k2 - k1))."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2211_15605_b200 as mfx  # noqa: E402

out = []
for cid in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3,2").split(",")]:
    g, pr, st = synth.config_case(cid)
    sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
    ws = mfx.Workspace(g)
    rng = np.random.default_rng(0)
    dv = [torch.from_numpy(rng.uniform(1e-4, 1e-3, g.n)).cuda() for _ in range(3)]
    systems = {"pp": (mfx.EQ_PP, mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=[sd["u"], sd["v"], sd["w"]] + dv)[0]),
               "w": (mfx.EQ_W, mfx.assemble_eq(mfx.EQ_W, g, pr, sd, ws)[0])}
    for name, (kind, sysd) in systems.items():
        for path, pname in ((mfx.PATH_TMA, "tma"), (mfx.PATH_GRID, "grid")):
            mfx.set_option("solver_path", path)
            x = torch.zeros(g.n, dtype=torch.float64, device="cuda")

            def t(k):
                ts = []
                for _ in range(5):
                    x.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    info = mfx.bicgstab_solve(kind, g, sysd, x, 0.0, k, ws)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                return statistics.median(ts), info["iters"]
            k1, k2 = 10, 110
            t(k1)
            (a, i1), (b, i2) = t(k1), t(k2)
            us = 1e3 * (b - a) / (i2 - i1)
            bpc = 184 if name == "pp" else 248
            out.append({"config": cid, "system": name, "path": pname, "us_per_iter": us,
                        "alg_GBps": bpc * g.n / (us * 1e-6) / 1e9, "iters": [i1, i2]})
            print(json.dumps(out[-1]), flush=True)
    mfx.set_option("solver_path", 0)
    del sd, systems, ws
    torch.cuda.empty_cache()
