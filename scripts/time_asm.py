"""Device time of the assembly / correction kernels at configuration 2 (CUDA
events, median of 9) -- used to tune their launch configuration."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2211_15605_b200 as mfx  # noqa: E402


def med(fn, reps=9):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return 1e3 * statistics.median(ts)


g, pr, st = synth.config_case(2, n_scalars=1)
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ws = mfx.Workspace(g)
out = {}
sysm = mfx.new_system(mfx.EQ_U, g.n)
for kind, name in ((mfx.EQ_U, "u"), (mfx.EQ_V, "v"), (mfx.EQ_W, "w")):
    out[f"assemble_{name}_us"] = med(lambda: mfx.assemble_eq(kind, g, pr, sd, ws, out=sysm))
star = [sd["u"], sd["v"], sd["w"], sysm["d"], sysm["d"], sysm["d"]]
sysp = mfx.new_system(mfx.EQ_PP, g.n)
out["assemble_pp_us"] = med(lambda: mfx.assemble_eq(mfx.EQ_PP, g, pr, sd, ws, star=star, out=sysp))
out["assemble_scalar_us"] = med(lambda: mfx.assemble_eq(mfx.EQ_SCALAR, g, pr, sd, ws, out=sysm, scalar_id=0))
outs = [torch.empty_like(sd["u"]) for _ in range(4)]
out["correct_us"] = med(lambda: mfx.correct(g, pr, star, sd["p"], sd["p"], out=outs))
for k in list(out):
    bpc = {"assemble_pp_us": 104, "correct_us": 96, "assemble_scalar_us": 120}.get(k, 144)
    out[k.replace("_us", "_GBps")] = bpc * g.n / (out[k] * 1e-6) / 1e9
print(json.dumps(out))
