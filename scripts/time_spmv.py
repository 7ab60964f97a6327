"""Standalone timing of the 7-point apply (TMA kernel, SPMV mode) at c2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2211_15605_b200 as mfx
g, pr, st = synth.config_case(2)
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ws = mfx.Workspace(g)
rng = np.random.default_rng(0)
dv = [torch.from_numpy(rng.uniform(1e-4, 1e-3, g.n)).cuda() for _ in range(3)]
for kind, name, bpc in ((mfx.EQ_PP, "pp", 40), (mfx.EQ_W, "w", 72)):
    if kind == mfx.EQ_PP:
        sysd, _ = mfx.assemble_eq(kind, g, pr, sd, ws, star=[sd["u"], sd["v"], sd["w"]] + dv)
    else:
        sysd, _ = mfx.assemble_eq(kind, g, pr, sd, ws)
    x = sd["w"].clone(); y = torch.empty_like(x)
    for _ in range(3): mfx.spmv(kind, g, sysd, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): mfx.spmv(kind, g, sysd, x, y)
    e1.record(); torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / 50
    print(f"spmv {name}: {us:.1f} us  {bpc * g.n / (us * 1e-6) / 1e9:.0f} GB/s algorithmic ({bpc} B/cell)")
