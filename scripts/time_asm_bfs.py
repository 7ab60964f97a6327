"""Device time of the three momentum assemblies on the paper's 10M-cell
backward-facing step (BLOCKED cells): TMA z-marching vs
grid-stride kernel (CUDA events, median of 9)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2211_15605_b200 as mfx  # noqa: E402

g, pr, st = synth.bfs_case(126, 63, 1260, seed=11)
sd = {k: torch.from_numpy(v).cuda() for k, v in st.items()}
ws = mfx.Workspace(g)
for path in (1, 0, 1, 0):
    mfx.set_option("asm_tma", path)
    ts = []
    for _ in range(9):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for comp in range(3):
            mfx.assemble_eq(comp, g, pr, sd, ws)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"BFS {g.nx}x{g.ny}x{g.nz} momentum assembly x3 ({'tma' if path else 'grid-stride'}): "
          f"{1e3 * statistics.median(ts):.0f} us", flush=True)
