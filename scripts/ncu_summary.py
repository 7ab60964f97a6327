"""Summarise ncu captures into profiles/: a compact per-launch CSV of the bench
command, per-kernel shares and DRAM traffic, key metrics of the full-set
reports, and profiles/ncu_traffic.json (DRAM bytes per launch per kernel class,
read by bench.py for roofline.traffic)."""
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def classify(name):
    m = re.search(r"k_stencil_rw<(\d)", name)
    if m:
        return {0: "spmv", 1: "setup", 2: "K1", 3: "K2"}[int(m.group(1))] + "_pp"
    if "k_bicg_rw" in name:
        return "persist_pp"
    m = re.search(r"k_stencil<(\d), (\d)", name)
    if m:
        mode, sym = int(m.group(1)), int(m.group(2))
        return {0: "spmv", 1: "setup", 2: "K1", 3: "K2"}[mode] + ("_pp" if sym else "_mom")
    for k in ("k3v", "k_asm_mom_tma", "k_assemble_mom", "k_assemble_pp", "k_assemble_scalar", "k_correct",
              "k_zero_if", "k_meta", "k_bicg_cluster", "k_pic_eps_final", "k_pic_eps", "k_pic_drag"):
        if k in name:
            return {"k3v": "K3"}.get(k, k)
    return "other:" + name.split("(")[0][-40:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        d[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki]
    return [(i, names[i], d[i]) for i in sorted(d)]


L = launches(os.path.join(GO, f"{tag}_launches_bench.csv"))
with open(os.path.join(PR, f"{tag}_launches_bench.csv"), "w") as f:
    f.write("id,kernel,class,gpu_time_ns,dram_read_bytes,dram_write_bytes\n")
    for i, n, m in L:
        f.write(f"{i},\"{n.split('(')[0][:80]}\",{classify(n)},{m.get('gpu__time_duration.sum', 0):.0f},"
                f"{m.get('dram__bytes_read.sum', 0):.0f},{m.get('dram__bytes_write.sum', 0):.0f}\n")
agg = defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for i, n, m in L:
    c = classify(n)
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[c]
    a[0] += 1
    a[1] += t
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot += t
traffic = {c: a[2] / a[0] for c, a in agg.items() if a[0]}
json.dump({"source": f"profiles/{tag}_launches_bench.csv (ncu, cache-control all, serialized)",
           "dram_bytes_per_launch": traffic}, open(os.path.join(PR, "ncu_traffic.json"), "w"), indent=1)

lines = [f"# ncu summary ({tag})", "",
         "## Launch list of `python bench.py --steps 1 --warmup 0` (ncu, gpu__time_duration + DRAM bytes)", "",
         "Serialized, cold-cache per-launch times: compare SHARES with bench.py's live CUDA-event timing.", "",
         "| class | launches | total ms | share | avg µs | DRAM MB / launch | DRAM GB/s |", "|---|---|---|---|---|---|---|"]
for c, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| {c} | {a[0]} | {a[1] / 1e6:.2f} | {a[1] / tot:.3f} | {a[1] / a[0] / 1e3:.1f} | "
                 f"{a[2] / a[0] / 1e6:.1f} | {a[2] / a[1]:.0f} |")

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
def raw_pages():
    # the box exports `ncu -i rep --page raw --csv` (reps exceed gpurun's copy-back limit); older tags have reps
    for x in sorted(os.listdir(GO)):
        if x.startswith(f"{tag}_prof") and x.endswith("_raw.csv"):
            yield x, open(os.path.join(GO, x)).read()
        elif x.startswith(f"{tag}_prof") and x.endswith(".ncu-rep"):
            yield x, subprocess.run(["ncu", "-i", os.path.join(GO, x), "--page", "raw", "--csv"],
                                    capture_output=True, text=True).stdout


for rep, out in raw_pages():
    lines_ = out.splitlines()
    k0 = next((i for i, l in enumerate(lines_) if "Kernel Name" in l), 0)
    rows = list(csv.reader(lines_[k0:]))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    lines += ["", f"## {rep} (ncu --set full)", ""]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        lines.append(f"### {classify(name)} — `{name.split('(')[0][:90]}`")
        for w in want:
            if w in h:
                lines.append(f"- {w} = {r[h.index(w)]} {units[h.index(w)]}")
        st = []
        for i, c in enumerate(h):
            if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        lines.append("- top stall samples: " + ", ".join(f"{c} {v:.0f}" for v, c in st[:6]))
open(os.path.join(PR, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:20]))
