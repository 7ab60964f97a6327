set -x
mkdir -p gpurun_out
MFX_REPORT_DIR=gpurun_out timeout 1200 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_dump.py -x -q > gpurun_out/pytest_next.log 2>&1; tail -30 gpurun_out/pytest_next.log
timeout 600 python -c "
import json, torch, bench, paper_2211_15605_b200 as mfx
print(json.dumps(bench.measure_bfs(mfx, torch)))
" > gpurun_out/bfs.json 2>&1; cat gpurun_out/bfs.json
