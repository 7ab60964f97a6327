# PIC coupling check on a B200: GPU parity tests + timing side measurement.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic.py -x -q > gpurun_out/pytest_pic.log 2>&1; tail -30 gpurun_out/pytest_pic.log
timeout 600 python -c "
import json, torch, bench, paper_2211_15605_b200 as mfx
print(json.dumps(bench.measure_pic(mfx, torch)))
" > gpurun_out/pic_time.json 2>&1; cat gpurun_out/pic_time.json
