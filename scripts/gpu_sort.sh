timeout 900 python -m pytest tests/test_gpu_pic.py -x -q > gpurun_out/pytest_sort.log 2>&1; tail -3 gpurun_out/pytest_sort.log
timeout 600 python -c "
import json, torch, bench, paper_2211_15605_b200 as mfx
print(json.dumps(bench.measure_pic(mfx, torch)))
"
