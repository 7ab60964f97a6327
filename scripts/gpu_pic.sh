timeout 1200 python -m pytest tests/test_gpu_pic.py tests/test_gpu_sanitize.py -x -q -k "pic or binned or sort" > gpurun_out/pytest_pic4.log 2>&1; tail -3 gpurun_out/pytest_pic4.log
timeout 600 python -c "
import json, torch, bench, paper_2211_15605_b200 as mfx
print(json.dumps(bench.measure_pic(mfx, torch)))
"
