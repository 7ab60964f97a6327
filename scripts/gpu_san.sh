timeout 1500 python -m pytest tests/test_gpu_sanitize.py -q -x > gpurun_out/pytest_san.log 2>&1; tail -20 gpurun_out/pytest_san.log
