timeout 900 python -m pytest tests/test_gpu_upwind.py tests/test_gpu_parity.py tests/test_gpu_blocked.py -x -q > gpurun_out/pytest_up.log 2>&1; tail -15 gpurun_out/pytest_up.log
