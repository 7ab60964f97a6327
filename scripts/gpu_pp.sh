timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_blocked.py tests/test_gpu_upwind.py -x -q -k "pp or blocked or bfs or upwind or simple" > gpurun_out/pytest_pp.log 2>&1; tail -3 gpurun_out/pytest_pp.log
timeout 300 python scripts/time_asm.py
