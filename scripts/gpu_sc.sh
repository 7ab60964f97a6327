timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_blocked.py tests/test_gpu_upwind.py tests/test_gpu_multirank.py -x -q -k "scalar or bfs or upwind or simple or multirank" > gpurun_out/pytest_sc.log 2>&1; tail -3 gpurun_out/pytest_sc.log
timeout 300 python scripts/time_asm.py
