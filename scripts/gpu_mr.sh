timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_blocked.py tests/test_gpu_upwind.py tests/test_gpu_fullsize.py tests/test_gpu_timeloop.py -x -q > gpurun_out/pytest_mr.log 2>&1; tail -3 gpurun_out/pytest_mr.log
timeout 300 python scripts/time_asm.py
MFX_ASM_TMA=0 timeout 300 python scripts/time_asm.py
