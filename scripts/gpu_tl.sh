set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_timeloop.py tests/test_gpu_parity.py -x -q -k "time or assemble" > gpurun_out/pytest_tl.log 2>&1; tail -30 gpurun_out/pytest_tl.log
