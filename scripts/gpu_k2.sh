set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_k2.log 2>&1; tail -5 gpurun_out/pytest_k2.log
timeout 300 python scripts/time_paths.py 2,3,4 2>&1 | grep tma
timeout 300 python scripts/prof_solve.py --kind pp --iters 200 --repeat 3
