timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sanitize.py tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_er.log 2>&1; tail -3 gpurun_out/pytest_er.log
timeout 300 python scripts/prof_solve.py --kind w --iters 200 --repeat 3 2>&1 | tail -3
timeout 300 python scripts/prof_solve.py --kind pp --iters 200 --repeat 3 2>&1 | tail -3
timeout 300 python scripts/time_paths.py 2,3 2>&1 | grep tma
