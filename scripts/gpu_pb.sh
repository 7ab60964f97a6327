timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sanitize.py -x -q -k "not pic and not bfs" > gpurun_out/pytest_pb.log 2>&1; tail -3 gpurun_out/pytest_pb.log
timeout 300 python scripts/prof_solve.py --kind pp --iters 200 --repeat 3 2>&1 | tail -3
timeout 300 python scripts/prof_solve.py --kind w --iters 200 --repeat 3 2>&1 | tail -3
timeout 300 python scripts/time_paths.py 2,3,4 2>&1 | grep tma
