timeout 900 python -m pytest tests/test_gpu_dist_solver.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
for cfg in 2 3; do timeout 300 python scripts/time_dist.py $cfg 200; done 2>&1 | tee gpurun_out/r02o_time_dist.log
