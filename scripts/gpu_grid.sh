set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bicgstab or simple" > gpurun_out/pytest_grid.log 2>&1; tail -15 gpurun_out/pytest_grid.log
timeout 600 python scripts/time_paths.py 3,2 > gpurun_out/paths.json 2>&1; cat gpurun_out/paths.json
