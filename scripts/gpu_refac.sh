timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_refac.log 2>&1; tail -4 gpurun_out/pytest_refac.log
timeout 300 python scripts/prof_solve.py --kind pp --iters 200 --repeat 3 2>&1 | tail -2
