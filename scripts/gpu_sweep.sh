timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster" 2>&1 | tail -2
MFX_CLUSTER_TRACE=1 python scripts/prof_solve.py --config 1 --kind pp --iters 30 --repeat 2 --path 2 2>&1 | tail -6
python scripts/prof_solve.py --config 1 --kind pp --iters 500 --repeat 3 --path 2 2>&1 | tail -3
