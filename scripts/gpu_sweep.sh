MFX_CLUSTER_TRACE=1 python scripts/prof_solve.py --config 1 --kind pp --iters 30 --repeat 2 --path 2 2>&1 | tail -14
