timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_solver.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not long_horizon" 2>&1 | tail -2
for rep in 1 2; do for dyn in 0 1; do
  for cfg in 2 3; do echo -n "MFX_DYN=$dyn c$cfg path 1: "; MFX_DYN=$dyn timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo; done
  echo -n "MFX_DYN=$dyn c2 w: "; MFX_DYN=$dyn timeout 300 python scripts/prof_solve.py --config 2 --kind w --iters 20 --repeat 3 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo
done; done
MFX_RW_TRACE=1 MFX_GRAPH=0 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 20 --repeat 1 2>&1 | grep "rw trace" | tail -2
