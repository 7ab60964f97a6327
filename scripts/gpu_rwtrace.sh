MFX_RW=12 MFX_RW_TRACE=1 MFX_GRAPH=0 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 20 --repeat 1 2>&1 | grep "rw trace" | tail -4
for cfg in 2 3; do for v in "8 1" "12 1" "8 5"; do set -- $v; echo "c$cfg MFX_RW=$1 path $2"
MFX_RW=$1 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path $2 2>&1 | tail -3
done; done
MFX_RW=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_solver.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not long_horizon" 2>&1 | tail -2
