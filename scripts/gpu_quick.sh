timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_solver.py -m gpu -x -q -k "pp or simple_iter_111 or dist or edge or deterministic or not_converged" 2>&1 | tail -2
for cfg in 3 2; do
MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 2 --path 5 2>&1 | grep "persist trace" | head -1
for path in 1 5; do echo "c$cfg path $path"; timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path $path 2>&1 | tail -3; done
done
MFX_RW_TRACE=1 MFX_GRAPH=0 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 20 --repeat 1 2>&1 | grep "rw trace" | tail -2
