# cluster push reductions: single-cluster solver (c1) and persistent solver (c3) -- parity + timing
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_blocked.py -m gpu -x -q -k "cluster or persist" 2>&1 | tail -3
for rep in 1 2; do for cl in 16 8; do
  echo -n "MFX_CLUSTER=$cl c1: "; MFX_CLUSTER=$cl timeout 300 python scripts/prof_solve.py --config 1 --kind pp --iters 400 --repeat 3 --path 2 2>&1 | grep timed | tail -1
done; done
MFX_CLUSTER_TRACE=1 timeout 300 python scripts/prof_solve.py --config 1 --kind pp --iters 50 --repeat 1 --path 2 2>&1 | grep -A5 "cluster trace"
for rep in 1 2; do for cl in 1 8 16; do
  echo -n "MFX_PERSIST_CL=$cl c3: "; MFX_PERSIST_CL=$cl timeout 300 python scripts/prof_solve.py --config 3 --kind pp --iters 200 --repeat 3 --path 5 2>&1 | grep timed | tail -1
done; done
for cl in 1 8; do
  echo -n "MFX_PERSIST_CL=$cl c2: "; MFX_PERSIST_CL=$cl timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 3 --path 5 2>&1 | grep timed | tail -1
done
echo -n "c2 path 1: "; timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep timed | tail -1
