for rep in 1 2; do for so in variants/libmfx_head.so variants/libmfx_new.so; do
  echo -n "$so c1: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config 1 --kind pp --iters 400 --repeat 3 --path 2 2>&1 | grep timed | tail -1
done; done
MFX_CLUSTER_TRACE=1 timeout 300 python scripts/prof_solve.py --config 1 --kind pp --iters 50 --repeat 1 --path 2 2>&1 | grep -A4 "cluster trace"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster" 2>&1 | tail -2
