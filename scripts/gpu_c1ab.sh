# c1 single-cluster solver: parity of the variant + A/B against the default build
MFX_SO_VARIANT=abv/libmfx_waitcta.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster" 2>&1 | tail -1
for rep in 1 2 3; do for so in "" abv/libmfx_waitcta.so; do for cl in 16; do
  echo -n "so=${so:-default} MFX_CLUSTER=$cl c1: "; MFX_SO_VARIANT=$so MFX_CLUSTER=$cl timeout 300 python scripts/prof_solve.py --config 1 --kind pp --iters 400 --repeat 3 --path 2 2>&1 | grep timed | tail -1
done; done; done
