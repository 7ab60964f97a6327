timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spmv or pp_ragged or c1_parity" 2>&1 | tail -2
for cfg in "MFX_TILE=1" "MFX_TILE=2" "MFX_TILE=5" "MFX_TILE=5 MFX_STAGES=4" "MFX_TILE=2 MFX_LZ=16" "MFX_TILE=5 MFX_LZ=16"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 100 --repeat 3 | tail -1
done
for cfg in "MFX_TILE=1" "MFX_TILE=5"; do
  echo "== w $cfg"; env $cfg python scripts/prof_solve.py --kind w --iters 100 --repeat 3 | tail -1
done
