timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "" "MFX_STAGES=3" "MFX_STAGES=6" "MFX_TILE=32" "MFX_TILE=32 MFX_STAGES=6" "MFX_LZ=32" "MFX_LZ=8"; do
  echo "== $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 100 --repeat 3 | tail -2
done
for cfg in "" "MFX_STAGES=4" "MFX_TILE=32"; do
  echo "== w $cfg"; env $cfg python scripts/prof_solve.py --kind w --iters 100 --repeat 3 | tail -2
done
