timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "" "MFX_TILE=1" "MFX_TILE=2" "MFX_TILE=2 MFX_STAGES=4" "MFX_TILE=4"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 100 --repeat 3 | tail -2
done
for cfg in "" "MFX_TILE=1" "MFX_TILE=2"; do
  echo "== w $cfg"; env $cfg python scripts/prof_solve.py --kind w --iters 100 --repeat 3 | tail -2
done
