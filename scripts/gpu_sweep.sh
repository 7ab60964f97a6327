timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "" "MFX_TILE=1"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 100 --repeat 3 | tail -2
done
echo "== w"; python scripts/prof_solve.py --kind w --iters 100 --repeat 3 | tail -2
