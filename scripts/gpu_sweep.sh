timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
for cfg in "" "MFX_STAGES=4" "MFX_TILE=2"; do echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 200 --repeat 3 2>&1 | tail -2; done
echo "== w"; python scripts/prof_solve.py --kind w --iters 200 --repeat 3 2>&1 | tail -2
