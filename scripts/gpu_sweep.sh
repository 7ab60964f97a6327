for cfg in "MFX_PDL=1" "MFX_PDL=0" "MFX_PDL=1" "MFX_PDL=0" "MFX_PDL=1 MFX_GRAPH=0" "MFX_PDL=0 MFX_GRAPH=0"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 400 --repeat 5 2>&1 | grep -E "timed|kernels"
done
for cfg in "MFX_PDL=1" "MFX_PDL=0"; do
  echo "== bench $cfg"; env $cfg timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pp_iteration'], d['clocks'])"
done
