timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "MFX_PDL=1" "MFX_PDL=0"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 400 --repeat 3 | tail -2
  echo "== pp graphs-only timing $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 400 --repeat 2 | head -1
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
