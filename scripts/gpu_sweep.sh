timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "" "MFX_GRAPH=0"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 200 --repeat 3 | tail -2
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
