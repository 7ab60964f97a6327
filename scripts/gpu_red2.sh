# after a reduction change: parity (all solver paths) + p' iteration times c2/c3 + short bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist_solver.py -m gpu -x -q -k "not long_horizon" 2>&1 | tail -2
for rep in 1 2; do
  for cfg in 2 3; do echo -n "c$cfg auto: "; timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo; done
  echo -n "c3 path 1: "; timeout 300 python scripts/prof_solve.py --config 3 --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed" | tail -1
done
MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config 3 --kind pp --iters 40 --repeat 2 --path 5 2>&1 | grep -A3 "persist trace" | head -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_red.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_red.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernel_avg_us'], d['pp_iteration'], d['clocks'])"
