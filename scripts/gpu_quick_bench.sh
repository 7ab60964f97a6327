# Quick check after a kernel change: solver/SIMPLE parity subset, p' and w iteration timings, short bench.
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "bicgstab or simple or spmv or c2 or c4" 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python scripts/prof_solve.py --kind pp --iters 200 2>&1 | tail -2; done
timeout 300 python scripts/prof_solve.py --kind w --iters 20 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_k2.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_k2.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernel_avg_us'], d['pp_iteration'], d['clocks'])"
