# One validation pass on a B200: smoke, GPU tests, bench, ncu launch list + full sets.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
t0=$(date +%s); timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench wall seconds: $(( $(date +%s) - t0 ))"; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
if [ "${MFX_NCU:-1}" = 1 ]; then
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k3v" -s 4 -c 3 -o gpurun_out/${TAG}_prof_pp python scripts/prof_solve.py --kind pp --iters 4 > gpurun_out/ncu_pp.log 2>&1; tail -1 gpurun_out/ncu_pp.log
ncu --set full --clock-control none --import-source on -k regex:"k_asm|k_assemble|k_correct" -c 3 -o gpurun_out/${TAG}_prof_asm python scripts/prof_solve.py --kind w --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pic" -c 2 -o gpurun_out/${TAG}_prof_pic python -c "import torch, bench, paper_2211_15605_b200 as m; bench.measure_pic(m, torch)" > /dev/null 2>&1
fi
ls -la gpurun_out/
