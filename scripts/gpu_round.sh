# One validation pass on a B200: smoke, GPU tests, bench, reference arm, ncu launch list +
# full-set captures of the top kernels (exported to CSV on the box; reps are too big to copy back).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
if [ "${MFX_TESTS:-1}" = 1 ]; then
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -25 gpurun_out/${TAG}_pytest_gpu.log
fi
t0=$(date +%s); timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench wall seconds: $(( $(date +%s) - t0 ))"; tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1; cat gpurun_out/${TAG}_bench_ref.json
if [ "${MFX_NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
for cap in "pp:k_stencil|k3v:4:3:--kind pp --iters 4" "pp3:k_bicg_rw:0:1:--config 3 --kind pp --iters 50" "c1:k_bicg_cluster:0:1:--config 1 --kind pp --iters 200" "asm:k_asm|k_assemble|k_correct:0:3:--kind w --iters 2"; do
  IFS=: read name rx skip cnt args <<< "$cap"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt -o /tmp/${TAG}_prof_$name python scripts/prof_solve.py $args > /dev/null 2>&1
  ncu -i /tmp/${TAG}_prof_$name.ncu-rep --page raw --csv > gpurun_out/${TAG}_prof_${name}_raw.csv 2>&1
  ncu -i /tmp/${TAG}_prof_$name.ncu-rep --page source --csv > gpurun_out/${TAG}_prof_${name}_source.csv 2>&1
  rm -f /tmp/${TAG}_prof_$name.ncu-rep
done
fi
ls -la gpurun_out/
