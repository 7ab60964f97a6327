set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py smoke 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
python scripts/prof_solve.py --kind pp --iters 200 --repeat 3
python scripts/prof_solve.py --kind w --iters 200 --repeat 2
MFX_KERNELS=v1 python scripts/prof_solve.py --kind pp --iters 200 --repeat 2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_pp.csv python scripts/prof_solve.py --kind pp --iters 15 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 6 -c 3 -o gpurun_out/prof_stencil python scripts/prof_solve.py --kind pp --iters 6 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
