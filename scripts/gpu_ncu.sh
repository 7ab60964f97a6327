# launch list of the bench command (single metric pass, serialized, cold cache)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
# full sets: K1 p', K2 p', K3 (launches 1,2,3 after setup in a p' solve)
ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k3v" -s 4 -c 3 -o gpurun_out/r01_prof_pp python scripts/prof_solve.py --kind pp --iters 4 > gpurun_out/ncu_pp.log 2>&1; tail -1 gpurun_out/ncu_pp.log
ncu --set full --clock-control none --import-source on -k regex:"k_assemble" -c 2 -o gpurun_out/r01_prof_asm python scripts/prof_solve.py --kind w --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_bicg_cluster" -c 1 -o gpurun_out/r01_prof_cluster python scripts/prof_solve.py --config 1 --kind pp --iters 200 > /dev/null 2>&1
ls -la gpurun_out/
