ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k3v" -s 4 -c 3 -o gpurun_out/r01b_prof_pp python scripts/prof_solve.py --kind pp --iters 4 > gpurun_out/ncu_pp.log 2>&1; tail -1 gpurun_out/ncu_pp.log
ls -la gpurun_out/
