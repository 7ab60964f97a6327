ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_active.avg --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/prof_solve.py --config 3 --kind pp --iters 20 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_stencil|k3v" -s 10 -c 3 -o gpurun_out/c3_full python scripts/prof_solve.py --config 3 --kind pp --iters 8 > /dev/null 2>&1
ls -la gpurun_out
