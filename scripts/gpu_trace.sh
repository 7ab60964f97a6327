mkdir -p gpurun_out
for cfg in 3 2; do
MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 2 --path 5 2>&1 | grep -A5 "persist trace"
done 2>&1 | tee gpurun_out/${TAG}_trace.log
