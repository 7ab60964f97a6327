mkdir -p gpurun_out
TAG=${TAG:-r02e}
for cfg in 2 3 1; do for v in "0 1" "8 1" "0 5" "15 5"; do
  set -- $v
  echo "c$cfg MFX_RW=$1 path $2"
  MFX_RW=$1 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path $2 2>&1 | tail -3
done; done 2>&1 | tee gpurun_out/${TAG}_red.log
MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config 3 --kind pp --iters 200 --repeat 2 --path 5 2>&1 | grep trace | tee -a gpurun_out/${TAG}_red.log
MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 2 --path 5 2>&1 | grep trace | tee -a gpurun_out/${TAG}_red.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -22 | tee gpurun_out/${TAG}_pytest_gpu.log
