mkdir -p gpurun_out
TAG=${TAG:-r02d}
for v in "0 2 4" "8 2 4" "8 1 0" "12 1 0"; do
  set -- $v
  echo "c2 MFX_RW=$1 MFX_RW_MB=$2 MFX_RW_STAGES=$3"
  MFX_RW=$1 MFX_RW_MB=$2 MFX_RW_STAGES=$3 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 3 2>&1 | tail -3
done 2>&1 | tee gpurun_out/${TAG}_k2_variants.log
for cfg in 3 2 1; do
  echo "config $cfg path 5 trace"
  MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 2 --path 5 2>&1 | tail -4
done 2>&1 | tee gpurun_out/${TAG}_persist_trace.log
MFX_RW=8 MFX_RW_MB=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pp and (tma or persist)" 2>&1 | tail -2
