# K2/K1 p' variants (row-warp, 3 CTAs/SM), dist solver with graphs, ncu CSV exports (reps deleted on the box).
mkdir -p gpurun_out
TAG=${TAG:-r02c}
MFX_RW=15 MFX_RW_MB=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_solver.py -m gpu -x -q -k "pp or spmv or dist or simple_iter_111" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dist_solver.py -m gpu -x -q 2>&1 | tail -2
for v in "0 2 4" "8 2 4" "8 3 3" "8 3 2" "12 3 0" "4 3 2" "15 3 0"; do
  set -- $v
  echo "c2 MFX_RW=$1 MFX_RW_MB=$2 MFX_RW_STAGES=$3"
  MFX_RW=$1 MFX_RW_MB=$2 MFX_RW_STAGES=$3 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 3 2>&1 | tail -3
done 2>&1 | tee gpurun_out/${TAG}_k2_variants.log
for cfg in 3 2; do MFX_RW=8 timeout 300 python scripts/time_dist.py $cfg 200; done 2>&1 | tee gpurun_out/${TAG}_time_dist.log
for v in "0 2" "8 2" "8 3"; do
  set -- $v
  MFX_RW=$1 MFX_RW_MB=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 2 -c 2 -o /tmp/k2_$1_$2 python scripts/prof_solve.py --kind pp --iters 3 > /dev/null 2>&1
  ncu -i /tmp/k2_$1_$2.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_rw$1_mb$2_raw.csv 2>&1
  ncu -i /tmp/k2_$1_$2.ncu-rep --page source --csv > gpurun_out/${TAG}_ncu_rw$1_mb$2_source.csv 2>&1
  rm -f /tmp/k2_$1_$2.ncu-rep
done
ls -la gpurun_out
