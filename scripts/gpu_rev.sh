for v in "8 1" "8 0" "12 1" "12 0" "15 0"; do
  set -- $v
  echo "c2 MFX_RW=$1 MFX_REVERSE=$2"
  MFX_RW=$1 MFX_REVERSE=$2 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 3 2>&1 | tail -3
done 2>&1 | tee gpurun_out/${TAG}_rev.log
