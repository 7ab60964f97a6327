set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for lz in 0 8 16 32 64; do
  if [ $lz = 0 ]; then unset MFX_LZ; else export MFX_LZ=$lz; fi
  echo "LZ=$lz"; python scripts/prof_solve.py --kind pp --iters 100 --repeat 3 | tail -2
done
unset MFX_LZ
python scripts/prof_solve.py --kind w --iters 100 --repeat 3 | tail -2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 20 --csv --log-file gpurun_out/launches_pp2.csv python scripts/prof_solve.py --kind pp --iters 5 > /dev/null 2>&1
