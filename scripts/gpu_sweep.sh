timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "" "MFX_REVERSE=0" "MFX_TILE=1"; do
  echo "== pp $cfg"; env $cfg python scripts/prof_solve.py --kind pp --iters 100 --repeat 3 | tail -2
done
for cfg in "" "MFX_REVERSE=0"; do
echo "== w $cfg"; env $cfg python scripts/prof_solve.py --kind w --iters 100 --repeat 3 | tail -2
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_rev.csv python scripts/prof_solve.py --kind pp --iters 8 > /dev/null 2>&1
