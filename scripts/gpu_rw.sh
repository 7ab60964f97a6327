# Round-2 session checks: row-warp p' kernels (MFX_RW mask: 1 SPMV, 2 SETUP, 4 K1, 8 K2),
# the persistent solver (path 5), the TMA slab solver, comm-stream exchange / packed BCAST.
mkdir -p gpurun_out
TAG=${TAG:-r02b}
timeout 900 python -m pytest tests/test_gpu_pic.py -m gpu -x -q -k "multirank or sort_is" --durations=5 2>&1 | tail -4
MFX_RW=15 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_solver.py tests/test_gpu_multirank.py -m gpu -x -q -k "pp or simple or spmv or graph or true_rel or dist or multirank or packed or edge or not_converged or deterministic" --durations=10 2>&1 | tail -16
for cfg in 2 3; do
for v in "0 4" "8 3" "8 4" "12 4" "15 4" "15 3"; do
  set -- $v
  echo "config $cfg MFX_RW=$1 MFX_RW_STAGES=$2"
  MFX_RW=$1 MFX_RW_STAGES=$2 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 2>&1 | tail -3
done
done 2>&1 | tee gpurun_out/${TAG}_rw_sweep.log
for cfg in 1 3 2; do for path in 1 5; do
  echo "config $cfg path $path (MFX_RW=15)"
  MFX_RW=15 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path $path 2>&1 | tail -3
done; done 2>&1 | tee gpurun_out/${TAG}_persist.log
MFX_RW=15 timeout 300 python scripts/time_dist.py 2 200 2>&1 | tee gpurun_out/${TAG}_time_dist.log
MFX_RW=15 timeout 300 python scripts/time_dist.py 3 200 2>&1 | tee -a gpurun_out/${TAG}_time_dist.log
MFX_RW=15 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k3v" -s 4 -c 3 -o gpurun_out/${TAG}_prof_pp_c2 python scripts/prof_solve.py --kind pp --iters 4 > gpurun_out/ncu_pp.log 2>&1; tail -1 gpurun_out/ncu_pp.log
MFX_RW=15 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil|k3v" -s 4 -c 3 -o gpurun_out/${TAG}_prof_pp_c3 python scripts/prof_solve.py --config 3 --kind pp --iters 4 > gpurun_out/ncu_pp3.log 2>&1; tail -1 gpurun_out/ncu_pp3.log
ls gpurun_out
