# tile x stage sweep of the p' stencil kernels at configuration 3 (64x64x256)
for t in 1 2 3 4 5; do
  for s in 3 4; do
    echo "tile=$t stages=$s"; MFX_TILE=$t MFX_STAGES=$s timeout 300 python scripts/prof_solve.py --config 3 --kind pp --iters 200 --repeat 3 2>&1 | tail -2
  done
done
