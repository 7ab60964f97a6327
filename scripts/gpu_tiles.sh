# tile sweep of the stencil kernels (MFX_TILE: 1 64x4, 2 64x8 pairs, 3 32x16 pairs, 5 64x8)
for t in 0 1 2 5; do
  for k in pp w; do
    echo "tile=$t kind=$k"; MFX_TILE=$t timeout 300 python scripts/prof_solve.py --kind $k --iters 100 --repeat 2 2>&1 | tail -1
  done
done
