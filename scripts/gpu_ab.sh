# same-box A/B of library builds (MFX_SO_VARIANT), interleaved
for rep in 1 2; do for so in abv/libmfx_ku1.so abv/libmfx_ku2.so abv/libmfx_ku4.so; do
  for cfg in 2 3; do echo -n "$so c$cfg path5: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 5 2>&1 | grep -E "timed" | tail -1; done
done; done
MFX_SO_VARIANT=abv/libmfx_ku2.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k persist 2>&1 | tail -1
