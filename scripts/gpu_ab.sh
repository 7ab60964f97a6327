# A/B of two library builds in one box session (MFX_SO_VARIANT), interleaved
MFX_SO_VARIANT=abv/libmfx_new.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not long_horizon" 2>&1 | tail -2
for rep in 1 2; do for so in abv/libmfx_head.so abv/libmfx_new.so; do
  for cfg in 2 3; do echo -n "$so c$cfg path 1: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo; done
  echo -n "$so c2 w: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config 2 --kind w --iters 20 --repeat 3 2>&1 | grep -E "timed" | tail -1
done; done
