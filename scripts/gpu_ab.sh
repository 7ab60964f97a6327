# same-box A/B of two library builds (MFX_SO_VARIANT), interleaved
MFX_SO_VARIANT=abv/libmfx_new.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bicgstab or simple" 2>&1 | tail -1
for rep in 1 2 3; do for so in abv/libmfx_head.so abv/libmfx_new.so; do
  for cfg in 2 3; do echo -n "$so c$cfg: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo; done
done; done
