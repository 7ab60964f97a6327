# A/B of two library builds in one box session (MFX_SO_VARIANT), interleaved
for rep in 1 2; do for so in variants/libmfx_head.so variants/libmfx_new.so; do
  for cfg in 3 2; do for path in 1 5; do echo -n "$so c$cfg path $path: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path $path 2>&1 | grep timed | tail -1; done; done
done; done
