# A/B of two library builds in one box session (MFX_SO_VARIANT), interleaved
for rep in 1 2; do for so in variants/libmfx_head.so variants/libmfx_new.so; do
  echo "== $so rep $rep"
  for cfg in 3 2; do
    MFX_SO_VARIANT=$so MFX_PERSIST_TRACE=1 timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 2 --path 5 2>&1 | grep "persist trace" | head -1 | cut -c1-400
    for path in 1 5; do echo -n "c$cfg path $path: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path $path 2>&1 | grep timed | tail -1; done
  done
done; done
