# persistent solver: 2 CTAs/SM x 3 stages vs 1 CTA/SM x 6 stages (MFX_PERSIST_S)
MFX_PERSIST_S=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "persist" 2>&1 | tail -1
for rep in 1 2 3; do for ps in 3 6; do for cfg in 3 2; do
  echo -n "MFX_PERSIST_S=$ps c$cfg path5: "; MFX_PERSIST_S=$ps timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 5 2>&1 | grep -E "timed" | tail -1
done; done; done
