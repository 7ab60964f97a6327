# row-warp consumer: stage released before the step-2 compute (MFX_RW_EARLY_RELEASE build) vs default
MFX_SO_VARIANT=abv/libmfx_er.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bicgstab_pp" 2>&1 | tail -1
for rep in 1 2 3; do for so in "" abv/libmfx_er.so; do for cfg in 2 3; do
  echo -n "so=${so:-default} c$cfg: "; MFX_SO_VARIANT=$so timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo
done; done; done
