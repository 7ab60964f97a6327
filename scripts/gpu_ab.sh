# K3 grid: CTAs per SM (MFX_K3_CPS; default = occupancy)
for rep in 1 2; do for cps in 0 2 4; do for cfg in 2 3; do
  echo -n "MFX_K3_CPS=$cps c$cfg path1: "; MFX_K3_CPS=$cps timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo
done; done; done
