for rep in 1 2; do for pdl in 0 1; do for cfg in 2 3; do
  echo -n "MFX_PDL=$pdl c$cfg path1: "; MFX_PDL=$pdl timeout 300 python scripts/prof_solve.py --config $cfg --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed" | tail -1
done; done; done
