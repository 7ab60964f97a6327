for v in "0 0" "1 0" "1 28" "1 19" "1 14" "0 0"; do set -- $v
  echo -n "MFX_DYN=$1 MFX_LZ=$2 c2: "; MFX_DYN=$1 MFX_LZ=$2 timeout 300 python scripts/prof_solve.py --config 2 --kind pp --iters 200 --repeat 3 --path 1 2>&1 | grep -E "timed|kernels" | tail -2 | tr '\n' ' '; echo
done
