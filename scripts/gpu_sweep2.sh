for t in 1 2 3 5; do for st in 3 4 6; do echo "TILE=$t STAGES=$st"; MFX_TILE=$t MFX_STAGES=$st timeout 120 python scripts/prof_solve.py --kind pp --iters 100 --repeat 2 2>&1 | tail -1; done; done
