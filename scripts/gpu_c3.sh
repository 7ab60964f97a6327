for t in 0 1 2 4 5; do for st in 3 4 6; do echo "TILE=$t STAGES=$st"; MFX_TILE=$t MFX_STAGES=$st timeout 120 python scripts/prof_solve.py --config 3 --kind pp --iters 200 --repeat 3 2>&1 | tail -3; done; done
for lz in 4 8 16 32; do echo "LZ=$lz"; MFX_LZ=$lz timeout 120 python scripts/prof_solve.py --config 3 --kind pp --iters 200 --repeat 3 2>&1 | tail -3; done
