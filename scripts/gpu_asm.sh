set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "assemble or simple" > gpurun_out/pytest_asm.log 2>&1; tail -15 gpurun_out/pytest_asm.log
timeout 300 python scripts/time_asm.py > gpurun_out/asm_tma.json 2>&1; cat gpurun_out/asm_tma.json
MFX_ASM_TMA=0 timeout 300 python scripts/time_asm.py > gpurun_out/asm_gs.json 2>&1; cat gpurun_out/asm_gs.json
