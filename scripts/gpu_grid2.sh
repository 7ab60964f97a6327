set -x
for c in 1 2 4 8; do MFX_GRID_CTAS_PER_SM=$c timeout 300 python scripts/time_paths.py 3 2>&1 | grep grid; done
