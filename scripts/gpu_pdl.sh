for p in 0 1; do echo "PDL=$p"; MFX_PDL=$p timeout 300 python scripts/time_paths.py 3,2 2>&1 | grep tma; done
