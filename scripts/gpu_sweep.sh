timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for path in 1 2; do echo "== c1 pp path $path"; python scripts/prof_solve.py --config 1 --kind pp --iters 500 --repeat 4 --path $path | tail -2; done
echo "== c1 w path 2"; python scripts/prof_solve.py --config 1 --kind w --iters 200 --repeat 4 --path 2 | tail -2
