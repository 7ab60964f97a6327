timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_sanitize.py -x -q -k "pic" > gpurun_out/pytest_pic2.log 2>&1; tail -3 gpurun_out/pytest_pic2.log
