timeout 300 python -m pytest tests/test_gpu_precond.py tests/test_gpu_dist.py -x -q > gpurun_out/t33.log 2>&1; echo t=$?
