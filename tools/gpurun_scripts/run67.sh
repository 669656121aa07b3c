timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_dist.py tests/test_gpu_stage23.py tests/test_gpu_fp64.py -x -q > gpurun_out/t67.log 2>&1; echo t=$?
timeout 600 python bench.py > gpurun_out/bench67.log 2>&1; echo b=$?
