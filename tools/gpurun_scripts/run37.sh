python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_stage1.py -x -q > gpurun_out/t37.log 2>&1; echo t=$?
