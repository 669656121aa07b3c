python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_fp64.py -x -q > gpurun_out/t51.log 2>&1; echo t=$?
