python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/t39.log 2>&1; echo t=$?
timeout 900 python tools/probe_parts.py C2 8 > gpurun_out/parts_c2.log 2>&1; echo a=$?
