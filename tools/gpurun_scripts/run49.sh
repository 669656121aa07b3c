python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t49.log 2>&1; echo t=$?
timeout 600 python tools/probe_stage1.py C2 > gpurun_out/p49.log 2>&1; echo p=$?
