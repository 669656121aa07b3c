python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t34.log 2>&1; echo t=$?
timeout 600 python tools/probe_stage1.py C2 > gpurun_out/p34.log 2>&1; echo p=$?
HF_LOOKAHEAD=0 timeout 600 python tools/probe_stage1.py C2 > gpurun_out/p34_serial.log 2>&1; echo p=$?
