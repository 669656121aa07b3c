timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t56.log 2>&1; echo t=$?
timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p56.log 2>&1; echo p=$?
HF_TRAIL_SIMPLE=1 timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p56s.log 2>&1; echo s=$?
timeout 300 python tools/probe_stage1.py C3 > gpurun_out/p56c3.log 2>&1; echo p=$?
