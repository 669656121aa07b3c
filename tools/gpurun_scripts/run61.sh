timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t61.log 2>&1; echo t=$?
timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p61.log 2>&1; echo p=$?
HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p61d.log 2>&1; echo p=$?
