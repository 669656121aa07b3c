timeout 600 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_dist.py -x -q > gpurun_out/t64.log 2>&1; echo t=$?
timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p64.log 2>&1; echo p=$?
HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p64d.log 2>&1; echo p=$?
HF_CHAIN_SMEMX=1 HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p64s.log 2>&1; echo p=$?
