python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/gpu_tests14.log 2>&1; echo tests=$?
HF_CHAIN_DEBUG=1 timeout 600 python tools/probe_stage1.py C2 > gpurun_out/chain14.log 2>&1; echo p=$?
HF_CHAIN_DEBUG=1 timeout 600 python tools/probe_stage1.py C2 128 >> gpurun_out/chain14.log 2>&1; echo p=$?
