timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p63.log 2>&1; echo p=$?
HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p63d.log 2>&1; echo p=$?
