HF_CHAIN_DEBUG=1 timeout 600 python tools/probe_stage1.py C2 > gpurun_out/chain13.log 2>&1; echo p=$?
