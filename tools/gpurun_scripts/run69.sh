HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 3 > gpurun_out/p69.log 2>&1; echo p=$?
