HF_TRSM_TRACE=1 timeout 300 python tools/prof_trsm.py C2 256 2 > gpurun_out/p71.log 2>&1; echo p=$?
