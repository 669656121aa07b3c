HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 1 > gpurun_out/p81.log 2>&1; echo p=$?
HF_TRSM_DEBUG=1 HF_TRSM_PW=4 timeout 300 python tools/prof_trsm.py C2 256 1 >> gpurun_out/p81.log 2>&1; echo p=$?
