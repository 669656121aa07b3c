HF_TRSM_TAIL=1 HF_TRSM_TRACE=1 timeout 300 python tools/prof_trsm.py C2 256 2 2>&1 | tail -7
