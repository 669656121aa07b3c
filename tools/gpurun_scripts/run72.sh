for tl in 1 2; do HF_TRSM_TAIL=$tl HF_TRSM_TRACE=1 timeout 300 python tools/prof_trsm.py C2 256 2 2>&1 | tail -3; done
