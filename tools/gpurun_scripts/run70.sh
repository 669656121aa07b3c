for la in 4 12 24 48 96; do echo "LA=$la $(HF_TRSM_LA=$la timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -1)"; done
for sg in 4 8 32; do echo "SEG=$sg $(HF_TRSM_SEG=$sg timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -1)"; done
