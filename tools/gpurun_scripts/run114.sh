for pw in 2 3; do for tl in 1 2; do for sg in 16 32; do for la in 24 48; do
echo "PW=$pw TAIL=$tl SEG=$sg LA=$la $(HF_TRSM_PW=$pw HF_TRSM_TAIL=$tl HF_TRSM_SEG=$sg HF_TRSM_LA=$la timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')"
done; done; done; done
