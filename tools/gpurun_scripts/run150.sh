#!/bin/bash
# TRSM parameter sweep with the current helpers (tools/prof_trsm.py includes the ~2.6 ms setup)
mkdir -p gpurun_out
for pw in 2 3; do for sg in 16 24; do for la in 16 24 40; do
echo "PW=$pw SEG=$sg LA=$la $(HF_TRSM_PW=$pw HF_TRSM_SEG=$sg HF_TRSM_LA=$la timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p150.log
done; done; done
