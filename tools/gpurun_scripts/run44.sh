for cfg in "8 16" "8 32" "24 32" "24 64" "0 32"; do set -- $cfg
HF_TRSM_LA=$1 HF_TRSM_SEG=$2 timeout 300 python tools/prof_trsm.py C2 256 3 > gpurun_out/p44.log 2>&1; echo "$1 $2 $(tail -1 gpurun_out/p44.log | cut -c60-140)"; done
