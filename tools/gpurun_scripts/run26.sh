for cfg in "64 192" "64 224" "32 96" "128 128" "64 160"; do set -- $cfg
HF_CHAIN_CTAS=$1 timeout 600 python tools/probe_stage1.py C2 $2 > gpurun_out/p26_$1_$2.log 2>&1; echo "$1 $2 $(grep '^chain\|^trailing (' gpurun_out/p26_$1_$2.log | tr '\n' ' ')"; done
