for v in "HF_X=0" "HF_CHAIN_SMEMX=1" "HF_CHAIN_FDIV=1" "HF_CHAIN_SMEMX=1 HF_CHAIN_FDIV=1" "HF_X=0"; do
env $v timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p66.log 2>&1; echo "$v $(grep -E '^chain' gpurun_out/p66.log)"
done
