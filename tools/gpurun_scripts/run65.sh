for v in "" "HF_CHAIN_SMEMX=1"; do
env $v timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p65.log 2>&1; echo "$v"; grep -E "^chain" gpurun_out/p65.log
env $v HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_stage1.py C2 2>&1 | grep "hf chain" | tail -1
done
