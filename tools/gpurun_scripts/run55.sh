HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p55_dbg.log 2>&1; echo a=$?
for g in 32 48 64 96; do HF_CHAIN_CTAS=$g timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p55_g$g.log 2>&1; echo g=$?; done
