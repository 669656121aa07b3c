python tools/probe_stage1.py C2 > gpurun_out/p43.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_chain -s 40 -c 1 -o gpurun_out/prof_chain2 python tools/probe_stage1.py C2 > gpurun_out/ncu43.log 2>&1; echo n=$?
