python tools/probe_stage1.py C2 > gpurun_out/p22.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trailing -s 20 -c 1 -o gpurun_out/prof_trailing python tools/probe_stage1.py C2 > gpurun_out/ncu22.log 2>&1; echo n=$?
