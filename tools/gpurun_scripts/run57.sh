timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p57.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trailing -s 140 -c 1 -o gpurun_out/trp python tools/probe_stage1.py C2 > gpurun_out/ncu57a.log 2>&1; echo a=$?
HF_TRAIL_SIMPLE=1 ncu --set full --clock-control none --import-source on -k regex:k_trailing -s 140 -c 1 -o gpurun_out/trs python tools/probe_stage1.py C2 > gpurun_out/ncu57b.log 2>&1; echo b=$?
