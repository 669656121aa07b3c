timeout 600 python tools/probe_config.py C2 1 > gpurun_out/p104.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_chain" -s 60 -c 1 -o gpurun_out/chain104 python tools/probe_config.py C2 1 > gpurun_out/ncu104a.log 2>&1; echo a=$?
ncu --set full --clock-control none --import-source on -k regex:"k_trsm" -s 2 -c 1 -o gpurun_out/trsm104 python tools/probe_config.py C2 1 > gpurun_out/ncu104b.log 2>&1; echo b=$?
ncu --set full --clock-control none --import-source on -k regex:"k_dgemm" -s 0 -c 1 -o gpurun_out/dgemm104 python tools/probe_config.py C2 1 > gpurun_out/ncu104c.log 2>&1; echo c=$?
