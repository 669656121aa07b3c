timeout 600 python tools/probe_config.py C2 1 > gpurun_out/p103.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_dgemm|k_reduce" --csv --log-file gpurun_out/dg103.csv python tools/probe_config.py C2 1 > gpurun_out/ncu103.log 2>&1; echo n=$?
