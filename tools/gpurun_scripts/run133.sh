#!/bin/bash
# ncu full capture of one large k_trailing_c launch (C2 stage 1), after a plain run
mkdir -p gpurun_out
timeout 300 python tools/probe_config.py C2 1 > gpurun_out/p133.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trailing_c -s 3 -c 1 -o gpurun_out/trail133 -f python tools/probe_config.py C2 1 > gpurun_out/ncu133.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu133.log
