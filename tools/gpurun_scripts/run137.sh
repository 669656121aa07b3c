#!/bin/bash
# ncu full capture of one large k_trailing_p launch (C2)
mkdir -p gpurun_out
timeout 300 python tools/probe_config.py C2 1 > gpurun_out/p137.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trailing_p -s 3 -c 1 -o gpurun_out/trail137 -f python tools/probe_config.py C2 1 > gpurun_out/ncu137.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu137.log
