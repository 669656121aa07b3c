#!/bin/bash
# ncu full capture of one forward k_trsm launch (C2, 256 columns), after a plain run
mkdir -p gpurun_out
timeout 300 python tools/prof_trsm.py C2 256 2 > gpurun_out/p122.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trsm -s 2 -c 1 -o gpurun_out/trsm122 -f python tools/prof_trsm.py C2 256 2 > gpurun_out/ncu122.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu122.log
