#!/bin/bash
# Table 1 analog refresh (C2, C3) with the current kernels
mkdir -p gpurun_out
timeout 900 python tools/table1.py C2 > gpurun_out/table1_c2.log 2>&1; echo "c2 rc $?" >> gpurun_out/table1_c2.log
timeout 900 python tools/table1.py C3 > gpurun_out/table1_c3.log 2>&1; echo "c3 rc $?" >> gpurun_out/table1_c3.log
