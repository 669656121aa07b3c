#!/bin/bash
# two-queue TRSM helper scheduler: parity + timing vs one queue
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py tests/test_gpu_nonsym.py -x -q > gpurun_out/t115.log 2>&1; echo "tests rc $?" >> gpurun_out/t115.log
for q in 1 0 1 0; do
  HF_TRSM_Q2=$q timeout 300 python tools/prof_trsm.py C2 256 5 >> gpurun_out/p115.log 2>&1; echo "q2=$q" >> gpurun_out/p115.log
done
HF_TRSM_Q2=1 timeout 300 python tools/prof_trsm.py C4 256 2 >> gpurun_out/p115.log 2>&1; echo "C4 q2=1" >> gpurun_out/p115.log
HF_TRSM_Q2=0 timeout 300 python tools/prof_trsm.py C4 256 2 >> gpurun_out/p115.log 2>&1; echo "C4 q2=0" >> gpurun_out/p115.log
HF_TRSM_Q2=1 timeout 300 python tools/prof_trsm.py C1 256 5 >> gpurun_out/p115.log 2>&1; echo "C1 q2=1" >> gpurun_out/p115.log
HF_TRSM_Q2=0 timeout 300 python tools/prof_trsm.py C1 256 5 >> gpurun_out/p115.log 2>&1; echo "C1 q2=0" >> gpurun_out/p115.log
