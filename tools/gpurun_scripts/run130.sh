#!/bin/bash
# Gram inverse: pivot blocks of 32 vs 16
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gram.py tests/test_gpu_stage23.py -q -x > gpurun_out/t130.log 2>&1; echo "tests rc $?" >> gpurun_out/t130.log
HF_SPD_BS=16 timeout 600 python -m pytest tests/test_gpu_gram.py -q -x >> gpurun_out/t130.log 2>&1; echo "tests bs16 rc $?" >> gpurun_out/t130.log
for n in 64 256 300 448; do
  timeout 120 python tools/prof_gram.py $n 20 >> gpurun_out/p130.log 2>&1
  HF_SPD_BS=16 timeout 120 python tools/prof_gram.py $n 20 >> gpurun_out/p130.log 2>&1
done
