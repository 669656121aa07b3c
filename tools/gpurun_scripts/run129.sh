#!/bin/bash
# Gram inverse timing: blocked vs scalar cluster kernels
mkdir -p gpurun_out
for n in 64 256 448; do
  timeout 120 python tools/prof_gram.py $n 20 >> gpurun_out/p129.log 2>&1
  HF_SPD_SCALAR=1 timeout 120 python tools/prof_gram.py $n 20 >> gpurun_out/p129.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_gram.py tests/test_gpu_stage23.py tests/test_gpu_krylov.py -q -x > gpurun_out/t129.log 2>&1; echo "tests rc $?" >> gpurun_out/t129.log
