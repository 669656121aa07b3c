#!/bin/bash
# dedicated near-queue helpers (HF_TRSM_NNH) sweep
mkdir -p gpurun_out
HF_TRSM_NNH=16 timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py -q -x > gpurun_out/t118.log 2>&1; echo "tests rc $?" >> gpurun_out/t118.log
for n in 0 8 16 24 32 48; do
echo "NNH=$n $(HF_TRSM_NNH=$n timeout 300 python tools/prof_trsm.py C2 256 5 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p118.log
done
HF_TRSM_NNH=16 HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 3 >> gpurun_out/p118.log 2>&1
