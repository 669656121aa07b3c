#!/bin/bash
# TRSM accumulate with one barrier per tile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py tests/test_gpu_fp64.py tests/test_gpu_nonsym.py -q -x > gpurun_out/t143.log 2>&1; echo "tests rc $?" >> gpurun_out/t143.log
for r in 1 2; do
echo "C2 $(timeout 300 python tools/prof_trsm.py C2 256 5 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p143.log
done
echo "C4 $(timeout 300 python tools/prof_trsm.py C4 256 2 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p143.log
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 2>&1 | tail -5 >> gpurun_out/p143.log
