#!/bin/bash
# TRSM thread mapping 8x4 per warp
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py tests/test_gpu_fp64.py -q -x > gpurun_out/t120.log 2>&1; echo "tests rc $?" >> gpurun_out/t120.log
for r in 1 2; do
echo "$(timeout 300 python tools/prof_trsm.py C2 256 5 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p120.log
done
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 >> gpurun_out/p120.log 2>&1
timeout 300 python tools/prof_trsm.py C4 256 2 >> gpurun_out/p120.log 2>&1
