#!/bin/bash
# near-item priority (HF_TRSM_NEARQ) with P-worker fallback
mkdir -p gpurun_out
HF_TRSM_NEARQ=1 timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py -q -x > gpurun_out/t119.log 2>&1; echo "tests rc $?" >> gpurun_out/t119.log
for q in 0 1; do for la in 8 24; do
echo "NEARQ=$q LA=$la $(HF_TRSM_NEARQ=$q HF_TRSM_LA=$la timeout 300 python tools/prof_trsm.py C2 256 5 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p119.log
done; done
HF_TRSM_NEARQ=1 HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 >> gpurun_out/p119.log 2>&1
