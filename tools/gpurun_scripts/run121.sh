#!/bin/bash
# helper PARTIAL items in 4x8 k-split form (HF_TRSM_H48)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py tests/test_gpu_fp64.py tests/test_gpu_nonsym.py -q -x > gpurun_out/t121.log 2>&1; echo "tests rc $?" >> gpurun_out/t121.log
for h in 1 0 1 0; do
echo "H48=$h C2 $(HF_TRSM_H48=$h timeout 300 python tools/prof_trsm.py C2 256 5 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p121.log
done
for h in 1 0; do
echo "H48=$h C4 $(HF_TRSM_H48=$h timeout 300 python tools/prof_trsm.py C4 256 2 2>&1 | grep -o 'trsm_ms_per_apply\": [0-9.]*')" >> gpurun_out/p121.log
done
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 >> gpurun_out/p121.log 2>&1
