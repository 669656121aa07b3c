timeout 600 python -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/t68.log 2>&1; echo t=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 3 > gpurun_out/p68.log 2>&1; echo p=$?
for tl in 1 3; do HF_TRSM_TAIL=$tl timeout 300 python tools/prof_trsm.py C2 256 3 > gpurun_out/p68_$tl.log 2>&1; echo p=$?; done
