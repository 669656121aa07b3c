timeout 300 python -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/t86.log 2>&1; echo t=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 > gpurun_out/p86.log 2>&1; echo p=$?
