timeout 300 python -X faulthandler tools/prof_trsm.py C2 256 1 > gpurun_out/p79.log 2>&1; echo p=$?
timeout 300 python -X faulthandler -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/t79.log 2>&1; echo t=$?
