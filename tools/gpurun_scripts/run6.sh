python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/gpu_tests6.log 2>&1; echo tests=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 > gpurun_out/trsm6.log 2>&1; echo prof=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 64 2 >> gpurun_out/trsm6.log 2>&1; echo prof=$?
timeout 300 python tools/prof_trsm.py C2 256 5 >> gpurun_out/trsm6.log 2>&1; echo prof=$?
