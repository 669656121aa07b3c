python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/t31.log 2>&1; echo t=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 3 > gpurun_out/p31.log 2>&1; echo p=$?
