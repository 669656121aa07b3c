timeout 600 python -m pytest tests/test_gpu_precond.py -x -q 2>&1 | tail -1
for tl in 1 2; do HF_TRSM_TAIL=$tl HF_TRSM_TRACE=1 timeout 300 python tools/prof_trsm.py C2 256 2 2>&1 | tail -3; done
for sg in 16 32 64; do echo "SEG=$sg $(HF_TRSM_TAIL=1 HF_TRSM_SEG=$sg timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -1)"; done
