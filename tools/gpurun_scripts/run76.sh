timeout 600 python -m pytest tests/test_gpu_precond.py -x -q 2>&1 | tail -1
HF_TRSM_TRACE=1 timeout 300 python tools/prof_trsm.py C2 256 2 2>&1 | tail -7
for v in "HF_TRSM_ELAG=6" "HF_TRSM_ELAG=2" "HF_TRSM_ELAG=12" "HF_TRSM_TAIL=2" "HF_TRSM_SEG=32"; do echo "$v $(env $v timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -1)"; done
