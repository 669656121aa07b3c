timeout 600 python -m pytest tests/test_gpu_precond.py -x -q 2>&1 | tail -1
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -3
for v in "HF_TRSM_PW=1" "HF_TRSM_PW=3" "HF_TRSM_TAIL=1" "HF_TRSM_TAIL=3" "HF_TRSM_ELAG=4" "HF_TRSM_ELAG=16" "HF_TRSM_LA=48"; do echo "$v $(env $v timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -1)"; done
