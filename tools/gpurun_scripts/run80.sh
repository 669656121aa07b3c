timeout 300 python -X faulthandler -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/t80.log 2>&1; echo t=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 3 > gpurun_out/p80.log 2>&1; echo p=$?
for v in "HF_TRSM_PW=1" "HF_TRSM_PW=3" "HF_TRSM_PW=4" "HF_TRSM_TAIL=1" "HF_TRSM_TAIL=3" "HF_TRSM_LA=48"; do echo "$v $(env $v timeout 300 python tools/prof_trsm.py C2 256 3 2>&1 | tail -1)" >> gpurun_out/p80.log; done
