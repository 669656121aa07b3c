timeout 300 python -X faulthandler -m pytest tests/test_gpu_precond.py tests/test_gpu_fp64.py -x -q > gpurun_out/t84.log 2>&1; echo t=$?
HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 2 > gpurun_out/p84.log 2>&1; echo p=$?
for v in "HF_TRSM_PW=1" "HF_TRSM_PW=3" "HF_TRSM_TAIL=1" "HF_TRSM_TAIL=4" "HF_TRSM_GEO=0 HF_TRSM_TAIL=8 HF_TRSM_PW=4" "HF_TRSM_GEO=0 HF_TRSM_TAIL=16 HF_TRSM_PW=6"; do echo "$v $(env $v HF_TRSM_DEBUG=1 timeout 300 python tools/prof_trsm.py C2 256 1 2>&1 | grep -o 'bwd.*P-workers.*\|trsm_ms_per_apply.*' | tail -2 | tr '\n' ' ')" >> gpurun_out/p84.log; done
