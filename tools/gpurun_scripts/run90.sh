for v in "HF_X=0" "HF_LOOKAHEAD=1"; do env $v timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p90.log 2>&1; echo "$v $(grep -E 'rep\": 1|^chain|^trailing|^other' gpurun_out/p90.log | tr '\n' ' ')"; done
HF_LOOKAHEAD=1 timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q 2>&1 | tail -1
