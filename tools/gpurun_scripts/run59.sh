HF_TRAIL=p timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t59.log 2>&1; echo t=$?
HF_TRAIL=p timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p59.log 2>&1 && \
HF_TRAIL=p ncu --set full --clock-control none --import-source on -k regex:k_trailing -s 140 -c 1 -o gpurun_out/tr59 python tools/probe_stage1.py C2 > gpurun_out/ncu59.log 2>&1; echo a=$?
