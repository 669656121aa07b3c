timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t87.log 2>&1; echo t=$?
timeout 300 python tools/probe_stage1.py C2 > gpurun_out/p87.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trailing -s 140 -c 1 -o gpurun_out/tr87 python tools/probe_stage1.py C2 > gpurun_out/ncu87.log 2>&1; echo a=$?
