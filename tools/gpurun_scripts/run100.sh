timeout 900 python -m pytest tests/test_gpu_multiblock.py tests/test_gpu_stage1.py -x -q > gpurun_out/t100.log 2>&1; echo t=$?
timeout 600 python tools/probe_mb.py C1 6 > gpurun_out/p100_c1.log 2>&1; echo a=$?
timeout 900 python tools/probe_mb.py C3 8 > gpurun_out/p100_c3.log 2>&1; echo b=$?
