timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_stage23.py tests/test_gpu_multiblock.py -x -q > gpurun_out/t106.log 2>&1; echo t=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench106.log 2>&1; echo b=$?
timeout 900 python tools/probe_stage1.py C4 > gpurun_out/p106_c4.log 2>&1; echo c=$?
