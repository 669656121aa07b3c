timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_dist.py tests/test_gpu_stage23.py -x -q > gpurun_out/t99.log 2>&1; echo t=$?
timeout 600 python tools/probe_mb.py C1 6 > gpurun_out/p99_c1.log 2>&1; echo a=$?
timeout 900 python tools/probe_mb.py C3 8 > gpurun_out/p99_c3.log 2>&1; echo b=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench99.log 2>&1; echo c=$?
