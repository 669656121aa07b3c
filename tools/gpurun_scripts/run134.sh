#!/bin/bash
# persistent trailing kernel with seed prefetch (k_trailing_p) vs k_trailing_c
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_multiblock.py tests/test_gpu_stage23.py -q -x > gpurun_out/t134.log 2>&1; echo "tests rc $?" >> gpurun_out/t134.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b134.json 2> gpurun_out/b134.err; echo "bench rc $?" >> gpurun_out/b134.err
HF_TRAIL_PERSIST=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b134c.json 2>> gpurun_out/b134.err; echo "bench c rc $?" >> gpurun_out/b134.err
