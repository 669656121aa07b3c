#!/bin/bash
# trailing prologue: map entries from global, no barrier before the seed loads
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_nonsym.py tests/test_gpu_multiblock.py -q -x > gpurun_out/t151.log 2>&1; echo "tests rc $?" >> gpurun_out/t151.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b151.json 2> gpurun_out/b151.err; echo "bench rc $?" >> gpurun_out/b151.err
