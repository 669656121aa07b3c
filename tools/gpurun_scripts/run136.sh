#!/bin/bash
# persistent trailing kernel: forced-parity tests, C2 bitwise probe, bench on/off
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_multiblock.py tests/test_gpu_stage23.py -q -x > gpurun_out/t136.log 2>&1; echo "tests rc $?" >> gpurun_out/t136.log
timeout 300 python tools/probe_trailp.py C2 > gpurun_out/p136.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b136.json 2> gpurun_out/b136.err; echo "bench rc $?" >> gpurun_out/b136.err
HF_TRAIL_PERSIST=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b136c.json 2>> gpurun_out/b136.err; echo "bench c rc $?" >> gpurun_out/b136.err
