#!/bin/bash
# split-K reduced in-kernel by the last CTA of each tile vs k_reduce
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage23.py tests/test_gpu_krylov.py tests/test_gpu_fp64.py tests/test_gpu_dist.py tests/test_gpu_nonsym.py -q -x > gpurun_out/t131.log 2>&1; echo "tests rc $?" >> gpurun_out/t131.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b131.json 2> gpurun_out/b131.err; echo "bench rc $?" >> gpurun_out/b131.err
HF_DGEMM_REDUCE=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b131r.json 2>> gpurun_out/b131.err; echo "bench reduce rc $?" >> gpurun_out/b131.err
