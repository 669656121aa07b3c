#!/bin/bash
# preconditioner setup: 16-byte stores in k_scale_op
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py tests/test_gpu_fp64.py tests/test_gpu_nonsym.py tests/test_gpu_dd.py tests/test_gpu_krylov.py -q -x > gpurun_out/t147.log 2>&1; echo "tests rc $?" >> gpurun_out/t147.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b147.json 2> gpurun_out/b147.err; echo "bench rc $?" >> gpurun_out/b147.err
