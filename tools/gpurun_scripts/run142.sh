#!/bin/bash
# paired block updates of Alg. 5 in one DMMA launch (dgemm2), problem selected without dynamic param indexing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage23.py tests/test_gpu_krylov.py tests/test_gpu_fp64.py tests/test_gpu_dist.py tests/test_gpu_nonsym.py tests/test_gpu_gram.py -q -x > gpurun_out/t142.log 2>&1; echo "tests rc $?" >> gpurun_out/t142.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b142.json 2> gpurun_out/b142.err; echo "bench rc $?" >> gpurun_out/b142.err
