#!/bin/bash
# blocked Gram inverse on the 16-CTA cluster: parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_stage23.py tests/test_gpu_krylov.py tests/test_gpu_dd.py -q -x > gpurun_out/t128.log 2>&1; echo "tests rc $?" >> gpurun_out/t128.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b128.json 2> gpurun_out/b128.err; echo "bench rc $?" >> gpurun_out/b128.err
HF_SPD_SCALAR=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b128s.json 2>> gpurun_out/b128.err; echo "bench scalar rc $?" >> gpurun_out/b128.err
