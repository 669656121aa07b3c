#!/bin/bash
# hard factorization on a 16-CTA cluster vs the cooperative kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage23.py tests/test_gpu_fullsize.py tests/test_gpu_multiblock.py tests/test_gpu_fp64.py -q -x > gpurun_out/t141.log 2>&1; echo "tests rc $?" >> gpurun_out/t141.log
HF_HARD_NOCLUSTER=1 timeout 900 python -m pytest tests/test_gpu_stage23.py -q -x >> gpurun_out/t141.log 2>&1; echo "tests nocluster rc $?" >> gpurun_out/t141.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b141.json 2> gpurun_out/b141.err; echo "bench rc $?" >> gpurun_out/b141.err
HF_HARD_NOCLUSTER=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b141n.json 2>> gpurun_out/b141.err; echo "bench n rc $?" >> gpurun_out/b141.err
