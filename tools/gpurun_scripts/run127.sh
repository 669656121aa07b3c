#!/bin/bash
# bench at HEAD (TRSM 4x8 helpers) + launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py -q -x > gpurun_out/t127.log 2>&1; echo "tests rc $?" >> gpurun_out/t127.log
timeout 600 python bench.py > gpurun_out/b127.json 2> gpurun_out/b127.err; echo "bench rc $?" >> gpurun_out/b127.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches127.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu127.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu127.log
