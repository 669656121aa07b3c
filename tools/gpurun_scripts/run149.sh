#!/bin/bash
# stage-1 lookahead schedule re-measured with the current kernels
mkdir -p gpurun_out
HF_LOOKAHEAD=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b149.json 2> gpurun_out/b149.err; echo "bench look rc $?" >> gpurun_out/b149.err
HF_LOOKAHEAD=1 HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_config.py C2 1 2>&1 | grep "hf chain" | tail -2 >> gpurun_out/b149.err
