#!/bin/bash
# chain: how often is the pivot the previous step's runner-up candidate (speculation statistics)
mkdir -p gpurun_out
for c in C2 C1 C3; do echo "== $c" >> gpurun_out/p138.log; HF_CHAIN_DEBUG=1 timeout 300 python tools/probe_config.py $c 1 2>&1 | grep "hf chain" | tail -2 >> gpurun_out/p138.log; done
