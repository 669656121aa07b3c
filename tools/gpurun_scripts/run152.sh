#!/bin/bash
# chain CTA count sweep at C2 with the current kernels (stage-1 ms)
mkdir -p gpurun_out
for g in 40 48 56 64 74; do
  echo "G=$g $(HF_CHAIN_CTAS=$g timeout 300 python tools/probe_config.py C2 2 2>&1 | grep -o '"stage_ms": \[[0-9., ]*\]' | tail -1)" >> gpurun_out/p152.log
done
