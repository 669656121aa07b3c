#!/bin/bash
# full GPU suite + smoke + bench at HEAD
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/t116.log 2>&1; echo "tests rc $?" >> gpurun_out/t116.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s116.log 2>&1; echo "smoke rc $?" >> gpurun_out/s116.log
timeout 600 python bench.py > gpurun_out/b116.json 2> gpurun_out/b116.err; echo "bench rc $?" >> gpurun_out/b116.err
