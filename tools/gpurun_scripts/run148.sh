#!/bin/bash
# final: full GPU suite + smoke + bench + reference + launch list at HEAD
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/t148.log 2>&1; echo "tests rc $?" >> gpurun_out/t148.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s148.log 2>&1; echo "smoke rc $?" >> gpurun_out/s148.log
timeout 600 python bench.py > gpurun_out/b148.json 2> gpurun_out/b148.err; echo "bench rc $?" >> gpurun_out/b148.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b148ref.json 2>> gpurun_out/b148.err; echo "ref rc $?" >> gpurun_out/b148.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches148.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu148.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu148.log
