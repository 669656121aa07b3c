timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t85.log 2>&1; echo t=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench85.log 2>&1; echo b=$?
timeout 300 python tools/determinism.py > gpurun_out/det85.log 2>&1; echo d=$?
