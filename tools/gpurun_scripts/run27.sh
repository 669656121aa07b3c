python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t27.log 2>&1; echo t=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench27.log 2>&1; echo b=$?
timeout 900 python tools/probe_stage1.py C4 > gpurun_out/p27_c4.log 2>&1; echo c=$?
