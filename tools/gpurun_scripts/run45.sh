python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_stage23.py tests/test_gpu_dist.py -x -q > gpurun_out/t45.log 2>&1; echo t=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench45.log 2>&1; echo b=$?
timeout 900 python tools/probe_config.py C3 2 > gpurun_out/c3_45.log 2>&1; echo c=$?
