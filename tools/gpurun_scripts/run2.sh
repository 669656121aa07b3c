python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_stage23.py -x -q > gpurun_out/gpu_tests23.log 2>&1; echo tests=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench2.log 2>&1; echo bench=$?
