python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_precond.py tests/test_gpu_stage23.py -x -q > gpurun_out/gpu_tests7.log 2>&1; echo tests=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench7.log 2>&1; echo bench=$?
