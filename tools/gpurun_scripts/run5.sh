python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_precond.py -x -q > gpurun_out/gpu_tests5.log 2>&1; echo tests=$?
timeout 300 python tools/prof_trsm.py C2 256 5 > gpurun_out/trsm5.log 2>&1; echo prof=$?
timeout 300 python tools/prof_trsm.py C2 64 5 >> gpurun_out/trsm5.log 2>&1; echo prof=$?
timeout 900 python -m pytest tests/test_gpu_stage23.py -x -q >> gpurun_out/gpu_tests5.log 2>&1; echo tests=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench5.log 2>&1; echo bench=$?
