timeout 600 python tools/probe_config.py C2 3 > gpurun_out/p102.log 2>&1; echo p=$?
timeout 600 python -m pytest tests/test_gpu_stage23.py tests/test_gpu_krylov.py -x -q > gpurun_out/t102.log 2>&1; echo t=$?
