timeout 1200 python tools/probe_config.py C3 2 > gpurun_out/c3.log 2>&1; echo c3=$?
timeout 900 python -m pytest tests/test_gpu_stage1.py tests/test_gpu_stage23.py -x -q -k "S12 or S24" > gpurun_out/gpu_tests16.log 2>&1; echo tests=$?
