timeout 900 python -X faulthandler -m pytest tests/test_gpu_dd.py -x -q > gpurun_out/t92.log 2>&1; echo t=$?
