timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -rs --durations=0 > gpurun_out/fullsize.log 2>&1; echo t=$?
