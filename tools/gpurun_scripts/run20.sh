HF_FULLSIZE_ORACLE=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -k c3 --durations=0 > gpurun_out/fullsize_c3_oracle.log 2>&1; echo t=$?
