HF_ALLOC_DEBUG=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench12_1.log 2>&1; echo bench=$?
