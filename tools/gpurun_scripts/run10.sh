for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench10_$i.log 2>&1; echo bench=$?; done
