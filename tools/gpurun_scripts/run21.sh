python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/gpu_dist.log 2>&1; echo t=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e --mode shard --steps 3 > gpurun_out/bench_shard.log 2>&1; echo b=$?
