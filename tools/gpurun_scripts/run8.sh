python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench8_$i.log 2>&1; echo bench=$?; done
nproc; lscpu | grep "Model name"
