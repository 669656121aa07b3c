python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b23.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu23.log 2>&1; echo n=$?
