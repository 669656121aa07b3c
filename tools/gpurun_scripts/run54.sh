python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_stage23.py -x -q > gpurun_out/t54.log 2>&1; echo t=$?
for c in C2 C3; do
timeout 600 python tools/probe_config.py $c 3 > gpurun_out/p54_$c.log 2>&1; echo p=$?
HF_HARD_UNFUSED=1 timeout 600 python tools/probe_config.py $c 3 > gpurun_out/p54u_$c.log 2>&1; echo u=$?
done
