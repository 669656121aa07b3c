python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q > gpurun_out/t25.log 2>&1; echo t=$?
HF_CHAIN_XCHG=slots timeout 600 python tools/probe_stage1.py C2 > gpurun_out/p25_slots.log 2>&1; echo a=$?
HF_CHAIN_XCHG=counter timeout 600 python tools/probe_stage1.py C2 > gpurun_out/p25_counter.log 2>&1; echo b=$?
