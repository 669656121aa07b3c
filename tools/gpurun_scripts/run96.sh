timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t96.log 2>&1; echo t=$?
timeout 600 python tools/probe_ns.py T96 > gpurun_out/p96.log 2>&1; echo p=$?
timeout 900 python tools/table1.py C2 > gpurun_out/table1_c2.log 2>&1; echo a=$?
