timeout 900 python tools/probe_parts.py C2 8 > gpurun_out/parts_c2.log 2>&1; echo a=$?
timeout 900 python tools/probe_parts.py C4 8 > gpurun_out/parts_c4.log 2>&1; echo b=$?
