timeout 900 python tools/probe_parts.py C2 1 > gpurun_out/parts1.log 2>&1; echo a=$?
timeout 900 python tools/probe_parts.py C2 2 > gpurun_out/parts2.log 2>&1; echo a=$?
