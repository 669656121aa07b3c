timeout 900 python tools/probe_gcr.py C4 30 512 > gpurun_out/c4_512.log 2>&1; echo a=$?
timeout 900 python tools/probe_gcr.py C4 30 1024 > gpurun_out/c4_1024.log 2>&1; echo b=$?
