timeout 900 python tools/probe_dd.py C2 > gpurun_out/p93.log 2>&1; echo p=$?
