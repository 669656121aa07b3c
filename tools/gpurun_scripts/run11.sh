timeout 600 python tools/probe_steps.py C2 > gpurun_out/steps.log 2>&1; echo p=$?
timeout 600 python tools/probe_steps.py C2 prof >> gpurun_out/steps.log 2>&1; echo p=$?
