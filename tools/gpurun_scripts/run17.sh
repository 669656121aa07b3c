timeout 1500 python tools/probe_config.py C4 1 > gpurun_out/c4.log 2>&1; echo c4=$?
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
free -g | head -2
