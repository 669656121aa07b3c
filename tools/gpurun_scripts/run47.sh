timeout 900 python tools/fig2.py C2 16 > gpurun_out/fig2_c2.log 2>&1; echo a=$?
timeout 900 python tools/fig2.py C3 16 > gpurun_out/fig2_c3.log 2>&1; echo b=$?
