timeout 900 python tools/table1.py C2 > gpurun_out/table1_c2.log 2>&1; echo a=$?
timeout 900 python tools/table1.py C3 > gpurun_out/table1_c3.log 2>&1; echo b=$?
