python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
python tools/prof_trsm.py C2 256 5 > gpurun_out/trsm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trsm -c 2 -o gpurun_out/prof_trsm python tools/prof_trsm.py C2 256 1 > gpurun_out/ncu_trsm.log 2>&1; echo ncu=$?
