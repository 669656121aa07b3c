python -c "from paper_2208_01907_b200 import build; build.build()" || exit 1
python tools/prof_trsm.py C2 256 2 > gpurun_out/p30.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trsm -s 2 -c 1 -o gpurun_out/prof_trsm2 python tools/prof_trsm.py C2 256 1 > gpurun_out/ncu30.log 2>&1; echo n=$?
