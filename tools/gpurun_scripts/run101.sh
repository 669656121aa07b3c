timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t101.log 2>&1; echo t=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke101.log 2>&1; echo s=$?
timeout 900 python bench.py > gpurun_out/bench101.log 2>&1; echo b=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref101.log 2>&1; echo r=$?
