python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke42.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputests42.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench42.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench42_ref.log 2>&1; echo ref=$?
