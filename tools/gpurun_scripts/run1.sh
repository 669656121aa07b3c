set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python tools/probe_gcr.py C2 60 64 > gpurun_out/probe_gcr64.log 2>&1; echo probe=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
