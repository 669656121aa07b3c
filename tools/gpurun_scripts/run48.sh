python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke48.log 2>&1; echo plain=$?
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck48.log 2>&1; echo memcheck=$?
