for nb in 128 160 192; do timeout 300 python tools/probe_stage1.py C2 $nb > gpurun_out/p89_$nb.log 2>&1; echo "$nb $(grep -E '^chain|^trailing|^other' gpurun_out/p89_$nb.log | tr '\n' ' ')"; done
