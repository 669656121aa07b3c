for g in 1 2 4 8 16 32; do echo "G=$g $(HF_HARD_CTAS=$g timeout 300 python tools/probe_config.py C2 2 2>&1 | grep -o "'hard': ([0-9.]*" )"; done
for g in 16 32 64 148; do echo "C3 G=$g $(HF_HARD_CTAS=$g timeout 600 python tools/probe_config.py C3 1 2>&1 | grep -o "'hard': ([0-9.]*" )"; done
