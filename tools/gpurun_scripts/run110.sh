for g in 32 64 128 148; do echo "G=$g $(HF_HARD_CTAS=$g timeout 300 python tools/probe_config.py C2 2 2>&1 | grep -o "'hard': ([0-9.]*" )"; done
