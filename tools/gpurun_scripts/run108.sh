for v in 0 3000 6000 9000 0; do echo "STAGGER=$v $(HF_TRAIL_STAGGER=$v timeout 300 python tools/probe_stage1.py C2 2>&1 | grep -E '^trailing \(|^chain \(' | tr '\n' ' ')"; done
