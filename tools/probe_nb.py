"""Stage-1 time at C2 for several panel widths nb (GPU)."""
import sys, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(name, 0, device="cuda").cuda()
ctx = hf.Context(0)
K = torch.empty_like(Kb)
for nb in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["128", "160", "192", "224"])]:
    ts = []
    for rep in range(3):
        K.copy_(Kb)
        hf.hf_scale(ctx, K)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, nb=nb)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        lf.close()
    print(json.dumps({"cfg": name, "nb": nb, "stage1_ms": min(ts[1:])}), flush=True)
