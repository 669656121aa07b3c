"""Stage 1 with the persistent trailing kernel vs k_trailing_c: bitwise comparison of
perm, D and L at a size where the persistent kernel runs (GPU)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(name, 0, device="cuda").cuda()
ctx = hf.Context(0)
hf.hf_scale(ctx, Kb)
out = {}
for mode in ("0", "1"):
    os.environ["HF_TRAIL_PERSIST"] = mode
    lf = hf.hf_factor_lowprec(ctx, Kb, tau=spec.tau, n_min=spec.n_min)
    perm, D, Lf = lf.export()
    out[mode] = (lf.N, perm, D, Lf.clone())
    lf.close()
a, b = out["0"], out["1"]
print("N", a[0], b[0], "perm eq", np.array_equal(a[1], b[1]), "D eq", np.array_equal(a[2], b[2]))
if a[0] == b[0]:
    d = (a[3] != b[3])
    nz = torch.nonzero(d)
    print("L mismatches", int(d.sum()), nz[:10].tolist())
