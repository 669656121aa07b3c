"""Run the whole path twice on the same input and compare everything bitwise."""
import sys, json
import numpy as np
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(spec, 0, device="cuda" if spec.kind == "planted" and spec.L > 4096 else "cpu").cuda()
ctx = hf.Context(0)
res = []
for rep in range(3):
    K = Kb.clone()
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
    perm, D, Lf = lf.export()
    hy, info, S22 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True)
    W = hf.hf_precond_apply(ctx, lf, K[:, :64].T.contiguous().T.contiguous().T if False else torch.randn(64, spec.L, generator=torch.Generator().manual_seed(1), dtype=torch.float64).cuda().T)
    kd = hf.hf_factor_hard(ctx, hy)
    res.append((perm.copy(), D.copy(), Lf.cpu().numpy(), S22.copy(), W.cpu().numpy(), kd, info.iters))
    hy.close(); lf.close()
out = {"cfg": name}
for q, nm in enumerate(["perm", "D", "L", "S22", "precond", "kernel_dim", "iters"]):
    a, b, c = res[0][q], res[1][q], res[2][q]
    if isinstance(a, np.ndarray):
        out[nm] = bool(np.array_equal(a, b) and np.array_equal(a, c))
        if not out[nm]:
            out[nm + "_maxdiff"] = float(max(np.abs(a - b).max(), np.abs(a - c).max()))
    else:
        out[nm] = [a, b, c]
print(json.dumps(out))
