"""Fig. 2 on the GPU at a config's size: iterations, final residual
and time of IR (Alg. 3), GCR per column (Alg. 4) and block GCR (Alg. 5) for the
config's K12 right-hand sides (the systems block GCR solves in Alg. 1 step 3).
    python tools/fig2.py C2 [ncol]"""
import sys, json, time
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(spec, 0, device="cuda" if spec.kind == "planted" and spec.L > 4096 else "cpu").cuda()
ctx = hf.Context(0)
hf.hf_scale(ctx, Kb)
lf = hf.hf_factor_lowprec(ctx, Kb, tau=spec.tau, n_min=spec.n_min)
perm, _, _ = lf.export(with_L=False)
ncol = int(sys.argv[2]) if len(sys.argv) > 2 else min(16, lf.n2)
lam2 = torch.from_numpy(perm[lf.N:lf.N + ncol]).cuda()
B = Kb[:, lam2].contiguous().T.contiguous().T        # K12 columns, column-major (L, ncol)
out = {"cfg": name, "L": spec.L, "N": lf.N, "ncol": ncol}
for m in ("bgcr", "gcr", "ir"):
    torch.cuda.synchronize()
    t = time.perf_counter()
    X, it, hist, st = hf.hf_krylov_solve(ctx, Kb, lf, B, m, max_iter=100, accept_failure=True)
    torch.cuda.synchronize()
    out[m] = {"iters": it, "converged": st == 0, "final_rel_res": float(hist[-1]),
              "ms": (time.perf_counter() - t) * 1e3, "history": [float(h) for h in hist[:12]]}
print(json.dumps(out))
