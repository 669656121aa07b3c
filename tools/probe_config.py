"""Run the whole GPU path on one config and print its statistics (GPU)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = hi.CONFIGS[name]
t0 = time.time()
Kb = hi.make_kbar(spec, 0, device="cuda" if spec.kind == "planted" and spec.L > 4096 else "cpu").cuda()
torch.cuda.synchronize()
print("gen s", round(time.time() - t0, 1), flush=True)
ctx = hf.Context(0)
K = torch.empty_like(Kb)
for rep in range(reps):
    ctx.set_profiling(rep == reps - 1)
    K.copy_(Kb)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    hf.hf_scale(ctx, K); ev[1].record()
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min); ev[2].record()
    hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, accept_failure=True); ev[3].record()
    kd = hf.hf_factor_hard(ctx, hy); ev[4].record()
    torch.cuda.synchronize()
    out = {"cfg": name, "rep": rep, "L": spec.L, "N": lf.N, "n2": lf.n2, "n2_tau_only": lf.n2_tau_only,
           "gcr_iters": info.iters, "status": info.status, "rec": info.max_rel_res_recursive,
           "true": info.max_rel_res_true, "kernel_dim": kd,
           "stage_ms": [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(4)]}
    print(json.dumps(out), flush=True)
    if rep < reps - 1:
        hy.close(); lf.close()
print({c: ctx.kernel_stats(c) for c in ("scale", "chain", "trailing", "dgemm", "trsm", "gram", "hard", "other")})
# solve with the manufactured RHS (scaled system)
xs = hi.manufactured_x(spec.L, device="cuda")
b = (K @ xs)
x, sinfo = hf.hf_solve(ctx, hy, b)
r = (K @ x - b).abs().max() / b.abs().max()
print(json.dumps({"solve_iters": sinfo.iters, "rho_manufactured": float(r)}))
