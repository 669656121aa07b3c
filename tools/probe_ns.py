"""NEXT-3: the nonsymmetric path at a full size (GPU): per-stage times and statistics.
    python tools/probe_ns.py T96"""
import sys, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "T96"
spec = hi.CONFIGS[name]
Kb = hi.colmajor(hi.make_kbar(spec, 0)).cuda()
ctx = hf.Context(0)
K = torch.empty_like(Kb)
for rep in range(2):
    ctx.set_profiling(rep == 1)
    K.copy_(Kb)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    hf.hf_scale_full(ctx, K); ev[1].record()
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, nonsym=True); ev[2].record()
    hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, accept_failure=True); ev[3].record()
    kd = hf.hf_factor_hard(ctx, hy); ev[4].record()
    torch.cuda.synchronize()
    xs = hi.manufactured_x(spec.L, device="cuda")
    Km = K.T            # the matrix (K's memory is column-major)
    b = Km @ xs
    x, sinfo = hf.hf_solve(ctx, hy, b)
    rho = float((Km @ x - b).abs().max() / b.abs().max())
    print(json.dumps({"cfg": name, "rep": rep, "L": spec.L, "N": lf.N, "n2": lf.n2, "n2_tau_only": lf.n2_tau_only,
                      "gcr_iters": info.iters, "true_rel_res": info.max_rel_res_true, "kernel_dim": kd,
                      "rho_manufactured": rho, "stage_ms": [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(4)],
                      "total_ms": round(ev[0].elapsed_time(ev[4]), 2)}), flush=True)
    hy.close(); lf.close()
print({c: ctx.kernel_stats(c) for c in ("scale", "chain", "trailing", "dgemm", "trsm", "gram", "hard", "other")})
