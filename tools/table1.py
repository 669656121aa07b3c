"""Table 1 analog on the GPU: the hybrid factorization with the
(float, double) pair (the north_star) against the pure-double run (stage 1 in
FP64, prec = 64) and the (double, double-double) pair (NEXT-1) on one config:
per-stage times, |Lambda_2| (tau-only and final), block-GCR iterations,
residual of the manufactured solution (not for the dd pair, whose
solve is not built).
    python tools/table1.py C2"""
import sys, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(spec, 0, device="cuda" if spec.kind == "planted" and spec.L > 4096 else "cpu").cuda()
ctx = hf.Context(0)
xs = hi.manufactured_x(spec.L, device="cuda")
out = {"cfg": name, "L": spec.L}
K = torch.empty_like(Kb)
for prec in (32, 64):
    for rep in range(2):
        if rep == 1:
            hy.close()
            lf.close()
        K.copy_(Kb)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        hf.hf_scale(ctx, K); ev[1].record()
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, prec=prec); ev[2].record()
        hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, accept_failure=True); ev[3].record()
        kd = hf.hf_factor_hard(ctx, hy); ev[4].record()
        torch.cuda.synchronize()
    b = K @ xs
    x, _ = hf.hf_solve(ctx, hy, b)
    rho = float((K @ x - b).abs().max() / b.abs().max())
    err = float((x - xs).abs().max() / xs.abs().max())
    out[f"fp{prec}"] = {"stage_ms": [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(4)],
                        "total_ms": round(ev[0].elapsed_time(ev[4]), 2), "N": lf.N, "n2": lf.n2,
                        "n2_tau_only": lf.n2_tau_only, "gcr_iters": info.iters,
                        "gcr_true_rel_res": info.max_rel_res_true, "kernel_dim": kd,
                        "rho_manufactured": rho, "x_err_inf_rel": err}
    hy.close()
    lf.close()
# the (double, double-double) pair: FP64 stage 1, double-double stages 2-3 (no solve)
for rep in range(2):
    K.copy_(Kb)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    hf.hf_scale(ctx, K); ev[1].record()
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, prec=64); ev[2].record()
    hy, info, _ = hf.hf_schur_gcr_dd(ctx, K, lf, accept_failure=True); ev[3].record()
    kd = hf.hf_factor_hard(ctx, hy, eps_ker=1e-20); ev[4].record()
    torch.cuda.synchronize()
    if rep == 1:
        out["fp64_dd"] = {"stage_ms": [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(4)],
                          "total_ms": round(ev[0].elapsed_time(ev[4]), 2), "N": lf.N, "n2": lf.n2,
                          "gcr_iters": info.iters, "gcr_true_rel_res": info.max_rel_res_true, "kernel_dim": kd}
    hy.close()
    lf.close()
print(json.dumps(out))
