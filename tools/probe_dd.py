"""NEXT-1 (double, double-double) pair: accuracy against the exact Schur
complement on small cases, and per-stage timing at a full config (GPU).
    python tools/probe_dd.py [C2]"""
import sys, json, time
import numpy as np
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from hf_inputs.configs import ConfigSpec
from oracle import exact
from paper_2208_01907_b200 import hf

ctx = hf.Context(0)
small = [ConfigSpec("P48", "planted", 48, n_min=3, n_hard=3, u_hard=(-10.0, -8.0)),
         ConfigSpec("P64", "planted", 64, n_min=4, n_hard=4, u_hard=(-12.0, -6.0)),
         ConfigSpec("S6", "saddle", 2 * 6 * 6 + 2 * 3 * 3, grid=6, jump=1e4),
         ConfigSpec("N8", "neumann", 64, grid=8, n_incl=1, incl_size=2)]
for spec in small:
    K = hi.make_kbar(spec, 0).to("cuda")
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, prec=64)
    perm, _, _ = lf.export64()
    lam1, lam2 = [int(i) for i in perm[:lf.N]], [int(i) for i in perm[lf.N:]]
    Kh = K.cpu().numpy()
    Sx = exact.schur(Kh, lam1, lam2)
    smax = max(abs(float(v)) for r in Sx for v in r)
    hyd, infd, (Sh, Sl) = hf.hf_schur_gcr_dd(ctx, K, lf, want_S22_host=True)
    hy6, inf6, S6 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True)
    kd_dd = hf.hf_factor_hard(ctx, hyd, eps_ker=1e-20)
    kd_64 = hf.hf_factor_hard(ctx, hy6, eps_ker=1e-10)
    print(json.dumps({"cfg": spec.name, "L": spec.L, "n2": lf.n2, "dd_iters": infd.iters, "dd_true_res": infd.max_rel_res_true,
                      "rel_err_dd": exact.rel_err(Sx, Sh, Sl), "rel_err_fp64": exact.rel_err(Sx, S6, np.zeros_like(S6)),
                      "fp64_iters": inf6.iters, "kd_dd": kd_dd, "kd_fp64": kd_64, "exact_kernel": lf.n2 - exact.rank(Sx),
                      "max_abs_S": smax}), flush=True)
    hyd.close(); hy6.close(); lf.close()

if len(sys.argv) > 1:
    name = sys.argv[1]
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(spec, 0, device="cuda" if spec.kind == "planted" and spec.L > 4096 else "cpu").cuda()
    K = torch.empty_like(Kb)
    for rep in range(2):
        ctx.set_profiling(rep == 1)
        K.copy_(Kb)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        hf.hf_scale(ctx, K); ev[1].record()
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, prec=64); ev[2].record()
        hy, info, _ = hf.hf_schur_gcr_dd(ctx, K, lf, accept_failure=True); ev[3].record()
        kd = hf.hf_factor_hard(ctx, hy, eps_ker=1e-20); ev[4].record()
        torch.cuda.synchronize()
        print(json.dumps({"cfg": name, "rep": rep, "pair": "(double, double-double)", "N": lf.N, "n2": lf.n2,
                          "gcr_iters": info.iters, "true_rel_res": info.max_rel_res_true, "status": info.status,
                          "kernel_dim": kd, "stage_ms": [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(4)],
                          "total_ms": round(ev[0].elapsed_time(ev[4]), 2)}), flush=True)
        hy.close(); lf.close()
    print({c: ctx.kernel_stats(c) for c in ("scale", "chain", "trailing", "ddgemm", "trsm", "gram", "hard", "other")})
