"""Block GCR residual trace + kernel-class breakdown on one config (GPU)."""
import os, sys, time, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf
os.environ.setdefault("HF_GCR_DEBUG", "1")
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 40
n_min = int(sys.argv[3]) if len(sys.argv) > 3 else None
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(name, 0, device="cuda" if spec.L > 4096 else "cpu").cuda()
ctx = hf.Context(0)
for rep in range(2):
    K = Kb.clone()
    t = time.time()
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min if n_min is None else n_min)
    t1 = time.time()
    ctx.set_profiling(rep == 1)
    hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, max_iter=maxit, accept_failure=True)
    torch.cuda.synchronize()
    print(json.dumps({"rep": rep, "n2": lf.n2, "factor_s": t1 - t, "gcr_s": time.time() - t1, "iters": info.iters,
                      "rec": info.max_rel_res_recursive, "true": info.max_rel_res_true, "status": info.status}), flush=True)
for c in ("dgemm", "trsm", "other", "hard"):
    print(c, ctx.kernel_stats(c))
