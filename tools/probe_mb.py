"""NEXT-4: multi-block postponing at a full config (GPU): ordering, stage 1 and
Alg. 1 with per-stage times, |Lambda_2| against the single-sequence rule.
    python tools/probe_mb.py C3 7"""
import sys, json, time
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 7
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(spec, 0).cuda()
ctx = hf.Context(0)
K = Kb.clone()
hf.hf_scale(ctx, K)
t0 = time.time()
blk, nblk = hf.hf_nd_blocks(ctx, K, levels)
t_nd = time.time() - t0
for rep in range(2):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    lf = hf.hf_factor_lowprec_blocks(ctx, K, blk, nblk, tau=spec.tau, n_min=spec.n_min, n_extra=4); ev[1].record()
    hy, info, _ = hf.hf_schur_gcr(ctx, K, lf, accept_failure=True); ev[2].record()
    kd = hf.hf_factor_hard(ctx, hy); ev[3].record()
    torch.cuda.synchronize()
    lf1 = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, n_extra=4)
    out = {"cfg": name, "rep": rep, "levels": levels, "nblk": nblk, "nd_s": round(t_nd, 3), "L": spec.L, "N": lf.N,
           "n2": lf.n2, "n2_tau_only": lf.n2_tau_only, "single_sequence_n2": lf1.n2, "gcr_iters": info.iters,
           "true_rel_res": info.max_rel_res_true, "kernel_dim": kd,
           "stage_ms": [round(ev[i].elapsed_time(ev[i + 1]), 2) for i in range(3)]}
    print(json.dumps(out), flush=True)
    hy.close(); lf.close(); lf1.close()
