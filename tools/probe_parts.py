"""Stage-1 timing of the column-partitioned (multi-GPU) algorithm emulated on one GPU:
chain (replicated on every rank) and trailing (split over the ranks) classes, and the
projected per-rank time chain + trailing / G (peer reads of the pivot column not
included: they are local here).  python tools/probe_parts.py C2 8"""
import sys, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(name, 0, device="cuda" if spec.L > 4096 else "cpu").cuda()
ctx = hf.Context(0)
out = {}
prev = {c: 0.0 for c in ("chain", "trailing", "other")}
for parts in (0, G):
    hf.hf_set_stage1_partitions(ctx, parts)
    for rep in range(2):
        K = Kb.clone()
        hf.hf_scale(ctx, K)
        ctx.set_profiling(rep == 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)
        e1.record()
        torch.cuda.synchronize()
        del lf, K
    tot = {c: ctx.kernel_stats(c)[0] for c in ("chain", "trailing", "other")}
    st = {c: tot[c] - prev[c] for c in tot}     # kernel_stats is cumulative
    prev = tot
    out[f"parts={parts}"] = {"factor_ms": e0.elapsed_time(e1), **st,
                             "projected_per_rank_ms": st["chain"] + st["other"] + st["trailing"] / max(parts, 1)}
    ctx.set_profiling(False)
print(json.dumps(out))
