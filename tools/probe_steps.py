"""Per-step host/device timing of the bench step (find one-off stalls)."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf
spec = hi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
prof = len(sys.argv) > 2 and sys.argv[2] == "prof"
Kb = hi.make_kbar(spec, 0, device="cuda").contiguous()
K = torch.empty_like(Kb)
ctx = hf.Context(0, torch.cuda.current_stream())
ctx.set_profiling(prof)
cls = ("chain", "trailing", "dgemm", "trsm", "gram", "hard", "other", "scale")
prev = {c: ctx.kernel_stats(c)[0] for c in cls}
for it in range(8):
    K.copy_(Kb)
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    hf.hf_scale(ctx, K); t.append(time.perf_counter())
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min); t.append(time.perf_counter())
    hy, info, _ = hf.hf_schur_gcr(ctx, K, lf); t.append(time.perf_counter())
    kd = hf.hf_factor_hard(ctx, hy); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    cur = {c: ctx.kernel_stats(c)[0] for c in cls}
    print(json.dumps({"it": it, "host_ms": [round((t[i + 1] - t[i]) * 1e3, 1) for i in range(5)],
                      "kern_ms": {c: round(cur[c] - prev[c], 1) for c in cls}}), flush=True)
    prev = cur
