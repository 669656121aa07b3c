"""Time steps a1-a3 on one config on the GPU (kernel-class breakdown)."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
spec = hi.CONFIGS[name]
dev = "cuda" if spec.L > 4096 else "cpu"
t = time.time()
Kb = hi.make_kbar(name, 0, device=dev).to("cuda")
torch.cuda.synchronize()
print("gen s", time.time() - t, flush=True)
ctx = hf.Context(0)
for rep in range(2):
    K = Kb.clone()
    ctx.set_profiling(rep == 1)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    q = hf.hf_scale(ctx, K)
    e1.record()
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, nb=nb)
    e2.record()
    torch.cuda.synchronize()
    print(json.dumps({"cfg": name, "rep": rep, "scale_ms": e0.elapsed_time(e1), "factor_ms": e1.elapsed_time(e2),
                      "N": lf.N, "n2": lf.n2, "n2_tau_only": lf.n2_tau_only}), flush=True)
for c in ("scale", "chain", "trailing", "other"):
    print(c, ctx.kernel_stats(c))
L = spec.L
F1 = sum((L - k - 1) * (L - k) for k in range(lf.N))
ms, n = ctx.kernel_stats("trailing")
print("trailing TFLOP/s", F1 / (ms * 1e-3) / 1e12 if ms else None)
cms, cn = ctx.kernel_stats("chain")
print("chain us/pivot", cms * 1e3 / max(lf.N, 1))
