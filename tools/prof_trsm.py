"""Time the FP32 preconditioner (k_trsm pair) at a config's sizes (GPU)."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import hf_inputs as hi
from paper_2208_01907_b200 import hf

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
ncol = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
spec = hi.CONFIGS[name]
Kb = hi.make_kbar(name, 0, device="cuda" if spec.L > 4096 else "cpu").cuda()
ctx = hf.Context(0)
hf.hf_scale(ctx, Kb)
lf = hf.hf_factor_lowprec(ctx, Kb, tau=spec.tau, n_min=spec.n_min)
R = torch.randn(ncol, lf.L, dtype=torch.float64, device="cuda").T
W = hf.hf_precond_apply(ctx, lf, R)
torch.cuda.synchronize()
ctx.set_profiling(True)
ctx.kernel_stats("trsm")
t0 = time.perf_counter()
for _ in range(reps):
    hf.hf_precond_apply(ctx, lf, R, W)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
ms, n = ctx.kernel_stats("trsm")
N = lf.N
fl = 2.0 * N * N * ncol
print(json.dumps({"cfg": name, "N": N, "ncol": ncol, "wall_ms_per_apply": wall * 1e3, "trsm_ms_per_apply": ms / reps,
                  "tflops": fl / (ms / reps * 1e-3) / 1e12}))
