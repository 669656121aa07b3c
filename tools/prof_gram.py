"""Time hf_gram_inverse (the Gram inverse of Alg. 5) at size n (GPU)."""
import sys, json
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2208_01907_b200 import hf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rng = np.random.default_rng(0)
B = rng.standard_normal((4 * n, n))
M = torch.from_numpy(np.asfortranarray(B.T @ B)).cuda()
ctx = hf.Context(0)
Mi, bd = hf.hf_gram_inverse(ctx, M)
ctx.set_profiling(True)
for _ in range(reps):
    hf.hf_gram_inverse(ctx, M)
ms, cnt = ctx.kernel_stats("gram")
err = float(np.linalg.norm(Mi.cpu().numpy() @ (B.T @ B) - np.eye(n)))
print(json.dumps({"n": n, "gram_ms_per_call": ms / reps, "launches": cnt, "breakdown": bd, "res": err}))
