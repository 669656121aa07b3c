"""DESIGN.md [R5] evidence: the ORACLE (plain CPU implementation) on C2 with a
given postponement floor n_min (default 64, the planted count) and max_iter
(default 100): block-GCR residual history (max over columns, recursive and the
true residual at exit).  Input generated on the GPU (hf_inputs, the same bytes
the CUDA path sees), everything else on the host.  Optionally the CUDA path on
the same matrix for comparison (--gpu).

    python tools/oracle_nmin.py [n_min] [max_iter] [--gpu] > gpurun_out/oracle_nmin64.log
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hf_inputs as hi  # noqa: E402
import oracle  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n_min = int(args[0]) if args else 64
    max_iter = int(args[1]) if len(args) > 1 else 100
    spec = hi.CONFIGS["C2"]
    import torch
    Kb = hi.make_kbar("C2", 0, device="cuda" if torch.cuda.is_available() else "cpu").cpu()
    if "--gpu" in sys.argv:
        from paper_2208_01907_b200 import hf
        with hf.Context(0) as ctx:
            Kd = Kb.to("cuda")
            hf.hf_scale(ctx, Kd)
            lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=n_min)
            hy, info, _ = hf.hf_schur_gcr(ctx, Kd, lf, max_iter=max_iter, accept_failure=True)
            print(json.dumps({"side": "cuda", "n_min": n_min, "n2": lf.n2, "iters": info.iters,
                              "rec": info.max_rel_res_recursive, "true": info.max_rel_res_true,
                              "status": info.status}), flush=True)
            del hy, lf, Kd
    t0 = time.time()
    Ko, _ = oracle.scale(Kb.numpy())
    del Kb
    F = oracle.factor_lowprec(Ko, spec.tau, n_min=n_min)
    t1 = time.time()
    print(json.dumps({"side": "oracle", "stage1_s": round(t1 - t0, 1), "N": F.N, "Ntau": F.Ntau,
                      "n2": F.n2}), flush=True)
    K11, K12, _, _ = oracle.extract_blocks(Ko, F)
    del Ko
    X, info = oracle.block_gcr(K11, F, K12, max_iter=max_iter, raise_on_fail=False)
    hist = [float(h.max()) for h in info.history]
    print(json.dumps({"side": "oracle", "n_min": n_min, "iters": info.iters, "converged": info.converged,
                      "rec": info.max_rel_res_recursive, "true": info.max_rel_res_true,
                      "gcr_s": round(time.time() - t1, 1), "history_max_rel_res": hist}), flush=True)


if __name__ == "__main__":
    main()
