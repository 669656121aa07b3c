"""Multi-GPU correctness check of the distributed stage 1 (k_dist.cu) and the
sharded stage 2, one process per GPU (run under torch.distributed.run, NCCL):
every rank factors the SAME matrix across all ranks; each rank also factors it
alone on its GPU (a non-distributed context) and Pi, Lambda_2, D and L must be
bit-identical [R8]; the allgathered S22 must be identical on every rank.
Rank 0 prints one JSON line; the exit code is non-zero on any mismatch.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/dist_check.py [config]
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import hf_inputs as hi  # noqa: E402
from paper_2208_01907_b200 import hf  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "P2048"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    idb = [hf.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(idb, src=0)
    ctx = hf.Context(local, nccl_id=idb[0], rank=rank, nranks=world)
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, 0, device="cuda" if spec.L > 4096 else "cpu").cuda()
    hf.hf_scale(ctx, Kb)
    lf = hf.hf_factor_lowprec(ctx, Kb, tau=spec.tau, n_min=spec.n_min)
    perm, D, Lf = lf.export()
    c1 = hf.Context(local)
    lf1 = hf.hf_factor_lowprec(c1, Kb, tau=spec.tau, n_min=spec.n_min)
    p1, D1, L1 = lf1.export()
    ok1 = bool(np.array_equal(perm, p1) and np.array_equal(D, D1) and torch.equal(Lf, L1))
    hy, info, S = hf.hf_schur_gcr(ctx, Kb, lf, want_S22_host=True)
    torch.cuda.synchronize()
    allS = [None] * world
    dist.all_gather_object(allS, S)
    oks = [None] * world
    dist.all_gather_object(oks, ok1)
    same_S = all(np.array_equal(allS[0], x) for x in allS)
    if rank == 0:
        print(json.dumps({"config": name, "world": world, "stage1_bitwise_vs_one_gpu": oks,
                          "S22_identical_on_ranks": same_S, "n2": lf.n2, "gcr_iters": info.iters,
                          "gcr_true_rel_res": info.max_rel_res_true}), flush=True)
    hy.close()
    lf.close()
    lf1.close()
    c1.close()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    if not (all(oks) and same_S):
        sys.exit(1)


if __name__ == "__main__":
    main()
