"""Host-side logic of the multi-GPU paths on CPU with torch.distributed/gloo,
world_size 2 (the GPU box has one GPU):
  * the stage-2 right-hand-side sharding plan of libhf (hf_shard_cols, a host
    function of the C-ABI) -- every rank computes its own slice, the gathered
    slices must tile [0, n2) exactly, in rank order, balanced to one column;
  * bench.py's max-over-ranks timing reduction (the contract's rule);
  * replica seeding (every rank a different matrix in replica mode, the same
    matrix in shard mode)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        from paper_2208_01907_b200 import hf
        out = {}
        for n2 in (0, 1, 3, 64, 256, 1344, 1345):
            mine = hf.hf_shard_cols(n2, world, rank)
            allp = [None] * world
            dist.all_gather_object(allp, mine)
            out[n2] = allp
        out["max"] = bench.max_over_ranks(float(10 * rank + 1))
        out["sum"] = bench.sum_over_ranks(float(10 * rank + 1))   # replicas: whole-job flops
        for L in (1, 300, 16384, 23040):
            cols = hf.hf_stage1_partition(L, world, rank)
            allc = [None] * world
            dist.all_gather_object(allc, cols.tolist())
            out[("s1", L)] = allc
        seeds = [None] * world
        dist.all_gather_object(seeds, [0 + rank, 0])     # replicas: seed + rank; shard: seed
        out["seeds"] = seeds
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))


@pytest.mark.timeout(300)
def test_shard_plan_and_rank_max_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=240)
        assert err is None, err
        res[r] = out
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert res[r]["max"] == 11.0
        assert res[r]["sum"] == 12.0
        for n2 in (0, 1, 3, 64, 256, 1344, 1345):
            sl = res[r][n2]
            assert sl == res[0][n2]                       # every rank sees the same plan
            assert sl[0][0] == 0 and sl[-1][1] == n2      # tiles [0, n2) ...
            for a, b in zip(sl, sl[1:]):
                assert a[1] == b[0]                       # ... contiguously, in rank order
            w = [c1 - c0 for c0, c1 in sl]
            assert max(w) - min(w) <= 1                   # balanced
        for L in (1, 300, 16384, 23040):
            allc = res[r][("s1", L)]
            flat = sorted(c for part in allc for c in part)
            assert flat == list(range(L))                                      # every column exactly once
            assert all(all((c // 128) % world == g for c in part) for g, part in enumerate(allc))
            sizes = [len(part) for part in allc]
            assert max(sizes) - min(sizes) <= 128                              # balanced to one block
    seeds = res[0]["seeds"]
    assert seeds[0][0] != seeds[1][0] and seeds[0][1] == seeds[1][1]


def test_shard_plan_single_rank():
    from paper_2208_01907_b200 import hf
    assert hf.hf_shard_cols(256, 1, 0) == (0, 256)
    with pytest.raises(hf.HFError):
        hf.hf_shard_cols(10, 2, 2)
