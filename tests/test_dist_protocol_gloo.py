"""The DATA FLOW of the distributed stage 1 (k_dist.cu) on
real ranks: world-size 2 and 3 torch.distributed/gloo processes on the CPU, each
holding only what its GPU would hold, exchanging only what the GPU ranks
exchange:

  * ownership: original index j belongs to rank (j // CB) % G; a rank stores
    the lower-triangle entries v_IJ (pos I >= pos J) of the indices J it owns;
  * per pivot: every rank's best key over its own chain rows (|d| bits, smallest
    position wins ties, sign) -> all_reduce(MAX) (the allreduce(max) of the
    north_star; on the GPU one tagged store into every rank's slot array);
    the pivot column's entries below the pivot and the pivot row's in-panel
    values come from the pivot's owner (broadcast from it; on the GPU a peer
    read); entries above the pivot are row P of the rank's own columns;
  * per panel: the panel's s values of all rows gathered from their owners
    (all_gather; on the GPU k_dgather), each rank updates its own columns.

The arithmetic is the canonical FP32 one ([R6]-[R8], one correctly rounded
fmaf per pivot per entry, emulated exactly with tests/exact_ldlt.py's binary32
rounding), so Pi, D and the factor must equal the ORACLE's bit for bit: this
pins the distribution logic (ownership, key encoding and tie rule, piece
assembly, panel broadcast) independently of the CUDA kernels."""
import math
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.exact_ldlt import f32, fmaf_exact

POS_MAX = 0x1FFFF


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _key(d: float, pos: int) -> int:
    ab = struct.unpack("<I", struct.pack("<f", abs(d)))[0]
    return (ab << 32) | ((POS_MAX - pos) << 15) | ((1 if d < 0 else 0) << 14) | 1


def _rank_factor(K, tau, nb, CB, rank, world):
    """One rank's share of the distributed stage 1 (tau rule only)."""
    L = K.shape[0]
    own = lambda j: (j // CB) % world == rank   # noqa: E731
    V = {}                                       # (I, J) -> v_IJ for own J, I >= J
    for J in range(L):
        if own(J):
            for I in range(J, L):
                V[(I, J)] = f32(K[I, J])
    active = list(range(L))                      # position order == original order
    dg = {I: V[(I, I)] for I in range(L) if own(I)}
    piv, D, Lcol = [], [], []
    dprev = None
    stopped = False
    while active and not stopped:
        pos = {I: p for p, I in enumerate(active)}
        panel = []                               # (P, d, sigma, {I: s_I}) of this panel
        S = {}                                   # own rows: I -> [s_I^t]
        done = set()
        for t in range(min(nb, len(active))):
            best = 0
            for I in active:
                if own(I) and I not in done:
                    best = max(best, _key(dg[I], pos[I]))
            kb = torch.tensor([best], dtype=torch.int64)
            dist.all_reduce(kb, op=dist.ReduceOp.MAX)
            bk = int(kb.item())
            absd = struct.unpack("<f", struct.pack("<I", (bk >> 32) & 0xFFFFFFFF))[0]
            d = -absd if (bk >> 14) & 1 else absd
            P = active[POS_MAX - ((bk >> 15) & POS_MAX)] if bk else None
            if bk == 0 or (dprev is None and absd == 0.0) or \
                    (dprev is not None and abs(d) < tau * abs(dprev)):
                stopped = True
                break
            owner = (P // CB) % world
            # the pivot's owner sends the pivot row's in-panel values and its column below P
            msg = [None]
            if rank == owner:
                msg = [([S.get(P, [])[u] for u in range(t)],
                        {I: V[(I, P)] for I in active if pos[I] > pos[P] and I not in done})]
            dist.broadcast_object_list(msg, src=owner)
            sP, colP = msg[0]
            r = f32(math.sqrt(absd))
            sg = 1.0 if d > 0 else -1.0
            Lk = {}
            for I in active:
                if not own(I) or I in done or I == P:
                    continue
                v = colP[I] if pos[I] > pos[P] else V[(P, I)]   # column P on its owner / row P of own column
                c = v
                for u in range(t):                             # [R8] in-panel pivots in order
                    c = fmaf_exact(-panel[u][2] * S[I][u], sP[u], c)
                s = f32(c / r)
                S.setdefault(I, []).append(s)
                Lk[I] = f32(c / d)
                dg[I] = fmaf_exact(-sg * s, s, dg[I])
            if own(P):
                S.setdefault(P, [])
            done.add(P)
            panel.append((P, d, sg))
            piv.append(P)
            D.append(d)
            Lcol.append(Lk)
            dprev = d
        # the panel broadcast: every row's s values from its owner, then the own-column update
        allS = [None] * world
        dist.all_gather_object(allS, {I: v for I, v in S.items() if I not in done})
        Sall = {}
        for part in allS:
            Sall.update(part)
        nt = len(panel)
        for P in done:
            active.remove(P)
        for J in active:
            if not own(J):
                continue
            for I in active:
                if pos[I] >= pos[J]:
                    v = V[(I, J)]
                    for u in range(nt):
                        v = fmaf_exact(-panel[u][2] * Sall[I][u], Sall[J][u], v)
                    V[(I, J)] = v
    allL = [None] * world
    dist.all_gather_object(allL, Lcol)
    Lfull = [{} for _ in piv]
    for part in allL:
        for k, col in enumerate(part):
            Lfull[k].update(col)
    return piv, D, Lfull


def _worker(rank, world, port, K, tau, nb, CB, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = _rank_factor(K, tau, nb, CB, rank, world)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,nb,CB,seed", [(2, 3, 2, 0), (3, 4, 1, 1), (2, 5, 3, 2)])
def test_distributed_stage1_protocol_gloo(world, nb, CB, seed):
    import hf_inputs as hi
    import oracle
    Kb = hi.make_kbar("C0", seed).numpy()[:22, :22].copy()
    Kb = 0.5 * (Kb + Kb.T)
    K, _ = oracle.scale(Kb)
    tau = 1e-2
    F = oracle.factor_lowprec(K, tau)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, K, tau, nb, CB, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = out
    for p in ps:
        p.join(timeout=60)
    piv, D, Lfull = res[0]
    for r in range(1, world):                    # identical on every rank
        assert res[r][0] == piv and res[r][1] == D
    assert len(piv) == F.Ntau
    assert np.array_equal(np.array(piv, dtype=np.int64), F.perm[:F.Ntau])            # Pi, bitwise
    assert np.array_equal(np.array(D, dtype=np.float32), F.D[:F.Ntau])               # D, bitwise
    rank_of = {P: k for k, P in enumerate(piv)}
    for k, col in enumerate(Lfull):              # the factor, bitwise on the Lambda_1 rows
        for I, v in col.items():
            if I in rank_of and rank_of[I] < F.N and k < F.N:
                assert np.float32(v) == F.Lfac[rank_of[I], k]
