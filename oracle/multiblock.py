"""oracle.multiblock -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

NEXT-4: multi-block threshold postponing along a
nested-dissection elimination tree (sec. 2.2):

  nd_blocks       nested-dissection ordering ("m-level bi-section tree"):
                  recursive level-structure bisection of the matrix graph,
                  blocks numbered in post-order (children before their
                  separator), 2^m - 1 blocks for m levels
  factor_blocks   per-block FP32 factorization with the tau-test against the
                  previously accepted pivot ([R21]),
                  the postponed entries collected in Lambda_0 and factored in a
                  final pass, floor and n-entry enlargement (oracle_factor_blocks_f32)
  hybrid_factor   Alg. 1 with that stage 1 (steps 2-5 as oracle.core)

Bisection rule (written out so the CUDA library's ordering can be checked
against it index for index): for a block S (sorted original indices) at depth
< m - 1 (the root has depth 0; an m-level tree has 2^m - 1 blocks) with
|S| > min_size: BFS in the graph restricted to S from the smallest
index r; u = the smallest index of the last BFS level; the level structure of
a BFS from u (neighbours in ascending order) gives levels V_0..V_h.  If h < 2
the block is a leaf.  Otherwise the separator is V_mid, mid = (h + 1) // 2,
S1 = V_0 u .. u V_{mid-1}, S2 = the rest of S (later levels and every index of
S the BFS from u did not reach).  Post-order: blocks of S1, blocks of S2, then
the separator.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import core
from .core import GcrInfo, Hybrid, LowFactor, _ptr, lib


def _lib():
    L = lib()
    if not getattr(L, "_mb_bound", False):
        i64, dp, fp, lp = (ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float),
                           ctypes.POINTER(ctypes.c_int64))
        ip = ctypes.POINTER(ctypes.c_int32)
        L.oracle_factor_blocks_f32.argtypes = [i64, dp, i64, ctypes.c_double, i64, i64, ip, ctypes.c_int32, lp, fp,
                                               fp, lp]
        L._mb_bound = True
    return L


def adjacency(K: np.ndarray):
    """Graph of the symmetric sparsity pattern: nbr[i] = sorted j != i with K_ij != 0 or K_ji != 0."""
    K = np.asarray(K)
    P = (K != 0) | (K.T != 0)
    np.fill_diagonal(P, False)
    return [np.nonzero(P[i])[0].tolist() for i in range(K.shape[0])]


def _bfs_levels(adj, members: set, start: int):
    levels, seen, front = [], {start}, [start]
    while front:
        levels.append(sorted(front))
        nxt = set()
        for v in front:
            for w in adj[v]:
                if w in members and w not in seen:
                    seen.add(w)
                    nxt.add(w)
        front = sorted(nxt)
    return levels, seen


def nd_blocks(adj, L: int, levels: int, min_size: int = 8):
    """Block number of every original index (int32[L]) and the number of blocks."""
    blk = np.full(L, -1, dtype=np.int32)
    counter = [0]

    def emit(S):
        for i in S:
            blk[i] = counter[0]
        counter[0] += 1

    def rec(S, depth):
        if depth >= levels - 1 or len(S) <= min_size:
            emit(S)
            return
        members = set(S)
        lv, _ = _bfs_levels(adj, members, S[0])
        u = lv[-1][0]
        lv, seen = _bfs_levels(adj, members, u)
        h = len(lv) - 1
        if h < 2:
            emit(S)
            return
        mid = (h + 1) // 2
        sep = lv[mid]
        S1 = sorted(i for lvl in lv[:mid] for i in lvl)
        S2 = sorted([i for lvl in lv[mid + 1:] for i in lvl] + [i for i in S if i not in seen])
        rec(S1, depth + 1)
        if S2:
            rec(S2, depth + 1)
        emit(sep)

    rec(list(range(L)), 0)
    return blk, counter[0]


def factor_blocks(K: np.ndarray, tau: float, blk: np.ndarray, nblk: int, n_min: int = 0,
                  n_extra: int = 0) -> LowFactor:
    K = np.asfortranarray(K, dtype=np.float64)
    L = K.shape[0]
    blk = np.ascontiguousarray(blk, dtype=np.int32)
    perm = np.empty(L, dtype=np.int64)
    Dk = np.zeros(max(L, 1), dtype=np.float32)
    Lf = np.empty((max(L, 1), max(L, 1)), dtype=np.float32, order="F")
    out = np.zeros(2, dtype=np.int64)
    rc = _lib().oracle_factor_blocks_f32(L, _ptr(K, ctypes.c_double), max(L, 1), float(tau), int(n_min),
                                         int(n_extra), _ptr(blk, ctypes.c_int32), int(nblk),
                                         _ptr(perm, ctypes.c_int64), _ptr(Dk, ctypes.c_float),
                                         _ptr(Lf, ctypes.c_float), _ptr(out, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_factor_blocks_f32: invalid arguments")
    N, Ntau = int(out[0]), int(out[1])
    return LowFactor(L=L, N=N, Ntau=Ntau, perm=perm, D=Dk[:N].copy(), Lfac=np.asfortranarray(Lf[:N, :N]),
                     dtype=np.float32)


def hybrid_factor(K: np.ndarray, tau: float, blk: np.ndarray, nblk: int, n_min: int = 0, n_extra: int = 4,
                  tol: float = 1e-14, max_iter: int = 100, eps_ker: float = 1e-10) -> Hybrid:
    """Algorithm 1 with the multi-block stage 1."""
    K = np.asfortranarray(K, dtype=np.float64)
    F = factor_blocks(K, tau, blk, nblk, n_min=n_min, n_extra=n_extra)
    K11, K12, K21, K22 = core.extract_blocks(K, F)
    if F.N > 0 and F.n2 > 0:
        X, info = core.block_gcr(K11, F, K12, tol=tol, max_iter=max_iter)
    else:
        X, info = np.zeros((F.N, F.n2)), GcrInfo(converged=True)
    S22 = core.schur(K22, K21, X)
    d_ref = float(np.min(np.abs(F.D.astype(np.float64)))) if F.N > 0 else 1.0
    H = core.factor_hard(S22, d_ref, eps_ker) if F.n2 > 0 else None
    return Hybrid(K=K, F=F, X=X, S22=S22, H=H, gcr=info, d_ref=d_ref)
