"""Pins of oracle/multiblock.py (NEXT-4, multi-block postponing): the
block path reduces to the pinned single-sequence factorization when there are no
blocks; bitwise agreement with an exact-rational left-looking replay of the block
rule; nested-dissection invariants (separation, post-order, 2^m - 1 blocks);
Alg. 1 + 2 with the multi-block stage 1 on grid Laplacians."""
import numpy as np
import pytest

import hf_inputs as hi
import oracle
from oracle import multiblock as mb
from tests.exact_ldlt import left_looking_ldlt_blocks


def test_no_blocks_is_the_single_sequence_factorization():
    K, _ = oracle.scale(hi.make_kbar("N16", 0).numpy())
    F0 = oracle.factor_lowprec(K, 1e-2, n_min=2, n_extra=1)
    F1 = mb.factor_blocks(K, 1e-2, np.zeros(K.shape[0], np.int32), 0, n_min=2, n_extra=1)
    assert F0.N == F1.N and F0.Ntau == F1.Ntau
    assert np.array_equal(F0.perm, F1.perm) and np.array_equal(F0.D, F1.D) and np.array_equal(F0.Lfac, F1.Lfac)


@pytest.mark.parametrize("L,seed,nblk", [(9, 0, 3), (10, 1, 4), (8, 2, 2)])
def test_blocks_match_exact_replay(L, seed, nblk):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((L, L))
    Kbar = B @ np.diag(rng.choice([1.0, -1.0, 1e-3, 1e-5], size=L)) @ B.T
    K, _ = oracle.scale(Kbar)
    blk = rng.integers(0, nblk, size=L).astype(np.int32)
    F = mb.factor_blocks(K, 1e-1, blk, nblk)
    piv, D, Lcols, Ntau = left_looking_ldlt_blocks(K, 1e-1, blk, nblk)
    assert F.Ntau == Ntau
    assert list(F.perm[:F.N]) == piv[:F.N]
    assert np.array_equal(F.D, np.array(D[:F.N], dtype=np.float32))
    pos = {p: k for k, p in enumerate(F.perm[:F.N])}
    for k in range(F.N):
        for i, v in Lcols[k].items():
            if i in pos and pos[i] > k:
                assert F.Lfac[pos[i], k] == np.float32(v)


def test_nested_dissection_invariants():
    K = hi.make_kbar("N32", 0).numpy()
    adj = mb.adjacency(K)
    L = K.shape[0]
    for levels in (1, 2, 3, 4):
        blk, nblk = mb.nd_blocks(adj, L, levels)
        assert np.all(blk >= 0) and blk.max() == nblk - 1
        assert nblk == 2 ** levels - 1          # a 32 x 32 grid bisects cleanly to 4 levels
    blk, nblk = mb.nd_blocks(adj, L, 3)
    # post-order on 3 levels: [leaf, leaf, sep], [leaf, leaf, sep], root sep (7 blocks);
    # the two halves (blocks 0-2 and 3-5) are separated by the root separator (block 6)
    A = set(np.nonzero(blk <= 2)[0].tolist())
    B = set(np.nonzero((blk >= 3) & (blk <= 5))[0].tolist())
    for i in A:
        assert not (set(adj[i]) & B)
    # leaves of the same parent are separated by that parent's separator
    for lo in (0, 3):
        X = set(np.nonzero(blk == lo)[0].tolist())
        Y = set(np.nonzero(blk == lo + 1)[0].tolist())
        for i in X:
            assert not (set(adj[i]) & Y)


@pytest.mark.parametrize("name,levels", [("N16", 3), ("N32", 4), ("S12", 3)])
def test_multiblock_hybrid_solve(name, levels):
    Kbar = hi.make_kbar(name, 0).numpy()
    K, _ = oracle.scale(Kbar)
    blk, nblk = mb.nd_blocks(mb.adjacency(K), K.shape[0], levels)
    HF = mb.hybrid_factor(K, 1e-2, blk, nblk, n_min=4, n_extra=4)
    assert HF.F.n2 >= 4
    xs = np.arange(K.shape[0]) % 11.0
    b = K @ xs
    x, info = oracle.hybrid_solve(HF, b)
    assert np.abs(K @ x - b).max() <= 1e-10 * np.abs(b).max()
