"""NEXT-4: multi-block threshold postponing along a nested-dissection tree
(sec. 2.2) on the GPU against oracle/multiblock.py: the ordering index
for index, stage 1 BITWISE (Pi, Lambda_2, D, L) including block transitions in
the middle of a panel, and Alg. 1 + 2 with it."""
import numpy as np
import pytest
import torch

import hf_inputs as hi
import oracle
from oracle import multiblock as mb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("name,levels", [("N16", 3), ("N32", 4), ("S12", 3), ("C1", 5), ("S24", 4)])
def test_nd_matches_oracle(ctx, name, levels):
    from paper_2208_01907_b200 import hf
    Kb = hi.make_kbar(name, 0)
    K = Kb.cuda()
    hf.hf_scale(ctx, K)
    blk, nblk = hf.hf_nd_blocks(ctx, K, levels)
    Ko, _ = oracle.scale(Kb.numpy())
    blk_o, nblk_o = mb.nd_blocks(mb.adjacency(Ko), Ko.shape[0], levels)
    assert nblk == nblk_o
    assert np.array_equal(blk, blk_o)


@pytest.mark.parametrize("name,levels,nb", [("N16", 3, 0), ("N32", 4, 0), ("N32", 4, 16), ("S12", 3, 0),
                                            ("S12", 3, 16), ("C1", 5, 0), ("S24", 4, 0)])
def test_stage1_blocks_bitwise(ctx, name, levels, nb):
    from paper_2208_01907_b200 import hf
    Kb = hi.make_kbar(name, 0)
    K = Kb.cuda()
    hf.hf_scale(ctx, K)
    Ko, _ = oracle.scale(Kb.numpy())
    assert np.array_equal(K.cpu().numpy(), Ko)
    blk, nblk = mb.nd_blocks(mb.adjacency(Ko), Ko.shape[0], levels)
    F = mb.factor_blocks(Ko, 1e-2, blk, nblk, n_min=2, n_extra=4)
    lf = hf.hf_factor_lowprec_blocks(ctx, K, blk, nblk, tau=1e-2, n_min=2, n_extra=4, nb=nb)
    perm, D, Lf = lf.export()
    assert lf.N == F.N and lf.L - lf.n2_tau_only == F.Ntau
    assert np.array_equal(perm, F.perm)
    assert np.array_equal(D, F.D)
    assert np.array_equal(Lf.cpu().numpy(), F.Lfac)
    lf.close()


def test_no_blocks_equals_single_sequence(ctx):
    from paper_2208_01907_b200 import hf
    K = hi.make_kbar("N32", 0).cuda()
    hf.hf_scale(ctx, K)
    a = hf.hf_factor_lowprec(ctx, K, tau=1e-2, n_min=2)
    b = hf.hf_factor_lowprec_blocks(ctx, K, np.zeros(K.shape[0], np.int32), 0, tau=1e-2, n_min=2)
    pa, Da, La = a.export()
    pb, Db, Lb = b.export()
    assert np.array_equal(pa, pb) and np.array_equal(Da, Db) and torch.equal(La, Lb)
    a.close()
    b.close()


@pytest.mark.parametrize("name,levels", [("N32", 4), ("S12", 3)])
def test_multiblock_hybrid_vs_oracle(ctx, name, levels):
    from paper_2208_01907_b200 import hf
    Kb = hi.make_kbar(name, 0)
    K = Kb.cuda()
    hf.hf_scale(ctx, K)
    Ko, _ = oracle.scale(Kb.numpy())
    blk, nblk = mb.nd_blocks(mb.adjacency(Ko), Ko.shape[0], levels)
    HF = mb.hybrid_factor(Ko, 1e-2, blk, nblk, n_min=4, n_extra=4)
    lf = hf.hf_factor_lowprec_blocks(ctx, K, blk, nblk, tau=1e-2, n_min=4, n_extra=4)
    hy, info, S22 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True)
    K11, K12, K21, K22 = oracle.extract_blocks(HF.K, HF.F)
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    assert np.linalg.norm(S22 - HF.S22) / den <= 1e-10
    hf.hf_factor_hard(ctx, hy)
    xs = hi.manufactured_x(lf.L, device="cuda")
    b = K @ xs
    x, _ = hf.hf_solve(ctx, hy, b)
    assert float((K @ x - b).abs().max() / b.abs().max()) <= 1e-12
    hy.close()
    lf.close()


def test_multiblock_edge_cases(ctx):
    """One block per index (every block a single candidate), all indices in one block, a
    block id out of range refused, L = 1, and a zero matrix (every block's first candidate
    is 0: all postponed)."""
    from paper_2208_01907_b200 import hf
    Kb = hi.make_kbar("N16", 0)
    K = Kb.cuda()
    hf.hf_scale(ctx, K)
    Ko, _ = oracle.scale(Kb.numpy())
    L = Ko.shape[0]
    for blk, nblk in ((np.arange(L, dtype=np.int32), L), (np.zeros(L, np.int32), 1),
                      ((np.arange(L) % 5).astype(np.int32), 5)):
        F = mb.factor_blocks(Ko, 1e-2, blk, nblk, n_min=1)
        lf = hf.hf_factor_lowprec_blocks(ctx, K, blk, nblk, tau=1e-2, n_min=1)
        perm, D, Lf = lf.export()
        assert lf.N == F.N and np.array_equal(perm, F.perm) and np.array_equal(D, F.D)
        assert np.array_equal(Lf.cpu().numpy(), F.Lfac)
        lf.close()
    with pytest.raises(hf.HFError):
        hf.hf_factor_lowprec_blocks(ctx, K, np.full(L, 7, np.int32), 3)
    one = torch.tensor([[2.0]], dtype=torch.float64, device="cuda")
    lf = hf.hf_factor_lowprec_blocks(ctx, one, np.zeros(1, np.int32), 1)
    assert lf.N == 1
    lf.close()
    z = torch.zeros(6, 6, dtype=torch.float64, device="cuda")
    lf = hf.hf_factor_lowprec_blocks(ctx, z, np.array([0, 0, 1, 1, 2, 2], np.int32), 3)
    assert lf.N == 0 and lf.n2 == 6
    lf.close()
