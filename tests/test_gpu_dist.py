"""Stage-2 right-hand-side sharding on one GPU:
  * every rank of a G-rank run emulated in turn (hf_set_virtual_rank: the
    rank's own block GCR on its column slice of K12 and its slice of S22,
    no collective); the slices put together must meet the same normwise bar
    against the oracle as the single-block run (e_S <= 1e-10, [R17]) even
    though every slice has its own Krylov space;
  * the real NCCL path of libhf (hf_create_dist, one rank): broadcast of the
    S22 / X12 slices and the max-reduction of the GCR statistics."""
import numpy as np
import pytest
import torch

import hf_inputs as hi
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


def _e_S(Sg, HF):
    K11, K12, K21, K22 = oracle.extract_blocks(HF.K, HF.F)
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    return np.linalg.norm(Sg - HF.S22) / den


@pytest.mark.parametrize("name,G", [("P2048", 2), ("P2048", 3), ("C0", 2), ("S24", 4)])
def test_virtual_ranks_compose(ctx, name, G):
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, 0)
    Ko, _ = oracle.scale(Kb.numpy())
    HF = oracle.hybrid_factor(Ko, tau=spec.tau, n_min=spec.n_min)
    Kd = Kb.cuda()
    hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min)
    n2 = lf.n2
    S = np.zeros((n2, n2))
    X = np.zeros((lf.N, n2))
    try:
        for r in range(G):
            hf.hf_set_virtual_rank(ctx, r, G)
            hy, info, Sr = hf.hf_schur_gcr(ctx, Kd, lf, want_S22_host=True)
            c0, c1 = hf.hf_shard_cols(n2, G, r)
            assert np.all(Sr[:, :c0] == 0) and np.all(Sr[:, c1:] == 0)
            S[:, c0:c1] = Sr[:, c0:c1]
            Xr, _ = hy.export()
            X[:, c0:c1] = Xr.cpu().numpy()[:, c0:c1]
            assert info.max_rel_res_true <= 1e-12
            hy.close()
    finally:
        hf.hf_set_virtual_rank(ctx, 0, 0)
    assert _e_S(S, HF) <= 1e-10
    assert np.linalg.norm(X - HF.X) <= 1e-8 * np.linalg.norm(HF.X)


def test_nccl_path_one_rank():
    from paper_2208_01907_b200 import hf
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = hi.CONFIGS["P1024"]
    Kb = hi.make_kbar("P1024", 0)
    Ko, _ = oracle.scale(Kb.numpy())
    HF = oracle.hybrid_factor(Ko, tau=spec.tau, n_min=spec.n_min)
    c = hf.Context(0, nccl_id=hf.nccl_unique_id(), rank=0, nranks=1)
    try:
        Kd = Kb.cuda()
        hf.hf_scale(c, Kd)
        lf = hf.hf_factor_lowprec(c, Kd, tau=spec.tau, n_min=spec.n_min)
        hy, info, S = hf.hf_schur_gcr(c, Kd, lf, want_S22_host=True)
        assert _e_S(S, HF) <= 1e-10 and info.max_rel_res_true <= 1e-12
        kd = hf.hf_factor_hard(c, hy)
        assert kd == HF.kernel_dim
    finally:
        c.close()


@pytest.mark.parametrize("name,seed,G,nb", [("P512", 0, 1, 0), ("P512", 2, 3, 0), ("P2048", 0, 2, 0),
                                            ("P2048", 1, 5, 64), ("P2048", 2, 8, 0), ("N32", 0, 4, 0),
                                            ("S24", 0, 3, 128), ("S24", 1, 6, 32), ("C1", 0, 8, 0),
                                            ("C1", 0, 7, 96), ("P1024", 0, 4, 16), ("C0", 1, 2, 8)])
@pytest.mark.parametrize("look", [0, 1])
def test_stage1_distributed_bitwise(ctx, name, seed, G, nb, look, monkeypatch):
    """The distributed stage 1 of the multi-GPU path (k_dist.cu: lower-triangle
    1D block-cyclic ownership, chain rows split over the ranks, per-pivot key
    exchange over every rank's slots, panel gathered from the owners), all G
    ranks emulated on this GPU in one cooperative chain launch: Pi, Lambda_2, D
    and L bit-identical to the oracle [R8] for G = 1..8 and several panel widths,
    with the serial schedule and with the lookahead one (the chain of panel p+1
    reads the matrix at the start of panel p and applies panel p's updates itself
    while panel p's trailing update runs on a second stream)."""
    from paper_2208_01907_b200 import hf
    monkeypatch.setenv("HF_DIST_LOOKAHEAD", str(look))
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    Kd = Kb.cuda()
    hf.hf_scale(ctx, Kd)
    try:
        hf.hf_set_stage1_partitions(ctx, G)
        lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min, nb=nb)
    finally:
        hf.hf_set_stage1_partitions(ctx, 0)
    perm, D, Lf = lf.export()
    assert lf.N == Fo.N and lf.L - lf.n2_tau_only == Fo.Ntau
    assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
    assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


@pytest.mark.slow
@pytest.mark.parametrize("G,look", [(2, 0), (8, 0), (8, 1)])
def test_stage1_distributed_c2_equals_one_gpu(ctx, G, look, monkeypatch):
    """C2 at full size (L = 16384, n_min 256): the G-rank emulation of the
    distributed stage 1 is bit-identical to the one-GPU path (which
    test_gpu_fullsize.py pins to the whole oracle)."""
    from paper_2208_01907_b200 import hf
    monkeypatch.setenv("HF_DIST_LOOKAHEAD", str(look))
    spec = hi.CONFIGS["C2"]
    Kb = hi.make_kbar("C2", 0, device="cuda")
    hf.hf_scale(ctx, Kb)
    lf1 = hf.hf_factor_lowprec(ctx, Kb, tau=spec.tau, n_min=spec.n_min)
    p1, D1, L1 = lf1.export()
    try:
        hf.hf_set_stage1_partitions(ctx, G)
        lfG = hf.hf_factor_lowprec(ctx, Kb, tau=spec.tau, n_min=spec.n_min)
    finally:
        hf.hf_set_stage1_partitions(ctx, 0)
    pG, DG, LG = lfG.export()
    assert np.array_equal(p1, pG) and np.array_equal(D1, DG)
    assert torch.equal(L1, LG)


@pytest.mark.parametrize("look", [0, 1])
def test_stage1_real_rank_path_one_gpu(look, monkeypatch):
    """The REAL-rank code path of the distributed stage 1 on one GPU: a one-rank NCCL
    context asked for one partition runs it exactly as a rank of a multi-GPU job does
    (CUDA-IPC handles all-gathered over NCCL, device-side NVLink barrier kernels,
    system-scope exchange words, the serial and the lookahead schedules with the chain's
    SMs reserved) -- only the peer mappings are absent.  Bitwise against the oracle."""
    from paper_2208_01907_b200 import hf
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    monkeypatch.setenv("HF_DIST_LOOKAHEAD", str(look))
    spec = hi.CONFIGS["P2048"]
    Kb = hi.make_kbar("P2048", 1)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    c = hf.Context(0, nccl_id=hf.nccl_unique_id(), rank=0, nranks=1)
    try:
        Kd = Kb.cuda()
        hf.hf_scale(c, Kd)
        hf.hf_set_stage1_partitions(c, 1)
        lf = hf.hf_factor_lowprec(c, Kd, tau=spec.tau, n_min=spec.n_min)
        perm, D, Lf = lf.export()
        assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
        assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)
        lf.close()
    finally:
        c.close()
