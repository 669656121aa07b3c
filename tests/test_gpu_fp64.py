"""NEXT-1, first part: stage 1 with the paper's (double,
double-double) pair's lower precision -- the FP64 factorization with the same
pivoting / postponing rules [R2]-[R10] in IEEE double (prec = 64), bitwise
against the oracle's FP64 variant (oracle_factor_f64): Pi, Lambda_2, D, L."""
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


CASES = [("C0", 0), ("C0", 1), ("P64", 0), ("N32", 0), ("S24", 0), ("P512", 0), ("P1024", 1), ("C1", 0)]


@pytest.mark.parametrize("name,seed", CASES)
def test_stage1_fp64_bitwise(ctx, name, seed):
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min, prec="f64")
    Kd = Kb.cuda()
    hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min, prec=64)
    perm, D, Lf = lf.export64()
    assert lf.N == Fo.N and lf.L - lf.n2_tau_only == Fo.Ntau
    assert np.array_equal(perm, Fo.perm)
    assert np.array_equal(D, Fo.D)
    if Fo.N:
        assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


@pytest.mark.parametrize("nb", [8, 32, 128])
def test_stage1_fp64_panel_width_invariance(ctx, nb):
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS["P512"]
    Kb = hi.make_kbar("P512", 2)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min, prec="f64")
    Kd = Kb.cuda()
    hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min, nb=nb, prec=64)
    perm, D, Lf = lf.export64()
    assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
    assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


def test_fp64_pivots_recover_the_planted_count(ctx):
    """with FP64 pivots the paper's tau-rule alone (no floor)
    postpones exactly the planted directions of the small planted configs."""
    from paper_2208_01907_b200 import hf
    for name, seed in (("C0", 0), ("C0", 1), ("P64", 0)):
        spec = hi.CONFIGS[name]
        Kd = hi.make_kbar(name, seed).cuda()
        hf.hf_scale(ctx, Kd)
        lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=0, prec=64)
        Fo = oracle.factor_lowprec(oracle.scale(hi.make_kbar(name, seed).numpy())[0], spec.tau, prec="f64")
        assert lf.n2_tau_only == spec.n_hard == Fo.L - Fo.Ntau, (name, seed, lf.n2_tau_only)


@pytest.mark.parametrize("name,seed", [("C0", 0), ("P512", 0), ("N32", 0), ("S24", 0), ("P2048", 1)])
def test_hybrid_fp64_pair_vs_oracle(ctx, name, seed):
    """The (double, double) hybrid -- FP64 factor + FP64 preconditioner (the k_trsm
    body instantiated for double) + FP64 block GCR, Schur, hard factor, solve --
    against the oracle's hybrid_factor(prec="f64"): the pure-precision column of the
    paper's Table 1 for the (float, double) pair."""
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    Ko, _ = oracle.scale(Kb.numpy())
    HF = oracle.hybrid_factor(Ko, tau=spec.tau, n_min=spec.n_min, prec="f64")
    Kd = Kb.cuda()
    hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min, prec=64)
    assert lf.N == HF.F.N
    hy, info, S22 = hf.hf_schur_gcr(ctx, Kd, lf, want_S22_host=True)
    K11, K12, K21, K22 = oracle.extract_blocks(HF.K, HF.F)
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    assert np.linalg.norm(S22 - HF.S22) / den <= 1e-10
    assert info.max_rel_res_true <= 1e-12
    assert info.iters <= max(4, HF.gcr.iters + 1)          # an FP64 preconditioner: very few iterations
    kd = hf.hf_factor_hard(ctx, hy)
    margin = min(abs(np.array(HF.H.mu_hist) - HF.H.thr)) if HF.H is not None and HF.H.mu_hist else np.inf
    if margin > 10 * np.linalg.norm(S22 - HF.S22):
        assert kd == HF.kernel_dim
    xs = hi.manufactured_x(Ko.shape[0]).numpy()
    b = Ko @ xs
    x, _ = hf.hf_solve(ctx, hy, torch.from_numpy(b).cuda())
    assert np.abs(Ko @ x.cpu().numpy() - b).max() / np.abs(b).max() <= 1e-12


def test_precond_fp64_vs_oracle(ctx):
    from paper_2208_01907_b200 import hf
    import scipy.linalg as sla
    spec = hi.CONFIGS["P1024"]
    Kb = hi.make_kbar("P1024", 0)
    Ko, _ = oracle.scale(Kb.numpy())
    F = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min, prec="f64")
    Kd = Kb.cuda()
    hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min, prec=64)
    rng = np.random.default_rng(5)
    R = rng.standard_normal((Ko.shape[0], 70))
    W = hf.hf_precond_apply(ctx, lf, torch.from_numpy(np.ascontiguousarray(R.T)).cuda().T).cpu().numpy()
    l1 = F.perm[: F.N]
    Wo = oracle.precond_apply(F, R[l1])
    assert np.linalg.norm(W[l1] - Wo) <= 1e-10 * np.linalg.norm(Wo)
