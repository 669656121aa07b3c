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
