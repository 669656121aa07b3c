"""NEXT-3: the nonsymmetric matrices of sec. 4.2-4.3 ([A B^T; -B delta D] and
[A B^T; -B 0]) through the GPU path against oracle/nonsym.py.

Stage 1 (FP32 LDU with symmetric pivoting and postponing, [R19]) is graded
BITWISE: Pi, Lambda_2, D, L and U.  Scaling (hf_scale_full) bitwise."""
import numpy as np
import pytest
import torch

import hf_inputs as hi
from hf_inputs.configs import ConfigSpec
from oracle import core as oracle_core
from oracle import nonsym

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


def _rand_ns(L, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((L, L))
    A[np.arange(L), np.arange(L)] = rng.choice([1.0, -1.0, 0.5, 2.0], size=L) * np.abs(rng.standard_normal(L) + 1)
    return A


CASES = [("T8", None, 0), ("H8", None, 0), ("T24", None, 0), ("rand", 300, 1), ("rand", 700, 2),
         ("T8", None, 3)]


def _kbar(name, L, seed):
    if name == "rand":
        return _rand_ns(L, seed)
    return hi.make_kbar(name, seed).numpy()


@pytest.mark.parametrize("name,L,seed", CASES)
@pytest.mark.parametrize("nb", [0, 16])
def test_stage1_nonsym_bitwise(ctx, name, L, seed, nb):
    from paper_2208_01907_b200 import hf
    Kbar = _kbar(name, L, seed)
    Ko, qo = nonsym.scale_full(Kbar)
    Kd = hi.colmajor(torch.from_numpy(Kbar)).cuda()
    q = hf.hf_scale_full(ctx, Kd)
    assert np.array_equal(q.cpu().numpy(), qo)
    assert np.array_equal(Kd.cpu().numpy().T, Ko)          # column-major bytes
    F = nonsym.factor_ldu(Ko, 1e-2, n_min=2)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=1e-2, n_min=2, nb=nb, nonsym=True)
    perm, D, Lf = lf.export()
    Uf = lf.export_u()
    assert lf.N == F.N and lf.L - lf.n2_tau_only == F.Ntau
    assert np.array_equal(perm, F.perm)
    assert np.array_equal(D, F.D)
    assert np.array_equal(Lf.cpu().numpy(), F.Lfac)
    assert np.array_equal(Uf.cpu().numpy(), F.Ufac)
    lf.close()


@pytest.mark.parametrize("name,L,seed", [("T8", None, 0), ("H8", None, 0), ("T24", None, 0), ("H8", None, 2),
                                         ("rand", 300, 1)])
def test_hybrid_nonsym_vs_oracle(ctx, name, L, seed):
    """Alg. 1 steps 2-5 and Alg. 2 on the nonsymmetric path: S22 normwise ([R17] form),
    X12, kernel dimension, manufactured solution, against oracle/nonsym.py."""
    from paper_2208_01907_b200 import hf
    Kbar = _kbar(name, L, seed)
    Ko, _ = nonsym.scale_full(Kbar)
    HF = nonsym.hybrid_factor(Ko, 1e-2, n_min=2)
    Kd = hi.colmajor(torch.from_numpy(Kbar)).cuda()
    hf.hf_scale_full(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=1e-2, n_min=2, nonsym=True)
    hy, info, S22 = hf.hf_schur_gcr(ctx, Kd, lf, want_S22_host=True)
    F = HF.F
    l1, l2 = F.lam1, F.lam2
    K21, K22 = Ko[np.ix_(l2, l1)], Ko[np.ix_(l2, l2)]
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    assert np.linalg.norm(S22 - HF.S22) / den <= 1e-10
    X, _ = hy.export()
    assert np.abs(X.cpu().numpy() - HF.X).max() <= 1e-8 * max(1.0, np.abs(HF.X).max())
    assert info.max_rel_res_true <= 1e-12
    kd = hf.hf_factor_hard(ctx, hy, eps_ker=1e-10)
    margin = min(abs(np.array(HF.H.mu_hist) - HF.H.thr)) if HF.H is not None else 1.0
    if margin > 10 * np.linalg.norm(S22 - HF.S22):
        assert kd == HF.kernel_dim
    xs = hi.manufactured_x(lf.L).numpy()
    b = Ko @ xs
    x, _ = hf.hf_solve(ctx, hy, torch.from_numpy(b).cuda())
    xg = x.cpu().numpy()
    assert np.abs(Ko @ xg - b).max() <= 1e-12 * np.abs(b).max()
    xo, _ = nonsym.hybrid_solve(HF, b)
    assert np.abs(Ko @ xo - b).max() <= 1e-12 * np.abs(b).max()
    hy.close()
    lf.close()


def test_precond_nonsym_vs_oracle(ctx):
    """Q^{-1} = U^{-1} D^{-1} L^{-1} in FP32 against the oracle's FP32 solves."""
    from paper_2208_01907_b200 import hf
    Kbar = _kbar("rand", 700, 2)
    Ko, _ = nonsym.scale_full(Kbar)
    F = nonsym.factor_ldu(Ko, 1e-2, n_min=2)
    Kd = hi.colmajor(torch.from_numpy(Kbar)).cuda()
    hf.hf_scale_full(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=1e-2, n_min=2, nonsym=True)
    rng = np.random.default_rng(0)
    R = rng.standard_normal((lf.L, 5))
    R[F.lam2] = 0.0
    W = hf.hf_precond_apply(ctx, lf, torch.from_numpy(R.T.copy()).cuda().T)
    Wg = W.cpu().numpy()
    Wo = np.zeros_like(R)
    Wo[F.lam1] = oracle_core.precond_apply(F, R[F.lam1])
    # both are FP32 solves of the same FP32 factors: agree to the FP32 error level of the solve
    eps32 = float(np.finfo(np.float32).eps)
    K11 = Ko[np.ix_(F.lam1, F.lam1)]
    exact = np.linalg.solve(K11, R[F.lam1])
    e_o = np.abs(Wo[F.lam1] - exact).max()
    e_g = np.abs(Wg[F.lam1] - exact).max()
    assert e_g <= max(10 * e_o, 100 * eps32 * np.abs(exact).max())
    lf.close()


def test_nonsym_edge_cases(ctx):
    """Degenerate inputs of the nonsymmetric path against the oracle: 1 x 1, a zero first
    pivot (everything postponed), a strictly triangular-dominant matrix with no postponement
    (n2 = 0: hf_schur_gcr returns an empty S22 and hf_factor_hard is a no-op), ragged sizes
    around the 128-row tile, NaN refused."""
    from paper_2208_01907_b200 import hf
    cases = [np.array([[-3.0]]), np.array([[0.0, 2.0], [-1.0, 0.0]]),
             np.eye(5) * 4 + np.triu(np.ones((5, 5)), 1)]
    rng = np.random.default_rng(9)
    for L in (127, 128, 129, 257):
        A = rng.standard_normal((L, L))
        A[np.arange(L), np.arange(L)] = rng.uniform(0.5, 2.0, L) * rng.choice([1, -1], L)
        cases.append(A)
    for Kbar in cases:
        Ko, _ = nonsym.scale_full(Kbar)
        F = nonsym.factor_ldu(Ko, 1e-2)
        Kd = hi.colmajor(torch.from_numpy(Kbar.copy())).cuda()
        hf.hf_scale_full(ctx, Kd)
        lf = hf.hf_factor_lowprec(ctx, Kd, tau=1e-2, nonsym=True)
        perm, D, Lf = lf.export()
        assert lf.N == F.N and np.array_equal(perm, F.perm) and np.array_equal(D, F.D)
        if F.N:
            assert np.array_equal(Lf.cpu().numpy(), F.Lfac)
            assert np.array_equal(lf.export_u().cpu().numpy(), F.Ufac)
        hy, info, S22 = hf.hf_schur_gcr(ctx, Kd, lf, want_S22_host=True)
        kd = hf.hf_factor_hard(ctx, hy)
        if lf.n2 == 0:
            assert kd == 0
        hy.close()
        lf.close()
    bad = torch.eye(4, dtype=torch.float64, device="cuda")
    bad[2, 1] = float("nan")
    with pytest.raises(hf.HFError):
        hf.hf_scale_full(ctx, bad)
