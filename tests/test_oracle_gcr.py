"""Pins for the oracle's preconditioner and Krylov solvers:
Algorithm 3, Algorithm 4, Algorithm 5."""
import numpy as np
import pytest

import oracle


def _moderate(n, seed, cond=1e3):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.geomspace(1.0, 1.0 / cond, n) * rng.choice([-1.0, 1.0], n)
    A = Q @ np.diag(lam) @ Q.T
    A = np.tril(A) + np.tril(A, -1).T
    K, _ = oracle.scale(A)
    return K


def _factor(K):
    F = oracle.factor_lowprec(K, 1e-6)
    assert F.N == K.shape[0]
    A = K[np.ix_(F.lam1, F.lam1)]
    return F, A


def test_precond_exact_cases():
    F = oracle.factor_lowprec(np.diag([2.0, 4.0]), 1e-2)   # pivots 4 then 2
    b = np.array([4.0, 2.0])                               # pivot order
    assert np.array_equal(oracle.precond_apply(F, b[:, None])[:, 0], [1.0, 1.0])
    Fi = oracle.factor_lowprec(np.eye(4), 1e-2)
    r = np.array([1.0 + 2**-30, 3.0, -7.0, np.pi])
    out = oracle.precond_apply(Fi, r[:, None])[:, 0]
    assert np.array_equal(out, r.astype(np.float32).astype(np.float64))   # truncate then lift


def test_precond_residual_bound():
    K = _moderate(30, 1, cond=10.0)
    F, A = _factor(K)
    rng = np.random.default_rng(3)
    b = rng.standard_normal((30, 1))
    x = oracle.precond_apply(F, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 100 * np.finfo(np.float32).eps


def test_identity_converges_at_iteration_zero():
    F = oracle.factor_lowprec(np.eye(8), 1e-2)
    B = np.arange(16.0).reshape(8, 2) % 5    # exactly representable in FP32
    X, info = oracle.block_gcr(np.eye(8), F, B)
    assert info.iters == 0 and info.converged and np.array_equal(X, B)


@pytest.mark.parametrize("seed", range(3))
def test_constructed_solution(seed):
    K = _moderate(40, seed, cond=1e4)
    F, A = _factor(K)
    rng = np.random.default_rng(seed)
    Xs = rng.standard_normal((40, 5))
    X, info = oracle.block_gcr(A, F, A @ Xs)
    assert info.converged and info.iters <= 15
    assert np.abs(X - Xs).max() <= 1e-12 * np.abs(Xs).max() * 1e3


@pytest.mark.parametrize("seed", range(3))
def test_block_orthogonality_and_monotone_residual(seed):
    K = _moderate(60, 10 + seed, cond=1e5)
    F, A = _factor(K)
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((60, 4))
    tr = {}
    X, info = oracle.block_gcr(A, F, B, trace=tr)
    Qs = tr["Q"]
    for n in range(len(Qs)):
        for m in range(n):
            G = Qs[m].T @ Qs[n]
            nm = np.linalg.norm(Qs[m], axis=0)[:, None] * np.linalg.norm(Qs[n], axis=0)[None, :]
            assert np.abs(G / nm).max() <= 1e-10          # Q_m^T Q_n = 0
    r0 = np.linalg.norm(B - A @ oracle.precond_apply(F, B), axis=0)
    for n, R in enumerate(tr["R"]):
        for m in range(min(n + 1, len(Qs))):
            G = Qs[m].T @ R                                 # Galerkin, relative
            nm = np.linalg.norm(Qs[m], axis=0)[:, None] * r0[None, :]   # to the initial residual
            assert np.abs(G / nm).max() <= 1e-12
    hist = np.array([h for h in info.history])
    assert np.all(np.linalg.norm(hist[1:], axis=1) <= np.linalg.norm(hist[:-1], axis=1) * (1 + 1e-12))


def test_block_with_one_column_equals_gcr():
    K = _moderate(50, 5, cond=1e5)
    F, A = _factor(K)
    b = np.random.default_rng(5).standard_normal(50)
    xb, ib = oracle.block_gcr(A, F, b[:, None])
    xg, ig = oracle.gcr(A, F, b)
    assert ib.iters == ig.iters
    hb = np.array([h[0] for h in ib.history])
    hg = np.array([h[0] for h in ig.history])
    assert np.allclose(hb, hg, rtol=1e-6, atol=1e-15)
    assert np.allclose(xb[:, 0], xg, rtol=1e-12, atol=1e-12 * np.abs(xg).max())


def test_iteration_ordering_bgcr_gcr_ir():
    """Fig. 2: IR converges slower than GCR; block GCR no slower."""
    K = _moderate(80, 21, cond=1e6)
    F, A = _factor(K)
    rng = np.random.default_rng(2)
    B = rng.standard_normal((80, 4))
    _, ib = oracle.block_gcr(A, F, B)
    its_g = max(oracle.gcr(A, F, B[:, j])[1].iters for j in range(4))
    its_ir = max(oracle.iterative_refinement(A, F, B[:, j], max_iter=200)[1].iters for j in range(4))
    assert ib.iters <= its_g <= its_ir
