"""Pins for Alg. 1 steps 2-5 and Alg. 2 of the oracle."""
import numpy as np
import pytest

import hf_inputs as hi
import oracle


def _hybrid(name, seed, **kw):
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed).numpy()
    K, q = oracle.scale(Kb)
    HF = oracle.hybrid_factor(K, tau=spec.tau, n_min=spec.n_min, **kw)
    return Kb, K, q, HF


def _normwise(Sa, Sb, K22, K21, X):
    return np.linalg.norm(Sa - Sb) / (np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(X))


@pytest.mark.parametrize("name,seed", [("C0", 0), ("C0", 1), ("N32", 0), ("S24", 0), ("P512", 0)])
def test_schur_matches_dense_eq2(name, seed):
    """S22 = K22 - K21 K11^{-1} K12 (Eq. 2) by LAPACK dense solve."""
    _, K, _, HF = _hybrid(name, seed)
    K11, K12, K21, K22 = oracle.extract_blocks(K, HF.F)
    Xd = np.linalg.solve(K11, K12)
    Sd = K22 - K21 @ Xd
    assert _normwise(HF.S22, Sd, K22, K21, Xd) <= 1e-10     # [R17] normwise form
    assert HF.gcr.converged and HF.gcr.iters <= 15


def _ld_solve(A, B):
    """Gaussian elimination in x87 long double, no pivoting beyond the given
    order (A is K11 in the oracle's pivot order)."""
    A = A.astype(np.longdouble).copy()
    B = B.astype(np.longdouble).copy()
    n = A.shape[0]
    for k in range(n):
        f = A[k + 1:, k] / A[k, k]
        A[k + 1:, k:] -= np.outer(f, A[k, k:])
        B[k + 1:] -= np.outer(f, B[k])
    X = np.zeros_like(B)
    for k in range(n - 1, -1, -1):
        X[k] = (B[k] - A[k, k + 1:] @ X[k + 1:]) / A[k, k]
    return X


@pytest.mark.parametrize("seed", range(3))
def test_schur_matches_long_double_small(seed):
    _, K, _, HF = _hybrid("P64", seed)
    K11, K12, K21, K22 = oracle.extract_blocks(K, HF.F)
    Xl = _ld_solve(K11, K12)
    Sl = (K22.astype(np.longdouble) - K21.astype(np.longdouble) @ Xl).astype(np.float64)
    assert _normwise(HF.S22, Sl, K22, K21, Xl.astype(np.float64)) <= 1e-12


def test_spec_acceptance_schur_forced_postponing():
    """SPEC acceptance #1: random 20-100 sized, 2-8 indices force-postponed,
    literal ||dS22||_F / ||S22||_F <= 1e-10 (S22 = O(1) here)."""
    rng = np.random.default_rng(42)
    for trial in range(20):
        n = int(rng.integers(20, 101))
        nm = int(rng.integers(2, 9))
        A = rng.standard_normal((n, n))
        Kb = A + A.T + np.diag(rng.uniform(2, 6, n) * rng.choice([-1, 1], n))
        K, _ = oracle.scale(Kb)
        HF = oracle.hybrid_factor(K, tau=1e-6, n_min=nm)
        K11, K12, K21, K22 = oracle.extract_blocks(K, HF.F)
        Sd = K22 - K21 @ np.linalg.solve(K11, K12)
        assert HF.F.n2 == nm
        assert np.linalg.norm(HF.S22 - Sd) <= 1e-10 * np.linalg.norm(Sd)


# ---------------------------------------------------------------- stage 3
def test_hard_factor_small_cases():
    H = oracle.factor_hard(np.diag([1.0, 0.0]), 1.0)
    assert H.kernel_dim == 1
    H = oracle.factor_hard(np.array([[0.0, 1.0], [1.0, 0.0]]), 1.0)
    assert H.blocks == [2] and H.kernel_dim == 0
    rng = np.random.default_rng(0)
    B = rng.standard_normal((11, 17))
    H = oracle.factor_hard(B.T @ B, 1.0)
    assert H.kernel_dim == 6


@pytest.mark.parametrize("rank_def", [0, 1, 2, 6])
def test_hard_factor_constructed_rank_and_reconstruction(rank_def):
    rng = np.random.default_rng(rank_def)
    m = 24
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    lam = rng.uniform(0.5, 2.0, m) * rng.choice([-1, 1], m)
    lam[m - rank_def:] = 0.0
    S = Q @ np.diag(lam) @ Q.T
    H = oracle.factor_hard(S, 1.0)
    assert H.kernel_dim == rank_def
    P = np.eye(m)[:, H.perm2]
    Rk = H.Lh @ H.Dh @ H.Lh.T
    Ssym = 0.5 * (S + S.T)
    assert np.abs(P @ Rk @ P.T - Ssym).max() <= 1e-12
    # a solve on a consistent right-hand side reproduces it
    y = S @ rng.standard_normal(m)
    x = oracle.hard_solve(H, y)
    assert np.abs(S @ x - y).max() <= 1e-11 * np.abs(y).max()


def test_neumann_and_saddle_kernel_dims_vs_eigen_count():
    """kernel_dim equals an independent FP64 count of |eig(K)| below the same
    threshold (C1 analog) and 2 translations for the saddle analog."""
    _, K, _, HF = _hybrid("N32", 0)
    thr = 1e-10 * HF.d_ref
    ev = np.abs(np.linalg.eigvalsh(K))
    assert HF.kernel_dim == int(np.sum(ev <= thr)) == 3
    _, K, _, HF = _hybrid("S24", 0)
    assert HF.kernel_dim == 2


# ---------------------------------------------------------------- Alg. 2
def test_identity_solve():
    HF = oracle.hybrid_factor(np.eye(6))
    b = np.arange(6.0)
    x, _ = oracle.hybrid_solve(HF, b)
    assert np.array_equal(x, b)


@pytest.mark.parametrize("name,seed", [("C0", 0), ("P512", 1), ("S24", 0), ("N32", 0)])
def test_manufactured_solution_residual(name, seed):
    """Table 1's RHS: x*_i = i mod 11, residual ||Kx-b||/||b|| <= 1e-12."""
    _, K, _, HF = _hybrid(name, seed)
    xs = hi.manufactured_x(K.shape[0]).numpy()
    b = K @ xs
    x, _ = oracle.hybrid_solve(HF, b)
    rho = np.abs(K @ x - b).max() / np.abs(b).max()
    assert rho <= 1e-12


@pytest.mark.parametrize("name,seed", [("C0", 2), ("P512", 0)])
def test_random_rhs_backward_error(name, seed):
    Kb, K, q, HF = _hybrid(name, seed)
    bb = hi.make_rhs(name, seed).numpy()
    b = q * bb
    x, _ = oracle.hybrid_solve(HF, b)
    eta = np.abs(K @ x - b).max() / (np.abs(K).sum(1).max() * np.abs(x).max() + np.abs(b).max())
    assert eta <= 1e-12
