"""Pins of oracle/nonsym.py (NEXT-3, the nonsymmetric matrices of sec. 4.2-4.3):
bitwise agreement of the FP32 LDU with an exact-rational left-looking replay,
reconstruction and pivot rule, constructed ranks of the LU of S22, manufactured
solutions of Alg. 2 on stokes-like and dd-hole-like inputs."""
import numpy as np
import pytest

import hf_inputs as hi
from oracle import nonsym
from tests.exact_ldlt import left_looking_ldu


def _rand_ns(L, seed, ties=False):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((L, L))
    if ties:
        A = np.round(A * 4) / 4
        np.fill_diagonal(A, rng.choice([1.0, -1.0, 0.5], size=L))
    return A


@pytest.mark.parametrize("L,seed,ties", [(7, 0, False), (9, 1, False), (8, 2, True), (10, 3, True)])
def test_ldu_matches_exact_replay(L, seed, ties):
    Kbar = _rand_ns(L, seed, ties) + 3 * np.eye(L) * (1 if not ties else 0)
    K, _ = nonsym.scale_full(Kbar)
    F = nonsym.factor_ldu(K, 1e-2)
    piv, D, Lcols, Urows = left_looking_ldu(K, 1e-2)
    assert F.Ntau == len(piv)
    assert list(F.perm[:F.N]) == piv[:F.N]
    assert np.array_equal(F.D, np.array(D[:F.N], dtype=np.float32))
    pos = {p: k for k, p in enumerate(F.perm[:F.N])}
    for k in range(F.N):
        for i, v in Lcols[k].items():
            if i in pos and pos[i] > k:
                assert F.Lfac[pos[i], k] == np.float32(v)
        for j, v in Urows[k].items():
            if j in pos and pos[j] > k:
                assert F.Ufac[pos[j], k] == np.float32(v)


def test_ldu_reconstruction_and_pivot_rule():
    K, _ = nonsym.scale_full(hi.make_kbar("T8", 0).numpy())
    F = nonsym.factor_ldu(K, 1e-2)
    N, l1 = F.N, F.lam1
    Lf, Uf, D = F.Lfac.astype(np.float64), F.Ufac.astype(np.float64), F.D.astype(np.float64)
    R = Lf @ np.diag(D) @ Uf.T
    K11 = K[np.ix_(l1, l1)]
    eps32 = float(np.finfo(np.float32).eps)
    assert np.abs(R - K11).max() <= 50 * N * eps32 * np.abs(K11).max()
    assert np.all(np.abs(D[1:]) >= 1e-2 * np.abs(D[:-1]))          # [R4]
    # each pivot is the largest remaining |diagonal| of the FP64 Schur complement (up to FP32 noise)
    for k in (1, N // 3, N - 1):
        S = K - K[:, l1[:k]] @ np.linalg.solve(K[np.ix_(l1[:k], l1[:k])], K[l1[:k], :])
        rest = [i for i in range(K.shape[0]) if i not in set(l1[:k])]
        dg = np.abs(np.diag(S)[rest])
        assert abs(S[l1[k], l1[k]]) >= dg.max() * (1 - 1e-3)


def test_hard_lu_constructed_ranks():
    rng = np.random.default_rng(7)
    for r in (0, 1, 3, 6):
        A = rng.standard_normal((9, r)) @ rng.standard_normal((r, 9)) if r else np.zeros((9, 9))
        H = nonsym.factor_hard_lu(A, 1.0, 1e-10)
        assert H.kernel_dim == 9 - r
        if r:
            P = np.eye(9)[H.prow]
            Q = np.eye(9)[:, H.pcol]
            LU = H.Lh[:, :r] @ H.Uh[:r, :]
            assert np.abs(P @ A @ Q - LU).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("name", ["T8", "H8"])
def test_hybrid_solve_manufactured(name):
    K, _ = nonsym.scale_full(hi.make_kbar(name, 0).numpy())
    HF = nonsym.hybrid_factor(K, 1e-2, n_min=2)
    xs = np.arange(K.shape[0]) % 11.0
    b = K @ xs
    # consistent right-hand side: the residual of the minimum-coordinate solution is at rounding level
    x, info = nonsym.hybrid_solve(HF, b)
    assert np.abs(K @ x - b).max() <= 1e-12 * np.abs(b).max()
    # S22 against the dense FP64 Schur complement (LAPACK)
    l1, l2 = HF.F.lam1, HF.F.lam2
    Sd = K[np.ix_(l2, l2)] - K[np.ix_(l2, l1)] @ np.linalg.solve(K[np.ix_(l1, l1)], K[np.ix_(l1, l2)])
    assert np.abs(HF.S22 - Sd).max() <= 1e-10 * (np.abs(K).max() + np.abs(K[np.ix_(l2, l1)]).max() * np.abs(HF.X).max())
