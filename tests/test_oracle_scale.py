"""Pins for the oracle's scaling step (sec. 2 opening) [R1]."""
import numpy as np
import pytest

import oracle


def test_spec_examples():
    # [[4,2],[2,1]] -> Q = diag(1/2, 1), K = [[1,1],[1,1]]  (forced analytically)
    K, q = oracle.scale(np.array([[4.0, 2.0], [2.0, 1.0]]))
    assert np.array_equal(q, [0.5, 1.0])
    assert np.array_equal(K, [[1.0, 1.0], [1.0, 1.0]])
    # identity -> identity
    K, q = oracle.scale(np.eye(5))
    assert np.array_equal(q, np.ones(5)) and np.array_equal(K, np.eye(5))
    # zero diagonal -> Q_ii = 1 ("otherwise [Q]_ii = 1")
    K, q = oracle.scale(np.array([[0.0, 3.0], [3.0, 0.0]]))
    assert np.array_equal(q, [1.0, 1.0]) and np.array_equal(K, [[0.0, 3.0], [3.0, 0.0]])


def test_negative_diagonal_takes_abs():
    K, q = oracle.scale(np.array([[-4.0, 2.0], [2.0, 9.0]]))
    assert np.array_equal(q, [0.5, 1.0 / 3.0])
    assert K[0, 0] == -1.0 and K[1, 1] == 1.0
    assert K[1, 0] == K[0, 1] == (1.0 / 3.0 * 2.0) * 0.5


@pytest.mark.parametrize("seed", range(3))
def test_random_matches_dense_formula_and_reads_lower_only(seed):
    rng = np.random.default_rng(seed)
    L = 37
    A = rng.standard_normal((L, L)) * 10.0 ** rng.uniform(-3, 3, (L, 1))
    Kb = np.tril(A) + np.tril(A, -1).T
    Kb[5, 5] = 0.0
    K, q = oracle.scale(Kb)
    dense = np.diag(q) @ Kb @ np.diag(q)          # different evaluation order
    off = ~np.eye(L, dtype=bool)
    assert np.allclose(K[off], dense[off], rtol=4e-16 * 4, atol=0)
    assert set(np.diag(K)) <= {-1.0, 0.0, 1.0}
    assert K[5, 5] == 0.0 and q[5] == 1.0
    assert np.array_equal(K, K.T)
    # garbage in the strict upper triangle must not matter
    Kg = Kb.copy()
    Kg[np.triu_indices(L, 1)] = np.nan
    K2, q2 = oracle.scale(Kg)
    assert np.array_equal(K2, K) and np.array_equal(q2, q)


def test_idempotent():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((20, 20))
    Kb = A + A.T + np.diag(rng.uniform(1, 5, 20))
    K, _ = oracle.scale(Kb)
    K2, q2 = oracle.scale(K)
    assert np.array_equal(q2, np.ones(20)) and np.array_equal(K2, K)
