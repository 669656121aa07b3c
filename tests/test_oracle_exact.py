"""Pins of oracle/exact.py (the exact-rational Schur complement and rank used as
the reference of the double-double path, NEXT-1): closed forms, a hand-worked
block case, LAPACK agreement to FP64 rounding, constructed ranks."""
from fractions import Fraction
from math import comb

import numpy as np
import scipy.linalg as sla

from oracle import exact


def test_solve_hilbert_inverse_closed_form():
    # (H^{-1})_ij = (-1)^(i+j) (i+j+1) C(n+i, n-j-1) C(n+j, n-i-1) C(i+j, i)^2  (0-based)
    n = 6
    H = [[Fraction(1, i + j + 1) for j in range(n)] for i in range(n)]
    I = [[Fraction(int(i == j)) for j in range(n)] for i in range(n)]
    X = exact.solve(H, I)
    for i in range(n):
        for j in range(n):
            want = (-1) ** (i + j) * (i + j + 1) * comb(n + i, n - j - 1) * comb(n + j, n - i - 1) * comb(i + j, i) ** 2
            assert X[i][j] == want


def test_schur_by_hand():
    # K11 = [[4, 2], [2, 3]] (det 8, inverse [[3, -2], [-2, 4]] / 8), K12 = [1, 0]^T, K22 = 2
    K = np.array([[4.0, 2.0, 1.0], [2.0, 3.0, 0.0], [1.0, 0.0, 2.0]])
    S = exact.schur(K, [0, 1], [2])
    assert S == [[Fraction(13, 8)]]
    # the partition may interleave: Lambda_1 = {0, 2}, Lambda_2 = {1}: 3 - [2 0] [[4 1][1 2]]^{-1} [2 0]^T
    S = exact.schur(K, [0, 2], [1])
    assert S == [[Fraction(3) - Fraction(4) * Fraction(2, 7)]]


def test_schur_matches_lapack_to_fp64_rounding():
    rng = np.random.default_rng(3)
    B = rng.standard_normal((24, 24))
    K = B @ B.T + 24 * np.eye(24)
    lam1, lam2 = list(range(0, 24, 2)) + list(range(1, 20, 2)), [21, 23]
    S = exact.schur(K, lam1, lam2)
    K11, K12, K22 = K[np.ix_(lam1, lam1)], K[np.ix_(lam1, lam2)], K[np.ix_(lam2, lam2)]
    Sd = K22 - K12.T @ sla.solve(K11, K12, assume_a="pos")
    hi, lo = exact.to_float_pair(S)
    assert np.max(np.abs(hi - Sd)) <= 1e-12 * np.max(np.abs(Sd))
    assert exact.rel_err(S, hi, lo) <= 1e-30          # the (hi, lo) pair carries ~106 bits


def test_rank_constructed():
    rng = np.random.default_rng(5)
    for r in (0, 1, 3, 6):
        B = rng.integers(-4, 5, size=(9, r)).astype(np.float64)
        A = B @ B.T
        want = np.linalg.matrix_rank(B) if r else 0      # small integers: FP64 rank is exact here
        assert exact.rank(exact.to_fractions(A)) == want
    assert exact.rank(exact.to_fractions(np.eye(5))) == 5
    # a rank deficiency far below FP64 resolution is still seen exactly
    A = np.array([[1.0, 1.0], [1.0, 1.0 + 2.0 ** -52]])
    assert exact.rank(exact.to_fractions(A)) == 2
    A = np.array([[1.0, 2.0 ** -40], [2.0 ** -40, 2.0 ** -80]])
    assert exact.rank(exact.to_fractions(A)) == 1
