"""oracle.exact -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Exact rational arithmetic (fractions.Fraction) for the NEXT-1 parity of the
(double, double-double) pair.  The double-double block GCR converges to the
Schur complement of Eq. (2) (Alg. 1 step 4 P:191),

    S22 = K22 - K21 K11^{-1} K12,

within double-double precision; its plain definition, evaluated exactly from
the (exactly representable) double inputs, is the reference.  Likewise the
hard factorization's kernel dimension is compared with the exact
rank deficiency of that S22.

Plain Gaussian elimination in Fractions -- slow (O(n^3) big-rational
operations), for the small sizes of the tests only (L <= ~96).

Pins (tests/test_oracle_exact.py): Hilbert-matrix inverse (closed form),
S22 of a 2x2 block case by hand, agreement with the FP64 LAPACK Schur
complement to FP64 rounding, rank of constructed rank-r matrices.
"""
from fractions import Fraction

import numpy as np


def to_fractions(A):
    """Every float64 entry exactly (Fraction(float) is exact for finite floats)."""
    A = np.asarray(A, dtype=np.float64)
    return [[Fraction(float(A[i, j])) for j in range(A.shape[1])] for i in range(A.shape[0])]


def solve(A, B):
    """X = A^{-1} B exactly (A square nonsingular, lists of Fractions); Gaussian
    elimination with partial pivoting on the first nonzero entry of each column."""
    n = len(A)
    m = len(B[0]) if n else 0
    M = [list(A[i]) + list(B[i]) for i in range(n)]
    for k in range(n):
        p = next((i for i in range(k, n) if M[i][k] != 0), None)
        if p is None:
            raise ZeroDivisionError("singular matrix")
        M[k], M[p] = M[p], M[k]
        piv = M[k][k]
        rowk = [v / piv for v in M[k]]
        M[k] = rowk
        for i in range(n):
            if i != k and M[i][k] != 0:
                f = M[i][k]
                M[i] = [a - f * b for a, b in zip(M[i], rowk)]
    return [row[n:n + m] for row in M]


def schur(K, lam1, lam2):
    """S22 = K22 - K21 K11^{-1} K12 exactly (Eq. 2).  K: float64 L x L,
    lam1 / lam2: index lists.  Returns an n2 x n2 list of Fractions."""
    F = to_fractions(K)
    K11 = [[F[i][j] for j in lam1] for i in lam1]
    K12 = [[F[i][j] for j in lam2] for i in lam1]
    K21 = [[F[i][j] for j in lam1] for i in lam2]
    K22 = [[F[i][j] for j in lam2] for i in lam2]
    X = solve(K11, K12) if lam1 else [[] for _ in lam1]
    n1, n2 = len(lam1), len(lam2)
    return [[K22[i][j] - sum((K21[i][k] * X[k][j] for k in range(n1)), Fraction(0)) for j in range(n2)]
            for i in range(n2)]


def rank(S):
    """Exact rank of a list-of-Fractions matrix (Gaussian elimination)."""
    M = [list(r) for r in S]
    n, m = len(M), (len(M[0]) if M else 0)
    r = 0
    for c in range(m):
        p = next((i for i in range(r, n) if M[i][c] != 0), None)
        if p is None:
            continue
        M[r], M[p] = M[p], M[r]
        for i in range(r + 1, n):
            if M[i][c] != 0:
                f = M[i][c] / M[r][c]
                M[i] = [a - f * b for a, b in zip(M[i], M[r])]
        r += 1
        if r == n:
            break
    return r


def to_float_pair(S):
    """Nearest (hi, lo) double pair of each Fraction: hi = RN(x), lo = RN(x - hi)."""
    n, m = len(S), len(S[0]) if S else 0
    hi = np.zeros((n, m))
    lo = np.zeros((n, m))
    for i in range(n):
        for j in range(m):
            h = float(S[i][j])
            hi[i, j] = h
            lo[i, j] = float(S[i][j] - Fraction(h))
    return hi, lo


def rel_err(S, hi, lo):
    """max |(hi + lo) - S| / max |S| evaluated exactly (S Fractions, hi/lo float arrays)."""
    n = len(S)
    num = Fraction(0)
    den = Fraction(0)
    for i in range(n):
        for j in range(n):
            d = abs(Fraction(float(hi[i, j])) + Fraction(float(lo[i, j])) - S[i][j])
            num = max(num, d)
            den = max(den, abs(S[i][j]))
    return float(num / den) if den else float(num)
