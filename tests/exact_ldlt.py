"""Exact-arithmetic emulation of the FP32 stage-1 rules, used ONLY as a pin
for the oracle (tests/test_oracle_lowprec.py).

It is structurally different from oracle/lowprec.c on purpose:
  * LEFT-looking: no trailing matrix is ever formed; every entry v_IJ^(k) is
    rebuilt from the FP32 start value by replaying the pivots in order;
  * no row/column swaps: indices stay original, the pivot set is a Python set;
  * arithmetic in exact rationals (fractions.Fraction) with an explicit,
    hand-written IEEE binary32 round-to-nearest-even, instead of the C
    library's fmaf / sqrtf / division.
Python's float is binary64; sqrt and division of binary32 operands computed
in binary64 and then rounded to binary32 are correctly rounded (p=53 >= 2*24+2),
so only the FMA needs the exact rational path.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def rn32(x: Fraction) -> float:
    """Round an exact rational to the nearest binary32 (ties to even)."""
    if x == 0:
        return 0.0
    sgn = -1 if x < 0 else 1
    a = abs(x)
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)                      # subnormal range: quantum 2^-149
    quantum = Fraction(2) ** (e - 23)
    n = a / quantum
    fl = n.numerator // n.denominator
    rem = n - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    val = fl * quantum
    if val >= Fraction(2) ** 128:
        return sgn * math.inf
    return float(np.float32(sgn * float(val)))   # exact: val is representable


def fmaf_exact(a: float, b: float, c: float) -> float:
    return rn32(Fraction(a) * Fraction(b) + Fraction(c))


def f32(x: float) -> float:
    return float(np.float32(x))


def left_looking_ldlt(K: np.ndarray, tau: float):
    """Returns (pivots, D, Lcols) with Lcols[k] = {I: L_{I,k}} for the
    tau-rule alone (no floor, no enlargement)."""
    L = K.shape[0]
    v0 = {}
    for i in range(L):
        for j in range(i + 1):
            v0[(i, j)] = f32(float(np.float32(K[i, j])))

    def key(i, j):
        return (i, j) if i >= j else (j, i)

    piv, D, S, sig, Lcols = [], [], [], [], []   # S[t] = {I: s_I^t}
    done = set()

    def entry(i, j, k):
        """v_IJ^(k): start value, then one exact-rounded FMA per pivot t < k."""
        v = v0[key(i, j)]
        for t in range(k):
            v = fmaf_exact(-sig[t] * S[t][i], S[t][j], v)
        return v

    for k in range(L):
        cands = [i for i in range(L) if i not in done]
        best, bd = None, None
        for i in cands:                              # ascending original index
            d = entry(i, i, k)
            if best is None or abs(d) > abs(bd):
                best, bd = i, d
        d = bd
        if k == 0 and d == 0.0:
            break
        if k > 0 and abs(float(d)) < tau * abs(float(D[-1])):
            break
        r = f32(math.sqrt(abs(d)))
        sg = 1.0 if d > 0 else -1.0
        s, lc = {}, {}
        for i in cands:
            if i == best:
                continue
            c = entry(i, best, k)
            s[i] = f32(c / r)
            lc[i] = f32(c / d)
        piv.append(best)
        D.append(d)
        S.append(s)
        sig.append(sg)
        Lcols.append(lc)
        done.add(best)
    return piv, D, Lcols


def left_looking_ldu(K: np.ndarray, tau: float):
    """NEXT-3 pin: the nonsymmetric FP32 rule [R19] by left-looking exact
    replay (no swaps, original indices): v_IJ^(k) = start value with one
    exact-rounded fmaf(-l_I^t, r_J^t, .) per earlier pivot t; l_I = RN32(c_I/d),
    r_J = v_{P J}.  Returns (pivots, D, Lcols, Urows) for the tau-rule alone,
    Lcols[k] = {I: l_I^k}, Urows[k] = {J: RN32(r_J^k / d_k)}."""
    L = K.shape[0]
    v0 = {(i, j): f32(float(np.float32(K[i, j]))) for i in range(L) for j in range(L)}
    piv, D, Ls, Rs, Lcols, Urows = [], [], [], [], [], []
    done = set()

    def entry(i, j, k):
        v = v0[(i, j)]
        for t in range(k):
            v = fmaf_exact(-Ls[t][i], Rs[t][j], v)
        return v

    for k in range(L):
        cands = [i for i in range(L) if i not in done]
        best, bd = None, None
        for i in cands:
            d = entry(i, i, k)
            if best is None or abs(d) > abs(bd):
                best, bd = i, d
        d = bd
        if k == 0 and d == 0.0:
            break
        if k > 0 and abs(float(d)) < tau * abs(float(D[-1])):
            break
        lc, rr, ur = {}, {}, {}
        for i in cands:
            if i == best:
                continue
            lc[i] = f32(entry(i, best, k) / d)
            rr[i] = entry(best, i, k)
            ur[i] = f32(rr[i] / d)
        piv.append(best)
        D.append(d)
        Ls.append(lc)
        Rs.append(rr)
        Lcols.append(lc)
        Urows.append(ur)
        done.add(best)
    return piv, D, Lcols, Urows


def left_looking_ldlt_blocks(K: np.ndarray, tau: float, blk, nblk: int):
    """NEXT-4 pin: the multi-block rule by left-looking exact replay: candidates of
    the current block only (ties -> smallest original index), ratio test against the
    previously accepted pivot [R21] (the very first pivot against 0 only), then a final
    pass over everything left.  Returns (pivots, D, Lcols, Ntau)."""
    L = K.shape[0]
    v0 = {}
    for i in range(L):
        for j in range(i + 1):
            v0[(i, j)] = f32(float(np.float32(K[i, j])))

    def key(i, j):
        return (i, j) if i >= j else (j, i)

    piv, D, S, sig, Lcols = [], [], [], [], []
    done = set()

    def entry(i, j, k):
        v = v0[key(i, j)]
        for t in range(k):
            v = fmaf_exact(-sig[t] * S[t][i], S[t][j], v)
        return v

    cur, first, k = 0, True, 0
    Ntau = L
    while k < L:
        cands = [i for i in range(L) if i not in done and (cur >= nblk or blk[i] == cur)]
        best, bd = None, None
        for i in cands:
            d = entry(i, i, k)
            if best is None or abs(d) > abs(bd):
                best, bd = i, d
        fail = best is None or (bd == 0.0 if first else abs(float(bd)) < tau * abs(float(D[-1])))
        if fail:
            if cur < nblk:
                cur += 1
                continue
            Ntau = k
            break
        d = bd
        r = f32(math.sqrt(abs(d)))
        sg = 1.0 if d > 0 else -1.0
        s, lc = {}, {}
        for i in range(L):
            if i in done or i == best:
                continue
            c = entry(i, best, k)
            s[i] = f32(c / r)
            lc[i] = f32(c / d)
        piv.append(best)
        D.append(d)
        S.append(s)
        sig.append(sg)
        Lcols.append(lc)
        done.add(best)
        first = False
        k += 1
    return piv, D, Lcols, Ntau
