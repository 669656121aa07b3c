"""Host checks of the residue (Chinese remainder) mat-vec's number theory (ozaki2.cu), read from
the kernel source so a changed constant is caught without a GPU: the 16 moduli are pairwise
coprime, their product covers the exact integer products' range, the int32 accumulation of one
modulus cannot overflow, and the chunked residue / Garner reconstruction steps the kernels take
recover random 106-bit products exactly (python integers as the reference), and the combine's
FP32 Garner steps -- every rounding emulated exactly -- give the canonical digits."""
from fractions import Fraction

import numpy as np
import math
import os
import random
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "paper_2208_01907_b200", "csrc", "ozaki2.cu")).read()
MODS = [int(x) for x in re.search(r"kModH\[NMOD\] = \{([^}]*)\}", SRC).group(1).split(",")]
LMAX = int(re.search(r"HF_REQUIRE\(L <= (\d+)", SRC).group(1))


def test_moduli_pairwise_coprime_and_in_int8_range():
    assert len(MODS) == 16 and len(set(MODS)) == 16
    assert all(2 <= m <= 256 for m in MODS)
    for i in range(16):
        for j in range(i):
            assert math.gcd(MODS[i], MODS[j]) == 1, (MODS[i], MODS[j])


def test_product_range_and_int32_accumulation():
    M = math.prod(MODS)
    # |C'| <= L 2^53 2^53 must lie in (-M/2, M/2) for every admissible L
    assert LMAX * 2 ** 106 < M // 2
    # one modulus' GEMM: L products of symmetric residues, |r| <= 128
    assert LMAX * 128 * 128 < 2 ** 31


def _residue(x, m):
    """The kernel's steps: signed chunks c0 + c1 2^18 + c2 2^36, offset, unsigned mod, symmetric."""
    c0, c1, c2 = x & 0x3FFFF, (x >> 18) & 0x3FFFF, x >> 36
    p18 = (1 << 18) % m
    p36 = p18 * p18 % m
    off = ((1 << 25) + m - 1) // m * m
    y = c0 + c1 * p18 + c2 * p36 + off
    assert 0 <= y < 2 ** 27
    r = y % m
    return r - m if 2 * r >= m else r


def _garner(res):
    """Symmetric mixed-radix digits and the Horner sum (exact here; FP64 in the kernel)."""
    v = []
    for l, m in enumerate(MODS):
        s = res[l] % m
        P = 1
        for j in range(l):
            s -= v[j] * (P % m)
            P *= MODS[j]
        t = s % m * pow(P % m, -1, m) % m
        v.append(t - m if 2 * t >= m else t)
    X = v[-1]
    for l in range(14, -1, -1):
        X = X * MODS[l] + v[l]
    return X


def test_chunked_residues_and_garner_recover_products():
    rng = random.Random(7)
    for _ in range(60):
        L = rng.choice([1, 2, 17, 300])
        a = [rng.randint(-(2 ** 53) + 1, 2 ** 53 - 1) for _ in range(L)]
        b = [rng.randint(-(2 ** 53) + 1, 2 ** 53 - 1) for _ in range(L)]
        exact = sum(x * y for x, y in zip(a, b))
        res = []
        for m in MODS:
            ra = [_residue(x, m) for x in a]
            rb = [_residue(y, m) for y in b]
            assert all(-128 <= r <= 127 for r in ra + rb)
            assert all((r - x) % m == 0 for r, x in zip(ra, a))
            res.append(sum(x * y for x, y in zip(ra, rb)))   # the int32 GEMM entry
        assert _garner(res) == exact


def test_garner_at_the_range_ends():
    """L = LMAX entries all at +-(2^53 - 1): the largest |C'| the kernels admit."""
    x = 2 ** 53 - 1
    for sa, sb in [(1, 1), (1, -1), (-1, -1)]:
        res = [LMAX * _residue(sa * x, m) * _residue(sb * x, m) for m in MODS]
        assert _garner(res) == LMAX * sa * sb * x * x


MAGIC = 3 * 2 ** 22   # 1.5 2^23


def _sym(r, m):
    r %= m
    return r - m if 2 * r > m else r


def _round_mod_f32(s, m):
    """r = s - m rint(s/m) with q from fma(s, fl32(1/m), 1.5 2^23) - 1.5 2^23 (FP32: the fma's one
    rounding lands in [2^23, 2^24), where the FP32 grid is the integers; ties to even)."""
    assert abs(s) < 2 ** 24
    inv = Fraction(float(np.float32(1.0) / np.float32(m)))
    t = round(Fraction(s) * inv + MAGIC)
    assert 2 ** 23 <= t < 2 ** 24
    return s - (t - MAGIC) * m


def _garner_f32(x):
    """k_oz2_combine's digits: s = lo + hi (2^16 mod m) - sum_j v_j (P_j mod m), r = round_mod(s),
    v = round_mod(r Pinv)."""
    v = []
    for l, m in enumerate(MODS):
        lo, hi = x[l] & 0xFFFF, x[l] >> 16
        s = lo + hi * _sym(65536, m)
        P = 1
        for j in range(l):
            s -= v[j] * _sym(P % m, m)
            P *= MODS[j]
        assert abs(s) < 4.6e6
        r = _round_mod_f32(s, m)
        assert 2 * abs(r) <= m
        d = _round_mod_f32(r * _sym(pow(P % m, -1, m), m), m)
        assert 2 * abs(d) <= m and (d - (x[l] - sum(v[j] * math.prod(MODS[:j]) for j in range(l))) *
                                     pow(P % m, -1, m)) % m == 0
        v.append(d)
    X = 0
    for l in range(15, -1, -1):
        X = X * MODS[l] + v[l]
    return X


def test_fp32_garner_digits_reconstruct():
    rng = random.Random(11)
    M = math.prod(MODS)
    lim = LMAX * 128 * 128   # |int32 GEMM sum|
    for _ in range(400):
        C = rng.randint(-LMAX * 2 ** 106, LMAX * 2 ** 106)
        # int32 sums congruent to C mod m_l anywhere in their admissible range
        x = [(_sym(C, m) + m * rng.randint(-(lim // m) + 1, lim // m - 1)) for m in MODS]
        assert all(abs(t) < 2 ** 31 for t in x)
        assert _garner_f32(x) == C
    for C in (LMAX * 2 ** 106, -LMAX * 2 ** 106, 0, 1, -1, M // 2 ** 3):
        assert _garner_f32([_sym(C, m) for m in MODS]) == C
