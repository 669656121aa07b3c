"""The FP64 block mat-vec emulated on the int8 tensor cores (ozaki.cu, hf_matvec /
hf_gcr_opts.matvec = 2): pinned by exactness on integer data, by its error bound
against an extended-precision reference, and by the block GCR / Schur complement it
drives agreeing with the FP64 DMMA path."""
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


def _sym(A):
    return np.tril(A) + np.tril(A, -1).T


@pytest.mark.parametrize("L,n,bits", [(700, 40, 20), (1031, 33, 12), (256, 64, 24)])
def test_integer_operands_exact(ctx, L, n, bits):
    """Integer K and W whose exact product fits in 53 bits: every slice product is exact
    and no product is dropped (the operands need fewer than 8 x 7 bits), so Z is the
    exact integer product, bitwise -- a dropped or mis-scaled slice, a wrong sign or
    a transposed operand fails it."""
    from paper_2208_01907_b200 import hf
    rng = np.random.default_rng(L + n)
    K = _sym(rng.integers(-2 ** bits, 2 ** bits, size=(L, L))).astype(np.float64)
    W = rng.integers(-2 ** bits, 2 ** bits, size=(n, L)).astype(np.float64)   # (n, L) = L x n column-major
    exact = (W.astype(object) @ K.astype(object)).astype(np.float64)          # Z^T = W^T K (K symmetric)
    assert np.abs(exact).max() < 2.0 ** 53
    Kd = torch.from_numpy(K).cuda()
    Wd = torch.from_numpy(W).cuda()
    Z = hf.hf_matvec(ctx, Kd, Wd, "ozaki").cpu().numpy()
    assert np.array_equal(Z, exact)
    Zd = hf.hf_matvec(ctx, Kd, Wd, "dmma").cpu().numpy()
    assert np.array_equal(Zd, exact)
    # the residue form reconstructs the exact integer product and rounds it by a Horner
    # evaluation in FP64: within 16 ulps of the exact product
    Z2 = hf.hf_matvec(ctx, Kd, Wd, "ozaki2").cpu().numpy()
    assert np.all(np.abs(Z2 - exact) <= 16 * 2.0 ** -53 * np.abs(exact))


def _exp_bound(v):
    m = np.abs(v).max()
    return 0 if m == 0 else int(np.frexp(m)[1])


@pytest.mark.parametrize("s", [3, 5, 8])
def test_error_bound_vs_extended_precision(ctx, s):
    """Rows / columns with magnitudes spread over 2^-12..2^12: |Z - KW| <= (s + 2) 2^(-7s)
    2^(e_m + f_c) L + 8u|KW| entrywise (e_m, f_c: the row / column exponent bounds, the
    ozaki.cu bound), against an 80-bit long-double reference; at s = 8 the normwise
    error is at the FP64 DMMA product's level."""
    from paper_2208_01907_b200 import hf
    rng = np.random.default_rng(s)
    L, n = 768, 40
    d = 2.0 ** rng.uniform(-12, 12, size=L)
    K = _sym(rng.standard_normal((L, L))) * d[:, None] * d[None, :]
    W = rng.standard_normal((n, L)) * (2.0 ** rng.uniform(-8, 8, size=n))[:, None]
    ref = W.astype(np.longdouble) @ K.astype(np.longdouble)          # (n, L)
    Kd = torch.from_numpy(K).cuda()
    Wd = torch.from_numpy(W).cuda()
    Z = hf.hf_matvec(ctx, Kd, Wd, "ozaki", slices=s).cpu().numpy()
    em = np.array([_exp_bound(K[:, m]) for m in range(L)])
    fc = np.array([_exp_bound(W[c]) for c in range(n)])
    bound = (s + 2) * 2.0 ** (-7 * s) * np.ldexp(1.0, em[None, :] + fc[:, None]) * L
    bound = bound + 8 * 2.0 ** -53 * np.abs(ref).astype(np.float64)
    err = np.abs((Z.astype(np.longdouble) - ref).astype(np.float64))
    assert (err <= bound).all(), float((err / bound).max())
    if s >= 3:   # the bound is not vacuous: the error grows as slices are removed
        Zs = hf.hf_matvec(ctx, Kd, Wd, "ozaki", slices=2).cpu().numpy()
        assert np.abs(Zs - ref.astype(np.float64)).max() > err.max()
    if s == 8:
        Zd = hf.hf_matvec(ctx, Kd, Wd, "dmma").cpu().numpy()
        nref = np.linalg.norm(ref.astype(np.float64))
        e_oz = np.linalg.norm((Z - ref).astype(np.float64)) / nref
        e_dm = np.linalg.norm((Zd - ref).astype(np.float64)) / nref
        # rows spread over 2^24: the slices bound the error by the ROW maximum, FP64 by the
        # entries -- within an order of magnitude of the DMMA product here
        assert e_oz <= max(10 * e_dm, 1e-15), (e_oz, e_dm)


def test_residue_form_error_bound_vs_extended_precision(ctx):
    """ozaki2.cu: |Z - KW| <= Lk 2^(e_m + f_c - 52) (the 53-bit truncations of both operands)
    + 2^-48 |KW| (the FP64 Horner evaluation) entrywise, rows / columns spread over 2^+-12;
    at the FP64 DMMA product's level normwise."""
    from paper_2208_01907_b200 import hf
    rng = np.random.default_rng(21)
    L, n = 768, 40
    d = 2.0 ** rng.uniform(-12, 12, size=L)
    K = _sym(rng.standard_normal((L, L))) * d[:, None] * d[None, :]
    W = rng.standard_normal((n, L)) * (2.0 ** rng.uniform(-8, 8, size=n))[:, None]
    ref = W.astype(np.longdouble) @ K.astype(np.longdouble)
    Kd, Wd = torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda()
    Z = hf.hf_matvec(ctx, Kd, Wd, "ozaki2").cpu().numpy()
    em = np.array([_exp_bound(K[:, m]) for m in range(L)])
    fc = np.array([_exp_bound(W[c]) for c in range(n)])
    bound = L * np.ldexp(1.0, em[None, :] + fc[:, None] - 52) + 2.0 ** -48 * np.abs(ref).astype(np.float64)
    err = np.abs((Z.astype(np.longdouble) - ref).astype(np.float64))
    assert (err <= bound).all(), float((err / bound).max())
    Zd = hf.hf_matvec(ctx, Kd, Wd, "dmma").cpu().numpy()
    nref = np.linalg.norm(ref.astype(np.float64))
    e2 = np.linalg.norm((Z - ref).astype(np.float64)) / nref
    ed = np.linalg.norm((Zd - ref).astype(np.float64)) / nref
    assert e2 <= max(10 * ed, 1e-15), (e2, ed)


@pytest.mark.parametrize("mv", ["ozaki", "ozaki2"])
@pytest.mark.parametrize("name,seed", [("P2048", 0), ("S24", 0), ("P4096", 1)])
def test_schur_gcr_ozaki_matches_dmma(ctx, name, seed, mv):
    """The block GCR + Schur complement with the emulated mat-vec: same iteration count
    (+-1) and S22 within 1e-9 of the FP64 DMMA run, true residuals <= 1e-12, and the
    oracle's S22 within the stage-2 parity tolerance."""
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    K = Kb.cuda().contiguous()
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=max(spec.n_min, 32))
    hy1, i1, S1 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True, matvec="dmma")
    hy2, i2, S2 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True, matvec=mv)
    assert abs(i1.iters - i2.iters) <= 1
    assert i2.max_rel_res_true <= 1e-12 and i1.max_rel_res_true <= 1e-12
    Ko, _ = oracle.scale(Kb.numpy())
    HF = oracle.hybrid_factor(Ko, tau=spec.tau, n_min=max(spec.n_min, 32))
    K11, K12, K21, K22 = oracle.extract_blocks(HF.K, HF.F)
    # S22 = K22 - K21 X12 cancels: differences are measured against the sizes of its two
    # terms, as the stage-2 parity bar does [R17]
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    assert np.linalg.norm(S2 - S1) / den <= 1e-12
    assert np.linalg.norm(S2 - HF.S22) / den <= 1e-10
    hy1.close()
    hy2.close()
    lf.close()


def test_edge_cases_extreme_scales_and_zeros(ctx):
    """Rows of K spread over 2^-600..2^600 (the row exponents must not overflow or lose the
    scale), an all-zero row / column of K, an all-zero column of W, a W column of subnormal
    magnitude, L not a multiple of 16 (the zero-padded slices): entrywise within the bound of
    test_error_bound_vs_extended_precision, zeros exactly zero."""
    from paper_2208_01907_b200 import hf
    rng = np.random.default_rng(11)
    L, n, s = 333, 36, 8
    d = 2.0 ** rng.integers(-300, 300, size=L).astype(np.float64)
    K = _sym(rng.standard_normal((L, L))) * d[:, None] * d[None, :]
    K[17, :] = 0.0
    K[:, 17] = 0.0
    W = rng.standard_normal((n, L))
    W[3] = 0.0
    W[5] *= 2.0 ** -1060                      # subnormal column
    W[:, 17] = 1.0
    ref = W.astype(np.longdouble) @ K.astype(np.longdouble)
    Z = hf.hf_matvec(ctx, torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda(), "ozaki").cpu().numpy()
    assert np.all(Z[3] == 0.0) and np.all(Z[:, 17] == 0.0)
    em = np.array([_exp_bound(K[:, m]) for m in range(L)])
    fc = np.array([_exp_bound(W[c]) for c in range(n)])
    bound = (s + 2) * np.ldexp(np.ldexp(1.0, -7 * s) * L, em[None, :] + fc[:, None])
    bound = bound + 8 * 2.0 ** -53 * np.abs(ref).astype(np.float64) + 1e-320
    err = np.abs((Z.astype(np.longdouble) - ref).astype(np.float64))
    assert np.all(np.isfinite(Z))
    assert (err <= bound).all(), float((err / bound).max())
