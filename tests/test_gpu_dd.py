"""NEXT-1, the (double, double-double) pair: FP64 canonical stage 1
(prec 64) + block GCR, Schur complement and hard factorization in double-double
(hf_schur_gcr_dd), against the EXACT rational Schur complement of Eq. (2)
 and its exact rank (oracle/exact.py).

Bars: normwise e_S = ||S22_dd - S||_max / (||K22|| + ||K21|| ||X||)_max <= 1e-26
(double-double unit roundoff 2^-104 ~ 5e-32, times the growth of the GCR's
stopping tolerance 1e-28 through X); the FP64 path on the same inputs is
reported beside it and must be >= 1e6 times less accurate unless it is itself
below 1e-26; kernel_dim == n2 - rank(S) exactly."""
import numpy as np
import pytest
import torch

import hf_inputs as hi
from hf_inputs.configs import ConfigSpec
from oracle import exact

pytestmark = pytest.mark.gpu

CASES = {
    "P48": ConfigSpec("P48", "planted", 48, n_min=3, n_hard=3, u_hard=(-10.0, -8.0)),
    "P64": ConfigSpec("P64", "planted", 64, n_min=4, n_hard=4, u_hard=(-12.0, -6.0)),
    "S4": ConfigSpec("S4", "saddle", 2 * 4 * 4 + 2 * 2 * 2, grid=4, jump=1e4),
    "S6": ConfigSpec("S6", "saddle", 2 * 6 * 6 + 2 * 3 * 3, grid=6, jump=1e4),
    "N8": ConfigSpec("N8", "neumann", 8 * 8, grid=8, n_incl=1, incl_size=2),
}


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


def _run(ctx, spec, seed):
    from paper_2208_01907_b200 import hf
    K = hi.make_kbar(spec, seed).to("cuda")
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min, prec=64)
    hy, info, S = hf.hf_schur_gcr_dd(ctx, K, lf, want_S22_host=True)
    return K, lf, hy, info, S


@pytest.mark.parametrize("name,seed", [("P48", 0), ("P48", 1), ("P64", 0), ("S4", 0), ("S6", 0), ("N8", 0)])
def test_dd_schur_vs_exact(ctx, name, seed):
    from paper_2208_01907_b200 import hf
    spec = CASES[name]
    K, lf, hy, info, S = _run(ctx, spec, seed)
    perm, _, _ = lf.export64()
    N, n2 = lf.N, lf.n2
    assert n2 >= 1
    lam1, lam2 = [int(i) for i in perm[:N]], [int(i) for i in perm[N:]]
    Kh = K.cpu().numpy()
    Sx = exact.schur(Kh, lam1, lam2)
    Shi, Slo = S
    # normwise error against the exact S22 ([R17] form)
    K22 = Kh[np.ix_(lam2, lam2)]
    K21 = Kh[np.ix_(lam2, lam1)]
    Xhi, Xlo, _, _ = hy.export_dd()
    X = Xhi.cpu().numpy()[lam1]
    den = np.abs(K22).max() + np.abs(K21).sum(1).max() * np.abs(X).max()
    num = exact.rel_err(Sx, Shi, Slo) * max(abs(float(v)) for r in Sx for v in r)
    e_dd = num / den
    assert e_dd <= 1e-26, e_dd
    assert info.max_rel_res_true <= 1e-26
    # the FP64 path on the same inputs (the (double, double) hybrid)
    hy64, _, S64 = hf.hf_schur_gcr(ctx, K, lf, want_S22_host=True)
    e_64 = exact.rel_err(Sx, S64, np.zeros_like(S64)) * max(abs(float(v)) for r in Sx for v in r) / den
    assert e_dd <= 1e-26 and (e_64 <= 1e-26 or e_64 >= 1e6 * e_dd), (e_dd, e_64)
    # hard factorization in double-double: kernel dimension = exact rank deficiency
    kd = hf.hf_factor_hard(ctx, hy, eps_ker=1e-20)
    assert kd == n2 - exact.rank(Sx)
    hy64.close()
    hy.close()
    lf.close()


def test_dd_requires_fp64_factor(ctx):
    from paper_2208_01907_b200 import hf
    spec = CASES["P48"]
    K = hi.make_kbar(spec, 0).to("cuda")
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=spec.tau, n_min=spec.n_min)   # FP32 factor
    with pytest.raises(hf.HFError) as e:
        hf.hf_schur_gcr_dd(ctx, K, lf)
    assert e.value.status == hf.HF_ERR_INVALID_ARG
    lf.close()


def test_dd_solve_is_refused_by_the_double_entry(ctx):
    from paper_2208_01907_b200 import hf
    K, lf, hy, info, S = _run(ctx, CASES["P48"], 0)
    hf.hf_factor_hard(ctx, hy, eps_ker=1e-20)
    b = torch.ones(lf.L, dtype=torch.float64, device="cuda")
    with pytest.raises(hf.HFError) as e:
        hf.hf_solve(ctx, hy, b)
    assert e.value.status == hf.HF_ERR_STATE
    hy.close()
    lf.close()


@pytest.mark.parametrize("name,seed", [("P48", 0), ("P64", 0), ("S4", 0), ("N8", 0)])
def test_dd_solve_exact_residual(ctx, name, seed):
    """Alg. 2 in double-double: the residual b - K x evaluated EXACTLY (Fractions), b = K x*
    with x*_i = i mod 11.  Bar: max |b - K x| / max |b| <= 1e-26 (the block-GCR
    tolerance 1e-28 times the size of b); the FP64 path's exact residual is reported beside
    it and must be >= 1e6 times larger unless itself below the bar.  (The FORWARD error is
    kappa(K) times this -- up to 1e13 on the planted cases -- so it is not the bar.)"""
    from fractions import Fraction
    from paper_2208_01907_b200 import hf
    spec = CASES[name]
    K, lf, hy, info, S = _run(ctx, spec, seed)
    hf.hf_factor_hard(ctx, hy, eps_ker=1e-20)
    Kh = K.cpu().numpy()
    L = Kh.shape[0]
    xs = hi.manufactured_x(L).numpy()
    b = Kh @ xs
    F = exact.to_fractions(Kh)
    bf = [Fraction(float(v)) for v in b]

    def exact_res(x):
        return float(max(abs(bf[i] - sum((F[i][j] * x[j] for j in range(L)), Fraction(0))) for i in range(L))
                     / max(abs(v) for v in bf))

    xh, xl, sinfo = hf.hf_solve_dd(ctx, hy, torch.from_numpy(b).cuda())
    xh, xl = xh.cpu().numpy(), xl.cpu().numpy()
    res_dd = exact_res([Fraction(float(xh[i])) + Fraction(float(xl[i])) for i in range(L)])
    assert res_dd <= 1e-26, res_dd
    hy64, _, _ = hf.hf_schur_gcr(ctx, K, lf)
    hf.hf_factor_hard(ctx, hy64, eps_ker=1e-10)
    x64, _ = hf.hf_solve(ctx, hy64, torch.from_numpy(b).cuda())
    x64 = x64.cpu().numpy()
    res_64 = exact_res([Fraction(float(x64[i])) for i in range(L)])
    assert res_64 <= 1e-26 or res_64 >= 1e6 * res_dd, (res_dd, res_64)
    hy64.close()
    hy.close()
    lf.close()


def test_dd_degenerate(ctx):
    """n2 = 0 (nothing postponed: empty S22, hard factor a no-op, the solve is the block GCR
    alone) and a 1 x 1 system through the double-double path."""
    from paper_2208_01907_b200 import hf
    K = torch.diag(torch.tensor([4.0, 2.0, 1.0, 0.5], dtype=torch.float64)).cuda()
    hf.hf_scale(ctx, K)
    lf = hf.hf_factor_lowprec(ctx, K, tau=1e-2, prec=64)
    assert lf.n2 == 0
    hy, info, _ = hf.hf_schur_gcr_dd(ctx, K, lf)
    assert hf.hf_factor_hard(ctx, hy, eps_ker=1e-20) == 0
    b = torch.tensor([1.0, -2.0, 3.0, 0.25], dtype=torch.float64, device="cuda")
    xh, xl, _ = hf.hf_solve_dd(ctx, hy, b)
    assert torch.equal(xh, b) and float(xl.abs().max()) == 0.0     # K = diag(+-1) after scaling
    hy.close()
    lf.close()
    one = torch.tensor([[-5.0]], dtype=torch.float64, device="cuda")
    hf.hf_scale(ctx, one)
    lf = hf.hf_factor_lowprec(ctx, one, tau=1e-2, n_min=1, prec=64)
    assert lf.n2 == 1
    hy, info, S = hf.hf_schur_gcr_dd(ctx, one, lf, want_S22_host=True)
    assert S[0][0, 0] == -1.0 and S[1][0, 0] == 0.0
    assert hf.hf_factor_hard(ctx, hy, eps_ker=1e-20) == 0
    hy.close()
    lf.close()
