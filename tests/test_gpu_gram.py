"""GPU parity of the Gram-matrix inverse of Algorithm 5 (M_n^{-1}) through
hf_gram_inverse, against the FP64 LAPACK inverse of the same matrix: the blocked
16-CTA cluster kernel (n <= 448, ragged last block), the scalar cluster kernel
(448 < n <= ~640) and the cooperative kernel (larger n); the breakdown flag [R11]
on indefinite and singular matrices."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


def _spd(n, seed, cond=1e4):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.logspace(0, np.log10(cond), n)
    rng.shuffle(ev)
    M = (Q * ev) @ Q.T
    return 0.5 * (M + M.T), cond


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 33, 100, 256, 300, 448, 449, 600, 700])
def test_gram_inverse_vs_lapack(ctx, n):
    from paper_2208_01907_b200 import hf
    M, cond = _spd(n, n)
    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    Mi, bd = hf.hf_gram_inverse(ctx, Md.T.contiguous().T)
    assert not bd
    Mi = Mi.cpu().numpy()
    X = np.linalg.inv(M)
    # Gauss-Jordan without pivoting on SPD M: forward error O(n cond eps) normwise
    err = np.linalg.norm(Mi - X) / np.linalg.norm(X)
    assert err <= 50 * n * cond * np.finfo(float).eps, err
    assert np.linalg.norm(Mi @ M - np.eye(n)) <= 50 * n * cond * np.finfo(float).eps


def test_gram_inverse_exact_cases(ctx):
    from paper_2208_01907_b200 import hf
    # diagonal with powers of two: every operation exact
    d = 2.0 ** np.arange(-8, 9, dtype=np.float64)
    Mi, bd = hf.hf_gram_inverse(ctx, torch.diag(torch.from_numpy(d)).cuda())
    assert not bd
    assert np.array_equal(Mi.cpu().numpy(), np.diag(1.0 / d))
    # [[4, 2], [2, 2]]^{-1} = [[1/2, -1/2], [-1/2, 1]] (exact in binary)
    M = torch.tensor([[4.0, 2.0], [2.0, 2.0]], dtype=torch.float64).cuda()
    Mi, bd = hf.hf_gram_inverse(ctx, M)
    assert not bd
    assert np.array_equal(Mi.cpu().numpy(), np.array([[0.5, -0.5], [-0.5, 1.0]]))


@pytest.mark.parametrize("n", [3, 40, 300, 600])
def test_gram_inverse_breakdown(ctx, n):
    from paper_2208_01907_b200 import hf
    M, _ = _spd(n, 7 + n, cond=10.0)
    # indefinite: one negative eigenvalue
    w, V = np.linalg.eigh(M)
    w[n // 2] = -1.0
    Mneg = (V * w) @ V.T
    _, bd = hf.hf_gram_inverse(ctx, torch.from_numpy(np.asfortranarray(0.5 * (Mneg + Mneg.T))).cuda())
    assert bd
    # a zero leading pivot
    Mz = M.copy()
    Mz[0, :] = 0.0
    Mz[:, 0] = 0.0
    _, bd = hf.hf_gram_inverse(ctx, torch.from_numpy(np.asfortranarray(Mz)).cuda())
    assert bd
