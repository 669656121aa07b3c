"""NEXT-3: the nonsymmetric matrices of sec. 4.2-4.3 ([A B^T; -B delta D] and
[A B^T; -B 0]) through the GPU path against oracle/nonsym.py.

Stage 1 (FP32 LDU with symmetric pivoting and postponing, [R19]) is graded
BITWISE: Pi, Lambda_2, D, L and U.  Scaling (hf_scale_full) bitwise."""
import numpy as np
import pytest
import torch

import hf_inputs as hi
from hf_inputs.configs import ConfigSpec
from oracle import nonsym

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


def _rand_ns(L, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((L, L))
    A[np.arange(L), np.arange(L)] = rng.choice([1.0, -1.0, 0.5, 2.0], size=L) * np.abs(rng.standard_normal(L) + 1)
    return A


CASES = [("T8", None, 0), ("H8", None, 0), ("T24", None, 0), ("rand", 300, 1), ("rand", 700, 2),
         ("T8", None, 3)]


def _kbar(name, L, seed):
    if name == "rand":
        return _rand_ns(L, seed)
    return hi.make_kbar(name, seed).numpy()


@pytest.mark.parametrize("name,L,seed", CASES)
@pytest.mark.parametrize("nb", [0, 16])
def test_stage1_nonsym_bitwise(ctx, name, L, seed, nb):
    from paper_2208_01907_b200 import hf
    Kbar = _kbar(name, L, seed)
    Ko, qo = nonsym.scale_full(Kbar)
    Kd = hi.colmajor(torch.from_numpy(Kbar)).cuda()
    q = hf.hf_scale_full(ctx, Kd)
    assert np.array_equal(q.cpu().numpy(), qo)
    assert np.array_equal(Kd.cpu().numpy().T, Ko)          # column-major bytes
    F = nonsym.factor_ldu(Ko, 1e-2, n_min=2)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=1e-2, n_min=2, nb=nb, nonsym=True)
    perm, D, Lf = lf.export()
    Uf = lf.export_u()
    assert lf.N == F.N and lf.L - lf.n2_tau_only == F.Ntau
    assert np.array_equal(perm, F.perm)
    assert np.array_equal(D, F.D)
    assert np.array_equal(Lf.cpu().numpy(), F.Lfac)
    assert np.array_equal(Uf.cpu().numpy(), F.Ufac)
    lf.close()
