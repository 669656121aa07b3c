"""Structure checks of the seeded workload generators (hf_inputs)."""
import numpy as np
import torch

import hf_inputs as hi


def test_planted_symmetric_deterministic():
    a = hi.make_kbar("C0", 3)
    b = hi.make_kbar("C0", 3)
    c = hi.make_kbar("C0", 4)
    assert a.shape == (256, 256) and a.dtype == torch.float64
    assert torch.equal(a, b) and not torch.equal(a, c)
    assert torch.equal(a, a.T)


def test_planted_spectrum_has_planted_small_directions():
    spec = hi.CONFIGS["P64"]
    K = hi.make_kbar("P64", 0).numpy()
    s = np.sort(np.abs(np.linalg.eigvalsh(K)))
    # n_hard eigenvalues far below the bulk
    assert s[spec.n_hard - 1] < 1e-5 * s[spec.n_hard]


def test_neumann_structure():
    spec = hi.CONFIGS["N32"]
    K = hi.make_kbar("N32", 0).numpy()
    assert K.shape == (spec.L, spec.L) and np.array_equal(K, K.T)
    assert np.abs(K.sum(1)).max() <= 1e-9 * np.abs(K).max()     # pure Neumann: K 1 = 0
    boxes = hi.configs._inclusions(spec, 0)
    s = spec.incl_size
    for i, (x0, y0) in enumerate(boxes):
        assert 1 <= x0 and x0 + s <= spec.grid - 1 and 1 <= y0 and y0 + s <= spec.grid - 1
        for (x1, y1) in boxes[i + 1:]:
            assert abs(x0 - x1) >= s + 1 or abs(y0 - y1) >= s + 1
    assert set(np.unique(np.round(-K[K < 0], 12))) <= {1e-8, 1.0, 1e6}


def test_saddle_structure():
    spec = hi.CONFIGS["S12"]
    K = hi.make_kbar("S12", 0).numpy()
    nv = 2 * spec.grid ** 2
    assert K.shape == (spec.L, spec.L) and np.array_equal(K, K.T)
    assert np.all(K[nv:, nv:] == 0)
    Bm = K[nv:, :nv]
    assert Bm.shape[0] == 2 * (spec.grid // 2) ** 2          # two divergence rows per 2x2 macro-cell
    assert np.all((Bm != 0).sum(1) == 4)
    assert np.linalg.matrix_rank(Bm) == Bm.shape[0]          # no spurious pressure modes
    # BASELINE.json config 3: L = 23040 = 18432 velocity dofs + 4608 constraint rows
    c3 = hi.CONFIGS["C3"]
    assert c3.L == 23040 and 2 * c3.grid ** 2 == 18432 and c3.L - 2 * c3.grid ** 2 == 4608
    # translations (u_x = 1 or u_y = 1, p = 0) are in the kernel
    for c in range(2):
        t = np.zeros(spec.L)
        t[c:nv:2] = 1.0
        assert np.abs(K @ t).max() <= 1e-8 * np.abs(K).max()


def test_rhs_and_manufactured():
    b = hi.make_rhs("N32", 1)
    assert abs(float(b.sum())) < 1e-9
    x = hi.manufactured_x(30)
    assert x.tolist() == [float(i % 11) for i in range(30)]
    bs = hi.make_rhs("S12", 0)
    assert torch.all(bs[2 * 12 * 12:] == 0)
