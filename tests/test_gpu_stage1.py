"""GPU parity of steps a1-a3 (scaling + FP32 factorization with postponing)
against the oracle: bitwise on q, K, Pi, Lambda_2, D and L ([R1]-[R10])."""
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


def _run(ctx, Kb_t, tau, n_min=0, n_extra=0, nb=0):
    from paper_2208_01907_b200 import hf
    Kd = Kb_t.to("cuda").contiguous()
    q = hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=tau, n_min=n_min, n_extra=n_extra, nb=nb)
    perm, D, Lf = lf.export()
    return Kd, q, lf, perm, D, Lf


CASES = [("C0", s) for s in range(6)] + [("P64", 0), ("N16", 0), ("N32", 0), ("S12", 0), ("S24", 0),
                                         ("P512", 0), ("P1024", 0)]


@pytest.mark.parametrize("name,seed", CASES)
def test_stage1_bitwise(ctx, name, seed):
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    Ko, qo = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    Kd, q, lf, perm, D, Lf = _run(ctx, Kb, spec.tau, n_min=spec.n_min)
    assert np.array_equal(q.cpu().numpy(), qo)
    assert np.array_equal(Kd.cpu().numpy(), Ko)            # symmetric: layout-free
    assert lf.N == Fo.N and lf.L - lf.n2_tau_only == Fo.Ntau
    assert np.array_equal(perm, Fo.perm)
    assert np.array_equal(D, Fo.D)
    if Fo.N:
        assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


@pytest.mark.parametrize("name,seed,pinned", [("C0", 0, True), ("P1024", 1, False), ("P512", 2, True)])
def test_scale_from_host_lower_triangle(ctx, name, seed, pinned):
    """hf_scale_host (the end-to-end entry: Kbar on the host) = the oracle's scaling, bitwise,
    reading only the lower triangle: the host matrix's upper triangle is overwritten with NaN
    and the result must not change; the bytes moved are the lower-triangle column panels."""
    from paper_2208_01907_b200 import hf
    Kb = hi.make_kbar(name, seed)
    Ko, qo = oracle.scale(Kb.numpy())
    L = Kb.shape[0]
    Kh = Kb.clone()
    # memory is column-major: element (i, j) of the matrix is Kh[j, i]; poison i < j
    iu = torch.triu_indices(L, L, offset=1)
    Kh[iu[1], iu[0]] = float("nan")
    if pinned:
        Kh = Kh.pin_memory()
    Kd = torch.empty(L, L, dtype=torch.float64, device="cuda")
    q, nbytes = hf.hf_scale_host(ctx, Kh, Kd)
    assert np.array_equal(q.cpu().numpy(), qo)
    assert np.array_equal(Kd.cpu().numpy(), Ko)
    W = 256
    assert nbytes == sum((L - j0) * min(W, L - j0) * 8 for j0 in range(0, L, W))
    assert nbytes <= (L * L + L * W) // 2 * 8             # the lower half + the diagonal blocks


def test_upload_pipelined_with_factorization(ctx):
    """hf_upload_lower (asynchronous, the library's upload stream) of matrix B while matrix A
    factors on the context stream, then hf_scale(B) (ordered after the upload) and B's
    factorization: both results bitwise equal to the oracle's."""
    from paper_2208_01907_b200 import hf
    specA, specB = hi.CONFIGS["P1024"], hi.CONFIGS["P512"]
    KbA, KbB = hi.make_kbar("P1024", 3), hi.make_kbar("P512", 4)
    KA = KbA.to("cuda").contiguous()
    KB = torch.empty(KbB.shape, dtype=torch.float64, device="cuda")
    hB = KbB.clone().pin_memory()
    hf.hf_scale(ctx, KA)
    lfA = hf.hf_factor_lowprec(ctx, KA, tau=specA.tau, n_min=specA.n_min)   # queued on the context stream
    hf.hf_upload_lower(ctx, hB, KB)                                        # concurrent copy
    hf.hf_scale(ctx, KB)
    lfB = hf.hf_factor_lowprec(ctx, KB, tau=specB.tau, n_min=specB.n_min)
    for Kb, spec, lf in ((KbA, specA, lfA), (KbB, specB, lfB)):
        Ko, _ = oracle.scale(Kb.numpy())
        Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
        perm, D, Lf = lf.export()
        assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
        if Fo.N:
            assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)
        lf.close()


@pytest.mark.parametrize("nb", [8, 16, 64, 128])
def test_stage1_panel_width_invariance(ctx, nb):
    """Panel width changes the blocking, never the bits (canonical order [R8])."""
    spec = hi.CONFIGS["P512"]
    Kb = hi.make_kbar("P512", 3)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    _, _, lf, perm, D, Lf = _run(ctx, Kb, spec.tau, n_min=spec.n_min, nb=nb)
    assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
    assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


def test_stage1_edge_cases(ctx):
    from paper_2208_01907_b200 import hf
    # first pivot 0 -> everything postponed
    _, _, lf, perm, D, _ = _run(ctx, torch.tensor([[0.0, 1.0], [1.0, 0.0]], dtype=torch.float64), 1e-2)
    assert lf.N == 0 and list(perm) == [0, 1]
    # diag(1, 0.9, 1e-9), tau 0.05 -- factor the matrix as given (no scaling)
    lf = hf.hf_factor_lowprec(ctx, torch.diag(torch.tensor([1.0, 0.9, 1e-9], dtype=torch.float64)).cuda(),
                              tau=0.05)
    perm, D, _ = lf.export()
    assert lf.N == 2 and list(perm) == [0, 1, 2] and list(D) == [1.0, np.float32(0.9)]
    # 1 x 1
    _, _, lf, perm, D, Lf = _run(ctx, torch.tensor([[-3.0]], dtype=torch.float64), 1e-2)
    assert lf.N == 1 and D[0] == -1.0
    # enlargement and floor together
    Kb = hi.make_kbar("P64", 1)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, 1e-2, n_min=5, n_extra=3)
    _, _, lf, perm, D, Lf = _run(ctx, Kb, 1e-2, n_min=5, n_extra=3)
    assert lf.N == Fo.N and np.array_equal(perm, Fo.perm) and np.array_equal(Lf.cpu().numpy(), Fo.Lfac)
    # bad tau
    with pytest.raises(hf.HFError):
        hf.hf_factor_lowprec(ctx, torch.eye(3, dtype=torch.float64, device="cuda"), tau=1.5)
    # NaN in K
    bad = torch.eye(4, dtype=torch.float64, device="cuda")
    bad[2, 1] = bad[1, 2] = float("nan")      # symmetric: hf_scale reads the lower triangle
    with pytest.raises(hf.HFError):
        hf.hf_scale(ctx, bad)


def test_stage1_c1_full_size(ctx):
    """Config 1 (L=4096) at full size, bitwise against the oracle."""
    spec = hi.CONFIGS["C1"]
    Kb = hi.make_kbar("C1", 0)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    _, _, lf, perm, D, Lf = _run(ctx, Kb, spec.tau, n_min=spec.n_min)
    assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
    assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


def test_stage1_lookahead_schedule_bitwise():
    """The lookahead schedule (HF_LOOKAHEAD=1: panel p+1's chain concurrent with panel p's
    trailing update, the chain applying panel p's updates to its pivot columns) gives the
    same bits as the oracle -- the canonical order [R8] does not depend on the schedule."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, hf_inputs as hi, oracle\n"
        "from paper_2208_01907_b200 import hf\n"
        "spec = hi.CONFIGS['P2048']; Kb = hi.make_kbar('P2048', 1)\n"
        "Ko, _ = oracle.scale(Kb.numpy()); Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)\n"
        "ctx = hf.Context(0); Kd = Kb.cuda(); hf.hf_scale(ctx, Kd)\n"
        "lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min, nb=64)\n"
        "perm, D, Lf = lf.export()\n"
        "assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)\n"
        "assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)\n"
        "print('ok')\n")
    env = dict(os.environ, HF_LOOKAHEAD="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("name,seed,nb", [("P512", 2, 0), ("P1024", 1, 0), ("P2048", 0, 64), ("S24", 0, 16),
                                         ("C0", 3, 8)])
def test_stage1_persistent_trailing_bitwise(ctx, name, seed, nb, monkeypatch):
    """The persistent trailing kernel (k_trailing_p: seeds of the next tile gathered by
    cp.async during the current one) forced at every size (HF_TRAIL_PERSIST=2; by default
    it runs only for launches of more than two tiles per CTA, C2-sized panels): same bits
    as the oracle, including ragged last chunks (nb = 8, 64) and tiny trailing matrices."""
    monkeypatch.setenv("HF_TRAIL_PERSIST", "2")
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    _, _, lf, perm, D, Lf = _run(ctx, Kb, spec.tau, n_min=spec.n_min, nb=nb)
    assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
    if Fo.N:
        assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)


@pytest.mark.parametrize("env,val", [("HF_TRAIL_BULK", "1"), ("HF_TRAIL_BULK", "2"), ("HF_TRAIL_PCTA", "1")])
@pytest.mark.parametrize("name,seed,nb", [("P1024", 1, 0), ("P2048", 0, 64), ("S24", 0, 16), ("C0", 3, 8)])
def test_stage1_trailing_variants_bitwise(ctx, name, seed, nb, env, val, monkeypatch):
    """The trailing update's opt-in variants, same bits as the oracle: the panel operands
    staged by the bulk-copy (TMA) engine with per-stage mbarriers, row by row
    (HF_TRAIL_BULK=1) or as 2D tensor-map boxes (HF_TRAIL_BULK=2), and
    persistent CTAs prefetching the next tile's compaction map (HF_TRAIL_PCTA) -- both
    measured slower than the default on C2."""
    monkeypatch.setenv(env, val)
    spec = hi.CONFIGS[name]
    Kb = hi.make_kbar(name, seed)
    Ko, _ = oracle.scale(Kb.numpy())
    Fo = oracle.factor_lowprec(Ko, spec.tau, n_min=spec.n_min)
    _, _, lf, perm, D, Lf = _run(ctx, Kb, spec.tau, n_min=spec.n_min, nb=nb)
    assert np.array_equal(perm, Fo.perm) and np.array_equal(D, Fo.D)
    if Fo.N:
        assert np.array_equal(Lf.cpu().numpy(), Fo.Lfac)
