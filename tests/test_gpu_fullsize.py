"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (default options, one context, the config's tau / n_min):

  C2 (L = 16384): the whole oracle (stage 1 bitwise on Pi, Lambda_2, D and the
      factor; block GCR + Schur + hard factor) against the CUDA path.
  C3 (L = 23040): the whole oracle (stage 1 bitwise on Pi, Lambda_2, D and the
      factor; S22 e_S, kernel dimension) plus S22 against the dense FP64 Schur
      complement of Eq. 2 (LAPACK solve with K11), kernel dimension 2 (the two
      translations), manufactured residual.  (~4 min)
  C4 (L = 65536, 34 GB in FP64): scaling bitwise on a sampled principal
      sub-block (K_ij depends only on Kbar_ij, Kbar_ii, Kbar_jj [R1]); stage 1
      BITWISE against the oracle's bounded run of its first 1024 pivots (Pi
      prefix, D, and the first 1024 factor columns on every Lambda_1 row);
      then properties that hold at any size, computed on the GPU in FP64 from
      the exported factor: the strict ratio test on every accepted pivot [R4],
      the reconstruction bound on sampled entries, the pivot rule at
      sampled steps [R3] (up to FP32 rounding), block-GCR true residual,
      manufactured residual.  (~4 min, ~60 GB of host memory)
"""
import os

import numpy as np
import pytest
import scipy.linalg as sla
import torch

import hf_inputs as hi
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2208_01907_b200 import hf
    c = hf.Context(0)
    yield c
    c.close()


def _gpu_path(ctx, spec, Kb):
    from paper_2208_01907_b200 import hf
    Kd = Kb.to("cuda")
    hf.hf_scale(ctx, Kd)
    lf = hf.hf_factor_lowprec(ctx, Kd, tau=spec.tau, n_min=spec.n_min)
    hy, info, S22 = hf.hf_schur_gcr(ctx, Kd, lf, want_S22_host=True)
    kd = hf.hf_factor_hard(ctx, hy)
    hf.hf_trim_cache(0)   # the library's cached workspaces (the mat-vec slices: as large as K) go back
    return Kd, lf, hy, info, S22, kd


def _rho_manufactured(ctx, hy, Kd):
    from paper_2208_01907_b200 import hf
    xs = hi.manufactured_x(Kd.shape[0], device="cuda")
    b = Kd @ xs
    x, _ = hf.hf_solve(ctx, hy, b)
    return float((Kd @ x - b).abs().max() / b.abs().max())


def test_c2_full_oracle(ctx):
    spec = hi.CONFIGS["C2"]
    Kb = hi.make_kbar("C2", 0, device="cuda").cpu()
    Ko, _ = oracle.scale(Kb.numpy())
    HF = oracle.hybrid_factor(Ko, tau=spec.tau, n_min=spec.n_min)
    Kd, lf, hy, info, S22, kd = _gpu_path(ctx, spec, Kb)
    assert np.array_equal(Kd.cpu().numpy(), Ko)
    perm, D, Lf = lf.export()
    assert lf.N == HF.F.N and lf.L - lf.n2_tau_only == HF.F.Ntau
    assert np.array_equal(perm, HF.F.perm)                  # Pi and Lambda_2, bitwise
    assert np.array_equal(D, HF.F.D)
    assert torch.equal(Lf.cpu(), torch.from_numpy(HF.F.Lfac))
    K11, K12, K21, K22 = oracle.extract_blocks(HF.K, HF.F)
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    assert np.linalg.norm(S22 - HF.S22) / den <= 1e-10      # [R17] e_S
    assert info.max_rel_res_true <= 1e-12
    thr = HF.H.thr
    margin = min(abs(np.array(HF.H.mu_hist) - thr))
    if margin > 10 * np.linalg.norm(S22 - HF.S22):
        assert kd == HF.kernel_dim
    assert _rho_manufactured(ctx, hy, Kd) <= 1e-12


def test_c3_full(ctx):
    spec = hi.CONFIGS["C3"]
    Kb = hi.make_kbar("C3", 0)
    Ko, _ = oracle.scale(Kb.numpy())
    Kd, lf, hy, info, S22, kd = _gpu_path(ctx, spec, Kb)
    assert np.array_equal(Kd.cpu().numpy(), Ko)
    perm, D, Lf = lf.export()
    # the whole oracle (Alg. 1 steps 1-5) on the same scaled matrix
    HF = oracle.hybrid_factor(Ko, tau=spec.tau, n_min=spec.n_min)
    assert lf.N == HF.F.N and lf.L - lf.n2_tau_only == HF.F.Ntau
    assert np.array_equal(perm, HF.F.perm)                  # Pi and Lambda_2, bitwise
    assert np.array_equal(D, HF.F.D)
    assert torch.equal(Lf.cpu(), torch.from_numpy(HF.F.Lfac))
    K11, K12, K21, K22 = oracle.extract_blocks(HF.K, HF.F)
    den = np.linalg.norm(K22) + np.linalg.norm(K21) * np.linalg.norm(HF.X)
    assert np.linalg.norm(S22 - HF.S22) / den <= 1e-10      # [R17] e_S
    thr = HF.H.thr
    margin = min(abs(np.array(HF.H.mu_hist) - thr))
    if margin > 10 * np.linalg.norm(S22 - HF.S22):
        assert kd == HF.kernel_dim
    del HF, K11, K21
    # S22 against the dense FP64 Schur complement of Eq. (2) (LAPACK solve with K11)
    l1, l2 = perm[: lf.N], perm[lf.N:]
    K11, K12, K22 = Ko[np.ix_(l1, l1)], Ko[np.ix_(l1, l2)], Ko[np.ix_(l2, l2)]
    Xd = sla.solve(K11, K12, assume_a="sym", check_finite=False)
    Sd = K22 - K12.T @ Xd
    den = np.linalg.norm(K22) + np.linalg.norm(K12) * np.linalg.norm(Xd)
    assert np.linalg.norm(S22 - Sd) / den <= 1e-10
    assert info.max_rel_res_true <= 1e-12
    assert kd == 2                       # the two rigid translations (pure Neumann reading)
    assert _rho_manufactured(ctx, hy, Kd) <= 1e-12


C4_PREFIX = 1024


def test_c4_full(ctx):
    from paper_2208_01907_b200 import hf
    spec = hi.CONFIGS["C4"]
    # C4 uses most of the device: release what the earlier full-size tests left cached in
    # torch's allocator and in the library's
    torch.cuda.empty_cache()
    hf.hf_trim_cache(0)
    Kb = hi.make_kbar("C4", 0, device="cuda")
    # [R1] scaling: a principal sub-block of Kbar scales to the same bits as in K
    sub = torch.from_numpy(np.sort(np.random.default_rng(4).choice(spec.L, 384, replace=False))).cuda()
    Kb_sub = Kb[sub][:, sub].cpu().numpy()
    Kd, lf, hy, info, S22, kd = _gpu_path(ctx, spec, Kb)
    del Kb
    torch.cuda.empty_cache()
    Ko_sub, _ = oracle.scale(Kb_sub)
    assert np.array_equal(Kd[sub][:, sub].cpu().numpy(), Ko_sub)
    perm, D, Lf = lf.export()
    N = lf.N
    assert N == spec.L - spec.n_min
    # stage 1, bitwise: the oracle's bounded run of the first C4_PREFIX pivots on the
    # same scaled K (the symmetric row-major tensor read as its column-major transpose)
    Kh = Kd.cpu().numpy().T
    pre = oracle.factor_lowprec_prefix(Kh, spec.tau, C4_PREFIX, n_min=spec.n_min)
    del Kh
    k = C4_PREFIX
    assert np.array_equal(perm[:k], pre.pivots)             # Pi prefix
    assert np.array_equal(D[:k], pre.D)
    rank = np.full(spec.L, -1, dtype=np.int64)
    rank[perm[:N]] = np.arange(N)
    rows = rank[pre.pos_orig]
    ok = rows >= 0                                          # every Lambda_1 row
    Lg = Lf[torch.from_numpy(rows[ok]).cuda(), :k].cpu().numpy()
    assert np.array_equal(Lg, pre.Lcols[ok])
    del pre, Lg
    # [R4] strict ratio test held at every accepted pivot
    Dd = np.abs(D.astype(np.float64))
    assert np.all(Dd[1:] >= spec.tau * Dd[:-1])
    # [R2]-[R8] reconstruction on sampled entries, in FP64 from the FP32 factor (S:291 bound)
    p1 = torch.from_numpy(perm[:N]).cuda()
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.integers(0, N, 256)).cuda()
    b = torch.from_numpy(rng.integers(0, N, 256)).cuda()
    La = Lf[a].double()
    Lb = Lf[b].double()
    Dt = torch.from_numpy(D.astype(np.float64)).cuda()
    rec = (La * Dt * Lb).sum(1)
    kab = Kd[p1[a], p1[b]]
    eps32 = float(np.finfo(np.float32).eps)
    assert float((rec - kab).abs().max()) <= 50 * N * eps32 * float(Kd.abs().max())
    # [R3] pivot rule at sampled steps: |d_k| is the largest remaining Schur diagonal
    # over the Lambda_1 rows (FP64 recomputation from the FP32 factor, equal up to the
    # FP32 rounding of the lazily updated diagonal: tol = 64 sqrt(k) eps32)
    Kdiag = Kd.diagonal()[torch.from_numpy(perm).cuda()]
    for k in (1, 1000, N // 2, N - 1):
        sd = torch.empty(N - k, dtype=torch.float64, device="cuda")
        for r0 in range(k, N, 4096):
            r1 = min(N, r0 + 4096)
            Lk = Lf[r0:r1, :k].double()
            sd[r0 - k:r1 - k] = Kdiag[r0:r1] - (Lk * Lk * Dt[:k]).sum(1)
            del Lk
        tol = 64 * np.sqrt(k) * eps32
        assert abs(float(sd[0])) >= float(sd.abs().max()) - tol
        assert abs(float(sd[0]) - float(D[k])) <= tol
    assert info.max_rel_res_true <= 1e-12
    # [R12]: the blocked tensor-core preconditioner may not cost iterations against the FP32
    # substitution (the dataflow form, HF_PRECOND=dataflow: 16 at C4); the blocked form takes
    # 11, and 18 when its bulk update accumulated the small bf16 parts after the large one
    assert info.iters <= 16
    assert _rho_manufactured(ctx, hy, Kd) <= 1e-12
