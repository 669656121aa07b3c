"""oracle.nonsym -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

NEXT-3: the hybrid factorization of the paper's
NONSYMMETRIC finite element matrices, [A B^T; -B delta D] (stokes)
and [A B^T; -B 0] (dd-hole), with the SAME symmetric pivoting and
threshold postponing ("Pi^T [K11 K12; K21 K22] Pi" of Eq. 1, P:46,
is written for a general K):

  scale_full      P:40 for a general matrix (every entry read)
  factor_ldu      FP32 LDU, canonical arithmetic [R19] (oracle/lowprec.c)
  precond_apply   Q^{-1} = U^{-1} D^{-1} L^{-1} in FP32, via core
  hybrid_factor   Alg. 1: block GCR (Alg. 5 is written for a
                  general matrix) on K11, S22 = K22 - K21 X12 with K21 the
                  actual lower-left block, LU with complete pivoting for S22
                  (the 1x1/2x2 symmetric pivots of [R15] do not apply)
  hybrid_solve    Alg. 2 with K21 and K12 separately

Pins: tests/test_oracle_nonsym.py (exact-rational left-looking emulation of
factor_ldu, reconstruction, constructed ranks of the LU, manufactured
solutions).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import core
from .core import GcrInfo, LowFactor, _ptr, block_gcr, lib


def _lib():
    L = lib()
    if not getattr(L, "_ns_bound", False):
        i64, dp, fp, lp = (ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float),
                           ctypes.POINTER(ctypes.c_int64))
        L.oracle_scale_full.argtypes = [i64, dp, i64, dp, dp]
        L.oracle_ldu_f32.argtypes = [i64, dp, i64, ctypes.c_double, i64, i64, lp, fp, fp, fp, lp]
        L._ns_bound = True
    return L


def scale_full(Kbar: np.ndarray):
    """K = Q Kbar Q for a general matrix.  Returns (K Fortran, q)."""
    Kbar = np.asfortranarray(Kbar, dtype=np.float64)
    L = Kbar.shape[0]
    K = np.empty_like(Kbar, order="F")
    q = np.empty(L, dtype=np.float64)
    _lib().oracle_scale_full(L, _ptr(Kbar, ctypes.c_double), L, _ptr(K, ctypes.c_double), _ptr(q, ctypes.c_double))
    return K, q


@dataclass
class LowFactorNS(LowFactor):
    Ufac: np.ndarray = None   # N x N: column k = row k of the unit upper U (U = Ufac^T)


def factor_ldu(K: np.ndarray, tau: float, n_min: int = 0, n_extra: int = 0) -> LowFactorNS:
    """FP32 LDU with symmetric pivoting and threshold postponing, [R19]."""
    K = np.asfortranarray(K, dtype=np.float64)
    L = K.shape[0]
    perm = np.empty(L, dtype=np.int64)
    Dk = np.zeros(max(L, 1), dtype=np.float32)
    Lf = np.empty((max(L, 1), max(L, 1)), dtype=np.float32, order="F")
    Uf = np.empty((max(L, 1), max(L, 1)), dtype=np.float32, order="F")
    out = np.zeros(2, dtype=np.int64)
    rc = _lib().oracle_ldu_f32(L, _ptr(K, ctypes.c_double), max(L, 1), float(tau), int(n_min), int(n_extra),
                               _ptr(perm, ctypes.c_int64), _ptr(Dk, ctypes.c_float), _ptr(Lf, ctypes.c_float),
                               _ptr(Uf, ctypes.c_float), _ptr(out, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_ldu_f32: invalid arguments (tau must be in (0,1))")
    N, Ntau = int(out[0]), int(out[1])
    return LowFactorNS(L=L, N=N, Ntau=Ntau, perm=perm, D=Dk[:N].copy(), Lfac=np.asfortranarray(Lf[:N, :N]),
                       dtype=np.float32, Ufac=np.asfortranarray(Uf[:N, :N]))


def extract_blocks(K: np.ndarray, F: LowFactor):
    """K11, K12, K21, K22 in Pi order, K21 the actual lower-left block."""
    l1, l2 = F.lam1, F.lam2
    return K[np.ix_(l1, l1)], K[np.ix_(l1, l2)], K[np.ix_(l2, l1)], K[np.ix_(l2, l2)]


# ------------------------------------------------------------ LU of S22
@dataclass
class HardLU:
    m: int
    r: int                  # rank found
    prow: np.ndarray        # pivot row labels (Lambda_2 positions) in order
    pcol: np.ndarray        # pivot column labels in order
    Lh: np.ndarray          # m x m unit lower (pivoted rows / cols)
    Uh: np.ndarray          # m x m upper, leading r x r block
    thr: float = 0.0
    mu_hist: list = field(default_factory=list)

    @property
    def kernel_dim(self) -> int:
        return self.m - self.r


def factor_hard_lu(S22: np.ndarray, d_ref: float, eps_ker: float = 1e-10) -> HardLU:
    """LU with complete pivoting of the nonsymmetric S22 in FP64: the pivot is
    the largest |entry| of the trailing block (ties -> smallest column label,
    then smallest row label); stop when it is <= eps_ker * d_ref, the size of
    the block left is the kernel dimension (the [R15] rule for a general S22)."""
    A = np.array(S22, dtype=np.float64, copy=True)
    m = A.shape[0]
    rl = np.arange(m, dtype=np.int64)
    cl = np.arange(m, dtype=np.int64)
    Lh = np.eye(m)
    thr = eps_ker * d_ref
    hist = []
    k = 0
    while k < m:
        sub = np.abs(A[k:, k:])
        mu = sub.max()
        hist.append(float(mu))
        if mu <= thr:
            break
        ii, jj = np.nonzero(sub == mu)
        ii, jj = ii + k, jj + k
        best = np.lexsort((rl[ii], cl[jj]))[0]
        i, j = ii[best], jj[best]
        A[[k, i], :] = A[[i, k], :]
        Lh[[k, i], :k] = Lh[[i, k], :k]
        rl[[k, i]] = rl[[i, k]]
        A[:, [k, j]] = A[:, [j, k]]
        cl[[k, j]] = cl[[j, k]]
        l = A[k + 1:, k] / A[k, k]
        A[k + 1:, k + 1:] -= np.outer(l, A[k, k + 1:])
        Lh[k + 1:, k] = l
        A[k + 1:, k] = 0.0
        k += 1
    return HardLU(m=m, r=k, prow=rl, pcol=cl, Lh=Lh, Uh=np.triu(A), thr=float(thr), mu_hist=hist)


def hard_solve_lu(H: HardLU, y: np.ndarray) -> np.ndarray:
    """x = S22^+ y on the factored part: P S Q = L U, kernel coordinates 0."""
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    r = H.r
    z = y[H.prow]
    w = np.linalg.solve(H.Lh[:r, :r], z[:r]) if r else np.zeros(0)
    v = np.linalg.solve(H.Uh[:r, :r], w) if r else np.zeros(0)
    x = np.zeros(H.m)
    x[H.pcol[:r]] = v
    return x


@dataclass
class HybridNS:
    K: np.ndarray
    F: LowFactorNS
    X: np.ndarray
    S22: np.ndarray
    H: HardLU | None
    gcr: GcrInfo
    d_ref: float

    @property
    def kernel_dim(self) -> int:
        return self.H.kernel_dim if self.H is not None else 0


def hybrid_factor(K: np.ndarray, tau: float = 1e-2, n_min: int = 0, n_extra: int = 0, tol: float = 1e-14,
                  max_iter: int = 100, eps_ker: float = 1e-10) -> HybridNS:
    """Algorithm 1 on a scaled general matrix K."""
    K = np.asfortranarray(K, dtype=np.float64)
    F = factor_ldu(K, tau, n_min=n_min, n_extra=n_extra)                   # step 1
    K11, K12, K21, K22 = extract_blocks(K, F)                              # step 2
    if F.N > 0 and F.n2 > 0:
        X, info = block_gcr(K11, F, K12, tol=tol, max_iter=max_iter)      # step 3
    else:
        X, info = np.zeros((F.N, F.n2)), GcrInfo(converged=True)
    S22 = core.schur(K22, K21, X)                                          # step 4
    d_ref = float(np.min(np.abs(F.D.astype(np.float64)))) if F.N > 0 else 1.0
    H = factor_hard_lu(S22, d_ref, eps_ker) if F.n2 > 0 else None          # step 5
    return HybridNS(K=K, F=F, X=X, S22=S22, H=H, gcr=info, d_ref=d_ref)


def hybrid_solve(HF: HybridNS, b: np.ndarray, tol: float = 1e-14, max_iter: int = 100):
    """Algorithm 2 with the actual K21."""
    F = HF.F
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    b1, b2 = b[F.lam1], b[F.lam2]
    K11, _, K21, _ = extract_blocks(HF.K, F)
    if F.N > 0:
        y1, info = block_gcr(K11, F, b1[:, None], tol=tol, max_iter=max_iter)   # step 1
        y1 = y1[:, 0]
    else:
        y1, info = np.zeros(0), GcrInfo(converged=True)
    y2 = b2 - K21 @ y1                                                     # step 2
    x2 = hard_solve_lu(HF.H, y2) if F.n2 > 0 else np.zeros(0)              # step 3
    x1 = y1 - HF.X @ x2 if F.n2 > 0 else y1                                # step 4
    x = np.empty(F.L)
    x[F.lam1] = x1
    x[F.lam2] = x2
    return x, info
