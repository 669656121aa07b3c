"""oracle.core -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Stage 1 (scaling and the lower-precision factorization) runs in plain C
(oracle/lowprec.c, loaded with ctypes); stages 2-3 and the solve are numpy /
scipy in FP64, following Algorithms 1, 2, 4 and 5 of the paper step by step.
A library primitive (matmul, Cholesky, triangular solve) serves as a step; no
blocking, fusion or reordering beyond what the algorithm states.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lowprec.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/lowprec.c into oracle/liboracle.so (plain gcc, IEEE,
    no contraction; OpenMP only parallelises independent per-entry chains)."""
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= os.path.getmtime(_SRC)):
        return _SO
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fno-math-errno",
           "-fopenmp", "-fPIC", "-shared", "-o", _SO + ".tmp", _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            i64, dp, fp, lp = (ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int64))
            L.oracle_scale.argtypes = [i64, dp, i64, dp, dp]
            L.oracle_factor_f32.argtypes = [i64, dp, i64, ctypes.c_double, i64, i64, i64, lp, fp, fp, lp, i64, lp]
            L.oracle_factor_f64.argtypes = [i64, dp, i64, ctypes.c_double, i64, i64, i64, lp, dp, dp, lp, i64, lp]
            _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class OracleBreakdown(RuntimeError):
    """Non-positive Cholesky pivot of a Gram matrix M_n ([R11])."""


class OracleNotConverged(RuntimeError):
    """Block GCR hit max_iter ([R13])."""


# --------------------------------------------------------------------------
# diagonal scaling
# --------------------------------------------------------------------------
def scale(Kbar: np.ndarray):
    """K = Q Kbar Q with Q_ii = 1/sqrt|Kbar_ii| (1 if 0), P:40 [R1].
    Kbar: L x L float64 (only its lower triangle is read).
    Returns (K full symmetric float64 Fortran-ordered, q)."""
    Kbar = np.asfortranarray(Kbar, dtype=np.float64)
    L = Kbar.shape[0]
    K = np.empty_like(Kbar, order="F")
    q = np.empty(L, dtype=np.float64)
    lib().oracle_scale(L, _ptr(Kbar, ctypes.c_double), L, _ptr(K, ctypes.c_double),
                       _ptr(q, ctypes.c_double))
    return K, q


# --------------------------------------------------------------------------
# Alg. 1 step 1, sec. 2.1-2.2
# --------------------------------------------------------------------------
@dataclass
class LowFactor:
    L: int
    N: int            # |Lambda_1|
    Ntau: int         # pure tau-rule count (no floor, no enlargement)
    perm: np.ndarray  # int64[L]: Lambda_1 in pivot order, then Lambda_2 ascending
    D: np.ndarray     # [N] pivots d_k (float32 or float64)
    Lfac: np.ndarray  # N x N unit lower, pivot order (Fortran)
    dtype: type = np.float32

    @property
    def n2(self) -> int:
        return self.L - self.N

    @property
    def lam1(self) -> np.ndarray:
        return self.perm[: self.N]

    @property
    def lam2(self) -> np.ndarray:
        return self.perm[self.N:]


def factor_lowprec(K: np.ndarray, tau: float, n_min: int = 0, n_extra: int = 0,
                   prec: str = "f32", max_steps: int = 0) -> LowFactor:
    """LDL^T with symmetric max-|diag| pivoting and threshold postponing in the
    lower precision, rules [R2]-[R10].  K: scaled, exactly
    symmetric float64 (only the lower triangle is read).  max_steps > 0 stops
    after that many pivots (bench.py's bounded CPU-baseline sample only)."""
    K = np.asfortranarray(K, dtype=np.float64)
    L = K.shape[0]
    dt = np.float32 if prec == "f32" else np.float64
    ct = ctypes.c_float if prec == "f32" else ctypes.c_double
    perm = np.empty(L, dtype=np.int64)
    Dk = np.zeros(max(L, 1), dtype=dt)
    Lf = np.empty((max(L, 1), max(L, 1)), dtype=dt, order="F")
    out = np.zeros(2, dtype=np.int64)
    fn = lib().oracle_factor_f32 if prec == "f32" else lib().oracle_factor_f64
    rc = fn(L, _ptr(K, ctypes.c_double), max(L, 1), float(tau), int(n_min), int(n_extra), int(max_steps),
            _ptr(perm, ctypes.c_int64), _ptr(Dk, ct), _ptr(Lf, ct), _ptr(out, ctypes.c_int64), -1, None)
    if rc != 0:
        raise ValueError("oracle_factor: invalid arguments (tau must be in (0,1))")
    N, Ntau = int(out[0]), int(out[1])
    return LowFactor(L=L, N=N, Ntau=Ntau, perm=perm, D=Dk[:N].copy(),
                     Lfac=np.asfortranarray(Lf[:N, :N]), dtype=dt)


@dataclass
class FactorPrefix:
    """The first `steps` pivots of stage 1 (a bounded run of the same algorithm)."""
    pivots: np.ndarray    # int64[steps] original index of pivot k
    D: np.ndarray         # [steps] d_k
    Lcols: np.ndarray     # L x steps: L_{i,k} = c_i / d_k for every row, rows in pos_orig order
    pos_orig: np.ndarray  # int64[L] original index at each position after the run


def factor_lowprec_prefix(K: np.ndarray, tau: float, steps: int, n_min: int = 0,
                          prec: str = "f32") -> FactorPrefix:
    """Stage 1 stopped after `steps` pivots (the same oracle_factor body
    as factor_lowprec): returns only the first `steps` factor columns, with every
    row, so an L = 65536 run fits in host memory (L x steps instead of L x L).
    An output-interface variant for the C4 prefix parity test, no arithmetic
    change.  Raises if the tau-rule stops before `steps` pivots."""
    K = np.asfortranarray(K, dtype=np.float64)
    L = K.shape[0]
    steps = int(min(steps, L))
    dt = np.float32 if prec == "f32" else np.float64
    ct = ctypes.c_float if prec == "f32" else ctypes.c_double
    perm = np.empty(L, dtype=np.int64)
    Dk = np.zeros(max(L, 1), dtype=dt)
    Lf = np.empty((max(L, 1), max(steps, 1)), dtype=dt, order="F")
    pos = np.empty(max(L, 1), dtype=np.int64)
    out = np.zeros(2, dtype=np.int64)
    fn = lib().oracle_factor_f32 if prec == "f32" else lib().oracle_factor_f64
    rc = fn(L, _ptr(K, ctypes.c_double), max(L, 1), float(tau), int(n_min), 0, steps,
            _ptr(perm, ctypes.c_int64), _ptr(Dk, ct), _ptr(Lf, ct), _ptr(out, ctypes.c_int64), steps,
            _ptr(pos, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_factor: invalid arguments (tau must be in (0,1))")
    if int(out[1]) < steps:
        raise ValueError(f"the tau rule stopped after {int(out[1])} < {steps} pivots")
    return FactorPrefix(pivots=pos[:steps].copy(), D=Dk[:steps].copy(), Lcols=Lf, pos_orig=pos[:L])


def precond_apply(F: LowFactor, R: np.ndarray) -> np.ndarray:
    """Q^{-1} R of P:242: truncate R to the lower precision, forward unit-lower
    solve, divide by D, backward L^T solve (U for a nonsymmetric LDU factor),
    lift back to FP64 [R12].
    R: N x m in pivot order (float64)."""
    R = np.atleast_2d(np.asarray(R, dtype=np.float64).reshape(F.N, -1))
    if F.N == 0:
        return np.zeros_like(R)
    dt = F.dtype
    r = R.astype(dt)                                                  # truncate
    y = sla.solve_triangular(F.Lfac, r, lower=True, unit_diagonal=True,
                             check_finite=False)                      # forward
    y = (y / F.D[:, None].astype(dt)).astype(dt)                      # D^{-1}
    Ub = getattr(F, "Ufac", None)          # nonsymmetric LDU (oracle/nonsym.py): U = Ufac^T
    e = sla.solve_triangular(F.Lfac if Ub is None else Ub, y, lower=True, trans="T", unit_diagonal=True,
                             check_finite=False)                      # backward
    return np.asarray(e, dtype=dt).astype(np.float64)                 # lift


# --------------------------------------------------------------------------
# Alg. 2 step 2 blocks
# --------------------------------------------------------------------------
def extract_blocks(K: np.ndarray, F: LowFactor):
    """K11 = K[L1,L1], K12 = K[L1,L2], K21 = K12^T, K22 = K[L2,L2] in Pi order."""
    l1, l2 = F.lam1, F.lam2
    K11 = K[np.ix_(l1, l1)]
    K12 = K[np.ix_(l1, l2)]
    K22 = K[np.ix_(l2, l2)]
    return K11, K12, K12.T.copy(), K22


@dataclass
class GcrInfo:
    iters: int = 0
    converged: bool = False
    history: list = field(default_factory=list)   # per iteration: per-column rel. res (recursive)
    max_rel_res_recursive: float = float("nan")
    max_rel_res_true: float = float("nan")


def _relres(R, bn):
    rn = np.linalg.norm(R, axis=0)
    out = np.zeros_like(rn)
    nz = bn > 0
    out[nz] = rn[nz] / bn[nz]
    out[~nz] = np.where(rn[~nz] == 0, 0.0, np.inf)
    return out


def block_gcr(A: np.ndarray, F: LowFactor, B: np.ndarray, tol: float = 1e-14,
              max_iter: int = 100, raise_on_fail: bool = True, trace: dict | None = None):
    """Algorithm 5: right-preconditioned block GCR with q_n = A p_n
    caching, readings [R13]:
      M_n = Q_n^T Q_n, A_n = Q_n^T R_n, X += P_n M_n^{-1} A_n, R -= Q_n M_n^{-1} A_n,
      B_mn = -Q_m^T Z_{n+1}, P_{n+1} = W_{n+1} + sum_m P_m M_m^{-1} B_mn (same for Q),
    orthogonalising against all previous blocks (Alg. 4, "for 0<=m<=n").
    Returns (X, GcrInfo).  If ``trace`` is a dict it receives the blocks
    P_n, Q_n and the residual after every iteration (tests only)."""
    B = np.atleast_2d(np.asarray(B, dtype=np.float64).reshape(A.shape[0], -1))
    info = GcrInfo()
    bn = np.linalg.norm(B, axis=0)
    X = precond_apply(F, B)                      # find x_0 satisfying Q x_0 = b
    R = B - A @ X                                # r_0 = b - A x_0
    res = _relres(R, bn)
    info.history.append(res)
    if res.size == 0 or res.max() <= tol:
        info.converged = True
    else:
        W = precond_apply(F, R)                  # w_0 = Q^{-1} r_0
        Ps, Qs, Ms = [W], [A @ W], []            # p_0 = w_0, q_0 = A p_0
        for n in range(max_iter):
            Qn = Qs[n]
            Mn = Qn.T @ Qn                       # [M_n]_{l,k} = (q_n^k, q_n^l)
            An = Qn.T @ R                        # [A_n]_{l,k} = (r_n^k, q_n^l)
            try:
                cf = sla.cho_factor(Mn, lower=True, check_finite=False)
            except np.linalg.LinAlgError as e:
                raise OracleBreakdown(f"Gram matrix M_{n} not positive definite") from e
            Ms.append(cf)
            C = sla.cho_solve(cf, An, check_finite=False)
            X = X + Ps[n] @ C                    # x_{n+1} = x_n + p_n M^{-1} A
            R = R - Qn @ C                       # r_{n+1} = r_n - q_n M^{-1} A
            res = _relres(R, bn)
            info.history.append(res)
            info.iters = n + 1
            if trace is not None:
                trace.setdefault("R", []).append(R.copy())
            if res.max() <= tol:
                info.converged = True
                break
            W = precond_apply(F, R)              # Q w_{n+1} = r_{n+1}
            Z = A @ W                            # z_{n+1} = A w_{n+1}
            Pn, Qn1 = W.copy(), Z.copy()
            for m in range(n + 1):
                Bmn = -(Qs[m].T @ Z)             # [B_mn]_{l,k} = -(z^k, q_m^l)
                G = sla.cho_solve(Ms[m], Bmn, check_finite=False)
                Pn = Pn + Ps[m] @ G
                Qn1 = Qn1 + Qs[m] @ G
            Ps.append(Pn)
            Qs.append(Qn1)
        if trace is not None:
            trace["P"], trace["Q"] = Ps, Qs
    info.max_rel_res_recursive = float(res.max()) if res.size else 0.0
    info.max_rel_res_true = float(_relres(B - A @ X, bn).max()) if bn.size else 0.0
    if not info.converged and raise_on_fail:
        raise OracleNotConverged(f"block GCR: {info.iters} iterations, res {res.max():.3e}")
    return X, info


def gcr(A: np.ndarray, F: LowFactor, b: np.ndarray, tol: float = 1e-14, max_iter: int = 100):
    """Algorithm 4, single right-hand side, q_n caching; the
    beta numerator read as (A w_{n+1}, A p_m) [R13, typo at P:289]."""
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    info = GcrInfo()
    bn = float(np.linalg.norm(b))
    x = precond_apply(F, b[:, None])[:, 0]
    r = b - A @ x
    rel = np.linalg.norm(r) / bn if bn > 0 else 0.0
    info.history.append(np.array([rel]))
    if rel <= tol:
        info.converged = True
    else:
        w = precond_apply(F, r[:, None])[:, 0]
        ps, qs = [w], [A @ w]
        for n in range(max_iter):
            qn = qs[n]
            qq = qn @ qn
            alpha = (r @ qn) / qq
            x = x + alpha * ps[n]
            r = r - alpha * qn
            rel = np.linalg.norm(r) / bn
            info.history.append(np.array([rel]))
            info.iters = n + 1
            if rel <= tol:
                info.converged = True
                break
            w = precond_apply(F, r[:, None])[:, 0]
            z = A @ w
            p, q = w.copy(), z.copy()
            for m in range(n + 1):
                beta = -(z @ qs[m]) / (qs[m] @ qs[m])
                p = p + beta * ps[m]
                q = q + beta * qs[m]
            ps.append(p)
            qs.append(q)
    info.max_rel_res_recursive = float(rel)
    info.max_rel_res_true = float(np.linalg.norm(b - A @ x) / bn) if bn > 0 else 0.0
    return x, info


def iterative_refinement(A: np.ndarray, F: LowFactor, b: np.ndarray, tol: float = 1e-14,
                         max_iter: int = 100):
    """Algorithm 3: mixed-precision iterative refinement."""
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    info = GcrInfo()
    bn = float(np.linalg.norm(b))
    x = precond_apply(F, b[:, None])[:, 0]       # steps 1-2
    r = b - A @ x                                # step 3
    rel = np.linalg.norm(r) / bn if bn > 0 else 0.0
    info.history.append(np.array([rel]))
    for n in range(max_iter):
        if rel <= tol:
            info.converged = True
            break
        e = precond_apply(F, r[:, None])[:, 0]   # 4a-4b
        x = x + e                                # 4c
        r = b - A @ x                            # 4d
        rel = np.linalg.norm(r) / bn
        info.history.append(np.array([rel]))
        info.iters = n + 1
    else:
        info.converged = rel <= tol
    info.max_rel_res_recursive = info.max_rel_res_true = float(rel)
    return x, info


def schur(K22: np.ndarray, K21: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Alg. 1 step 4: S22 = K22 - K21 X12 in FP64 (Eq. 2)."""
    return K22 - K21 @ X


# --------------------------------------------------------------------------
# Alg. 1 step 5: FP64 factorization of S22 with 1x1/2x2 pivots [R15]
# --------------------------------------------------------------------------
ALPHA_BP = (1.0 + np.sqrt(17.0)) / 8.0


@dataclass
class HardFactor:
    m: int                 # n2
    r: int                 # rank found (m - kernel_dim)
    perm2: np.ndarray      # position -> Lambda_2 position label
    Lh: np.ndarray         # m x m unit lower (kernel part: identity columns)
    Dh: np.ndarray         # m x m block diagonal (1x1 / 2x2 blocks on [:r,:r])
    blocks: list           # pivot block sizes in order
    mu_stop: float = 0.0   # max |S_ij| of the block left at the stop (or of the last pivot)
    thr: float = 0.0
    mu_hist: list = field(default_factory=list)   # max |S_ij| of the trailing block at every step

    @property
    def kernel_dim(self) -> int:
        return self.m - self.r


def factor_hard(S22: np.ndarray, d_ref: float, eps_ker: float = 1e-10) -> HardFactor:
    """Symmetric Bunch-Parlett complete pivoting in FP64 (alpha = (1+sqrt17)/8):
    1x1 pivot at the max |diag| if it is >= alpha * max|S_ij|, else a 2x2
    pivot on the max off-diagonal pair; ties -> smallest Lambda_2 position.
    Stop when max |S_ij| of the trailing block <= eps_ker * d_ref; the size of
    the block left is the kernel dimension [R15]."""
    S = 0.5 * (np.asarray(S22, dtype=np.float64) + np.asarray(S22, dtype=np.float64).T)
    m = S.shape[0]
    A = S.copy()
    lab = np.arange(m, dtype=np.int64)
    Lh = np.eye(m)
    Dh = np.zeros((m, m))
    blocks = []
    thr = eps_ker * d_ref
    k = 0
    mu_stop = 0.0
    mu_hist = []

    def swap(i, j):
        if i == j:
            return
        A[[i, j], :] = A[[j, i], :]
        A[:, [i, j]] = A[:, [j, i]]
        Lh[[i, j], :k] = Lh[[j, i], :k]
        lab[[i, j]] = lab[[j, i]]

    while k < m:
        sub = np.abs(A[k:, k:])
        mu0 = sub.max()
        mu_stop = mu0
        mu_hist.append(float(mu0))
        if mu0 <= thr:
            break
        dg = np.diag(sub)
        mu1 = dg.max()
        if mu1 >= ALPHA_BP * mu0:
            cand = np.nonzero(dg == mu1)[0] + k
            p = cand[np.argmin(lab[cand])]
            swap(k, p)
            d = A[k, k]
            col = A[k + 1:, k].copy()
            l = col / d
            A[k + 1:, k + 1:] -= np.outer(col, col) / d        # exactly symmetric
            Lh[k + 1:, k] = l
            Dh[k, k] = d
            A[k + 1:, k] = 0.0
            A[k, k + 1:] = 0.0
            blocks.append(1)
            k += 1
        else:
            off = sub.copy()
            np.fill_diagonal(off, -1.0)
            ii, jj = np.nonzero(off == mu0)
            sel = ii < jj
            ii, jj = ii[sel] + k, jj[sel] + k
            la, lb = np.minimum(lab[ii], lab[jj]), np.maximum(lab[ii], lab[jj])
            best = np.lexsort((lb, la))[0]
            i, j = (ii[best], jj[best]) if lab[ii[best]] < lab[jj[best]] else (jj[best], ii[best])
            swap(k, i)
            if j == k:
                j = i
            swap(k + 1, j)
            E = A[k:k + 2, k:k + 2].copy()
            C = A[k + 2:, k:k + 2].copy()
            Lc = C @ np.linalg.inv(E)
            T = Lc @ C.T
            A[k + 2:, k + 2:] -= 0.5 * (T + T.T)               # keep A exactly symmetric
            Lh[k + 2:, k:k + 2] = Lc
            Dh[k:k + 2, k:k + 2] = E
            A[k + 2:, k:k + 2] = 0.0
            A[k:k + 2, k + 2:] = 0.0
            blocks.append(2)
            k += 2
    return HardFactor(m=m, r=k, perm2=lab, Lh=Lh, Dh=Dh, blocks=blocks, mu_stop=float(mu_stop),
                      thr=float(thr), mu_hist=mu_hist)


def hard_solve(H: HardFactor, y: np.ndarray) -> np.ndarray:
    """Solve S22 x2 = y2 with the kernel coordinates of the pivoted x2 set to
    zero (basic solution, [R16]).  y: m or m x k."""
    y = np.asarray(y, dtype=np.float64)
    vec = y.ndim == 1
    Y = y.reshape(H.m, -1)
    r = H.r
    z = Y[H.perm2]
    out = np.zeros_like(z)
    if r > 0:
        L11 = H.Lh[:r, :r]
        w = sla.solve_triangular(L11, z[:r], lower=True, unit_diagonal=True)
        v = np.linalg.solve(H.Dh[:r, :r], w)
        out[:r] = sla.solve_triangular(L11, v, lower=True, trans="T", unit_diagonal=True)
    x = np.zeros_like(out)
    x[H.perm2] = out
    return x[:, 0] if vec else x


# --------------------------------------------------------------------------
# Algorithms 1 and 2
# --------------------------------------------------------------------------
@dataclass
class Hybrid:
    K: np.ndarray
    F: LowFactor
    X: np.ndarray           # N x n2 (Pi order)
    S22: np.ndarray         # n2 x n2 (unsymmetrised)
    H: HardFactor | None
    gcr: GcrInfo
    d_ref: float

    @property
    def kernel_dim(self) -> int:
        return 0 if self.H is None else self.H.kernel_dim


def hybrid_factor(K: np.ndarray, tau: float = 1e-2, n_min: int = 0, n_extra: int = 0,
                  tol: float = 1e-14, max_iter: int = 100, eps_ker: float = 1e-10,
                  prec: str = "f32") -> Hybrid:
    """Algorithm 1 on the scaled matrix K."""
    K = np.asfortranarray(K, dtype=np.float64)
    F = factor_lowprec(K, tau, n_min=n_min, n_extra=n_extra, prec=prec)   # step 1
    K11, K12, K21, K22 = extract_blocks(K, F)                              # step 2
    if F.N > 0 and F.n2 > 0:
        X, info = block_gcr(K11, F, K12, tol=tol, max_iter=max_iter)      # step 3
    else:
        X, info = np.zeros((F.N, F.n2)), GcrInfo(converged=True)
    S22 = schur(K22, K21, X)                                               # step 4
    d_ref = float(np.min(np.abs(F.D.astype(np.float64)))) if F.N > 0 else 1.0
    H = factor_hard(S22, d_ref, eps_ker) if F.n2 > 0 else None             # step 5
    return Hybrid(K=K, F=F, X=X, S22=S22, H=H, gcr=info, d_ref=d_ref)


def hybrid_solve(HF: Hybrid, b: np.ndarray, tol: float = 1e-14, max_iter: int = 100):
    """Algorithm 2 for the scaled system K x = b [R16]."""
    F = HF.F
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    b1, b2 = b[F.lam1], b[F.lam2]
    K11, _, K21, _ = extract_blocks(HF.K, F)
    if F.N > 0:
        y1, info = block_gcr(K11, F, b1[:, None], tol=tol, max_iter=max_iter)  # step 1
        y1 = y1[:, 0]
    else:
        y1, info = np.zeros(0), GcrInfo(converged=True)
    y2 = b2 - K21 @ y1                                                     # step 2
    x2 = hard_solve(HF.H, y2) if F.n2 > 0 else np.zeros(0)                 # step 3
    x1 = y1 - HF.X @ x2 if F.n2 > 0 else y1                                # step 4
    x = np.empty(F.L)
    x[F.lam1] = x1
    x[F.lam2] = x2
    return x, info


def kernel_dimension(HF: Hybrid) -> int:
    return HF.kernel_dim
