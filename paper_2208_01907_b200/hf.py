"""Thin ctypes binding of libhf.so (include/hf.h).  Argument marshalling only:
every step of the path runs in the CUDA kernels behind the C ABI.  There is
no CPU fallback -- if libhf.so is missing or a call fails, this raises.

Matrices cross the boundary as column-major device buffers.  A contiguous
torch tensor T of shape (n, m) is the column-major m x n matrix T^T; for the
symmetric K that distinction vanishes.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhf.so")

HF_OK, HF_ERR_INVALID_ARG, HF_ERR_CUDA, HF_ERR_NCCL, HF_ERR_OOM = 0, 1, 2, 3, 4
HF_ERR_NOT_CONVERGED, HF_ERR_BREAKDOWN, HF_ERR_STATE = 5, 6, 7
_NAMES = {0: "HF_OK", 1: "HF_ERR_INVALID_ARG", 2: "HF_ERR_CUDA", 3: "HF_ERR_NCCL", 4: "HF_ERR_OOM",
          5: "HF_ERR_NOT_CONVERGED", 6: "HF_ERR_BREAKDOWN", 7: "HF_ERR_STATE"}

EXPORTED = [
    "hf_create", "hf_create_dist", "hf_nccl_unique_id", "hf_destroy", "hf_last_error",
    "hf_set_profiling", "hf_kernel_stats", "hf_kernel_work", "hf_chain_exchange_floor", "hf_launch_count", "hf_scale", "hf_scale_host", "hf_upload_lower", "hf_matvec", "hf_factor_lowprec",
    "hf_lowfactor_export", "hf_lowfactor_destroy", "hf_schur_gcr", "hf_hybrid_export",
    "hf_factor_hard", "hf_hard_export", "hf_solve", "hf_hybrid_destroy", "hf_trim_cache",
    "hf_precond_apply", "hf_shard_cols", "hf_set_virtual_rank", "hf_set_stage1_partitions",
    "hf_stage1_partition", "hf_krylov_solve", "hf_lowfactor_export64", "hf_schur_gcr_dd",
    "hf_hybrid_export_dd", "hf_lowfactor_export_u", "hf_scale_full", "hf_solve_dd",
    "hf_nd_blocks", "hf_factor_lowprec_blocks", "hf_gram_inverse",
]


class HFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class lowprec_opts(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_double), ("n_extra", ctypes.c_int64), ("n_min", ctypes.c_int64),
                ("nb", ctypes.c_int32), ("prec", ctypes.c_int32), ("nonsym", ctypes.c_int32)]


class gcr_opts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int32), ("matvec", ctypes.c_int32),
                ("slices", ctypes.c_int32)]


MATVEC = {"auto": 0, "dmma": 1, "ozaki": 2, "ozaki2": 3}


class gcr_info(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("max_rel_res_recursive", ctypes.c_double),
                ("max_rel_res_true", ctypes.c_double), ("matvec", ctypes.c_int32)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libhf.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run `python -m paper_2208_01907_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    pi64, pdbl = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)
    sig = {
        "hf_create": [ctypes.c_int, vp, ctypes.POINTER(vp)],
        "hf_create_dist": [ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
        "hf_nccl_unique_id": [vp],
        "hf_destroy": [vp],
        "hf_set_profiling": [vp, ctypes.c_int],
        "hf_kernel_stats": [vp, ctypes.c_char_p, pdbl, pi64],
        "hf_kernel_work": [vp, ctypes.c_char_p, pdbl, pdbl],
        "hf_chain_exchange_floor": [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, pdbl],
        "hf_launch_count": [vp, pi64],
        "hf_scale": [vp, i64, vp, i64, vp],
        "hf_scale_host": [vp, i64, vp, i64, vp, i64, vp, vp],
        "hf_upload_lower": [vp, i64, vp, i64, vp, i64, vp],
        "hf_matvec": [vp, i64, vp, i64, vp, i64, i64, vp, i64, i32, i32],
        "hf_scale_full": [vp, i64, vp, i64, vp],
        "hf_factor_lowprec": [vp, i64, vp, i64, ctypes.POINTER(lowprec_opts), ctypes.POINTER(vp), pi64, pi64, pi64],
        "hf_lowfactor_export": [vp, vp, vp, vp, vp, i64],
        "hf_lowfactor_destroy": [vp],
        "hf_lowfactor_export64": [vp, vp, vp, vp, vp, i64],
        "hf_lowfactor_export_u": [vp, vp, vp, i64],
        "hf_schur_gcr": [vp, vp, i64, vp, ctypes.POINTER(gcr_opts), ctypes.POINTER(vp), vp,
                         ctypes.POINTER(gcr_info)],
        "hf_hybrid_export": [vp, vp, vp, i64, vp, i64],
        "hf_schur_gcr_dd": [vp, vp, i64, vp, ctypes.POINTER(gcr_opts), ctypes.POINTER(vp), vp, vp,
                            ctypes.POINTER(gcr_info)],
        "hf_hybrid_export_dd": [vp, vp, vp, vp, i64, vp, vp, i64],
        "hf_solve_dd": [vp, vp, vp, vp, vp, ctypes.POINTER(gcr_info)],
        "hf_nd_blocks": [vp, i64, vp, i64, i32, i32, vp, ctypes.POINTER(i32)],
        "hf_factor_lowprec_blocks": [vp, i64, vp, i64, ctypes.POINTER(lowprec_opts), vp, i32, ctypes.POINTER(vp),
                                     pi64, pi64, pi64],
        "hf_factor_hard": [vp, vp, dbl, pi64],
        "hf_hard_export": [vp, vp, vp, vp, pi64],
        "hf_solve": [vp, vp, vp, vp, ctypes.POINTER(gcr_info)],
        "hf_hybrid_destroy": [vp],
        "hf_trim_cache": [ctypes.c_int],
        "hf_precond_apply": [vp, vp, i64, vp, i64, vp, i64],
        "hf_gram_inverse": [vp, i64, vp, i64, vp, ctypes.POINTER(ctypes.c_int32)],
        "hf_shard_cols": [i64, ctypes.c_int, ctypes.c_int, pi64, pi64],
        "hf_set_virtual_rank": [vp, ctypes.c_int, ctypes.c_int],
        "hf_set_stage1_partitions": [vp, ctypes.c_int],
        "hf_stage1_partition": [i64, ctypes.c_int, ctypes.c_int, pi64, vp],
        "hf_krylov_solve": [vp, vp, i64, vp, ctypes.c_int, i64, vp, vp, dbl, i32, ctypes.POINTER(i32), pdbl, i32],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.hf_last_error.argtypes = [vp]
    L.hf_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def hf_trim_cache(device: int = 0) -> None:
    """Return the library's cached (free) device blocks of `device` to the driver."""
    st = load().hf_trim_cache(device)
    if st != HF_OK:
        raise HFError(st, "hf_trim_cache")


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def _dev(t: torch.Tensor, dtype) -> None:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise TypeError(f"expected a contiguous CUDA {dtype} tensor")


class Context:
    """hf_ctx: one CUDA device + stream (+ optional NCCL communicator)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None,
                 nccl_id: bytes | None = None, rank: int = 0, nranks: int = 1):
        self.lib = load()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        if nccl_id is None:
            st = self.lib.hf_create(device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        else:
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            st = self.lib.hf_create_dist(device, ctypes.c_void_p(self.stream.cuda_stream), buf, rank,
                                         nranks, ctypes.byref(h))
        if st != HF_OK:
            msg = self.lib.hf_last_error(h if h.value else None).decode()
            if h.value:
                self.lib.hf_destroy(h)
            raise HFError(st, msg)
        self.h = h

    def check(self, st: int, accept=()):
        if st != HF_OK and st not in accept:
            raise HFError(st, self.lib.hf_last_error(self.h).decode())
        return st

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.hf_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # instrumentation
    def set_profiling(self, on: bool):
        self.check(self.lib.hf_set_profiling(self.h, int(bool(on))))

    def kernel_stats(self, cls: str):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self.check(self.lib.hf_kernel_stats(self.h, cls.encode(), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def kernel_work(self, cls: str):
        """(flops, bytes) of algorithmic work of a kernel class while profiling (cumulative)."""
        fl, by = ctypes.c_double(), ctypes.c_double()
        self.check(self.lib.hf_kernel_work(self.h, cls.encode(), ctypes.byref(fl), ctypes.byref(by)))
        return fl.value, by.value

    def chain_exchange_floor(self, nctas: int, nthreads: int, steps: int = 4096) -> float:
        """us per step of the chain's grid-wide exchange alone (instrumentation)."""
        us = ctypes.c_double()
        self.check(self.lib.hf_chain_exchange_floor(self.h, int(nctas), int(nthreads), int(steps), ctypes.byref(us)))
        return us.value

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        self.check(self.lib.hf_launch_count(self.h, ctypes.byref(n)))
        return n.value


def hf_shard_cols(n2: int, nranks: int, rank: int) -> tuple[int, int]:
    """Column slice [c0, c1) of the n2 right-hand sides owned by `rank` (host only)."""
    c0, c1 = ctypes.c_int64(), ctypes.c_int64()
    st = load().hf_shard_cols(int(n2), int(nranks), int(rank), ctypes.byref(c0), ctypes.byref(c1))
    if st != HF_OK:
        raise HFError(st, "hf_shard_cols: bad arguments")
    return c0.value, c1.value


def hf_set_virtual_rank(ctx: "Context", rank: int, nranks: int) -> None:
    ctx.check(ctx.lib.hf_set_virtual_rank(ctx.h, int(rank), int(nranks)))


def hf_set_stage1_partitions(ctx: "Context", nparts: int) -> None:
    """Run stage 1 column-partitioned over `nparts` partitions on this GPU (emulation of the
    multi-GPU factorization; 0 = single-GPU path)."""
    ctx.check(ctx.lib.hf_set_stage1_partitions(ctx.h, int(nparts)))


def hf_stage1_partition(L: int, nparts: int, part: int) -> np.ndarray:
    """Original column indices partition `part` owns in the multi-GPU stage 1 (host only)."""
    n = ctypes.c_int64()
    cols = np.empty(max(L, 1), dtype=np.int64)
    st = load().hf_stage1_partition(int(L), int(nparts), int(part), ctypes.byref(n), cols.ctypes.data)
    if st != HF_OK:
        raise HFError(st, "hf_stage1_partition: bad arguments")
    return cols[: n.value]


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load().hf_nccl_unique_id(buf)
    if st != HF_OK:
        raise HFError(st, "ncclGetUniqueId failed")
    return buf.raw


# ---------------------------------------------------------------------- a1
def hf_scale(ctx: Context, K: torch.Tensor) -> torch.Tensor:
    """In-place diagonal scaling; returns q (device FP64[L])."""
    _dev(K, torch.float64)
    L = K.shape[0]
    q = torch.empty(L, dtype=torch.float64, device=K.device)
    ctx.check(ctx.lib.hf_scale(ctx.h, L, _ptr(K), L, _ptr(q)))
    return q


def hf_scale_host(ctx: Context, Kbar_host: torch.Tensor, K: torch.Tensor):
    """P:40 scaling from a host matrix: the lower triangle of Kbar_host (CPU FP64 L x L,
    column-major memory = a transposed-contiguous or symmetric tensor; pin it for an
    asynchronous copy) is copied into the device K and scaled there.  Returns
    (q device FP64[L], bytes copied host -> device)."""
    _dev(K, torch.float64)
    if Kbar_host.device.type != "cpu" or Kbar_host.dtype != torch.float64 or not Kbar_host.is_contiguous():
        raise ValueError("Kbar_host must be a contiguous CPU float64 tensor")
    L = K.shape[0]
    if tuple(Kbar_host.shape) != (L, L):
        raise ValueError("Kbar_host and K differ in shape")
    q = torch.empty(L, dtype=torch.float64, device=K.device)
    nb = ctypes.c_int64(0)
    ctx.check(ctx.lib.hf_scale_host(ctx.h, L, _ptr(Kbar_host), L, _ptr(K), L, _ptr(q),
                                    ctypes.byref(nb)))
    return q, int(nb.value)


def hf_upload_lower(ctx: Context, Kbar_host: torch.Tensor, K: torch.Tensor) -> int:
    """Asynchronous copy of the lower triangle of Kbar_host (CPU FP64 L x L, pinned for
    asynchrony) into the device K on the context's upload stream; the next hf_scale on
    this context waits for it.  K must not be in use by queued work.  Returns the bytes."""
    _dev(K, torch.float64)
    if Kbar_host.device.type != "cpu" or Kbar_host.dtype != torch.float64 or not Kbar_host.is_contiguous():
        raise ValueError("Kbar_host must be a contiguous CPU float64 tensor")
    L = K.shape[0]
    if tuple(Kbar_host.shape) != (L, L):
        raise ValueError("Kbar_host and K differ in shape")
    nb = ctypes.c_int64(0)
    ctx.check(ctx.lib.hf_upload_lower(ctx.h, L, _ptr(Kbar_host), L, _ptr(K), L, ctypes.byref(nb)))
    return int(nb.value)


def hf_matvec(ctx: Context, K: torch.Tensor, W: torch.Tensor, matvec: str = "ozaki", slices: int = 0) -> torch.Tensor:
    """Z = K W for a symmetric device FP64 K (L x L) and W (L x n as a column-major
    matrix: a (n, L) contiguous tensor, i.e. W.T of a row-major L x n); returns Z in the
    same (n, L) layout.  matvec "dmma" or "ozaki"."""
    _dev(K, torch.float64)
    _dev(W, torch.float64)
    L = K.shape[0]
    n = W.shape[0]
    if W.shape[1] != L or not W.is_contiguous():
        raise ValueError("W must be a contiguous (n, L) tensor")
    Z = torch.empty_like(W)
    ctx.check(ctx.lib.hf_matvec(ctx.h, L, _ptr(K), L, _ptr(W), L, n, _ptr(Z), L, MATVEC[matvec], int(slices)))
    return Z


def hf_scale_full(ctx: Context, K: torch.Tensor) -> torch.Tensor:
    """NEXT-3: in-place scaling of a general matrix (memory = column-major K); returns q."""
    _dev(K, torch.float64)
    L = K.shape[0]
    q = torch.empty(L, dtype=torch.float64, device=K.device)
    ctx.check(ctx.lib.hf_scale_full(ctx.h, L, _ptr(K), L, _ptr(q)))
    return q


# ---------------------------------------------------------------------- a2-a3
class LowFactor:
    def __init__(self, ctx: Context, h, L: int, N: int, n2: int, n2_tau: int):
        self.ctx, self.h, self.L, self.N, self.n2, self.n2_tau_only = ctx, h, L, N, n2, n2_tau

    def export(self, with_L: bool = True):
        """(perm np.int64[L], D np.float32[N], Lfac device float32 N x N (matrix view))."""
        perm = np.empty(self.L, dtype=np.int64)
        D = np.empty(max(self.N, 1), dtype=np.float32)
        Lf = None
        if with_L and self.N > 0:
            Lf = torch.empty(self.N, self.N, dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        self.ctx.check(self.ctx.lib.hf_lowfactor_export(self.ctx.h, self.h, _ptr(perm), _ptr(D),
                                                        _ptr(Lf), self.N))
        return perm, D[: self.N], (Lf.T if Lf is not None else None)

    def export_u(self):
        """Nonsymmetric factor: Ufac (device float32 N x N, pivot order) with U = Ufac^T."""
        U = torch.empty(max(self.N, 1), max(self.N, 1), dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        self.ctx.check(self.ctx.lib.hf_lowfactor_export_u(self.ctx.h, self.h, _ptr(U), max(self.N, 1)))
        return U[: self.N, : self.N].T

    def export64(self, with_L: bool = True):
        """prec-64 factors: (perm np.int64[L], D np.float64[N], Lfac device float64 N x N)."""
        perm = np.empty(self.L, dtype=np.int64)
        D = np.empty(max(self.N, 1), dtype=np.float64)
        Lf = None
        if with_L and self.N > 0:
            Lf = torch.empty(self.N, self.N, dtype=torch.float64, device=f"cuda:{self.ctx.device}")
        self.ctx.check(self.ctx.lib.hf_lowfactor_export64(self.ctx.h, self.h, _ptr(perm), _ptr(D),
                                                          _ptr(Lf), self.N))
        return perm, D[: self.N], (Lf.T if Lf is not None else None)

    def close(self):
        if self.h is not None and self.h.value:
            self.ctx.lib.hf_lowfactor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hf_factor_lowprec(ctx: Context, K: torch.Tensor, tau: float = 1e-2, n_extra: int = 0,
                      n_min: int = 0, nb: int = 0, prec: int = 32, nonsym: bool = False) -> LowFactor:
    """nonsym=True (NEXT-3): K is a general matrix whose COLUMN-major bytes are the
    tensor's memory (pass hf_inputs.colmajor(Kbar-like tensor))."""
    _dev(K, torch.float64)
    L = K.shape[0]
    o = lowprec_opts(float(tau), int(n_extra), int(n_min), int(nb), int(prec), int(bool(nonsym)))
    h = ctypes.c_void_p()
    N, n2, n2t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ctx.check(ctx.lib.hf_factor_lowprec(ctx.h, L, _ptr(K), L, ctypes.byref(o), ctypes.byref(h),
                                        ctypes.byref(N), ctypes.byref(n2), ctypes.byref(n2t)))
    return LowFactor(ctx, h, L, N.value, n2.value, n2t.value)


# ---------------------------------------------------------------------- a4-a7
@dataclass
class GcrInfo:
    iters: int
    max_rel_res_recursive: float
    max_rel_res_true: float
    status: int = HF_OK
    matvec: int = 0        # the mat-vec form that ran: 1 DMMA, 2 int8 slices, 3 int8 residues


class Hybrid:
    def __init__(self, ctx: Context, h, lf: LowFactor, K: torch.Tensor):
        self.ctx, self.h, self.lf, self.K = ctx, h, lf, K    # keeps K alive (borrowed)
        self.kernel_dim = None

    @property
    def n2(self):
        return self.lf.n2

    def export(self):
        """(X device FP64 N x n2 matrix view, S22 device FP64 n2 x n2 matrix view)."""
        N, n2 = self.lf.N, self.lf.n2
        dev = f"cuda:{self.ctx.device}"
        X = torch.empty(max(n2, 1), max(N, 1), dtype=torch.float64, device=dev)
        S = torch.empty(max(n2, 1), max(n2, 1), dtype=torch.float64, device=dev)
        self.ctx.check(self.ctx.lib.hf_hybrid_export(self.ctx.h, self.h, _ptr(X), max(N, 1), _ptr(S),
                                                     max(n2, 1)))
        return X[:n2, :N].T, S[:n2, :n2].T

    def export_dd(self):
        """Double-double hybrid: (Xhi, Xlo: device L x n2, original row order; S22hi, S22lo: device n2 x n2)."""
        L, n2 = self.lf.L, self.lf.n2
        dev = f"cuda:{self.ctx.device}"
        out = [torch.empty(max(n2, 1), max(L, 1), dtype=torch.float64, device=dev) for _ in range(2)]
        out += [torch.empty(max(n2, 1), max(n2, 1), dtype=torch.float64, device=dev) for _ in range(2)]
        self.ctx.check(self.ctx.lib.hf_hybrid_export_dd(self.ctx.h, self.h, _ptr(out[0]), _ptr(out[1]), max(L, 1),
                                                        _ptr(out[2]), _ptr(out[3]), max(n2, 1)))
        return out[0][:n2, :L].T, out[1][:n2, :L].T, out[2][:n2, :n2].T, out[3][:n2, :n2].T

    def hard_export(self):
        n2 = self.lf.n2
        p = np.zeros(max(n2, 1), dtype=np.int64)
        b = np.zeros(max(n2, 1), dtype=np.int32)
        r = ctypes.c_int64()
        self.ctx.check(self.ctx.lib.hf_hard_export(self.ctx.h, self.h, _ptr(p), _ptr(b), ctypes.byref(r)))
        return p[:n2], b[:n2], r.value

    def close(self):
        if self.h is not None and self.h.value:
            self.ctx.lib.hf_hybrid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hf_precond_apply(ctx: Context, lf: LowFactor, R: torch.Tensor, W: torch.Tensor | None = None) -> torch.Tensor:
    """W = Q^{-1} R (FP32 preconditioner, [R12]).  R: device FP64 L x ncol in
    column-major layout (R.stride() == (1, L), e.g. ``t.T`` of a contiguous
    (ncol, L) tensor), original row order.  Returns W in the same layout."""
    if not (isinstance(R, torch.Tensor) and R.is_cuda and R.dtype == torch.float64 and R.dim() == 2
            and R.shape[0] == lf.L and (R.shape[1] <= 1 or R.stride() == (1, lf.L))):
        raise TypeError("R must be a column-major CUDA float64 (L, ncol) tensor")
    ncol = R.shape[1]
    if W is None:
        W = torch.empty(ncol, lf.L, dtype=torch.float64, device=R.device).T
    ctx.check(ctx.lib.hf_precond_apply(ctx.h, lf.h, ncol, _ptr(R), lf.L, _ptr(W), lf.L))
    return W


def hf_gram_inverse(ctx: Context, M: torch.Tensor) -> tuple[torch.Tensor, bool]:
    """(M^{-1}, breakdown) for the SPD Gram matrix of Alg. 5.  M: CUDA float64
    (n, n), column-major or symmetric.  Returns Minv column-major (n, n) and the breakdown flag."""
    if not (isinstance(M, torch.Tensor) and M.is_cuda and M.dtype == torch.float64 and M.dim() == 2
            and M.shape[0] == M.shape[1]):
        raise TypeError("M must be a square CUDA float64 tensor")
    n = M.shape[0]
    Mc = M if (n <= 1 or M.stride() == (1, n)) else M.T.contiguous().T
    Minv = torch.empty(n, n, dtype=torch.float64, device=M.device).T
    bd = ctypes.c_int32(0)
    ctx.check(ctx.lib.hf_gram_inverse(ctx.h, n, _ptr(Mc), max(n, 1), _ptr(Minv), ctypes.byref(bd)))
    return Minv, bool(bd.value)


KRYLOV = {"ir": 0, "gcr": 1, "bgcr": 2}


def hf_krylov_solve(ctx: Context, K: torch.Tensor, lf: LowFactor, B: torch.Tensor, method: str = "bgcr",
                    tol: float = 1e-14, max_iter: int = 100, accept_failure: bool = False):
    """K11 X = B by IR (Alg. 3), GCR (Alg. 4, per column) or block GCR (Alg. 5).
    B: column-major CUDA float64 (L, ncol).  Returns (X, iters, history np.ndarray, status)."""
    _dev(K, torch.float64)
    if not (isinstance(B, torch.Tensor) and B.is_cuda and B.dtype == torch.float64 and B.dim() == 2
            and B.shape[0] == lf.L and (B.shape[1] <= 1 or B.stride() == (1, lf.L))):
        raise TypeError("B must be a column-major CUDA float64 (L, ncol) tensor")
    X = torch.empty(B.shape[1], lf.L, dtype=torch.float64, device=B.device).T
    it = ctypes.c_int32()
    hist = np.full(max_iter + 2, -1.0)
    st = ctx.lib.hf_krylov_solve(ctx.h, _ptr(K), K.shape[0], lf.h, KRYLOV[method], B.shape[1], _ptr(B), _ptr(X),
                                 float(tol), int(max_iter), ctypes.byref(it),
                                 hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(hist))
    ctx.check(st, (HF_ERR_NOT_CONVERGED,) if accept_failure else ())
    return X, it.value, hist[hist >= 0], st


def hf_schur_gcr(ctx: Context, K: torch.Tensor, lf: LowFactor, tol: float = 1e-14, max_iter: int = 100,
                 want_S22_host: bool = False, accept_failure: bool = False, matvec: str = "auto",
                 slices: int = 0):
    """Returns (Hybrid, GcrInfo, S22 host np.ndarray or None).  matvec: "auto" | "dmma" |
    "ozaki" (hf_gcr_opts.matvec), slices: the Ozaki slices (0 = default)."""
    _dev(K, torch.float64)
    o = gcr_opts(float(tol), int(max_iter), MATVEC[matvec], int(slices))
    info = gcr_info()
    h = ctypes.c_void_p()
    S = np.empty((lf.n2, lf.n2), dtype=np.float64, order="F") if (want_S22_host and lf.n2) else None
    st = ctx.lib.hf_schur_gcr(ctx.h, _ptr(K), K.shape[0], lf.h, ctypes.byref(o), ctypes.byref(h),
                              _ptr(S), ctypes.byref(info))
    ok = (HF_ERR_NOT_CONVERGED, HF_ERR_BREAKDOWN) if accept_failure else ()
    ctx.check(st, ok)
    gi = GcrInfo(info.iters, info.max_rel_res_recursive, info.max_rel_res_true, st, info.matvec)
    return Hybrid(ctx, h, lf, K), gi, S


def hf_schur_gcr_dd(ctx: Context, K: torch.Tensor, lf: LowFactor, tol: float = 1e-28, max_iter: int = 100,
                    want_S22_host: bool = False, accept_failure: bool = False):
    """NEXT-1: block GCR + Schur complement in double-double with the FP64 factor lf
    (prec = 64) as preconditioner.  Returns (Hybrid, GcrInfo, (S22hi, S22lo) host or None)."""
    _dev(K, torch.float64)
    o = gcr_opts(float(tol), int(max_iter), 0, 0)
    info = gcr_info()
    h = ctypes.c_void_p()
    want = want_S22_host and lf.n2
    Sh = np.empty((lf.n2, lf.n2), dtype=np.float64, order="F") if want else None
    Sl = np.empty((lf.n2, lf.n2), dtype=np.float64, order="F") if want else None
    st = ctx.lib.hf_schur_gcr_dd(ctx.h, _ptr(K), K.shape[0], lf.h, ctypes.byref(o), ctypes.byref(h),
                                 _ptr(Sh), _ptr(Sl), ctypes.byref(info))
    ok = (HF_ERR_NOT_CONVERGED, HF_ERR_BREAKDOWN) if accept_failure else ()
    ctx.check(st, ok)
    gi = GcrInfo(info.iters, info.max_rel_res_recursive, info.max_rel_res_true, st)
    return Hybrid(ctx, h, lf, K), gi, ((Sh, Sl) if want else None)


def hf_factor_hard(ctx: Context, hy: Hybrid, eps_ker: float = 1e-10) -> int:
    kd = ctypes.c_int64()
    ctx.check(ctx.lib.hf_factor_hard(ctx.h, hy.h, float(eps_ker), ctypes.byref(kd)))
    hy.kernel_dim = kd.value
    return kd.value


def hf_solve(ctx: Context, hy: Hybrid, b: torch.Tensor, x: torch.Tensor | None = None):
    """Alg. 2 on the scaled system; b, x device FP64[L].  Returns (x, GcrInfo)."""
    _dev(b, torch.float64)
    if x is None:
        x = torch.empty_like(b)
    info = gcr_info()
    ctx.check(ctx.lib.hf_solve(ctx.h, hy.h, _ptr(b), _ptr(x), ctypes.byref(info)))
    return x, GcrInfo(info.iters, info.max_rel_res_recursive, info.max_rel_res_true)


def hf_solve_dd(ctx: Context, hy: Hybrid, b: torch.Tensor):
    """NEXT-1: Alg. 2 in double-double on a double-double hybrid.  Returns (xhi, xlo, GcrInfo)."""
    _dev(b, torch.float64)
    xh = torch.empty_like(b)
    xl = torch.empty_like(b)
    info = gcr_info()
    ctx.check(ctx.lib.hf_solve_dd(ctx.h, hy.h, _ptr(b), _ptr(xh), _ptr(xl), ctypes.byref(info)))
    return xh, xl, GcrInfo(info.iters, info.max_rel_res_recursive, info.max_rel_res_true)


def hf_nd_blocks(ctx: Context, K: torch.Tensor, levels: int, min_size: int = 8):
    """NEXT-4: nested-dissection blocks of K's pattern.  Returns (blk np.int32[L], nblk)."""
    _dev(K, torch.float64)
    L = K.shape[0]
    blk = np.empty(max(L, 1), dtype=np.int32)
    n = ctypes.c_int32()
    ctx.check(ctx.lib.hf_nd_blocks(ctx.h, L, _ptr(K), L, int(levels), int(min_size), _ptr(blk), ctypes.byref(n)))
    return blk[:L], n.value


def hf_factor_lowprec_blocks(ctx: Context, K: torch.Tensor, blk: np.ndarray, nblk: int, tau: float = 1e-2,
                             n_extra: int = 0, n_min: int = 0, nb: int = 0) -> LowFactor:
    """NEXT-4: stage 1 with multi-block postponing (blk: host int32[L], block ids in tree order)."""
    _dev(K, torch.float64)
    L = K.shape[0]
    b = np.ascontiguousarray(blk, dtype=np.int32)
    o = lowprec_opts(float(tau), int(n_extra), int(n_min), int(nb), 32, 0)
    h = ctypes.c_void_p()
    N, n2, n2t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ctx.check(ctx.lib.hf_factor_lowprec_blocks(ctx.h, L, _ptr(K), L, ctypes.byref(o), _ptr(b), int(nblk),
                                               ctypes.byref(h), ctypes.byref(N), ctypes.byref(n2), ctypes.byref(n2t)))
    return LowFactor(ctx, h, L, N.value, n2.value, n2t.value)
