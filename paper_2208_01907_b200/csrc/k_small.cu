// k_small.cu -- FP64 helper kernels of steps a4-a8:
//   block extraction (Alg. 1 step 2), per-column residual norms and
//   the convergence test [R13], inversion of the Gram matrices M_n (Alg. 5
//   P:322-330, via Cholesky) and the hard factorization of S22 (Alg. 1
//   step 5; 1x1/2x2 pivots P:84; kernel rule [R15]).
#include <cooperative_groups.h>

#include <algorithm>

#include "k_dgemm.cuh"
#include "k_small.cuh"

namespace cg = cooperative_groups;

namespace hf {
namespace {

// ------------------------------------------------------------------ gathers
// B[i + j*L] = mask1[i] ? K[i + lam2[j]*ld] : 0     (K12 in original row order)
__global__ void k_gather_cols(int64_t L, const double *__restrict__ K, int64_t ld, const int64_t *__restrict__ lam2,
                              int64_t n2, const uint8_t *__restrict__ mask1, double *__restrict__ B) {
    for (int64_t j = blockIdx.y; j < n2; j += gridDim.y) {
        const double *src = K + lam2[j] * ld;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (int64_t)gridDim.x * blockDim.x)
            B[i + j * L] = mask1[i] ? src[i] : 0.0;
    }
}

// K22[a + b*n2] = K[lam2[a] + lam2[b]*ld]
__global__ void k_gather_k22(int64_t n2, const double *__restrict__ K, int64_t ld, const int64_t *__restrict__ lam2,
                             double *__restrict__ K22) {
    const int64_t tot = n2 * n2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = e % n2, b = e / n2;
        K22[e] = K[lam2[a] + lam2[b] * ld];
    }
}

__global__ void k_mask_from_pos(int64_t L, const int32_t *__restrict__ pos1, uint8_t *__restrict__ m) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < L) m[i] = pos1[i] >= 0 ? 1 : 0;
}

// out[j] = sum_i X[i + j*ldx]^2 ; one CTA per column, fixed reduction order
__global__ void __launch_bounds__(256) k_colnorm2(int64_t M, const double *__restrict__ X, int64_t ldx,
                                                  double *__restrict__ out) {
    __shared__ double red[256];
    const int64_t j = blockIdx.x;
    const double *x = X + j * ldx;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < M; i += 256) s = fma(x[i], x[i], s);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = red[0];
}

// res = max_j sqrt(rn2_j / bn2_j) (0 if both 0, inf if only bn2 is 0)
__global__ void k_maxres(int64_t n, const double *__restrict__ rn2, const double *__restrict__ bn2, double *out) {
    __shared__ double red[256];
    double m = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += 256) {
        double r;
        if (bn2[j] > 0.0) r = sqrt(rn2[j] / bn2[j]);
        else r = (rn2[j] == 0.0) ? 0.0 : INFINITY;
        m = fmax(m, r);
    }
    red[threadIdx.x] = m;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// ------------------------------------------------------------------ SPD inverse
// Minv = M^{-1} for the SPD Gram matrix M_n of Alg. 5 by in-place
// Gauss-Jordan elimination without pivoting (for SPD M its pivots are the
// squared Cholesky diagonals, so "pivot <= 0" is exactly Cholesky breakdown
// [R11] -> status[0] |= 1).  One cooperative launch: CTA c owns a contiguous
// slice of columns; per step k every CTA reads snapshots of column k and row k
// (written by their owners at the end of step k-1) and updates its columns;
// one grid barrier per step.
//   p = a_kk;  a_ij -= a_ik a_kj / p;  a_kj /= p;  a_ik = -a_ik / p;  a_kk = 1/p
__global__ void __launch_bounds__(256) k_spd_inv(int64_t n, const double *__restrict__ M, int64_t ldm,
                                                 double *__restrict__ A, double *__restrict__ cbuf,
                                                 double *__restrict__ rbuf, int *status) {
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, tid = threadIdx.x, nt = blockDim.x;
    const int64_t per = (n + G - 1) / G;
    const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(n, j0 + per);
    for (int64_t j = j0; j < j1; ++j)
        for (int64_t i = tid; i < n; i += nt) {
            const double v = M[i + j * ldm];
            A[i + j * n] = v;
            if (j == 0) cbuf[i] = v;
            if (i == 0) rbuf[j] = v;
        }
    int bad = 0;
    grid.sync();
    for (int64_t k = 0; k < n; ++k) {
        const double *ck = cbuf + (k & 1) * n, *rk = rbuf + (k & 1) * n;
        double *cn = cbuf + ((k + 1) & 1) * n, *rn = rbuf + ((k + 1) & 1) * n;
        double p = ck[k];
        if (!(p > 0.0)) {
            bad = 1;
            p = 1.0;
        }
        const double ip = 1.0 / p;
        for (int64_t j = j0; j < j1; ++j) {
            double *aj = A + j * n;
            if (j == k) {
                for (int64_t i = tid; i < n; i += nt) {
                    const double v = (i == k) ? ip : -ck[i] / p;
                    aj[i] = v;
                    if (j == k + 1) cn[i] = v;
                    if (i == k + 1) rn[j] = v;
                }
            } else {
                const double r = rk[j] / p;
                for (int64_t i = tid; i < n; i += nt) {
                    const double v = (i == k) ? r : fma(-ck[i], r, aj[i]);
                    aj[i] = v;
                    if (j == k + 1) cn[i] = v;
                    if (i == k + 1) rn[j] = v;
                }
            }
        }
        grid.sync();
    }
    if (blockIdx.x == 0 && tid == 0 && bad) atomicOr(status, 1);
}

// ------------------------------------------------------------------ hard factorization
// Bunch-Parlett complete pivoting on A = (S22 + S22^T)/2 [R15].  Single CTA.
// A: n x n workspace (full symmetric), Lh: n x n, Dh: n x n, lab: labels.
struct Best {
    double v;
    int64_t k1, k2;   // tie keys (smaller wins)
    int64_t i, j;
};

__device__ __forceinline__ bool better(const Best &a, const Best &b) {
    if (a.v != b.v) return a.v > b.v;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    return a.k2 < b.k2;
}

__device__ Best block_best(Best b, Best *sh) {
    const int tid = threadIdx.x, nt = blockDim.x;
    sh[tid] = b;
    __syncthreads();
    for (int w = nt / 2; w > 0; w >>= 1) {
        if (tid < w && better(sh[tid + w], sh[tid])) sh[tid] = sh[tid + w];
        __syncthreads();
    }
    Best r = sh[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(512) k_hard_factor(int64_t n, const double *__restrict__ S, double thr,
                                                     double *__restrict__ A, double *__restrict__ Lh,
                                                     double *__restrict__ Dh, int32_t *__restrict__ lab,
                                                     int32_t *__restrict__ blocks, int64_t *rank_out) {
    __shared__ Best sh[512];
    __shared__ double E[4];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t tot = n * n;
    for (int64_t e = tid; e < tot; e += nt) {
        const int64_t i = e % n, j = e / n;
        A[e] = 0.5 * (S[i + j * n] + S[j + i * n]);
        Lh[e] = (i == j) ? 1.0 : 0.0;
        Dh[e] = 0.0;
    }
    for (int64_t i = tid; i < n; i += nt) {
        lab[i] = (int32_t)i;
        blocks[i] = 0;
    }
    __syncthreads();
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int64_t k = 0, nblk = 0;
    while (k < n) {
        // mu0: max |A_ij| over the trailing block (lower part suffices: A symmetric)
        // off: best off-diagonal (i > j) with label tie-break; dg: best diagonal
        Best bo{-1.0, 0, 0, -1, -1}, bd{-1.0, 0, 0, -1, -1};
        const int64_t m = n - k;
        for (int64_t e = tid; e < m * m; e += nt) {
            const int64_t i = k + e % m, j = k + e / m;
            if (i < j) continue;
            const double v = fabs(A[i + j * n]);
            if (i == j) {
                Best c{v, lab[i], 0, i, i};
                if (better(c, bd)) bd = c;
            } else {
                const int64_t la = min(lab[i], lab[j]), lb = max(lab[i], lab[j]);
                Best c{v, la, lb, i, j};
                if (better(c, bo)) bo = c;
            }
        }
        bd = block_best(bd, sh);
        bo = block_best(bo, sh);
        const double mu1 = bd.v, mu0 = fmax(bd.v, bo.v);
        if (mu0 <= thr) break;
        if (mu1 >= alpha * mu0) {
            // ---- 1x1 pivot at bd.i
            const int64_t p = bd.i;
            // swap k <-> p (rows/cols of A, rows of Lh[:, :k], labels)
            if (p != k) {
                for (int64_t c = tid; c < n; c += nt) {
                    double t = A[k + c * n]; A[k + c * n] = A[p + c * n]; A[p + c * n] = t;
                }
                __syncthreads();
                for (int64_t r = tid; r < n; r += nt) {
                    double t = A[r + k * n]; A[r + k * n] = A[r + p * n]; A[r + p * n] = t;
                }
                for (int64_t c = tid; c < k; c += nt) {
                    double t = Lh[k + c * n]; Lh[k + c * n] = Lh[p + c * n]; Lh[p + c * n] = t;
                }
                if (tid == 0) { int32_t t = lab[k]; lab[k] = lab[p]; lab[p] = t; }
                __syncthreads();
            }
            const double d = A[k + k * n];
            // A[i,j] -= (c_i c_j) / d  for i, j > k  (exactly symmetric)
            for (int64_t e = tid; e < (m - 1) * (m - 1); e += nt) {
                const int64_t i = k + 1 + e % (m - 1), j = k + 1 + e / (m - 1);
                A[i + j * n] -= (A[i + k * n] * A[j + k * n]) / d;
            }
            __syncthreads();
            for (int64_t i = k + 1 + tid; i < n; i += nt) {
                Lh[i + k * n] = A[i + k * n] / d;
                A[i + k * n] = 0.0;
                A[k + i * n] = 0.0;
            }
            if (tid == 0) { Dh[k + k * n] = d; blocks[nblk] = 1; }
            ++nblk;
            k += 1;
        } else {
            // ---- 2x2 pivot on the best off-diagonal pair, smaller label first
            int64_t i = bo.i, j = bo.j;
            if (lab[i] > lab[j]) { int64_t t = i; i = j; j = t; }
            for (int s = 0; s < 2; ++s) {
                const int64_t dst = k + s;
                int64_t p = (s == 0) ? i : j;
                if (s == 1 && j == k) p = i;   // j was moved by the first swap
                if (p != dst) {
                    for (int64_t c = tid; c < n; c += nt) {
                        double t = A[dst + c * n]; A[dst + c * n] = A[p + c * n]; A[p + c * n] = t;
                    }
                    __syncthreads();
                    for (int64_t r = tid; r < n; r += nt) {
                        double t = A[r + dst * n]; A[r + dst * n] = A[r + p * n]; A[r + p * n] = t;
                    }
                    for (int64_t c = tid; c < k; c += nt) {
                        double t = Lh[dst + c * n]; Lh[dst + c * n] = Lh[p + c * n]; Lh[p + c * n] = t;
                    }
                    if (tid == 0) { int32_t t = lab[dst]; lab[dst] = lab[p]; lab[p] = t; }
                    __syncthreads();
                }
            }
            if (tid == 0) {
                const double a = A[k + k * n], b = A[k + 1 + k * n], c = A[k + 1 + (k + 1) * n];
                const double det = a * c - b * b;
                E[0] = c / det; E[1] = -b / det; E[2] = -b / det; E[3] = a / det;   // inv(E), symmetric
                Dh[k + k * n] = a; Dh[k + 1 + k * n] = b; Dh[k + (k + 1) * n] = b; Dh[k + 1 + (k + 1) * n] = c;
                blocks[nblk] = 2;
            }
            __syncthreads();
            // Lc = C E^{-1} (C = A[k+2:, k:k+2]); A -= 0.5 (Lc C^T + C Lc^T)
            for (int64_t e = tid; e < (m - 2) * (m - 2); e += nt) {
                const int64_t r = k + 2 + e % (m - 2), c = k + 2 + e / (m - 2);
                const double cr0 = A[r + k * n], cr1 = A[r + (k + 1) * n];
                const double cc0 = A[c + k * n], cc1 = A[c + (k + 1) * n];
                const double lr0 = cr0 * E[0] + cr1 * E[1], lr1 = cr0 * E[2] + cr1 * E[3];
                const double lc0 = cc0 * E[0] + cc1 * E[1], lc1 = cc0 * E[2] + cc1 * E[3];
                const double t1 = lr0 * cc0 + lr1 * cc1, t2 = lc0 * cr0 + lc1 * cr1;
                A[r + c * n] -= 0.5 * (t1 + t2);
            }
            __syncthreads();
            for (int64_t r = k + 2 + tid; r < n; r += nt) {
                const double cr0 = A[r + k * n], cr1 = A[r + (k + 1) * n];
                Lh[r + k * n] = cr0 * E[0] + cr1 * E[1];
                Lh[r + (k + 1) * n] = cr0 * E[2] + cr1 * E[3];
                A[r + k * n] = A[r + (k + 1) * n] = 0.0;
                A[k + r * n] = A[k + 1 + r * n] = 0.0;
            }
            ++nblk;
            k += 2;
        }
        __syncthreads();
    }
    if (tid == 0) *rank_out = k;
}

// x2 = S22^+ y2 with the kernel coordinates of the pivoted vector set to 0 [R16].
// Single CTA; y, x: n-vectors (device).
__global__ void __launch_bounds__(256) k_hard_solve(int64_t n, int64_t r, const double *__restrict__ Lh,
                                                    const double *__restrict__ Dh, const int32_t *__restrict__ lab,
                                                    const int32_t *__restrict__ blocks, const double *__restrict__ y,
                                                    double *__restrict__ x, double *__restrict__ z) {
    __shared__ double red[256];
    const int tid = threadIdx.x;
    for (int64_t i = tid; i < n; i += 256) z[i] = y[lab[i]];
    __syncthreads();
    // forward: unit lower L11 (r x r)
    for (int64_t i = 0; i < r; ++i) {
        double s = 0.0;
        for (int64_t kk = tid; kk < i; kk += 256) s = fma(Lh[i + kk * n], z[kk], s);
        red[tid] = s;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (tid < w) red[tid] += red[tid + w];
            __syncthreads();
        }
        if (tid == 0) z[i] -= red[0];
        __syncthreads();
    }
    // block diagonal
    if (tid == 0) {
        int64_t k = 0;
        for (int64_t b = 0; k < r; ++b) {
            if (blocks[b] == 1) {
                z[k] = z[k] / Dh[k + k * n];
                k += 1;
            } else {
                const double a = Dh[k + k * n], bb = Dh[k + 1 + k * n], c = Dh[k + 1 + (k + 1) * n];
                const double det = a * c - bb * bb;
                const double z0 = z[k], z1 = z[k + 1];
                z[k] = (c * z0 - bb * z1) / det;
                z[k + 1] = (a * z1 - bb * z0) / det;
                k += 2;
            }
        }
    }
    __syncthreads();
    for (int64_t i = r + tid; i < n; i += 256) z[i] = 0.0;   // kernel coordinates
    __syncthreads();
    // backward: L11^T
    for (int64_t i = r - 1; i >= 0; --i) {
        double s = 0.0;
        for (int64_t kk = i + 1 + tid; kk < r; kk += 256) s = fma(Lh[kk + i * n], z[kk], s);
        red[tid] = s;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (tid < w) red[tid] += red[tid + w];
            __syncthreads();
        }
        if (tid == 0) z[i] -= red[0];
        __syncthreads();
    }
    for (int64_t i = tid; i < n; i += 256) x[lab[i]] = z[i];
}

__global__ void k_scatter_rows(int64_t n, const int64_t *__restrict__ idx, const double *__restrict__ src,
                               double *__restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[idx[i]] = src[i];
}
__global__ void k_gather_rows(int64_t n, const int64_t *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_mask_vec(int64_t L, const uint8_t *__restrict__ m, const double *__restrict__ src,
                           double *__restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < L) dst[i] = m[i] ? src[i] : 0.0;
}
// X_out (n x ncol, ld n) = X_in[perm[0..n), :] (ld L)
__global__ void k_gather_block_rows(int64_t n, int64_t ncol, const int64_t *__restrict__ perm,
                                    const double *__restrict__ X, int64_t ldx, double *__restrict__ out, int64_t ldo) {
    const int64_t tot = n * ncol;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        out[i + j * ldo] = X[perm[i] + j * ldx];
    }
}

}  // namespace

// ------------------------------------------------------------------ launchers
void gather_K12(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const int64_t *lam2, int64_t n2,
                const uint8_t *mask1, double *B) {
    ClassTimer tm_(ctx, "other");
    dim3 g((unsigned)std::min<int64_t>(cdiv(L, 256), 64), (unsigned)std::min<int64_t>(n2, 65535));
    k_gather_cols<<<g, 256, 0, ctx->stream>>>(L, K, ld, lam2, n2, mask1, B);
    HF_CHECK_LAUNCH(ctx);
}
void gather_K22(hf_ctx *ctx, int64_t n2, const double *K, int64_t ld, const int64_t *lam2, double *K22) {
    ClassTimer tm_(ctx, "other");
    k_gather_k22<<<(unsigned)std::min<int64_t>(cdiv(n2 * n2, 256), 4096), 256, 0, ctx->stream>>>(n2, K, ld, lam2, K22);
    HF_CHECK_LAUNCH(ctx);
}
void mask_from_pos(hf_ctx *ctx, int64_t L, const int32_t *pos1, uint8_t *m) {
    k_mask_from_pos<<<(unsigned)cdiv(L, 256), 256, 0, ctx->stream>>>(L, pos1, m);
    HF_CHECK_LAUNCH(ctx);
}
void colnorm2(hf_ctx *ctx, int64_t M, int64_t ncol, const double *X, int64_t ldx, double *out) {
    ClassTimer tm_(ctx, "other");
    k_colnorm2<<<(unsigned)ncol, 256, 0, ctx->stream>>>(M, X, ldx, out);
    HF_CHECK_LAUNCH(ctx);
}
void maxres(hf_ctx *ctx, int64_t n, const double *rn2, const double *bn2, double *out) {
    ClassTimer tm_(ctx, "other");
    k_maxres<<<1, 256, 0, ctx->stream>>>(n, rn2, bn2, out);
    HF_CHECK_LAUNCH(ctx);
}
void spd_inverse(hf_ctx *ctx, int64_t n, const double *M, int64_t ldm, double *Minv, DBuf<double> &wk,
                 DBuf<double> &dg, int *status) {
    (void)dg;
    ClassTimer tm_(ctx, "gram");
    wk.alloc((size_t)4 * n, ctx->stream);
    double *cb = wk.p, *rb = wk.p + 2 * n;
    int G = (int)std::min<int64_t>(std::max<int64_t>(1, cdiv(n, 4)), ctx->num_sms);
    void *args[] = {&n, &M, &ldm, &Minv, &cb, &rb, &status};
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_spd_inv, dim3(G), dim3(256), args, 0, ctx->stream));
    HF_CHECK_LAUNCH(ctx);
}
void hard_factor(hf_ctx *ctx, int64_t n, const double *S, double thr, double *A, double *Lh, double *Dh,
                 int32_t *lab, int32_t *blocks, int64_t *rank_dev) {
    ClassTimer tm(ctx, "hard");
    k_hard_factor<<<1, 512, 0, ctx->stream>>>(n, S, thr, A, Lh, Dh, lab, blocks, rank_dev);
    HF_CHECK_LAUNCH(ctx);
}
void hard_solve(hf_ctx *ctx, int64_t n, int64_t r, const double *Lh, const double *Dh, const int32_t *lab,
                const int32_t *blocks, const double *y, double *x, double *z) {
    k_hard_solve<<<1, 256, 0, ctx->stream>>>(n, r, Lh, Dh, lab, blocks, y, x, z);
    HF_CHECK_LAUNCH(ctx);
}
void scatter_rows(hf_ctx *ctx, int64_t n, const int64_t *idx, const double *src, double *dst) {
    if (n <= 0) return;
    k_scatter_rows<<<(unsigned)cdiv(n, 256), 256, 0, ctx->stream>>>(n, idx, src, dst);
    HF_CHECK_LAUNCH(ctx);
}
void gather_rows(hf_ctx *ctx, int64_t n, const int64_t *idx, const double *src, double *dst) {
    if (n <= 0) return;
    k_gather_rows<<<(unsigned)cdiv(n, 256), 256, 0, ctx->stream>>>(n, idx, src, dst);
    HF_CHECK_LAUNCH(ctx);
}
void mask_vec(hf_ctx *ctx, int64_t L, const uint8_t *m, const double *src, double *dst) {
    k_mask_vec<<<(unsigned)cdiv(L, 256), 256, 0, ctx->stream>>>(L, m, src, dst);
    HF_CHECK_LAUNCH(ctx);
}
void gather_block_rows(hf_ctx *ctx, int64_t n, int64_t ncol, const int64_t *perm, const double *X, int64_t ldx,
                       double *out, int64_t ldo) {
    ClassTimer tm_(ctx, "other");
    if (n <= 0 || ncol <= 0) return;
    k_gather_block_rows<<<(unsigned)std::min<int64_t>(cdiv(n * ncol, 256), 8192), 256, 0, ctx->stream>>>(
        n, ncol, perm, X, ldx, out, ldo);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
