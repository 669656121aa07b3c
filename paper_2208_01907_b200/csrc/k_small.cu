// k_small.cu -- FP64 helper kernels of steps a4-a8:
//   block extraction (Alg. 1 step 2), per-column residual norms and
//   the convergence test [R13], inversion of the Gram matrices M_n (Alg. 5
//   P:322-330, via Cholesky) and the hard factorization of S22 (Alg. 1
//   step 5; 1x1/2x2 pivots P:84; kernel rule [R15]).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

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

// NEXT-3: B2[i + j*L] = K[lam2[j] + i*ld] on Lambda_1 rows (K21^T in original row order)
__global__ void k_gather_rows_t(int64_t L, const double *__restrict__ K, int64_t ld, const int64_t *__restrict__ lam2,
                                int64_t n2, const uint8_t *__restrict__ mask1, double *__restrict__ B) {
    for (int64_t j = blockIdx.y; j < n2; j += gridDim.y) {
        const int64_t r = lam2[j];
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (int64_t)gridDim.x * blockDim.x)
            B[i + j * L] = mask1[i] ? K[r + i * ld] : 0.0;
    }
}

// NEXT-3: LU with complete pivoting of the nonsymmetric S22 in FP64, one CTA, in
// place: pivot = largest |entry| of the trailing block, ties -> smallest column
// label, then smallest row label (the oracle's rule); rows and columns are swapped
// physically; stop when the pivot is <= thr; A ends as [L \ U] with P S Q = L U.
__global__ void __launch_bounds__(1024) k_hard_lu(int n, const double *__restrict__ S, double thr, double *A,
                                                  int32_t *prow, int32_t *pcol, int64_t *rank_out) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    for (int64_t e = tid; e < (int64_t)n * n; e += nt) A[e] = S[e];
    for (int i = tid; i < n; i += nt) {
        prow[i] = i;
        pcol[i] = i;
    }
    __shared__ double rv[32];
    __shared__ int ri[32], rj[32], bi_s, bj_s;
    __shared__ double bv_s;
    __syncthreads();
    auto better = [&](double v, int i, int j, double bv, int bi, int bj) {
        // larger |value|; ties: smaller column label, then smaller row label
        if (v != bv) return v > bv;
        if (j < 0 || bj < 0) return bj < 0 && j >= 0;
        const int cj = pcol[j], cb = pcol[bj];
        if (cj != cb) return cj < cb;
        return prow[i] < prow[bi];
    };
    int k = 0;
    for (; k < n; ++k) {
        double bv = -1.0;
        int bi = -1, bj = -1;
        for (int64_t e = tid; e < (int64_t)(n - k) * (n - k); e += nt) {
            const int i = k + (int)(e % (n - k)), j = k + (int)(e / (n - k));
            const double v = fabs(A[i + (int64_t)j * n]);
            if (better(v, i, j, bv, bi, bj)) { bv = v; bi = i; bj = j; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (better(ov, oi, oj, bv, bi, bj)) { bv = ov; bi = oi; bj = oj; }
        }
        if (lane == 0) { rv[wid] = bv; ri[wid] = bi; rj[wid] = bj; }
        __syncthreads();
        if (tid == 0) {
            double v = -1.0;
            int i2 = -1, j2 = -1;
            for (int w = 0; w < nw; ++w)
                if (better(rv[w], ri[w], rj[w], v, i2, j2)) { v = rv[w]; i2 = ri[w]; j2 = rj[w]; }
            bv_s = v; bi_s = i2; bj_s = j2;
        }
        __syncthreads();
        if (bv_s <= thr) break;   // uniform
        const int pi = bi_s, pj = bj_s;
        // swap rows k, pi (all columns) and columns k, pj (all rows)
        if (pi != k)
            for (int j = tid; j < n; j += nt) {
                const double t = A[k + (int64_t)j * n];
                A[k + (int64_t)j * n] = A[pi + (int64_t)j * n];
                A[pi + (int64_t)j * n] = t;
            }
        __syncthreads();
        if (pj != k)
            for (int i = tid; i < n; i += nt) {
                const double t = A[i + (int64_t)k * n];
                A[i + (int64_t)k * n] = A[i + (int64_t)pj * n];
                A[i + (int64_t)pj * n] = t;
            }
        if (tid == 0) {
            const int a = prow[k]; prow[k] = prow[pi]; prow[pi] = a;
            const int b = pcol[k]; pcol[k] = pcol[pj]; pcol[pj] = b;
        }
        __syncthreads();
        const double d = A[k + (int64_t)k * n];
        for (int i = k + 1 + tid; i < n; i += nt) A[i + (int64_t)k * n] = A[i + (int64_t)k * n] / d;   // L column
        __syncthreads();
        for (int64_t e = tid; e < (int64_t)(n - k - 1) * (n - k - 1); e += nt) {
            const int i = k + 1 + (int)(e % (n - k - 1)), j = k + 1 + (int)(e / (n - k - 1));
            A[i + (int64_t)j * n] = fma(-A[i + (int64_t)k * n], A[k + (int64_t)j * n], A[i + (int64_t)j * n]);
        }
        __syncthreads();
    }
    if (tid == 0) *rank_out = k;
}

// x = S^+ y on the factored part: z = y[prow], L z' = z (r x r), U v = z', x[pcol[:r]] = v, 0 elsewhere
__global__ void k_hard_lu_solve(int n, int64_t r, const double *__restrict__ A, const int32_t *__restrict__ prow,
                                const int32_t *__restrict__ pcol, const double *__restrict__ y, double *x, double *z) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < n; i += nt) {
        z[i] = y[prow[i]];
        x[i] = 0.0;
    }
    __syncthreads();
    for (int64_t k = 0; k < r; ++k) {          // forward, unit lower
        const double zk = z[k];
        for (int64_t i = k + 1 + tid; i < r; i += nt) z[i] -= A[i + k * n] * zk;
        __syncthreads();
    }
    for (int64_t k = r - 1; k >= 0; --k) {     // backward, upper
        if (tid == 0) z[k] = z[k] / A[k + k * n];
        __syncthreads();
        const double zk = z[k];
        for (int64_t i = tid; i < k; i += nt) z[i] -= A[i + k * n] * zk;
        __syncthreads();
    }
    for (int64_t i = tid; i < r; i += nt) x[pcol[i]] = z[i];
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
// The same Gauss-Jordan inverse on one thread-block CLUSTER of 16 CTAs with the matrix in
// distributed shared memory (n <= ~640): CTA r holds the columns j = r + 16 c; after a
// step's update the owner of the next pivot column stores it into every CTA's shared buffer
// (double buffered by step parity), so one cluster barrier per step replaces the grid
// barrier and all reads are local.  Same arithmetic per entry as k_spd_inv.
constexpr int SPD_CL = 16;
__global__ void __launch_bounds__(512) k_spd_inv_cl(int n, const double *__restrict__ M, int64_t ldm,
                                                    double *__restrict__ Minv, int *status) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double smd[];
    const int r = (int)cl.block_rank(), tid = threadIdx.x, nt = blockDim.x;
    const int ncl = (n - r + SPD_CL - 1) / SPD_CL;                 // local columns
    const int ncmax = (n + SPD_CL - 1) / SPD_CL;
    double *A = smd;                                              // [ncmax][n], local column c = global r + 16 c
    double *cb = smd + (size_t)ncmax * n;                         // [2][n] pivot column buffers, then [ncmax]
    for (int e = tid; e < ncl * n; e += nt) {
        const int c = e / n, i = e % n;
        A[e] = M[i + (int64_t)(r + SPD_CL * c) * ldm];
    }
    if (r == 0)   // column 0 is the first pivot column: every CTA's buffer 0
        for (int e = tid; e < SPD_CL * n; e += nt) {
            const int dst = e / n, i = e % n;
            double *rb = cl.map_shared_rank(cb, dst);
            rb[i] = M[i];
        }
    cl.sync();
    int bad = 0;
    for (int k = 0; k < n; ++k) {
        const double *ck = cb + (k & 1) * n;
        double p = ck[k];
        if (!(p > 0.0)) {
            bad = 1;
            p = 1.0;
        }
        const double ip = 1.0 / p;
        // the row-k multipliers of the local columns first (row k is overwritten below)
        double *rrow = cb + 2 * (size_t)n;   // [ncmax]
        for (int c = tid; c < ncl; c += nt) rrow[c] = A[(size_t)c * n + k] / p;
        __syncthreads();
        for (int e = tid; e < ncl * n; e += nt) {
            const int c = e / n, i = e % n;
            const int j = r + SPD_CL * c;
            double *aj = A + (size_t)c * n;
            if (j == k) aj[i] = (i == k) ? ip : -ck[i] / p;
            else aj[i] = (i == k) ? rrow[c] : fma(-ck[i], rrow[c], aj[i]);
        }
        __syncthreads();
        if (k + 1 < n && (k + 1) % SPD_CL == r) {   // broadcast the next pivot column
            const double *src = A + (size_t)((k + 1) / SPD_CL) * n;
            for (int e = tid; e < SPD_CL * n; e += nt) {
                const int dst = e / n, i = e % n;
                double *rb = cl.map_shared_rank(cb + ((k + 1) & 1) * n, dst);
                rb[i] = src[i];
            }
        }
        cl.sync();
    }
    for (int e = tid; e < ncl * n; e += nt) {
        const int c = e / n, i = e % n;
        Minv[i + (int64_t)(r + SPD_CL * c) * n] = A[e];
    }
    if (r == 0 && tid == 0 && bad) atomicOr(status, 1);
}

// BLOCKED Gauss-Jordan on the same 16-CTA cluster (n <= ~450): the pivot block P = 16
// consecutive indices is one column per CTA, so per block step every owner broadcasts its
// column into every CTA's panel buffer (double buffered by step parity), one cluster barrier,
// then each CTA inverts A_PP (16 x 16, scalar Gauss-Jordan: its pivots are those of the
// scalar elimination, so the breakdown test [R11] is unchanged) and applies the block pivot
//   A_PP <- D = A_PP^{-1},  A_Pj <- D A_Pj,  A_iP <- -A_iP D,  A_ij <- A_ij - A_iP D A_Pj
// to its own columns: n / 16 barriers instead of n.
constexpr int SPD_BS = SPD_CL;   // one column of every pivot block per CTA (the layout requires it)
__global__ void __launch_bounds__(512) k_spd_inv_blk(int n, const double *__restrict__ M, int64_t ldm,
                                                     double *__restrict__ Minv, int *status) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double smd[];
    const int r = (int)cl.block_rank(), tid = threadIdx.x, nt = blockDim.x;
    const int ncl = (n - r + SPD_CL - 1) / SPD_CL;                // local columns (global r + 16 c)
    const int ncmax = (n + SPD_CL - 1) / SPD_CL;
    double *A = smd;                                             // [ncmax][n]
    double *PB = A + (size_t)ncmax * n;                          // [2][SPD_BS][n] panel: column k of block
    double *Rs = PB + 2 * (size_t)SPD_BS * n;                    // [ncmax][SPD_BS]  D A_Pj of own columns
    __shared__ double Ds[SPD_BS][SPD_BS + 1];
    __shared__ double dcol[SPD_BS], drow[SPD_BS];
    for (int e = tid; e < ncl * n; e += nt) {
        const int c = e / n, i = e % n;
        A[e] = M[i + (int64_t)(r + SPD_CL * c) * ldm];
    }
    __syncthreads();
    auto bcast = [&](int m) {   // own column of block m -> panel slot r of every CTA
        if (SPD_BS * m + r >= n) return;
        const double *src = A + (size_t)m * n;
        double *dstb = PB + (size_t)(m & 1) * SPD_BS * n + (size_t)r * n;
        for (int e = tid; e < SPD_CL * n; e += nt) {
            const int dst = e / n, i = e % n;
            cl.map_shared_rank(dstb, dst)[i] = src[i];
        }
    };
    bcast(0);
    cl.sync();
    int bad = 0;
    const int nblk = (n + SPD_BS - 1) / SPD_BS;
    for (int m = 0; m < nblk; ++m) {
        const int p0 = SPD_BS * m, bs = min(SPD_BS, n - p0);
        const double *P = PB + (size_t)(m & 1) * SPD_BS * n;    // P[k * n + i] = A(i, p0 + k)
        // D = A_PP^{-1} by scalar Gauss-Jordan (threads 0..bs*bs-1 own one entry each)
        const int di = tid / SPD_BS, dj = tid % SPD_BS;
        const bool dact = tid < SPD_BS * SPD_BS && di < bs && dj < bs;
        if (dact) Ds[di][dj] = P[(size_t)dj * n + p0 + di];
        __syncthreads();
        for (int k = 0; k < bs; ++k) {
            double pk = Ds[k][k];
            if (!(pk > 0.0)) {
                bad = 1;
                pk = 1.0;
            }
            if (tid < bs) {
                dcol[tid] = Ds[tid][k];
                drow[tid] = Ds[k][tid] / pk;
            }
            __syncthreads();
            if (dact) {
                double v;
                if (di == k && dj == k) v = 1.0 / pk;
                else if (di == k) v = drow[dj];
                else if (dj == k) v = -dcol[di] / pk;
                else v = fma(-dcol[di], drow[dj], Ds[di][dj]);
                Ds[di][dj] = v;
            }
            __syncthreads();
        }
        // Rs[c][k] = (D A_Pj)_k for own columns j = r + 16 c outside P (rows P read before the update)
        for (int e = tid; e < ncl * SPD_BS; e += nt) {
            const int c = e / SPD_BS, k = e % SPD_BS;
            if (c == m || k >= bs) continue;
            const double *aj = A + (size_t)c * n + p0;
            double sacc = 0.0;
            for (int l = 0; l < bs; ++l) sacc = fma(Ds[k][l], aj[l], sacc);
            Rs[c * SPD_BS + k] = sacc;
        }
        __syncthreads();
        for (int e = tid; e < ncl * n; e += nt) {
            const int c = e / n, i = e % n;
            double *aj = A + (size_t)c * n;
            const bool inP = i >= p0 && i < p0 + bs;
            if (c != m) {
                if (inP) {
                    aj[i] = Rs[c * SPD_BS + (i - p0)];
                } else {
                    double v = aj[i];
                    for (int k = 0; k < bs; ++k) v = fma(-P[(size_t)k * n + i], Rs[c * SPD_BS + k], v);
                    aj[i] = v;
                }
            } else {   // own column p0 + r of the pivot block
                if (inP) {
                    aj[i] = Ds[i - p0][r];
                } else {
                    double v = 0.0;
                    for (int k = 0; k < bs; ++k) v = fma(-P[(size_t)k * n + i], Ds[k][r], v);
                    aj[i] = v;
                }
            }
        }
        __syncthreads();
        if (m + 1 < nblk) bcast(m + 1);
        cl.sync();
    }
    for (int e = tid; e < ncl * n; e += nt) {
        const int c = e / n, i = e % n;
        Minv[i + (int64_t)(r + SPD_CL * c) * n] = A[e];
    }
    if (r == 0 && tid == 0 && bad) atomicOr(status, 1);
}

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
// Bunch-Parlett complete pivoting on A = (S22 + S22^T)/2 [R15].
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

// Multi-CTA version (one cooperative launch, any n): no physical swaps --
// indices keep their Lambda_2 position as label, an active flag marks the
// trailing block.  CTA c owns columns j = c, c+G, ... of the FULL symmetric
// work matrix (both triangles are updated with commutative formulas, so A
// stays bitwise symmetric).  Per step: search (per-CTA best diagonal and
// off-diagonal, ties by labels) -> grid barrier -> every CTA reduces the G
// partial bests and takes the same decision -> rank-1 / rank-2 update of its
// columns + the L column(s) -> grid barrier.  Two grid barriers per pivot.
__global__ void __launch_bounds__(256) k_hard_factor_mc(int64_t n, const double *__restrict__ S, double thr,
                                                        double *__restrict__ A, double *__restrict__ Lcol,
                                                        int32_t *__restrict__ act, int32_t *__restrict__ posof,
                                                        Best *__restrict__ gbest, double *__restrict__ Dh,
                                                        int32_t *__restrict__ blocks, int32_t *__restrict__ pivots,
                                                        int64_t *rank_out) {
    cg::grid_group grid = cg::this_grid();
    __shared__ Best sh[256];
    __shared__ Best sdg, soff;
    const int G = gridDim.x, tid = threadIdx.x, nt = blockDim.x;
    const int c = blockIdx.x;
    // A = (S + S^T)/2, Dh = 0, flags
    for (int64_t j = c; j < n; j += G)
        for (int64_t i = tid; i < n; i += nt) {
            A[i + j * n] = 0.5 * (S[i + j * n] + S[j + i * n]);
            Dh[i + j * n] = 0.0;
        }
    if (c == 0)
        for (int64_t i = tid; i < n; i += nt) {
            act[i] = 1;
            posof[i] = -1;
            blocks[i] = 0;
        }
    grid.sync();
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int64_t k = 0, nblk = 0;
    while (k < n) {
        // ---- search over own active columns
        Best bo{-1.0, 0, 0, -1, -1}, bd{-1.0, 0, 0, -1, -1};
        for (int64_t j = c; j < n; j += G) {
            if (!act[j]) continue;
            const double *aj = A + j * n;
            for (int64_t i = tid; i < n; i += nt) {
                if (!act[i]) continue;
                const double v = fabs(aj[i]);
                if (i == j) {
                    Best cd{v, i, 0, i, i};
                    if (better(cd, bd)) bd = cd;
                } else {
                    Best cd{v, min(i, j), max(i, j), i, j};
                    if (better(cd, bo)) bo = cd;
                }
            }
        }
        bd = block_best(bd, sh);
        bo = block_best(bo, sh);
        if (tid == 0) {
            gbest[2 * c] = bd;
            gbest[2 * c + 1] = bo;
        }
        grid.sync();
        // ---- every CTA: the same decision from the G partial bests
        if (tid < 32) {
            Best d0{-1.0, 0, 0, -1, -1}, o0{-1.0, 0, 0, -1, -1};
            for (int g = tid; g < G; g += 32) {
                if (better(gbest[2 * g], d0)) d0 = gbest[2 * g];
                if (better(gbest[2 * g + 1], o0)) o0 = gbest[2 * g + 1];
            }
            for (int o = 16; o > 0; o >>= 1) {
                Best x{__shfl_xor_sync(0xffffffffu, d0.v, o), __shfl_xor_sync(0xffffffffu, d0.k1, o),
                       __shfl_xor_sync(0xffffffffu, d0.k2, o), __shfl_xor_sync(0xffffffffu, d0.i, o),
                       __shfl_xor_sync(0xffffffffu, d0.j, o)};
                if (better(x, d0)) d0 = x;
                Best y{__shfl_xor_sync(0xffffffffu, o0.v, o), __shfl_xor_sync(0xffffffffu, o0.k1, o),
                       __shfl_xor_sync(0xffffffffu, o0.k2, o), __shfl_xor_sync(0xffffffffu, o0.i, o),
                       __shfl_xor_sync(0xffffffffu, o0.j, o)};
                if (better(y, o0)) o0 = y;
            }
            if (tid == 0) {
                sdg = d0;
                soff = o0;
            }
        }
        __syncthreads();
        const Best d0 = sdg, o0 = soff;
        const double mu1 = d0.v, mu0 = fmax(d0.v, o0.v);
        if (mu0 <= thr) break;   // uniform across the grid
        if (mu1 >= alpha * mu0) {
            // ---- 1x1 pivot at p = d0.i
            const int64_t p = d0.i;
            const double d = A[p + p * n];
            const double *ap = A + p * n;
            for (int64_t j = c; j < n; j += G) {
                if (!act[j] || j == p) continue;
                double *aj = A + j * n;
                const double apj = ap[j];
                for (int64_t i = tid; i < n; i += nt)
                    if (act[i] && i != p) aj[i] -= (ap[i] * apj) / d;
            }
            if (c == 0) {
                for (int64_t i = tid; i < n; i += nt) Lcol[i + k * n] = (act[i] && i != p) ? ap[i] / d : 0.0;
                if (tid == 0) {
                    Dh[k + k * n] = d;
                    blocks[nblk] = 1;
                    pivots[k] = (int32_t)p;
                }
            }
            grid.sync();   // column p / labels read above before the flags change
            if (c == 0 && tid == 0) {
                act[p] = 0;
                posof[p] = (int32_t)k;
            }
            ++nblk;
            k += 1;
        } else {
            // ---- 2x2 pivot on (p, q), smaller label first
            const int64_t p = min(o0.i, o0.j), q = max(o0.i, o0.j);
            const double a_ = A[p + p * n], b_ = A[q + p * n], c_ = A[q + q * n];
            const double det = a_ * c_ - b_ * b_;
            const double E0 = c_ / det, E1 = -b_ / det, E2 = -b_ / det, E3 = a_ / det;
            const double *ap = A + p * n, *aq = A + q * n;
            for (int64_t j = c; j < n; j += G) {
                if (!act[j] || j == p || j == q) continue;
                double *aj = A + j * n;
                const double cc0 = ap[j], cc1 = aq[j];
                const double lc0 = cc0 * E0 + cc1 * E1, lc1 = cc0 * E2 + cc1 * E3;
                for (int64_t i = tid; i < n; i += nt) {
                    if (!act[i] || i == p || i == q) continue;
                    const double cr0 = ap[i], cr1 = aq[i];
                    const double lr0 = cr0 * E0 + cr1 * E1, lr1 = cr0 * E2 + cr1 * E3;
                    const double t1 = lr0 * cc0 + lr1 * cc1, t2 = lc0 * cr0 + lc1 * cr1;
                    aj[i] -= 0.5 * (t1 + t2);
                }
            }
            if (c == 0) {
                for (int64_t i = tid; i < n; i += nt) {
                    const bool ok = act[i] && i != p && i != q;
                    const double cr0 = ap[i], cr1 = aq[i];
                    Lcol[i + k * n] = ok ? cr0 * E0 + cr1 * E1 : 0.0;
                    Lcol[i + (k + 1) * n] = ok ? cr0 * E2 + cr1 * E3 : 0.0;
                }
                if (tid == 0) {
                    Dh[k + k * n] = a_;
                    Dh[k + 1 + k * n] = b_;
                    Dh[k + (k + 1) * n] = b_;
                    Dh[k + 1 + (k + 1) * n] = c_;
                    blocks[nblk] = 2;
                    pivots[k] = (int32_t)p;
                    pivots[k + 1] = (int32_t)q;
                }
            }
            grid.sync();
            if (c == 0 && tid == 0) {
                act[p] = act[q] = 0;
                posof[p] = (int32_t)k;
                posof[q] = (int32_t)(k + 1);
            }
            ++nblk;
            k += 2;
        }
        grid.sync();
    }
    if (c == 0 && tid == 0) *rank_out = k;
}

// Fused variant (default): ONE grid barrier per pivot.  The update of pivot
// step k and the search for step k+1 are one pass over each CTA's columns
// (the search reads the freshly updated values and skips the step-k pivots);
// the per-CTA bests are double buffered by step parity, so a CTA that has
// decided and moved on never overwrites bests another CTA is still reading.
__device__ __forceinline__ void warp_best(Best &b) {
    for (int o = 16; o > 0; o >>= 1) {
        Best x{__shfl_xor_sync(0xffffffffu, b.v, o), __shfl_xor_sync(0xffffffffu, b.k1, o),
               __shfl_xor_sync(0xffffffffu, b.k2, o), __shfl_xor_sync(0xffffffffu, b.i, o),
               __shfl_xor_sync(0xffffffffu, b.j, o)};
        if (better(x, b)) b = x;
    }
}

// both bests of the CTA at once: warp shuffles, then one pass over the per-warp winners
// (two barriers instead of the nine of two block_best trees)
__device__ __forceinline__ void block_best2(Best &bd, Best &bo, Best *sh) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    warp_best(bd);
    warp_best(bo);
    if (lane == 0) {
        sh[wid] = bd;
        sh[32 + wid] = bo;
    }
    __syncthreads();
    if (wid == 0) {
        Best d = lane < nw ? sh[lane] : Best{-1.0, 0, 0, -1, -1};
        Best o = lane < nw ? sh[32 + lane] : Best{-1.0, 0, 0, -1, -1};
        warp_best(d);
        warp_best(o);
        if (lane == 0) {
            sh[64] = d;
            sh[65] = o;
        }
    }
    __syncthreads();
    bd = sh[64];
    bo = sh[65];
}

__global__ void __launch_bounds__(256) k_hard_factor_f(int64_t n, const double *__restrict__ S, double thr,
                                                       double *__restrict__ A, double *__restrict__ Lcol,
                                                       int32_t *__restrict__ act, int32_t *__restrict__ posof,
                                                       Best *__restrict__ gbest, double *__restrict__ Dh,
                                                       int32_t *__restrict__ blocks, int32_t *__restrict__ pivots,
                                                       int64_t *rank_out) {
    cg::grid_group grid = cg::this_grid();
    __shared__ Best sh[256];
    __shared__ Best sdg, soff;
    const int G = gridDim.x, tid = threadIdx.x, nt = blockDim.x;
    const int c = blockIdx.x;
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    // A = (S + S^T)/2 and the first search, fused
    Best bo{-1.0, 0, 0, -1, -1}, bd{-1.0, 0, 0, -1, -1};
    for (int64_t j = c; j < n; j += G)
        for (int64_t i = tid; i < n; i += nt) {
            const double v = 0.5 * (S[i + j * n] + S[j + i * n]);
            A[i + j * n] = v;
            Dh[i + j * n] = 0.0;
            if (i == j) {
                Best cd{fabs(v), i, 0, i, i};
                if (better(cd, bd)) bd = cd;
            } else {
                Best cd{fabs(v), min(i, j), max(i, j), i, j};
                if (better(cd, bo)) bo = cd;
            }
        }
    if (c == 0)
        for (int64_t i = tid; i < n; i += nt) {
            act[i] = 1;
            posof[i] = -1;
            blocks[i] = 0;
        }
    int par = 0;
    block_best2(bd, bo, sh);
    if (tid == 0) {
        gbest[(size_t)par * 2 * G + 2 * c] = bd;
        gbest[(size_t)par * 2 * G + 2 * c + 1] = bo;
    }
    grid.sync();
    int64_t k = 0, nblk = 0;
    while (k < n) {
        // ---- the same decision in every CTA from the G partial bests of this step
        if (tid < 32) {
            Best d0{-1.0, 0, 0, -1, -1}, o0{-1.0, 0, 0, -1, -1};
            const Best *gb = gbest + (size_t)par * 2 * G;
            for (int g = tid; g < G; g += 32) {
                if (better(gb[2 * g], d0)) d0 = gb[2 * g];
                if (better(gb[2 * g + 1], o0)) o0 = gb[2 * g + 1];
            }
            warp_best(d0);
            warp_best(o0);
            if (tid == 0) {
                sdg = d0;
                soff = o0;
            }
        }
        __syncthreads();
        const Best d0 = sdg, o0 = soff;
        const double mu1 = d0.v, mu0 = fmax(d0.v, o0.v);
        if (mu0 <= thr) break;   // uniform
        par ^= 1;
        bo = Best{-1.0, 0, 0, -1, -1};
        bd = Best{-1.0, 0, 0, -1, -1};
        if (mu1 >= alpha * mu0) {
            // ---- 1x1 pivot at p: update + next search in one pass
            const int64_t p = d0.i;
            const double d = A[p + p * n];
            const double *ap = A + p * n;
            for (int64_t j = c; j < n; j += G) {
                if (!act[j] || j == p) continue;
                double *aj = A + j * n;
                const double apj = ap[j];
                for (int64_t i = tid; i < n; i += nt) {
                    if (!act[i] || i == p) continue;
                    const double v = aj[i] - (ap[i] * apj) / d;
                    aj[i] = v;
                    if (i == j) {
                        Best cd{fabs(v), i, 0, i, i};
                        if (better(cd, bd)) bd = cd;
                    } else {
                        Best cd{fabs(v), min(i, j), max(i, j), i, j};
                        if (better(cd, bo)) bo = cd;
                    }
                }
            }
            if (c == 0) {
                for (int64_t i = tid; i < n; i += nt) Lcol[i + k * n] = (act[i] && i != p) ? ap[i] / d : 0.0;
                if (tid == 0) {
                    Dh[k + k * n] = d;
                    blocks[nblk] = 1;
                    pivots[k] = (int32_t)p;
                    posof[p] = (int32_t)k;
                }
            }
            block_best2(bd, bo, sh);
            if (tid == 0) {
                gbest[(size_t)par * 2 * G + 2 * c] = bd;
                gbest[(size_t)par * 2 * G + 2 * c + 1] = bo;
                // p leaves the active set BEFORE the barrier (this step skips p explicitly, so
                // no reader of this step depends on act[p]); the barrier publishes it to the
                // next step's readers
                act[p] = 0;
            }
            grid.sync();
            ++nblk;
            k += 1;
        } else {
            // ---- 2x2 pivot on (p, q), smaller label first
            const int64_t p = min(o0.i, o0.j), q = max(o0.i, o0.j);
            const double a_ = A[p + p * n], b_ = A[q + p * n], c_ = A[q + q * n];
            const double det = a_ * c_ - b_ * b_;
            const double E0 = c_ / det, E1 = -b_ / det, E2 = -b_ / det, E3 = a_ / det;
            const double *ap = A + p * n, *aq = A + q * n;
            for (int64_t j = c; j < n; j += G) {
                if (!act[j] || j == p || j == q) continue;
                double *aj = A + j * n;
                const double cc0 = ap[j], cc1 = aq[j];
                const double lc0 = cc0 * E0 + cc1 * E1, lc1 = cc0 * E2 + cc1 * E3;
                for (int64_t i = tid; i < n; i += nt) {
                    if (!act[i] || i == p || i == q) continue;
                    const double cr0 = ap[i], cr1 = aq[i];
                    const double lr0 = cr0 * E0 + cr1 * E1, lr1 = cr0 * E2 + cr1 * E3;
                    const double t1 = lr0 * cc0 + lr1 * cc1, t2 = lc0 * cr0 + lc1 * cr1;
                    const double v = aj[i] - 0.5 * (t1 + t2);
                    aj[i] = v;
                    if (i == j) {
                        Best cd{fabs(v), i, 0, i, i};
                        if (better(cd, bd)) bd = cd;
                    } else {
                        Best cd{fabs(v), min(i, j), max(i, j), i, j};
                        if (better(cd, bo)) bo = cd;
                    }
                }
            }
            if (c == 0) {
                for (int64_t i = tid; i < n; i += nt) {
                    const bool ok = act[i] && i != p && i != q;
                    const double cr0 = ap[i], cr1 = aq[i];
                    Lcol[i + k * n] = ok ? cr0 * E0 + cr1 * E1 : 0.0;
                    Lcol[i + (k + 1) * n] = ok ? cr0 * E2 + cr1 * E3 : 0.0;
                }
                if (tid == 0) {
                    Dh[k + k * n] = a_;
                    Dh[k + 1 + k * n] = b_;
                    Dh[k + (k + 1) * n] = b_;
                    Dh[k + 1 + (k + 1) * n] = c_;
                    blocks[nblk] = 2;
                    pivots[k] = (int32_t)p;
                    pivots[k + 1] = (int32_t)q;
                    posof[p] = (int32_t)k;
                    posof[q] = (int32_t)(k + 1);
                }
            }
            block_best2(bd, bo, sh);
            if (tid == 0) {
                gbest[(size_t)par * 2 * G + 2 * c] = bd;
                gbest[(size_t)par * 2 * G + 2 * c + 1] = bo;
                act[p] = act[q] = 0;   // before the barrier, as for the 1x1 pivot
            }
            grid.sync();
            ++nblk;
            k += 2;
        }
    }
    if (c == 0 && tid == 0) *rank_out = k;
}

// The fused factorization on one 16-CTA CLUSTER (n <= 600): CTA r holds the columns
// j = r + 16 c of the symmetrized S22 in shared memory; the pivot column(s) are read from
// their owner's shared memory (never modified after the decision), the per-CTA bests go into
// every CTA's shared slot array (double buffered by step parity), and one cluster barrier
// per pivot replaces the grid barrier.  Per-entry arithmetic, tie rules and outputs are
// those of k_hard_factor_f (bit-identical results).
constexpr int HC = 16;
__global__ void __launch_bounds__(512) k_hard_factor_cl(int n, const double *__restrict__ S, double thr,
                                                        double *__restrict__ Lcol, int32_t *__restrict__ posof,
                                                        double *__restrict__ Dh, int32_t *__restrict__ blocks,
                                                        int32_t *__restrict__ pivots, int64_t *rank_out) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double smh[];
    __shared__ Best sh[72];
    __shared__ Best BB[2][HC][2];
    __shared__ Best sdg, soff;
    const int r = (int)cl.block_rank(), tid = threadIdx.x, nt = blockDim.x;
    const int ncl = (n - r + HC - 1) / HC;
    const int ncmax = (n + HC - 1) / HC;
    // (c, i) of this thread's flat entries e = tid, tid + nt, ... advanced without a division
    const int c0 = tid / n, i0 = tid % n, dc = nt / n, di = nt % n;
    double *A = smh;                                  // [ncmax][n], local column c = global r + 16 c
    double *PC = A + (size_t)ncmax * n;               // [2][n] pivot column(s) of this step
    int32_t *act = reinterpret_cast<int32_t *>(PC + 2 * (size_t)n);   // [n]
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    Best bo{-1.0, 0, 0, -1, -1}, bd{-1.0, 0, 0, -1, -1};
    for (int e = tid; e < ncl * n; e += nt) {
        const int c = e / n, i = e % n;
        const int64_t j = r + HC * c;
        const double v = 0.5 * (S[i + j * n] + S[j + (int64_t)i * n]);
        A[e] = v;
        Dh[i + j * n] = 0.0;
        if (i == j) {
            Best cd{fabs(v), i, 0, i, i};
            if (better(cd, bd)) bd = cd;
        } else {
            Best cd{fabs(v), min((int64_t)i, j), max((int64_t)i, j), i, j};
            if (better(cd, bo)) bo = cd;
        }
    }
    for (int i = tid; i < n; i += nt) {
        act[i] = 1;
        if (r == 0) {
            posof[i] = -1;
            blocks[i] = 0;
        }
    }
    int par = 0;
    auto publish = [&]() {   // this CTA's bests -> slot r of every CTA (parity par)
        block_best2(bd, bo, sh);
        if (tid < HC) {
            Best *dst = cl.map_shared_rank(&BB[par][r][0], tid);
            dst[0] = bd;
            dst[1] = bo;
        }
    };
    publish();
    cl.sync();
    int k = 0, nblk = 0;
    while (k < n) {
        if (tid < 32) {
            Best d0 = tid < HC ? BB[par][tid][0] : Best{-1.0, 0, 0, -1, -1};
            Best o0 = tid < HC ? BB[par][tid][1] : Best{-1.0, 0, 0, -1, -1};
            warp_best(d0);
            warp_best(o0);
            if (tid == 0) {
                sdg = d0;
                soff = o0;
            }
        }
        __syncthreads();
        const Best d0 = sdg, o0 = soff;
        const double mu1 = d0.v, mu0 = fmax(d0.v, o0.v);
        if (mu0 <= thr) break;   // uniform across the cluster
        par ^= 1;
        bo = Best{-1.0, 0, 0, -1, -1};
        bd = Best{-1.0, 0, 0, -1, -1};
        const bool one = mu1 >= alpha * mu0;
        const int p = one ? (int)d0.i : (int)min(o0.i, o0.j), q = one ? -1 : (int)max(o0.i, o0.j);
        {   // pivot column(s) from their owners' shared memory (not modified in this step)
            const double *sp = cl.map_shared_rank(A, p % HC) + (size_t)(p / HC) * n;
            for (int i = tid; i < n; i += nt) PC[i] = sp[i];
            if (!one) {
                const double *sq = cl.map_shared_rank(A, q % HC) + (size_t)(q / HC) * n;
                for (int i = tid; i < n; i += nt) PC[n + i] = sq[i];
            }
        }
        __syncthreads();
        const double *ap = PC, *aq = PC + n;
        if (one) {
            const double d = ap[p];
            for (int e = tid, c = c0, i = i0; e < ncl * n; e += nt, c += dc, i += di, (i >= n ? (i -= n, ++c) : 0)) {
                const int j = r + HC * c;
                if (!act[j] || j == p || !act[i] || i == p) continue;
                const double v = A[e] - (ap[i] * ap[j]) / d;
                A[e] = v;
                if (i == j) {
                    Best cd{fabs(v), i, 0, i, i};
                    if (better(cd, bd)) bd = cd;
                } else {
                    Best cd{fabs(v), min(i, j), max(i, j), i, j};
                    if (better(cd, bo)) bo = cd;
                }
            }
            if (r == 0) {
                for (int i = tid; i < n; i += nt) Lcol[i + (int64_t)k * n] = (act[i] && i != p) ? ap[i] / d : 0.0;
                if (tid == 0) {
                    Dh[k + (int64_t)k * n] = d;
                    blocks[nblk] = 1;
                    pivots[k] = p;
                    posof[p] = k;
                }
            }
        } else {
            const double a_ = ap[p], b_ = ap[q], c_ = aq[q];
            const double det = a_ * c_ - b_ * b_;
            const double E0 = c_ / det, E1 = -b_ / det, E2 = -b_ / det, E3 = a_ / det;
            for (int e = tid, c = c0, i = i0; e < ncl * n; e += nt, c += dc, i += di, (i >= n ? (i -= n, ++c) : 0)) {
                const int j = r + HC * c;
                if (!act[j] || j == p || j == q || !act[i] || i == p || i == q) continue;
                const double cc0 = ap[j], cc1 = aq[j];
                const double lc0 = cc0 * E0 + cc1 * E1, lc1 = cc0 * E2 + cc1 * E3;
                const double cr0 = ap[i], cr1 = aq[i];
                const double lr0 = cr0 * E0 + cr1 * E1, lr1 = cr0 * E2 + cr1 * E3;
                const double t1 = lr0 * cc0 + lr1 * cc1, t2 = lc0 * cr0 + lc1 * cr1;
                const double v = A[e] - 0.5 * (t1 + t2);
                A[e] = v;
                if (i == j) {
                    Best cd{fabs(v), i, 0, i, i};
                    if (better(cd, bd)) bd = cd;
                } else {
                    Best cd{fabs(v), min(i, j), max(i, j), i, j};
                    if (better(cd, bo)) bo = cd;
                }
            }
            if (r == 0) {
                for (int i = tid; i < n; i += nt) {
                    const bool ok = act[i] && i != p && i != q;
                    const double cr0 = ap[i], cr1 = aq[i];
                    Lcol[i + (int64_t)k * n] = ok ? cr0 * E0 + cr1 * E1 : 0.0;
                    Lcol[i + (int64_t)(k + 1) * n] = ok ? cr0 * E2 + cr1 * E3 : 0.0;
                }
                if (tid == 0) {
                    Dh[k + (int64_t)k * n] = a_;
                    Dh[k + 1 + (int64_t)k * n] = b_;
                    Dh[k + (int64_t)(k + 1) * n] = b_;
                    Dh[k + 1 + (int64_t)(k + 1) * n] = c_;
                    blocks[nblk] = 2;
                    pivots[k] = p;
                    pivots[k + 1] = q;
                    posof[p] = k;
                    posof[q] = k + 1;
                }
            }
        }
        __syncthreads();   // every reader of act[] in this CTA is done
        if (tid == 0) {
            act[p] = 0;
            if (!one) act[q] = 0;
        }
        publish();          // (block_best2's barriers order the act[] writes for this CTA)
        cl.sync();
        ++nblk;
        k += one ? 1 : 2;
    }
    if (r == 0 && tid == 0) *rank_out = k;
}

// lab[pos] = Lambda_2 position at pivoted position pos (pivots first, then the
// kernel indices ascending); Lh (n x n, pivoted positions) unit lower with
// Lh[pos(i), kk] = Lcol[i, kk] for kk < pos(i), kk < r.
__global__ void k_hard_assemble(int64_t n, const int64_t *__restrict__ rank, const double *__restrict__ Lcol,
                                const int32_t *__restrict__ posof, const int32_t *__restrict__ pivots,
                                int32_t *__restrict__ lab, double *__restrict__ Lh) {
    const int64_t r = *rank;
    // kernel indices in ascending order get positions r, r+1, ... (one thread: n <= a few 1000)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int32_t w = (int32_t)r;
        for (int64_t i = 0; i < n; ++i)
            if (posof[i] < 0) lab[w++] = (int32_t)i;
        for (int64_t q = 0; q < r; ++q) lab[q] = pivots[q];
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e % n, kk = e / n;   // Lh[row + kk*n] for pivoted position row
        double v = (row == kk) ? 1.0 : 0.0;
        if (row > kk && kk < r && row < r) v = Lcol[(int64_t)pivots[row] + kk * n];
        Lh[e] = v;
    }
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
// Y[:, c] += alpha X[:, c]
__global__ void k_axpy_cols(int64_t L, int64_t n, double alpha, const double *__restrict__ X, int64_t ldx,
                            double *__restrict__ Y, int64_t ldy) {
    const int64_t tot = L * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % L, c = e / L;
        Y[i + c * ldy] = fma(alpha, X[i + c * ldx], Y[i + c * ldy]);
    }
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
void gather_K21T(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const int64_t *lam2, int64_t n2,
                 const uint8_t *mask1, double *B) {
    ClassTimer tm_(ctx, "other");
    dim3 g((unsigned)std::min<int64_t>(cdiv(L, 256), 64), (unsigned)std::min<int64_t>(n2, 65535));
    k_gather_rows_t<<<g, 256, 0, ctx->stream>>>(L, K, ld, lam2, n2, mask1, B);
    HF_CHECK_LAUNCH(ctx);
}
void hard_lu(hf_ctx *ctx, int64_t n, const double *S, double thr, double *A, int32_t *prow, int32_t *pcol,
             int64_t *rank_dev) {
    ClassTimer tm(ctx, "hard");
    k_hard_lu<<<1, 1024, 0, ctx->stream>>>((int)n, S, thr, A, prow, pcol, rank_dev);
    HF_CHECK_LAUNCH(ctx);
}
void hard_lu_solve(hf_ctx *ctx, int64_t n, int64_t r, const double *A, const int32_t *prow, const int32_t *pcol,
                   const double *y, double *x, double *z) {
    k_hard_lu_solve<<<1, 256, 0, ctx->stream>>>((int)n, r, A, prow, pcol, y, x, z);
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
    const size_t shm_cl = ((size_t)cdiv(n, SPD_CL) * n + 2 * (size_t)n + (size_t)cdiv(n, SPD_CL)) * sizeof(double);
    static DevState cl_ok_dev(-1);   // the 16-CTA cluster path: non-portable cluster size, checked once per device
    int &cl_ok = cl_ok_dev[ctx->device];
    if (cl_ok < 0) {
        cl_ok = getenv("HF_SPD_NOCLUSTER") ? 0 : 1;
        if (cl_ok && (cudaFuncSetAttribute(k_spd_inv_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
                      cudaFuncSetAttribute(k_spd_inv_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess))
            cl_ok = 0;
        cudaGetLastError();
    }
    const size_t shm_blk = ((size_t)cdiv(n, SPD_CL) * n + 2 * (size_t)SPD_BS * n + (size_t)cdiv(n, SPD_CL) * SPD_BS) *
                           sizeof(double);
    static DevState blk_ok_dev(-1);
    int &blk_ok = blk_ok_dev[ctx->device];
    if (blk_ok < 0) {
        blk_ok = (cl_ok && !getenv("HF_SPD_SCALAR")) ? 1 : 0;
        if (blk_ok && (cudaFuncSetAttribute(k_spd_inv_blk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
                       cudaFuncSetAttribute(k_spd_inv_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 223 * 1024) != cudaSuccess))
            blk_ok = 0;   // 223 KB: its static shared arrays count against the 227 KB
        cudaGetLastError();
    }
    if (cl_ok && n >= 1 && (shm_cl <= (size_t)227 * 1024 || (blk_ok && shm_blk <= (size_t)223 * 1024))) {
        const bool blk = blk_ok && shm_blk <= (size_t)223 * 1024;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(SPD_CL);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = blk ? shm_blk : shm_cl;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = SPD_CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int ni = (int)n;
        if (blk) HF_CUDA(cudaLaunchKernelEx(&cfg, k_spd_inv_blk, ni, M, ldm, Minv, status));
        else HF_CUDA(cudaLaunchKernelEx(&cfg, k_spd_inv_cl, ni, M, ldm, Minv, status));
        HF_CHECK_LAUNCH(ctx);
        return;
    }
    int G = (int)std::min<int64_t>(std::max<int64_t>(1, cdiv(n, 4)), ctx->num_sms);
    void *args[] = {&n, &M, &ldm, &Minv, &cb, &rb, &status};
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_spd_inv, dim3(G), dim3(256), args, 0, ctx->stream));
    HF_CHECK_LAUNCH(ctx);
}
void hard_factor(hf_ctx *ctx, int64_t n, const double *S, double thr, double *A, double *Lh, double *Dh,
                 int32_t *lab, int32_t *blocks, int64_t *rank_dev) {
    ClassTimer tm(ctx, "hard");
    cudaStream_t st = ctx->stream;
    DBuf<double> Lcol;
    Lcol.alloc((size_t)n * n, st);
    DBuf<int32_t> flags;
    flags.alloc((size_t)3 * n, st);   // act | posof | pivots
    int32_t *act = flags.p, *posof = flags.p + n, *piv = flags.p + 2 * n;
    static DevState per_sm_dev(0);
    int &per_sm = per_sm_dev[ctx->device];
    if (!per_sm) {
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hard_factor_mc, 256, 0));
        per_sm = std::max(1, per_sm);
    }
    int G = (int)std::min<int64_t>(std::max<int64_t>(1, cdiv(n, 8)), (int64_t)ctx->num_sms * std::min(per_sm, 1));
    DBuf<Best> gb;
    gb.alloc((size_t)4 * G, st);   // [2 step parities][2 G]
    void *args[] = {&n, &S, &thr, &A, &Lcol.p, &act, &posof, &gb.p, &Dh, &blocks, &piv, &rank_dev};
    static const bool unfused = getenv("HF_HARD_UNFUSED") != nullptr;   // the 3-barrier reference variant
    // the 16-CTA cluster kernel for n <= 600 (HF_HARD_NOCLUSTER: the cooperative one)
    const size_t shm_cl = ((size_t)cdiv(n, HC) * n + 2 * (size_t)n) * sizeof(double) + (size_t)n * sizeof(int32_t);
    static DevState hcl_ok_dev(-1);
    int &hcl_ok = hcl_ok_dev[ctx->device];
    if (hcl_ok < 0) {
        hcl_ok = getenv("HF_HARD_NOCLUSTER") ? 0 : 1;
        if (hcl_ok && (cudaFuncSetAttribute(k_hard_factor_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
                       cudaFuncSetAttribute(k_hard_factor_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess))
            hcl_ok = 0;
        cudaGetLastError();
    }
    if (hcl_ok && !unfused && n >= 1 && n <= 600 && shm_cl <= (size_t)200 * 1024) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(HC);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = shm_cl;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = HC;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const int ni = (int)n;
        HF_CUDA(cudaLaunchKernelEx(&cfg, k_hard_factor_cl, ni, S, thr, Lcol.p, posof, Dh, blocks, piv, rank_dev));
    } else {
        HF_CUDA(cudaLaunchCooperativeKernel(unfused ? (void *)k_hard_factor_mc : (void *)k_hard_factor_f, dim3(G),
                                            dim3(256), args, 0, st));
    }
    HF_CHECK_LAUNCH(ctx);
    k_hard_assemble<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 4096), 256, 0, st>>>(n, rank_dev, Lcol.p, posof,
                                                                                        piv, lab, Lh);
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
void axpy_cols(hf_ctx *ctx, int64_t L, int64_t n, double alpha, const double *X, int64_t ldx, double *Y,
               int64_t ldy) {
    if (L <= 0 || n <= 0) return;
    k_axpy_cols<<<(unsigned)std::min<int64_t>(cdiv(L * n, 256), 8192), 256, 0, ctx->stream>>>(L, n, alpha, X, ldx, Y, ldy);
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
