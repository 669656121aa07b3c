// k_trsm.cu -- the lower-precision preconditioner Q^{-1} of P:242 ("find e^
// satisfying Q^ e^ = r^ in lower precision ... up-converting"), used by block
// GCR (Alg. 5) and Alg. 2 step 1:
//   W = scatter_Pi( L^{-T} D^{-1} L^{-1} RN32(gather_Pi(R)) )  in FP32,
// with the FP64->FP32 truncation fused into the forward solve's load and the
// FP32->FP64 lift + scatter to original row order fused into the backward
// solve's store ("forward/backward substitution in lower precision ...
// BLAS level 3 TRSM").
//
// Design: persistent row-block-owner kernels.  Work item = (64-row block b,
// 64-column RHS chunk); items are handed out in dependency order by an atomic
// counter, each item accumulates the off-diagonal block products of the
// blocks it depends on as soon as their release flags are set (FFMA, 64x64x64
// register-tiled), then applies the precomputed inverse of its 64x64 unit
// diagonal block and releases its own flag.  No host round trips.
#include <algorithm>

#include "k_dgemm.cuh"

namespace hf {
namespace {

constexpr int TBS = 64;

__device__ __forceinline__ void st_release32(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Poll with RELAXED loads and acquire once afterwards: an ld.acquire in a spin
// loop emits an L1 invalidate (CCTL.IVALL) per iteration, which stalls every
// other CTA on the SM.
__device__ __forceinline__ int ld_relaxed32(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// inverse of each 64x64 unit-lower diagonal block (identity-padded at the edge)
__global__ void __launch_bounds__(64) k_diag_inv(int64_t N, const float *__restrict__ Lf, int64_t ldl,
                                                 float *__restrict__ Linv) {
    __shared__ float Ls[TBS][TBS + 1];
    __shared__ float Xs[TBS][TBS + 1];
    const int64_t r0 = (int64_t)blockIdx.x * TBS;
    const int j = threadIdx.x;
    for (int i = 0; i < TBS; ++i) {
        const bool ok = r0 + i < N && r0 + j < N;
        Ls[i][j] = ok ? Lf[(r0 + i) + (r0 + j) * ldl] : (i == j ? 1.f : 0.f);
    }
    __syncthreads();
    // column j of the inverse: x_i = delta_ij - sum_{j<=k<i} L_ik x_k
    for (int i = 0; i < TBS; ++i) {
        float s = (i == j) ? 1.f : 0.f;
        if (i > j)
            for (int k = j; k < i; ++k) s = __fmaf_rn(-Ls[i][k], Xs[k][j], s);
        Xs[i][j] = (i < j) ? 0.f : s;
    }
    __syncthreads();
    float *dst = Linv + (size_t)blockIdx.x * TBS * TBS;
    for (int i = 0; i < TBS; ++i) dst[i + j * TBS] = Xs[i][j];
}

struct TrsmArgs {
    int64_t N;
    int ncol, nch, nblk;
    const float *Lf;
    int64_t ldl;
    const float *Linv;
    const float *D;
    const int64_t *perm;
    const double *R;
    int64_t ldr;
    float *Y;      // forward result y (N x ncol, ld N)
    float *Xb;     // backward result x (N x ncol, ld N)
    double *W;     // output, original row order
    int64_t ldw;
    int *flags;    // [2][nblk*nch]
    int *counter;  // [2]
    int epoch;
};

// acc(4x4 per thread) -= Lt^T-ish product: acc[i][j] -= sum_k Ls[k][tr*4+i] * Ys[k][tc*4+j]
__device__ __forceinline__ void tile_fma(float (&acc)[4][4], const float (*Ls)[TBS], const float (*Ys)[TBS],
                                         int tr, int tc, float sgn) {
#pragma unroll 8
    for (int k = 0; k < TBS; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(&Ls[k][tr * 4]);
        const float4 y = *reinterpret_cast<const float4 *>(&Ys[k][tc * 4]);
        const float av[4] = {sgn * a.x, sgn * a.y, sgn * a.z, sgn * a.w};
        const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], yv[j], acc[i][j]);
    }
}

// acc[i][j] -= sum_k Ls[k][tr*4+i] * Ys[k][tc*4+j]  (negation folded into the FFMA)
__device__ __forceinline__ void tile_fma_neg(float (&acc)[4][4], const float (*Ls)[TBS], const float (*Ys)[TBS],
                                             int tr, int tc) {
#pragma unroll 8
    for (int k = 0; k < TBS; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(&Ls[k][tr * 4]);
        const float4 y = *reinterpret_cast<const float4 *>(&Ys[k][tc * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(-av[i], yv[j], acc[i][j]);
    }
}

template <bool BWD>
__global__ void __launch_bounds__(256) k_trsm(TrsmArgs a) {
    __shared__ __align__(16) float Ls[TBS][TBS];
    __shared__ __align__(16) float Ys[TBS][TBS];
    __shared__ int item_s;
    const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
    const int nitems = a.nblk * a.nch;
    int *flags = a.flags + (BWD ? nitems : 0);
    int *counter = a.counter + (BWD ? 1 : 0);
    for (;;) {
        if (tid == 0) item_s = atomicAdd(counter, 1);
        __syncthreads();
        const int item = item_s;
        __syncthreads();
        if (item >= nitems) return;
        const int b = BWD ? (a.nblk - 1 - item / a.nch) : (item / a.nch);
        const int cc = item % a.nch;
        const int64_t r0 = (int64_t)b * TBS;
        const int c0 = cc * TBS;
        float acc[4][4];
        // ---- right-hand side: forward truncates R (FP64, original order) to FP32;
        //      backward starts from z = D^{-1} y
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t r = r0 + tr * 4 + i;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = c0 + tc * 4 + j;
                float v = 0.f;
                if (r < a.N && c < a.ncol) {
                    if (!BWD) v = __double2float_rn(a.R[a.perm[r] + (int64_t)c * a.ldr]);
                    else v = __fdiv_rn(a.Y[r + (int64_t)c * a.N], a.D[r]);
                }
                acc[i][j] = v;
            }
        }
        // ---- off-diagonal blocks, earliest-finished dependency first
        //      (forward: 0, 1, ..., b-1; backward: nblk-1, ..., b+1)
        const int ndep = BWD ? (a.nblk - 1 - b) : b;
        for (int dq = 0; dq < ndep; ++dq) {
            const int cb = BWD ? (a.nblk - 1 - dq) : dq;
            if (tid == 0) {
                if (ld_relaxed32(&flags[cb * a.nch + cc]) != a.epoch) {
                    while (ld_relaxed32(&flags[cb * a.nch + cc]) != a.epoch) __nanosleep(64);
                }
                fence_acquire();
            }
            __syncthreads();
            const int64_t q0 = (int64_t)cb * TBS;
            const float *src = BWD ? a.Xb : a.Y;
#pragma unroll 4
            for (int q = 0; q < 16; ++q) {
                const int e = tid + q * 256;
                const int x = e & 63, y = e >> 6;
                // forward: Ls[k][r] = L(r0+r, q0+k)  (x = r, y = k): column q0+k contiguous in r
                // backward: Ls[k][r] = L(q0+k, r0+r) (x = k, y = r): column r0+r contiguous in k
                float lv;
                if (!BWD) {
                    const bool ok = r0 + x < a.N;
                    lv = ok ? a.Lf[(r0 + x) + (q0 + y) * a.ldl] : 0.f;
                    Ls[y][x] = lv;
                } else {
                    const bool ok = q0 + x < a.N && r0 + y < a.N;
                    lv = ok ? a.Lf[(q0 + x) + (r0 + y) * a.ldl] : 0.f;
                    Ls[x][y] = lv;
                }
                // Ys[k][c] = src(q0+k, c0+c)   (x = k, y = c)
                const bool okb = q0 + x < a.N && c0 + y < a.ncol;
                Ys[x][y] = okb ? src[(q0 + x) + (int64_t)(c0 + y) * a.N] : 0.f;
            }
            __syncthreads();
            tile_fma_neg(acc, Ls, Ys, tr, tc);
            __syncthreads();
        }
        // ---- diagonal block: out = Linv_b (or Linv_b^T) * acc
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) Ys[tr * 4 + i][tc * 4 + j] = acc[i][j];
        const float *Li = a.Linv + (size_t)b * TBS * TBS;
#pragma unroll 4
        for (int q = 0; q < 16; ++q) {
            const int e = tid + q * 256;
            const int x = e & 63, y = e >> 6;
            // forward: Ls[k][r] = Linv(r, k) (x = r, y = k);  backward: Ls[k][r] = Linv(k, r) (x = k, y = r)
            if (!BWD) Ls[y][x] = Li[x + y * TBS];
            else Ls[y][x] = Li[y + x * TBS];
        }
        __syncthreads();
        float out[4][4] = {};
        tile_fma(out, Ls, Ys, tr, tc, 1.f);
        // ---- store
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t r = r0 + tr * 4 + i;
            if (r >= a.N) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = c0 + tc * 4 + j;
                if (c >= a.ncol) continue;
                if (!BWD) {
                    a.Y[r + (int64_t)c * a.N] = out[i][j];
                } else {
                    a.Xb[r + (int64_t)c * a.N] = out[i][j];
                    a.W[a.perm[r] + (int64_t)c * a.ldw] = (double)out[i][j];   // lift + scatter
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release32(&flags[b * a.nch + cc], a.epoch);
        }
    }
}

}  // namespace

void precond_setup(hf_ctx *ctx, Precond &p, int64_t N, int64_t L, const float *Lfac, const float *D,
                   const int64_t *perm) {
    p.N = N;
    p.L = L;
    p.Lfac = Lfac;
    p.D = D;
    p.perm = perm;
    if (N == 0) return;
    const int64_t nblk = cdiv(N, TBS);
    p.Linv.alloc((size_t)nblk * TBS * TBS, ctx->stream);
    ClassTimer tm(ctx, "trsm");
    k_diag_inv<<<(unsigned)nblk, TBS, 0, ctx->stream>>>(N, Lfac, N, p.Linv.p);
    HF_CHECK_LAUNCH(ctx);
}

void precond_apply(hf_ctx *ctx, Precond &p, int64_t ncol, const double *R, int64_t ldr, double *W, int64_t ldw) {
    cudaStream_t st = ctx->stream;
    HF_CUDA(cudaMemset2DAsync(W, ldw * sizeof(double), 0, p.L * sizeof(double), ncol, st));
    if (p.N == 0 || ncol == 0) return;
    const int nblk = (int)cdiv(p.N, TBS);
    const int nch = (int)cdiv(ncol, TBS);
    p.Y.alloc((size_t)p.N * ncol, st);
    p.Xb.alloc((size_t)p.N * ncol, st);
    if (p.flags.n < (size_t)2 * nblk * nch) {
        p.flags.alloc((size_t)2 * nblk * nch, st);
        p.flags.zero(st);
        p.epoch = 0;
    }
    p.counter.alloc(2, st);
    HF_CUDA(cudaMemsetAsync(p.counter.p, 0, 2 * sizeof(int), st));
    p.epoch += 1;
    TrsmArgs a{p.N, (int)ncol, nch, nblk, p.Lfac, p.N, p.Linv.p, p.D, p.perm, R, ldr, p.Y.p, p.Xb.p, W, ldw,
               p.flags.p, p.counter.p, p.epoch};
    const int nitems = nblk * nch;
    const int grid = std::min(nitems, ctx->num_sms * 4);
    ClassTimer tm(ctx, "trsm");
    k_trsm<false><<<grid, 256, 0, st>>>(a);
    HF_CHECK_LAUNCH(ctx);
    k_trsm<true><<<grid, 256, 0, st>>>(a);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
