// k_scale.cu -- step a1: diagonal scaling K = Q Kbar Q (sec. 2 opening) [R1].
//
// HBM-bound: reads the lower triangle once (4 L^2 B) and writes the full
// symmetric FP64 matrix (8 L^2 B).  32x32 tiles of the lower triangle are
// staged in shared memory so the mirrored (transposed) write is coalesced.
#include <algorithm>

#include "hf_internal.cuh"

namespace hf {
namespace {

__global__ void k_scale_q(int64_t L, const double *__restrict__ K, int64_t ld, double *__restrict__ q,
                          int *bad) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    double d = K[i + i * ld];
    if (!isfinite(d)) atomicOr(bad, 1);
    // q_i = 1/sqrt|d| (IEEE division and square root), 1 if d == 0
    q[i] = (d != 0.0) ? __ddiv_rn(1.0, __dsqrt_rn(fabs(d))) : 1.0;
}

// One 32x32 tile (bi >= bj) of the lower triangle per CTA of 32x8 threads.
__global__ void __launch_bounds__(256) k_scale_tiles(int64_t L, double *__restrict__ K, int64_t ld,
                                                     const double *__restrict__ q, int *bad) {
    __shared__ double tile[32][33];
    const int64_t t = blockIdx.x;
    int64_t bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int64_t bj = t - bi * (bi + 1) / 2;
    const int64_t r0 = bi * 32, c0 = bj * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t qi = r0 + tx;
    const double qr = (qi < L) ? q[qi] : 0.0;
    int badl = 0;
#pragma unroll
    for (int yy = 0; yy < 32; yy += 8) {
        const int64_t j = c0 + ty + yy;   // column
        const int64_t i = r0 + tx;        // row
        double v = 0.0;
        if (i < L && j < L && i >= j) {
            double kb = K[i + j * ld];
            if (!isfinite(kb)) badl = 1;
            if (i == j) {
                v = (kb > 0.0) ? 1.0 : ((kb < 0.0) ? -1.0 : 0.0);
            } else {
                v = __dmul_rn(__dmul_rn(qr, kb), q[j]);   // (q_i Kbar_ij) q_j
            }
            K[i + j * ld] = v;
        }
        tile[ty + yy][tx] = v;   // tile[col][row]
    }
    if (badl) atomicOr(bad, 1);
    __syncthreads();
    // mirrored write: element (row i, col j) -> (row j, col i), rows of the upper tile contiguous
#pragma unroll
    for (int yy = 0; yy < 32; yy += 8) {
        const int64_t i = r0 + ty + yy;   // original row -> new column
        const int64_t j = c0 + tx;        // original col -> new row
        if (i < L && j < L && i > j) K[j + i * ld] = tile[tx][ty + yy];
    }
}

// NEXT-3: every entry of a general matrix, K_ij = (q_i Kbar_ij) q_j, diagonal sign.
__global__ void k_scale_full(int64_t L, double *__restrict__ K, int64_t ld, const double *__restrict__ q, int *bad) {
    for (int64_t j = blockIdx.x; j < L; j += gridDim.x) {
        const double qj = q[j];
        int badl = 0;
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
            const double kb = K[i + j * ld];
            if (!isfinite(kb)) badl = 1;
            K[i + j * ld] = (i == j) ? ((kb > 0.0) ? 1.0 : ((kb < 0.0) ? -1.0 : 0.0))
                                     : __dmul_rn(__dmul_rn(q[i], kb), qj);
        }
        if (badl) atomicOr(bad, 1);
    }
}

}  // namespace

void launch_scale_full(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q, int *bad_flag) {
    ClassTimer tm(ctx, "scale");
    k_scale_q<<<(unsigned)cdiv(L, 256), 256, 0, ctx->stream>>>(L, K, ld, q, bad_flag);
    HF_CHECK_LAUNCH(ctx);
    k_scale_full<<<(unsigned)std::min<int64_t>(L, 65535), 256, 0, ctx->stream>>>(L, K, ld, q, bad_flag);
    HF_CHECK_LAUNCH(ctx);
}

void launch_scale(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q, int *bad_flag) {
    ClassTimer tm(ctx, "scale");
    k_scale_q<<<(unsigned)cdiv(L, 256), 256, 0, ctx->stream>>>(L, K, ld, q, bad_flag);
    HF_CHECK_LAUNCH(ctx);
    const int64_t T = cdiv(L, 32);
    const int64_t ntiles = T * (T + 1) / 2;
    k_scale_tiles<<<(unsigned)ntiles, dim3(32, 8), 0, ctx->stream>>>(L, K, ld, q, bad_flag);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
