// ozaki.cu -- the block mat-vec Z = beta Z + alpha mask o (K W) of the block GCR
// (Alg. 5; the "SpMM in higher precision" of P:507) with the FP64
// products emulated EXACTLY on the integer tensor cores (Ozaki scheme, error-free
// splitting into int8 slices):
//
//   K_mk = 2^{e_m} sum_{p=1..s} 2^{-7p} a_p(m,k),   a_p in [-127, 127]   (rows m)
//   W_kc = 2^{f_c} sum_{q=1..s} 2^{-7q} b_q(k,c),   b_q in [-127, 127]   (columns c)
//
// with e_m / f_c the smallest exponents bounding the row / column (max < 2^e) and
// the slices taken by truncation (x <- 128 x - trunc(128 x), exact in FP64), so
// |K_mk - 2^{e_m} sum_p ...| < 2^{e_m - 7s}.  Then
//
//   (K W)_mc ~= 2^{e_m + f_c} sum_{g=2}^{s+1} 2^{-7g} sum_{p+q=g} (A_p B_q)_mc
//
// where every A_p B_q is an int8 x int8 -> int32 GEMM, EXACT (|entry| <= Lk 127^2
// < 2^31 for Lk <= 133,000), each group's sum is exact in int64, and only the s
// group terms are rounded in FP64 (summed from the smallest).  The dropped
// products (p + q > s + 1) and the truncation bound the error by
// ~(2 + s/128) 2^{-7s} 2^{e_m + f_c} Lk, relative to max_k|K_mk| max_k|W_kc| Lk --
// the form of the FP64 GEMM bound Lk u |K||W| with 2^{-7s} in place of u:
// the default s = 8 gives 2^{-56} (FP64: u = 2^{-53}); measured at C2, s = 7 leaves
// the block GCR's true residual at 6e-12 (FP64 DMMA: 3.6e-14), s = 8 at 6.1e-14.
//
// Layout: A_p row m = column m of the symmetric K (contiguous, k-major), ldA =
// L rounded up to 16 with zero padding, slices [p][m][ldA]; B_q column c
// k-major, [q][c][ldA]; the products for one p run as ONE int8 GEMM against
// the concatenated [B_1 .. B_{s+1-p}] (A_p read once per mat-vec), on
// cuBLASLt's IMMA kernels (a plain library GEMM); the splitting and the
// combination are the kernels below.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "lt.cuh"
#include "ozaki.cuh"

namespace hf {
namespace {

// smallest e with max |x| < 2^e over the masked entries of one vector; 0 for a zero vector
__device__ __forceinline__ int exp_bound(double mx) {
    if (!(mx > 0.0)) return 0;
    int e;
    frexp(mx, &e);   // mx = f 2^e, f in [0.5, 1)
    return e;
}

__device__ __forceinline__ double block_max(double v) {
    __shared__ double red[32];
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}

// One block per vector v (a column of K = row of the symmetric K, or a column of W):
// exponent of its masked max, then its s slices, four entries (one 32-bit word per
// slice) per thread step.  Entries with mask 0 (and the padding) are 0 in every slice.
__global__ void __launch_bounds__(256) k_oz_split(int64_t len, int64_t ldA, const double *__restrict__ X,
                                                  int64_t ldx, const uint8_t *__restrict__ mask, int s,
                                                  int64_t slice_stride, int8_t *__restrict__ out,
                                                  int32_t *__restrict__ ex) {
    const int64_t v = blockIdx.x;
    const double *x = X + v * ldx;
    double mx = 0.0;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x)
        if (!mask || mask[k]) mx = fmax(mx, fabs(x[k]));
    const int e = exp_bound(block_max(mx));
    if (threadIdx.x == 0) ex[v] = e;
    uint32_t *o32 = reinterpret_cast<uint32_t *>(out + v * ldA);
    const int64_t s32 = slice_stride / 4;
    for (int64_t k4 = threadIdx.x; k4 < ldA / 4; k4 += blockDim.x) {
        double r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t k = 4 * k4 + u;
            r[u] = (k < len && (!mask || mask[k])) ? scalbn(x[k], -e) : 0.0;   // exact, |r| < 1
        }
        for (int p = 0; p < s; ++p) {
            uint32_t w = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double t = r[u] * 128.0;         // exact
                const double a = trunc(t);             // |a| <= 127
                r[u] = t - a;                          // exact, |r| < 1
                w |= (uint32_t)(uint8_t)(int8_t)a << (8 * u);
            }
            o32[p * s32 + k4] = w;
        }
    }
}

// Z_mc = beta Z_mc + alpha mask_m 2^{e_m + f_c} sum_g 2^{-7g} S_g,  S_g = sum_{p+q=g} C_p[m, (q-1) n + c]
// (int64, exact), groups summed from the smallest (g = S + 1) in FP64.  S is a template
// parameter so the S(S+1)/2 loads of an entry are all issued before the sums.
template <int S>
__global__ void __launch_bounds__(256) k_oz_combine(int64_t L, int64_t n, const int32_t *__restrict__ C, int64_t ldc,
                                                    const int32_t *__restrict__ em, const int32_t *__restrict__ fc,
                                                    const uint8_t *__restrict__ mask, double alpha, double beta,
                                                    double *__restrict__ Z, int64_t ldz) {
    const int64_t total = L * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = e % L, c = e / L;
        const bool keep = !mask || mask[m];
        double acc = 0.0;
        if (keep) {
            int32_t v[S * (S + 1) / 2];
            {
                int i = 0;
                int64_t off = 0;   // first column of product block p
#pragma unroll
                for (int p = 1; p <= S; ++p) {
#pragma unroll
                    for (int q = 1; q <= S + 1 - p; ++q) v[i++] = __ldcs(&C[(off + (int64_t)(q - 1) * n + c) * ldc + m]);
                    off += (int64_t)(S + 1 - p) * n;
                }
            }
            long long sg[S + 2];
#pragma unroll
            for (int g = 0; g < S + 2; ++g) sg[g] = 0;
            {
                int i = 0;
#pragma unroll
                for (int p = 1; p <= S; ++p)
#pragma unroll
                    for (int q = 1; q <= S + 1 - p; ++q) sg[p + q] += v[i++];
            }
#pragma unroll
            for (int g = S + 1; g >= 2; --g) acc += scalbn((double)sg[g], -7 * g);
            acc = scalbn(acc, em[m] + fc[c]);
        }
        double *z = Z + m + c * ldz;
        const double ab = keep ? __dmul_rn(alpha, acc) : 0.0;
        *z = (beta == 0.0) ? ab : fma(beta, *z, ab);
    }
}

}  // namespace

int ozaki_slices() {
    int s = 8;
    if (const char *e = getenv("HF_OZAKI_SLICES")) s = std::max(2, std::min(9, atoi(e)));
    return s;
}

void ozaki_prepare(hf_ctx *ctx, Ozaki &oz, const double *K, int64_t ld, int64_t L, const uint8_t *mask, int s,
                   int64_t n) {
    cudaStream_t st = ctx->stream;
    HF_REQUIRE(L <= 130000, "ozaki: L too large for exact int32 products");
    oz.L = L;
    oz.s = s;
    oz.ldA = (L + 15) / 16 * 16;
    oz.mask = mask;
    // rows padded to ldA too (the int8 GEMM wants every dimension a multiple of 16); the
    // padding rows are zero slices and their products are never read
    oz.A.alloc((size_t)s * oz.ldA * oz.ldA, st);
    if (oz.ldA > L) HF_CUDA(cudaMemsetAsync(oz.A.p, 0, (size_t)s * oz.ldA * oz.ldA, st));
    oz.e.alloc((size_t)std::max<int64_t>(L, 1), st);
    // the per-mat-vec buffers for blocks of up to n columns, allocated here so that a
    // caller can fall back to the DMMA product when they do not fit (hf_gcr_opts.matvec 0)
    oz.B.alloc((size_t)s * std::max<int64_t>(n, 1) * oz.ldA, st);
    oz.f.alloc((size_t)std::max<int64_t>(n, 1), st);
    oz.C.alloc((size_t)s * (s + 1) / 2 * std::max<int64_t>(n, 1) * oz.ldA, st);
    ClassTimer tm(ctx, "ozaki_split", st, 0.0, 8.0 * (double)L * L + (double)s * L * oz.ldA);
    // row m of K = column m (K symmetric): contiguous; only the masked (Lambda_1) columns
    // enter, as W is zero on the others
    k_oz_split<<<(unsigned)L, 256, 0, st>>>(L, oz.ldA, K, ld, mask, s, oz.ldA * oz.ldA, oz.A.p, oz.e.p);
    HF_CHECK_LAUNCH(ctx);
}

void ozaki_matvec(hf_ctx *ctx, Ozaki &oz, const double *W, int64_t ldw, int64_t n, double *Z, int64_t ldz,
                  double beta, double alpha) {
    cudaStream_t st = ctx->stream;
    const int64_t L = oz.L, ldA = oz.ldA;
    const int s = oz.s;
    oz.B.alloc((size_t)s * n * ldA, st);
    oz.f.alloc((size_t)std::max<int64_t>(n, 1), st);
    const int64_t ncols = (int64_t)s * (s + 1) / 2 * n;   // all products' columns
    oz.C.alloc((size_t)ncols * ldA, st);
    {
        ClassTimer tm(ctx, "ozaki_split", st, 0.0, 8.0 * (double)L * n + (double)s * n * ldA);
        k_oz_split<<<(unsigned)n, 256, 0, st>>>(L, ldA, W, ldw, oz.mask, s, n * ldA, oz.B.p, oz.f.p);
        HF_CHECK_LAUNCH(ctx);
    }
    {
        // algorithmic work of the emulated FP64 product: 2 L^2 n flop; its int8 tensor work
        // is s(s+1)/2 times that in int8 ops
        ClassTimer tm(ctx, "ozaki_imma", st, 2.0 * (double)L * L * n, (double)s * L * ldA);
        int64_t off = 0;
        for (int p = 1; p <= s; ++p) {
            const int64_t nc = (int64_t)(s + 1 - p) * n;
            lt_imma(ctx, ldA, nc, ldA, oz.A.p + (size_t)(p - 1) * ldA * ldA, ldA, oz.B.p, ldA, oz.C.p + off * ldA, ldA);
            off += nc;
        }
    }
    ClassTimer tm(ctx, "ozaki_combine", st, 0.0, 4.0 * (double)ncols * L + 16.0 * (double)L * n);
    const int64_t total = L * n;
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 16);
    switch (s) {
#define HF_OZ_COMB(S) \
    case S: k_oz_combine<S><<<grid, 256, 0, st>>>(L, n, oz.C.p, ldA, oz.e.p, oz.f.p, oz.mask, alpha, beta, Z, ldz); break;
        HF_OZ_COMB(2) HF_OZ_COMB(3) HF_OZ_COMB(4) HF_OZ_COMB(5) HF_OZ_COMB(6) HF_OZ_COMB(7) HF_OZ_COMB(8) HF_OZ_COMB(9)
#undef HF_OZ_COMB
        default: HF_REQUIRE(false, "ozaki: slices out of range");
    }
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
