// ozaki2.cu -- the block mat-vec Z = beta Z + alpha mask o (K W) of the block GCR with the
// FP64 product emulated EXACTLY on the int8 tensor cores by residue arithmetic (the Chinese
// remainder form of the Ozaki scheme; hf_gcr_opts.matvec = 3):
//
//   K'_mk = trunc(K_mk 2^{53 - e_m}),  W'_kc = trunc(W_kc 2^{53 - f_c})     (|.| < 2^53, exact
//                                                                            integers in FP64)
//   C' = K' W' is an integer with |C'| <= Lk 2^106 < M / 2,  M = prod m_l  (16 pairwise
//   coprime moduli <= 256: M ~ 2^125.4, so Lk <= 2^18)
//   C'_l = (K' mod m_l)(W' mod m_l)  -- one EXACT int8 x int8 -> int32 GEMM per modulus
//          (symmetric residues in [-128, 127]; |entries| <= Lk 2^14 < 2^31 for Lk <= 130000)
//   C'   = the unique value in (-M/2, M/2) with C' = C'_l (mod m_l) for every l: Garner's
//          mixed-radix digits with symmetric digits, then Horner in FP64 (16 roundings)
//   (K W)_mc ~= C'_mc 2^{e_m + f_c - 106}
//
// The only approximations are the truncations of K and W to 53-bit integers under their row
// / column scales (|error| < Lk 2^{e_m + f_c - 52}) and the final FP64 rounding of C' (< 16
// ulps): the FP64 GEMM bound's form with the row / column maxima in place of |K||W|, 16
// int8 GEMMs per mat-vec instead of the 36 slice products of ozaki.cu.  The residues of K are
// made once per solve (16 int8 copies of K: twice the slices' memory).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "lt.cuh"
#include "ozaki.cuh"

namespace hf {
namespace {

constexpr int NMOD = 16;
constexpr int kModH[NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
// modulus l as a compile-time constant once the loops over l are unrolled (so every x % m is a
// multiply-high sequence, not a division)
__host__ __device__ constexpr int modulus(int l) {
    return l == 0 ? 256 : l == 1 ? 255 : l == 2 ? 253 : l == 3 ? 251 : l == 4 ? 247 : l == 5 ? 241 : l == 6 ? 239
         : l == 7 ? 233 : l == 8 ? 229 : l == 9 ? 227 : l == 10 ? 223 : l == 11 ? 217 : l == 12 ? 211
         : l == 13 ? 199 : l == 14 ? 197 : 193;
}
// Garner with partial products: v_l = ((r_l - sum_{j<l} v_j (P_j mod m_l)) mod m_l) Pinv_l mod m_l,
// P_j = m_0 ... m_{j-1} (P_0 = 1), Pinv_l = P_l^{-1} mod m_l
__constant__ int kPm[NMOD][NMOD];   // kPm[l][j] = P_j mod m_l (j < l)
__constant__ int kPinv[NMOD];

int inv_mod(int a, int m) {   // a^{-1} mod m (gcd 1)
    a %= m;
    for (int x = 1; x < m; ++x)
        if ((a * x) % m == 1) return x;
    return 1;
}

void upload_constants() {
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(once[dev % 64], [] {
        int pm[NMOD][NMOD] = {}, pinv[NMOD] = {};
        for (int l = 0; l < NMOD; ++l) {
            const int m = kModH[l];
            long long P = 1 % m;   // P_j mod m_l
            for (int j = 0; j < l; ++j) {
                pm[l][j] = (int)P;
                P = (P * kModH[j]) % m;
            }
            pinv[l] = inv_mod((int)P, m);   // P_l^{-1} mod m_l
        }
        cudaMemcpyToSymbol(kPm, pm, sizeof(pm));
        cudaMemcpyToSymbol(kPinv, pinv, sizeof(pinv));
    });
    HF_CUDA(cudaGetLastError());
}

__device__ __forceinline__ int exp_bound2(double mx) {
    if (!(mx > 0.0)) return 0;
    int e;
    frexp(mx, &e);
    return e;
}

__device__ __forceinline__ double block_max2(double v) {
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

// one block per vector (a column of K = row of the symmetric K, or a column of W): the
// exponent of its masked maximum, then its 16 residue vectors.  The 53-bit integer
// x' = trunc(x 2^{53-e}) (signed, two's complement) is cut into c2 2^36 + c1 2^18 + c0 with
// 0 <= c0, c1 < 2^18 and |c2| < 2^17: x' mod m = (c0 + c1 (2^18 mod m) + c2 (2^36 mod m) + O_m)
// mod m, the offset O_m (a multiple of m above 2^25) making the sum non-negative and below
// 2^27; then the symmetric range [-m/2, m/2).
__host__ __device__ constexpr unsigned pow18(int l) { return (1u << 18) % (unsigned)modulus(l); }
__host__ __device__ constexpr unsigned pow36(int l) { return pow18(l) * pow18(l) % (unsigned)modulus(l); }
__host__ __device__ constexpr int offset(int l) { return ((1 << 25) + modulus(l) - 1) / modulus(l) * modulus(l); }

__device__ __forceinline__ void chunks(double w, int &c0, int &c1, int &c2) {
    const long long s = (long long)w;   // exact: |w| < 2^53
    c0 = (int)(s & 0x3FFFF);
    c1 = (int)((s >> 18) & 0x3FFFF);
    c2 = (int)(s >> 36);
}

template <int L0>
__device__ __forceinline__ unsigned residue_byte(int c0, int c1, int c2) {
    constexpr unsigned M = (unsigned)modulus(L0);
    const unsigned y = (unsigned)(c0 + c1 * (int)pow18(L0) + c2 * (int)pow36(L0) + offset(L0));
    const unsigned r = y % M;                                           // [0, M)
    return (2 * r >= M ? r - M : r) & 0xFFu;                            // the symmetric residue's byte
}

// four consecutive entries per thread: per modulus one 32-bit store of their four residues
template <int L0>
__device__ __forceinline__ void store_residues(const int (&c)[4][3], int8_t *o, int64_t res_stride) {
    if constexpr (L0 < NMOD) {
        unsigned packed = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) packed |= residue_byte<L0>(c[i][0], c[i][1], c[i][2]) << (8 * i);
        *reinterpret_cast<unsigned *>(o + (int64_t)L0 * res_stride) = packed;
        store_residues<L0 + 1>(c, o, res_stride);
    }
}

// ldA and res_stride are multiples of 16, so every 4-entry group is 4-byte aligned
__global__ void __launch_bounds__(256) k_oz2_residues(int64_t len, int64_t ldA, const double *__restrict__ X,
                                                      int64_t ldx, const uint8_t *__restrict__ mask,
                                                      int64_t res_stride, int8_t *__restrict__ out,
                                                      int32_t *__restrict__ ex) {
    const int64_t v = blockIdx.x;
    const double *x = X + v * ldx;
    double mx = 0.0;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x)
        if (!mask || mask[k]) mx = fmax(mx, fabs(x[k]));
    const int e = exp_bound2(block_max2(mx));
    if (threadIdx.x == 0) ex[v] = e;
    int8_t *o = out + v * ldA;
    for (int64_t k0 = 4 * (int64_t)threadIdx.x; k0 < ldA; k0 += 4 * (int64_t)blockDim.x) {
        int c[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t k = k0 + i;
            const double w = (k < len && (!mask || mask[k])) ? trunc(scalbn(x[k], 53 - e)) : 0.0;   // |w| < 2^53
            chunks(w, c[i][0], c[i][1], c[i][2]);
        }
        store_residues<0>(c, o + k0, res_stride);
    }
}

// per entry: the 16 residues -> Garner's symmetric mixed-radix digits (partial products: one
// reduction per digit) -> Horner in FP64 -> the scaling, the mask, alpha and beta
template <int L0>
__device__ __forceinline__ void garner(const int32_t (&x)[NMOD], int (&v)[NMOD]) {
    if constexpr (L0 < NMOD) {
        constexpr int M = modulus(L0);
        int s = x[L0] % M;   // |x| < 2^31 -> (-M, M)
#pragma unroll
        for (int j = 0; j < L0; ++j) s -= v[j] * kPm[L0][j];   // |s| < 2^20
        int t = s % M;
        if (t < 0) t += M;
        t = (t * kPinv[L0]) % M;
        v[L0] = (2 * t >= M) ? t - M : t;                       // symmetric digit
        garner<L0 + 1>(x, v);
    }
}

__global__ void __launch_bounds__(256) k_oz2_combine(int64_t L, int64_t n, const int32_t *__restrict__ C,
                                                     int64_t ldc, int64_t cstride, const int32_t *__restrict__ em,
                                                     const int32_t *__restrict__ fc, const uint8_t *__restrict__ mask,
                                                     double alpha, double beta, double *__restrict__ Z, int64_t ldz) {
    const int64_t total = L * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = e % L, c = e / L;
        const bool keep = !mask || mask[m];
        double acc = 0.0;
        if (keep) {
            int32_t x[NMOD];
#pragma unroll
            for (int l = 0; l < NMOD; ++l) x[l] = __ldcs(&C[(int64_t)l * cstride + m + c * ldc]);
            int v[NMOD];
            garner<0>(x, v);
            double X = (double)v[NMOD - 1];
#pragma unroll
            for (int l = NMOD - 2; l >= 0; --l) X = fma(X, (double)modulus(l), (double)v[l]);
            acc = scalbn(X, em[m] + fc[c] - 106);
        }
        double *z = Z + m + c * ldz;
        const double ab = keep ? __dmul_rn(alpha, acc) : 0.0;
        *z = (beta == 0.0) ? ab : fma(beta, *z, ab);
    }
}

unsigned grid2(hf_ctx *ctx, int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16));
}

}  // namespace

void ozaki2_prepare(hf_ctx *ctx, Ozaki2 &oz, const double *K, int64_t ld, int64_t L, const uint8_t *mask,
                    int64_t n) {
    cudaStream_t st = ctx->stream;
    HF_REQUIRE(L <= 130000, "ozaki2: L too large for exact int32 residue products");
    upload_constants();
    oz.L = L;
    oz.ldA = (L + 15) / 16 * 16;
    oz.mask = mask;
    const int64_t ldA = oz.ldA;
    oz.A.alloc((size_t)NMOD * ldA * ldA, st);
    if (ldA > L) HF_CUDA(cudaMemsetAsync(oz.A.p, 0, (size_t)NMOD * ldA * ldA, st));
    oz.e.alloc((size_t)std::max<int64_t>(L, 1), st);
    oz.B.alloc((size_t)NMOD * std::max<int64_t>(n, 1) * ldA, st);
    oz.f.alloc((size_t)std::max<int64_t>(n, 1), st);
    oz.C.alloc((size_t)NMOD * std::max<int64_t>(n, 1) * ldA, st);
    ClassTimer tm(ctx, "ozaki_split", st, 0.0, 8.0 * (double)L * L + (double)NMOD * L * ldA);
    k_oz2_residues<<<(unsigned)L, 256, 0, st>>>(L, ldA, K, ld, mask, ldA * ldA, oz.A.p, oz.e.p);
    HF_CHECK_LAUNCH(ctx);
}

void ozaki2_matvec(hf_ctx *ctx, Ozaki2 &oz, const double *W, int64_t ldw, int64_t n, double *Z, int64_t ldz,
                   double beta, double alpha) {
    cudaStream_t st = ctx->stream;
    const int64_t L = oz.L, ldA = oz.ldA;
    oz.B.alloc((size_t)NMOD * n * ldA, st);
    oz.f.alloc((size_t)std::max<int64_t>(n, 1), st);
    oz.C.alloc((size_t)NMOD * n * ldA, st);
    {
        ClassTimer tm(ctx, "ozaki_split", st, 0.0, 8.0 * (double)L * n + (double)NMOD * n * ldA);
        k_oz2_residues<<<(unsigned)n, 256, 0, st>>>(L, ldA, W, ldw, oz.mask, n * ldA, oz.B.p, oz.f.p);
        HF_CHECK_LAUNCH(ctx);
    }
    {
        ClassTimer tm(ctx, "ozaki_imma", st, 2.0 * (double)L * L * n, (double)NMOD * L * ldA);
        for (int l = 0; l < NMOD; ++l)
            lt_imma(ctx, ldA, n, ldA, oz.A.p + (size_t)l * ldA * ldA, ldA, oz.B.p + (size_t)l * n * ldA, ldA,
                    oz.C.p + (size_t)l * n * ldA, ldA);
    }
    ClassTimer tm(ctx, "ozaki_combine", st, 0.0, 4.0 * NMOD * (double)n * L + 16.0 * (double)L * n);
    k_oz2_combine<<<grid2(ctx, L * n), 256, 0, st>>>(L, n, oz.C.p, ldA, n * ldA, oz.e.p, oz.f.p, oz.mask, alpha,
                                                      beta, Z, ldz);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
