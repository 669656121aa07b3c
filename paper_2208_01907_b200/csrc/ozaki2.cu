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
// P_j = m_0 ... m_{j-1} (P_0 = 1), Pinv_l = P_l^{-1} mod m_l (k_oz2_combine)

int inv_mod(int a, int m) {   // a^{-1} mod m (gcd 1)
    a %= m;
    for (int x = 1; x < m; ++x)
        if ((a * x) % m == 1) return x;
    return 1;
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
// exponent e of its masked maximum, then its 16 residue vectors.  The 53-bit integer
// x' = trunc(x 2^{53-e}) (two's complement) is cut into five 13-bit chunks,
// x' = c0 + c1 2^13 + c2 2^26 + c3 2^39 + c4 2^52 (0 <= c0..c3 < 2^13, c4 in [-2, 1]), and per
// modulus, all in exact FP32 arithmetic (every value an integer below 2^24):
//   y = sum_i c_i p_i,  p_i = 2^{13 i} mod m in [-m/2, m/2]     (|y| < 3.2e6 < 2^22)
//   q = rint(y / m)  as  fma(y, fl(1/m), 1.5 2^23) - 1.5 2^23   (|y fl(1/m) - y/m| < 1e-3, while
//                     y/m is >= 1/(2m) >= 2e-3 from a half-integer for odd m; exact for m = 256)
//   r = y - q m, |r| <= m/2, taken as the low byte of the float r + 1.5 2^23
// so r = x' (mod m) with |r| <= 128 (-128 for the one tie of m = 256): a residue the int8 GEMM
// takes as is (the combine reduces its sums mod m again).
__host__ __device__ constexpr int pchunk(int l, int i) {   // 2^{13 i} mod m, symmetric
    int r = 1;
    for (int k = 0; k < i; ++k) r = r * (1 << 13) % modulus(l);
    return 2 * r > modulus(l) ? r - modulus(l) : r;
}
constexpr float kMagic = 12582912.0f;   // 1.5 2^23: adding it rounds to an integer, keeps two's complement bits

// two entries at once (FFMA2 / FADD2: two independent IEEE operations per instruction); the
// per-modulus constants as float2 pairs in constant memory so FFMA2 reads them as operands
__constant__ float2 kRc[NMOD][6];   // p_1..p_4, 1/m, -m (each duplicated)

template <int L0>
__device__ __forceinline__ float2 residue_pair(const float2 (&c)[5]) {
    const float2 mg = make_float2(kMagic, kMagic);
    float2 y = __ffma2_rn(c[1], kRc[L0][0], c[0]);
    y = __ffma2_rn(c[2], kRc[L0][1], y);
    y = __ffma2_rn(c[3], kRc[L0][2], y);
    y = __ffma2_rn(c[4], kRc[L0][3], y);
    const float2 q = __fadd2_rn(__ffma2_rn(y, kRc[L0][4], mg), make_float2(-kMagic, -kMagic));
    return __ffma2_rn(q, kRc[L0][5], __fadd2_rn(y, mg));   // r + 1.5 2^23: r in byte 0
}

// four consecutive entries per thread (two pairs): per modulus one 32-bit store of their four
// residues
template <int L0>
__device__ __forceinline__ void store_residues(const float2 (&c01)[5], const float2 (&c23)[5], int8_t *o,
                                               int64_t res_stride) {
    if constexpr (L0 < NMOD) {
        const float2 r01 = residue_pair<L0>(c01), r23 = residue_pair<L0>(c23);
        const unsigned lo = __byte_perm(__float_as_uint(r01.x), __float_as_uint(r01.y), 0x0040);
        const unsigned hi = __byte_perm(__float_as_uint(r23.x), __float_as_uint(r23.y), 0x0040);
        *reinterpret_cast<unsigned *>(o + (int64_t)L0 * res_stride) = __byte_perm(lo, hi, 0x5410);
        store_residues<L0 + 1>(c01, c23, o, res_stride);
    }
}

__device__ __forceinline__ float chunk_f(unsigned bits) {   // 0 <= bits < 2^13, exactly
    return __int_as_float((int)(bits | 0x4B000000u)) - 8388608.0f;
}

// ldA and res_stride are multiples of 16, so every 4-entry group is 4-byte aligned
// the exponent of a vector's masked maximum (one block per vector)
__device__ __forceinline__ int vector_exponent(const double *x, int64_t len, const uint8_t *mask) {
    double mx = 0.0;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x)
        if (!mask || mask[k]) mx = fmax(mx, fabs(x[k]));
    return exp_bound2(block_max2(mx));
}

__global__ void __launch_bounds__(256) k_oz2_exponents(int64_t len, const double *__restrict__ X, int64_t ldx,
                                                       const uint8_t *__restrict__ mask, int32_t *__restrict__ ex) {
    const int e = vector_exponent(X + (int64_t)blockIdx.x * ldx, len, mask);
    if (threadIdx.x == 0) ex[blockIdx.x] = e;
}

// given = 0: one block per vector finds the exponent itself (K: L blocks fill the GPU);
// given = 1: the exponents are in ex already (k_oz2_exponents) and blockIdx.y cuts each vector
// into gridDim.y pieces (W: n vectors alone would leave most SMs idle)
__global__ void __launch_bounds__(256) k_oz2_residues(int64_t len, int64_t ldA, const double *__restrict__ X,
                                                      int64_t ldx, const uint8_t *__restrict__ mask,
                                                      int64_t res_stride, int8_t *__restrict__ out,
                                                      int32_t *__restrict__ ex, int given) {
    const int64_t v = blockIdx.x;
    const double *x = X + v * ldx;
    int e;
    if (given) {
        e = ex[v];
    } else {
        e = vector_exponent(x, len, mask);
        if (threadIdx.x == 0) ex[v] = e;
    }
    // x 2^{53-e} as (x 2^a) 2^b with both factors normal doubles (e can be as low as -1073)
    const int a = min(53 - e, 1000);
    const double sa = ldexp(1.0, a), sb = ldexp(1.0, 53 - e - a);
    const int64_t piece = (ldA / 4 + gridDim.y - 1) / gridDim.y * 4;   // entries per piece, a multiple of 4
    const int64_t kbeg = (int64_t)blockIdx.y * piece, kend = min(ldA, kbeg + piece);
    int8_t *o = out + v * ldA;
    for (int64_t k0 = kbeg + 4 * (int64_t)threadIdx.x; k0 < kend; k0 += 4 * (int64_t)blockDim.x) {
        float2 c01[5], c23[5];   // the chunks of entries (k0, k0+1) and (k0+2, k0+3) as FFMA2 pairs
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            // branch-free: loads at a clamped index (len >= 1), then the selection
            const int64_t k = k0 + i, kc = min(k, len - 1);
            const double xl = __ldg(x + kc);
            const bool keep = k < len && (!mask || __ldg(mask + kc));
            const double xv = keep ? xl : 0.0;
            const long long s = __double2ll_rz((xv * sa) * sb);   // |s| < 2^53, exact scaling
            const unsigned lo = (unsigned)s, hi = (unsigned)((unsigned long long)s >> 32);
            float2 *c = i < 2 ? c01 : c23;
            float *cc[5] = {i & 1 ? &c[0].y : &c[0].x, i & 1 ? &c[1].y : &c[1].x, i & 1 ? &c[2].y : &c[2].x,
                            i & 1 ? &c[3].y : &c[3].x, i & 1 ? &c[4].y : &c[4].x};
            *cc[0] = chunk_f(lo & 0x1FFFu);
            *cc[1] = chunk_f((lo >> 13) & 0x1FFFu);
            *cc[2] = chunk_f(__funnelshift_r(lo, hi, 26) & 0x1FFFu);
            *cc[3] = chunk_f((hi >> 7) & 0x1FFFu);
            *cc[4] = (float)((int)hi >> 20);                    // s >> 52 in [-2, 1]
        }
        store_residues<0>(c01, c23, o + k0, res_stride);
    }
}


// Garner in exact FP32 arithmetic, two entries at once (FFMA2).  Digit l of the symmetric
// mixed radix, v_l = ((x_l - sum_{j<l} v_j P_j) Pinv_l) mod m_l in [-m_l/2, m_l/2]:
//   s = x_lo + x_hi (2^16 mod m) - sum_j v_j (P_j mod m)   (x_l = x_hi 2^16 + x_lo, int32 sum of
//       the GEMM; |s| < 2^22 + 2^16 + 15 2^14 < 4.6e6, an exact FP32 integer)
//   r = s - m rint(s/m)       (rint by the 1.5 2^23 constant: |s fl(1/m) - s/m| < 1.4e-3 < 1/(2m)
//                              for every odd m <= 255, exact for m = 256, so r is the symmetric
//                              residue)
//   v = w - m rint(w/m), w = r Pinv_l  (|w| <= 2^14: exact, symmetric again)
// then Horner in FP64 (16 roundings) as before.
__constant__ float2 kGc[NMOD][NMOD + 5];   // [l][j < l]: -(P_j mod m_l); [l][16..20]: 2^16 mod m_l, Pinv_l, 1/m_l, -m_l, 0

__device__ __forceinline__ float2 round_mod(float2 s, const float2 &invm, const float2 &negm) {
    const float2 mg = make_float2(kMagic, kMagic);
    const float2 q = __fadd2_rn(__ffma2_rn(s, invm, mg), make_float2(-kMagic, -kMagic));
    return __ffma2_rn(q, negm, s);
}

template <int L0>
__device__ __forceinline__ void garner2(const float2 (&xlo)[NMOD], const float2 (&xhi)[NMOD], float2 (&v)[NMOD]) {
    if constexpr (L0 < NMOD) {
        float2 s = __ffma2_rn(xhi[L0], kGc[L0][16], xlo[L0]);
#pragma unroll
        for (int j = 0; j < L0; ++j) s = __ffma2_rn(v[j], kGc[L0][j], s);
        const float2 r = round_mod(s, kGc[L0][18], kGc[L0][19]);
        v[L0] = round_mod(__fmul2_rn(r, kGc[L0][17]), kGc[L0][18], kGc[L0][19]);
        garner2<L0 + 1>(xlo, xhi, v);
    }
}

__device__ __forceinline__ void split16(int32_t x, float &lo, float &hi) {   // exact: x = hi 2^16 + lo
    lo = __int_as_float((int)(((unsigned)x & 0xFFFFu) | 0x4B000000u)) - 8388608.0f;
    hi = __int_as_float((int)((((unsigned)x >> 16) ^ 0x8000u) | 0x4B000000u)) - 8421376.0f;   // 2^23 + 2^15
}

// two entries per thread, rows m and m + 1 of column c = blockIdx.y (one 8-byte load per
// modulus: ldc and cstride are multiples of 16 and row ldA - 1 >= L - 1 exists): the 16 int32
// sums -> digits -> Horner (digit pairs first, exactly in FP32: |v_{2k+1} m_{2k} + v_{2k}| < 2^16)
// -> the scaling, the mask, alpha and beta
__global__ void __launch_bounds__(256) k_oz2_combine(int64_t L, const int32_t *__restrict__ C, int64_t ldc,
                                                     int64_t cstride, const int32_t *__restrict__ em,
                                                     const int32_t *__restrict__ fc, const uint8_t *__restrict__ mask,
                                                     double alpha, double beta, double *__restrict__ Z, int64_t ldz) {
    const int64_t c = blockIdx.y, m = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (m >= L) return;
    const bool two = m + 1 < L;
    const bool keep0 = !mask || mask[m], keep1 = two && (!mask || mask[m + 1]);
    float2 xlo[NMOD], xhi[NMOD];
    const int32_t *cp = C + m + c * ldc;
#pragma unroll
    for (int l = 0; l < NMOD; ++l) {
        const int2 x = __ldcs(reinterpret_cast<const int2 *>(cp + (int64_t)l * cstride));
        float lo0, hi0, lo1, hi1;
        split16(x.x, lo0, hi0);
        split16(x.y, lo1, hi1);
        xlo[l] = make_float2(lo0, lo1);
        xhi[l] = make_float2(hi0, hi1);
    }
    float2 v[NMOD];
    garner2<0>(xlo, xhi, v);
    double X0 = 0.0, X1 = 0.0;
#pragma unroll
    for (int k = NMOD / 2 - 1; k >= 0; --k) {
        const float mk = (float)modulus(2 * k);
        const float2 u = __ffma2_rn(v[2 * k + 1], make_float2(mk, mk), v[2 * k]);
        const double R = (double)modulus(2 * k) * (double)modulus(2 * k + 1);
        X0 = fma(X0, R, (double)u.x);
        X1 = fma(X1, R, (double)u.y);
    }
    const int32_t fcol = fc[c];
    double *z = Z + m + c * ldz;
    {
        const double ab = keep0 ? __dmul_rn(alpha, scalbn(X0, em[m] + fcol - 106)) : 0.0;
        z[0] = (beta == 0.0) ? ab : fma(beta, z[0], ab);
    }
    if (two) {
        const double ab = keep1 ? __dmul_rn(alpha, scalbn(X1, em[m + 1] + fcol - 106)) : 0.0;
        z[1] = (beta == 0.0) ? ab : fma(beta, z[1], ab);
    }
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
        float2 rc[NMOD][6];
        for (int l = 0; l < NMOD; ++l) {
            for (int i = 1; i <= 4; ++i) rc[l][i - 1] = make_float2((float)pchunk(l, i), (float)pchunk(l, i));
            rc[l][4] = make_float2(1.0f / (float)kModH[l], 1.0f / (float)kModH[l]);
            rc[l][5] = make_float2(-(float)kModH[l], -(float)kModH[l]);
        }
        cudaMemcpyToSymbol(kRc, rc, sizeof(rc));
        float2 gc[NMOD][NMOD + 5] = {};
        auto sym = [](long long r, int m) { r %= m; if (r < 0) r += m; return (float)(2 * r > m ? r - m : r); };
        for (int l = 0; l < NMOD; ++l) {
            const int m = kModH[l];
            for (int j = 0; j < l; ++j) gc[l][j] = make_float2(-sym(pm[l][j], m), -sym(pm[l][j], m));
            gc[l][16] = make_float2(sym(65536, m), sym(65536, m));
            gc[l][17] = make_float2(sym(pinv[l], m), sym(pinv[l], m));
            gc[l][18] = make_float2(1.0f / (float)m, 1.0f / (float)m);
            gc[l][19] = make_float2(-(float)m, -(float)m);
        }
        cudaMemcpyToSymbol(kGc, gc, sizeof(gc));
    });
    HF_CUDA(cudaGetLastError());
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
    k_oz2_residues<<<(unsigned)L, 256, 0, st>>>(L, ldA, K, ld, mask, ldA * ldA, oz.A.p, oz.e.p, 0);
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
        k_oz2_exponents<<<(unsigned)n, 256, 0, st>>>(L, W, ldw, oz.mask, oz.f.p);
        HF_CHECK_LAUNCH(ctx);
        // pieces of >= 4096 entries, about eight blocks per SM over all columns
        const int64_t want = std::max<int64_t>(1, (int64_t)ctx->num_sms * 8 / std::max<int64_t>(n, 1));
        const unsigned pieces = (unsigned)std::min<int64_t>(want, std::max<int64_t>(1, ldA / 4096));
        k_oz2_residues<<<dim3((unsigned)n, pieces), 256, 0, st>>>(L, ldA, W, ldw, oz.mask, n * ldA, oz.B.p,
                                                                  oz.f.p, 1);
        HF_CHECK_LAUNCH(ctx);
    }
    {
        ClassTimer tm(ctx, "ozaki_imma", st, 2.0 * (double)L * L * n, (double)NMOD * L * ldA);
        // the 16 products as one strided batch (16 x the tiles of one product: no partial last wave)
        static const bool batched = !(getenv("HF_OZ2_BATCH") && atoi(getenv("HF_OZ2_BATCH")) == 0);
        if (batched)
            lt_imma(ctx, ldA, n, ldA, oz.A.p, ldA, oz.B.p, ldA, oz.C.p, ldA, NMOD, ldA * ldA, n * ldA, n * ldA);
        else
            for (int l = 0; l < NMOD; ++l)
                lt_imma(ctx, ldA, n, ldA, oz.A.p + (size_t)l * ldA * ldA, ldA, oz.B.p + (size_t)l * n * ldA, ldA,
                        oz.C.p + (size_t)l * n * ldA, ldA);
    }
    ClassTimer tm(ctx, "ozaki_combine", st, 0.0, 4.0 * NMOD * (double)n * L + 16.0 * (double)L * n);
    k_oz2_combine<<<dim3((unsigned)((L + 511) / 512), (unsigned)n), 256, 0, st>>>(L, oz.C.p, ldA, n * ldA, oz.e.p,
                                                                                oz.f.p, oz.mask, alpha, beta, Z, ldz);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
