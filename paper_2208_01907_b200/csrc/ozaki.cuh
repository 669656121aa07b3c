// ozaki.cuh -- FP64 block mat-vec emulated on the int8 tensor cores (ozaki.cu).
#pragma once
#include "hf_internal.cuh"

namespace hf {

struct Ozaki {
    int64_t L = 0, ldA = 0;
    int s = 0;
    const uint8_t *mask = nullptr;   // Lambda_1 rows / columns (borrowed)
    DBuf<int8_t> A;                  // [s][ldA][ldA] slices of K (row m = column m; rows >= L zero)
    DBuf<int32_t> e;                 // [L] row exponents
    DBuf<int8_t> B;                  // [s][n][ldA] slices of the current W
    DBuf<int32_t> f;                 // [n] column exponents
    DBuf<int32_t> C;                 // int32 products, s(s+1)/2 x n columns of ldA
};

// the residue (Chinese remainder) form, ozaki2.cu: 16 int8 residues of the 53-bit integer
// scalings of K and W, one exact int8 GEMM per modulus, Garner reconstruction
struct Ozaki2 {
    int64_t L = 0, ldA = 0;
    const uint8_t *mask = nullptr;
    DBuf<int8_t> A;                  // [16][ldA][ldA] residues of K (row m = column m; rows >= L zero)
    DBuf<int32_t> e;                 // [L] row exponents
    DBuf<int8_t> B;                  // [16][n][ldA] residues of the current W
    DBuf<int32_t> f;                 // [n] column exponents
    DBuf<int32_t> C;                 // [16][n][ldA] int32 products
};
void ozaki2_prepare(hf_ctx *ctx, Ozaki2 &oz, const double *K, int64_t ld, int64_t L, const uint8_t *mask,
                    int64_t n);
void ozaki2_matvec(hf_ctx *ctx, Ozaki2 &oz, const double *W, int64_t ldw, int64_t n, double *Z, int64_t ldz,
                   double beta, double alpha);

// slices per operand (HF_OZAKI_SLICES, default 8: 56 bits)
int ozaki_slices();
// split the symmetric K (L x L, ld) restricted to the masked columns, once per solve, and
// allocate the buffers of mat-vecs with up to n columns (HF_ERR_OOM when they do not fit)
void ozaki_prepare(hf_ctx *ctx, Ozaki &oz, const double *K, int64_t ld, int64_t L, const uint8_t *mask, int s,
                   int64_t n);
// Z = beta Z + alpha mask o (K W)   (W: L x n, ldw, zero outside the mask)
void ozaki_matvec(hf_ctx *ctx, Ozaki &oz, const double *W, int64_t ldw, int64_t n, double *Z, int64_t ldz,
                  double beta, double alpha);

}  // namespace hf
