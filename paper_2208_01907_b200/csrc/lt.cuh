// lt.cuh -- the plain library GEMMs libhf issues through cuBLASLt (lt.cu): the exact
// int8 slice products of the emulated FP64 mat-vec (ozaki.cu) and the FP32 / 3xTF32
// block products of the blocked preconditioner (k_trsm_blk.cu).  Descriptors and the
// heuristic's algorithm are cached per shape; one handle per device, one workspace per stream.
#pragma once
#include <cuda_bf16.h>

#include "hf_internal.cuh"

namespace hf {

// D (rows x cols, int32, ldd) = A^T B;  A: k x rows int8 (lda), B: k x cols int8 (ldb);
// `batch` problems at the given element strides
void lt_imma(hf_ctx *ctx, int64_t rows, int64_t cols, int64_t k, const int8_t *A, int64_t lda, const int8_t *B,
             int64_t ldb, int32_t *D, int64_t ldd, int batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sD = 0);

// C = alpha op(A) op(B) + beta C, FP32 column-major, `batch` problems at the given element
// strides; tf32: the tensor-core TF32 path (inputs rounded to TF32 by the hardware, FP32
// accumulation), else IEEE FP32 arithmetic.
void lt_sgemm(hf_ctx *ctx, bool tA, bool tB, int64_t m, int64_t n, int64_t k, float alpha, const float *A,
              int64_t lda, int64_t sA, const float *B, int64_t ldb, int64_t sB, float beta, float *C, int64_t ldc,
              int64_t sC, int batch, bool tf32);

// C = alpha op(A) B + beta C with bfloat16 operands, FP32 output and accumulation, on stream st
// (0: the context stream), `batch` problems at the given element strides
void lt_bgemm(hf_ctx *ctx, bool tA, int64_t m, int64_t n, int64_t k, float alpha, const __nv_bfloat16 *A,
              int64_t lda, const __nv_bfloat16 *B, int64_t ldb, float beta, float *C, int64_t ldc,
              cudaStream_t st = nullptr, int batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0);

// frees the workspace kept for stream s (call before destroying s, after synchronising it)
void lt_release_stream(hf_ctx *ctx, cudaStream_t s);

}  // namespace hf
