// k_dgemm.cuh -- FP64 DMMA GEMM interface (see k_dgemm.cu).
#pragma once
#include "hf_internal.cuh"

namespace hf {

struct DgemmArgs {
    int64_t M, N, K;
    double alpha;
    const double *A;
    int64_t lda;
    const double *B;
    int64_t ldb;
    double beta;
    double *C;
    int64_t ldc;
    const uint8_t *rowmask;  // optional: rows with 0 get beta*C only
    double *W;               // split-K partials
};

// C = beta*C + alpha * rowmask o (op(A) B); splits <= 0 = automatic.
void dgemm(hf_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
           int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
           const uint8_t *rowmask, DBuf<double> *work, int splits = 0);

// FP32 preconditioner Q^{-1} (k_trsm.cu); struct Precond is in hf_internal.cuh
void precond_setup(hf_ctx *ctx, Precond &p, const hf_lowfactor *lf);
// W (L x ncol, original order, ldw) = Q^{-1} R (R: L x ncol, original order, ldr);
// rows of Lambda_2 in W are set to 0.
void precond_apply(hf_ctx *ctx, Precond &p, int64_t ncol, const double *R, int64_t ldr, double *W,
                   int64_t ldw);

}  // namespace hf
