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

// Two problems of the same shape (no row mask) in one launch: C_b = beta_b C_b + alpha_b op(A_b) B_b
// (better wave fill for the small block updates of Alg. 5); separate split-K work buffers.
void dgemm2(hf_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha0, const double *A0,
            int64_t lda0, const double *B0, int64_t ldb0, double beta0, double *C0, int64_t ldc0, double alpha1,
            const double *A1, int64_t lda1, const double *B1, int64_t ldb1, double beta1, double *C1, int64_t ldc1,
            DBuf<double> *work0, DBuf<double> *work1, int splits = 0);

// C = beta*C + alpha * rowmask o (op(A) B); splits <= 0 = automatic.
void dgemm(hf_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
           int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
           const uint8_t *rowmask, DBuf<double> *work, int splits = 0);

// the blocked tensor-core form of the FP32 preconditioner (k_trsm_blk.cu; HF_PRECOND=dataflow
// selects the k_trsm.cu dataflow kernels instead)
bool precond_blocked_enabled();
void precond_blk_setup(hf_ctx *ctx, PrecondBlk &p, int64_t N, int64_t L, const float *Lfac, const float *D,
                       const int64_t *perm, const int32_t *pos1);
void precond_blk_apply(hf_ctx *ctx, PrecondBlk &p, int64_t ncol, const double *R, int64_t ldr, double *W,
                       int64_t ldw);

// FP32 preconditioner Q^{-1} (k_trsm.cu); struct Precond is in hf_internal.cuh
void precond_setup(hf_ctx *ctx, Precond &p, const hf_lowfactor *lf);
// W (L x ncol, original order, ldw) = Q^{-1} R (R: L x ncol, original order, ldr);
// rows of Lambda_2 in W are set to 0.
void precond_apply(hf_ctx *ctx, Precond &p, int64_t ncol, const double *R, int64_t ldr, double *W,
                   int64_t ldw);

}  // namespace hf
