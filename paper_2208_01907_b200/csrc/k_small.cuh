// k_small.cuh -- launchers of k_small.cu
#pragma once
#include "hf_internal.cuh"

namespace hf {
void gather_K12(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const int64_t *lam2, int64_t n2,
                const uint8_t *mask1, double *B);
void gather_K22(hf_ctx *ctx, int64_t n2, const double *K, int64_t ld, const int64_t *lam2, double *K22);
// NEXT-3 (nonsymmetric): K21^T gather, LU with complete pivoting of S22 and its solve
void gather_K21T(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const int64_t *lam2, int64_t n2,
                 const uint8_t *mask1, double *B);
void hard_lu(hf_ctx *ctx, int64_t n, const double *S, double thr, double *A, int32_t *prow, int32_t *pcol,
             int64_t *rank_dev);
void hard_lu_solve(hf_ctx *ctx, int64_t n, int64_t r, const double *A, const int32_t *prow, const int32_t *pcol,
                   const double *y, double *x, double *z);
void mask_from_pos(hf_ctx *ctx, int64_t L, const int32_t *pos1, uint8_t *m);
void colnorm2(hf_ctx *ctx, int64_t M, int64_t ncol, const double *X, int64_t ldx, double *out);
void maxres(hf_ctx *ctx, int64_t n, const double *rn2, const double *bn2, double *out);
void spd_inverse(hf_ctx *ctx, int64_t n, const double *M, int64_t ldm, double *Minv, DBuf<double> &wk,
                 DBuf<double> &dg, int *status);
void hard_factor(hf_ctx *ctx, int64_t n, const double *S, double thr, double *A, double *Lh, double *Dh,
                 int32_t *lab, int32_t *blocks, int64_t *rank_dev);
void hard_solve(hf_ctx *ctx, int64_t n, int64_t r, const double *Lh, const double *Dh, const int32_t *lab,
                const int32_t *blocks, const double *y, double *x, double *z);
void scatter_rows(hf_ctx *ctx, int64_t n, const int64_t *idx, const double *src, double *dst);
void gather_rows(hf_ctx *ctx, int64_t n, const int64_t *idx, const double *src, double *dst);
void mask_vec(hf_ctx *ctx, int64_t L, const uint8_t *m, const double *src, double *dst);
void axpy_cols(hf_ctx *ctx, int64_t L, int64_t n, double alpha, const double *X, int64_t ldx, double *Y,
               int64_t ldy);
void gather_block_rows(hf_ctx *ctx, int64_t n, int64_t ncol, const int64_t *perm, const double *X, int64_t ldx,
                       double *out, int64_t ldo);
}  // namespace hf
