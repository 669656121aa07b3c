/*
 * hf.h -- C ABI of the B200 hybrid mixed-precision factorization hot path
 * (Suzuki, "A Hybrid Factorization Algorithm for Sparse Matrix with Mixed
 * Precision Arithmetic", arXiv 2208.01907).  Implemented by libhf.so
 * (paper_2208_01907_b200/csrc, hand-written CUDA for sm_100a).
 *
 * Citations: P:n = line n of the paper's LaTeX source.  [Rn] are
 * the readings of silent/ambiguous passages listed in DESIGN.md section 3.
 *
 * Conventions (all entry points)
 *  - Pointers are DEVICE pointers unless the name ends in _host.
 *  - Matrices are column-major FP64 with leading dimension ld >= L.  K must be
 *    exactly symmetric; only its lower triangle (row >= col) is read where
 *    stated.  Index arrays are int64, 0-based, ORIGINAL indices of K.
 *  - Every call is ordered on the context's CUDA stream.  Calls that return
 *    *_host values synchronise that stream before returning.
 *  - Functions return an hf_status and never abort/exit.  On error the
 *    outputs are unspecified, handles can still be destroyed, and
 *    hf_last_error(ctx) describes the error.
 *  - Ownership: the caller owns K, q, b, x and every *_host buffer.  The
 *    library owns the memory behind hf_lowfactor / hf_hybrid handles and frees
 *    it in the *_destroy calls.  An hf_hybrid BORROWS the caller's K (used
 *    again by hf_solve): K must stay valid and unmodified until
 *    hf_hybrid_destroy.
 */
#ifndef HF_H
#define HF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hf_ctx hf_ctx;             /* device, stream, optional NCCL comm, counters */
typedef struct hf_lowfactor hf_lowfactor; /* Pi, Lambda_1/2, FP32 factor L, D (device)   */
typedef struct hf_hybrid hf_hybrid;       /* X12, S22, hard factors, borrowed K          */

typedef enum {
    HF_OK = 0,
    HF_ERR_INVALID_ARG = 1,    /* bad size/pointer, tau outside (0,1), NaN/Inf found   */
    HF_ERR_CUDA = 2,           /* CUDA runtime error (message in hf_last_error)        */
    HF_ERR_NCCL = 3,           /* NCCL error (multi-GPU contexts)                      */
    HF_ERR_OOM = 4,            /* device allocation failed                             */
    HF_ERR_NOT_CONVERGED = 5,  /* block GCR reached max_iter (info filled)             */
    HF_ERR_BREAKDOWN = 6,      /* Gram matrix M_n not positive definite [R11]          */
    HF_ERR_STATE = 7           /* handle in the wrong state (e.g. solve before hard)   */
} hf_status;

/* ---------------------------------------------------------------- context */
/* device: CUDA ordinal; cuda_stream: a cudaStream_t (NULL = legacy default). */
hf_status hf_create(int device, void *cuda_stream, hf_ctx **out);
/* Multi-GPU context (sec. 8(e) of SURVEY.md): nccl_unique_id128 points to the
 * 128-byte ncclUniqueId produced by hf_nccl_unique_id on rank 0 and broadcast
 * by the caller (torch.distributed).  rank in [0, nranks). */
hf_status hf_create_dist(int device, void *cuda_stream, const void *nccl_unique_id128,
                         int rank, int nranks, hf_ctx **out);
hf_status hf_nccl_unique_id(void *id128_host);
/* Multi-GPU stage 2: on a context of nranks > 1, hf_schur_gcr
 * gives rank r the contiguous column slice [c0, c1) of K12 (c0 = r n2 / G,
 * c1 = (r+1) n2 / G), runs block GCR on it, forms S22[:, c0:c1] and broadcasts
 * the S22 and X12 slices from their owners (one NCCL group); every rank ends
 * with the full S22 and X12 (block-GCR statistics max-reduced).  Stage 1, the
 * hard factorization and hf_solve are replicated (deterministic kernels:
 * identical on every rank).  Pure host function, needs no device. */
hf_status hf_shard_cols(int64_t n2, int nranks, int rank, int64_t *c0_host, int64_t *c1_host);
/* Multi-GPU stage 1 (P:64-67, P:72-75 distributed): on a context of
 * nranks > 1, hf_factor_lowprec distributes the FP32 factorization in a 1D
 * block-cyclic layout of the LOWER triangle: rank r owns the original indices
 * j with (j / 128) % nranks == r and stores, for each, the entries v_IJ of the
 * active I at or below it (every pair on exactly one rank: the trailing-update
 * work over the ranks equals one GPU's).  The pivot chain's rows are split the
 * same way; per pivot every chain CTA stores its tagged (|d|, position) key into
 * every rank's slot array over NVLink (the max-reduction that picks the pivot),
 * the pivot column's entries below the pivot are read from its owner and the
 * pivot row's in-panel values from the winner's mailbox; after each panel every
 * rank gathers the panel from the owners and updates its own columns.  Peer
 * buffers are CUDA-IPC mappings (handles all-gathered over NCCL), barriers are
 * device-side; a peer that stops answering for 60 s makes the call fail with
 * HF_ERR_NCCL ("peer did not answer") instead of hanging.  Pi, D and L
 * are bitwise those of one GPU on every rank.
 * hf_set_stage1_partitions(ctx, G > 0) runs the same distributed algorithm with
 * all G ranks on this GPU (one cooperative chain launch over every rank's CTAs:
 * single-process emulation, tests and the time model); 0 = the single-GPU path. */
hf_status hf_set_stage1_partitions(hf_ctx *ctx, int nparts);
/* The indices (original, increasing) rank `part` of `nparts` owns in that
 * factorization: j with (j / 128) % nparts == part.  Host only; the
 * list is written if cols_host is not NULL (room for L entries). */
hf_status hf_stage1_partition(int64_t L, int nparts, int part, int64_t *ncols_host, int64_t *cols_host);
/* Single-GPU emulation of one rank of that sharding (tests): with nranks > 0,
 * hf_schur_gcr computes only rank's slice of S22 / X12 and leaves the other
 * columns zero (no collective); nranks = 0 switches the emulation off. */
hf_status hf_set_virtual_rank(hf_ctx *ctx, int rank, int nranks);
hf_status hf_destroy(hf_ctx *ctx);
/* Last error message of ctx (never NULL; "" when none).  ctx may be NULL for
 * errors raised before a context existed. */
const char *hf_last_error(const hf_ctx *ctx);

/* Instrumentation: number of kernels this context launched so far, and the
 * summed device time of one kernel class measured with CUDA events on the
 * context stream while profiling is enabled.  class: "trailing", "chain",
 * "dgemm", "trsm" (the triangular-solve applications), "trsm_setup" (their
 * operator setup), "gram", "scale", "hard", "other".  Every entry point runs on
 * the context's device and restores the caller's current device. */
hf_status hf_set_profiling(hf_ctx *ctx, int enable);
hf_status hf_kernel_stats(hf_ctx *ctx, const char *kernel_class, double *ms_host,
                          int64_t *launches_host);
hf_status hf_launch_count(const hf_ctx *ctx, int64_t *launches_host);
/* The ALGORITHMIC work of one kernel class summed over the launches made while
 * profiling was enabled (what the method must compute: e.g. one FMA
 * per lower-triangle entry per pivot for "trailing", 2 N^2 n per application for
 * "trsm", 2 M N K per product for "dgemm"); 0 for classes that do not report it.
 * Cumulative like hf_kernel_stats. */
hf_status hf_kernel_work(hf_ctx *ctx, const char *kernel_class, double *flops_host, double *bytes_host);
/* Instrumentation (the pivot chain's roofline): microseconds per step of the chain's
 * grid-wide exchange ALONE -- nctas cooperative CTAs of nthreads threads, per step a
 * block max-reduction of a key, one tag-validated slot store per CTA and a poll of every
 * slot -- with no column fetch and no arithmetic.  The floor under the chain's per-pivot
 * time for that geometry. */
hf_status hf_chain_exchange_floor(hf_ctx *ctx, int nctas, int nthreads, int steps, double *us_per_step_host);
/* Device workspaces and handle buffers come from a per-(device, stream) cache
 * that reuses freed blocks in stream order (no memory is re-mapped by a
 * repeated factorization); this synchronises the device and returns every
 * cached (free) block of `device` to the driver.  Live handles are untouched. */
hf_status hf_trim_cache(int device);

/* ------------------------------------------------- a1: scaling, P:40 [R1] */
/* In place: q_i = 1/sqrt|K_ii| (1 if K_ii == 0); K_ij = (q_i K_ij) q_j for
 * i > j from the LOWER triangle, mirrored to the upper triangle; K_ii set to
 * exactly +1, -1 or 0 by the sign of the input diagonal.  K: L x L (ld),
 * q: FP64[L].  Returns HF_ERR_INVALID_ARG if K holds NaN/Inf on or below the
 * diagonal. */
hf_status hf_scale(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q);
/* The same scaling from a HOST matrix: the lower triangle (i >= j, the only part
 * hf_scale reads) of Kbar_host (L x L, column-major, ldh >= L; pinned memory makes
 * the copy asynchronous, pageable memory works) is copied into the device K (ld)
 * in column panels of 256 on the context stream, then scaled in place as above
 * (the upper triangle of K is written from the lower one; that of Kbar_host is
 * never read).  *h2d_bytes_host (if not NULL) = bytes moved host -> device.
 * Synchronises the stream.  Same errors as hf_scale. */
hf_status hf_scale_host(hf_ctx *ctx, int64_t L, const double *Kbar_host, int64_t ldh, double *K, int64_t ld,
                        double *q, int64_t *h2d_bytes_host);
/* Asynchronous form of hf_scale_host's copy, for pipelining the next matrix's
 * transfer behind the current factorization: the same lower-triangle panels of
 * Kbar_host into K, issued on the context's own upload stream (created on first
 * use) and returning at once (pinned Kbar_host: the host must keep it unchanged
 * until the copy is done; pageable memory makes the call synchronous).  The copy
 * is NOT ordered after work already queued on the context stream: the caller
 * must not upload into a K that queued work still reads.  The next hf_scale /
 * hf_scale_host on this context orders the context stream after every upload
 * issued before it.  *h2d_bytes_host (if not NULL) = bytes the copy moves.  The
 * paper's scaling step then runs by hf_scale(K). */
hf_status hf_upload_lower(hf_ctx *ctx, int64_t L, const double *Kbar_host, int64_t ldh, double *K, int64_t ld,
                          int64_t *h2d_bytes_host);
/* NEXT-3: the same scaling for a GENERAL matrix (every entry read and written:
 * K_ij = (q_i Kbar_ij) q_j, K_ii = sign Kbar_ii).  Same errors as hf_scale. */
hf_status hf_scale_full(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q);

/* ---------------------------- a2-a3: lower-precision factor, P:64-85 [R2-R10] */
typedef struct {
    double tau;       /* threshold of P:73, in (0,1)                                  */
    int64_t n_extra;  /* P:82 enlargement: move the last n_extra pivots to Lambda_2   */
    int64_t n_min;    /* postponement floor [R5]: |Lambda_2| >= n_min                 */
    int32_t nb;       /* panel width (0 = automatic)                                  */
    int32_t prec;     /* 0 or 32: FP32 factor (Alg. 1's lower precision for the       */
                      /* (float, double) pair); 64: FP64 factor, the lower precision  */
                      /* of the paper's (double, double-double) pair (NEXT-1)  */
    int32_t nonsym;   /* NEXT-3: 1 = K is a GENERAL matrix (every entry read):       */
                      /* FP32 LDU with the same pivoting / postponing, rule [R19]     */
                      /* (d = v_PP, l_I = c_I / d, r_J = v_PJ, v_IJ <- fmaf(-l_I,     */
                      /* r_J, v_IJ)); prec 32, one GPU.  0 = symmetric LDL^T.        */
} hf_lowprec_opts;

/* FP32 LDL^T of the scaled K (lower triangle read) with symmetric max-|diag|
 * pivoting (ties -> smallest original index), the strict ratio test
 * |d_k| < tau |d_{k-1}| of P:73 evaluated in FP64, and the role-symmetric
 * update v_IJ <- fmaf(-sigma s_I, s_J, v_IJ) applied once per pivot in
 * increasing order [R8], so Pi, D and L are bit-identical to the oracle.
 * Outputs N = |Lambda_1|, n2 = |Lambda_2| and the pure tau-rule count.
 * A first pivot of exactly 0 is legal and postpones everything (N = 0). */
hf_status hf_factor_lowprec(hf_ctx *ctx, int64_t L, const double *K, int64_t ld,
                            const hf_lowprec_opts *opts, hf_lowfactor **out,
                            int64_t *N_host, int64_t *n2_host, int64_t *n2_tau_only_host);
/* perm_host[L]: Pi = [Lambda_1 in pivot order, Lambda_2 ascending] [R10];
 * D_host[N]: FP32 pivots; Lfac: DEVICE N x N column-major (ldl >= N) unit
 * lower factor in pivot order (U = L^T), zeros above the diagonal.  Any output
 * pointer may be NULL to skip it. */
hf_status hf_lowfactor_export(hf_ctx *ctx, const hf_lowfactor *lf, int64_t *perm_host,
                              float *D_host, float *Lfac, int64_t ldl);
/* prec 64 factors: perm_host[L], D_host[N] (double), Lfac: DEVICE N x N double. */
hf_status hf_lowfactor_export64(hf_ctx *ctx, const hf_lowfactor *lf, int64_t *perm_host,
                                double *D_host, double *Lfac, int64_t ldl);
hf_status hf_lowfactor_destroy(hf_lowfactor *lf);
/* ----------- NEXT-4: multi-block threshold postponing, sec. 2.2 */
/* Nested-dissection blocks of the symmetric sparsity pattern of K (DEVICE,
 * column-major, only K_ij != 0 is used): an m-level bisection tree (P:70,
 * 2^m - 1 blocks when every level splits), recursive level-structure
 * bisection (rule in nd.cu), blocks in post-order (children before their
 * separator).  blk_host[L] = block of every index, *nblk_host = count.
 * Synchronises. */
hf_status hf_nd_blocks(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, int32_t levels, int32_t min_size,
                       int32_t *blk_host, int32_t *nblk_host);
/* Stage 1 with multi-block postponing: blocks 0..nblk-1 in order, the pivots of
 * block j chosen among its remaining indices (rule [R3]), the ratio test [R4]
 * against the previously accepted pivot (across blocks, [R21]; the very first
 * pivot only against 0), the rest of a stopped block postponed to Lambda_0; then a final
 * pass over every remaining index with the same rules, whose stop is
 * N_tau; floor and enlargement (opts n_min, n_extra; "usually n = 4") as
 * hf_factor_lowprec.  nblk = 0: exactly hf_factor_lowprec.  FP32 symmetric,
 * one GPU.  blk_host: HOST int32[L], values in [0, nblk). */
hf_status hf_factor_lowprec_blocks(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts *opts,
                                   const int32_t *blk_host, int32_t nblk, hf_lowfactor **out, int64_t *N_host,
                                   int64_t *n2_host, int64_t *n2_tau_only_host);

/* NEXT-3: the unit upper factor U of a nonsymmetric LDU as Ufac = U^T (N x N,
 * DEVICE, ldu >= N, pivot order): Ufac[i + k ldu] = U_ki.  HF_ERR_STATE on a
 * symmetric factor. */
hf_status hf_lowfactor_export_u(hf_ctx *ctx, const hf_lowfactor *lf, float *Ufac, int64_t ldu);

/* --------------------------- a5: the preconditioner Q^{-1}, P:231-242 [R12] */
/* W = lift( L^{-T} D^{-1} L^{-1} truncate(R) ) in FP32 for the Lambda_1 rows
 * ("find e^ satisfying Q^ e^ = r^ in lower precision ... up-converting"),
 * 0 on the Lambda_2 rows.  R, W: DEVICE L x ncol column-major FP64 in ORIGINAL
 * row order (ldr, ldw >= L); only the Lambda_1 rows of R are read.  The same
 * kernels serve every preconditioner application inside hf_schur_gcr and
 * hf_solve (SPEC precond_solve).  Synchronises. */
hf_status hf_precond_apply(hf_ctx *ctx, const hf_lowfactor *lf, int64_t ncol, const double *R,
                           int64_t ldr, double *W, int64_t ldw);

/* Minv = M^{-1} for the SPD Gram matrix M_n = q_n^T q_n of Algorithm 5 (P:322-330:
 * alpha_n = M_n^{-1} q_n^T r_n, beta_{n,m} = -M_m^{-1} q_m^T z), the step hf_schur_gcr runs
 * once per iteration.  M: DEVICE n x n column-major FP64 (ldm >= n, only read); Minv:
 * DEVICE n x n (ld n).  Gauss-Jordan without pivoting (16-CTA cluster, blocked by 16 for
 * n <= 448); *breakdown_host = 1 when a pivot is not positive (M not numerically SPD,
 * [R11]; Minv is then not meaningful), else 0.  Synchronises. */
hf_status hf_gram_inverse(hf_ctx *ctx, int64_t n, const double *M, int64_t ldm, double *Minv,
                          int32_t *breakdown_host);

/* ------------- NEXT-2: IR / GCR / block GCR comparison (Fig. 2) */
/* K11 X = B with the FP32 preconditioner of lf: method 0 = Algorithm 3 (mixed-
 * precision iterative refinement), 1 = Algorithm 4 (GCR, P:277-295,
 * one column at a time), 2 = Algorithm 5 (block GCR).  B, X: DEVICE
 * L x ncol column-major (ld L), original row order (Lambda_2 rows of B ignored,
 * of X set to 0).  Stops when every column's ||r||_2/||b||_2 <= tol or after
 * max_iter iterations (HF_ERR_NOT_CONVERGED); iters_host = iterations (max over
 * columns for method 1), hist_host[0..hist_len) = max relative residual after
 * iteration 0, 1, ... (-1 past the end).  Synchronises. */
hf_status hf_krylov_solve(hf_ctx *ctx, const double *K, int64_t ld, const hf_lowfactor *lf, int method,
                          int64_t ncol, const double *B, double *X, double tol, int32_t max_iter,
                          int32_t *iters_host, double *hist_host, int32_t hist_len);

/* The block mat-vec of Alg. 5 alone (P:507's "SpMM in higher
 * precision"): Z = K W for a SYMMETRIC K (L x L, ld; the Ozaki path reads row m
 * as column m), W: L x n (ldw), Z: L x n (ldz), all DEVICE FP64.  matvec 1 = FP64
 * DMMA, 2 = FP64 emulated on the int8 tensor cores with `slices` slices (0 = 8;
 * see hf_gcr_opts), 3 = the residue form.  Synchronises. */
hf_status hf_matvec(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const double *W, int64_t ldw, int64_t n,
                    double *Z, int64_t ldz, int32_t matvec, int32_t slices);

/* ------------------------ a4-a6: block GCR + Schur */
typedef struct {
    double tol;        /* per-column recursive ||r||_2/||b||_2 target [R13] (1e-14) */
    int32_t max_iter;  /* iteration cap (100)                                       */
    /* the FP64 block mat-vec K11 W (P:507's "SpMM in higher precision"):
     *   1: FP64 DMMA tensor-core GEMM;
     *   3: FP64 emulated on the int8 tensor cores in residue (Chinese remainder)
     *      form (ozaki2.cu): K and W scaled by powers of two to 53-bit integers,
     *      16 pairwise coprime moduli <= 256, one exact int8 GEMM per modulus,
     *      the exact integer product rebuilt by Garner's mixed radix and
     *      rounded in FP64 -- error below Lk 2^(e_m + f_c - 52) + 16 ulps;
     *      16 int8 copies of K of memory, Lk <= 130000;
     *   2: FP64 emulated on the int8 tensor cores (Ozaki scheme, ozaki.cu): K's
     *      rows and W's columns split into `slices` exact 7-bit fixed-point
     *      slices under a power-of-two scale, every slice product an exact
     *      int8 GEMM, the products with p + q <= slices + 1 summed exactly per
     *      group and the groups in FP64 -- error below
     *      ~2^(-7 slices) Lk max|K_m.| max|W_.c| per entry (8 slices: 2^-56,
     *      against FP64's Lk 2^-53 |K||W|);
     *   0: automatic: for blocks of >= 32 columns 3, else 2, else 1, as device
     *      memory allows (the K copies and the block GCR's growth); else 1.
     * The environment variable HF_MATVEC=dmma|ozaki|ozaki2 overrides 0.      */
    int32_t matvec;
    int32_t slices;    /* matvec 2: slices per operand, 2..9 (0 = 8)               */
} hf_gcr_opts;
typedef struct {
    int32_t iters;                 /* completed block-GCR iterations          */
    double max_rel_res_recursive;  /* max over columns at exit (recursive r)  */
    double max_rel_res_true;       /* max over columns of ||K12 - K11 X||/||K12|| */
    int32_t matvec;                /* the mat-vec form that ran (hf_gcr_opts.matvec 1..3) */
} hf_gcr_info;

/* Alg. 1 steps 2-4: K11 X12 = K12 by right-preconditioned block GCR in FP64
 * with Q^{-1} = FP32 (L D L^T)^{-1} (casts fused), then S22 = K22 - K21 X12 in
 * FP64.  K: the SAME scaled full symmetric matrix given to hf_factor_lowprec
 * (borrowed by the returned handle).  S22_host_or_null: n2 x n2 column-major,
 * rows/cols in Lambda_2 ascending order.  Returns HF_ERR_NOT_CONVERGED or
 * HF_ERR_BREAKDOWN with *out still valid and info filled. */
hf_status hf_schur_gcr(hf_ctx *ctx, const double *K, int64_t ld, const hf_lowfactor *lf,
                       const hf_gcr_opts *opts, hf_hybrid **out, double *S22_host_or_null,
                       hf_gcr_info *info_host);
/* X: DEVICE N x n2 (ldx >= N, rows in Pi_1 order); S22: DEVICE n2 x n2 (lds). */
hf_status hf_hybrid_export(hf_ctx *ctx, const hf_hybrid *hy, double *X, int64_t ldx,
                           double *S22, int64_t lds);

/* ------------------- NEXT-1: the (double, double-double) pair */
/* Alg. 1 steps 2-4 with the higher precision raised to double-double (Table 1's
 * (double, quadruple) row): block GCR (Alg. 5) with every N x n2
 * block as (hi, lo) double pairs, K11 W formed with error-free products and
 * double-double sums, Gram inverses and updates in double-double, and
 * S22 = K22 - K21 X12 in double-double.  lf must be the FP64 factorization
 * (hf_factor_lowprec with prec = 64): its FP64 L D L^T is the lower-precision
 * preconditioner, applied to the residual rounded to double.  opts: tol is
 * the per-column recursive ||r||/||b|| target (default 1e-28).  S22hi/lo_host:
 * n2 x n2 column-major (S22 = hi + lo exactly).  The returned hybrid is a
 * double-double one: hf_factor_hard factors S22 in double-double (same rule
 * as below), hf_hard_export works, hf_solve_dd solves (hf_solve returns
 * HF_ERR_STATE).  One rank
 * only (HF_ERR_INVALID_ARG on a distributed or virtual-rank context). */
hf_status hf_schur_gcr_dd(hf_ctx *ctx, const double *K, int64_t ld, const hf_lowfactor *lf,
                          const hf_gcr_opts *opts, hf_hybrid **out, double *S22hi_host_or_null,
                          double *S22lo_host_or_null, hf_gcr_info *info_host);
/* X (L x n2, ORIGINAL row order, zero on Lambda_2 rows) and S22 of a
 * double-double hybrid as hi / lo parts; DEVICE pointers (any may be NULL);
 * HF_ERR_STATE on a double hybrid. */
hf_status hf_hybrid_export_dd(hf_ctx *ctx, const hf_hybrid *hy, double *Xhi, double *Xlo, int64_t ldx,
                              double *S22hi, double *S22lo, int64_t lds);
/* Alg. 2 in double-double on a double-double hybrid after
 * hf_factor_hard: b DEVICE FP64[L] (scaled system, original order), x = xhi + xlo
 * DEVICE FP64[L] each; block GCR tolerance 1e-28; kernel coordinates 0 [R16].
 * HF_ERR_STATE on a double hybrid or before hf_factor_hard. */
hf_status hf_solve_dd(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *xhi, double *xlo,
                      hf_gcr_info *info_host);

/* ---------------------------- a7: hard factorization, P:192, P:84 [R15] */
/* FP64 Bunch-Parlett (complete pivoting, alpha = (1+sqrt17)/8) LDL^T of
 * (S22 + S22^T)/2 with 1x1/2x2 pivots; stops when max|S_ij| of the trailing
 * block <= eps_ker * min_k |D_k|; kernel_dim = size of the block left.
 * n2 = 0 is a no-op (kernel_dim = 0). */
hf_status hf_factor_hard(hf_ctx *ctx, hf_hybrid *hy, double eps_ker, int64_t *kernel_dim_host);
/* perm2_host[n2]: pivot order as Lambda_2 positions; blocks_host[n2]: pivot
 * sizes (1 or 2) in order, the rest 0; rank_host: n2 - kernel_dim. */
hf_status hf_hard_export(hf_ctx *ctx, const hf_hybrid *hy, int64_t *perm2_host,
                         int32_t *blocks_host, int64_t *rank_host);

/* ------------------------------------------ a8: hybrid solve, Alg. 2 [R16] */
/* Solves the SCALED system K x = b (b, x: device FP64[L], original order):
 * y1 = block GCR on K11 with one column, y2 = b2 - K21 y1, x2 = S22^+ y2
 * (kernel coordinates 0), x1 = y1 - X12 x2.  Requires hf_factor_hard. */
hf_status hf_solve(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *x,
                   hf_gcr_info *info_host);
hf_status hf_hybrid_destroy(hf_hybrid *hy);

#ifdef __cplusplus
}
#endif
#endif /* HF_H */
