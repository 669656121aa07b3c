/*
 * oracle/lowprec.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU implementation of the first part of the
 * hybrid factorization of Suzuki (arXiv 2208.01907).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code with the CUDA path
 * (paper_2208_01907_b200/csrc) and includes no header of it.
 *
 * Citations: P:n = PAPER.md line n (LaTeX source of the paper).
 * Readings of silent/ambiguous passages are listed in DESIGN.md section 3 and
 * referred to here as [Rn].
 *
 * Functions
 *   oracle_scale          P:40 (sec. 2 opening): K = Q Kbar Q, diag(K) in {-1,0,1}.
 *   oracle_factor_f32     P:64-67 (sec. 2.1) symmetric max-|diag| pivoting with
 *                         rank-1 Schur update, P:72-75 (sec. 2.2) threshold
 *                         postponing, P:82-83 enlargement, in FP32 (the lower
 *                         precision of Alg. 1 step 1).
 *   oracle_factor_f64     the same algorithm in FP64 (used by the planted-count
 *                         pin of the tests and by the (double, double-double)
 *                         pair of sec. 4.3).
 *
 * max_steps > 0 stops after that many pivots (a bounded sample for bench.py's
 * CPU baseline, and the bitwise PREFIX comparison at C4 in the tests; results
 * of such a run are not a factorization).  Output-only options (round 2,
 * no arithmetic change): ncol >= 0 writes only the first ncol columns of Lfac
 * (an L x ncol array; -1: all L), and a bounded run writes every row of them
 * in its own position order, which pos_orig (nullable, [L]) receives as the
 * original index of each position.
 *
 * Arithmetic is IEEE round-to-nearest, no contraction (compiled with
 * -ffp-contract=off); every FMA is an explicit fmaf/fma call.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* "scaled so that diagonal entries take one of -1, 0 and 1, ...        */
/* [Q]_ii = 1/sqrt([Kbar]_ii) when [Kbar]_ii != 0, otherwise [Q]_ii = 1 ...   */
/* Q Kbar Q = K".  Only the lower triangle (i >= j) of Kbar is read [R1].     */
/* Kbar, K: column-major L x L with leading dimension ld (may alias).         */
/* K is written as a full symmetric matrix.  Returns 0.                      */
/* ------------------------------------------------------------------------- */
int oracle_scale(int64_t L, const double *Kbar, int64_t ld, double *K, double *q)
{
    for (int64_t i = 0; i < L; ++i) {
        double d = Kbar[i + i * ld];
        q[i] = (d != 0.0) ? 1.0 / sqrt(fabs(d)) : 1.0;
    }
    for (int64_t j = 0; j < L; ++j) {
        for (int64_t i = j + 1; i < L; ++i) {
            double v = (q[i] * Kbar[i + j * ld]) * q[j];
            K[i + j * ld] = v;
            K[j + i * ld] = v;
        }
    }
    for (int64_t i = 0; i < L; ++i) {
        double d = Kbar[i + i * ld];
        K[i + i * ld] = (d > 0.0) ? 1.0 : ((d < 0.0) ? -1.0 : 0.0);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Stage 1 (Alg. 1 step 1): LDL^T with symmetric pivoting and         */
/* threshold postponing.  Written once as a macro body for the two scalar    */
/* types so the FP64 variant is the same algorithm letter for letter.        */
/*                                                                           */
/* Storage: A is a full L x L column-major array of which only the lower     */
/* triangle (row >= col) in POSITION space is used.  The paper's step         */
/* (P:65-67): find k0 = argmax |diag| of the trailing block, swap rows and   */
/* columns k and k0 (physically), then the rank-1 update                      */
/*   S'_22 = K~'_22 - [K~_22]_{down 1} d^{-1} [K~_22]_{1 right}.              */
/* The update is evaluated in the role-symmetric form [R7, R8]               */
/*   s_i = c_i / sqrt|d|, sigma = sign d,  v_ij <- fma(-sigma*s_i, s_j, v_ij) */
/* which is the same rank-1 update (c_i c_j / d = sigma s_i s_j) with one    */
/* correctly rounded FMA per pivot per entry.                                */
/*                                                                           */
/* Outputs:                                                                  */
/*   perm[L]   : perm[k] = original index of the k-th pivot for k < N,       */
/*               then Lambda_2 in ascending original index [R10]             */
/*   Dk[L]     : pivot values d_k for k < N_tau (first N are D)              */
/*   Lfac      : L x L column-major (ld = L); column k < N holds the unit-   */
/*               lower factor column in pivot (position) order:              */
/*               Lfac[i + k L] = c_i / d_k for k < i < N, 1 on the diagonal,  */
/*               0 above.  Only the leading N x N block is meaningful.       */
/*   out[0]=N, out[1]=N_tau (pure tau-rule count, no floor, no enlargement)  */
/* Returns 0, or -1 on bad arguments / allocation failure.                   */
/* ------------------------------------------------------------------------- */
#define ORACLE_FACTOR_BODY(T, FMA, SQRT, FABS)                                  \
    if (L < 0 || !(tau > 0.0 && tau < 1.0) || n_min < 0 || n_extra < 0)       \
        return -1;                                                            \
    T *A = (T *)malloc((size_t)(L > 0 ? L : 1) * (size_t)(L > 0 ? L : 1) * sizeof(T)); \
    T *s = (T *)malloc((size_t)(L > 0 ? L : 1) * sizeof(T));                  \
    int64_t *orig = (int64_t *)malloc((size_t)(L > 0 ? L : 1) * sizeof(int64_t)); \
    if (!A || !s || !orig) { free(A); free(s); free(orig); return -1; }       \
    /* [R2] lower-precision start values, rounded once from the FP64 K */     \
    for (int64_t j = 0; j < L; ++j)                                           \
        for (int64_t i = j; i < L; ++i)                                       \
            A[i + j * L] = (T)K[i + j * ld];                                  \
    for (int64_t p = 0; p < L; ++p) orig[p] = p;                              \
    int64_t Ntau = L;                                                         \
    const int64_t kmax = (max_steps > 0 && max_steps < L) ? max_steps : L;   \
    for (int64_t k = 0; k < kmax; ++k) {                                      \
        /* [R3] P:65 max |diag|, ties -> smallest original index */           \
        int64_t best = k;                                                     \
        for (int64_t p = k + 1; p < L; ++p) {                                 \
            T a = FABS(A[p + p * L]), b = FABS(A[best + best * L]);           \
            if (a > b || (a == b && orig[p] < orig[best])) best = p;          \
        }                                                                     \
        T d = A[best + best * L];                                             \
        /* [R4] P:73 |K_{i+1,i+1}/K_{ii}| < tau -> stop (ratio in FP64) */    \
        if (k == 0 && d == (T)0) { Ntau = 0; break; }                         \
        if (k > 0 && fabs((double)d) < tau * fabs((double)Dk[k - 1])) {      \
            Ntau = k; break;                                                  \
        }                                                                     \
        /* P:66 "rows and columns ... k+1 and k0 are exchanged" */            \
        if (best != k) {                                                      \
            int64_t p = best; T t;                                            \
            for (int64_t j = 0; j < k; ++j) {          /* rows of L part */   \
                t = A[k + j * L]; A[k + j * L] = A[p + j * L]; A[p + j * L] = t; \
            }                                                                 \
            t = A[k + k * L]; A[k + k * L] = A[p + p * L]; A[p + p * L] = t;  \
            for (int64_t i = k + 1; i < p; ++i) {      /* col k <-> row p */  \
                t = A[i + k * L]; A[i + k * L] = A[p + i * L]; A[p + i * L] = t; \
            }                                                                 \
            for (int64_t i = p + 1; i < L; ++i) {      /* below p */          \
                t = A[i + k * L]; A[i + k * L] = A[i + p * L]; A[i + p * L] = t; \
            }                                                                 \
            int64_t o = orig[k]; orig[k] = orig[p]; orig[p] = o;              \
        }                                                                     \
        Dk[k] = d;                                                            \
        /* [R7] r = sqrt|d|, sigma = sign d, s_i = c_i / r (IEEE division) */ \
        T r = SQRT(FABS(d));                                                  \
        T sg = (d > (T)0) ? (T)1 : (T)-1;                                     \
        for (int64_t i = k + 1; i < L; ++i) {                                 \
            T c = A[i + k * L];                                               \
            s[i] = c / r;                                                     \
            A[i + k * L] = c / d;                 /* [R10] L_ik = c_i / d */  \
        }                                                                     \
        /* [R8] P:67 rank-1 Schur update of the trailing lower triangle */    \
        _Pragma("omp parallel for schedule(dynamic, 16)")                     \
        for (int64_t j = k + 1; j < L; ++j) {                                 \
            T nsj = -sg * s[j];                                               \
            T *col = A + j * L;                                               \
            for (int64_t i = j; i < L; ++i)                                   \
                col[i] = FMA(nsj, s[i], col[i]);                              \
        }                                                                     \
    }                                                                         \
    if (kmax < L && Ntau == L) Ntau = kmax;   /* sampling run (bench only) */ \
    /* [R5] floor, [R9] P:82 enlargement by moving the last accepted pivots */ \
    int64_t N = Ntau;                                                         \
    if (L - n_min < N) N = (L - n_min > 0) ? L - n_min : 0;                   \
    if (N < L) N = (N - n_extra > 0) ? N - n_extra : 0;                       \
    /* [R10] Pi = [pivots, Lambda_2 ascending] */                             \
    for (int64_t p = 0; p < N; ++p) perm[p] = orig[p];                        \
    {                                                                         \
        char *used = (char *)calloc((size_t)(L > 0 ? L : 1), 1);              \
        if (!used) { free(A); free(s); free(orig); return -1; }               \
        for (int64_t p = 0; p < N; ++p) used[orig[p]] = 1;                    \
        int64_t w = N;                                                        \
        for (int64_t i = 0; i < L; ++i) if (!used[i]) perm[w++] = i;          \
        free(used);                                                           \
    }                                                                         \
    /* a bounded run (kmax < L) keeps EVERY row of its kmax columns, in its   \
       own position order (pos_orig below): output only, no arithmetic change */ \
    const int64_t nrow = (kmax < L) ? L : N;                                  \
    const int64_t nc = (ncol >= 0 && ncol < L) ? ncol : L;                    \
    for (int64_t j = 0; j < nc; ++j)                                          \
        for (int64_t i = 0; i < L; ++i) {                                     \
            T v = (T)0;                                                       \
            if (j < N && i < nrow) v = (i == j) ? (T)1 : ((i > j) ? A[i + j * L] : (T)0); \
            Lfac[i + j * L] = v;                                              \
        }                                                                     \
    if (pos_orig) for (int64_t p = 0; p < L; ++p) pos_orig[p] = orig[p];      \
    out[0] = N; out[1] = Ntau;                                                \
    free(A); free(s); free(orig);                                             \
    return 0;

int oracle_factor_f32(int64_t L, const double *K, int64_t ld, double tau,
                      int64_t n_min, int64_t n_extra, int64_t max_steps,
                      int64_t *perm, float *Dk, float *Lfac, int64_t *out,
                      int64_t ncol, int64_t *pos_orig)
{
    ORACLE_FACTOR_BODY(float, fmaf, sqrtf, fabsf)
}

int oracle_factor_f64(int64_t L, const double *K, int64_t ld, double tau,
                      int64_t n_min, int64_t n_extra, int64_t max_steps,
                      int64_t *perm, double *Dk, double *Lfac, int64_t *out,
                      int64_t ncol, int64_t *pos_orig)
{
    ORACLE_FACTOR_BODY(double, fma, sqrt, fabs)
}

/* ========================================================================= */
/* NEXT-3: the NONSYMMETRIC matrices of sec. 4.2-4.3     */
/* ([A B^T; -B delta D], [A B^T; -B 0]) with the same   */
/* symmetric pivoting and postponing.                               */
/* ========================================================================= */

/* P:40 scaling for a general matrix: K_ij = (q_i Kbar_ij) q_j for i != j,    */
/* every entry read (no symmetry assumed), diag(K) in {-1, 0, 1}.             */
int oracle_scale_full(int64_t L, const double *Kbar, int64_t ld, double *K, double *q)
{
    for (int64_t i = 0; i < L; ++i) {
        double d = Kbar[i + i * ld];
        q[i] = (d != 0.0) ? 1.0 / sqrt(fabs(d)) : 1.0;
    }
    for (int64_t j = 0; j < L; ++j)
        for (int64_t i = 0; i < L; ++i) {
            if (i == j) continue;
            K[i + j * ld] = (q[i] * Kbar[i + j * ld]) * q[j];
        }
    for (int64_t i = 0; i < L; ++i) {
        double d = Kbar[i + i * ld];
        K[i + i * ld] = (d > 0.0) ? 1.0 : ((d < 0.0) ? -1.0 : 0.0);
    }
    return 0;
}

/* FP32 LDU with symmetric pivoting and threshold postponing ("S'_22 */
/* = K~'_22 - [K~_22]_{down 1} d^{-1} [K~_22]_{1 right}"), right-looking on   */
/* the full matrix with physical row and column swaps.  Canonical arithmetic */
/* [R19] (fixed roles, one FMA per entry per pivot, pivots in order):        */
/*   d = v_PP, l_i = c_i / d (c_i = v_iP, IEEE division), r_j = v_Pj,         */
/*   v_ij <- fmaf(-l_i, r_j, v_ij)  for every active (i, j), diagonal too.    */
/* Pivot rule [R3], stop test [R4], floor [R5], enlargement [R9], Pi [R10]    */
/* exactly as oracle_factor_f32.  Factors (pivot order, ld = L):              */
/*   Lfac[i + k L] = l_i (unit lower), Ufac[i + k L] = r_i / d_k: column k    */
/*   holds ROW k of the unit upper U (so U = Ufac^T), Dk[k] = d_k.            */
int oracle_ldu_f32(int64_t L, const double *K, int64_t ld, double tau, int64_t n_min, int64_t n_extra,
                   int64_t *perm, float *Dk, float *Lfac, float *Ufac, int64_t *out)
{
    if (L < 0 || !(tau > 0.0 && tau < 1.0) || n_min < 0 || n_extra < 0) return -1;
    const size_t LL = (size_t)(L > 0 ? L : 1) * (size_t)(L > 0 ? L : 1);
    float *A = (float *)malloc(LL * sizeof(float));
    float *l = (float *)malloc((size_t)(L > 0 ? L : 1) * sizeof(float));
    float *r = (float *)malloc((size_t)(L > 0 ? L : 1) * sizeof(float));
    int64_t *orig = (int64_t *)malloc((size_t)(L > 0 ? L : 1) * sizeof(int64_t));
    if (!A || !l || !r || !orig) { free(A); free(l); free(r); free(orig); return -1; }
    for (int64_t j = 0; j < L; ++j)
        for (int64_t i = 0; i < L; ++i) A[i + j * L] = (float)K[i + j * ld];   /* [R2] */
    for (int64_t p = 0; p < L; ++p) orig[p] = p;
    int64_t Ntau = L;
    for (int64_t k = 0; k < L; ++k) {
        int64_t best = k;                                                     /* [R3] */
        for (int64_t p = k + 1; p < L; ++p) {
            float a = fabsf(A[p + p * L]), b = fabsf(A[best + best * L]);
            if (a > b || (a == b && orig[p] < orig[best])) best = p;
        }
        float d = A[best + best * L];
        if (k == 0 && d == 0.0f) { Ntau = 0; break; }                        /* [R4] */
        if (k > 0 && fabs((double)d) < tau * fabs((double)Dk[k - 1])) { Ntau = k; break; }
        if (best != k) {                      /* swap rows k, best and columns k, best */
            for (int64_t j = 0; j < L; ++j) {
                float t = A[k + j * L]; A[k + j * L] = A[best + j * L]; A[best + j * L] = t;
            }
            for (int64_t i = 0; i < L; ++i) {
                float t = A[i + k * L]; A[i + k * L] = A[i + best * L]; A[i + best * L] = t;
            }
            int64_t o = orig[k]; orig[k] = orig[best]; orig[best] = o;
        }
        Dk[k] = d;
        for (int64_t i = k + 1; i < L; ++i) {
            l[i] = A[i + k * L] / d;          /* column: c_i / d */
            r[i] = A[k + i * L];              /* row value r_i = v_{P i} */
        }
        for (int64_t i = k + 1; i < L; ++i) {
            A[i + k * L] = l[i];              /* L_ik stored in place (below the pivot) */
            A[k + i * L] = r[i] / d;          /* U_ki stored in place (right of the pivot) */
        }
        _Pragma("omp parallel for schedule(static)")
        for (int64_t j = k + 1; j < L; ++j) {
            const float rj = r[j];
            float *col = A + j * L;
            for (int64_t i = k + 1; i < L; ++i) col[i] = fmaf(-l[i], rj, col[i]);
        }
    }
    int64_t N = Ntau;
    if (L - n_min < N) N = (L - n_min > 0) ? L - n_min : 0;
    if (N < L) N = (N - n_extra > 0) ? N - n_extra : 0;
    for (int64_t p = 0; p < N; ++p) perm[p] = orig[p];
    {
        char *used = (char *)calloc((size_t)(L > 0 ? L : 1), 1);
        if (!used) { free(A); free(l); free(r); free(orig); return -1; }
        for (int64_t p = 0; p < N; ++p) used[orig[p]] = 1;
        int64_t w = N;
        for (int64_t i = 0; i < L; ++i) if (!used[i]) perm[w++] = i;
        free(used);
    }
    for (int64_t j = 0; j < L; ++j)
        for (int64_t i = 0; i < L; ++i) {
            float vl = 0.0f, vu = 0.0f;
            if (j < N && i < N) {
                vl = (i == j) ? 1.0f : ((i > j) ? A[i + j * L] : 0.0f);
                vu = (i == j) ? 1.0f : ((i > j) ? A[j + i * L] : 0.0f);
            }
            Lfac[i + j * L] = vl;
            Ufac[i + j * L] = vu;
        }
    out[0] = N; out[1] = Ntau;
    free(A); free(l); free(r); free(orig);
    return 0;
}

/* ========================================================================= */
/* NEXT-4: multi-block threshold postponing (sec. 2.2,  */
/* P:69-85).  The indices are split into blocks in elimination-tree order    */
/* (blk[original index] = block number 0..nblk-1, e.g. the post-order of a   */
/* nested-dissection tree).  "During the LDU-factorization of the sub- */
/* matrix with index Lambda_j, if |K_{i+1,i+1}/K_ii| < tau, then the lower   */
/* block of the matrix is not factorized": the pivots of block j are  */
/* chosen among ITS remaining indices only (max |diag|, ties -> smallest     */
/* original index [R3]), the ratio test [R4] compares each candidate with the */
/* previously ACCEPTED pivot of the elimination sequence (across blocks:     */
/* reading [R21]; only the very first pivot is tested against 0 alone); the  */
/* rest of a stopped block is postponed to Lambda_0.  "At the end of all     */
/* threshold                                                                 */
/* factorization following the elimination tree, we will again apply the     */
/* LDU-factorization to the last Schur complement with indices Lambda_0"     */
/* (P:80): a final pass over every remaining index with the same rules; its  */
/* tau-stop ends the factorization (Ntau).  Floor [R5] and the enlargement   */
/* by n_extra entries ("usually n = 4") as in oracle_factor_f32.       */
/* Arithmetic exactly [R2]-[R10] (this function IS oracle_factor_f32 when    */
/* nblk = 0).  Outputs as oracle_factor_f32.                                 */
/* ========================================================================= */
int oracle_factor_blocks_f32(int64_t L, const double *K, int64_t ld, double tau, int64_t n_min, int64_t n_extra,
                             const int32_t *blk, int32_t nblk, int64_t *perm, float *Dk, float *Lfac, int64_t *out)
{
    if (L < 0 || !(tau > 0.0 && tau < 1.0) || n_min < 0 || n_extra < 0 || nblk < 0) return -1;
    const size_t LL = (size_t)(L > 0 ? L : 1) * (size_t)(L > 0 ? L : 1);
    float *A = (float *)malloc(LL * sizeof(float));
    float *s = (float *)malloc((size_t)(L > 0 ? L : 1) * sizeof(float));
    int64_t *orig = (int64_t *)malloc((size_t)(L > 0 ? L : 1) * sizeof(int64_t));
    if (!A || !s || !orig) { free(A); free(s); free(orig); return -1; }
    for (int64_t j = 0; j < L; ++j)
        for (int64_t i = j; i < L; ++i) A[i + j * L] = (float)K[i + j * ld];
    for (int64_t p = 0; p < L; ++p) orig[p] = p;
    int64_t Ntau = L;
    int32_t cur = 0;          /* current block; cur == nblk: the final pass over Lambda_0 */
    int first = 1;            /* no pivot accepted yet */
    int64_t k = 0;
    while (k < L) {
        int64_t best = -1;
        for (int64_t p = k; p < L; ++p) {
            if (cur < nblk && blk[orig[p]] != cur) continue;
            if (best < 0) { best = p; continue; }
            float a = fabsf(A[p + p * L]), b = fabsf(A[best + best * L]);
            if (a > b || (a == b && orig[p] < orig[best])) best = p;
        }
        int fail = (best < 0);
        float d = 0.0f;
        if (!fail) {
            d = A[best + best * L];
            fail = first ? (d == 0.0f) : (fabs((double)d) < tau * fabs((double)Dk[k - 1]));
        }
        if (fail) {
            if (cur < nblk) { ++cur; continue; }   /* the rest of the block -> Lambda_0 */
            Ntau = k;                                         /* the final pass stops */
            break;
        }
        if (best != k) {   /* swap in the lower-triangle storage, exactly as oracle_factor_f32 */
            int64_t p = best; float t;
            for (int64_t j = 0; j < k; ++j) { t = A[k + j * L]; A[k + j * L] = A[p + j * L]; A[p + j * L] = t; }
            t = A[k + k * L]; A[k + k * L] = A[p + p * L]; A[p + p * L] = t;
            for (int64_t i = k + 1; i < p; ++i) { t = A[i + k * L]; A[i + k * L] = A[p + i * L]; A[p + i * L] = t; }
            for (int64_t i = p + 1; i < L; ++i) { t = A[i + k * L]; A[i + k * L] = A[i + p * L]; A[i + p * L] = t; }
            int64_t o = orig[k]; orig[k] = orig[p]; orig[p] = o;
        }
        Dk[k] = d;
        float r = sqrtf(fabsf(d)), sg = (d > 0.0f) ? 1.0f : -1.0f;
        for (int64_t i = k + 1; i < L; ++i) {
            float c = A[i + k * L];
            s[i] = c / r;
            A[i + k * L] = c / d;
        }
        _Pragma("omp parallel for schedule(dynamic, 16)")
        for (int64_t j = k + 1; j < L; ++j) {
            float nsj = -sg * s[j];
            float *col = A + j * L;
            for (int64_t i = j; i < L; ++i) col[i] = fmaf(nsj, s[i], col[i]);
        }
        first = 0;
        ++k;
    }
    int64_t N = Ntau;
    if (L - n_min < N) N = (L - n_min > 0) ? L - n_min : 0;
    if (N < L) N = (N - n_extra > 0) ? N - n_extra : 0;
    for (int64_t p = 0; p < N; ++p) perm[p] = orig[p];
    {
        char *used = (char *)calloc((size_t)(L > 0 ? L : 1), 1);
        if (!used) { free(A); free(s); free(orig); return -1; }
        for (int64_t p = 0; p < N; ++p) used[orig[p]] = 1;
        int64_t w = N;
        for (int64_t i = 0; i < L; ++i) if (!used[i]) perm[w++] = i;
        free(used);
    }
    for (int64_t j = 0; j < L; ++j)
        for (int64_t i = 0; i < L; ++i) {
            float v = 0.0f;
            if (j < N && i < N) v = (i == j) ? 1.0f : ((i > j) ? A[i + j * L] : 0.0f);
            Lfac[i + j * L] = v;
        }
    out[0] = N; out[1] = Ntau;
    free(A); free(s); free(orig);
    return 0;
}
