// gcr_dd.cu -- NEXT-1, the higher-precision half of the
// (double, double-double) pair of the paper's Table 1 ("quadruple
// precision" P:26-27): with the FP64 canonical factorization
// (prec 64) as the lower-precision preconditioner Q^{-1}, Alg. 1
// steps 3-5 run in double-double:
//   * block GCR (Alg. 5) with every N x n2 block (X, R, P_m, Q_m)
//     held as (hi, lo) pairs; K11 W is formed with error-free products
//     (two-product by FMA) and double-double sums; Gram matrices, their
//     inverses and all block updates in double-double;
//   * S22 = K22 - K21 X12 (Eq. 2) in double-double;
//   * the Bunch-Parlett factorization of S22 with the kernel rule [R15]
//      in double-double.
// The preconditioner consumes the hi part of the residual (the residual
// rounded to double, which is exactly what "find e^ in lower precision" of
// P:242 does) and returns double corrections (lo = 0).
//
// Arithmetic: Knuth two-sum, Dekker/FMA two-product, the accurate
// double-double addition (two two-sums, two renormalisations) and the
// FMA-based double-double product; every operation is an explicit
// round-to-nearest intrinsic so the compiler cannot contract an error-free
// transformation.  All summation orders are fixed (deterministic results).
//
// Kernels: k_ddgemm (64 x 64 CTA tiles, 4 x 4 double-double accumulators per
// thread, K in chunks of 16 through shared memory, optional split-K reduced in
// split order), k_dd_reduce, k_dd_spd_inv (Gauss-Jordan, one CTA), k_dd_hard
// (Bunch-Parlett, one CTA), small element-wise kernels.  Bound: the FP64 FMA
// pipe (about 24 FP64 operations per double-double multiply-add).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "k_dgemm.cuh"
#include "k_small.cuh"

namespace hf {
namespace {

// ------------------------------------------------------------------ dd arithmetic
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {   // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
    dd s = two_sum(x.hi, y.hi);
    const dd t = two_sum(x.lo, y.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    dd p = two_prod(x.hi, y.hi);
    p.lo = __fma_rn(x.hi, y.lo, p.lo);
    p.lo = __fma_rn(x.lo, y.hi, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {   // three-term long division
    const double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = dd_sub(a, dd_mul({q1, 0.0}, b));
    const double q2 = __ddiv_rn(r.hi, b.hi);
    r = dd_sub(r, dd_mul({q2, 0.0}, b));
    const double q3 = __ddiv_rn(r.hi, b.hi);
    return dd_add(quick_two_sum(q1, q2), {q3, 0.0});
}
__device__ __forceinline__ double dd_abs_hi(dd x) { return fabs(x.hi); }

// ------------------------------------------------------------------ dd GEMM
// C = beta C + sgn * mask o (op(A) B): A M x K (TA: stored K x M), B K x N,
// column-major; A and B each double (lo pointer null) or double-double.
struct DDG {
    int64_t M, N, K;
    double sgn;
    const double *Ah, *Al;
    int64_t lda;
    const double *Bh, *Bl;
    int64_t ldb;
    int beta;                 // 0 or 1
    double *Ch, *Cl;
    int64_t ldc;
    const uint8_t *mask;      // rows with 0 get beta C only
    double *Wh, *Wl;          // split-K partials [split][M x N] (splits > 1)
    int64_t kper;             // K per split
};
constexpr int DBT = 64, DKC = 16;

template <bool TA, bool ADD, bool BDD>
__global__ void __launch_bounds__(256) k_ddgemm(DDG g) {
    __shared__ double Ash[DKC][DBT], Asl[DKC][DBT], Bsh[DKC][DBT], Bsl[DKC][DBT];
    const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.x * DBT, n0 = (int64_t)blockIdx.y * DBT;
    const int64_t k_lo = (int64_t)blockIdx.z * g.kper, k_hi = min(g.K, k_lo + g.kper);
    dd acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = {0.0, 0.0};
    for (int64_t k0 = k_lo; k0 < k_hi; k0 += DKC) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + u * 256;
            int kk, m;
            if (TA) { kk = e & 15; m = e >> 4; }
            else { m = e & 63; kk = e >> 6; }
            const int64_t gm = m0 + m, gk = k0 + kk;
            double vh = 0.0, vl = 0.0;
            if (gm < g.M && gk < k_hi) {
                const int64_t o = TA ? gk + gm * g.lda : gm + gk * g.lda;
                vh = g.Ah[o];
                if (ADD) vl = g.Al[o];
            }
            Ash[kk][m] = vh;
            Asl[kk][m] = vl;
            const int kb = e & 15, nb = e >> 4;
            const int64_t gn = n0 + nb, gkb = k0 + kb;
            double bh = 0.0, bl = 0.0;
            if (gn < g.N && gkb < k_hi) {
                bh = g.Bh[gkb + gn * g.ldb];
                if (BDD) bl = g.Bl[gkb + gn * g.ldb];
            }
            Bsh[kb][nb] = bh;
            Bsl[kb][nb] = bl;
        }
        __syncthreads();
        const int kmax = (int)min((int64_t)DKC, k_hi - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            double ah[4], al[4], bh[4], bl[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                ah[i] = Ash[kk][tr * 4 + i];
                al[i] = Asl[kk][tr * 4 + i];
                bh[i] = Bsh[kk][tc * 4 + i];
                bl[i] = Bsl[kk][tc * 4 + i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    dd p = two_prod(ah[i], bh[j]);
                    if (BDD) p.lo = __fma_rn(ah[i], bl[j], p.lo);
                    if (ADD) p.lo = __fma_rn(al[i], bh[j], p.lo);
                    acc[i][j] = dd_add(acc[i][j], p);
                }
        }
        __syncthreads();
    }
    const bool split = gridDim.z > 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = m0 + tr * 4 + i;
        if (r >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = n0 + tc * 4 + j;
            if (c >= g.N) continue;
            if (split) {
                const size_t o = (size_t)blockIdx.z * g.M * g.N + r + c * g.M;
                g.Wh[o] = acc[i][j].hi;
                g.Wl[o] = acc[i][j].lo;
                continue;
            }
            dd v = (g.mask && !g.mask[r]) ? dd{0.0, 0.0} : acc[i][j];
            if (g.sgn < 0) v = dd_neg(v);
            const int64_t o = r + c * g.ldc;
            if (g.beta) v = dd_add({g.Ch[o], g.Cl[o]}, v);
            g.Ch[o] = v.hi;
            g.Cl[o] = v.lo;
        }
    }
}

// split-K partials summed in split order, then masked, signed and added to beta C
__global__ void k_dd_reduce(DDG g, int splits) {
    const int64_t n = g.M * g.N;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % g.M, c = e / g.M;
        dd v{0.0, 0.0};
        for (int z = 0; z < splits; ++z) v = dd_add(v, {g.Wh[(size_t)z * n + e], g.Wl[(size_t)z * n + e]});
        if (g.mask && !g.mask[r]) v = {0.0, 0.0};
        if (g.sgn < 0) v = dd_neg(v);
        const int64_t o = r + c * g.ldc;
        if (g.beta) v = dd_add({g.Ch[o], g.Cl[o]}, v);
        g.Ch[o] = v.hi;
        g.Cl[o] = v.lo;
    }
}

struct DDWork {
    DBuf<double> h, l;
};

void ddgemm(hf_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double sgn, const double *Ah,
            const double *Al, int64_t lda, const double *Bh, const double *Bl, int64_t ldb, bool beta, double *Ch,
            double *Cl, int64_t ldc, const uint8_t *mask, DDWork &w) {
    if (M <= 0 || N <= 0) return;
    cudaStream_t st = ctx->stream;
    const int64_t mt = cdiv(M, DBT), nt = cdiv(N, DBT);
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(2 * (int64_t)ctx->num_sms, mt * nt), K / 512));
    splits = std::min(splits, 64);
    if (K == 0) splits = 1;
    DDG g{M, N, K, sgn, Ah, Al, lda, Bh, Bl, ldb, beta ? 1 : 0, Ch, Cl, ldc, mask, nullptr, nullptr, 0};
    g.kper = cdiv(std::max<int64_t>(K, 1), splits);
    g.kper = cdiv(g.kper, DKC) * DKC;
    splits = (int)std::max<int64_t>(1, cdiv(std::max<int64_t>(K, 1), g.kper));
    if (splits > 1) {
        w.h.alloc((size_t)splits * M * N, st);
        w.l.alloc((size_t)splits * M * N, st);
        g.Wh = w.h.p;
        g.Wl = w.l.p;
    }
    ClassTimer tm(ctx, "ddgemm");
    dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)splits);
    const bool add = Al != nullptr, bdd = Bl != nullptr;
#define DDG_LAUNCH(TA_, A_, B_) k_ddgemm<TA_, A_, B_><<<grid, 256, 0, st>>>(g)
    if (transA) {
        if (add && bdd) DDG_LAUNCH(true, true, true);
        else if (add) DDG_LAUNCH(true, true, false);
        else if (bdd) DDG_LAUNCH(true, false, true);
        else DDG_LAUNCH(true, false, false);
    } else {
        if (add && bdd) DDG_LAUNCH(false, true, true);
        else if (add) DDG_LAUNCH(false, true, false);
        else if (bdd) DDG_LAUNCH(false, false, true);
        else DDG_LAUNCH(false, false, false);
    }
#undef DDG_LAUNCH
    HF_CHECK_LAUNCH(ctx);
    if (splits > 1) {
        k_dd_reduce<<<(unsigned)std::min<int64_t>(cdiv(M * N, 256), 4096), 256, 0, st>>>(g, splits);
        HF_CHECK_LAUNCH(ctx);
    }
}

// ------------------------------------------------------------------ small dd kernels
// Inverse of the SPD n x n dd matrix M (Gauss-Jordan without pivoting on [M | I],
// one CTA; W: 2 n^2 dd workspace); status = 1 on a non-positive pivot.
__global__ void __launch_bounds__(1024) k_dd_spd_inv(int n, const double *Mh, const double *Ml, int ldm, double *Wh,
                                                     double *Wl, double *Ih, double *Il, int *status) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t ldw = n;   // W: n x 2n column-major
    for (int64_t e = tid; e < (int64_t)n * 2 * n; e += nt) {
        const int64_t r = e % n, c = e / n;
        if (c < n) {
            Wh[e] = Mh[r + c * ldm];
            Wl[e] = Ml[r + c * ldm];
        } else {
            Wh[e] = (c - n == r) ? 1.0 : 0.0;
            Wl[e] = 0.0;
        }
    }
    __syncthreads();
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        const dd piv{Wh[k + k * ldw], Wl[k + k * ldw]};
        if (!(piv.hi > 0.0)) {
            if (tid == 0) bad = 1;
            break;
        }
        __syncthreads();
        // row k /= piv (columns k..2n-1)
        for (int c = k + tid; c < 2 * n; c += nt) {
            const dd v = dd_div({Wh[k + c * ldw], Wl[k + c * ldw]}, piv);
            Wh[k + c * ldw] = v.hi;
            Wl[k + c * ldw] = v.lo;
        }
        __syncthreads();
        // rows i != k: row_i -= W(i,k) row_k  (column k is read first by every thread)
        for (int64_t e = tid; e < (int64_t)n * (2 * n - k - 1); e += nt) {
            const int i = (int)(e % n);
            const int c = k + 1 + (int)(e / n);
            if (i == k) continue;
            const dd f{Wh[i + k * ldw], Wl[i + k * ldw]};
            const dd v = dd_sub({Wh[i + (int64_t)c * ldw], Wl[i + (int64_t)c * ldw]},
                                dd_mul(f, {Wh[k + (int64_t)c * ldw], Wl[k + (int64_t)c * ldw]}));
            Wh[i + (int64_t)c * ldw] = v.hi;
            Wl[i + (int64_t)c * ldw] = v.lo;
        }
        __syncthreads();
        for (int i = tid; i < n; i += nt) {
            Wh[i + k * ldw] = (i == k) ? 1.0 : 0.0;
            Wl[i + k * ldw] = 0.0;
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0 && bad) *status = 1;
    for (int64_t e = tid; e < (int64_t)n * n; e += nt) {
        Ih[e] = Wh[e + (int64_t)n * n];
        Il[e] = Wl[e + (int64_t)n * n];
    }
}

__global__ void k_dd_copy(int64_t n, const double *sh, const double *sl, double *dh, double *dl) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        dh[e] = sh[e];
        dl[e] = sl ? sl[e] : 0.0;
    }
}

// Bunch-Parlett (complete pivoting, alpha = (1 + sqrt 17) / 8) LDL^T of the dd
// matrix A = (S + S^T) / 2 with 1x1 / 2x2 pivots, one CTA; stops when the largest
// |entry| (hi part) of the active block is <= thr.  Pivot search on hi parts,
// ties to the smallest (label) pair -- the FP64 kernel's rule.  Outputs the rank
// and the pivot sequence (labels, block sizes).
__global__ void __launch_bounds__(1024) k_dd_hard(int n, const double *Sh, const double *Sl, double thr, double *Ah,
                                                  double *Al, double *Lch, double *Lcl, int32_t *act, int32_t *pivots,
                                                  int32_t *blocks, int64_t *rank_out) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t e = tid; e < (int64_t)n * n; e += nt) {
        const int64_t i = e % n, j = e / n;
        const dd v = dd_mul({0.5, 0.0}, dd_add({Sh[i + j * n], Sl[i + j * n]}, {Sh[j + i * n], Sl[j + i * n]}));
        Ah[e] = v.hi;
        Al[e] = v.lo;
        Lch[e] = 0.0;
        Lcl[e] = 0.0;
    }
    for (int i = tid; i < n; i += nt) {
        act[i] = 1;
        blocks[i] = 0;
    }
    __shared__ double rv[32];
    __shared__ int ri[32], rj[32];
    __shared__ double sd_v, so_v;
    __shared__ int sd_i, so_i, so_j;
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    __syncthreads();
    int k = 0, nblk = 0;
    auto better = [](double v, int i, int j, double bv, int bi, int bj) {
        return v > bv || (v == bv && (i < bi || (i == bi && j < bj)));
    };
    while (k < n) {
        // search: max |diagonal| and max |off-diagonal| over the active block (hi parts)
        for (int pass = 0; pass < 2; ++pass) {
            double bv = -1.0;
            int bi = 0x7fffffff, bj = 0x7fffffff;
            if (pass == 0) {
                for (int i = tid; i < n; i += nt)
                    if (act[i]) {
                        const double v = fabs(Ah[i + (int64_t)i * n]);
                        if (better(v, i, i, bv, bi, bj)) { bv = v; bi = i; bj = i; }
                    }
            } else {
                for (int64_t e = tid; e < (int64_t)n * n; e += nt) {
                    const int i = (int)(e % n), j = (int)(e / n);
                    if (i <= j || !act[i] || !act[j]) continue;
                    const double v = fabs(Ah[e]);
                    if (better(v, j, i, bv, bi, bj)) { bv = v; bi = j; bj = i; }
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (better(ov, oi, oj, bv, bi, bj)) { bv = ov; bi = oi; bj = oj; }
            }
            if (lane == 0) { rv[wid] = bv; ri[wid] = bi; rj[wid] = bj; }
            __syncthreads();
            if (tid == 0) {
                double v = -1.0;
                int i2 = 0x7fffffff, j2 = 0x7fffffff;
                for (int w = 0; w < nw; ++w)
                    if (better(rv[w], ri[w], rj[w], v, i2, j2)) { v = rv[w]; i2 = ri[w]; j2 = rj[w]; }
                if (pass == 0) { sd_v = v; sd_i = i2; }
                else { so_v = v; so_i = i2; so_j = j2; }
            }
            __syncthreads();
        }
        const double mu1 = sd_v, mu0 = fmax(sd_v, so_v);
        if (mu0 <= thr) break;   // uniform
        if (mu1 >= alpha * mu0) {
            const int p = sd_i;
            const dd d{Ah[p + (int64_t)p * n], Al[p + (int64_t)p * n]};
            for (int64_t e = tid; e < (int64_t)n * n; e += nt) {
                const int i = (int)(e % n), j = (int)(e / n);
                if (!act[i] || !act[j] || i == p || j == p) continue;
                const dd lip = dd_div({Ah[i + (int64_t)p * n], Al[i + (int64_t)p * n]}, d);
                const dd v = dd_sub({Ah[e], Al[e]}, dd_mul(lip, {Ah[p + (int64_t)j * n], Al[p + (int64_t)j * n]}));
                Ah[e] = v.hi;
                Al[e] = v.lo;
            }
            for (int i = tid; i < n; i += nt)   // L column (label space): l_ip = A_ip / d
                if (act[i] && i != p) {
                    const dd l = dd_div({Ah[i + (int64_t)p * n], Al[i + (int64_t)p * n]}, d);
                    Lch[i + (int64_t)p * n] = l.hi;
                    Lcl[i + (int64_t)p * n] = l.lo;
                }
            __syncthreads();
            if (tid == 0) {
                act[p] = 0;
                pivots[k] = p;
                blocks[nblk] = 1;
            }
            ++nblk;
            k += 1;
        } else {
            const int p = min(so_i, so_j), q = max(so_i, so_j);
            const dd a_{Ah[p + (int64_t)p * n], Al[p + (int64_t)p * n]}, b_{Ah[q + (int64_t)p * n], Al[q + (int64_t)p * n]},
                c_{Ah[q + (int64_t)q * n], Al[q + (int64_t)q * n]};
            const dd det = dd_sub(dd_mul(a_, c_), dd_mul(b_, b_));
            for (int64_t e = tid; e < (int64_t)n * n; e += nt) {
                const int i = (int)(e % n), j = (int)(e / n);
                if (!act[i] || !act[j] || i == p || j == p || i == q || j == q) continue;
                // A_ij -= [A_ip A_iq] E^{-1} [A_pj; A_qj],  E^{-1} = [c -b; -b a] / det
                const dd aip{Ah[i + (int64_t)p * n], Al[i + (int64_t)p * n]}, aiq{Ah[i + (int64_t)q * n], Al[i + (int64_t)q * n]};
                const dd apj{Ah[p + (int64_t)j * n], Al[p + (int64_t)j * n]}, aqj{Ah[q + (int64_t)j * n], Al[q + (int64_t)j * n]};
                const dd l0 = dd_div(dd_sub(dd_mul(aip, c_), dd_mul(aiq, b_)), det);
                const dd l1 = dd_div(dd_sub(dd_mul(aiq, a_), dd_mul(aip, b_)), det);
                const dd v = dd_sub({Ah[e], Al[e]}, dd_add(dd_mul(l0, apj), dd_mul(l1, aqj)));
                Ah[e] = v.hi;
                Al[e] = v.lo;
            }
            for (int i = tid; i < n; i += nt)   // the two L columns: [l0 l1] = [A_ip A_iq] E^{-1}
                if (act[i] && i != p && i != q) {
                    const dd aip{Ah[i + (int64_t)p * n], Al[i + (int64_t)p * n]}, aiq{Ah[i + (int64_t)q * n], Al[i + (int64_t)q * n]};
                    const dd l0 = dd_div(dd_sub(dd_mul(aip, c_), dd_mul(aiq, b_)), det);
                    const dd l1 = dd_div(dd_sub(dd_mul(aiq, a_), dd_mul(aip, b_)), det);
                    Lch[i + (int64_t)p * n] = l0.hi;
                    Lcl[i + (int64_t)p * n] = l0.lo;
                    Lch[i + (int64_t)q * n] = l1.hi;
                    Lcl[i + (int64_t)q * n] = l1.lo;
                }
            __syncthreads();
            if (tid == 0) {
                act[p] = act[q] = 0;
                pivots[k] = p;
                pivots[k + 1] = q;
                blocks[nblk] = 2;
            }
            ++nblk;
            k += 2;
        }
        __syncthreads();
    }
    if (tid == 0) *rank_out = k;
}

// x = S22^+ y in double-double with the factors of k_dd_hard (label space: D blocks at
// A[p, p] / A[q, p] / A[q, q], L columns in Lc), kernel coordinates 0 [R16]; one CTA.
__global__ void __launch_bounds__(256) k_dd_hard_solve(int n, int64_t r, const double *Ah, const double *Al,
                                                       const double *Lch, const double *Lcl, const int32_t *pivots,
                                                       const int32_t *blocks, const double *yh, const double *yl,
                                                       double *xh, double *xl, int32_t *act) {
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ double rh[256], rl[256];
    for (int i = tid; i < n; i += nt) {
        xh[i] = yh[i];
        xl[i] = yl ? yl[i] : 0.0;
        act[i] = 1;
    }
    __syncthreads();
    // forward: z_i -= l_ip z_p (pivot blocks in order)
    for (int64_t k = 0, b = 0; k < r; ++b) {
        const int bs = blocks[b];
        const int p = pivots[k], q = bs == 2 ? pivots[k + 1] : -1;
        const dd zp{xh[p], xl[p]}, zq = q >= 0 ? dd{xh[q], xl[q]} : dd{0.0, 0.0};
        __syncthreads();
        for (int i = tid; i < n; i += nt) {
            if (!act[i] || i == p || i == q) continue;
            dd v = dd_mul({Lch[i + (int64_t)p * n], Lcl[i + (int64_t)p * n]}, zp);
            if (q >= 0) v = dd_add(v, dd_mul({Lch[i + (int64_t)q * n], Lcl[i + (int64_t)q * n]}, zq));
            const dd z = dd_sub({xh[i], xl[i]}, v);
            xh[i] = z.hi;
            xl[i] = z.lo;
        }
        __syncthreads();
        if (tid == 0) {
            act[p] = 0;
            if (q >= 0) act[q] = 0;
        }
        __syncthreads();
        k += bs;
    }
    // block diagonal, then kernel coordinates 0
    if (tid == 0) {
        for (int64_t k = 0, b = 0; k < r; ++b) {
            const int bs = blocks[b];
            const int p = pivots[k];
            if (bs == 1) {
                const dd z = dd_div({xh[p], xl[p]}, {Ah[p + (int64_t)p * n], Al[p + (int64_t)p * n]});
                xh[p] = z.hi;
                xl[p] = z.lo;
            } else {
                const int q = pivots[k + 1];
                const dd a_{Ah[p + (int64_t)p * n], Al[p + (int64_t)p * n]}, b_{Ah[q + (int64_t)p * n], Al[q + (int64_t)p * n]},
                    c_{Ah[q + (int64_t)q * n], Al[q + (int64_t)q * n]};
                const dd det = dd_sub(dd_mul(a_, c_), dd_mul(b_, b_));
                const dd z0{xh[p], xl[p]}, z1{xh[q], xl[q]};
                const dd w0 = dd_div(dd_sub(dd_mul(c_, z0), dd_mul(b_, z1)), det);
                const dd w1 = dd_div(dd_sub(dd_mul(a_, z1), dd_mul(b_, z0)), det);
                xh[p] = w0.hi; xl[p] = w0.lo;
                xh[q] = w1.hi; xl[q] = w1.lo;
            }
            k += bs;
        }
    }
    __syncthreads();
    for (int i = tid; i < n; i += nt)
        if (act[i]) {   // never pivoted: kernel coordinate
            xh[i] = 0.0;
            xl[i] = 0.0;
        }
    __syncthreads();
    // backward: z_p -= sum_i l_ip z_i over the rows eliminated after p (blocks in reverse)
    int64_t nb = 0;
    for (int64_t k = 0; k < r; ++nb) k += blocks[nb];
    for (int64_t b = nb - 1, k = r; b >= 0; --b) {
        const int bs = blocks[b];
        k -= bs;
        for (int c = 0; c < bs; ++c) {
            const int p = pivots[k + c];
            // rows after the block: every i whose L entry in column p is set (zero elsewhere)
            dd s{0.0, 0.0};
            for (int i = tid; i < n; i += nt) {
                const dd l{Lch[i + (int64_t)p * n], Lcl[i + (int64_t)p * n]};
                if (l.hi != 0.0 || l.lo != 0.0) s = dd_add(s, dd_mul(l, {xh[i], xl[i]}));
            }
            rh[tid] = s.hi;
            rl[tid] = s.lo;
            __syncthreads();
            if (tid == 0) {
                dd t{0.0, 0.0};
                for (int w = 0; w < nt; ++w) t = dd_add(t, {rh[w], rl[w]});
                const dd z = dd_sub({xh[p], xl[p]}, t);
                xh[p] = z.hi;
                xl[p] = z.lo;
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ Alg. 5 in dd
struct GcrDD {
    DBuf<double> Ph, Pl, Qh, Ql;   // L x cap*n
    int64_t cap = 0;
    DBuf<double> Mih, Mil;         // cap * n * n inverses
    DBuf<double> Rh, Rl, Wd, Mh, Ml, Anh, Anl, Ch, Cl, Hh, Hl, Gh, Gl, Gwh, Gwl;
    DBuf<double> bn2, rn2, res;
    DBuf<int> status;
    DDWork w;
};

void grow_dd(hf_ctx *ctx, GcrDD &g, int64_t L, int64_t n, int64_t need) {
    if (need <= g.cap) return;
    const int64_t nc = std::max<int64_t>(need, std::max<int64_t>(8, 2 * g.cap));
    cudaStream_t st = ctx->stream;
    DBuf<double> *bufs[6] = {&g.Ph, &g.Pl, &g.Qh, &g.Ql, &g.Mih, &g.Mil};
    const size_t per[6] = {(size_t)L * n, (size_t)L * n, (size_t)L * n, (size_t)L * n, (size_t)n * n, (size_t)n * n};
    for (int b = 0; b < 6; ++b) {
        DBuf<double> nb;
        nb.alloc(per[b] * nc, st);
        if (g.cap > 0)
            HF_CUDA(cudaMemcpyAsync(nb.p, bufs[b]->p, per[b] * g.cap * sizeof(double), cudaMemcpyDeviceToDevice, st));
        *bufs[b] = std::move(nb);
    }
    g.cap = nc;
}

double read_res_dd(hf_ctx *ctx, GcrDD &g, int *bad) {
    double r = 0.0;
    int s = 0;
    HF_CUDA(cudaMemcpyAsync(&r, g.res.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    HF_CUDA(cudaMemcpyAsync(&s, g.status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    HF_CUDA(cudaStreamSynchronize(ctx->stream));
    *bad = s;
    return r;
}

void spd_inverse_dd(hf_ctx *ctx, int64_t n, const double *Mh, const double *Ml, double *Ih, double *Il, GcrDD &g) {
    g.Gwh.alloc((size_t)2 * n * n, ctx->stream);
    g.Gwl.alloc((size_t)2 * n * n, ctx->stream);
    ClassTimer tm(ctx, "gram");
    k_dd_spd_inv<<<1, 1024, 0, ctx->stream>>>((int)n, Mh, Ml, (int)n, g.Gwh.p, g.Gwl.p, Ih, Il, g.status.p);
    HF_CHECK_LAUNCH(ctx);
}

// K11 X = B (L x n, original order, Lambda_2 rows zero; B double, X dd)
void block_gcr_dd(hf_ctx *ctx, const double *K, int64_t ld, int64_t L, const uint8_t *mask, Precond &pc,
                  const double *B, int64_t n, double *Xh, double *Xl, const hf_gcr_opts &o, hf_gcr_info *info,
                  GcrDD &g) {
    cudaStream_t st = ctx->stream;
    const size_t Ln = (size_t)L * n;
    g.Rh.alloc(Ln, st);
    g.Rl.alloc(Ln, st);
    g.Wd.alloc(Ln, st);
    g.bn2.alloc(n, st);
    g.rn2.alloc(n, st);
    g.res.alloc(1, st);
    g.status.alloc(1, st);
    g.status.zero(st);
    for (DBuf<double> *b : {&g.Mh, &g.Ml, &g.Anh, &g.Anl, &g.Ch, &g.Cl}) b->alloc((size_t)n * n, st);
    colnorm2(ctx, L, n, B, L, g.bn2.p);
    // x_0 = Q^{-1} b (double, lo = 0);  r_0 = b - K11 x_0 in dd
    precond_apply(ctx, pc, n, B, L, g.Wd.p, L);
    k_dd_copy<<<1024, 256, 0, st>>>((int64_t)Ln, g.Wd.p, nullptr, Xh, Xl);
    HF_CHECK_LAUNCH(ctx);
    k_dd_copy<<<1024, 256, 0, st>>>((int64_t)Ln, B, nullptr, g.Rh.p, g.Rl.p);
    HF_CHECK_LAUNCH(ctx);
    ddgemm(ctx, false, L, n, L, -1.0, K, nullptr, ld, Xh, Xl, L, true, g.Rh.p, g.Rl.p, L, mask, g.w);
    colnorm2(ctx, L, n, g.Rh.p, L, g.rn2.p);
    maxres(ctx, n, g.rn2.p, g.bn2.p, g.res.p);
    int bad = 0;
    double res = read_res_dd(ctx, g, &bad);
    int iters = 0;
    bool conv = res <= o.tol;
    if (!conv) {
        grow_dd(ctx, g, L, n, 2);
        precond_apply(ctx, pc, n, g.Rh.p, L, g.Wd.p, L);                       // w_0 = Q^{-1} r_0 (hi part)
        k_dd_copy<<<1024, 256, 0, st>>>((int64_t)Ln, g.Wd.p, nullptr, g.Ph.p, g.Pl.p);   // p_0 = w_0
        HF_CHECK_LAUNCH(ctx);
        ddgemm(ctx, false, L, n, L, 1.0, K, nullptr, ld, g.Wd.p, nullptr, L, false, g.Qh.p, g.Ql.p, L, mask, g.w);
        for (int it = 0; it < o.max_iter; ++it) {
            const size_t off = (size_t)it * Ln;
            const double *Pnh = g.Ph.p + off, *Pnl = g.Pl.p + off, *Qnh = g.Qh.p + off, *Qnl = g.Ql.p + off;
            double *Mih = g.Mih.p + (size_t)it * n * n, *Mil = g.Mil.p + (size_t)it * n * n;
            ddgemm(ctx, true, n, n, L, 1.0, Qnh, Qnl, L, Qnh, Qnl, L, false, g.Mh.p, g.Ml.p, n, nullptr, g.w);      // M_n
            ddgemm(ctx, true, n, n, L, 1.0, Qnh, Qnl, L, g.Rh.p, g.Rl.p, L, false, g.Anh.p, g.Anl.p, n, nullptr, g.w);  // A_n
            spd_inverse_dd(ctx, n, g.Mh.p, g.Ml.p, Mih, Mil, g);
            ddgemm(ctx, false, n, n, n, 1.0, Mih, Mil, n, g.Anh.p, g.Anl.p, n, false, g.Ch.p, g.Cl.p, n, nullptr, g.w);
            ddgemm(ctx, false, L, n, n, 1.0, Pnh, Pnl, L, g.Ch.p, g.Cl.p, n, true, Xh, Xl, L, nullptr, g.w);       // x += p C
            ddgemm(ctx, false, L, n, n, -1.0, Qnh, Qnl, L, g.Ch.p, g.Cl.p, n, true, g.Rh.p, g.Rl.p, L, nullptr, g.w);  // r -= q C
            colnorm2(ctx, L, n, g.Rh.p, L, g.rn2.p);
            maxres(ctx, n, g.rn2.p, g.bn2.p, g.res.p);
            res = read_res_dd(ctx, g, &bad);
            iters = it + 1;
            if (res <= o.tol) {
                conv = true;
                break;
            }
            if (bad) {
                info->iters = iters;
                info->max_rel_res_recursive = res;
                throw Error{HF_ERR_BREAKDOWN, "double-double block GCR: Gram matrix M_n is not positive definite"};
            }
            if (it + 1 >= o.max_iter) break;
            grow_dd(ctx, g, L, n, it + 2);
            const size_t off1 = (size_t)(it + 1) * Ln;
            const int64_t nb = (int64_t)(it + 1) * n;
            precond_apply(ctx, pc, n, g.Rh.p, L, g.Wd.p, L);                                                  // w_{n+1}
            k_dd_copy<<<1024, 256, 0, st>>>((int64_t)Ln, g.Wd.p, nullptr, g.Ph.p + off1, g.Pl.p + off1);
            HF_CHECK_LAUNCH(ctx);
            ddgemm(ctx, false, L, n, L, 1.0, K, nullptr, ld, g.Wd.p, nullptr, L, false, g.Qh.p + off1, g.Ql.p + off1, L,
                   mask, g.w);                                                                                 // z = A w
            g.Hh.alloc((size_t)nb * n, st);
            g.Hl.alloc((size_t)nb * n, st);
            g.Gh.alloc((size_t)nb * n, st);
            g.Gl.alloc((size_t)nb * n, st);
            ddgemm(ctx, true, nb, n, L, 1.0, g.Qh.p, g.Ql.p, L, g.Qh.p + off1, g.Ql.p + off1, L, false, g.Hh.p, g.Hl.p, nb,
                   nullptr, g.w);                                                                              // Q_m^T z
            for (int m = 0; m <= it; ++m)                                                                      // G_m = -M_m^{-1} Q_m^T z
                ddgemm(ctx, false, n, n, n, -1.0, g.Mih.p + (size_t)m * n * n, g.Mil.p + (size_t)m * n * n, n,
                       g.Hh.p + (size_t)m * n, g.Hl.p + (size_t)m * n, nb, false, g.Gh.p + (size_t)m * n,
                       g.Gl.p + (size_t)m * n, nb, nullptr, g.w);
            ddgemm(ctx, false, L, n, nb, 1.0, g.Ph.p, g.Pl.p, L, g.Gh.p, g.Gl.p, nb, true, g.Ph.p + off1, g.Pl.p + off1, L,
                   nullptr, g.w);                                                                              // p_{n+1}
            ddgemm(ctx, false, L, n, nb, 1.0, g.Qh.p, g.Ql.p, L, g.Gh.p, g.Gl.p, nb, true, g.Qh.p + off1, g.Ql.p + off1, L,
                   nullptr, g.w);                                                                              // q_{n+1}
        }
    }
    info->iters = iters;
    info->max_rel_res_recursive = res;
    // true residual ||B - K11 X|| / ||B|| in dd (reported)
    k_dd_copy<<<1024, 256, 0, st>>>((int64_t)Ln, B, nullptr, g.Rh.p, g.Rl.p);
    HF_CHECK_LAUNCH(ctx);
    ddgemm(ctx, false, L, n, L, -1.0, K, nullptr, ld, Xh, Xl, L, true, g.Rh.p, g.Rl.p, L, mask, g.w);
    colnorm2(ctx, L, n, g.Rh.p, L, g.rn2.p);
    maxres(ctx, n, g.rn2.p, g.bn2.p, g.res.p);
    info->max_rel_res_true = read_res_dd(ctx, g, &bad);
    if (!conv) throw Error{HF_ERR_NOT_CONVERGED, "double-double block GCR reached max_iter"};
}

}  // namespace

// ------------------------------------------------------------------ Alg. 1 steps 2-4 in dd
void schur_gcr_dd(hf_ctx *ctx, hf_hybrid *hy, const hf_gcr_opts &o, hf_gcr_info *info) {
    cudaStream_t st = ctx->stream;
    const hf_lowfactor *lf = hy->lf;
    HF_REQUIRE(lf->prec == 64, "double-double Schur complement: the factor must be FP64 (prec 64)");
    const int64_t L = hy->L, N = hy->N, n2 = hy->n2;
    info->iters = 0;
    info->max_rel_res_recursive = info->max_rel_res_true = 0.0;
    hy->dd = true;
    hy->mask1.alloc(std::max<int64_t>(L, 1), st);
    if (L > 0) mask_from_pos(ctx, L, lf->pos1.p, hy->mask1.p);
    hy->lam2.alloc(std::max<int64_t>(n2, 1), st);
    if (n2 > 0)
        HF_CUDA(cudaMemcpyAsync(hy->lam2.p, lf->perm.p + N, n2 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    precond_setup(ctx, hy->pc, lf);
    const size_t Ln = (size_t)std::max<int64_t>(L * n2, 1), nn = (size_t)std::max<int64_t>(n2 * n2, 1);
    hy->X.alloc(Ln, st);
    hy->Xlo.alloc(Ln, st);
    hy->B.alloc(Ln, st);
    hy->S22.alloc(nn, st);
    hy->S22lo.alloc(nn, st);
    if (n2 == 0) return;
    gather_K12(ctx, L, hy->K, hy->ld, hy->lam2.p, n2, hy->mask1.p, hy->B.p);   // step 2
    gather_K22(ctx, n2, hy->K, hy->ld, hy->lam2.p, hy->S22.p);
    HF_CUDA(cudaMemsetAsync(hy->S22lo.p, 0, nn * sizeof(double), st));
    GcrDD g;
    int local_st = HF_OK;
    std::string msg;
    if (N > 0) {
        try {
            block_gcr_dd(ctx, hy->K, hy->ld, L, hy->mask1.p, hy->pc, hy->B.p, n2, hy->X.p, hy->Xlo.p, o, info, g);
        } catch (const Error &e) {
            if (e.st != HF_ERR_NOT_CONVERGED && e.st != HF_ERR_BREAKDOWN) throw;
            local_st = e.st;
            msg = e.msg;
        }
        // step 4: S22 = K22 - K21 X  (K21 X = B^T X: X is zero on Lambda_2 rows), in dd
        ddgemm(ctx, true, n2, n2, L, -1.0, hy->B.p, nullptr, L, hy->X.p, hy->Xlo.p, L, true, hy->S22.p, hy->S22lo.p,
               n2, nullptr, g.w);
    } else {
        HF_CUDA(cudaMemsetAsync(hy->X.p, 0, Ln * sizeof(double), st));
        HF_CUDA(cudaMemsetAsync(hy->Xlo.p, 0, Ln * sizeof(double), st));
    }
    if (local_st != HF_OK) throw Error{(hf_status)local_st, msg};
}

// ------------------------------------------------------------------ Alg. 1 step 5 in dd
void factor_hard_dd(hf_ctx *ctx, hf_hybrid *hy, double eps_ker) {
    cudaStream_t st = ctx->stream;
    const int64_t n2 = hy->n2;
    hy->hard_done = false;
    if (n2 == 0) {
        hy->rank = hy->kernel_dim = 0;
        hy->hard_done = true;
        return;
    }
    double dref = 1.0;
    const auto &D = hy->lf->h_D64;
    if (!D.empty()) {
        dref = INFINITY;
        for (double d : D) dref = std::min(dref, std::fabs(d));
    }
    hy->perm2.alloc(n2, st);
    hy->blocks.alloc(n2, st);
    HF_CUDA(cudaMemsetAsync(hy->blocks.p, 0, n2 * sizeof(int32_t), st));
    const size_t nn = (size_t)n2 * n2;
    hy->Dh.alloc(nn, st);      // the eliminated matrix (D blocks at the pivot entries), hi
    hy->Dhlo.alloc(nn, st);
    hy->Lh.alloc(nn, st);      // L columns in label space, hi
    hy->Lhlo.alloc(nn, st);
    DBuf<int32_t> act;
    act.alloc(n2, st);
    DBuf<int64_t> rk;
    rk.alloc(1, st);
    {
        ClassTimer tm(ctx, "hard");
        k_dd_hard<<<1, 1024, 0, st>>>((int)n2, hy->S22.p, hy->S22lo.p, eps_ker * dref, hy->Dh.p, hy->Dhlo.p, hy->Lh.p,
                                       hy->Lhlo.p, act.p, hy->perm2.p, hy->blocks.p, rk.p);
        HF_CHECK_LAUNCH(ctx);
    }
    int64_t r = 0;
    HF_CUDA(cudaMemcpyAsync(&r, rk.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    hy->rank = r;
    hy->kernel_dim = n2 - r;
    hy->hard_done = true;
}

// ------------------------------------------------------------------ Alg. 2 in dd
// The scaled system K x = b (b double, original order) solved in double-double:
// y1 = K11^{-1} b1 (dd block GCR, one column), y2 = b2 - K21 y1, x2 = S22^+ y2 (dd
// Bunch-Parlett factors, kernel coordinates 0 [R16]), x1 = y1 - X12 x2; x = hi + lo.
void hybrid_solve_dd(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *xh, double *xl,
                     const hf_gcr_opts &o, hf_gcr_info *info) {
    cudaStream_t st = ctx->stream;
    const int64_t L = hy->L, N = hy->N, n2 = hy->n2;
    info->iters = 0;
    info->max_rel_res_recursive = info->max_rel_res_true = 0.0;
    if (L == 0) return;
    DBuf<double> bm, y2h, y2l, x2h, x2l;
    GcrDD g;
    if (N > 0) {
        bm.alloc(L, st);
        mask_vec(ctx, L, hy->mask1.p, b, bm.p);
        block_gcr_dd(ctx, hy->K, hy->ld, L, hy->mask1.p, hy->pc, bm.p, 1, xh, xl, o, info, g);   // step 1
    } else {
        HF_CUDA(cudaMemsetAsync(xh, 0, L * sizeof(double), st));
        HF_CUDA(cudaMemsetAsync(xl, 0, L * sizeof(double), st));
    }
    if (n2 > 0) {
        y2h.alloc(n2, st);
        y2l.alloc(n2, st);
        x2h.alloc(n2, st);
        x2l.alloc(n2, st);
        gather_rows(ctx, n2, hy->lam2.p, b, y2h.p);
        HF_CUDA(cudaMemsetAsync(y2l.p, 0, n2 * sizeof(double), st));
        ddgemm(ctx, true, n2, 1, L, -1.0, hy->B.p, nullptr, L, xh, xl, L, true, y2h.p, y2l.p, n2, nullptr, g.w);  // step 2
        DBuf<int32_t> act;
        act.alloc(n2, st);
        k_dd_hard_solve<<<1, 256, 0, st>>>((int)n2, hy->rank, hy->Dh.p, hy->Dhlo.p, hy->Lh.p, hy->Lhlo.p,
                                           hy->perm2.p, hy->blocks.p, y2h.p, y2l.p, x2h.p, x2l.p, act.p);   // step 3
        HF_CHECK_LAUNCH(ctx);
        ddgemm(ctx, false, L, 1, n2, -1.0, hy->X.p, hy->Xlo.p, L, x2h.p, x2l.p, n2, true, xh, xl, L, nullptr, g.w);   // step 4
        scatter_rows(ctx, n2, hy->lam2.p, x2h.p, xh);
        scatter_rows(ctx, n2, hy->lam2.p, x2l.p, xl);
    }
    HF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hf
