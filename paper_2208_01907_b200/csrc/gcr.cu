// gcr.cu -- host orchestration of steps a4-a8 on the context stream:
//   Alg. 1 steps 2-5 and Alg. 2, with Algorithm 5
//   (preconditioned block GCR) as the inner solver.
//
// All N x n2 blocks live in ORIGINAL row order as L x n2 arrays whose
// Lambda_2 rows are zero: the block mat-vec K11 W is then the plain dense
// product K W (K is the full scaled matrix, read contiguously by the DMMA
// GEMM) with the Lambda_2 rows of the result masked to zero, and the Gram
// products are plain column dot products.  Only the FP32 preconditioner
// works in pivot order (gather/scatter fused into its kernels).
//
// Readings [R13]: M_n = Q_n^T Q_n, A_n = Q_n^T R_n, X += P_n M_n^{-1} A_n,
// R -= Q_n M_n^{-1} A_n, G_mn = -M_m^{-1} Q_m^T Z_{n+1} for all m <= n,
// P_{n+1} = W + sum_m P_m G_mn, Q_{n+1} = Z + sum_m Q_m G_mn; convergence when
// every column's recursive ||r||_2 / ||b||_2 <= tol (one 8-byte D2H per
// iteration).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "k_dgemm.cuh"
#include "k_small.cuh"
#include "ozaki.cuh"

#include <string>
#include <vector>

namespace hf {
namespace {

struct GcrWork {
    DBuf<double> P, Q;       // L x cap*n
    int64_t cap = 0;         // blocks
    DBuf<double> Minv;       // cap * n * n
    DBuf<double> R, H, G, Mn, An, C;
    DBuf<double> bn2, rn2, res;
    DBuf<double> dgw, dgw2, chw, chdg;
    DBuf<int> status;
    std::vector<double> *hist = nullptr;   // optional: max relative residual after every iteration
    Ozaki *oz = nullptr;                   // the mat-vec on the int8 tensor cores (ozaki.cu), else DMMA
    std::unique_ptr<Ozaki> ozown;
    std::unique_ptr<Ozaki2> oz2;           // the residue form (ozaki2.cu, matvec 3)
};

// hf_gcr_opts.matvec: 3 = the residue (CRT) form of the int8 emulation (ozaki2.cu), 2 = the
// slice form (ozaki.cu), 1 = DMMA, 0 = automatic: for blocks of >= 96 columns the residue
// form, for >= 32 (or when the residues do not fit) the slice form, else DMMA, as device
// memory allows; HF_MATVEC=dmma|ozaki|ozaki2 overrides the automatic choice
void setup_matvec(hf_ctx *ctx, const double *K, int64_t ld, int64_t L, const uint8_t *mask, int64_t n,
                  const hf_gcr_opts &o, GcrWork &w) {
    if (w.oz || w.oz2) return;
    const bool dbg = getenv("HF_MATVEC_DEBUG") != nullptr;
    int mode = o.matvec;
    const bool autom = mode == 0;
    if (autom) {
        // the residue form reads 16 int8 copies of K per mat-vec, the slice form 8 (one per A
        // slice, the B slices side by side) but computes 36 products instead of 16: with few
        // columns the mat-vec is bound by those reads (C4, n = 64: residues 11.3 ms, slices
        // 8.3 ms per mat-vec; n = 512: residues 23 ms, slices 46 ms; C2 n = 256: residues)
        mode = n >= 96 ? 3 : (n >= 32 ? 2 : 1);
        if (const char *e = getenv("HF_MATVEC")) {
            if (std::string(e) == "dmma") mode = 1;
            else if (std::string(e) == "ozaki") mode = 2;
            else if (std::string(e) == "ozaki2") mode = 3;
        }
    }
    if (L == 0 || mode == 1) return;
    // the automatic choice also leaves room for the block GCR's own growth: P and Q for 16
    // blocks while the 8-block ones are still alive (grow() doubles them), plus 1 GB
    auto room = [&]() {
        auto it = ctx->matvec_room.find({L, n});
        if (it != ctx->matvec_room.end()) return it->second;
        size_t fr = 0, tot = 0;
        HF_CUDA(cudaMemGetInfo(&fr, &tot));
        const size_t need = (size_t)3 * 8 * (size_t)L * (size_t)n * 8 + ((size_t)1 << 30);
        const size_t have = fr + cached_free_bytes(ctx->device);
        if (have < need && dbg) fprintf(stderr, "[hf matvec] %zu of %zu bytes left\n", have, need);
        ctx->matvec_room[{L, n}] = have >= need;
        return have >= need;
    };
    if (mode == 3) {   // the residue form (16 int8 residue copies of K)
        w.oz2.reset(new Ozaki2());
        try {
            ozaki2_prepare(ctx, *w.oz2, K, ld, L, mask, n);
            host_trace("ozaki2_prepare");
        } catch (const Error &e) {
            if (e.st != HF_ERR_OOM || !autom) throw;
            if (dbg) fprintf(stderr, "[hf matvec] int8 residues do not fit (%s)\n", e.msg.c_str());
            w.oz2.reset();
        }
        const bool fits = w.oz2 && (!autom || room());
        host_trace("room");
        if (fits) {
            if (dbg) fprintf(stderr, "[hf matvec] int8 residues (CRT), n = %lld\n", (long long)n);
            return;
        }
        w.oz2.reset();
        mode = 2;   // the automatic choice tries the slice form (8 copies' worth) next
    }
    w.ozown.reset(new Ozaki());
    try {
        ozaki_prepare(ctx, *w.ozown, K, ld, L, mask, o.slices > 0 ? o.slices : ozaki_slices(), n);
    } catch (const Error &e) {
        // the slices take as much memory as K itself; the automatic choice falls back to
        // the DMMA product when they do not fit (e.g. C4 beside the FP32 preconditioner)
        if (e.st != HF_ERR_OOM || !autom) throw;
        if (dbg) fprintf(stderr, "[hf matvec] int8 slices do not fit (%s): DMMA\n", e.msg.c_str());
        w.ozown.reset();
        return;
    }
    if (autom && !room()) {
        if (dbg) fprintf(stderr, "[hf matvec] int8 slices: DMMA\n");
        w.ozown.reset();
        return;
    }
    w.oz = w.ozown.get();
    if (dbg) fprintf(stderr, "[hf matvec] int8 slices, n = %lld\n", (long long)n);
}

void grow(hf_ctx *ctx, GcrWork &w, int64_t L, int64_t n, int64_t need) {
    if (need <= w.cap) return;
    int64_t nc = std::max<int64_t>(need, std::max<int64_t>(8, 2 * w.cap));
    DBuf<double> P2, Q2, M2;
    P2.alloc((size_t)L * n * nc, ctx->stream);
    Q2.alloc((size_t)L * n * nc, ctx->stream);
    M2.alloc((size_t)n * n * nc, ctx->stream);
    if (w.cap > 0) {
        HF_CUDA(cudaMemcpyAsync(P2.p, w.P.p, (size_t)L * n * w.cap * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        HF_CUDA(cudaMemcpyAsync(Q2.p, w.Q.p, (size_t)L * n * w.cap * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        HF_CUDA(cudaMemcpyAsync(M2.p, w.Minv.p, (size_t)n * n * w.cap * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    w.P = std::move(P2);
    w.Q = std::move(Q2);
    w.Minv = std::move(M2);
    w.cap = nc;
}

// Z = mask o (K W)   (K11 W in original row order)
inline void matvec(hf_ctx *ctx, const double *K, int64_t ld, int64_t L, const uint8_t *mask, const double *W,
                   int64_t n, double *Z, double beta, double alpha, GcrWork &w) {
    if (w.oz) {
        ozaki_matvec(ctx, *w.oz, W, L, n, Z, L, beta, alpha);
        return;
    }
    if (w.oz2) {
        ozaki2_matvec(ctx, *w.oz2, W, L, n, Z, L, beta, alpha);
        return;
    }
    dgemm(ctx, false, L, n, L, alpha, K, ld, W, L, beta, Z, L, mask, &w.dgw);
}

double read_res(hf_ctx *ctx, GcrWork &w, int *bad) {
    double r = 0.0;
    int st = 0;
    HF_CUDA(cudaMemcpyAsync(&r, w.res.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    HF_CUDA(cudaMemcpyAsync(&st, w.status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    host_trace("residual sync");
    HF_CUDA(cudaStreamSynchronize(ctx->stream));
    host_trace("residual sync done");
    *bad = st;
    return r;
}

// Algorithm 5: solve K11 X = B (L x n, original order, Lambda_2 rows zero).
void block_gcr(hf_ctx *ctx, const double *K, int64_t ld, int64_t L, const uint8_t *mask, Precond &pc,
               const double *B, int64_t n, double *X, const hf_gcr_opts &o, hf_gcr_info *info, GcrWork &w) {
    cudaStream_t st = ctx->stream;
    setup_matvec(ctx, K, ld, L, mask, n, o, w);
    host_trace("setup_matvec");
    info->matvec = w.oz2 ? 3 : (w.oz ? 2 : 1);
    w.R.alloc((size_t)L * n, st);
    w.bn2.alloc(n, st);
    w.rn2.alloc(n, st);
    w.res.alloc(1, st);
    w.status.alloc(1, st);
    w.status.zero(st);
    w.Mn.alloc((size_t)n * n, st);
    w.An.alloc((size_t)n * n, st);
    w.C.alloc((size_t)n * n, st);
    double *R = w.R.p;

    colnorm2(ctx, L, n, B, L, w.bn2.p);
    precond_apply(ctx, pc, n, B, L, X, L);                       // find x_0: Q x_0 = b
    host_trace("precond_apply x0");
    HF_CUDA(cudaMemcpyAsync(R, B, (size_t)L * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    matvec(ctx, K, ld, L, mask, X, n, R, 1.0, -1.0, w);          // r_0 = b - A x_0
    colnorm2(ctx, L, n, R, L, w.rn2.p);
    maxres(ctx, n, w.rn2.p, w.bn2.p, w.res.p);
    int bad = 0;
    double res = read_res(ctx, w, &bad);
    if (w.hist) w.hist->push_back(res);
    int iters = 0;
    bool conv = res <= o.tol;
    if (!conv) {
        grow(ctx, w, L, n, 2);
        precond_apply(ctx, pc, n, R, L, w.P.p, L);               // p_0 = w_0 = Q^{-1} r_0
        matvec(ctx, K, ld, L, mask, w.P.p, n, w.Q.p, 0.0, 1.0, w);  // q_0 = A p_0
        for (int it = 0; it < o.max_iter; ++it) {
            const double *Pn = w.P.p + (size_t)it * n * L;
            const double *Qn = w.Q.p + (size_t)it * n * L;
            double *Minv = w.Minv.p + (size_t)it * n * n;
            dgemm2(ctx, true, n, n, L, 1.0, Qn, L, Qn, L, 0.0, w.Mn.p, n,                    // M_n
                   1.0, Qn, L, R, L, 0.0, w.An.p, n, &w.dgw, &w.dgw2);                      // A_n
            spd_inverse(ctx, n, w.Mn.p, n, Minv, w.chw, w.chdg, w.status.p);
            dgemm(ctx, false, n, n, n, 1.0, Minv, n, w.An.p, n, 0.0, w.C.p, n, nullptr, &w.dgw, 1);
            dgemm2(ctx, false, L, n, n, 1.0, Pn, L, w.C.p, n, 1.0, X, L,                      // x += p C
                   -1.0, Qn, L, w.C.p, n, 1.0, R, L, &w.dgw, &w.dgw2, 1);                     // r -= q C
            colnorm2(ctx, L, n, R, L, w.rn2.p);
            maxres(ctx, n, w.rn2.p, w.bn2.p, w.res.p);
            res = read_res(ctx, w, &bad);
            if (w.hist) w.hist->push_back(res);
            iters = it + 1;
            if (getenv("HF_GCR_DEBUG")) fprintf(stderr, "[hf gcr] n2=%lld it=%d res=%.3e bad=%d\n", (long long)n, iters, res, bad);
            if (res <= o.tol) {
                conv = true;
                break;
            }
            if (bad) {
                info->iters = iters;
                info->max_rel_res_recursive = res;
                throw Error{HF_ERR_BREAKDOWN, "block GCR: Gram matrix M_n is not positive definite"};
            }
            if (it + 1 >= o.max_iter) break;
            grow(ctx, w, L, n, it + 2);
            double *Pn1 = w.P.p + (size_t)(it + 1) * n * L;
            double *Qn1 = w.Q.p + (size_t)(it + 1) * n * L;
            const int64_t nb = (int64_t)(it + 1) * n;
            precond_apply(ctx, pc, n, R, L, Pn1, L);                       // w_{n+1}
            matvec(ctx, K, ld, L, mask, Pn1, n, Qn1, 0.0, 1.0, w);         // z_{n+1} = A w_{n+1}
            w.H.alloc((size_t)nb * n, st);
            w.G.alloc((size_t)nb * n, st);
            dgemm(ctx, true, nb, n, L, 1.0, w.Q.p, L, Qn1, L, 0.0, w.H.p, nb, nullptr, &w.dgw);   // Q_m^T z
            for (int m = 0; m <= it; ++m)                                   // G_m = -M_m^{-1} Q_m^T z
                dgemm(ctx, false, n, n, n, -1.0, w.Minv.p + (size_t)m * n * n, n, w.H.p + (size_t)m * n, nb, 0.0,
                      w.G.p + (size_t)m * n, nb, nullptr, &w.dgw, 1);
            dgemm2(ctx, false, L, n, nb, 1.0, w.P.p, L, w.G.p, nb, 1.0, Pn1, L,               // p_{n+1}
                   1.0, w.Q.p, L, w.G.p, nb, 1.0, Qn1, L, &w.dgw, &w.dgw2);                   // q_{n+1}
        }
    }
    info->iters = iters;
    info->max_rel_res_recursive = res;
    // true residual ||B - K11 X|| / ||B|| (reported)
    HF_CUDA(cudaMemcpyAsync(R, B, (size_t)L * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    matvec(ctx, K, ld, L, mask, X, n, R, 1.0, -1.0, w);
    colnorm2(ctx, L, n, R, L, w.rn2.p);
    maxres(ctx, n, w.rn2.p, w.bn2.p, w.res.p);
    info->max_rel_res_true = read_res(ctx, w, &bad);
    if (!conv) throw Error{HF_ERR_NOT_CONVERGED, "block GCR reached max_iter"};
}

}  // namespace

// ------------------------------------------------------------------ Alg. 3 (IR) and the comparison
// Algorithm 3, mixed-precision iterative refinement on the same
// kernels: x_0 = Q^{-1} b, r = b - A x, repeat e = Q^{-1} r, x += e, r = b - A x
// (A = K11 in original row order); all columns at once, stop when every column's
// ||r||_2 / ||b||_2 <= tol.
void iterative_refinement(hf_ctx *ctx, const double *K, int64_t ld, int64_t L, const uint8_t *mask, Precond &pc,
                          const double *B, int64_t n, double *X, const hf_gcr_opts &o, hf_gcr_info *info,
                          GcrWork &w) {
    cudaStream_t st = ctx->stream;
    setup_matvec(ctx, K, ld, L, mask, n, o, w);
    host_trace("setup_matvec");
    info->matvec = w.oz2 ? 3 : (w.oz ? 2 : 1);
    w.R.alloc((size_t)L * n, st);
    w.bn2.alloc(n, st);
    w.rn2.alloc(n, st);
    w.res.alloc(1, st);
    w.status.alloc(1, st);
    w.status.zero(st);
    DBuf<double> E;
    E.alloc((size_t)L * n, st);
    colnorm2(ctx, L, n, B, L, w.bn2.p);
    precond_apply(ctx, pc, n, B, L, X, L);                                // steps 1-2
    int bad = 0, iters = 0;
    double res = 0.0;
    for (;;) {
        HF_CUDA(cudaMemcpyAsync(w.R.p, B, (size_t)L * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        matvec(ctx, K, ld, L, mask, X, n, w.R.p, 1.0, -1.0, w);           // r = b - A x
        colnorm2(ctx, L, n, w.R.p, L, w.rn2.p);
        maxres(ctx, n, w.rn2.p, w.bn2.p, w.res.p);
        res = read_res(ctx, w, &bad);
        if (w.hist) w.hist->push_back(res);
        if (res <= o.tol || iters >= o.max_iter) break;
        precond_apply(ctx, pc, n, w.R.p, L, E.p, L);                      // e = Q^{-1} r
        axpy_cols(ctx, L, n, 1.0, E.p, L, X, L);                           // x += e
        ++iters;
    }
    info->iters = iters;
    info->max_rel_res_recursive = info->max_rel_res_true = res;
    if (res > o.tol) throw Error{HF_ERR_NOT_CONVERGED, "iterative refinement reached max_iter"};
}

// ------------------------------------------------------------------ Alg. 1 steps 2-4
// Multi-GPU (stage 2): the n2 right-hand sides (columns of K12)
// are split into contiguous slices, one per rank (hf_shard_cols); every rank
// runs its own block GCR on its slice and forms S22[:, slice] = K22[:, slice]
// - K21 X[:, slice]; the slices of S22 and X are then broadcast from their
// owners in one NCCL group (ncclBroadcast per rank: unequal slice widths, no
// padding), and the GCR statistics are max-reduced.  Errors of one rank are
// carried through the collectives (no rank leaves early) and raised after.
// A "virtual" rank set with hf_set_virtual_rank computes only its slice and
// leaves the other columns zero (single-GPU emulation of one rank, no
// collective).
void schur_gcr(hf_ctx *ctx, hf_hybrid *hy, const hf_gcr_opts &o, hf_gcr_info *info) {
    cudaStream_t st = ctx->stream;
    const hf_lowfactor *lf = hy->lf;
    const int64_t L = hy->L, N = hy->N, n2 = hy->n2;
    info->iters = 0;
    info->max_rel_res_recursive = info->max_rel_res_true = 0.0;
    hy->mask1.alloc(std::max<int64_t>(L, 1), st);
    if (L > 0) mask_from_pos(ctx, L, lf->pos1.p, hy->mask1.p);
    hy->lam2.alloc(std::max<int64_t>(n2, 1), st);
    if (n2 > 0)
        HF_CUDA(cudaMemcpyAsync(hy->lam2.p, lf->perm.p + N, n2 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    host_trace("schur_gcr start");
    precond_setup(ctx, hy->pc, lf);
    host_trace("precond_setup");
    hy->X.alloc((size_t)std::max<int64_t>(L * n2, 1), st);
    hy->B.alloc((size_t)std::max<int64_t>(L * n2, 1), st);
    hy->S22.alloc((size_t)std::max<int64_t>(n2 * n2, 1), st);
    if (n2 == 0) return;
    gather_K12(ctx, L, hy->K, hy->ld, hy->lam2.p, n2, hy->mask1.p, hy->B.p);   // step 2
    gather_K22(ctx, n2, hy->K, hy->ld, hy->lam2.p, hy->S22.p);
    hy->nonsym = lf->nonsym;
    if (hy->nonsym) {   // NEXT-3: the actual K21 (K21 != K12^T)
        hy->B2.alloc((size_t)L * n2, st);
        gather_K21T(ctx, L, hy->K, hy->ld, hy->lam2.p, n2, hy->mask1.p, hy->B2.p);
    }
    const double *K21T = hy->nonsym ? hy->B2.p : hy->B.p;
    const bool virt = ctx->vnranks > 0;
    const int nr = virt ? ctx->vnranks : ctx->nranks, rk = virt ? ctx->vrank : ctx->rank;
    int64_t c0 = 0, c1 = n2;
    shard_cols(n2, nr, rk, &c0, &c1);
    const int64_t ns = c1 - c0;
    if (nr > 1) HF_CUDA(cudaMemsetAsync(hy->X.p, 0, (size_t)L * n2 * sizeof(double), st));
    int local_st = HF_OK;
    std::string local_msg;
    if (N > 0 && ns > 0) {
        GcrWork w;
        try {
            block_gcr(ctx, hy->K, hy->ld, L, hy->mask1.p, hy->pc, hy->B.p + c0 * L, ns, hy->X.p + c0 * L, o, info,
                      w);                                                                           // step 3
        } catch (const Error &e) {
            if (e.st != HF_ERR_NOT_CONVERGED && e.st != HF_ERR_BREAKDOWN) throw;   // CUDA errors: unrecoverable
            local_st = e.st;
            local_msg = e.msg;
        }
        // step 4: S22[:, slice] = K22[:, slice] - K21 X[:, slice]  (K21 X = B^T X: X is zero on Lambda_2 rows)
        dgemm(ctx, true, n2, ns, L, -1.0, K21T, L, hy->X.p + c0 * L, L, 1.0, hy->S22.p + c0 * n2, n2, nullptr,
              &w.dgw);
    } else if (N == 0) {
        HF_CUDA(cudaMemsetAsync(hy->X.p, 0, (size_t)L * n2 * sizeof(double), st));
    }
    if (virt && nr > 1) {
        // single-GPU emulation of rank rk: the other ranks' columns of S22 are not computed
        if (c0 > 0) HF_CUDA(cudaMemsetAsync(hy->S22.p, 0, (size_t)c0 * n2 * sizeof(double), st));
        if (c1 < n2) HF_CUDA(cudaMemsetAsync(hy->S22.p + c1 * n2, 0, (size_t)(n2 - c1) * n2 * sizeof(double), st));
    }
#ifdef HF_WITH_NCCL
    if (!virt && ctx->comm) {   // (also with one rank: the same NCCL path, trivially)
        DBuf<double> red;
        red.alloc(4, st);
        double h[4] = {(double)info->iters, info->max_rel_res_recursive, info->max_rel_res_true, (double)local_st};
        HF_CUDA(cudaMemcpyAsync(red.p, h, sizeof(h), cudaMemcpyHostToDevice, st));
        collective_begin(ctx);
        for (int r = 0; r < nr; ++r) {
            int64_t a0, a1;
            shard_cols(n2, nr, r, &a0, &a1);
            if (a1 == a0) continue;
            collective_bcast(ctx, hy->S22.p + a0 * n2, (size_t)(a1 - a0) * n2, r);
            collective_bcast(ctx, hy->X.p + a0 * L, (size_t)(a1 - a0) * L, r);
        }
        collective_max(ctx, red.p, 4);
        collective_end(ctx);
        HF_CUDA(cudaMemcpyAsync(h, red.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        HF_CUDA(cudaStreamSynchronize(st));
        info->iters = (int32_t)h[0];
        info->max_rel_res_recursive = h[1];
        info->max_rel_res_true = h[2];
        if (local_st == HF_OK && (int)h[3] != HF_OK) {
            local_st = (int)h[3];
            local_msg = "block GCR failed on another rank";
        }
    }
#endif
    if (local_st != HF_OK) throw Error{(hf_status)local_st, local_msg};
}

// ------------------------------------------------------------------ Alg. 1 step 5
void factor_hard(hf_ctx *ctx, hf_hybrid *hy, double eps_ker) {
    cudaStream_t st = ctx->stream;
    const int64_t n2 = hy->n2;
    hy->hard_done = false;
    if (n2 == 0) {
        hy->rank = hy->kernel_dim = 0;
        hy->hard_done = true;
        return;
    }
    double dref = 1.0;
    if (hy->lf->prec == 64) {
        const auto &D = hy->lf->h_D64;
        if (!D.empty()) {
            dref = INFINITY;
            for (double d : D) dref = std::min(dref, std::fabs(d));
        }
    } else {
        const auto &D = hy->lf->h_D;
        if (!D.empty()) {
            dref = INFINITY;
            for (float d : D) dref = std::min(dref, std::fabs((double)d));
        }
    }
    if (hy->nonsym) {   // NEXT-3: LU with complete pivoting (the 1x1 / 2x2 symmetric pivots do not apply)
        hy->LUh.alloc((size_t)n2 * n2, st);
        hy->perm2.alloc(n2, st);
        hy->pcol2.alloc(n2, st);
        hy->blocks.alloc(n2, st);
        HF_CUDA(cudaMemsetAsync(hy->blocks.p, 0, n2 * sizeof(int32_t), st));
        DBuf<int64_t> rk;
        rk.alloc(1, st);
        hard_lu(ctx, n2, hy->S22.p, eps_ker * dref, hy->LUh.p, hy->perm2.p, hy->pcol2.p, rk.p);
        int64_t r = 0;
        HF_CUDA(cudaMemcpyAsync(&r, rk.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        HF_CUDA(cudaStreamSynchronize(st));
        hy->rank = r;
        hy->kernel_dim = n2 - r;
        hy->hard_done = true;
        return;
    }
    hy->Lh.alloc((size_t)n2 * n2, st);
    hy->Dh.alloc((size_t)n2 * n2, st);
    hy->perm2.alloc(n2, st);
    hy->blocks.alloc(n2, st);
    DBuf<double> A;
    A.alloc((size_t)n2 * n2, st);
    DBuf<int64_t> rk;
    rk.alloc(1, st);
    hard_factor(ctx, n2, hy->S22.p, eps_ker * dref, A.p, hy->Lh.p, hy->Dh.p, hy->perm2.p, hy->blocks.p, rk.p);
    int64_t r = 0;
    HF_CUDA(cudaMemcpyAsync(&r, rk.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    hy->rank = r;
    hy->kernel_dim = n2 - r;
    hy->hard_done = true;
}

// ------------------------------------------------------------------ Alg. 2
void hybrid_solve(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *x, const hf_gcr_opts &o,
                  hf_gcr_info *info) {
    cudaStream_t st = ctx->stream;
    const int64_t L = hy->L, N = hy->N, n2 = hy->n2;
    info->iters = 0;
    info->max_rel_res_recursive = info->max_rel_res_true = 0.0;
    if (L == 0) return;
    DBuf<double> bm, y1, y2, x2, z;
    y1.alloc(L, st);
    if (N > 0) {
        bm.alloc(L, st);
        mask_vec(ctx, L, hy->mask1.p, b, bm.p);
        GcrWork w;
        block_gcr(ctx, hy->K, hy->ld, L, hy->mask1.p, hy->pc, bm.p, 1, y1.p, o, info, w);   // step 1
    } else {
        HF_CUDA(cudaMemsetAsync(y1.p, 0, L * sizeof(double), st));
    }
    HF_CUDA(cudaMemcpyAsync(x, y1.p, L * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (n2 > 0) {
        y2.alloc(n2, st);
        x2.alloc(n2, st);
        z.alloc(n2, st);
        DBuf<double> dg;
        gather_rows(ctx, n2, hy->lam2.p, b, y2.p);
        dgemm(ctx, true, n2, 1, L, -1.0, hy->nonsym ? hy->B2.p : hy->B.p, L, y1.p, L, 1.0, y2.p, n2, nullptr,
              &dg);                                                                                   // step 2
        if (hy->nonsym)
            hard_lu_solve(ctx, n2, hy->rank, hy->LUh.p, hy->perm2.p, hy->pcol2.p, y2.p, x2.p, z.p);   // step 3
        else
            hard_solve(ctx, n2, hy->rank, hy->Lh.p, hy->Dh.p, hy->perm2.p, hy->blocks.p, y2.p, x2.p, z.p);
        dgemm(ctx, false, L, 1, n2, -1.0, hy->X.p, L, x2.p, n2, 1.0, x, L, nullptr, &dg, 1);   // step 4
        scatter_rows(ctx, n2, hy->lam2.p, x2.p, x);
    }
    HF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hf

extern "C" hf_status hf_hybrid_export(hf_ctx *ctx, const hf_hybrid *hy, double *X, int64_t ldx, double *S22,
                                      int64_t lds) {
    if (!ctx || !hy) return HF_ERR_INVALID_ARG;
    try {
        const int64_t N = hy->N, n2 = hy->n2;
        if (X && N > 0 && n2 > 0) {
            if (ldx < N) throw hf::Error{HF_ERR_INVALID_ARG, "hf_hybrid_export: ldx < N"};
            hf::gather_block_rows(ctx, N, n2, hy->lf->perm.p, hy->X.p, hy->L, X, ldx);
        }
        if (S22 && n2 > 0) {
            if (lds < n2) throw hf::Error{HF_ERR_INVALID_ARG, "hf_hybrid_export: lds < n2"};
            HF_CUDA(cudaMemcpy2DAsync(S22, lds * sizeof(double), hy->S22.p, n2 * sizeof(double), n2 * sizeof(double),
                                      n2, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (const hf::Error &e) {
        ctx->last_error = e.msg;
        return e.st;
    }
    return HF_OK;
}

// ------------------------------------------------------------------ Fig. 2 comparison
// hf_krylov_solve (include/hf.h): K11 X = B by Algorithm 3 (IR), Algorithm 4 (GCR,
// one column at a time) or Algorithm 5 (block GCR), with the FP32 preconditioner
// of lf; the maximum relative residual after every iteration goes to hist_host.
extern "C" hf_status hf_krylov_solve(hf_ctx *ctx, const double *K, int64_t ld, const hf_lowfactor *lf, int method,
                                     int64_t ncol, const double *B, double *X, double tol, int32_t max_iter,
                                     int32_t *iters_host, double *hist_host, int32_t hist_len) {
    if (!ctx || !lf) return HF_ERR_INVALID_ARG;
    hf::DeviceGuard dg(ctx);
    try {
        const int64_t L = lf->L;
        if (!(method >= 0 && method <= 2) || ncol < 0 || ld < L || tol <= 0.0 || max_iter < 1 ||
            (ncol > 0 && L > 0 && (!K || !B || !X)))
            throw hf::Error{HF_ERR_INVALID_ARG, "hf_krylov_solve: bad arguments"};
        if (iters_host) *iters_host = 0;
        if (ncol == 0 || L == 0 || lf->N == 0) return HF_OK;
        cudaStream_t st = ctx->stream;
        hf::DBuf<uint8_t> mask;
        mask.alloc(L, st);
        hf::mask_from_pos(ctx, L, lf->pos1.p, mask.p);
        hf::Precond pc;
        hf::precond_setup(ctx, pc, lf);
        hf::DBuf<double> Bm;
        Bm.alloc((size_t)L * ncol, st);
        for (int64_t c = 0; c < ncol; ++c) hf::mask_vec(ctx, L, mask.p, B + c * L, Bm.p + c * L);
        hf_gcr_opts o{tol, max_iter, 0, 0};
        hf_gcr_info info{0, 0.0, 0.0, 0};
        std::vector<double> hist;
        int32_t iters = 0;
        hf_status fail = HF_OK;
        std::string fail_msg;
        auto run = [&](auto &&f) {   // outputs are filled even when the solver does not converge
            try {
                f();
            } catch (const hf::Error &e) {
                if (e.st != HF_ERR_NOT_CONVERGED && e.st != HF_ERR_BREAKDOWN) throw;
                fail = e.st;
                fail_msg = e.msg;
            }
        };
        if (method == 0) {
            hf::GcrWork w;
            w.hist = &hist;
            run([&] { hf::iterative_refinement(ctx, K, ld, L, mask.p, pc, Bm.p, ncol, X, o, &info, w); });
            iters = info.iters;
        } else if (method == 2) {
            hf::GcrWork w;
            w.hist = &hist;
            run([&] { hf::block_gcr(ctx, K, ld, L, mask.p, pc, Bm.p, ncol, X, o, &info, w); });
            iters = info.iters;
        } else {
            // Algorithm 4 column by column; the history is the max over columns per iteration
            std::vector<double> hmax;
            for (int64_t c = 0; c < ncol; ++c) {
                hf::GcrWork w;
                std::vector<double> h1;
                w.hist = &h1;
                run([&] { hf::block_gcr(ctx, K, ld, L, mask.p, pc, Bm.p + c * L, 1, X + c * L, o, &info, w); });
                iters = std::max(iters, info.iters);
                if (hmax.size() < h1.size()) hmax.resize(h1.size(), 0.0);
                for (size_t q = 0; q < h1.size(); ++q) hmax[q] = std::max(hmax[q], h1[q]);
                for (size_t q = h1.size(); q < hmax.size(); ++q) hmax[q] = std::max(hmax[q], h1.empty() ? 0.0 : h1.back());
            }
            hist = hmax;
        }
        if (iters_host) *iters_host = iters;
        if (hist_host)
            for (int32_t q = 0; q < hist_len; ++q) hist_host[q] = q < (int32_t)hist.size() ? hist[q] : -1.0;
        HF_CUDA(cudaStreamSynchronize(st));
        if (fail != HF_OK) throw hf::Error{fail, fail_msg};
    } catch (const hf::Error &e) {
        ctx->last_error = e.msg;
        return e.st;
    }
    return HF_OK;
}
