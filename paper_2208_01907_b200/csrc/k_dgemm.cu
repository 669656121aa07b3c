// k_dgemm.cu -- FP64 GEMM on the legacy FP64 tensor path (DMMA m8n8k4 via
// mma.sync; tcgen05 has no f64 kind on sm_100), used for every FP64
// contraction of steps a5/a6 (Alg. 5, Alg. 1 step 4 P:191):
//   K11 W (the block mat-vec, "SpMM in higher precision"),
//   Gram blocks Q^T Q, Q^T R, Q^T Z, the n2 x n2 coefficient products, the
//   block updates X += P C etc., and S22 = K22 - K21 X.
//
//   C[M x N] = beta * C + alpha * rowmask o (op(A) B),  column-major,
//   op(A) = A (M x K, lda) or A^T (A stored K x M, lda);  B: K x N (ldb).
// Split-K writes deterministic partial tiles that k_reduce sums in order.
//
// CTA tile 64x64x16, 4 warps (2x2, 32x32 each = 4x4 DMMA tiles), 3-stage
// cp.async pipeline; shared layouts [k][m+4] / [k][n+4] make the DMMA
// fragment loads bank-conflict free (8-byte words, 16 pairs per half warp).
#include <algorithm>
#include <cmath>

#include "hf_internal.cuh"
#include "k_dgemm.cuh"

namespace hf {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4, STAGES = 3;
constexpr int SA = BM + PAD, SB = BN + PAD;
constexpr int STAGE_ELEMS = BK * SA + BK * SB;

__device__ __forceinline__ void cp_async8(double *smem_dst, const double *gsrc, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int n = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// up to two problems of the same shape in one launch (blockIdx.z = problem * splits + split)
struct DgemmBatch {
    DgemmArgs g[2];
    int splits;
};

template <bool TRANS_A>
__global__ void __launch_bounds__(128) k_dgemm(DgemmBatch gb) {
    extern __shared__ __align__(16) double sm[];
    const int zs = (int)blockIdx.z % gb.splits, nsplit = gb.splits;
    const DgemmArgs g = ((int)blockIdx.z >= gb.splits) ? gb.g[1] : gb.g[0];   // no dynamic param indexing
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    // grid.x = N tiles (fastest): the N tiles of one M tile run side by side, so each A
    // (= K11) tile comes from DRAM once and from L2 for the other N tiles
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    // K range of this split
    const int64_t kper = ((g.K + nsplit - 1) / nsplit + BK - 1) / BK * BK;
    const int64_t kbeg = (int64_t)zs * kper;
    const int64_t kend = min(g.K, kbeg + kper);
    const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

    auto load_tile = [&](int stage, int kt) {
        double *As = sm + stage * STAGE_ELEMS;
        double *Bs = As + BK * SA;
        const int64_t k0 = kbeg + (int64_t)kt * BK;
        // A: 64 x 16 elements, 8 per thread
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int e = tid + q * 128;
            int mm, kk;
            if (!TRANS_A) { mm = e & 63; kk = e >> 6; }      // column k contiguous in m
            else { kk = e & 15; mm = e >> 4; }                // row m of A^T contiguous in k
            const int64_t gm = m0 + mm, gk = k0 + kk;
            const bool ok = gm < g.M && gk < kend;
            const double *src = g.A + (ok ? (TRANS_A ? gk + gm * g.lda : gm + gk * g.lda) : 0);
            cp_async8(&As[kk * SA + mm], src, ok);
        }
        // B: 16 x 64, column n contiguous in k
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int e = tid + q * 128;
            const int kk = e & 15, nn = e >> 4;
            const int64_t gn = n0 + nn, gk = k0 + kk;
            const bool ok = gn < g.N && gk < kend;
            const double *src = g.B + (ok ? gk + gn * g.ldb : 0);
            cp_async8(&Bs[kk * SB + nn], src, ok);
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ntiles) load_tile(s, s);
        cp_commit();
    }
    const int ar = lane >> 2, ak = lane & 3;
    for (int kt = 0; kt < ntiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nxt = kt + STAGES - 1;
            if (nxt < ntiles) load_tile(nxt % STAGES, nxt);
            cp_commit();
        }
        const double *As = sm + (kt % STAGES) * STAGE_ELEMS;
        const double *Bs = As + BK * SA;
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[(k4 + ak) * SA + wm * 32 + i * 8 + ar];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[(k4 + ak) * SB + wn * 32 + j * 8 + ar];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_wait<0>();

    // epilogue: fragment (row = lane/4, cols 2*(lane%4) + {0,1})
    const bool partial = nsplit > 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gm = m0 + wm * 32 + i * 8 + (lane >> 2);
        if (gm >= g.M) continue;
        const bool keep = !g.rowmask || g.rowmask[gm];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gn = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
                if (gn >= g.N) continue;
                if (partial) {
                    g.W[(size_t)zs * g.M * g.N + gm + gn * g.M] = acc[i][j][h];
                } else {
                    double *c = g.C + gm + gn * g.ldc;
                    const double ab = keep ? __dmul_rn(g.alpha, acc[i][j][h]) : 0.0;
                    *c = (g.beta == 0.0) ? ab : fma(g.beta, *c, ab);
                }
            }
        }
    }
}

__global__ void k_reduce(DgemmArgs g, int splits) {
    const int64_t total = g.M * g.N;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gm = e % g.M, gn = e / g.M;
        // the partials are summed in split order (deterministic); their loads are issued
        // eight at a time ahead of the adds so their latencies overlap
        double s = 0.0;
        int z = 0;
        for (; z + 8 <= splits; z += 8) {
            double w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = __ldcs(&g.W[(size_t)(z + u) * total + e]);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += w[u];
        }
        for (; z < splits; ++z) s += __ldcs(&g.W[(size_t)z * total + e]);
        const bool keep = !g.rowmask || g.rowmask[gm];
        double *c = g.C + gm + gn * g.ldc;
        const double ab = keep ? __dmul_rn(g.alpha, s) : 0.0;
        *c = (g.beta == 0.0) ? ab : fma(g.beta, *c, ab);
    }
}

}  // namespace

static void dgemm_launch(hf_ctx *ctx, bool transA, int nprob, const DgemmArgs *gs, DBuf<double> *const *work,
                         int splits) {
    const int64_t M = gs[0].M, N = gs[0].N, K = gs[0].K;
    if (M <= 0 || N <= 0) return;
    cudaStream_t st = ctx->stream;
    const int64_t mt = cdiv(M, BM), nt = cdiv(N, BN);
    const size_t shm0 = (size_t)STAGES * STAGE_ELEMS * sizeof(double);
    static DevState per_sm_dev(0);   // per device: kernel attributes apply per device context
    int &per_sm = per_sm_dev[ctx->device];
    if (!per_sm) {
        HF_CUDA(cudaFuncSetAttribute(k_dgemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm0));
        HF_CUDA(cudaFuncSetAttribute(k_dgemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm0));
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dgemm<false>, 128, shm0));
        per_sm = std::max(1, per_sm);
    }
    if (splits <= 0) {
        // wave-aware split-K: among splits whose depth is >= 256, take the one whose CTA count
        // fills the last wave best (the plain 1024-tile mat-vec fills 1.73 waves of 592 CTA
        // slots -> 87 %; 4 splits give 6.92 waves -> 99 %); ties -> fewer splits
        const int64_t slots = (int64_t)per_sm * ctx->num_sms;
        const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(16, K / 256));
        double best = -1.0;
        splits = 1;
        for (int64_t sp = 1; sp <= smax; ++sp) {
            const double w = (double)(mt * nt * sp * nprob) / (double)slots;
            const double eff = w / std::ceil(w);
            if (eff > best + 0.02) {
                best = eff;
                splits = (int)sp;
            }
        }
    }
    if (K == 0) splits = 1;
    DgemmBatch gb;
    gb.splits = splits;
    for (int b = 0; b < nprob; ++b) {
        gb.g[b] = gs[b];
        if (splits > 1) {
            work[b]->alloc((size_t)splits * M * N, st);
            gb.g[b].W = work[b]->p;
        }
    }
    if (nprob == 1) gb.g[1] = gb.g[0];
    const size_t shm = shm0;
    ClassTimer tm(ctx, "dgemm", st, 2.0 * (double)M * (double)N * (double)K * nprob,
                  8.0 * nprob * ((double)M * K + (double)K * N + 2.0 * (double)M * N));
    HF_REQUIRE(mt <= 65535, "dgemm: too many row tiles for grid.y");
    dim3 grid((unsigned)nt, (unsigned)mt, (unsigned)(splits * nprob));
    if (transA) k_dgemm<true><<<grid, 128, shm, st>>>(gb);
    else k_dgemm<false><<<grid, 128, shm, st>>>(gb);
    HF_CHECK_LAUNCH(ctx);
    if (splits > 1) {
        const int64_t total = M * N;
        for (int b = 0; b < nprob; ++b) {
            k_reduce<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 4096), 256, 0, st>>>(gb.g[b], splits);
            HF_CHECK_LAUNCH(ctx);
        }
    }
}

void dgemm(hf_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
           int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
           const uint8_t *rowmask, DBuf<double> *work, int splits) {
    const DgemmArgs g{M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, rowmask, nullptr};
    DBuf<double> *w[1] = {work};
    dgemm_launch(ctx, transA, 1, &g, w, splits);
}

void dgemm2(hf_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha0, const double *A0,
            int64_t lda0, const double *B0, int64_t ldb0, double beta0, double *C0, int64_t ldc0, double alpha1,
            const double *A1, int64_t lda1, const double *B1, int64_t ldb1, double beta1, double *C1, int64_t ldc1,
            DBuf<double> *work0, DBuf<double> *work1, int splits) {
    const DgemmArgs g[2] = {{M, N, K, alpha0, A0, lda0, B0, ldb0, beta0, C0, ldc0, nullptr, nullptr},
                            {M, N, K, alpha1, A1, lda1, B1, ldb1, beta1, C1, ldc1, nullptr, nullptr}};
    DBuf<double> *w[2] = {work0, work1};
    dgemm_launch(ctx, transA, 2, g, w, splits);
}

}  // namespace hf
