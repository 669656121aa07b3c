// k_trsm_blk.cu -- the lower-precision preconditioner Q^{-1} = L^{-T} D^{-1} L^{-1} of
// P:242 / P:506 ("forward/backward substitution in lower precision ... BLAS level 3
// TRSM") as a BLOCKED solve whose work is tensor-core GEMMs:
//
//   forward  L Y = R:  for j = 0..nb-1:  Y_j = Linv_j R_j;   R_{>j} -= L_{>j,j} Y_j
//   Z = D^{-1} Y
//   backward L^T X = Z: for j = nb-1..0: X_j = Linv_j^T Z_j; Z_{<j} -= (L_{j,<j})^T X_j
//
// with blocks of BS = 2048 rows (nb = 8 at C2), Linv_j the inverse of the unit lower
// diagonal block L_jj (formed once per factorization by recursive doubling from the
// 64 x 64 inverses: inv([A 0; C B]) = [A^-1 0; -B^-1 C A^-1  B^-1], FP32 GEMMs), and
// every product in FP32 precision on the BF16 tensor cores by an exact three-way split
// x = x1 + x2 + x3 (x1 = RN_bf16(x), x2 = RN_bf16(x - x1), x3 = x - x1 - x2: 3 x 8 bits
// hold FP32's 24 exactly) and the six products with i + j <= 4:
//   A B ~= A1 B1 + (A1 B2 + A2 B1) + (A1 B3 + A3 B1 + A2 B2)   (FP32 accumulation,
//   summed from the smallest; the dropped A2 B3 + A3 B2 + A3 B3 are ~2^-25 |A||B|, below
//   FP32's unit roundoff; an exactly representable identity block stays exact).
// The sequential chain of the substitution is nb GEMM pairs per direction instead
// of N / 64 dependent 64-row links (k_trsm.cu), and the products run at tensor-core
// rate.  Any summation order is allowed for the preconditioner [R12]; the L factor
// and D are the FP32 ones of stage 1, pivot order, unchanged.
//
// Operand layouts (column-major, ld Nb = nb BS; L padded with the identity):
//   L1..L3  Nb x Nb bf16 parts, only the tiles on / below the diagonal are read;
//   I1..I3  block j's BS x BS inverse at j BS (BS + 1) with ld BS (the FP32 inverse is
//           built there first: the diagonal offset g of any doubling pair maps to
//           g (BS + 1), so the pairs of one level across all blocks form ONE strided
//           batched GEMM);
//   X, Y (FP32), S1..S3 (bf16 parts of the current block)  Nb x ncp, the right-hand
//           sides in pivot order (ncp = ncol rounded to 8).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "k_dgemm.cuh"
#include "lt.cuh"

using bf16 = __nv_bfloat16;

namespace hf {
namespace {

// x = p1 + p2 + p3 exactly, each a bfloat16 (round to nearest at every step)
__device__ __forceinline__ void split3(float x, bf16 &p1, bf16 &p2, bf16 &p3) {
    p1 = __float2bfloat16_rn(x);
    const float r = x - __bfloat162float(p1);   // exact
    p2 = __float2bfloat16_rn(r);
    p3 = __float2bfloat16_rn(r - __bfloat162float(p2));   // exact: at most 8 bits remain
}

// Lp (Nb x Nb) = Lfac (N x N, ld N) padded with the identity; lower 32 x 32 tiles only
__global__ void __launch_bounds__(256) k_blk_pad(int64_t N, int64_t Nb, const float *__restrict__ Lf,
                                                 float *__restrict__ Lp) {
    if (blockIdx.x < blockIdx.y) return;
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int q = ty; q < 32; q += 8) {
        const int64_t i = i0 + tx, j = j0 + q;
        Lp[i + j * Nb] = (i < N && j < N) ? Lf[i + j * N] : (i == j ? 1.f : 0.f);
    }
}

// inverse of each 64 x 64 unit lower diagonal block of Lp into the packed Inv (column j of
// the inverse by forward substitution, one thread per column)
__global__ void __launch_bounds__(64) k_blk_inv64(int64_t Nb, const float *__restrict__ Lp, int64_t BS,
                                                  float *__restrict__ Inv) {
    __shared__ float Ls[64][65], Xs[64][65];
    const int64_t r0 = (int64_t)blockIdx.x * 64;
    const int j = threadIdx.x;
    for (int i = 0; i < 64; ++i) Ls[i][j] = Lp[(r0 + i) + (r0 + j) * Nb];
    __syncthreads();
    for (int i = 0; i < 64; ++i) {
        float s = (i == j) ? 1.f : 0.f;
        if (i > j)
            for (int k = j; k < i; ++k) s = __fmaf_rn(-Ls[i][k], Xs[k][j], s);
        Xs[i][j] = (i < j) ? 0.f : s;
    }
    __syncthreads();
    float *dst = Inv + r0 * (BS + 1);   // diagonal offset r0 -> packed r0 (BS + 1)
    for (int i = 0; i < 64; ++i) dst[i + (int64_t)j * BS] = Xs[i][j];
}

// n elements of x -> the three bf16 parts
__global__ void k_blk_split_all(int64_t n, const float *__restrict__ x, bf16 *__restrict__ p1, bf16 *__restrict__ p2,
                                bf16 *__restrict__ p3) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        split3(x[e], p1[e], p2[e], p3[e]);
}

// the lower 32 x 32 tiles of the Nb x Nb matrix x -> the three bf16 parts
__global__ void __launch_bounds__(256) k_blk_split_lower(int64_t Nb, const float *__restrict__ x,
                                                         bf16 *__restrict__ p1, bf16 *__restrict__ p2,
                                                         bf16 *__restrict__ p3) {
    if (blockIdx.x < blockIdx.y) return;
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int q = ty; q < 32; q += 8) {
        const int64_t e = (i0 + tx) + (j0 + q) * Nb;
        split3(x[e], p1[e], p2[e], p3[e]);
    }
}

// rows [r0, r0 + nr) x ncp columns of X (+ X2 if given; ld) -> the parts (same positions)
__global__ void k_blk_split_rows(int64_t r0, int64_t nr, int64_t ncp, const float *__restrict__ X,
                                 const float *__restrict__ X2, int64_t ld, bf16 *__restrict__ p1,
                                 bf16 *__restrict__ p2, bf16 *__restrict__ p3) {
    const int64_t total = nr * ncp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = (r0 + e % nr) + (e / nr) * ld;
        split3(X2 ? X[q] + X2[q] : X[q], p1[q], p2[q], p3[q]);
    }
}

// C (BS x ncp, ld ldc) = alpha (P0 + P1 + ... + P5) + beta C, the six part products of a
// small product in their SMALL order (smallest first), summed in IEEE FP32 in that order
__global__ void __launch_bounds__(256) k_blk_sum6(int64_t BS, int64_t ncp, const float *__restrict__ P, float alpha,
                                                  float beta, float *__restrict__ C, int64_t ldc) {
    const int64_t per = BS * ncp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (int64_t)gridDim.x * blockDim.x) {
        float v = P[e];
#pragma unroll
        for (int q = 1; q < 6; ++q) v += P[e + q * per];
        float *c = C + (e % BS) + (e / BS) * ldc;
        *c = beta == 0.f ? alpha * v : fmaf(beta, *c, alpha * v);
    }
}

// Part orders of the K-concatenated products.  The six part products with i + j <= 4 as ONE
// GEMM over K' = 6 BS:  [A3 A1 A2 A2 A1 A1] . [B1; B3; B2; B1; B2; B1]  (SMALL order, for the
// latency-critical diagonal-inverse and coupling products, whose A operands are stored with
// their parts duplicated), or as three GEMMs over the three-part L layout, stored reversed
// ([L3 L2 L1] along K) and issued smallest first: L1 . B3,  [L2 L1] . [B2; B2],
// [L3 L2 L1] . [B1; B1; B1]  (BULK order of the B stack).  Within one GEMM the tensor cores
// accumulate along K, so a small part placed after L1 B1 is added into the large sum:
// with the forward order [L1 L2 L3] . [B1; B1; B1] first, C4 needed 18 block-GCR iterations
// instead of 11 (stage 2 2.57 s vs 1.55 s; C2 6 either way, true residual 6.2e-15 vs 3.6e-15).
__constant__ int kOrdSmall[6] = {2, 0, 1, 1, 0, 0};   // A part per K block (B: kOrdSmallB)
__constant__ int kOrdSmallB[6] = {0, 2, 1, 0, 1, 0};
__constant__ int kOrdBulkB[6] = {0, 0, 0, 1, 1, 2};

__device__ __forceinline__ bf16 part_of(const bf16 (&pp)[3], int q) { return q == 0 ? pp[0] : (q == 1 ? pp[1] : pp[2]); }

// BS x BS FP32 blocks (ld lds, block stride sstride) -> the six-part concatenation with
// duplicated A parts: cols != 0: BS x 6BS, part kOrdSmall[q] in columns [q BS, (q+1) BS)
// (A operand, op N); cols == 0: 6BS x BS, part kOrdSmall[q] in rows [q BS, (q+1) BS) (op T).
// Two consecutive rows per thread: 4-byte stores of bf16 pairs.
__global__ void k_blk_cat6(int nblk, int64_t BS, const float *__restrict__ src, int64_t lds, int64_t sstride,
                           bf16 *__restrict__ dst, int cols) {
    const int64_t per = BS * BS, hper = per / 2, total = (int64_t)nblk * hper;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / hper, w = e % hper, r = 2 * (w % (BS / 2)), c = w / (BS / 2);
        const float *sp = src + b * sstride + r + c * lds;
        bf16 pa[3], pb[3];
        split3(sp[0], pa[0], pa[1], pa[2]);
        split3(sp[1], pb[0], pb[1], pb[2]);
        bf16 *d = dst + b * 6 * per;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const int pq = kOrdSmall[q];
            const __nv_bfloat162 v = __halves2bfloat162(part_of(pa, pq), part_of(pb, pq));
            bf16 *t = cols ? d + r + (q * BS + c) * BS : d + (q * BS + r) + c * 6 * BS;
            *reinterpret_cast<__nv_bfloat162 *>(t) = v;
        }
    }
}

// rows [r0, r0 + BS) x ncp columns of X (+ X2; ld) -> a 6BS x ncp stack (ld 6BS) of their
// parts in the SMALL (bulk == 0) or BULK B order; two consecutive rows per thread
__global__ void k_blk_split6(int64_t r0, int64_t BS, int64_t ncp, const float *__restrict__ X,
                             const float *__restrict__ X2, int64_t ld, bf16 *__restrict__ dst, int bulk) {
    const int64_t hb = BS / 2, total = hb * ncp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = 2 * (e % hb), c = e / hb, q0 = (r0 + r) + c * ld;
        float2 v = *reinterpret_cast<const float2 *>(X + q0);
        if (X2) {
            const float2 v2 = *reinterpret_cast<const float2 *>(X2 + q0);
            v.x += v2.x;
            v.y += v2.y;
        }
        bf16 pa[3], pb[3];
        split3(v.x, pa[0], pa[1], pa[2]);
        split3(v.y, pb[0], pb[1], pb[2]);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const int pq = bulk ? kOrdBulkB[q] : kOrdSmallB[q];
            *reinterpret_cast<__nv_bfloat162 *>(dst + (q * BS + r) + c * 6 * BS) =
                __halves2bfloat162(part_of(pa, pq), part_of(pb, pq));
        }
    }
}

// few columns: the bulk update's B operand as ONE 3BS x 3ncp matrix (ld 3BS) against the
// packed [L3 L2 L1], so a single GEMM reads L once:  column block 0 = [B1; B1; B1],
// 1 = [0; B2; B2], 2 = [0; 0; B3]  ->  T = [L3B1 + L2B1 + L1B1, L2B2 + L1B2, L1B3]
__global__ void k_blk_split_cat(int64_t r0, int64_t BS, int64_t ncp, const float *__restrict__ X, int64_t ld,
                                bf16 *__restrict__ dst) {
    const int64_t hb = BS / 2, total = hb * ncp, ldd = 3 * BS;
    const bf16 z = __float2bfloat16_rn(0.f);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = 2 * (e % hb), c = e / hb;
        const float2 v = *reinterpret_cast<const float2 *>(X + (r0 + r) + c * ld);
        bf16 pa[3], pb[3];
        split3(v.x, pa[0], pa[1], pa[2]);
        split3(v.y, pb[0], pb[1], pb[2]);
#pragma unroll
        for (int cb = 0; cb < 3; ++cb)
#pragma unroll
            for (int sl = 0; sl < 3; ++sl) {   // slot sl pairs with L part 3 - sl
                const bool on = sl >= cb;
                *reinterpret_cast<__nv_bfloat162 *>(dst + (sl * BS + r) + (cb * ncp + c) * ldd) =
                    on ? __halves2bfloat162(part_of(pa, cb), part_of(pb, cb)) : __halves2bfloat162(z, z);
            }
    }
}

// C (m x ncp, ldc) -= (T2 + T1) + T0, the bulk update's three partials smallest first
__global__ void k_blk_sub3(int64_t m, int64_t ncp, const float *__restrict__ T, int64_t ldt, float *__restrict__ C,
                           int64_t ldc) {
    const int64_t total = m * ncp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % m, c = e / m;
        const float s = (T[r + (2 * ncp + c) * ldt] + T[r + (ncp + c) * ldt]) + T[r + c * ldt];
        C[r + c * ldc] -= s;
    }
}

// offsets of the packed L layouts (nb blocks of BS):
//   Lc: block column j (j < nb - 1) = rows (j+1)BS .. Nb-1 (height h_j = (nb-1-j) BS) x the
//       three parts side by side, L3 L2 L1 (3BS columns), ld h_j, at 3 BS^2 (j (nb-1) - j (j-1) / 2)
//   Lr: block row i (i >= 1) = the three parts stacked, L3 L2 L1 (3BS rows) x columns 0 .. iBS-1,
//       ld 3BS, at 3 BS^2 (i-1) i / 2
// the small products as a batch of six part GEMMs (HF_PRECOND_SPLITK=0/1 forces; default:
// fewer than 256 right-hand-side columns)
static bool splitk_small(int64_t ncp) {
    if (const char *e = getenv("HF_PRECOND_SPLITK")) return atoi(e) != 0;
    return ncp < 256;
}
// the bulk update as one GEMM against the 3BS x 3ncp part matrix (HF_PRECOND_BCAT=0/1 forces;
// default: fewer than 256 columns, where the three-GEMM form is bound by its repeated L reads)
static bool bcat_bulk(int64_t ncp) {
    if (const char *e = getenv("HF_PRECOND_BCAT")) return atoi(e) != 0;
    return ncp < 256;
}
__host__ __device__ __forceinline__ int64_t lc_off(int64_t j, int64_t nb, int64_t BS) {
    return 3 * BS * BS * (j * (nb - 1) - j * (j - 1) / 2);
}
__host__ __device__ __forceinline__ int64_t lr_off(int64_t i, int64_t BS) { return 3 * BS * BS * ((i - 1) * i / 2); }

// the strictly-below-block-diagonal entries of Lp (Nb x Nb FP32) -> their parts in Lc and Lr;
// 64 x 32 tiles, two consecutive rows per thread (4-byte stores of bf16 pairs)
__global__ void __launch_bounds__(256) k_blk_pack_L(int64_t Nb, int64_t BS, const float *__restrict__ Lp,
                                                    bf16 *__restrict__ Lc, bf16 *__restrict__ Lr) {
    const int64_t i0 = (int64_t)blockIdx.x * 64, j0 = (int64_t)blockIdx.y * 32;
    if (i0 / BS <= j0 / BS) return;   // tiles never straddle a BS block (BS >= 64)
    const int64_t nb = Nb / BS;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t r = i0 + 2 * tx, bi = r / BS;
    for (int q = ty; q < 32; q += 8) {
        const int64_t c = j0 + q, bj = c / BS;
        const float2 v = *reinterpret_cast<const float2 *>(Lp + r + c * Nb);
        bf16 pa[3], pb[3];
        split3(v.x, pa[0], pa[1], pa[2]);
        split3(v.y, pb[0], pb[1], pb[2]);
        const int64_t h = (nb - 1 - bj) * BS;
        bf16 *dc = Lc + lc_off(bj, nb, BS) + (r - (bj + 1) * BS);
        bf16 *dr = Lr + lr_off(bi, BS) + (r - bi * BS) + c * 3 * BS;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const __nv_bfloat162 w = __halves2bfloat162(pa[p], pb[p]);
            const int s = 2 - p;   // stored [L3 L2 L1] along K (smallest first, see gemm_bulk)
            *reinterpret_cast<__nv_bfloat162 *>(dc + (s * BS + (c - bj * BS)) * h) = w;
            *reinterpret_cast<__nv_bfloat162 *>(dr + s * BS) = w;
        }
    }
}

// X (Nb x ncp, pivot order) = RN32(R[perm]) (FP64 -> FP32 truncation), zero padding
__global__ void k_blk_gather(int64_t N, int64_t Nb, int64_t ncol, int64_t ncp, const int64_t *__restrict__ perm,
                             const double *__restrict__ R, int64_t ldr, float *__restrict__ X) {
    const int64_t total = Nb * ncp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % Nb, c = e / Nb;
        X[e] = (i < N && c < ncol) ? __double2float_rn(R[perm[i] + c * ldr]) : 0.f;
    }
}

// Y <- D^{-1} Y (rows < N; IEEE quotient)
__global__ void k_blk_dscale(int64_t N, int64_t Nb, int64_t ncp, const float *__restrict__ D, float *__restrict__ Y) {
    const int64_t total = Nb * ncp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % Nb;
        if (i < N) Y[e] = __fdiv_rn(Y[e], D[i]);
    }
}

// W (L x ncol, original order, FP64) = lift(X[pos1]), 0 on Lambda_2 rows
__global__ void k_blk_scatter(int64_t L, int64_t Nb, int64_t ncol, const int32_t *__restrict__ pos1,
                              const float *__restrict__ X, double *__restrict__ W, int64_t ldw) {
    const int64_t total = L * ncol;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % L, c = e / L;
        const int32_t r = pos1[i];
        W[i + c * ldw] = r >= 0 ? (double)X[r + c * Nb] : 0.0;
    }
}

unsigned grid_for(hf_ctx *ctx, int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8));
}

// C = alpha op(A) B + beta C in FP32 precision: the six bf16 part products with i + j <= 4,
// smallest first, on stream st, `batch` problems at element strides sA / sB / sC
void gemm6(hf_ctx *ctx, cudaStream_t st, bool tA, int64_t m, int64_t n, int64_t k, float alpha, bf16 *const A[3],
           int64_t lda, bf16 *const B[3], int64_t ldb, float beta, float *C, int64_t ldc, int batch = 1,
           int64_t sA = 0, int64_t sB = 0, int64_t sC = 0) {
    static const int ord[6][2] = {{2, 0}, {0, 2}, {1, 1}, {1, 0}, {0, 1}, {0, 0}};
    for (int q = 0; q < 6; ++q)
        lt_bgemm(ctx, tA, m, n, k, alpha, A[ord[q][0]], lda, B[ord[q][1]], ldb, q ? 1.f : beta, C, ldc, st, batch, sA,
                 sB, sC);
}

bf16 *bp(DBuf<uint16_t> &b) { return reinterpret_cast<bf16 *>(b.p); }
void parts(DBuf<uint16_t> (&b)[3], int64_t off, bf16 *out[3]) {
    for (int q = 0; q < 3; ++q) out[q] = bp(b[q]) + off;
}

cudaStream_t aux_stream(hf_ctx *ctx, int i) {
    if (!ctx->aux[i]) HF_CUDA(cudaStreamCreateWithFlags(&ctx->aux[i], cudaStreamNonBlocking));
    return ctx->aux[i];
}

}  // namespace

bool precond_blocked_enabled() {
    const char *e = getenv("HF_PRECOND");
    return !(e && std::string(e) == "dataflow");
}

void precond_blk_setup(hf_ctx *ctx, PrecondBlk &p, int64_t N, int64_t L, const float *Lfac, const float *D,
                       const int64_t *perm, const int32_t *pos1) {
    cudaStream_t st = ctx->stream;
    p.N = N;
    p.L = L;
    p.D = D;
    p.perm = perm;
    p.pos1 = pos1;
    if (N == 0) return;
    int64_t bsmax = 2048;   // HF_PRECOND_BS: tuning (a power of two times 64)
    if (const char *e = getenv("HF_PRECOND_BS")) bsmax = std::max<int64_t>(64, atoll(e));
    int64_t BS = 64;
    while (BS < bsmax && BS < N) BS *= 2;
    p.BS = BS;
    p.nb = (int)cdiv(N, BS);
    p.Nb = p.nb * BS;
    const int64_t Nb = p.Nb, nb = p.nb;
    ClassTimer tm(ctx, "trsm_setup");
    const size_t ninv = (size_t)nb * BS * (BS + 1), per6 = (size_t)6 * BS * BS;
    DBuf<float> Lp, Inv, T;   // FP32 working copies, released at the end
    Lp.alloc((size_t)Nb * Nb, st);
    Inv.alloc(ninv, st);
    T.alloc(std::max<size_t>((size_t)Nb * BS / 4, (size_t)std::max<int64_t>(nb - 1, 1) * BS * BS), st);
    HF_CUDA(cudaMemsetAsync(Inv.p, 0, ninv * sizeof(float), st));
    dim3 g((unsigned)(Nb / 32), (unsigned)(Nb / 32));
    k_blk_pad<<<g, 256, 0, st>>>(N, Nb, Lfac, Lp.p);
    HF_CHECK_LAUNCH(ctx);
    k_blk_inv64<<<(unsigned)(Nb / 64), 64, 0, st>>>(Nb, Lp.p, BS, Inv.p);
    HF_CHECK_LAUNCH(ctx);
    // recursive doubling, IEEE FP32 GEMMs: all pairs of one level in one batched call each
    for (int64_t h = 64; h < BS; h *= 2) {
        const int batch = (int)(Nb / (2 * h));
        const int64_t sd = 2 * h * (BS + 1), sl = 2 * h * (Nb + 1);
        // T_p = C_p Ainv_p,  C_p = L[g+h : g+2h, g : g+h]
        lt_sgemm(ctx, false, false, h, h, h, 1.f, Lp.p + h, Nb, sl, Inv.p, BS, sd, 0.f, T.p, h, h * h, batch, false);
        // Inv[g+h : g+2h, g : g+h] = -Binv_p T_p
        lt_sgemm(ctx, false, false, h, h, h, -1.f, Inv.p + h * (BS + 1), BS, sd, T.p, h, h * h, 0.f, Inv.p + h, BS, sd,
                 batch, false);
    }
    // the operands of the solves
    const size_t nlc = (size_t)lc_off(nb - 1, nb, BS), nlr = (size_t)lr_off(nb, BS);
    p.Lc.alloc(std::max<size_t>(nlc, 1), st);
    p.Lr.alloc(std::max<size_t>(nlr, 1), st);
    if (nb > 1) {
        k_blk_pack_L<<<dim3((unsigned)(Nb / 64), (unsigned)(Nb / 32)), 256, 0, st>>>(Nb, BS, Lp.p, bp(p.Lc), bp(p.Lr));
        HF_CHECK_LAUNCH(ctx);
    }
    p.Ic.alloc(nb * per6, st);
    p.It.alloc(nb * per6, st);
    k_blk_cat6<<<grid_for(ctx, nb * BS * BS / 2), 256, 0, st>>>(nb, BS, Inv.p, BS, BS * (BS + 1), bp(p.Ic), 1);
    HF_CHECK_LAUNCH(ctx);
    k_blk_cat6<<<grid_for(ctx, nb * BS * BS / 2), 256, 0, st>>>(nb, BS, Inv.p, BS, BS * (BS + 1), bp(p.It), 0);
    HF_CHECK_LAUNCH(ctx);
    // the couplings of consecutive blocks, so that the next block's update needs the current
    // block's right-hand side, not its solution:  G_j = L_{j+1,j} Linv_j (forward),
    // H_j = Linv_{j+1} L_{j+1,j} (backward), FP32 precision (the six part products, batched)
    if (nb > 1) {
        const int nc = (int)nb - 1;
        DBuf<uint16_t> Ls[3], Is[3];   // parts of the sub-diagonal blocks and of the inverses
        for (int q = 0; q < 3; ++q) {
            Ls[q].alloc((size_t)nc * BS * BS, st);
            Is[q].alloc(ninv, st);
        }
        k_blk_split_all<<<grid_for(ctx, (int64_t)ninv), 256, 0, st>>>((int64_t)ninv, Inv.p, bp(Is[0]), bp(Is[1]),
                                                                      bp(Is[2]));
        HF_CHECK_LAUNCH(ctx);
        // the sub-diagonal blocks L_{j+1,j} into a packed FP32 copy (T), then parts
        HF_CUDA(cudaMemcpy2DAsync(T.p, BS * sizeof(float), Lp.p + BS, Nb * sizeof(float), BS * sizeof(float), BS, 
                                  cudaMemcpyDeviceToDevice, st));   // block 0 (the batched form follows)
        for (int j = 1; j < nc; ++j)
            HF_CUDA(cudaMemcpy2DAsync(T.p + (size_t)j * BS * BS, BS * sizeof(float), Lp.p + (j + 1) * BS + j * BS * Nb,
                                      Nb * sizeof(float), BS * sizeof(float), BS, cudaMemcpyDeviceToDevice, st));
        k_blk_split_all<<<grid_for(ctx, (int64_t)nc * BS * BS), 256, 0, st>>>((int64_t)nc * BS * BS, T.p, bp(Ls[0]),
                                                                              bp(Ls[1]), bp(Ls[2]));
        HF_CHECK_LAUNCH(ctx);
        bf16 *A[3], *B[3];
        p.Gc.alloc((size_t)nc * per6, st);
        p.Ht.alloc((size_t)nc * per6, st);
        // G_j = L_{j+1,j} Inv_j -> T -> Gc
        parts(Ls, 0, A);
        parts(Is, 0, B);
        gemm6(ctx, st, false, BS, BS, BS, 1.f, A, BS, B, BS, 0.f, T.p, BS, nc, BS * BS, BS * (BS + 1), BS * BS);
        k_blk_cat6<<<grid_for(ctx, nc * BS * BS / 2), 256, 0, st>>>(nc, BS, T.p, BS, BS * BS, bp(p.Gc), 1);
        HF_CHECK_LAUNCH(ctx);
        // H_j = Inv_{j+1} L_{j+1,j} -> T -> Ht
        parts(Is, BS * (BS + 1), A);
        parts(Ls, 0, B);
        gemm6(ctx, st, false, BS, BS, BS, 1.f, A, BS, B, BS, 0.f, T.p, BS, nc, BS * (BS + 1), BS * BS, BS * BS);
        k_blk_cat6<<<grid_for(ctx, nc * BS * BS / 2), 256, 0, st>>>(nc, BS, T.p, BS, BS * BS, bp(p.Ht), 0);
        HF_CHECK_LAUNCH(ctx);
    }
    if (p.ev.empty()) {
        p.ev.resize((size_t)4 * nb + 4);
        for (auto &e : p.ev) HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
}

// Three streams per direction: A (the context stream) stacks block j's right-hand side and
// forms its solution; C applies the coupling to block j +- 1 from the right-hand side (the
// sequential path: stack -> one coupling GEMM -> stack); B runs the bulk update of the
// blocks beyond from the solution (three GEMMs over the packed three-part L).  The coupling
// updates accumulate into Xa, the bulk ones into Xb, so the two never write the same words;
// block j's right-hand side is Xa + Xb.
void precond_blk_apply(hf_ctx *ctx, PrecondBlk &p, int64_t ncol, const double *R, int64_t ldr, double *W,
                       int64_t ldw) {
    cudaStream_t st = ctx->stream;
    if (ncol == 0) return;
    if (p.N == 0) {
        HF_CUDA(cudaMemset2DAsync(W, ldw * sizeof(double), 0, p.L * sizeof(double), ncol, st));
        return;
    }
    const int64_t Nb = p.Nb, BS = p.BS, ncp = (ncol + 7) / 8 * 8, nb = p.nb;
    const size_t per6 = (size_t)6 * BS * BS, stk = (size_t)6 * BS * ncp;
    p.Xa.alloc((size_t)Nb * ncp, st);
    p.Xb.alloc((size_t)Nb * ncp, st);
    p.Y.alloc((size_t)Nb * ncp, st);
    p.S6.alloc(nb * stk, st);
    p.SB.alloc(nb * stk, st);
    const double nn = (double)p.N * (double)p.N;
    ClassTimer tm(ctx, "trsm", st, 2.0 * nn * (double)ncol, 3.0 * nn + 16.0 * (double)p.N * (double)ncol);
    cudaStream_t sb = aux_stream(ctx, 0), sc = aux_stream(ctx, 1);
    cudaEvent_t *evX = p.ev.data(), *evY = evX + nb, *evC = evY + nb, *evB = evC + nb, *evS = evB + nb;
    float *Xa = p.Xa.p, *Xb = p.Xb.p, *Y = p.Y.p;
    bf16 *S6 = bp(p.S6), *SB = bp(p.SB), *Lc = bp(p.Lc), *Lr = bp(p.Lr);
    auto stack = [&](cudaStream_t s, const float *src, const float *src2, int64_t j, bf16 *dst, int bulk) {
        k_blk_split6<<<grid_for(ctx, BS * ncp / 2), 256, 0, s>>>(j * BS, BS, ncp, src, src2, Nb, dst + j * stk, bulk);
        HF_CHECK_LAUNCH(ctx);
    };
    // one GEMM over K' = 6BS (the duplicated-part A operands), or (split) the six part products
    // as one strided batch of K = BS GEMMs into partials summed smallest first by k_blk_sum6:
    // with few right-hand sides the single GEMM has BS ncp / 64^2 CTAs walking a 6BS-long K
    // (C4 with 64 columns per rank: 32 CTAs; trsm 183 -> 169 ms per stage 2 there, neutral at
    // C2's 256 columns, where the default keeps the single GEMM)
    const bool split = splitk_small(ncp);
    if (split) {
        p.P6a.alloc((size_t)6 * BS * ncp, st);
        p.P6c.alloc((size_t)6 * BS * ncp, st);
    }
    auto gemm_small = [&](cudaStream_t s, bool tA, const bf16 *A, int64_t j, float alpha, float beta, float *C) {
        if (split) {
            float *P6 = (s == sc) ? p.P6c.p : p.P6a.p;
            lt_bgemm(ctx, tA, BS, ncp, BS, 1.f, A, tA ? 6 * BS : BS, S6 + j * stk, 6 * BS, 0.f, P6, BS, s, 6,
                     tA ? BS : BS * BS, BS, BS * ncp);
            k_blk_sum6<<<grid_for(ctx, BS * ncp), 256, 0, s>>>(BS, ncp, P6, alpha, beta, C, Nb);
            HF_CHECK_LAUNCH(ctx);
            return;
        }
        lt_bgemm(ctx, tA, BS, ncp, 6 * BS, alpha, A, tA ? 6 * BS : BS, S6 + j * stk, 6 * BS, beta, C, Nb, s);
    };
    // the bulk product from the three-part L: K' = 3BS, 2BS, BS over the stack's BULK blocks
    const bool bcat = bcat_bulk(ncp);
    const size_t stc = (size_t)9 * BS * ncp;
    if (bcat) {
        p.SC.alloc(nb * stc, st);
        p.TB.alloc((size_t)Nb * 3 * ncp, st);
    }
    auto gemm_bulk = [&](cudaStream_t s, bool tA, int64_t m, const bf16 *A, int64_t lda, int64_t j, float *C) {
        if (bcat) {   // one GEMM reads [L3 L2 L1] once; the partials are subtracted smallest first
            if (m <= 0) return;
            lt_bgemm(ctx, tA, m, 3 * ncp, 3 * BS, 1.f, A, lda, bp(p.SC) + j * stc, 3 * BS, 0.f, p.TB.p, m, s);
            k_blk_sub3<<<grid_for(ctx, m * ncp), 256, 0, s>>>(m, ncp, p.TB.p, m, C, Nb);
            HF_CHECK_LAUNCH(ctx);
            return;
        }
        const bf16 *Bj = SB + j * stk;
        // smallest first: L1 B3, [L2 L1] [B2; B2], [L3 L2 L1] [B1; B1; B1] (parts stored reversed)
        const int64_t po = tA ? BS : BS * lda;   // one part further along K in A
        lt_bgemm(ctx, tA, m, ncp, BS, -1.f, A + 2 * po, lda, Bj + 5 * BS, 6 * BS, 1.f, C, Nb, s);
        lt_bgemm(ctx, tA, m, ncp, 2 * BS, -1.f, A + po, lda, Bj + 3 * BS, 6 * BS, 1.f, C, Nb, s);
        lt_bgemm(ctx, tA, m, ncp, 3 * BS, -1.f, A, lda, Bj, 6 * BS, 1.f, C, Nb, s);
    };
    auto fork = [&]() {   // B and C start after everything queued on A so far
        HF_CUDA(cudaEventRecord(evS[0], st));
        HF_CUDA(cudaStreamWaitEvent(sb, evS[0], 0));
        HF_CUDA(cudaStreamWaitEvent(sc, evS[0], 0));
    };
    auto join = [&]() {   // A continues after everything queued on B and C
        HF_CUDA(cudaEventRecord(evS[1], sb));
        HF_CUDA(cudaEventRecord(evS[2], sc));
        HF_CUDA(cudaStreamWaitEvent(st, evS[1], 0));
        HF_CUDA(cudaStreamWaitEvent(st, evS[2], 0));
    };
    k_blk_gather<<<grid_for(ctx, Nb * ncp), 256, 0, st>>>(p.N, Nb, ncol, ncp, p.perm, R, ldr, Xa);
    HF_CHECK_LAUNCH(ctx);
    HF_CUDA(cudaMemsetAsync(Xb, 0, (size_t)Nb * ncp * sizeof(float), st));
    fork();
    // ---- forward: L Y = X
    for (int64_t j = 0; j < nb; ++j) {
        const int64_t j0 = j * BS;
        if (j >= 1) HF_CUDA(cudaStreamWaitEvent(st, evC[j - 1], 0));   // coupling of j-1 wrote Xa_j
        if (j >= 2) HF_CUDA(cudaStreamWaitEvent(st, evB[j - 2], 0));   // bulk of j-2 wrote Xb_j
        stack(st, Xa, Xb, j, S6, 0);
        HF_CUDA(cudaEventRecord(evX[j], st));
        if (j + 1 < nb) {   // C: Xa_{j+1} -= G_j X_j
            HF_CUDA(cudaStreamWaitEvent(sc, evX[j], 0));
            gemm_small(sc, false, bp(p.Gc) + j * per6, j, -1.f, 1.f, Xa + j0 + BS);
            HF_CUDA(cudaEventRecord(evC[j], sc));
        }
        gemm_small(st, false, bp(p.Ic) + j * per6, j, 1.f, 0.f, Y + j0);   // A: Y_j = Linv_j X_j
        if (j + 2 < nb) {   // B: Xb_{>j+1} -= L_{>j+1,j} Y_j
            if (bcat) {
                k_blk_split_cat<<<grid_for(ctx, BS * ncp / 2), 256, 0, st>>>(j * BS, BS, ncp, Y, Nb,
                                                                              bp(p.SC) + j * stc);
                HF_CHECK_LAUNCH(ctx);
            } else {
                stack(st, Y, nullptr, j, SB, 1);
            }
            HF_CUDA(cudaEventRecord(evY[j], st));
            HF_CUDA(cudaStreamWaitEvent(sb, evY[j], 0));
            const int64_t h = (nb - 1 - j) * BS;
            gemm_bulk(sb, false, h - BS, Lc + lc_off(j, nb, BS) + BS, h, j, Xb + j0 + 2 * BS);
            HF_CUDA(cudaEventRecord(evB[j], sb));
        }
    }
    join();
    k_blk_dscale<<<grid_for(ctx, Nb * ncp), 256, 0, st>>>(p.N, Nb, ncp, p.D, Y);
    HF_CHECK_LAUNCH(ctx);
    // ---- backward: L^T X = Z (Z = D^-1 Y: Za = Y, Zb = 0; the solution goes to Xa)
    float *Za = Y, *Zb = Xb, *Xo = Xa;
    HF_CUDA(cudaMemsetAsync(Zb, 0, (size_t)Nb * ncp * sizeof(float), st));
    fork();
    for (int64_t j = nb - 1; j >= 0; --j) {
        const int64_t j0 = j * BS;
        if (j + 1 < nb) HF_CUDA(cudaStreamWaitEvent(st, evC[j + 1], 0));   // coupling of j+1 wrote Za_j
        if (j + 2 < nb) HF_CUDA(cudaStreamWaitEvent(st, evB[j + 2], 0));   // bulk of j+2 wrote Zb_j
        stack(st, Za, Zb, j, S6, 0);
        HF_CUDA(cudaEventRecord(evX[j], st));
        if (j >= 1) {   // C: Za_{j-1} -= H_{j-1}^T Z_j
            HF_CUDA(cudaStreamWaitEvent(sc, evX[j], 0));
            gemm_small(sc, true, bp(p.Ht) + (j - 1) * per6, j, -1.f, 1.f, Za + j0 - BS);
            HF_CUDA(cudaEventRecord(evC[j], sc));
        }
        gemm_small(st, true, bp(p.It) + j * per6, j, 1.f, 0.f, Xo + j0);   // A: X_j = Linv_j^T Z_j
        if (j >= 2) {   // B: Zb_{<j-1} -= (L_{j,<j-1})^T X_j
            if (bcat) {
                k_blk_split_cat<<<grid_for(ctx, BS * ncp / 2), 256, 0, st>>>(j * BS, BS, ncp, Xo, Nb,
                                                                              bp(p.SC) + j * stc);
                HF_CHECK_LAUNCH(ctx);
            } else {
                stack(st, Xo, nullptr, j, SB, 1);
            }
            HF_CUDA(cudaEventRecord(evY[j], st));
            HF_CUDA(cudaStreamWaitEvent(sb, evY[j], 0));
            gemm_bulk(sb, true, j0 - BS, Lr + lr_off(j, BS), 3 * BS, j, Zb);
            HF_CUDA(cudaEventRecord(evB[j], sb));
        }
    }
    join();
    k_blk_scatter<<<grid_for(ctx, p.L * ncol), 256, 0, st>>>(p.L, Nb, ncol, p.pos1, Xo, W, ldw);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
