// k_trsm.cu -- the lower-precision preconditioner Q^{-1} of P:242 ("find e^
// satisfying Q^ e^ = r^ in lower precision ... up-converting"), used by block
// GCR (Alg. 5) and Alg. 2 step 1:
//   W = scatter_Pi( L^{-T} D^{-1} L^{-1} RN32(gather_Pi(R)) )  in FP32,
// with the FP64->FP32 truncation fused into the forward solve's load and the
// FP32->FP64 lift + scatter to original row order fused into the backward
// solve's store ("forward/backward substitution in lower precision ...
// BLAS level 3 TRSM").  Any summation order is allowed here [R12].
//
// Design (B200): persistent dataflow kernels, one per direction.
//  * Work item = (64-row block b, 64-column RHS chunk).  Items are handed out
//    in dependency order by an atomic counter; an item accumulates the
//    off-diagonal products L_bq Y_q of its dependencies q in the order they
//    finish (release flags, relaxed polling + one acquire), then applies the
//    precomputed inverse of its 64x64 unit diagonal block and releases its own
//    flag.  No host round trips, no launch per block.
//  * Operands are laid out so every tile load is a contiguous 16-byte
//    cp.async (LDGSTS) into a conflict-free shared layout, double buffered so
//    the next dependency's tiles stream in while the current one is used:
//      - forward reads L (padded Np x Np, column-major): tile[k][r] = L(r0+r, q0+k)
//      - backward reads U = L^T (padded, column-major):   tile[k][r] = U(r0+r, q0+k)
//      - the intermediate y and x are ROW-major (Np x ncolp), so tile[k][c] is
//        a contiguous row segment.
//  * 256 threads, 4x4 register tile per thread, FFMA.
#include <algorithm>

#include "k_dgemm.cuh"

namespace hf {
namespace {

constexpr int TBS = 64;          // row block
constexpr int CW = 64;           // RHS chunk width
constexpr int TILE = TBS * TBS;  // floats per 64x64 tile

__device__ __forceinline__ void st_release32(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Poll with RELAXED loads and acquire once afterwards: an ld.acquire in a spin
// loop emits an L1 invalidate per iteration, which stalls every other CTA on the SM.
__device__ __forceinline__ int ld_relaxed32(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void cp_async16(float *smem_dst, const float *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// ------------------------------------------------------------------ setup kernels
// Lp (Np x Np, ld Np) = Lfac (N x N, ld N) padded with the identity; Up = Lp^T.
// 32x32 tiles through shared memory so both the read and the transposed write
// are coalesced.
__global__ void __launch_bounds__(256) k_pad_transpose(int64_t N, int64_t Np, const float *__restrict__ Lf,
                                                       float *__restrict__ Lp, float *__restrict__ Up) {
    __shared__ float t[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int q = ty; q < 32; q += 8) {
        const int64_t i = i0 + tx, j = j0 + q;
        float v;
        if (i < N && j < N) v = Lf[i + j * N];
        else v = (i == j) ? 1.f : 0.f;
        t[q][tx] = v;
        Lp[i + j * Np] = v;
    }
    __syncthreads();
    for (int q = ty; q < 32; q += 8) Up[(j0 + tx) + (i0 + q) * Np] = t[tx][q];   // Up(j, i) = L(i, j)
}

// Inverse of each 64x64 unit-lower diagonal block, stored directly in the
// shared-tile layouts of the two solves:
//   LinvF[b][k][r] = Linv_b(r, k)   (forward:  out = Linv_b acc)
//   LinvB[b][k][r] = Linv_b(k, r)   (backward: out = Linv_b^T acc)
__global__ void __launch_bounds__(64) k_diag_inv(int64_t Np, const float *__restrict__ Lp, float *__restrict__ LinvF,
                                                 float *__restrict__ LinvB) {
    __shared__ float Ls[TBS][TBS + 1];
    __shared__ float Xs[TBS][TBS + 1];
    const int64_t r0 = (int64_t)blockIdx.x * TBS;
    const int j = threadIdx.x;
    for (int i = 0; i < TBS; ++i) Ls[i][j] = Lp[(r0 + i) + (r0 + j) * Np];
    __syncthreads();
    // column j of the inverse: x_i = delta_ij - sum_{j<=k<i} L_ik x_k
    for (int i = 0; i < TBS; ++i) {
        float s = (i == j) ? 1.f : 0.f;
        if (i > j)
            for (int k = j; k < i; ++k) s = __fmaf_rn(-Ls[i][k], Xs[k][j], s);
        Xs[i][j] = (i < j) ? 0.f : s;
    }
    __syncthreads();
    float *F = LinvF + (size_t)blockIdx.x * TILE;
    float *B = LinvB + (size_t)blockIdx.x * TILE;
    for (int k = 0; k < TBS; ++k) {
        F[k * TBS + j] = Xs[j][k];
        B[k * TBS + j] = Xs[k][j];
    }
}

struct TrsmArgs {
    int64_t N, Np;
    int ncol, ncolp, nch, nblk;
    const float *Lp;     // forward operand  (Np x Np, col-major)
    const float *Up;     // backward operand (Np x Np, col-major) = Lp^T
    const float *LinvF;  // [nblk][64][64]
    const float *LinvB;
    const float *D;      // [N]
    const int64_t *perm; // [L] pivot order -> original index
    const double *R;     // input, original row order (L x ncol, ldr)
    int64_t ldr;
    float *Y;            // forward result, row-major Np x ncolp
    float *Xb;           // backward result, row-major Np x ncolp
    double *W;           // output, original row order (L x ncol, ldw)
    int64_t ldw;
    int *flags;          // [2][nblk*nch]
    int *counter;        // [2]
    int epoch;
};

// acc[i][j] -= sum_k As[k][tr*4+i] * Bs[k][tc*4+j]
__device__ __forceinline__ void tile_fms(float (&acc)[4][4], const float *As, const float *Bs, int tr, int tc) {
#pragma unroll 16
    for (int k = 0; k < TBS; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(&As[k * TBS + tr * 4]);
        const float4 y = *reinterpret_cast<const float4 *>(&Bs[k * CW + tc * 4]);
        const float av[4] = {-a.x, -a.y, -a.z, -a.w};
        const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], yv[j], acc[i][j]);
    }
}

template <bool BWD>
__global__ void __launch_bounds__(256, 3) k_trsm(TrsmArgs a) {
    extern __shared__ __align__(16) float sm[];   // [2 stages][A tile | B tile]
    __shared__ int item_s;
    const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
    const int nitems = a.nblk * a.nch;
    int *flags = a.flags + (BWD ? nitems : 0);
    int *counter = a.counter + (BWD ? 1 : 0);
    const float *Op = BWD ? a.Up : a.Lp;
    const float *src = BWD ? a.Xb : a.Y;

    // copy the (A, B) tiles of dependency block q, chunk c0, into stage s
    auto load_dep = [&](int s, int64_t r0, int64_t q0, int c0) {
        float *As = sm + s * 2 * TILE;
        float *Bs = As + TILE;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + u * 256;          // 1024 16-byte chunks per tile
            const int k = e >> 4, r4 = (e & 15) * 4;
            cp_async16(&As[k * TBS + r4], Op + (r0 + r4) + (q0 + k) * a.Np);
            cp_async16(&Bs[k * CW + r4], src + (q0 + k) * a.ncolp + c0 + r4);
        }
    };

    for (;;) {
        if (tid == 0) item_s = atomicAdd(counter, 1);
        __syncthreads();
        const int item = item_s;
        if (item >= nitems) return;
        const int b = BWD ? (a.nblk - 1 - item / a.nch) : (item / a.nch);
        const int cc = item % a.nch;
        const int64_t r0 = (int64_t)b * TBS;
        const int c0 = cc * CW;
        float acc[4][4];
        // ---- right-hand side: forward truncates R (FP64, original order) to FP32;
        //      backward starts from z = D^{-1} y
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t r = r0 + tr * 4 + i;
            if (!BWD) {
                const int64_t pr = r < a.N ? a.perm[r] : 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int c = c0 + tc * 4 + j;
                    acc[i][j] = (r < a.N && c < a.ncol) ? __double2float_rn(a.R[pr + (int64_t)c * a.ldr]) : 0.f;
                }
            } else {
                const float4 y = *reinterpret_cast<const float4 *>(&a.Y[r * a.ncolp + c0 + tc * 4]);
                const float d = r < a.N ? a.D[r] : 1.f;
                acc[i][0] = __fdiv_rn(y.x, d);
                acc[i][1] = __fdiv_rn(y.y, d);
                acc[i][2] = __fdiv_rn(y.z, d);
                acc[i][3] = __fdiv_rn(y.w, d);
            }
        }
        // ---- off-diagonal blocks (forward: 0 .. b-1; backward: nblk-1 .. b+1),
        //      double buffered: tiles of dependency dq+1 stream in during dq
        const int ndep = BWD ? (a.nblk - 1 - b) : b;
        auto dep_block = [&](int dq) { return BWD ? (a.nblk - 1 - dq) : dq; };
        auto wait_flag = [&](int q) {
            if (tid == 0) {
                const int *f = &flags[q * a.nch + cc];
                if (ld_relaxed32(f) != a.epoch) {
                    while (ld_relaxed32(f) != a.epoch) __nanosleep(32);
                }
                fence_acquire();
            }
            __syncthreads();
        };
        if (ndep > 0) {
            wait_flag(dep_block(0));
            load_dep(0, r0, (int64_t)dep_block(0) * TBS, c0);
            cp_commit();
        }
        for (int dq = 0; dq < ndep; ++dq) {
            if (dq + 1 < ndep) {
                wait_flag(dep_block(dq + 1));
                load_dep((dq + 1) & 1, r0, (int64_t)dep_block(dq + 1) * TBS, c0);
                cp_commit();
                cp_wait_1();
            } else {
                cp_wait_all();
            }
            __syncthreads();
            const float *As = sm + (dq & 1) * 2 * TILE;
            tile_fms(acc, As, As + TILE, tr, tc);
            __syncthreads();
        }
        // ---- diagonal block: out = Linv_b acc (forward) or Linv_b^T acc (backward)
        {
            float *As = sm, *Bs = sm + TILE;
            const float *Li = (BWD ? a.LinvB : a.LinvF) + (size_t)b * TILE;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = tid + u * 256;
                cp_async16(&As[e * 4], Li + e * 4);
            }
            cp_commit();
            // Bs[k][c] = -acc (tile_fms subtracts)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                *reinterpret_cast<float4 *>(&Bs[(tr * 4 + i) * CW + tc * 4]) =
                    make_float4(-acc[i][0], -acc[i][1], -acc[i][2], -acc[i][3]);
            cp_wait_all();
            __syncthreads();
            float out[4][4] = {};
            tile_fms(out, As, Bs, tr, tc);
            // ---- store
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t r = r0 + tr * 4 + i;
                float *dst = (BWD ? a.Xb : a.Y) + r * a.ncolp + c0 + tc * 4;
                *reinterpret_cast<float4 *>(dst) = make_float4(out[i][0], out[i][1], out[i][2], out[i][3]);
                if (BWD && r < a.N) {
                    const int64_t pr = a.perm[r];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int c = c0 + tc * 4 + j;
                        if (c < a.ncol) a.W[pr + (int64_t)c * a.ldw] = (double)out[i][j];   // lift + scatter
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release32(&flags[b * a.nch + cc], a.epoch);
        }
    }
}

}  // namespace

void precond_setup(hf_ctx *ctx, Precond &p, int64_t N, int64_t L, const float *Lfac, const float *D,
                   const int64_t *perm) {
    p.N = N;
    p.L = L;
    p.Lfac = Lfac;
    p.D = D;
    p.perm = perm;
    if (N == 0) return;
    cudaStream_t st = ctx->stream;
    const int64_t nblk = cdiv(N, TBS);
    p.Np = nblk * TBS;
    p.Lp.alloc((size_t)p.Np * p.Np, st);
    p.Up.alloc((size_t)p.Np * p.Np, st);
    p.LinvF.alloc((size_t)nblk * TILE, st);
    p.LinvB.alloc((size_t)nblk * TILE, st);
    ClassTimer tm(ctx, "trsm");
    dim3 g((unsigned)(p.Np / 32), (unsigned)(p.Np / 32));
    k_pad_transpose<<<g, 256, 0, st>>>(N, p.Np, Lfac, p.Lp.p, p.Up.p);
    HF_CHECK_LAUNCH(ctx);
    k_diag_inv<<<(unsigned)nblk, TBS, 0, st>>>(p.Np, p.Lp.p, p.LinvF.p, p.LinvB.p);
    HF_CHECK_LAUNCH(ctx);
}

void precond_apply(hf_ctx *ctx, Precond &p, int64_t ncol, const double *R, int64_t ldr, double *W, int64_t ldw) {
    cudaStream_t st = ctx->stream;
    HF_CUDA(cudaMemset2DAsync(W, ldw * sizeof(double), 0, p.L * sizeof(double), ncol, st));
    if (p.N == 0 || ncol == 0) return;
    const int nblk = (int)(p.Np / TBS);
    const int nch = (int)cdiv(ncol, CW);
    const int ncolp = nch * CW;
    p.Y.alloc((size_t)p.Np * ncolp, st);
    p.Xb.alloc((size_t)p.Np * ncolp, st);
    if (p.flags.n < (size_t)2 * nblk * nch) {
        p.flags.alloc((size_t)2 * nblk * nch, st);
        p.flags.zero(st);
        p.epoch = 0;
    }
    p.counter.alloc(2, st);
    HF_CUDA(cudaMemsetAsync(p.counter.p, 0, 2 * sizeof(int), st));
    p.epoch += 1;
    TrsmArgs a{p.N, p.Np, (int)ncol, ncolp, nch, nblk, p.Lp.p, p.Up.p, p.LinvF.p, p.LinvB.p, p.D, p.perm,
               R, ldr, p.Y.p, p.Xb.p, W, ldw, p.flags.p, p.counter.p, p.epoch};
    const size_t shm = (size_t)4 * TILE * sizeof(float);   // 2 stages x (A + B) = 64 KB
    static bool attr = false;
    if (!attr) {
        HF_CUDA(cudaFuncSetAttribute(k_trsm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        HF_CUDA(cudaFuncSetAttribute(k_trsm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        attr = true;
    }
    const int nitems = nblk * nch;
    const int grid = std::min(nitems, ctx->num_sms * 3);
    ClassTimer tm(ctx, "trsm");
    k_trsm<false><<<grid, 256, shm, st>>>(a);
    HF_CHECK_LAUNCH(ctx);
    k_trsm<true><<<grid, 256, shm, st>>>(a);
    HF_CHECK_LAUNCH(ctx);
}

}  // namespace hf
