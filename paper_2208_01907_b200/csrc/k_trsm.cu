// k_trsm.cu -- the lower-precision preconditioner Q^{-1} of P:242 ("find e^
// satisfying Q^ e^ = r^ in lower precision ... up-converting"), used by block
// GCR (Alg. 5) and Alg. 2 step 1:
//   W = scatter_Pi( L^{-T} D^{-1} L^{-1} RN32(gather_Pi(R)) )  in FP32,
// with the FP64->FP32 truncation fused into the forward solve's load and the
// FP32->FP64 lift + scatter to original row order fused into the backward
// solve's store ("forward/backward substitution in lower precision ...
// BLAS level 3 TRSM").  Any summation order is allowed here [R12].
//
// Design (B200): one cooperative persistent launch per direction, blocks of
// 64 rows, RHS chunks of 64 columns.  With Dinv_b the inverse of the unit
// diagonal block (L_bb^{-1} forward, L_bb^{-T} backward), Op = L / L^T and
// the block-row-scaled operator G_bq = Dinv_b Op_bq (formed once, in place,
// at setup), the solve is  Y_b = Dinv_b RHS_b - sum_{q<b} G_bq Y_q, split as
//     Y_b = P_b - G_{b,b-1} Y_{b-1} - G_{b,b-2} Y_{b-2},
//     P_b = Dinv_b RHS_b - sum_{q < b-2} G_bq Y_q
// (block indices in the direction of the solve); no Dinv product is left
// behind the last dependency of P_b.
//  * CHAIN CTAs (one per chunk, alone on their SM: the helper that shares
//    the SM exits) walk the blocks in order and keep Y_{b-1}, Y_{b-2} in a
//    3-slot shared ring: a link of the sequential chain is two 64x64x64
//    tile products (G tiles prefetched by cp.async during the previous
//    link); two STORE warps copy each finished Y_b to global memory, fence
//    and release it while the 8 compute warps already run the next link
//    (per-slot FULL/EMPTY named barriers hand the ring slots over).
//  * ROLES BY SM: the first CTA to reach an SM takes the next role ticket
//    (chain chunks, then P-workers); a CTA landing on a role's SM leaves, so
//    every latency-critical CTA has its SM alone.
//  * P-WORKERS (two per chunk, blocks j alternating) form P_j = base_j - (near
//    partial slots) - (tail: G_{j,j-3} Y_{j-3}), the short sums that remain
//    once Y_{j-3} is out.
//  * HELPER CTAs (all others) take items from a host-built table in
//    topological order (atomic counter): PARTIAL items sum one segment of
//    dependency blocks into a slot (segments grow geometrically away from the
//    diagonal: 1, 2, 4, ..., SEG blocks); EARLY items form base_j = Dinv_j RHS_j
//    - (bulk slots) well ahead of the chain.  Dependency flags are checked
//    eight at a time and three stages of tile loads are in flight.
//  * Release flags + relaxed polling + one acquire; the cooperative launch
//    guarantees chain and helpers are co-resident (no deadlock by design:
//    every table item depends only on earlier items and on chain stages
//    earlier than its own position).
//  * Operands are laid out so every tile load is a contiguous 16-byte
//    cp.async (LDGSTS) into a conflict-free shared layout, double buffered so
//    the next dependency's tiles stream in while the current one is used:
//      - forward reads L (padded Np x Np, column-major): tile[k][r] = L(r0+r, q0+k)
//      - backward reads U = L^T (padded, column-major):   tile[k][r] = U(r0+r, q0+k)
//      - the intermediate y and x are ROW-major (Np x ncolp), so tile[k][c] is
//        a contiguous row segment.
//  * 256 threads, 4x4 register tile per thread, FFMA.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "k_dgemm.cuh"

namespace hf {
namespace {

constexpr int TBS = 64;          // row block
constexpr int CW = 64;           // RHS chunk width
constexpr int TILE = TBS * TBS;  // elements per 64x64 tile

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

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void wait_epoch(const int *f, int epoch) {
    if (ld_relaxed32(f) != epoch) {
        while (ld_relaxed32(f) != epoch) __nanosleep(20);
    }
    fence_acquire();
}


// ---- precision-generic helpers of the solve bodies (T = float for the paper's FP32
//      preconditioner, T = double for the FP64 one of the (double, dd) pair, NEXT-1)
template <typename T> struct V4 { T x, y, z, w; };
template <typename T> __device__ __forceinline__ V4<T> ld4(const T *p);
template <> __device__ __forceinline__ V4<float> ld4<float>(const float *p) {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    return {v.x, v.y, v.z, v.w};
}
template <> __device__ __forceinline__ V4<double> ld4<double>(const double *p) {
    const double2 a = *reinterpret_cast<const double2 *>(p), b = *reinterpret_cast<const double2 *>(p + 2);
    return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st4(float *p, float a, float b, float c, float d) {
    *reinterpret_cast<float4 *>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st4(double *p, double a, double b, double c, double d) {
    *reinterpret_cast<double2 *>(p) = make_double2(a, b);
    *reinterpret_cast<double2 *>(p + 2) = make_double2(c, d);
}
template <typename T> __device__ __forceinline__ void st4v(T *p, const V4<T> &v) { st4(p, v.x, v.y, v.z, v.w); }
__device__ __forceinline__ float cvt_down(double x, float) { return __double2float_rn(x); }
__device__ __forceinline__ double cvt_down(double x, double) { return x; }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

}  // namespace

namespace p32 {
namespace {
using T = float;
#include "k_trsm_body.cuh"
}  // namespace
}  // namespace p32

namespace p64 {
namespace {
using T = double;
#include "k_trsm_body.cuh"
}  // namespace
}  // namespace p64

// ------------------------------------------------------------------ precision dispatch
void precond_setup(hf_ctx *ctx, Precond &p, const hf_lowfactor *lf) {
    p.prec = lf->prec;
    p.blk = lf->prec != 64 && !lf->nonsym && precond_blocked_enabled();
    if (p.blk) {
        precond_blk_setup(ctx, p.b, lf->N, lf->L, lf->Lfac.p, lf->D.p, lf->perm.p, lf->pos1.p);
        return;
    }
    if (lf->prec == 64)
        p64::precond_setup_t(ctx, p.d, lf->N, lf->L, lf->Lfac64.p, lf->D64.p, lf->perm.p, lf->pos1.p);
    else
        p32::precond_setup_t(ctx, p.f, lf->N, lf->L, lf->Lfac.p, lf->D.p, lf->perm.p, lf->pos1.p,
                             lf->nonsym ? lf->Ufac.p : nullptr);
}

void precond_apply(hf_ctx *ctx, Precond &p, int64_t ncol, const double *R, int64_t ldr, double *W, int64_t ldw) {
    if (p.blk) precond_blk_apply(ctx, p.b, ncol, R, ldr, W, ldw);
    else if (p.prec == 64) p64::precond_apply_t(ctx, p.d, ncol, R, ldr, W, ldw);
    else p32::precond_apply_t(ctx, p.f, ncol, R, ldr, W, ldw);
}

}  // namespace hf
