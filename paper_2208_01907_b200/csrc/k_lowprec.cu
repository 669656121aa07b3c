// k_lowprec.cu -- steps a2/a3: FP32 LDL^T with symmetric max-|diag| pivoting
// and threshold postponing (Alg. 1 step 1; sec. 2.1; sec. 2.2
// P:72-75), rules [R2]-[R10] of DESIGN.md.
//
// B200 design:
//  * Blocked LEFT-looking over panels of nb pivots with a lazily updated
//    diagonal.  No physical row/column swaps: after every panel the active
//    (not yet pivoted) indices are compacted STABLY, so position order equals
//    original-index order and "ties -> smallest original index" [R3] is
//    "ties -> smallest position".
//  * k_chain: one cooperative persistent launch per panel, one CTA per SM.
//    Each CTA owns a contiguous slice of rows and keeps their panel values
//    -sigma_u s_i^u in shared memory.  Per pivot: local argmax -> red.max of
//    a 64-bit key + one release-add on an arrival counter (the only
//    grid-wide exchange) -> the pivot column is assembled
//    from the panel-start matrix plus the in-panel updates, one fmaf per
//    earlier in-panel pivot in increasing order [R8] -> s_i = c_i / sqrt|d|,
//    L_ik = c_i / d, lazy diagonal update.
//  * k_trailing: symmetric rank-nb update of the trailing lower triangle,
//    FP32 FFMA register-tiled (128x128 CTA tile, 8x8 per thread).  Every
//    entry is ONE accumulator seeded from its value and updated with one
//    fmaf per pivot in increasing order -- no split-K, no reassociation, no
//    tensor cores -- which is what makes Pi, D, L bit-identical to the
//    oracle.  The stable compaction is fused into its loads.
//
// Role symmetry: fmaf(-sigma s_I, s_J, v) == fmaf(-sigma s_J, s_I, v) bit for
// bit because the product is exact inside the FMA, so the row/column roles of
// the oracle (right-looking) and of these kernels need not match.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "hf_internal.cuh"

namespace hf {
namespace {

constexpr uint32_t POS_MAX = 0x1FFFF;   // 17-bit position field -> L <= 131071

// ------------------------------------------------------------------ keys
// (|d| bits, smallest position wins ties, sign of d): the unsigned max of the
// keys is the pivot of [R3]; 0 is neutral (no candidate).
__device__ __forceinline__ uint64_t mkkey(float d, uint32_t pos) {
    const uint64_t ab = __float_as_uint(fabsf(d));
    return (ab << 32) | ((uint64_t)(POS_MAX - pos) << 15) | ((uint64_t)(d < 0.f) << 14) | 1ull;
}

__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// unsigned max of a 64-bit key over the warp: two single-instruction reductions
// (redux.sync) on the high word, then on the low word among the lanes holding it
__device__ __forceinline__ uint64_t warp_max64(uint64_t v) {
    const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((uint64_t)mh << 32) | ml;
}

__device__ __forceinline__ void red_release_add(unsigned int *p, unsigned int v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// spin with relaxed loads, acquire once (an ld.acquire per spin iteration
// would invalidate L1 every time)
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_max_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// c <- fmaf(x_u, y_u, c) for u = 0..n-1 in order [R8].  x_u: the own row's panel values in
// shared memory, interleaved by four (x_u at xs[(u >> 2) * R4 + (u & 3)], R4 = 4 x rows per
// CTA: one 16-byte load per thread per four pivots, four wavefronts per warp); y_u = ys[u]
// (broadcast, 16-byte aligned: one 16-byte load per four pivots, one wavefront).  The scalar
// form (one 4-byte load of each operand and an address IMAD per fmaf) was bound by the
// shared-memory wavefronts of the broadcast loads.
__device__ __forceinline__ float fma_chain(float c, const float *xs, const float *ys, int n, int R4) {
    int u = 0;
    for (; u + 8 <= n; u += 8) {
        const float4 x0 = *reinterpret_cast<const float4 *>(xs);
        const float4 x1 = *reinterpret_cast<const float4 *>(xs + R4);
        const float4 y0 = *reinterpret_cast<const float4 *>(ys + u);
        const float4 y1 = *reinterpret_cast<const float4 *>(ys + u + 4);
        xs += 2 * R4;
        c = __fmaf_rn(x0.x, y0.x, c);
        c = __fmaf_rn(x0.y, y0.y, c);
        c = __fmaf_rn(x0.z, y0.z, c);
        c = __fmaf_rn(x0.w, y0.w, c);
        c = __fmaf_rn(x1.x, y1.x, c);
        c = __fmaf_rn(x1.y, y1.y, c);
        c = __fmaf_rn(x1.z, y1.z, c);
        c = __fmaf_rn(x1.w, y1.w, c);
    }
    if (u + 4 <= n) {
        const float4 x0 = *reinterpret_cast<const float4 *>(xs);
        const float4 y0 = *reinterpret_cast<const float4 *>(ys + u);
        xs += R4;
        u += 4;
        c = __fmaf_rn(x0.x, y0.x, c);
        c = __fmaf_rn(x0.y, y0.y, c);
        c = __fmaf_rn(x0.z, y0.z, c);
        c = __fmaf_rn(x0.w, y0.w, c);
    }
    for (int q = 0; u < n; ++u, ++q) c = __fmaf_rn(xs[q], ys[u], c);
    return c;
}
__host__ __device__ __forceinline__ int64_t ceil4(int64_t n) { return (n + 3) & ~(int64_t)3; }

// ------------------------------------------------------------------ cast [R2]
__global__ void k_cast_lower(int64_t L, const double *__restrict__ K, int64_t ldk, float *__restrict__ V,
                             int64_t ldv) {
    for (int64_t j = blockIdx.x; j < L; j += gridDim.x) {
        const double *kc = K + j * ldk;
        float *vc = V + j * ldv;
        for (int64_t i = j + threadIdx.x; i < L; i += blockDim.x) vc[i] = __double2float_rn(kc[i]);
    }
}

__global__ void k_iota32(int64_t n, int32_t *a) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

// ------------------------------------------------------------------ chain
struct ChainArgs {
    int64_t m;          // active size at panel start
    int64_t K0;         // global index of the panel's first pivot
    int nbp;            // pivots to attempt in this panel
    int R;              // rows per CTA (smem stride)
    double tau;
    const float *V;     // trailing matrix (position space), lower triangle
    int64_t ldv;
    const int32_t *orig;  // position -> original index
    float *S;           // S[i + t*lds] = s_i^t (positive sign), this panel
    float *Sn;          // Sn[i + t*lds] = -sigma_t s_i^t
    int64_t lds;
    float *sigma;       // [nb] sign of d_t
    int32_t *pivpos;    // [nb] pivot positions of this panel
    float *Lorig;       // Lorig[orig + k*ldl] = L_{orig,k}
    int64_t ldl;
    float *Dk;          // [L] d_k
    int32_t *pivorig;   // [L] original index of pivot k
    unsigned long long *keys;    // [nbp] per-step max key (zeroed before the launch)    (xmode 0)
    unsigned int *cnt;           // arrival counter (zeroed before the launch)          (xmode 0)
    unsigned long long *slots;   // [2][G][sstride] per-CTA key | step tag (xmode 1)
    int sstride;                 // words between two CTAs' slots (HF_SLOT_STRIDE; 32 = one L2 line each)
    int spec;                    // prefetch the runner-up candidates' columns (HF_CHAIN_SPEC, xmode 1, no blocks)
    int dpoll;                   // two poll rounds in flight (HF_CHAIN_DPOLL)
    int xmode;                   // 0: red.max + counter; 1: spread LL slots (HF_CHAIN_XCHG)
    unsigned long long *mbox;    // [2][G][nb] candidate-row values: float bits << 32 | step tag
    int32_t *status;    // [0] Ntau if stopped, [1] pivots done in last panel, [2] stopped
    // NEXT-4, multi-block postponing: blk[original index] = block number in
    // elimination-tree order, nblk blocks, then the final pass over Lambda_0; bstate =
    // {current block, no pivot accepted yet, exchange attempt counter}
    // carried across panels (null blk: the single-sequence rule)
    const int32_t *blk;
    int nblk;
    int32_t *bstate;
    unsigned long long *dbg;   // optional per-phase time sums (CTA 0), HF_CHAIN_DEBUG
    // lookahead (the previous panel's trailing update runs concurrently): V is the
    // matrix at the START of the previous panel, in its position space; the
    // previous panel's updates of the pivot columns are applied here
    const int32_t *mapprev;   // current position -> previous position (null: none)
    const float *SNprev;      // [prev pos][nbmax] -sigma_u s_i^u of the previous panel
    const float *sigprev;     // [nbprev] sigma of the previous panel
    const float *DGprev;      // [prev pos] lazy diagonal at the end of the previous panel
    int nbprev, nbmax;
    float *SNout;             // [pos][nbmax] this panel's values (for the next panel)
    float *DGout;             // [pos] lazy diagonal at the end of this panel
};

constexpr int SLOT_STRIDE = 32;     // 256 B between slots: no two CTAs' slots share an L2 line
constexpr uint64_t TAGM = 0x3FFF;   // 14-bit step tag in the low bits of every exchanged word
__device__ __forceinline__ uint64_t step_tag(int64_t k) { return (uint64_t)(k % 16383) + 1; }

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Per pivot k = K0 + t (all CTAs in lock step):
//  A  local argmax over own active rows -> CTA key (warp shuffles + smem)
//  B  warp 0: red.max of the key into keys[t], then red.release.add on the
//     arrival counter (the release orders only that red.max);
//     warp 1: the candidate row's panel values to this CTA's mailbox as
//     "LL" words (float bits << 32 | step tag), so no fence orders them --
//     a reader validates every word by its tag (double buffered by step
//     parity, so a fast CTA never overwrites a word a slow one still needs)
//  C  the PREVIOUS step's s / L values of own rows go to global memory now
//  D  one thread per CTA polls the counter, acquires, reads keys[t]
//  E  stop test [R4]; F  pivot-row panel values from the winner's mailbox
//     (tag-checked) and the panel-start column V[:, P] for own rows;
//  G  c_i = chain of fmaf over the earlier in-panel pivots in order [R8],
//     s = c/r, L = c/d, diagonal.
// MAXT: the launch bound (threads = own rows rounded to a warp: 256 at C2, 448 at C4).  A
// bound of 256 / 512 lifts the register cap from 64 to 255 / 128 (108 used at 256): C2 chain
// 52.0 -> 49.5 ms per step, same box, alternating runs.  Software-pipelining the fmaf chain's
// shared loads with those registers was slower (51.6 ms).  HF_CHAIN_LB=1024 forces the
// 1024-thread build.
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_chain(ChainArgs a) {
    extern __shared__ __align__(16) float smem[];
    __shared__ unsigned long long red[32];
    __shared__ unsigned long long bkey;
    __shared__ int32_t spec_p[2];   // speculative next-pivot positions (a.spec)
    if (*(volatile int32_t *)&a.status[2]) return;   // uniform: set by an earlier launch
    const int G = gridDim.x;
    const int tid = threadIdx.x, nthr = blockDim.x, nwarp = nthr >> 5, lane = tid & 31, wid = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * a.R;
    const int64_t nown = max((int64_t)0, min((int64_t)a.R, a.m - r0));
    const int nb = a.nbp;
    const int nbq = a.nbprev;                 // previous panel's pivots (lookahead) or 0
    // panel values interleaved by four (fma_chain): value u of own row r at
    // [(u >> 2) * 4R + 4r + (u & 3)]; every array starts 16-byte aligned
    const int R4 = 4 * a.R;
    auto sx = [&](int u, int r) -> size_t { return (size_t)(u >> 2) * R4 + 4 * r + (u & 3); };
    float *sneg = smem;                            // [nbp][R]  -sigma_u s_i^u for own rows
    float *snp = sneg + (size_t)ceil4(nb) * a.R;   // [nbq][R]  the same for the previous panel
    float *sp = snp + (size_t)ceil4(nbq) * a.R;    // [nbp] s_P^u of the current pivot row
    float *spp = sp + ceil4(nb);                   // [nbq]     s_P^u of the previous panel
    float *sgm = spp + ceil4(nbq);                 // [nbp]     sigma_u

    const bool has = tid < nown;
    const int64_t i = r0 + tid;
    const int64_t io = (has && a.mapprev) ? (int64_t)a.mapprev[i] : i;   // own row in V's position space
    const int32_t oi = has ? a.orig[i] : 0;
    float dg = 0.f;   // lazy diagonal of own row
    if (has) dg = a.DGprev ? a.DGprev[io] : a.V[i + i * a.ldv];
    if (has)
        for (int u = 0; u < nbq; ++u) snp[sx(u, tid)] = a.SNprev[io * a.nbmax + u];
    bool piv = !has;
    float dprev = a.K0 > 0 ? a.Dk[a.K0 - 1] : 0.f;
    const bool BLK = a.blk != nullptr;
    int curblk = BLK ? a.bstate[0] : 0;
    bool first = BLK ? (a.bstate[1] != 0) : (a.K0 == 0);
    int64_t att = BLK ? (int64_t)a.bstate[2] : a.K0;   // exchange attempt: tags and buffer parity
    const int32_t myblk = (BLK && has) ? a.blk[oi] : 0;
    // deferred stores of the previous step
    bool pend = false;
    float ps = 0.f, pn = 0.f, pc = 0.f, pd = 1.f;   // (L = c / d is formed at the deferred store)
    int t = 0;
    bool stopped = false;
    const bool dbg = a.dbg && blockIdx.x == 0 && tid == 0;
    const bool dbga = a.dbg && tid == 0;   // per-CTA phase sums (HF_CHAIN_DEBUG=2: the skew)
    unsigned long long ph[5] = {0, 0, 0, 0, 0}, tp = dbga ? gtimer() : 0;
    uint32_t spec2 = 0xFFFFFFFFu, spec3 = 0xFFFFFFFFu;   // HF_CHAIN_DEBUG speculation statistics
#define PH(q) if (dbga) { unsigned long long n_ = gtimer(); ph[q] += n_ - tp; tp = n_; }
    for (; t < nb;) {
        const int64_t k = a.K0 + t;
        const uint64_t tag = step_tag(att);
        const int par = (int)(att & 1);
        // ---- A: [R3] local argmax of |diag| over own active rows (of the current block)
        const bool cand = !piv && (!BLK || curblk >= a.nblk || myblk == curblk);
        uint64_t key = cand ? mkkey(dg, (uint32_t)i) : 0ull;
        key = warp_max64(key);
        if (lane == 0) red[wid] = key;
        __syncthreads();
        // ---- B: publish
        if (wid < 2) {
            uint64_t v = (lane < nwarp) ? red[lane] : 0ull;
            v = warp_max64(v);
            if (wid == 0) {
                if (lane == 0) {
                    if (a.xmode == 1) {
                        unsigned long long *slot = &a.slots[((size_t)par * G + blockIdx.x) * a.sstride];
                        st_relaxed_u64(slot, (v & ~TAGM) | tag);
                    } else {
                        if (v) red_max_u64(&a.keys[t], v);
                        red_release_add(a.cnt, 1u);
                    }
                }
            } else if (v) {
                unsigned long long *mb = a.mbox + ((size_t)par * G + blockIdx.x) * (nb + 1);
                const int lr = (int)((int64_t)(POS_MAX - (uint32_t)((v >> 15) & POS_MAX)) - r0);
                for (int u = lane; u < t; u += 32)
                    st_relaxed_u64(&mb[u], ((unsigned long long)__float_as_uint(sneg[sx(u, lr)]) << 32) | tag);
            }
        }
        // ---- C: deferred global stores of step t-1
        if (pend) {
            a.S[i + (int64_t)(t - 1) * a.lds] = ps;
            a.Sn[i + (int64_t)(t - 1) * a.lds] = pn;
            a.Lorig[(int64_t)oi + (k - 1) * a.ldl] = __fdiv_rn(pc, pd);   // [R10] L = c / d, off the critical path
            pend = false;
        }
        PH(0)
        // ---- D: wait for all CTAs, read the winning key
        if (a.xmode == 1) {
            if (wid == 1 && a.spec) {
                // speculation: the runner-up and third of this step's per-CTA candidates are
                // the likeliest next pivots (C2: 22 / 33 %); their column entries of this
                // CTA's rows are prefetched into L2 after the barrier (warp 1 polls the same
                // slots as warp 0 and ranks them, off warp 0's path)
                const unsigned long long *sl = a.slots + (size_t)par * G * a.sstride;
                uint64_t v0, v1;
                for (;;) {
                    v0 = lane < G ? ld_relaxed_u64(&sl[(size_t)lane * a.sstride]) : tag;
                    v1 = lane + 32 < G ? ld_relaxed_u64(&sl[(size_t)(lane + 32) * a.sstride]) : tag;
                    if (__all_sync(0xffffffffu, ((v0 & TAGM) == tag) && ((v1 & TAGM) == tag))) break;
                }
                v0 = lane < G ? (v0 & ~TAGM) : 0;
                v1 = lane + 32 < G ? (v1 & ~TAGM) : 0;
                const uint64_t k1 = warp_max64(umax64(v0, v1));
                const uint64_t k2 = warp_max64(umax64(v0 < k1 ? v0 : 0, v1 < k1 ? v1 : 0));
                const uint64_t k3 = warp_max64(umax64(v0 < k2 ? v0 : 0, v1 < k2 ? v1 : 0));
                if (lane == 0) {
                    spec_p[0] = k2 ? (int32_t)(POS_MAX - (uint32_t)((k2 >> 15) & POS_MAX)) : -1;
                    spec_p[1] = k3 ? (int32_t)(POS_MAX - (uint32_t)((k3 >> 15) & POS_MAX)) : -1;
                }
            }
            if (wid == 0) {   // every slot of this step (tags), max = the pivot key; no fence needed
                const unsigned long long *sl = a.slots + (size_t)par * G * a.sstride;
                uint64_t mx;
                if (G <= 64 && a.dpoll) {
                    // two poll rounds in flight (the second issued half a round trip after the
                    // first), so the last slot's arrival is seen sooner; G <= 64: two slots per lane
                    const unsigned long long *s0 = &sl[(size_t)lane * a.sstride];
                    const unsigned long long *s1 = &sl[(size_t)(lane + 32) * a.sstride];
                    const bool h0 = lane < G, h1 = lane + 32 < G;
                    uint64_t a0 = h0 ? ld_relaxed_u64(s0) : tag, a1 = h1 ? ld_relaxed_u64(s1) : tag;
                    uint64_t b0 = h0 ? ld_relaxed_u64(s0) : tag, b1 = h1 ? ld_relaxed_u64(s1) : tag;
                    for (;;) {
                        if (__all_sync(0xffffffffu, ((a0 & TAGM) == tag) && ((a1 & TAGM) == tag))) {
                            mx = umax64(h0 ? a0 : 0, h1 ? a1 : 0);
                            break;
                        }
                        a0 = h0 ? ld_relaxed_u64(s0) : tag;
                        a1 = h1 ? ld_relaxed_u64(s1) : tag;
                        if (__all_sync(0xffffffffu, ((b0 & TAGM) == tag) && ((b1 & TAGM) == tag))) {
                            mx = umax64(h0 ? b0 : 0, h1 ? b1 : 0);
                            break;
                        }
                        b0 = h0 ? ld_relaxed_u64(s0) : tag;
                        b1 = h1 ? ld_relaxed_u64(s1) : tag;
                    }
                } else {
                    for (;;) {
                        bool ok = true;
                        mx = 0;
                        for (int g = lane; g < G; g += 32) {
                            const uint64_t sv = ld_relaxed_u64(&sl[(size_t)g * a.sstride]);
                            ok &= (sv & TAGM) == tag;
                            mx = umax64(mx, sv);
                        }
                        if (__all_sync(0xffffffffu, ok)) break;
                    }
                }
                mx = warp_max64(mx);
                if (lane == 0) bkey = mx;
                if (a.dbg && blockIdx.x == 0) {
                    // speculation statistics: is this step's pivot the runner-up (or third) of
                    // the previous step's per-CTA candidates? (positions; HF_CHAIN_DEBUG only)
                    const unsigned long long *sl = a.slots + (size_t)par * G * a.sstride;
                    uint64_t v0 = lane < G ? (ld_relaxed_u64(&sl[(size_t)lane * a.sstride]) & ~TAGM) : 0;
                    uint64_t v1 = lane + 32 < G ? (ld_relaxed_u64(&sl[(size_t)(lane + 32) * a.sstride]) & ~TAGM) : 0;
                    const uint64_t k1 = warp_max64(umax64(v0, v1));
                    const uint64_t k2 = warp_max64(umax64(v0 < k1 ? v0 : 0, v1 < k1 ? v1 : 0));
                    const uint64_t k3 = warp_max64(umax64(v0 < k2 ? v0 : 0, v1 < k2 ? v1 : 0));
                    const uint32_t p1 = (uint32_t)((k1 >> 15) & POS_MAX);
                    if (lane == 0) {
                        if (t > 0) {
                            a.dbg[7] += 1;
                            if (p1 == spec2) a.dbg[5] += 1;
                            if (p1 == spec2 || p1 == spec3) a.dbg[6] += 1;
                        }
                        spec2 = k2 ? (uint32_t)((k2 >> 15) & POS_MAX) : 0xFFFFFFFFu;
                        spec3 = k3 ? (uint32_t)((k3 >> 15) & POS_MAX) : 0xFFFFFFFFu;
                    }
                }
            }
        } else if (tid == 0) {
            const unsigned int want = (unsigned int)G * (unsigned int)(t + 1);
            while (ld_relaxed_u32(a.cnt) < want) {
            }
            fence_acquire();
            bkey = ld_relaxed_u64(&a.keys[t]);
        }
        __syncthreads();
        const uint64_t bk = bkey;
        PH(1)
        const float absd = __uint_as_float((uint32_t)(bk >> 32));
        const int64_t P = (int64_t)(POS_MAX - (uint32_t)((bk >> 15) & POS_MAX));
        const float d = ((bk >> 14) & 1) ? -absd : absd;
        // ---- E: [R4] stop test, ratio evaluated in FP64, strict, against the previously
        //      accepted pivot (across blocks [R21]; the very first pivot only against 0)
        const bool stop = (bk == 0) || (first ? (absd == 0.f)
                                              : ((double)absd < __dmul_rn(a.tau, fabs((double)dprev))));
        if (stop && BLK && curblk < a.nblk) {   // the rest of this block -> Lambda_0; next block, same step
            ++curblk;
            ++att;
            continue;
        }
        if (stop) {
            if (blockIdx.x == 0 && tid == 0) {
                a.status[0] = (int32_t)k;
                a.status[1] = t;
                a.status[2] = 1;
            }
            stopped = true;
            break;
        }
        const float sg = d > 0.f ? 1.f : -1.f;
        // ---- F: [R6] pivot row from the winner's mailbox, stale column for own rows
        const int64_t Po = a.mapprev ? (int64_t)a.mapprev[P] : P;   // pivot in V's position space
        // the column load is issued first so its latency overlaps the mailbox poll below
        // (one unconditional load from a selected address, its value used only after the
        // barrier below: a conditional load merged into a register stalls the thread here)
        const float *vp = (io >= Po) ? (a.V + io + Po * a.ldv) : (a.V + Po + io * a.ldv);
        const float v = __ldcg((!piv && i != P) ? vp : a.V);
        {
            const int owner = (int)(P / a.R);
            const unsigned long long *mb = a.mbox + ((size_t)par * G + owner) * (nb + 1);
            for (int u = tid; u < t; u += nthr) {
                uint64_t w;
                do {
                    w = ld_relaxed_u64(&mb[u]);
                } while ((w & TAGM) != tag);
                sp[u] = -sgm[u] * __uint_as_float((uint32_t)(w >> 32));   // s_P^u (exact sign flip)
            }
            for (int u = tid; u < nbq; u += nthr) spp[u] = -a.sigprev[u] * a.SNprev[Po * a.nbmax + u];
            if (tid == 0) sgm[t] = sg;
        }
        __syncthreads();
        if (a.spec && !piv) {   // L2 prefetch of this row's entries of the speculative next pivots
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int32_t ps_ = spec_p[q];
                if (ps_ >= 0 && ps_ != (int32_t)P && ps_ < a.m) {
                    const int64_t pso = a.mapprev ? (int64_t)a.mapprev[ps_] : ps_;
                    const float *pp = (io >= pso) ? (a.V + io + pso * a.ldv) : (a.V + pso + io * a.ldv);
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pp));
                }
            }
        }
        PH(2)
        // ---- G: column, scaled column, lazy diagonal
        const float r = __fsqrt_rn(absd);               // [R7]
        if (has && i == P) {
            piv = true;
            a.Dk[k] = d;                                // the owner records the pivot (no loads)
            a.pivorig[k] = oi;
            a.pivpos[t] = (int32_t)P;
            a.sigma[t] = sg;
        } else if (!piv) {
            float c = v;
            c = fma_chain(c, snp + 4 * tid, spp, nbq, R4);   // [R8] the previous panel's pivots first
            c = fma_chain(c, sneg + 4 * tid, sp, t, R4);   // [R8] one fmaf per earlier pivot, in order
            const float sv = __fdiv_rn(c, r);
            const float ns = -sg * sv;                  // exact
            sneg[sx(t, tid)] = ns;
            ps = sv;
            pn = ns;
            pc = c;
            pd = d;
            pend = true;
            dg = __fmaf_rn(ns, sv, dg);                 // lazy diagonal, same fma as the update
        }
        dprev = d;
        first = false;
        ++att;
        ++t;
        PH(3)
    }
    if (pend) {   // flush the last step's values
        a.S[i + (int64_t)(t - 1) * a.lds] = ps;
        a.Sn[i + (int64_t)(t - 1) * a.lds] = pn;
        a.Lorig[(int64_t)oi + (a.K0 + t - 1) * a.ldl] = __fdiv_rn(pc, pd);
    }
    if (!stopped && blockIdx.x == 0 && tid == 0) a.status[1] = t;
    if (BLK && blockIdx.x == 0 && tid == 0) {
        a.bstate[0] = curblk;
        a.bstate[1] = first ? 1 : 0;
        a.bstate[2] = (int32_t)att;
    }
    if (a.SNout && has) {   // this panel's values and the lazy diagonal, for the next panel's lookahead
        for (int u = 0; u < t; ++u) a.SNout[i * a.nbmax + u] = sneg[sx(u, tid)];
        a.DGout[i] = dg;
    }
    if (dbg) {
        for (int q = 0; q < 4; ++q) a.dbg[q] += ph[q];
        a.dbg[4] += t;
    }
    if (dbga)
        for (int q = 0; q < 4; ++q) a.dbg[8 + 4 * blockIdx.x + q] += ph[q];
#undef PH
}

// ------------------------------------------------------------------ exchange floor
// The chain's grid-wide step with nothing else in it (instrumentation, the chain's
// roofline): per step every CTA reduces a key over its threads (warp redux + shared
// memory, as phase A), one thread stores it into its spread slot (phase B) and warp 0
// polls every slot until all carry the step's tag (phase D), then a block barrier.
__global__ void __launch_bounds__(1024, 1) k_xchg_floor(unsigned long long *slots, int sstride, int steps,
                                                       unsigned long long *out) {
    __shared__ unsigned long long red[32], bkey;
    const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
    unsigned long long acc = 0;
    const unsigned long long t0 = gtimer();
    for (int t = 0; t < steps; ++t) {
        const uint64_t tag = step_tag(t);
        const int par = t & 1;
        uint64_t key = mkkey((float)((tid * 7 + t * 13 + blockIdx.x) & 1023), (uint32_t)(blockIdx.x * 1024 + tid));
        key = warp_max64(key);
        if (lane == 0) red[wid] = key;
        __syncthreads();
        if (wid == 0) {
            uint64_t v = lane < nwarp ? red[lane] : 0ull;
            v = warp_max64(v);
            if (lane == 0) st_relaxed_u64(&slots[((size_t)par * G + blockIdx.x) * sstride], (v & ~TAGM) | tag);
            const unsigned long long *sl = slots + (size_t)par * G * sstride;
            uint64_t mx;
            for (;;) {
                bool ok = true;
                mx = 0;
                for (int g = lane; g < G; g += 32) {
                    const uint64_t sv = ld_relaxed_u64(&sl[(size_t)g * sstride]);
                    ok &= (sv & TAGM) == tag;
                    mx = umax64(mx, sv);
                }
                if (__all_sync(0xffffffffu, ok)) break;
            }
            mx = warp_max64(mx);
            if (lane == 0) bkey = mx;
        }
        __syncthreads();
        acc += bkey & 1;
    }
    if (blockIdx.x == 0 && tid == 0) {
        out[0] = gtimer() - t0;
        out[1] = acc;
    }
}

// ------------------------------------------------------------------ compaction
// map[j'] = old position of the j'-th surviving index (stable), norig likewise.
__global__ void k_compact(int64_t m, int nbp, const int32_t *__restrict__ pivpos,
                          const int32_t *__restrict__ orig, int32_t *__restrict__ map,
                          int32_t *__restrict__ norig, const int32_t *status) {
    __shared__ int32_t srt[1024];
    if (status[2]) return;
    for (int q = threadIdx.x; q < nbp; q += blockDim.x) {
        const int32_t v = pivpos[q];
        int rk = 0;
        for (int w = 0; w < nbp; ++w) rk += (pivpos[w] < v);
        srt[rk] = v;
    }
    __syncthreads();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nbp;   // count of pivots < p
        while (lo < hi) {
            int md = (lo + hi) >> 1;
            if (srt[md] < p) lo = md + 1; else hi = md;
        }
        const bool isp = lo < nbp && srt[lo] == p;
        if (!isp) {
            map[p - lo] = (int32_t)p;
            norig[p - lo] = orig[p];
        }
    }
}

// ------------------------------------------------------------------ trailing update
struct TrailArgs {
    int64_t mp;            // new active size
    int nbp;               // pivots in the panel
    const float *Vold;
    float *Vnew;
    int64_t ldv;
    const int32_t *map;    // new position -> old position
    const float *S;        // S[old + t*lds]    =  s_i^t
    const float *Sn;       // Sn[old + t*lds]   = -sigma_t s_i^t
    int64_t lds;
    const int32_t *status;
    int64_t ntiles;        // k_trailing_c: tiles of the launch (persistent CTAs)
    const float *Sc;       // Sc[t*ldc + new]  = s^t of the row at NEW position (compacted panel)
    const float *Snc;      // Snc[t*ldc + new] = -sigma_t s^t
    int64_t ldc;           // multiple of 4; >= the padded tile extent
};

constexpr int TB = 128;    // CTA tile (rows and columns)
constexpr int TK = 16;     // k chunk

// One 128x128 tile of the new lower triangle per CTA, 256 threads, 8x8 entries
// per thread held as 8x4 float2 accumulators and updated with FFMA2
// (__ffma2_rn: two independent IEEE fmaf, bit-identical to the scalar form)
// -- one fused multiply-add per entry per pivot, pivots in increasing order.
__global__ void __launch_bounds__(256, 2) k_trailing(TrailArgs a) {
    if (a.status[2]) return;
    __shared__ __align__(16) float As[2][TK][TB];
    __shared__ __align__(16) float Bs[2][TK][TB];
    __shared__ int32_t rmap[TB], cmap[TB];

    const int64_t t = blockIdx.x;
    int64_t bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int64_t bj = t - bi * (bi + 1) / 2;
    const int64_t row0 = bi * TB, col0 = bj * TB;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int mpr = (int)min((int64_t)TB, a.mp - row0), mpc = (int)min((int64_t)TB, a.mp - col0);

    if (tid < TB) rmap[tid] = (tid < mpr) ? a.map[row0 + tid] : -1;
    else cmap[tid - TB] = (tid - TB < mpc) ? a.map[col0 + tid - TB] : -1;
    __syncthreads();

#define RR(q) (((q) < 4) ? tx * 4 + (q) : 64 + tx * 4 + ((q)-4))
#define CC(q) (((q) < 4) ? ty * 4 + (q) : 64 + ty * 4 + ((q)-4))
    // accumulators seeded from the current values (compaction fused in the gather):
    // one 64-bit column pointer per column, 32-bit row offsets
    float2 acc[8][4];
    {
        int32_t rm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) rm[q] = rmap[RR(q)];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int32_t cm = cmap[CC(2 * j + h)];
                const float *colp = a.Vold + (int64_t)(cm >= 0 ? cm : 0) * a.ldv;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float v = (cm >= 0 && rm[q] >= cm) ? __ldg(colp + rm[q]) : 0.f;
                    if (h) acc[q][j].y = v;
                    else acc[q][j].x = v;
                }
            }
        }
    }

    // global -> register staging: per chunk 8 A (-sigma s) and 8 B (s) values per thread
    const int lr = tid & 127, lk = tid >> 7;   // element (row lr, k = lk + 2*q)
    const int32_t arow = rmap[lr], bcol = cmap[lr];
    const float *Ap = a.Sn + (arow >= 0 ? arow : 0) + (int64_t)lk * a.lds;
    const float *Bp = a.S + (bcol >= 0 ? bcol : 0) + (int64_t)lk * a.lds;
    const int64_t lds2 = 2 * a.lds, ldsk = (int64_t)TK * a.lds;
    const bool aok = arow >= 0, bok = bcol >= 0;
    float ra[TK / 2], rb[TK / 2];
    auto gload = [&](int t0) {
#pragma unroll
        for (int q = 0; q < TK / 2; ++q) {
            const bool ok = t0 + lk + 2 * q < a.nbp;
            ra[q] = (ok && aok) ? __ldg(Ap + q * lds2) : 0.f;
            rb[q] = (ok && bok) ? __ldg(Bp + q * lds2) : 0.f;
        }
        Ap += ldsk;
        Bp += ldsk;
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < TK / 2; ++q) {
            As[buf][lk + 2 * q][lr] = ra[q];
            Bs[buf][lk + 2 * q][lr] = rb[q];
        }
    };

    gload(0);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int t0 = 0; t0 < a.nbp; t0 += TK) {
        const bool more = t0 + TK < a.nbp;
        if (more) gload(t0 + TK);
        const int kmax = min(TK, a.nbp - t0);
        if (kmax == TK) {
#pragma unroll
            for (int kk = 0; kk < TK; ++kk) {
                const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][tx * 4]);
                const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + tx * 4]);
                const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][ty * 4]);
                const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + ty * 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                      make_float2(b1.z, b1.w)};
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[q][j] = __ffma2_rn(make_float2(av[q], av[q]), bv[j], acc[q][j]);
            }
        } else {
            for (int kk = 0; kk < kmax; ++kk) {   // ragged last chunk: exactly nbp updates, no padding
                const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][tx * 4]);
                const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + tx * 4]);
                const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][ty * 4]);
                const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + ty * 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                      make_float2(b1.z, b1.w)};
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[q][j] = __ffma2_rn(make_float2(av[q], av[q]), bv[j], acc[q][j]);
            }
        }
        if (more) {
            sstore(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }

    // store the lower triangle of the new trailing matrix: 16-byte stores on full
    // off-diagonal tiles (rows tx*4..+3 are contiguous), masked scalar stores elsewhere
    const bool full = (row0 > col0) && mpr == TB && mpc == TB && (a.ldv & 3) == 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int cl = CC(2 * j + h);
            float *colp = a.Vnew + (col0 + cl) * a.ldv + row0;
            if (full) {
                *reinterpret_cast<float4 *>(colp + tx * 4) =
                    h ? make_float4(acc[0][j].y, acc[1][j].y, acc[2][j].y, acc[3][j].y)
                      : make_float4(acc[0][j].x, acc[1][j].x, acc[2][j].x, acc[3][j].x);
                *reinterpret_cast<float4 *>(colp + 64 + tx * 4) =
                    h ? make_float4(acc[4][j].y, acc[5][j].y, acc[6][j].y, acc[7][j].y)
                      : make_float4(acc[4][j].x, acc[5][j].x, acc[6][j].x, acc[7][j].x);
            } else if (cl < mpc) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int rl = RR(q);
                    if (rl < mpr && row0 + rl >= col0 + cl) colp[rl] = h ? acc[q][j].y : acc[q][j].x;
                }
            }
        }
    }
#undef RR
#undef CC
}

// The panel in the NEW position space: Sc[t*ldc + new] = S[map[new] + t*lds] (and Sn),
// so the trailing kernel streams contiguous 128-row slices of it with 16-byte cp.async.
__global__ void k_gather_panel(int64_t mp, int nbp, const int32_t *__restrict__ map, const float *__restrict__ S,
                               const float *__restrict__ Sn, int64_t lds, float *__restrict__ Sc,
                               float *__restrict__ Snc, int64_t ldc, const int32_t *status) {
    if (status[2]) return;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= mp) return;
    const int64_t o = map[p];
    const int t0 = blockIdx.y * 16, t1 = min(nbp, t0 + 16);
#pragma unroll 4
    for (int t = t0; t < t1; ++t) {
        Sc[(int64_t)t * ldc + p] = S[o + (int64_t)t * lds];
        Snc[(int64_t)t * ldc + p] = Sn[o + (int64_t)t * lds];
    }
}

__device__ __forceinline__ void cp_async16_s(unsigned sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_g(void *sdst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}

// k_trailing with the panel operands streamed from the compacted panel by 16-byte
// cp.async, three stages in flight (no register staging, no per-element address
// arithmetic); the same single fmaf chain per entry in pivot order.
constexpr int TNS = 3;   // cp.async stages (k_trailing_p)
#ifndef HF_TNSC
#define HF_TNSC 2
#endif
// k_trailing_c's operand stages (TNSC - 1 chunks in flight).  Two stages (32 KB per CTA) beat
// three (48 KB) and four: C2 trailing 29.2 vs 29.8 / 29.8 ms per step (two alternating runs
// each) -- the smaller shared carve-out leaves more L1 to the once-per-tile seed gathers
constexpr int TNSC = HF_TNSC;
constexpr size_t TRAIL_C_SMEM = (size_t)2 * TNSC * TK * TB * sizeof(float);
// NS (NEXT-3, nonsymmetric LDU): the FULL square trailing matrix (T x T tiles),
// A operand -l_I, B operand r_J, v_IJ <- fmaf(-l_I, r_J, v_IJ) [R19].
// TMA (BULK): the panel operands staged by the bulk-copy engine (cp.async.bulk, one 512-byte
// row per instruction, issued by 32 threads per chunk, completion counted in bytes on a
// per-stage mbarrier) instead of 16-byte cp.async from every thread.
// BULK = 2: one 2D tensor copy (cp.async.bulk.tensor, a 16 x 128 box) per operand per chunk
// through the tensor maps tmA (Snc) / tmB (Sc).
template <bool NS, int BULK = 0>
__global__ void __launch_bounds__(256, 2) k_trailing_c(TrailArgs a, const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB) {
    if (a.status[2]) return;
    extern __shared__ __align__(16) float dsm_t[];   // [TNSC][TK][TB] x 2 (48 KB: dynamic)
    // the tensor copies need 128 B aligned destinations; the dynamic window starts 32 B past
    // one (measured), so BULK = 2 launches with 128 B more and rounds up
    float *dsm = BULK == 2 ? reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(dsm_t) + 127) & ~uintptr_t(127))
                           : dsm_t;
    float (*As)[TK][TB] = reinterpret_cast<float (*)[TK][TB]>(dsm);
    float (*Bs)[TK][TB] = reinterpret_cast<float (*)[TK][TB]>(dsm + TNSC * TK * TB);
    __shared__ int32_t rmap[TB], cmap[TB];
    __shared__ __align__(8) unsigned long long mbar[TNSC];   // BULK: one per operand stage
    // persistent: CTA b takes tiles b, b + grid, ... (the order of the one-tile-per-CTA
    // launch); the next tile's compaction-map entry is loaded into a register while the
    // current tile computes, so a tile's seed gather waits for one memory latency, not two
    auto tile_of = [&](int64_t t, int64_t &bi, int64_t &bj) {
        if (NS) {
            const int64_t T = (a.mp + TB - 1) / TB;
            bi = t % T;
            bj = t / T;
        } else {
            bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
            while (bi * (bi + 1) / 2 > t) --bi;
            while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
            bj = t - bi * (bi + 1) / 2;
        }
    };
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    auto map_entry = [&](int64_t t) -> int32_t {   // this thread's rmap / cmap entry of tile t
        int64_t bi, bj;
        tile_of(t, bi, bj);
        const int64_t base = (tid < TB ? bi : bj) * TB + (tid & (TB - 1));
        return base < a.mp ? a.map[base] : -1;
    };
    int64_t t = blockIdx.x;
    if (t >= a.ntiles) return;
    {
        const int32_t m0 = map_entry(t);
        if (tid < TB) rmap[tid] = m0;
        else cmap[tid - TB] = m0;
    }
    for (;;) {
    int64_t bi, bj;
    tile_of(t, bi, bj);
    const int64_t row0 = bi * TB, col0 = bj * TB;
    const int mpr = (int)min((int64_t)TB, a.mp - row0), mpc = (int)min((int64_t)TB, a.mp - col0);
    const int nchunk = (a.nbp + TK - 1) / TK;

    // chunk c -> stage c % TNSC: TK pivots x 128 positions of each operand, 2 x 16 B per
    // thread each.  The four source pointers advance by one chunk per issue (64-bit adds
    // on the ALU pipe) and the stage rotates: no per-chunk multiplies or modulo on the FMA
    // pipe, which the update saturates (IMAD runs on it, rt 2 like FFMA2).
    // (piece 2 of a thread is piece 1 eight panel rows further: + 8 ldc in global memory,
    // + 8 TB floats in shared memory)
    const int ek0 = tid >> 5, er0 = (tid & 31) * 4;
    const float *pa = a.Snc + (int64_t)ek0 * a.ldc + row0 + er0;
    const float *pb = a.Sc + (int64_t)ek0 * a.ldc + col0 + er0;
    const int64_t cstride = (int64_t)TK * a.ldc, eight = (int64_t)8 * a.ldc;
    const unsigned sA = (unsigned)__cvta_generic_to_shared(&As[0][ek0][er0]);
    const unsigned sB = (unsigned)__cvta_generic_to_shared(&Bs[0][ek0][er0]);
    constexpr unsigned STGB = TK * TB * sizeof(float), EIGHTB = 8 * TB * sizeof(float);
    unsigned soff = 0;   // stage of the next issue, in bytes
    int sidx = 0;        // its index
    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(&mbar[0]);
    auto issue = [&](int c) {
        if (BULK == 2) {
            if (c < nchunk && tid == 0) {
                const unsigned mb = mb0 + 8u * (unsigned)sidx;
                const unsigned dA = (unsigned)__cvta_generic_to_shared(&As[0][0][0]) + soff;
                const unsigned dB = (unsigned)__cvta_generic_to_shared(&Bs[0][0][0]) + soff;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                             "r"((unsigned)(2 * TK * TB * sizeof(float))) : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(dA), "l"(&tmA), "r"((int)row0), "r"(c * TK), "r"(mb) : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(dB), "l"(&tmB), "r"((int)col0), "r"(c * TK), "r"(mb) : "memory");
            }
        } else if (BULK) {
            if (c < nchunk && tid < 2 * TK) {
                // thread k < 16: row k of the A operand; 16 <= k < 32: row k - 16 of B
                const int k = tid & (TK - 1);
                const bool isb = tid >= TK;
                const unsigned dst = (isb ? (unsigned)__cvta_generic_to_shared(&Bs[0][0][0])
                                          : (unsigned)__cvta_generic_to_shared(&As[0][0][0])) +
                                     soff + (unsigned)(k * TB * sizeof(float));
                const float *src = (isb ? a.Sc + col0 : a.Snc + row0) + (int64_t)(c * TK + k) * a.ldc;
                const unsigned mb = mb0 + 8u * (unsigned)sidx;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // after the generic reads
                if (tid == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                                 "r"((unsigned)(2 * TK * TB * sizeof(float))) : "memory");
                __syncwarp();
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(dst), "l"(src), "r"((unsigned)(TB * sizeof(float))), "r"(mb) : "memory");
            }
        } else {
            if (c < nchunk) {
                cp_async16_s(sA + soff, pa);
                cp_async16_s(sA + soff + EIGHTB, pa + eight);
                cp_async16_s(sB + soff, pb);
                cp_async16_s(sB + soff + EIGHTB, pb + eight);
                pa += cstride;
                pb += cstride;
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        soff = (soff == (TNSC - 1) * STGB) ? 0u : soff + STGB;
        sidx = (sidx == TNSC - 1) ? 0 : sidx + 1;
    };
    if (BULK && tid == 0) {   // the stage mbarriers: one arrival (the expect_tx) per use
        for (int q = 0; q < TNSC; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8u * q) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (BULK) __syncthreads();
    unsigned phase_bits = 0;   // BULK: parity of each stage's next completion
#pragma unroll
    for (int q = 0; q < TNSC - 1; ++q) issue(q);
    __syncthreads();   // this tile's maps (stored before the loop or at the end of the previous tile)

#define RR(q) (((q) < 4) ? tx * 4 + (q) : 64 + tx * 4 + ((q)-4))
#define CC(q) (((q) < 4) ? ty * 4 + (q) : 64 + ty * 4 + ((q)-4))
    float2 acc[8][4];
    // an interior tile (strictly below the diagonal, no ragged edge; every tile but the edges
    // for NS): all 64 seeds exist, so no masks; the column bases are computed once and kept
    // as 64-bit pointers for the row offsets (fewer FMA-pipe IMADs and parameter reloads)
    const bool interior = (NS || row0 > col0) && mpr == TB && mpc == TB;
    if (interior) {
        int32_t rm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) rm[q] = rmap[RR(q)];
        const float *vold = a.Vold;
        const int64_t ldv = a.ldv;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float *c0p = vold + (int64_t)cmap[CC(2 * j)] * ldv;
            const float *c1p = vold + (int64_t)cmap[CC(2 * j + 1)] * ldv;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                acc[q][j].x = __ldg(c0p + rm[q]);
                acc[q][j].y = __ldg(c1p + rm[q]);
            }
        }
    } else {
        int32_t rm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) rm[q] = rmap[RR(q)];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int32_t cm = cmap[CC(2 * j + h)];
                const float *colp = a.Vold + (int64_t)(cm >= 0 ? cm : 0) * a.ldv;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const bool ok = NS ? (cm >= 0 && rm[q] >= 0) : (cm >= 0 && rm[q] >= cm);
                    const float v = ok ? __ldg(colp + rm[q]) : 0.f;
                    if (h) acc[q][j].y = v;
                    else acc[q][j].x = v;
                }
            }
        }
    }

    const int64_t tn = t + gridDim.x;
    const int32_t mnext = tn < a.ntiles ? map_entry(tn) : -1;   // consumed after the main loop
    int st = 0;   // stage of chunk c
    for (int c = 0; c < nchunk; ++c, st = (st == TNSC - 1) ? 0 : st + 1) {
        if (BULK) {
            const unsigned mb = mb0 + 8u * (unsigned)st;
            const unsigned ph = (phase_bits >> st) & 1u;
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(mb), "r"(ph) : "memory");
            phase_bits ^= 1u << st;
            __syncthreads();                // every thread is done with stage (c+2)%3 (read in c-1)
        } else {
            asm volatile("cp.async.wait_group %0;" ::"n"(TNSC - 2) : "memory");
            __syncthreads();                // chunk c landed for all threads; stage (c-1)%TNSC is free
        }
        issue(c + TNSC - 1);
        const int kmax = min(TK, a.nbp - c * TK);
        if (kmax == TK) {
#pragma unroll
            for (int kk = 0; kk < TK; ++kk) {
                const float4 a0 = *reinterpret_cast<const float4 *>(&As[st][kk][tx * 4]);
                const float4 a1 = *reinterpret_cast<const float4 *>(&As[st][kk][64 + tx * 4]);
                const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[st][kk][ty * 4]);
                const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[st][kk][64 + ty * 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                      make_float2(b1.z, b1.w)};
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[q][j] = __ffma2_rn(make_float2(av[q], av[q]), bv[j], acc[q][j]);
            }
        } else {
            for (int kk = 0; kk < kmax; ++kk) {   // ragged last chunk: exactly nbp updates
                const float4 a0 = *reinterpret_cast<const float4 *>(&As[st][kk][tx * 4]);
                const float4 a1 = *reinterpret_cast<const float4 *>(&As[st][kk][64 + tx * 4]);
                const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[st][kk][ty * 4]);
                const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[st][kk][64 + ty * 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                      make_float2(b1.z, b1.w)};
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[q][j] = __ffma2_rn(make_float2(av[q], av[q]), bv[j], acc[q][j]);
            }
        }
    }

    const bool full = (NS || row0 > col0) && mpr == TB && mpc == TB && (a.ldv & 3) == 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int cl = CC(2 * j + h);
            float *colp = a.Vnew + (col0 + cl) * a.ldv + row0;
            if (full) {
                *reinterpret_cast<float4 *>(colp + tx * 4) =
                    h ? make_float4(acc[0][j].y, acc[1][j].y, acc[2][j].y, acc[3][j].y)
                      : make_float4(acc[0][j].x, acc[1][j].x, acc[2][j].x, acc[3][j].x);
                *reinterpret_cast<float4 *>(colp + 64 + tx * 4) =
                    h ? make_float4(acc[4][j].y, acc[5][j].y, acc[6][j].y, acc[7][j].y)
                      : make_float4(acc[4][j].x, acc[5][j].x, acc[6][j].x, acc[7][j].x);
            } else if (cl < mpc) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int rl = RR(q);
                    if (rl < mpr && (NS || row0 + rl >= col0 + cl)) colp[rl] = h ? acc[q][j].y : acc[q][j].x;
                }
            }
        }
    }
    __syncthreads();   // every thread is done with this tile's maps and operand stages
    if (tn >= a.ntiles) break;
    if (tid < TB) rmap[tid] = mnext;
    else cmap[tid - TB] = mnext;
    t = tn;
    }
#undef RR
#undef CC
}

// Persistent form of k_trailing_c (symmetric): two CTAs per SM walk the lower-triangle
// tiles t = blockIdx.x, + gridDim.x, ...  While a tile is computed, each thread gathers the
// 64 start values (seeds) IT will need for its next tile into shared memory with 4-byte
// cp.async (zero-filled outside the triangle), so the scattered gather through the
// compaction map -- most of a tile's non-FMA time in k_trailing_c -- overlaps the FMA
// loop.  Each thread reads back only what it gathered itself: no barrier on the seed
// buffer.  Same single fmaf chain per entry in pivot order (bit-identical).
constexpr size_t TRAIL_P_SMEM = (size_t)2 * TNS * TK * TB * sizeof(float) + (size_t)TB * TB * sizeof(float);   // + seeds
__device__ __forceinline__ void cp_async4_z(void *sdst, const void *gsrc, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gsrc), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void tile_of(int64_t t, int64_t &bi, int64_t &bj) {
    bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    bj = t - bi * (bi + 1) / 2;
}
__global__ void __launch_bounds__(256, 2) k_trailing_p(TrailArgs a, int64_t ntiles) {
    if (a.status[2]) return;
    extern __shared__ __align__(16) float dsm_t[];
    float (*As)[TK][TB] = reinterpret_cast<float (*)[TK][TB]>(dsm_t);
    float (*Bs)[TK][TB] = reinterpret_cast<float (*)[TK][TB]>(dsm_t + TNS * TK * TB);
    float *Sd = dsm_t + 2 * TNS * TK * TB;   // [TB cols][TB rows] seeds of the current tile
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int nchunk = (a.nbp + TK - 1) / TK;
#define RR(q) (((q) < 4) ? tx * 4 + (q) : 64 + tx * 4 + ((q)-4))
#define CC(q) (((q) < 4) ? ty * 4 + (q) : 64 + ty * 4 + ((q)-4))
    // this thread's 64 seeds of tile t -> Sd (its own entries only), one commit group
    auto gather = [&](int64_t t) {
        if (t < ntiles) {
            int64_t bi, bj;
            tile_of(t, bi, bj);
            const int64_t row0 = bi * TB, col0 = bj * TB;
            int32_t rm[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) rm[q] = (row0 + RR(q) < a.mp) ? a.map[row0 + RR(q)] : -1;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int cl = CC(c);
                const int32_t cm = (col0 + cl < a.mp) ? a.map[col0 + cl] : -1;
                const float *colp = a.Vold + (int64_t)(cm >= 0 ? cm : 0) * a.ldv;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const bool ok = cm >= 0 && rm[q] >= cm;
                    cp_async4_z(&Sd[cl * TB + RR(q)], ok ? colp + rm[q] : a.Vold, ok);
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    gather(blockIdx.x);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int64_t bi, bj;
        tile_of(t, bi, bj);
        const int64_t row0 = bi * TB, col0 = bj * TB;
        const int mpr = (int)min((int64_t)TB, a.mp - row0), mpc = (int)min((int64_t)TB, a.mp - col0);
        auto issue = [&](int c) {
            if (c < nchunk) {
                const int st = c % TNS;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int e = tid + u * 256;
                    const int k = e >> 5, r4 = (e & 31) * 4;
                    const int64_t off = (int64_t)(c * TK + k) * a.ldc;
                    cp_async16_g(&As[st][k][r4], a.Snc + off + row0 + r4);
                    cp_async16_g(&Bs[st][k][r4], a.Sc + off + col0 + r4);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // the previous tile's readers of the operand stages are done (barrier at its loop end)
        issue(0);
        issue(1);
        // groups now: [seeds(t)], chunk0, chunk1 -> seeds(t) complete
        asm volatile("cp.async.wait_group 2;" ::: "memory");
        float2 acc[8][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float *sc = Sd + CC(2 * j + h) * TB;
                const float4 lo = *reinterpret_cast<const float4 *>(sc + tx * 4);
                const float4 hi = *reinterpret_cast<const float4 *>(sc + 64 + tx * 4);
                const float v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (h) acc[q][j].y = v[q];
                    else acc[q][j].x = v[q];
                }
            }
        }
        for (int c = 0; c < nchunk; ++c) {
            // commit order: chunk0, chunk1, [wait c=0] chunk2, seeds(next), [c=1] chunk3, [c=2]
            // chunk4, ... -> chunk c is complete when at most 1 (c = 0), 2 (c = 1, 2) or
            // 1 (c >= 3) newer groups are pending
            if (c == 1 || c == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
            else asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
            issue(c + 2);
            const int st = c % TNS;
            const int kmax = min(TK, a.nbp - c * TK);
            if (kmax == TK) {
#pragma unroll
                for (int kk = 0; kk < TK; ++kk) {
                    const float4 a0 = *reinterpret_cast<const float4 *>(&As[st][kk][tx * 4]);
                    const float4 a1 = *reinterpret_cast<const float4 *>(&As[st][kk][64 + tx * 4]);
                    const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[st][kk][ty * 4]);
                    const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[st][kk][64 + ty * 4]);
                    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                          make_float2(b1.z, b1.w)};
#pragma unroll
                    for (int q = 0; q < 8; ++q)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[q][j] = __ffma2_rn(make_float2(av[q], av[q]), bv[j], acc[q][j]);
                }
            } else {
                for (int kk = 0; kk < kmax; ++kk) {
                    const float4 a0 = *reinterpret_cast<const float4 *>(&As[st][kk][tx * 4]);
                    const float4 a1 = *reinterpret_cast<const float4 *>(&As[st][kk][64 + tx * 4]);
                    const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[st][kk][ty * 4]);
                    const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[st][kk][64 + ty * 4]);
                    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                          make_float2(b1.z, b1.w)};
#pragma unroll
                    for (int q = 0; q < 8; ++q)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[q][j] = __ffma2_rn(make_float2(av[q], av[q]), bv[j], acc[q][j]);
                }
            }
            // the next tile's seeds into this thread's own Sd entries: issued after the first
            // chunk's FMAs consumed the values read from them
            if (c == 0) gather(t + gridDim.x);
        }
        __syncthreads();   // every thread is done with the operand stages before the next tile's issue
        const bool full = row0 > col0 && mpr == TB && mpc == TB && (a.ldv & 3) == 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cl = CC(2 * j + h);
                float *colp = a.Vnew + (col0 + cl) * a.ldv + row0;
                if (full) {
                    *reinterpret_cast<float4 *>(colp + tx * 4) =
                        h ? make_float4(acc[0][j].y, acc[1][j].y, acc[2][j].y, acc[3][j].y)
                          : make_float4(acc[0][j].x, acc[1][j].x, acc[2][j].x, acc[3][j].x);
                    *reinterpret_cast<float4 *>(colp + 64 + tx * 4) =
                        h ? make_float4(acc[4][j].y, acc[5][j].y, acc[6][j].y, acc[7][j].y)
                          : make_float4(acc[4][j].x, acc[5][j].x, acc[6][j].x, acc[7][j].x);
                } else if (cl < mpc) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int rl = RR(q);
                        if (rl < mpr && row0 + rl >= col0 + cl) colp[rl] = h ? acc[q][j].y : acc[q][j].x;
                    }
                }
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#undef RR
#undef CC
}

// ------------------------------------------------------------------ partitioned trailing update
// ------------------------------------------------------------------ factor gather
// Lfac[a + k*N] = Lorig[pivorig[a] + k*ldl] (a > k), 1 (a == k), 0 (a < k)
__global__ void k_gather_L(int64_t N, const int32_t *__restrict__ pivorig, const float *__restrict__ Lorig,
                           int64_t ldl, float *__restrict__ Lfac, int64_t ldf) {
    for (int64_t k = blockIdx.x; k < N; k += gridDim.x) {
        const float *src = Lorig + k * ldl;
        float *dst = Lfac + k * ldf;
        for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
            float v = 0.f;
            if (r == k) v = 1.f;
            else if (r > k) v = src[pivorig[r]];
            dst[r] = v;
        }
    }
}

}  // namespace

// ------------------------------------------------------------------ host driver
// tensor map of a compacted panel buffer (ldc positions x nrows pivots, FP32, row = one
// pivot's values): the 2D TMA box of the trailing update is 128 positions x 16 pivots
static void make_panel_tmap(CUtensorMap *m, const float *base, int64_t ldc, int64_t nrows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        HF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        HF_REQUIRE(fn && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)ldc, (cuuint64_t)nrows};
    const cuuint64_t strides[1] = {(cuuint64_t)ldc * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)TB, (cuuint32_t)TK};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error{HF_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
}

// algorithmic work per launch, reported through hf_kernel_work:
//  trailing update of a panel of nbp pivots leaving mp active indices: one FMA per
//    lower-triangle entry (diagonal included) per pivot; bytes = the triangle read
//    and written once plus the two panel operands;
//  chain: per pivot t of the panel, the column c_I of every active row brought up to
//    date over the t earlier in-panel pivots (one FMA each), and 16 bytes per row
//    (the panel-start column read, s, -sigma s, L written).
static double trail_flops(int64_t mp, int nbp) { return (double)mp * (double)(mp + 1) * nbp; }
static double trail_bytes(int64_t mp, int nbp) { return (double)mp * (mp + 1) * 4.0 + 8.0 * mp * nbp; }
static double chain_flops(int64_t m, int nbp) {
    double f = 0.0;
    for (int t = 0; t < nbp; ++t) f += 2.0 * (double)(m - t) * t;
    return f;
}
static double chain_bytes(int64_t m, int nbp) { return 16.0 * ((double)m * nbp - 0.5 * (double)nbp * (nbp - 1)); }
// N, Pi, D (host and device) and the factor buffer of lf from the chain's outputs
// (status = {N_tau if stopped, -, stopped}, pivorig, Dk); the caller gathers the factor
void lowprec_outputs(hf_ctx *ctx, int64_t L, const hf_lowprec_opts &o, hf_lowfactor *lf, const int32_t *status,
                     const int32_t *pivorig, const float *Dk) {
    cudaStream_t st = ctx->stream;
    int32_t hs[4];
    HF_CUDA(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    if (hs[3] != 0) throw Error{HF_ERR_NCCL, "stage 1: a peer did not answer within the exchange timeout (multi-GPU chain)"};
    const int64_t Ntau = hs[2] ? hs[0] : L;
    // [R5] floor and [R9] enlargement: the last accepted pivots move to Lambda_2
    int64_t N = Ntau;
    if (L - o.n_min < N) N = std::max<int64_t>(0, L - o.n_min);
    if (N < L) N = std::max<int64_t>(0, N - o.n_extra);
    lf->Ntau = Ntau;
    lf->N = N;
    lf->n2 = L - N;

    // [R10] Pi = [pivots, Lambda_2 ascending]
    std::vector<int32_t> po(std::max<int64_t>(N, 1));
    if (N > 0) HF_CUDA(cudaMemcpyAsync(po.data(), pivorig, N * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    lf->h_D.assign(std::max<int64_t>(N, 1), 0.f);
    if (N > 0) HF_CUDA(cudaMemcpyAsync(lf->h_D.data(), Dk, N * sizeof(float), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    lf->h_D.resize(N);
    std::vector<int32_t> rank(L, -1);
    lf->h_perm.resize(L);
    for (int64_t k = 0; k < N; ++k) {
        lf->h_perm[k] = po[k];
        rank[po[k]] = (int32_t)k;
    }
    int64_t w = N;
    for (int64_t i = 0; i < L; ++i)
        if (rank[i] < 0) lf->h_perm[w++] = i;
    lf->perm.alloc(L, st);
    lf->pos1.alloc(L, st);
    HF_CUDA(cudaMemcpyAsync(lf->perm.p, lf->h_perm.data(), L * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    HF_CUDA(cudaMemcpyAsync(lf->pos1.p, rank.data(), L * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    lf->D.alloc(std::max<int64_t>(N, 1), st);
    if (N > 0) HF_CUDA(cudaMemcpyAsync(lf->D.p, Dk, N * sizeof(float), cudaMemcpyDeviceToDevice, st));
    lf->Lfac.alloc((size_t)std::max<int64_t>(N, 1) * std::max<int64_t>(N, 1), st);
    HF_CUDA(cudaStreamSynchronize(st));   // host vectors used by the copies above must outlive them
}

static void lowprec_finish(hf_ctx *ctx, int64_t L, const hf_lowprec_opts &o, hf_lowfactor *lf, DBuf<int32_t> &status,
                           DBuf<int32_t> &pivorig, DBuf<float> &Dk, DBuf<float> &Lorig, DBuf<unsigned long long> *dbg) {
    cudaStream_t st = ctx->stream;
    if (dbg) {
        unsigned long long hd[8];
        HF_CUDA(cudaMemcpy(hd, dbg->p, sizeof(hd), cudaMemcpyDeviceToHost));
        const double np = hd[4] ? (double)hd[4] : 1.0;
        {   // per-CTA sums: min / mean / max over the chain CTAs of every phase
            std::vector<unsigned long long> pc((size_t)4 * ctx->num_sms);
            HF_CUDA(cudaMemcpy(pc.data(), dbg->p + 8, pc.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            int nact = 0;
            for (int b = 0; b < ctx->num_sms; ++b) nact += pc[(size_t)4 * b] > 0;
            for (int q = 0; q < 4; ++q) {
                double mn = 1e30, mx = 0.0, sm = 0.0;
                for (int b = 0; b < nact; ++b) {
                    const double v = pc[(size_t)4 * b + q] / np * 1e-3;
                    mn = std::min(mn, v);
                    mx = std::max(mx, v);
                    sm += v;
                }
                fprintf(stderr, "[hf chain] phase %d over %d CTAs: min %.3f mean %.3f max %.3f us/step\n", q, nact, mn,
                        sm / std::max(nact, 1), mx);
            }
        }
        fprintf(stderr, "[hf chain] steps %llu  us/step: publish %.3f  exchange %.3f  fetch %.3f  compute %.3f\n",
                hd[4], hd[0] / np * 1e-3, hd[1] / np * 1e-3, hd[2] / np * 1e-3, hd[3] / np * 1e-3);
        if (hd[7])
            fprintf(stderr, "[hf chain] pivot = previous step's runner-up candidate: %.1f %%, runner-up or third: %.1f %%\n",
                    100.0 * hd[5] / hd[7], 100.0 * hd[6] / hd[7]);
    }
    lowprec_outputs(ctx, L, o, lf, status.p, pivorig.p, Dk.p);
    const int64_t N = lf->N;
    if (N > 0) {
        ClassTimer tm(ctx, "other");
        k_gather_L<<<(unsigned)std::min<int64_t>(N, 65535), 256, 0, st>>>(N, pivorig.p, Lorig.p, L, lf->Lfac.p, N);
        HF_CHECK_LAUNCH(ctx);
    }
    HF_CUDA(cudaStreamSynchronize(st));
}

void lowprec_factor(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                    hf_lowfactor *lf, const int32_t *blk_host, int nblk_in) {
    cudaStream_t st = ctx->stream;
    const int nsm = ctx->num_sms;
    const int o_nblk = blk_host ? nblk_in : 0;   // NEXT-4: multi-block postponing
    lf->L = L;
    lf->stream = st;
    if (L == 0) {
        lf->N = lf->Ntau = lf->n2 = 0;
        return;
    }
    HF_REQUIRE(L <= (int64_t)POS_MAX - 1, "L too large for the 17-bit position key");

    // panel width: the chain keeps R x nb floats per CTA in shared memory
    int maxsmem = 0;
    HF_CUDA(cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    cudaFuncAttributes fa;
    HF_CUDA(cudaFuncGetAttributes(&fa, k_chain<1024>));
    maxsmem -= (int)fa.sharedSizeBytes;
    // Chain geometry (measured on B200 at C2, chain + trailing ms: 148 CTAs / nb 256: 106.3,
    // 148 / 128: 103.3, 74 / 128: 100.6, 64 / 128: 95.0, 64 / 192: 95.8, 32 / 96: 98.8):
    // fewer CTAs make the per-pivot exchange cheaper until the rows per CTA no longer fit the
    // panel in shared memory, so G = max(64, L / rows-that-fit) CTAs.
    // nb = 160 (measured at C2 with the streaming trailing kernel, chain + trailing + other ms:
    // nb 128: 88.4, 160: 87.9, 192: 87.9; the trailing update alone 32.2 / 30.9 / 29.6)
    const int nb_def = 160;
    // Lookahead (HF_LOOKAHEAD=1, off by default): the chain of panel p+1 runs while panel
    // p's trailing update runs on a second stream, applying panel p's updates to its pivot
    // columns itself (the same fmaf, so the bits do not change).  Measured at C2: 103 ms
    // (chain 5.5 us/pivot: the concurrent update's memory traffic slows every exchange and
    // column read) against 99 ms serial, so the serial schedule is the default.
    const bool look = !blk_host && getenv("HF_LOOKAHEAD") && atoi(getenv("HF_LOOKAHEAD")) != 0;
    const int64_t per_row = look ? 2 * nb_def + 3 : nb_def + 2;   // floats of shared memory per row
    int gmax = (int)std::min<int64_t>(nsm, std::max<int64_t>(64, cdiv(L, (int64_t)(maxsmem / 4 / per_row))));
    if (const char *e = getenv("HF_CHAIN_CTAS")) gmax = std::max(1, std::min(nsm, atoi(e)));
    const int64_t G0 = std::min<int64_t>(gmax, std::max<int64_t>(1, cdiv(L, 32)));
    const int64_t R0 = cdiv(L, G0);
    HF_REQUIRE(R0 <= 1024, "L too large for one chain CTA per SM (R > 1024)");
    int nb = o.nb > 0 ? o.nb : nb_def;
    if (o.nb <= 0 && getenv("HF_NB")) nb = std::max(8, atoi(getenv("HF_NB")));   // sweeps
    // with lookahead the chain holds both panels' values of its rows in shared memory
    const int nbf = (look ? 2 : 1);
    // the widest multiple of 16 (the trailing kernel's k chunk) that fits, e.g. 112 at C4
    auto chain_fits = [&](int w) { return (int64_t)(nbf * ceil4(w) * R0 + 3 * ceil4(w) + 4) * 4 <= (int64_t)maxsmem; };
    while (nb > 16 && !chain_fits(nb)) nb -= 16;
    while (nb > 8 && !chain_fits(nb)) nb /= 2;
    HF_REQUIRE(nb >= 8 && nb <= 1024, "panel width out of range");

    DBuf<float> V[2];
    V[0].alloc((size_t)L * L, st);
    V[1].alloc((size_t)L * L, st);
    DBuf<int32_t> orig[2], map[2];
    orig[0].alloc(L, st);
    orig[1].alloc(L, st);
    map[0].alloc(L, st);
    if (look) map[1].alloc(L, st);
    DBuf<float> S[2], Sn[2], sigma[2], SNrow[2], DG[2], Lorig, Dk, Sc, Snc;
    const int64_t ldc = cdiv(L, TB) * TB;   // compacted panel: padded to whole 128-row tiles
    for (int b = 0; b < (look ? 2 : 1); ++b) {
        S[b].alloc((size_t)L * nb, st);
        Sn[b].alloc((size_t)L * nb, st);
        sigma[b].alloc(nb, st);
        if (b == 0) {   // the compacted panel of the streaming trailing kernel (gathered on its stream)
            Sc.alloc((size_t)ldc * cdiv(nb, TK) * TK, st);
            Snc.alloc((size_t)ldc * cdiv(nb, TK) * TK, st);
        }
        if (look) {
            SNrow[b].alloc((size_t)L * nb, st);
            DG[b].alloc(L, st);
        }
    }
    Lorig.alloc((size_t)L * L, st);
    Dk.alloc(L, st);
    DBuf<int32_t> pivpos, pivorig, status;
    pivpos.alloc(nb, st);
    pivorig.alloc(L, st);
    status.alloc(4, st);
    // per-launch exchange state: keys[nb] + counter, zeroed before every chain launch;
    // mailbox words are tagged (self-validating), zeroed once
    DBuf<unsigned long long> xchg, mbox, slots;
    xchg.alloc((size_t)nb + 2, st);
    mbox.alloc((size_t)2 * nsm * (nb + 1), st);
    mbox.zero(st);
    int sstride = SLOT_STRIDE;
    // HF_CHAIN_SPEC=1: L2 prefetch of the runner-up candidates' columns (measured slower at C2:
    // chain 53.3 vs 51.5 ms -- a 22-33 % hit rate does not pay for the extra poll and traffic)
    int chain_spec = 0;
    if (const char *e = getenv("HF_CHAIN_SPEC")) chain_spec = atoi(e);
    // HF_CHAIN_DPOLL=1: two poll rounds in flight (measured 52.5 vs 52.1 ms chain at C2: off;
    // with the launch bound matched to the block: 49.2 / 49.2 / 49.8 / 49.2 vs 49.5 / 49.7 /
    // 49.4 / 49.4 ms over four alternating pairs -- within the run-to-run spread, still off)
    int chain_dpoll = 0;
    if (const char *e = getenv("HF_CHAIN_DPOLL")) chain_dpoll = atoi(e);
    if (const char *e = getenv("HF_SLOT_STRIDE")) sstride = std::max(1, std::min(64, atoi(e)));
    slots.alloc((size_t)2 * nsm * SLOT_STRIDE, st);
    slots.zero(st);
    int xmode = 1;
    if (const char *e = getenv("HF_CHAIN_XCHG")) xmode = (strcmp(e, "counter") == 0) ? 0 : 1;
    if (blk_host) xmode = 1;   // block transitions repeat a step: tagged slots only
    HF_CUDA(cudaMemsetAsync(status.p, 0, 4 * sizeof(int32_t), st));

    {
        ClassTimer tm(ctx, "other");
        k_cast_lower<<<(unsigned)std::min<int64_t>(L, 65535), 256, 0, st>>>(L, K, ld, V[0].p, L);
        HF_CHECK_LAUNCH(ctx);
        k_iota32<<<(unsigned)cdiv(L, 256), 256, 0, st>>>(L, orig[0].p);
        HF_CHECK_LAUNCH(ctx);
    }
    cudaStream_t st2 = st;
    if (look) {
        if (!ctx->side) {
            HF_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
            for (auto &e : ctx->ev) HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        st2 = ctx->side;
        HF_CUDA(cudaEventRecord(ctx->ev[0], st));        // the side stream starts after the setup above
        HF_CUDA(cudaStreamWaitEvent(st2, ctx->ev[0], 0));
    }

    HF_CUDA(cudaFuncSetAttribute(k_chain<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_chain<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_chain<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    const int chain_lb = getenv("HF_CHAIN_LB") ? atoi(getenv("HF_CHAIN_LB")) : 0;
    HF_CUDA(cudaFuncSetAttribute(k_trailing_c<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRAIL_C_SMEM));
    HF_CUDA(cudaFuncSetAttribute(k_trailing_c<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRAIL_C_SMEM));
    HF_CUDA(cudaFuncSetAttribute(k_trailing_c<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRAIL_C_SMEM + 128));
    // HF_TRAIL_BULK=1: the panel operands staged by the bulk-copy (TMA) engine row by row;
    // =2: by 2D tensor copies (a 16 x 128 box per operand per chunk)
    const int trail_bulk = getenv("HF_TRAIL_BULK") ? atoi(getenv("HF_TRAIL_BULK")) : 0;
    CUtensorMap tmA, tmB;
    std::memset(&tmA, 0, sizeof(tmA));
    std::memset(&tmB, 0, sizeof(tmB));
    if (trail_bulk == 2) {
        make_panel_tmap(&tmA, Snc.p, ldc, cdiv(nb, TK) * TK);
        make_panel_tmap(&tmB, Sc.p, ldc, cdiv(nb, TK) * TK);
    }
    // k_trailing_c: one tile per CTA (default) or persistent CTAs, occupancy x SMs, each
    // prefetching its next tile's compaction map while the current one computes
    // (HF_TRAIL_PCTA=1; measured slower: C2 32.0 vs 29.7 ms, C4 1926 vs 1780 ms per
    // factorization -- the hardware's CTA launch overlaps the next tile's prologue better)
    int cocc = 0;
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cocc, k_trailing_c<false>, 256, TRAIL_C_SMEM));
    const bool trail_pcta = getenv("HF_TRAIL_PCTA") && atoi(getenv("HF_TRAIL_PCTA")) != 0;
    const int64_t cgrid = trail_pcta ? (int64_t)std::max(1, cocc) * nsm : INT64_MAX;
    // persistent trailing kernel (seed prefetch), two CTAs per SM -- OFF by default: measured
    // 38.3 vs 31.0 ms per C2 step (FMA pipe 64.8 vs 71.5 % active; the 4-byte cp.async seed
    // gather adds 155 MB of DRAM reads per large launch and leaves fewer warps resident).
    // HF_TRAIL_PERSIST=1: for launches of more than two tiles per CTA, =2: at any size (tests)
    const int pmode = getenv("HF_TRAIL_PERSIST") ? atoi(getenv("HF_TRAIL_PERSIST")) : 0;
    const bool persist = pmode != 0;
    int pgrid = 0;
    if (persist) {
        HF_CUDA(cudaFuncSetAttribute(k_trailing_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRAIL_P_SMEM));
        int occ = 0;
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_trailing_p, 256, TRAIL_P_SMEM));
        pgrid = std::max(1, occ) * nsm;
    }
    DBuf<int32_t> blkd, bstate;   // NEXT-4: block of every original index; {block, first, attempt}
    if (blk_host) {
        blkd.alloc(std::max<int64_t>(L, 1), st);
        HF_CUDA(cudaMemcpyAsync(blkd.p, blk_host, L * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        bstate.alloc(3, st);
        const int32_t b0[3] = {0, 1, 0};
        HF_CUDA(cudaMemcpyAsync(bstate.p, b0, sizeof(b0), cudaMemcpyHostToDevice, st));
        HF_CUDA(cudaStreamSynchronize(st));   // the host arrays may die after the call
    }
    DBuf<unsigned long long> dbg;
    const bool want_dbg = getenv("HF_CHAIN_DEBUG") != nullptr;
    if (want_dbg) {
        dbg.alloc(8 + 4 * 1024, st);
        dbg.zero(st);
    }
    // buffers of panel p: V[vb] is the matrix at the START of panel p (its position space),
    // S/Sn/sigma/SNrow/DG[p & 1] its values, map[p & 1] its compaction (p+1 space -> p space)
    int cur = 0, vb = 0, pidx = 0, nbprev = 0;
    bool tr_pending = false;   // a trailing update is in flight on the side stream
    int64_t m = L, K0 = 0;
    while (m > 0) {
        const int nbp = (int)std::min<int64_t>(nb, m);
        const int64_t G = std::min<int64_t>(gmax, std::max<int64_t>(1, cdiv(m, 32)));
        const int64_t R = cdiv(m, G);
        const int nthr = (int)std::max<int64_t>(64, cdiv(R, 32) * 32);
        const int pb = look ? (pidx & 1) : 0, qb = pb ^ 1;
        const int64_t nbq_ = look ? nbprev : 0;
        const size_t shm = ((size_t)(ceil4(nbp) + ceil4(nbq_)) * R + 2 * ceil4(nbp) + ceil4(nbq_) + 4) * sizeof(float);
        if (xmode == 0) HF_CUDA(cudaMemsetAsync(xchg.p, 0, xchg.n * sizeof(unsigned long long), st));
        ChainArgs ca;
        ca.m = m; ca.K0 = K0; ca.nbp = nbp; ca.R = (int)R; ca.tau = o.tau;
        ca.V = V[vb].p; ca.ldv = L; ca.orig = orig[cur].p;
        ca.S = S[pb].p; ca.Sn = Sn[pb].p; ca.lds = L; ca.sigma = sigma[pb].p; ca.pivpos = pivpos.p;
        ca.Lorig = Lorig.p; ca.ldl = L; ca.Dk = Dk.p; ca.pivorig = pivorig.p;
        ca.keys = xchg.p; ca.cnt = reinterpret_cast<unsigned int *>(xchg.p + nb); ca.mbox = mbox.p;
        ca.slots = slots.p; ca.xmode = xmode; ca.sstride = sstride;
        ca.spec = (xmode == 1 && !blk_host && G <= 64) ? chain_spec : 0;
        ca.dpoll = chain_dpoll;
        ca.status = status.p; ca.dbg = want_dbg ? dbg.p : nullptr;
        ca.blk = blkd.p; ca.nblk = o_nblk; ca.bstate = bstate.p;
        ca.nbmax = nb;
        if (look && pidx > 0) {
            ca.mapprev = map[qb].p; ca.SNprev = SNrow[qb].p; ca.sigprev = sigma[qb].p; ca.DGprev = DG[qb].p;
            ca.nbprev = nbprev;
        } else {
            ca.mapprev = nullptr; ca.SNprev = nullptr; ca.sigprev = nullptr; ca.DGprev = nullptr; ca.nbprev = 0;
        }
        ca.SNout = look ? SNrow[pb].p : nullptr;
        ca.DGout = look ? DG[pb].p : nullptr;
        {
            ClassTimer tm(ctx, "chain", st, chain_flops(m, nbp), chain_bytes(m, nbp));
            void *args[] = {&ca};
            const int lb = std::max(nthr, chain_lb);
            void *kf = lb <= 256 ? (void *)k_chain<256> : lb <= 512 ? (void *)k_chain<512> : (void *)k_chain<1024>;
            HF_CUDA(cudaLaunchCooperativeKernel(kf, dim3((unsigned)G), dim3(nthr), args, shm, st));
            HF_CHECK_LAUNCH(ctx);
        }
        const int64_t mp = m - nbp;
        if (mp > 0) {
            {
                ClassTimer tm(ctx, "other");
                k_compact<<<(unsigned)std::min<int64_t>(cdiv(m, 256), 4096), 256, 0, st>>>(
                    m, nbp, pivpos.p, orig[cur].p, map[pb].p, orig[cur ^ 1].p, status.p);
                HF_CHECK_LAUNCH(ctx);
            }
            // trailing update of this panel: V at the start of panel p (V[?]) -> V at the start
            // of panel p+1.  Serial: V[cur] -> V[cur^1].  Lookahead: the chain of panel p
            // read V[vb] (start of panel p-1); the trailing update of panel p-1 (in flight)
            // writes the start of panel p into the other buffer, and this one then turns it
            // into the start of panel p+1 in V[vb], which the next chain no longer needs.
            TrailArgs ta;
            ta.mp = mp; ta.nbp = nbp; ta.ldv = L; ta.ntiles = 0;
            ta.map = map[pb].p; ta.S = S[pb].p; ta.Sn = Sn[pb].p; ta.lds = L; ta.status = status.p;
            ta.Sc = Sc.p; ta.Snc = Snc.p; ta.ldc = ldc;
            const int64_t T = cdiv(mp, TB);
            const int64_t ntiles = T * (T + 1) / 2;
            ta.ntiles = ntiles;
            if (!look) {
                ta.Vold = V[cur].p; ta.Vnew = V[cur ^ 1].p;
                if (Sc.p) {
                    ClassTimer tg(ctx, "other");
                    k_gather_panel<<<dim3((unsigned)cdiv(mp, 256), (unsigned)cdiv(nbp, 16)), 256, 0, st>>>(
                        mp, nbp, map[pb].p, S[pb].p, Sn[pb].p, L, Sc.p, Snc.p, ldc, status.p);
                    HF_CHECK_LAUNCH(ctx);
                }
                ClassTimer tm(ctx, "trailing", st, trail_flops(mp, nbp), trail_bytes(mp, nbp));
                if (Sc.p && persist && (ntiles > 2 * pgrid || pmode == 2)) {
                    k_trailing_p<<<(unsigned)pgrid, 256, TRAIL_P_SMEM, st>>>(ta, ntiles);
                } else if (Sc.p) {
                    const unsigned tg = (unsigned)std::min<int64_t>(ntiles, cgrid);
                    if (trail_bulk == 2) k_trailing_c<false, 2><<<tg, 256, TRAIL_C_SMEM + 128, st>>>(ta, tmA, tmB);
                    else if (trail_bulk) k_trailing_c<false, 1><<<tg, 256, TRAIL_C_SMEM, st>>>(ta, tmA, tmB);
                    else k_trailing_c<false><<<tg, 256, TRAIL_C_SMEM, st>>>(ta, tmA, tmB);
                } else {
                    k_trailing<<<(unsigned)ntiles, 256, 0, st>>>(ta);
                }
                HF_CHECK_LAUNCH(ctx);
                vb ^= 1;
            } else {
                // the side stream: wait for this chain (S, Sn, map of panel p)
                HF_CUDA(cudaEventRecord(ctx->ev[1], st));
                HF_CUDA(cudaStreamWaitEvent(st2, ctx->ev[1], 0));
                const int vsrc = (pidx == 0) ? vb : (vb ^ 1);   // start of panel p
                ta.Vold = V[vsrc].p; ta.Vnew = V[vsrc ^ 1].p;
                {
                    ClassTimer tg(ctx, "other", st2);
                    k_gather_panel<<<dim3((unsigned)cdiv(mp, 256), (unsigned)cdiv(nbp, 16)), 256, 0, st2>>>(
                        mp, nbp, map[pb].p, S[pb].p, Sn[pb].p, L, Sc.p, Snc.p, ldc, status.p);
                    HF_CHECK_LAUNCH(ctx);
                }
                {
                    ClassTimer tm(ctx, "trailing", st2, trail_flops(mp, nbp), trail_bytes(mp, nbp));
                    k_trailing_c<false><<<(unsigned)std::min<int64_t>(ntiles, cgrid), 256, TRAIL_C_SMEM, st2>>>(ta, tmA, tmB);
                    HF_CHECK_LAUNCH(ctx);
                }
                // the next chain reads the start of panel p (vsrc); before it runs, the trailing
                // update of panel p-1 (which wrote vsrc) must be done -- it is, being earlier on st2;
                // wait for everything on st2 except this launch: record after the previous one
                if (tr_pending) HF_CUDA(cudaStreamWaitEvent(st, ctx->ev[2], 0));
                HF_CUDA(cudaEventRecord(ctx->ev[2], st2));
                tr_pending = true;
                vb = vsrc;
            }
            cur ^= 1;
        }
        nbprev = nbp;
        K0 += nbp;
        m = mp;
        ++pidx;
    }
    if (look) {   // join the side stream before the trailing buffers can be released
        HF_CUDA(cudaEventRecord(ctx->ev[3], st2));
        HF_CUDA(cudaStreamWaitEvent(st, ctx->ev[3], 0));
    }
    V[0].release();   // the trailing buffers are done: keep the peak at K + Lorig + Lfac
    V[1].release();
    lowprec_finish(ctx, L, o, lf, status, pivorig, Dk, Lorig, want_dbg ? &dbg : nullptr);
}

// ========================================================================= NEXT-3
// Nonsymmetric LDU with symmetric pivoting and threshold postponing (the
// paper's stokes / dd-hole matrices; Eq. 1 P:46 is
// written for a general K), canonical FP32 arithmetic [R19]:
//   d = v_PP, l_I = c_I / d (IEEE), r_J = v_PJ, v_IJ <- fmaf(-l_I, r_J, v_IJ),
// one fmaf per entry per pivot in pivot order -- bit-identical to the
// right-looking oracle (oracle_ldu_f32) by the same argument as [R8] with the
// roles fixed (the product -l_I r_J is exact inside the FMA).
namespace {

__global__ void k_cast_full(int64_t L, const double *__restrict__ K, int64_t ldk, float *__restrict__ V, int64_t ldv) {
    for (int64_t j = blockIdx.x; j < L; j += gridDim.x)
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) V[i + j * ldv] = __double2float_rn(K[i + j * ldk]);
}

struct ChainNSArgs {
    int64_t m, K0;
    int nbp, R;
    double tau;
    const float *V;               // full trailing matrix at the panel start (position space)
    int64_t ldv;
    const int32_t *orig;
    float *S;                     // S[i + t*lds]  = r_i^t  (trailing B operand)
    float *Sn;                    // Sn[i + t*lds] = -l_i^t (trailing A operand)
    int64_t lds;
    int32_t *pivpos;
    float *Lorig, *Uorig;         // [orig + k*ldl]: l = c / d, r / d
    int64_t ldl;
    float *Dk;
    int32_t *pivorig;
    unsigned long long *slots;    // [2][G][SLOT_STRIDE] key | tag
    unsigned long long *mbox;     // [2][G][2 (nb+1)] candidate row: (-l, r) words, float bits << 32 | tag
    int32_t *status;
};

// Per pivot (CTA = a slice of rows; each row i also stands for COLUMN i):
//  A local argmax of the lazy diagonal -> this CTA's slot; the candidate's panel
//    values (-l_P^u, r_P^u), u < t, to the mailbox (tagged words)
//  D every slot of this step -> the pivot key (smallest position on ties)
//  E stop test [R4]
//  F pivot row's (-l_P^u, r_P^u) from the winner's mailbox; column V[:, P] and
//    row V[P, :] entries of own indices from the panel-start matrix
//  G c_i = V_iP + sum_u fmaf(-l_i^u, r_P^u), r_i = V_Pi + sum_u fmaf(-l_P^u, r_i^u)
//    (u ascending), l_i = c_i / d, lazy diagonal fmaf(-l_i, r_i, v_ii)
// MAXT: the launch bound, as k_chain's (a 256 / 512 bound lifts the 64-register cap)
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_chain_ns(ChainNSArgs a) {
    extern __shared__ float smem[];
    __shared__ unsigned long long red[32];
    __shared__ unsigned long long bkey;
    if (*(volatile int32_t *)&a.status[2]) return;
    const int G = gridDim.x;
    const int tid = threadIdx.x, nthr = blockDim.x, nwarp = nthr >> 5, lane = tid & 31, wid = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * a.R;
    const int64_t nown = max((int64_t)0, min((int64_t)a.R, a.m - r0));
    const int nb = a.nbp;
    float *nl = smem;                          // [nb][R] -l_i^u of own indices
    float *rr = nl + (size_t)nb * a.R;         // [nb][R]  r_i^u of own indices
    float *spl = rr + (size_t)nb * a.R;        // [nb] -l_P^u of the pivot
    float *spr = spl + nb;                     // [nb]  r_P^u of the pivot
    const bool has = tid < nown;
    const int64_t i = r0 + tid;
    const int32_t oi = has ? a.orig[i] : 0;
    float dg = has ? a.V[i + i * a.ldv] : 0.f;
    bool piv = !has;
    float dprev = a.K0 > 0 ? a.Dk[a.K0 - 1] : 0.f;
    bool pend = false;
    float ps = 0.f, pn = 0.f, pl = 0.f, pu = 0.f;
    int t = 0;
    bool stopped = false;
    for (; t < nb; ++t) {
        const int64_t k = a.K0 + t;
        const uint64_t tag = step_tag(k);
        uint64_t key = piv ? 0ull : mkkey(dg, (uint32_t)i);
        key = warp_max64(key);
        if (lane == 0) red[wid] = key;
        __syncthreads();
        if (wid < 2) {
            uint64_t v = (lane < nwarp) ? red[lane] : 0ull;
            v = warp_max64(v);
            if (wid == 0) {
                if (lane == 0) {
                    unsigned long long *slot = &a.slots[((size_t)(t & 1) * G + blockIdx.x) * SLOT_STRIDE];
                    st_relaxed_u64(slot, (v & ~TAGM) | tag);
                }
            } else if (v) {
                unsigned long long *mb = a.mbox + ((size_t)(t & 1) * G + blockIdx.x) * 2 * (nb + 1);
                const int lr = (int)((int64_t)(POS_MAX - (uint32_t)((v >> 15) & POS_MAX)) - r0);
                for (int u = lane; u < t; u += 32) {
                    st_relaxed_u64(&mb[2 * u], ((unsigned long long)__float_as_uint(nl[(size_t)u * a.R + lr]) << 32) | tag);
                    st_relaxed_u64(&mb[2 * u + 1], ((unsigned long long)__float_as_uint(rr[(size_t)u * a.R + lr]) << 32) | tag);
                }
            }
        }
        if (pend) {   // deferred global stores of step t-1
            a.S[i + (int64_t)(t - 1) * a.lds] = ps;
            a.Sn[i + (int64_t)(t - 1) * a.lds] = pn;
            a.Lorig[(int64_t)oi + (k - 1) * a.ldl] = pl;
            a.Uorig[(int64_t)oi + (k - 1) * a.ldl] = pu;
            pend = false;
        }
        if (wid == 0) {
            const unsigned long long *sl = a.slots + (size_t)(t & 1) * G * SLOT_STRIDE;
            uint64_t mx;
            for (;;) {
                bool ok = true;
                mx = 0;
                for (int g = lane; g < G; g += 32) {
                    const uint64_t sv = ld_relaxed_u64(&sl[(size_t)g * SLOT_STRIDE]);
                    ok &= (sv & TAGM) == tag;
                    mx = umax64(mx, sv);
                }
                if (__all_sync(0xffffffffu, ok)) break;
            }
            mx = warp_max64(mx);
            if (lane == 0) bkey = mx;
        }
        __syncthreads();
        const uint64_t bk = bkey;
        const float absd = __uint_as_float((uint32_t)(bk >> 32));
        const int64_t P = (int64_t)(POS_MAX - (uint32_t)((bk >> 15) & POS_MAX));
        const float d = ((bk >> 14) & 1) ? -absd : absd;
        const bool stop = (k == 0) ? (absd == 0.f) : ((double)absd < __dmul_rn(a.tau, fabs((double)dprev)));
        if (stop) {
            if (blockIdx.x == 0 && tid == 0) {
                a.status[0] = (int32_t)k;
                a.status[1] = t;
                a.status[2] = 1;
            }
            stopped = true;
            break;
        }
        float vc = 0.f, vr = 0.f;   // panel-start column / row entries of own index
        if (!piv && i != P) {
            vc = a.V[i + P * a.ldv];
            vr = a.V[P + i * a.ldv];
        }
        {
            const int owner = (int)(P / a.R);
            const unsigned long long *mb = a.mbox + ((size_t)(t & 1) * G + owner) * 2 * (nb + 1);
            for (int u = tid; u < 2 * t; u += nthr) {
                uint64_t w;
                do {
                    w = ld_relaxed_u64(&mb[u]);
                } while ((w & TAGM) != tag);
                const float x = __uint_as_float((uint32_t)(w >> 32));
                if (u & 1) spr[u >> 1] = x;
                else spl[u >> 1] = x;
            }
        }
        __syncthreads();
        if (has && i == P) {
            piv = true;
            a.Dk[k] = d;
            a.pivorig[k] = oi;
            a.pivpos[t] = (int32_t)P;
        } else if (!piv) {
            float c = vc, r = vr;
            const float *xl = nl + tid, *xr = rr + tid;
            for (int u = 0; u < t; ++u) {                      // [R19] one fmaf per earlier pivot, in order
                c = __fmaf_rn(xl[(size_t)u * a.R], spr[u], c);
                r = __fmaf_rn(spl[u], xr[(size_t)u * a.R], r);
            }
            const float l = __fdiv_rn(c, d);
            nl[(size_t)t * a.R + tid] = -l;
            rr[(size_t)t * a.R + tid] = r;
            ps = r;
            pn = -l;
            pl = l;
            pu = __fdiv_rn(r, d);
            pend = true;
            dg = __fmaf_rn(-l, r, dg);                         // lazy diagonal, the trailing update's fma
        }
        dprev = d;
    }
    if (pend) {
        a.S[i + (int64_t)(t - 1) * a.lds] = ps;
        a.Sn[i + (int64_t)(t - 1) * a.lds] = pn;
        a.Lorig[(int64_t)oi + (a.K0 + t - 1) * a.ldl] = pl;
        a.Uorig[(int64_t)oi + (a.K0 + t - 1) * a.ldl] = pu;
    }
    if (!stopped && blockIdx.x == 0 && tid == 0) a.status[1] = t;
}

}  // namespace

void lowprec_factor_ns(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                       hf_lowfactor *lf) {
    cudaStream_t st = ctx->stream;
    lf->L = L;
    lf->nonsym = true;
    if (L == 0) {
        lf->N = lf->Ntau = lf->n2 = 0;
        return;
    }
    HF_REQUIRE(L <= (int64_t)POS_MAX - 1, "L too large for the 17-bit position key");
    const int nsm = ctx->num_sms;
    int maxsmem = 0;
    HF_CUDA(cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    cudaFuncAttributes fa;
    HF_CUDA(cudaFuncGetAttributes(&fa, k_chain_ns<1024>));
    maxsmem -= (int)fa.sharedSizeBytes;
    const int nb_def = 64;   // two panel values per own index
    int gmax = (int)std::min<int64_t>(nsm, std::max<int64_t>(64, cdiv(L, (int64_t)(maxsmem / 4 / (2 * nb_def + 2)))));
    const int64_t G0 = std::min<int64_t>(gmax, std::max<int64_t>(1, cdiv(L, 32)));
    const int64_t R0 = cdiv(L, G0);
    HF_REQUIRE(R0 <= 1024, "L too large for one chain CTA per SM (R > 1024)");
    int nb = o.nb > 0 ? o.nb : nb_def;
    while (nb > 8 && (int64_t)(2 * nb * R0 + 2 * nb) * 4 > (int64_t)maxsmem) nb /= 2;
    nb = std::max(TK, (nb / TK) * TK);
    HF_REQUIRE((int64_t)(2 * nb * R0 + 2 * nb) * 4 <= (int64_t)maxsmem, "panel does not fit in shared memory");

    DBuf<float> V[2], S, Sn, Sc, Snc, Lorig, Uorig, Dk;
    V[0].alloc((size_t)L * L, st);
    V[1].alloc((size_t)L * L, st);
    DBuf<int32_t> orig[2], map, pivpos, pivorig, status;
    orig[0].alloc(L, st);
    orig[1].alloc(L, st);
    map.alloc(L, st);
    S.alloc((size_t)L * nb, st);
    Sn.alloc((size_t)L * nb, st);
    const int64_t ldc = cdiv(L, TB) * TB;
    Sc.alloc((size_t)ldc * nb, st);
    Snc.alloc((size_t)ldc * nb, st);
    Lorig.alloc((size_t)L * L, st);
    Uorig.alloc((size_t)L * L, st);
    Dk.alloc(L, st);
    pivpos.alloc(nb, st);
    pivorig.alloc(L, st);
    status.alloc(4, st);
    DBuf<unsigned long long> mbox, slots;
    mbox.alloc((size_t)2 * nsm * 2 * (nb + 1), st);
    mbox.zero(st);
    slots.alloc((size_t)2 * nsm * SLOT_STRIDE, st);
    slots.zero(st);
    HF_CUDA(cudaMemsetAsync(status.p, 0, 4 * sizeof(int32_t), st));
    {
        ClassTimer tm(ctx, "other");
        k_cast_full<<<(unsigned)std::min<int64_t>(L, 65535), 256, 0, st>>>(L, K, ld, V[0].p, L);
        HF_CHECK_LAUNCH(ctx);
        k_iota32<<<(unsigned)cdiv(L, 256), 256, 0, st>>>(L, orig[0].p);
        HF_CHECK_LAUNCH(ctx);
    }
    HF_CUDA(cudaFuncSetAttribute(k_chain_ns<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_chain_ns<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_chain_ns<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_trailing_c<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRAIL_C_SMEM));
    int cur = 0;
    int64_t m = L, K0 = 0;
    while (m > 0) {
        const int nbp = (int)std::min<int64_t>(nb, m);
        const int64_t G = std::min<int64_t>(gmax, std::max<int64_t>(1, cdiv(m, 32)));
        const int64_t R = cdiv(m, G);
        const int nthr = (int)std::max<int64_t>(64, cdiv(R, 32) * 32);
        const size_t shm = ((size_t)2 * nbp * R + 2 * nbp) * sizeof(float);
        ChainNSArgs ca;
        ca.m = m; ca.K0 = K0; ca.nbp = nbp; ca.R = (int)R; ca.tau = o.tau;
        ca.V = V[cur].p; ca.ldv = L; ca.orig = orig[cur].p;
        ca.S = S.p; ca.Sn = Sn.p; ca.lds = L; ca.pivpos = pivpos.p;
        ca.Lorig = Lorig.p; ca.Uorig = Uorig.p; ca.ldl = L; ca.Dk = Dk.p; ca.pivorig = pivorig.p;
        ca.slots = slots.p; ca.mbox = mbox.p; ca.status = status.p;
        {
            ClassTimer tm(ctx, "chain");
            void *args[] = {&ca};
            const int lb = std::max(nthr, getenv("HF_CHAIN_LB") ? atoi(getenv("HF_CHAIN_LB")) : 0);
            void *kf = lb <= 256 ? (void *)k_chain_ns<256> : lb <= 512 ? (void *)k_chain_ns<512> : (void *)k_chain_ns<1024>;
            HF_CUDA(cudaLaunchCooperativeKernel(kf, dim3((unsigned)G), dim3(nthr), args, shm, st));
            HF_CHECK_LAUNCH(ctx);
        }
        const int64_t mp = m - nbp;
        if (mp > 0) {
            {
                ClassTimer tm(ctx, "other");
                k_compact<<<(unsigned)std::min<int64_t>(cdiv(m, 256), 4096), 256, 0, st>>>(
                    m, nbp, pivpos.p, orig[cur].p, map.p, orig[cur ^ 1].p, status.p);
                HF_CHECK_LAUNCH(ctx);
                k_gather_panel<<<dim3((unsigned)cdiv(mp, 256), (unsigned)cdiv(nbp, 16)), 256, 0, st>>>(
                    mp, nbp, map.p, S.p, Sn.p, L, Sc.p, Snc.p, ldc, status.p);
                HF_CHECK_LAUNCH(ctx);
            }
            TrailArgs ta;
            ta.mp = mp; ta.nbp = nbp; ta.ldv = L; ta.ntiles = cdiv(mp, TB) * cdiv(mp, TB); ta.map = map.p; ta.S = S.p; ta.Sn = Sn.p; ta.lds = L;
            ta.status = status.p; ta.Sc = Sc.p; ta.Snc = Snc.p; ta.ldc = ldc;
            ta.Vold = V[cur].p; ta.Vnew = V[cur ^ 1].p;
            const int64_t T = cdiv(mp, TB);
            {
                ClassTimer tm(ctx, "trailing");
                CUtensorMap tz;
                std::memset(&tz, 0, sizeof(tz));
                k_trailing_c<true><<<(unsigned)(T * T), 256, TRAIL_C_SMEM, st>>>(ta, tz, tz);
                HF_CHECK_LAUNCH(ctx);
            }
            cur ^= 1;
        }
        K0 += nbp;
        m = mp;
    }
    V[0].release();
    V[1].release();
    lowprec_finish(ctx, L, o, lf, status, pivorig, Dk, Lorig, nullptr);
    const int64_t N = lf->N;
    lf->Ufac.alloc((size_t)std::max<int64_t>(N, 1) * std::max<int64_t>(N, 1), st);
    if (N > 0) {
        ClassTimer tm(ctx, "other");
        k_gather_L<<<(unsigned)std::min<int64_t>(N, 65535), 256, 0, st>>>(N, pivorig.p, Uorig.p, L, lf->Ufac.p, N);
        HF_CHECK_LAUNCH(ctx);
    }
    HF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hf

namespace hf {
// microseconds per exchange step of the chain's grid-wide exchange alone
double chain_exchange_floor(hf_ctx *ctx, int nctas, int nthreads, int steps) {
    cudaStream_t st = ctx->stream;
    nctas = std::max(1, std::min(nctas, ctx->num_sms));
    nthreads = std::max(32, std::min(1024, (nthreads + 31) / 32 * 32));
    DBuf<unsigned long long> slots, out;
    slots.alloc((size_t)2 * nctas * SLOT_STRIDE, st);
    slots.zero(st);
    out.alloc(2, st);
    int ss = SLOT_STRIDE;
    void *args[] = {&slots.p, &ss, &steps, &out.p};
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_xchg_floor, dim3((unsigned)nctas), dim3(nthreads), args, 0, st));
    HF_CHECK_LAUNCH(ctx);
    unsigned long long h[2];
    HF_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    return (double)h[0] * 1e-3 / std::max(steps, 1);
}
}  // namespace hf
