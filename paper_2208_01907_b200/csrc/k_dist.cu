// k_dist.cu -- stage 1 (steps a2/a3: FP32 LDL^T with symmetric max-|diag| pivoting
// and threshold postponing, rules [R2]-[R10]) DISTRIBUTED over G
// ranks (BASELINE north_star: "1D block-column-cyclic layout ...
// allreduce(max) picks the pivot ... broadcast distributes each factored panel").
//
// Layout: original index j is OWNED by rank (j / 128) % G.
// Rank g stores, for every active index J it owns ("local column" c, kept in
// position order), the LOWER-triangle entries v_IJ of all active I with
// pos(I) >= pos(J), rows by global position (compacted stably after each panel,
// as on one GPU).  Every unordered pair {I, J} is stored once, so the total
// trailing-update work over the ranks equals one GPU's (no full columns).
//
// Pivot chain (k_chain_d, one cooperative launch per panel per rank): the chain
// ROWS of rank g are the indices it owns.  Per pivot:
//   A  local argmax over own rows -> (|d|, position, sign) key + (rank, local col)
//   B  every CTA stores its key into the slot array of EVERY rank (one hop over
//      NVLink, tag-validated "LL" words, no fences) and its candidate row's panel
//      values into its own rank's mailbox
//   C  each CTA polls its own rank's slots: the max key is the pivot P ([R3]),
//      identical on every rank (it is the allreduce(max) of the north_star)
//   D  column entries for own rows I: pos(I) < pos(P): row P of own column I
//      (local); pos(I) > pos(P): column P on its owner (a peer read); the pivot
//      row's panel values from the winner's mailbox (a peer read)
//   E  c_I, s_I = c_I / sqrt|d|, L = c_I / d, lazy diagonal -- the same fmaf
//      sequence as the one-GPU chain [R8], so the bits do not depend on G.
// After the chain each rank gathers the panel S of ALL rows from the owners
// (k_dgather: the panel broadcast), compacts its local columns and updates its
// own lower-triangle columns (k_trailing_d, the FFMA2 tile of k_trailing_c over a
// device-built tile list).  The factor rows are gathered from their owners at the
// end.
//
// One code path for real ranks and their one-GPU emulation: every peer buffer is
// reached through a per-rank pointer table (CUDA-IPC mappings on a multi-GPU
// context; plain buffers of this GPU when G ranks are emulated, where ONE
// cooperative launch runs all ranks' chain CTAs -- the profiling guide forbids
// separate launches that wait on one another on one GPU).  Cross-rank spins carry
// a timeout (status[3] = 1, HF_ERR) so a lost peer cannot hang the GPU.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hf_internal.cuh"

namespace hf {
namespace {

constexpr uint32_t DPOS_MAX = 0x1FFFF;   // 17-bit position field -> L <= 131071
constexpr int DCB = 128;                 // ownership block: owner(j) = (j / DCB) % G
constexpr int DTB = 128;                 // trailing tile
constexpr int DTK = 16;                  // trailing k chunk
constexpr int DTNS = 3;                  // cp.async stages
constexpr size_t DTRAIL_SMEM = (size_t)2 * DTNS * DTK * DTB * sizeof(float);
constexpr int DSLOT = 32;                // 256 B between slots
constexpr uint64_t DTAGM = 0x3FFF;

__device__ __forceinline__ int owner_of(int64_t j, int G) { return (int)((j / DCB) % G); }
__host__ __device__ __forceinline__ int64_t col_orig(int64_t c, int h, int G) {
    return (c / DCB) * ((int64_t)DCB * G) + (int64_t)h * DCB + (c % DCB);
}
__device__ __forceinline__ uint64_t dkey(float d, uint32_t pos) {
    const uint64_t ab = __float_as_uint(fabsf(d));
    return (ab << 32) | ((uint64_t)(DPOS_MAX - pos) << 15) | ((uint64_t)(d < 0.f) << 14) | 1ull;
}
__device__ __forceinline__ uint64_t dtag(int64_t k) { return (uint64_t)(k % 16383) + 1; }
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
}  // namespace

// per-rank buffers, reached through a device table (peer mappings on a real run).
// [2] arrays are indexed by the parity `cur` of the panel that wrote / reads them.
struct DRank {
    float *V[2];             // L x ncols, rows = global position, ld = ldp (ping-pong)
    int32_t *lpos[2];        // local column -> global position (by panel parity)
    int32_t *lorig[2];       // local column -> original index
    int32_t *nloc;           // [2] active local columns
    int32_t *cmapL;          // new local column -> old local column (last compaction)
    float *S[2];             // own rows' s_i^t at the panel's positions, ld = lds
    float *DG[2];            // own rows' lazy diagonal at the end of the panel (lookahead)
    float *Lorig;            // L_{orig, k} (may alias across emulated ranks)
    unsigned long long *slots;   // [2][G * Cmax][DSLOT]  {key, info} pairs
    unsigned long long *mbox;    // [2][Cmax][nbmax + 1]
    float *Dk;               // [L] pivots d_k
    int32_t *pivorig;        // [L] original index of pivot k
    int32_t *pivpos[2];      // [nbmax] pivot positions of the panel
    float *sigma[2];         // [nbmax] sign of d_t
    int32_t *status;         // [4]: N_tau if stopped, pivots in last panel, stopped, peer timeout
    int32_t *orig[2];        // global position -> original index (identical on every rank)
    int32_t *map;            // new position -> old position (last compaction)
    int32_t *tiles;          // [CTmax + 1] tile prefix | [CTmax] first row tile | [1] tile counter
    float *Sc, *Snc;         // the panel in the NEW position space (all rows), ld = ldc
    float *Scol;             // s of own local columns (new local order), ld = ldcol
    unsigned int *bar;       // [2] cross-rank barrier counters (chain stream, trailing stream)
};

namespace {

struct DChainArgs {
    const DRank *rp;
    int G, rank0, Cper, R, cur, nbp, nbmax;
    int nbq;                 // lookahead: pivots of the previous panel applied here (0: serial)
    int64_t m, K0, ldp, lds, ldl;
    double tau;
    unsigned long long timeout_ns;
    unsigned long long *dbg;   // optional per-phase time sums of CTA 0 (HF_CHAIN_DEBUG)
};

// c <- fmaf(x_u, y_u, c) for u = 0..n-1 in order [R8]; x_u = xs[u * R] (own row's
// panel values, shared memory, stride R), y_u = ys[u] (broadcast).  (Issuing the next
// 8 loads ahead of the current 8 FMAs measured slower: 0.96 vs 0.80 us per C2 pivot.)
__device__ __forceinline__ float fma_chain(float c, const float *xs, const float *ys, int n, int R) {
    int u = 0;
    for (; u + 8 <= n; u += 8) {
        float x[8], y[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            x[q] = xs[(size_t)(u + q) * R];
            y[q] = ys[u + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) c = __fmaf_rn(x[q], y[q], c);
    }
    for (; u < n; ++u) c = __fmaf_rn(xs[(size_t)u * R], ys[u], c);
    return c;
}

// warp max of a 64-bit key (redux.sync on the high then the low word) and the payload
// of the lane holding it (keys are distinct when non-zero: they carry the position)
__device__ __forceinline__ void warp_argmax(uint64_t &key, uint32_t &p1, uint32_t &p2) {
    const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const unsigned win = __ballot_sync(0xffffffffu, hi == mh && lo == ml);
    const int src = __ffs(win) - 1;
    p1 = __shfl_sync(0xffffffffu, p1, src);
    p2 = __shfl_sync(0xffffffffu, p2, src);
    key = ((uint64_t)mh << 32) | ml;
}

template <bool SYS>
__device__ __forceinline__ void st_x_v2(unsigned long long *p, unsigned long long a, unsigned long long b) {
    if (SYS) asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
    else asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
template <bool SYS>
__device__ __forceinline__ void ld_x_v2(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
    if (SYS) asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
template <bool SYS>
__device__ __forceinline__ void st_x(unsigned long long *p, unsigned long long v) {
    if (SYS) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <bool SYS>
__device__ __forceinline__ unsigned long long ld_x(const unsigned long long *p) {
    unsigned long long v;
    if (SYS) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// One cooperative launch: CTA b belongs to rank rank0 + b / Cper (its local
// index lb = b % Cper) and owns local columns [lb R, lb R + R) of that rank.
// SYS: the exchange words cross NVLink (real ranks, system scope); else the
// ranks are emulated on this GPU (gpu scope).
// Lookahead (nbq > 0): the previous panel's trailing update is still running, so
// the matrix read here is the one at the START of the previous panel (V[cur ^ 1],
// index spaces of that panel) and its nbq updates of the pivot column are applied
// here first, one fmaf per pivot in order -- the same operands the trailing update
// uses (role-symmetric [R8]), so the bits equal the serial schedule's.
// MAXT: the launch bound, as k_chain's (a 256 / 512 bound lifts the 64-register cap)
template <bool SYS, int MAXT = 1024>
__global__ void __launch_bounds__(MAXT, 1) k_chain_d(DChainArgs a) {
    extern __shared__ __align__(16) float smem[];
    __shared__ unsigned long long red[32];
    __shared__ uint32_t redi[32], redl[32];
    __shared__ unsigned long long bkey;
    __shared__ uint32_t binfo, blb;
    __shared__ int bail;
    const int grp = blockIdx.x / a.Cper, lb = blockIdx.x % a.Cper;
    const int h = a.rank0 + grp;
    const DRank &me = a.rp[h];
    if (*(volatile int32_t *)&me.status[2] || *(volatile int32_t *)&me.status[3]) return;   // uniform per rank
    const int GT = a.G * a.Cper;
    const int gid = h * a.Cper + lb;
    const int tid = threadIdx.x, nthr = blockDim.x, nwarp = nthr >> 5, lane = tid & 31, wid = tid >> 5;
    const int cur = a.cur, prv = cur ^ 1;
    const bool look = a.nbq > 0;
    const int nbq = a.nbq;
    const int64_t nl = me.nloc[cur];
    const int64_t c0 = (int64_t)lb * a.R;
    const int64_t nown = max((int64_t)0, min((int64_t)a.R, nl - c0));
    const int nb = a.nbp;
    float *sneg = smem;                                          // [nbp][R] -sigma_u s_i^u, own rows
    float *snp = sneg + (size_t)nb * a.R;                        // [nbq][R] the same, previous panel
    float *sp = smem + (((size_t)(nb + nbq) * a.R + 3) & ~(size_t)3);   // [nbp] s_P^u of the pivot row
    float *spp = sp + nb;                                        // [nbq] s_P^u, previous panel
    float *sgm = spp + nbq;                                      // [nbp] sigma_u
    __shared__ int32_t pvs[256];                                 // [nbp] pivot positions (nb <= 256)
    const bool has = tid < nown;
    const int64_t c = c0 + tid;                                  // own local column = own row
    const int64_t i = has ? (int64_t)me.lpos[cur][c] : 0;        // its position (this panel)
    const int32_t oi = has ? me.lorig[cur][c] : 0;
    const int64_t cr = (has && look) ? (int64_t)me.cmapL[c] : c;            // its column in the V read
    const int64_t io = (has && look) ? (int64_t)me.lpos[prv][cr] : i;       // its row in the V read
    const float *Vme = me.V[look ? prv : cur];
    float dg = 0.f;                                              // lazy diagonal
    if (has) dg = look ? me.DG[prv][cr] : Vme[io + cr * a.ldp];
    if (has && look) {
        const float *Sq = me.S[prv] + io;
        const float *sq = me.sigma[prv];
        for (int u = 0; u < nbq; ++u) snp[(size_t)u * a.R + tid] = -sq[u] * Sq[(int64_t)u * a.lds];
    }
    const uint32_t myinfo = has ? (((uint32_t)h << 20) | (uint32_t)cr) : 0u;
    // every pointer the step loop uses, in registers / shared memory (the exchange asm's
    // memory clobbers would otherwise reload them from the table on the critical path)
    __shared__ const float *sV[64], *sSp[64];
    __shared__ const unsigned long long *sMb[64];
    __shared__ unsigned long long *sSl[64];
    for (int q = tid; q < a.G; q += nthr) {
        sV[q] = a.rp[q].V[look ? prv : cur];
        sSp[q] = a.rp[q].S[prv];
        sMb[q] = a.rp[q].mbox;
        sSl[q] = a.rp[q].slots;
    }
    float *const Sme = me.S[cur];
    float *const Lor = me.Lorig;
    float *const Dk = me.Dk;
    int32_t *const pvme = me.pivpos[cur];
    float *const sgme = me.sigma[cur];
    int32_t *const stat = me.status;
    const int32_t *const mapme = me.map;
    unsigned long long *const mbme = me.mbox;
    bool piv = !has;
    float dprev = a.K0 > 0 ? Dk[a.K0 - 1] : 0.f;
    bool pend = false;
    float ps = 0.f, pc = 0.f, pd = 1.f;   // (L = c / d is formed at the deferred store)
    int t = 0;
    bool stopped = false;
    if (tid == 0) bail = 0;
    const unsigned long long deadline = gtime() + a.timeout_ns;
    const unsigned long long *myslots = me.slots;
    const bool dbgon = a.dbg && blockIdx.x == 0 && tid == 0;
    unsigned long long ph[6] = {0, 0, 0, 0, 0, 0}, tp = dbgon ? gtime() : 0;
#define PH(q) if (dbgon) { const unsigned long long n_ = gtime(); ph[q] += n_ - tp; tp = n_; }
    for (; t < nb;) {
        const int64_t k = a.K0 + t;
        const uint64_t tag = dtag(k);
        const int par = (int)(k & 1);
        PH(4)
        // ---- A: [R3] local argmax over own active rows, carrying (rank, column in the V read)
        uint64_t key = !piv ? dkey(dg, (uint32_t)i) : 0ull;
        uint32_t kinfo = myinfo, klr = (uint32_t)tid;
        warp_argmax(key, kinfo, klr);
        if (lane == 0) {
            red[wid] = key;
            redi[wid] = kinfo;
            redl[wid] = klr;
        }
        __syncthreads();
        PH(0)
        // ---- B: publish {key, info | lb} to every rank; the candidate's panel values to the mailbox
        if (wid < 2) {
            uint64_t v = (lane < nwarp) ? red[lane] : 0ull;
            uint32_t vinfo = (lane < nwarp) ? redi[lane] : 0u;
            uint32_t vlr = (lane < nwarp) ? redl[lane] : 0u;
            warp_argmax(v, vinfo, vlr);
            if (wid == 0) {
                const unsigned long long w1 =
                    ((unsigned long long)(v ? vinfo : 0u) << 32) | ((unsigned long long)lb << 14) | tag;
                // one slot per CTA in every rank's array (emulated ranks share one array: one
                // store, as each real rank's poll of its own array sees one store per CTA)
                for (int q = lane; q < (SYS ? a.G : 1); q += 32)
                    st_x_v2<SYS>(sSl[q] + ((size_t)par * GT + gid) * DSLOT, (v & ~DTAGM) | tag, w1);
            } else if (v) {
                unsigned long long *mb = mbme + ((size_t)par * a.Cper + lb) * (a.nbmax + 1);
                for (int u = lane; u < t; u += 32)
                    st_x<SYS>(&mb[u], ((unsigned long long)__float_as_uint(sneg[(size_t)u * a.R + vlr]) << 32) | tag);
            }
        }
        // ---- deferred global stores of step t-1 (own rows)
        if (pend) {
            Sme[i + (int64_t)(t - 1) * a.lds] = ps;
            Lor[(int64_t)oi + (k - 1) * a.ldl] = __fdiv_rn(pc, pd);   // [R10], off the critical path
            pend = false;
        }
        PH(1)
        // ---- C: every slot of this step (tags); the max key is the pivot
        if (wid == 0) {
            const unsigned long long *sl = myslots + (size_t)par * GT * DSLOT;
            uint64_t mx, mi = 0;
            unsigned spins = 0;
            for (;;) {
                bool ok = true;
                mx = 0;
                for (int g = lane; g < GT; g += 32) {
                    unsigned long long sv, si;
                    ld_x_v2<SYS>(&sl[(size_t)g * DSLOT], sv, si);
                    ok &= ((sv & DTAGM) == tag) && ((si & DTAGM) == tag);
                    if (sv > mx) {
                        mx = sv;
                        mi = si;
                    }
                }
                if (__all_sync(0xffffffffu, ok)) break;
                if ((++spins & 1023u) == 0 && gtime() > deadline) {
                    if (lane == 0) {
                        bail = 1;
                        stat[3] = 1;
                    }
                    break;
                }
            }
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) {
                const uint64_t ox = __shfl_xor_sync(0xffffffffu, mx, o2);
                const uint64_t oi2 = __shfl_xor_sync(0xffffffffu, mi, o2);
                if (ox > mx) {
                    mx = ox;
                    mi = oi2;
                }
            }
            if (lane == 0) {
                bkey = mx;
                binfo = (uint32_t)(mi >> 32);
                blb = (uint32_t)((mi >> 14) & 0x3FFFF);
            }
        }
        __syncthreads();
        if (bail) return;
        const uint64_t bk = bkey;
        const float absd = __uint_as_float((uint32_t)(bk >> 32));
        const int64_t P = (int64_t)(DPOS_MAX - (uint32_t)((bk >> 15) & DPOS_MAX));
        const float d = ((bk >> 14) & 1) ? -absd : absd;
        // ---- [R4] stop test, in FP64, strict, against the previous accepted pivot
        const bool stop = (bk == 0) || (a.K0 + t == 0 ? (absd == 0.f)
                                                       : ((double)absd < __dmul_rn(a.tau, fabs((double)dprev))));
        if (stop) {
            if (lb == 0 && tid == 0) {
                stat[0] = (int32_t)k;
                stat[1] = t;
                stat[2] = 1;
            }
            stopped = true;
            break;
        }
        const float sg = d > 0.f ? 1.f : -1.f;
        const uint32_t w = binfo;
        const int hP = (int)(w >> 20);
        const int64_t cP = (int64_t)(w & 0xFFFFF);
        const int64_t Po = look ? (int64_t)mapme[P] : P;            // the pivot's row in the V read
        PH(2)
        // ---- D: own rows' column entries from the matrix read (peer for rows below P), then
        //      the pivot row's panel values from the winner's mailbox (+ previous panel's)
        // one unconditional global load (the address selected first), issued before the
        // mailbox poll so the two latencies overlap (threads without an entry read Vme[0])
        const float *vp = (io > Po) ? (sV[hP] + io + cP * a.ldp)    // column P on its owner
                                    : (Vme + Po + cr * a.ldp);     // row P of own column
        const bool want = !piv && i != P;
        const float v = __ldcg(want ? vp : Vme);   // consumed only after the barrier (phase E)
        {
            const unsigned long long *mb = sMb[hP] + ((size_t)par * a.Cper + blb) * (a.nbmax + 1);
            for (int u = tid; u < t; u += nthr) {
                uint64_t ww;
                unsigned spins = 0;
                for (;;) {
                    ww = ld_x<SYS>(&mb[u]);
                    if ((ww & DTAGM) == tag) break;
                    if ((++spins & 1023u) == 0 && gtime() > deadline) {
                        bail = 1;
                        stat[3] = 1;
                        break;
                    }
                }
                sp[u] = -sgm[u] * __uint_as_float((uint32_t)(ww >> 32));   // s_P^u (exact sign flip)
            }
            if (look) {
                const float *Sp = sSp[hP] + Po;
                for (int u = tid; u < nbq; u += nthr) spp[u] = Sp[(int64_t)u * a.lds];
            }
            if (tid == 0) {
                sgm[t] = sg;
                pvs[t] = (int32_t)P;
            }
        }
        __syncthreads();
        if (bail) return;
        PH(3)
        // ---- E: column, scaled column, lazy diagonal [R6]-[R8], [R10]
        const float r = __fsqrt_rn(absd);
        if (lb == 0 && tid == 0) {   // every rank records the pivot (identical everywhere)
            Dk[k] = d;
            pvme[t] = (int32_t)P;
            sgme[t] = sg;
        }
        if (has && i == P) {
            piv = true;
        } else if (!piv) {
            float cc = v;
            cc = fma_chain(cc, snp + tid, spp, nbq, a.R);   // [R8] the previous panel's pivots first
            cc = fma_chain(cc, sneg + tid, sp, t, a.R);     // then the earlier in-panel pivots, in order
            const float sv = __fdiv_rn(cc, r);
            const float ns = -sg * sv;
            sneg[(size_t)t * a.R + tid] = ns;
            ps = sv;
            pc = cc;
            pd = d;
            pend = true;
            dg = __fmaf_rn(ns, sv, dg);
        }
        dprev = d;
        ++t;
    }
    if (pend) {
        Sme[i + (int64_t)(t - 1) * a.lds] = ps;
        Lor[(int64_t)oi + (a.K0 + t - 1) * a.ldl] = __fdiv_rn(pc, pd);
    }
    if (dbgon) {
        for (int q = 0; q < 5; ++q) a.dbg[q] += ph[q];
        a.dbg[5] += t;
    }
#undef PH
    if (has && !piv) me.DG[cur][c] = dg;   // for the next panel's lookahead
    if (lb == 0) {   // off the critical path: the pivots' original indices
        for (int u = tid; u < t; u += nthr) me.pivorig[a.K0 + u] = me.orig[cur][pvs[u]];
        if (!stopped && tid == 0) me.status[1] = t;
    }
}

// --------------------------------------------------------------- per-rank setup
// V_h[i + c ldp] = RN32(K(i, j)) for own column c (original j) and rows i >= j
// (lower triangle of K [R1], [R2]); lpos = lorig = j; orig = iota
__global__ void k_dcast(int64_t L, const double *__restrict__ K, int64_t ld, int h, int G, float *__restrict__ V,
                        int64_t ldp, int64_t ncols, int32_t *lpos, int32_t *lorig) {
    for (int64_t c = blockIdx.x; c < ncols; c += gridDim.x) {
        const int64_t j = col_orig(c, h, G);
        if (threadIdx.x == 0) {
            lpos[c] = (int32_t)j;
            lorig[c] = (int32_t)j;
        }
        const double *kc = K + j * ld;
        float *vc = V + c * ldp;
        for (int64_t i = j + threadIdx.x; i < L; i += blockDim.x) vc[i] = __double2float_rn(kc[i]);
    }
}

__global__ void k_diota(int64_t n, int32_t *a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

// global stable compaction (identical on every rank): map[new] = old, orig_new
__global__ void k_dcompact(int64_t m, int nbp, const int32_t *__restrict__ pivpos, const int32_t *__restrict__ orig,
                           int32_t *__restrict__ map, int32_t *__restrict__ norig, const int32_t *status) {
    __shared__ int32_t srt[1024];
    if (status[2] || status[3]) return;
    for (int q = threadIdx.x; q < nbp; q += blockDim.x) {
        const int32_t v = pivpos[q];
        int rk = 0;
        for (int w = 0; w < nbp; ++w) rk += (pivpos[w] < v);
        srt[rk] = v;
    }
    __syncthreads();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nbp;
        while (lo < hi) {
            const int md = (lo + hi) >> 1;
            if (srt[md] < p) lo = md + 1;
            else hi = md;
        }
        if (!(lo < nbp && srt[lo] == p)) {
            map[p - lo] = (int32_t)p;
            norig[p - lo] = orig[p];
        }
    }
}

// local compaction of rank h: old local column c (position pos) -> c - #own pivots
// below pos, at position pos - #pivots below pos; cmapL[new] = old
__global__ void k_dlocal(int h, int G, int nbp, const int32_t *__restrict__ pivpos, const int32_t *__restrict__ orig,
                         const int32_t *__restrict__ lpos, const int32_t *__restrict__ lorig, int32_t *__restrict__ nlpos,
                         int32_t *__restrict__ nlorig, int32_t *__restrict__ cmapL, int32_t *nloc, int cur,
                         const int32_t *status) {
    __shared__ int32_t srt[1024], ownp[1025];
    if (status[2] || status[3]) return;
    for (int q = threadIdx.x; q < nbp; q += blockDim.x) {
        const int32_t v = pivpos[q];
        int rk = 0;
        for (int w = 0; w < nbp; ++w) rk += (pivpos[w] < v);
        srt[rk] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {   // prefix count of own pivots in sorted order
        int cnt = 0;
        ownp[0] = 0;
        for (int q = 0; q < nbp; ++q) {
            cnt += owner_of(orig[srt[q]], G) == h;
            ownp[q + 1] = cnt;
        }
        if (blockIdx.x == 0) nloc[cur ^ 1] = nloc[cur] - cnt;
    }
    __syncthreads();
    const int64_t nl = nloc[cur];
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nl; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = lpos[c];
        int lo = 0, hi = nbp;
        while (lo < hi) {
            const int md = (lo + hi) >> 1;
            if (srt[md] < p) lo = md + 1;
            else hi = md;
        }
        if (lo < nbp && srt[lo] == p) continue;   // pivoted
        const int64_t cn = c - ownp[lo];
        nlpos[cn] = p - lo;
        nlorig[cn] = lorig[c];
        cmapL[cn] = (int32_t)c;
    }
}

// the panel broadcast: Sc[t ldc + p'] = s of the row at new position p', read from
// the rank owning it (a peer read on a real run), Snc = -sigma_t s
struct DGatherArgs {
    const DRank *rp;
    int h, G, nbp, cur;
    int64_t mp, lds, ldc;
};
__global__ void k_dgather(DGatherArgs a) {
    const DRank &me = a.rp[a.h];
    if (me.status[2] || me.status[3]) return;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.mp) return;
    const int64_t o = me.map[p];                          // panel-start position of the row
    const float *src = a.rp[owner_of(me.orig[a.cur][o], a.G)].S[a.cur];
    const float *sg = me.sigma[a.cur];
    const int t0 = blockIdx.y * 16, t1 = min(a.nbp, t0 + 16);
    for (int t = t0; t < t1; ++t) {
        const float sv = src[o + (int64_t)t * a.lds];
        me.Sc[(int64_t)t * a.ldc + p] = sv;
        me.Snc[(int64_t)t * a.ldc + p] = -sg[t] * sv;
    }
}

// s of own local columns in their new order: Scol[t ldcol + c'] = Sc[t ldc + lpos'[c']];
// the tile list of the trailing update: column tile ct starts at row tile lpos'[128 ct] / 128
__global__ void k_dcols(int nbp, int64_t mp, const float *__restrict__ Sc, int64_t ldc, const int32_t *__restrict__ nlpos,
                        const int32_t *nloc, int nxt, float *__restrict__ Scol, int64_t ldcol, int32_t *tiles, int ctmax,
                        const int32_t *status) {
    if (status[2] || status[3]) return;
    const int64_t nl = nloc[nxt];
    if (blockIdx.x == 0) {   // tile prefix (one CTA)
        __shared__ int32_t cnt[1024];
        const int RT = (int)((mp + DTB - 1) / DTB);
        const int CT = (int)((nl + DTB - 1) / DTB);
        for (int ct = threadIdx.x; ct < ctmax; ct += blockDim.x) {
            int rt0 = 0, n = 0;
            if (ct < CT) {
                rt0 = nlpos[(int64_t)ct * DTB] / DTB;
                n = RT - rt0;
            }
            cnt[ct] = n;
            tiles[ctmax + 1 + ct] = rt0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int ct = 0; ct < ctmax; ++ct) {
                tiles[ct] = s;
                s += cnt[ct];
            }
            tiles[ctmax] = s;
            tiles[2 * ctmax + 1] = 0;   // the trailing kernel's tile counter
        }
        return;
    }
    const int64_t cn = (int64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
    if (cn >= ldcol) return;
    const int64_t pp = cn < nl ? (int64_t)nlpos[cn] : -1;
    for (int t = 0; t < nbp; ++t) Scol[(int64_t)t * ldcol + cn] = pp >= 0 ? Sc[(int64_t)t * ldc + pp] : 0.f;
}

__device__ __forceinline__ void cp_async16_sd(unsigned sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_d(void *sdst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}

// Trailing update of rank h's own lower-triangle columns (persistent over the tile
// list): entry (row p', local column c') starts from Vold[map[p'] + cmapL[c'] ldp]
// and receives one fmaf(-sigma_t s_I^t, s_J^t, v) per pivot t in order [R8] -- the
// inner loop of k_trailing_c; rows above the column's position are not stored.
struct DTrailArgs {
    int64_t mp;
    int nbp, ctmax, reserve;
    const float *Vold;
    float *Vnew;
    int64_t ldp;
    const int32_t *map;     // new position -> old position (rows)
    const int32_t *cmapL;   // new local column -> old local column
    const int32_t *nlpos;   // new local column -> new position
    const int32_t *nloc;    // [2]
    int nxt;
    const int32_t *tiles;
    const float *Snc, *Scol;
    int64_t ldc, ldcol;
    const int32_t *status;
};
__global__ void __launch_bounds__(256, 2) k_trailing_d(DTrailArgs a) {
    if (a.status[2] || a.status[3]) return;
    extern __shared__ __align__(16) float dsm[];
    float (*As)[DTK][DTB] = reinterpret_cast<float (*)[DTK][DTB]>(dsm);
    float (*Bs)[DTK][DTB] = reinterpret_cast<float (*)[DTK][DTB]>(dsm + DTNS * DTK * DTB);
    __shared__ int32_t rmap[DTB], cmap[DTB], cpos[DTB];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int nchunk = (a.nbp + DTK - 1) / DTK;
    if (a.reserve > 0) {   // lookahead: the first `reserve` SMs stay free for the next chain
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if ((int)smid < a.reserve) return;
    }
    __shared__ int64_t next;
    __shared__ int32_t tpre[1025], trt0[1024];   // the tile list (ctmax <= 1024), once per CTA
    for (int q = threadIdx.x; q <= a.ctmax; q += blockDim.x) tpre[q] = a.tiles[q];
    for (int q = threadIdx.x; q < a.ctmax; q += blockDim.x) trt0[q] = a.tiles[a.ctmax + 1 + q];
    const int64_t ntiles = a.tiles[a.ctmax];
    const int64_t nl = a.nloc[a.nxt];
    int *ctr = const_cast<int *>(a.tiles) + 2 * a.ctmax + 1;
#define RR(q) (((q) < 4) ? tx * 4 + (q) : 64 + tx * 4 + ((q)-4))
#define CC(q) (((q) < 4) ? ty * 4 + (q) : 64 + ty * 4 + ((q)-4))
    // the next tile's index is fetched (atomic) while the current one computes
    __shared__ int64_t after;
    if (tid == 0) next = atomicAdd(ctr, 1);
    for (;;) {
        __syncthreads();   // the previous tile's readers of As / Bs / maps are done; next is set
        const int64_t tt = next;
        if (tt >= ntiles) break;
        if (tid == 0) after = atomicAdd(ctr, 1);
        int lo = 0, hi = a.ctmax - 1;   // column tile: last ct with tiles[ct] <= tt
        while (lo < hi) {
            const int md = (lo + hi + 1) >> 1;
            if (tpre[md] <= tt) lo = md;
            else hi = md - 1;
        }
        const int ct = lo;
        const int64_t rt = trt0[ct] + (tt - tpre[ct]);
        const int64_t row0 = rt * DTB, col0 = (int64_t)ct * DTB;
        const int mpr = (int)min((int64_t)DTB, a.mp - row0), mpc = (int)min((int64_t)DTB, nl - col0);
        // source pointers advanced by one chunk per issue, rotating stage (no per-chunk
        // multiplies on the FMA pipe; see k_trailing_c)
        const int ek0 = tid >> 5, er0 = (tid & 31) * 4;
        const float *pa = a.Snc + (int64_t)ek0 * a.ldc + row0 + er0;
        const float *pb = a.Scol + (int64_t)ek0 * a.ldcol + col0 + er0;
        const unsigned sA = (unsigned)__cvta_generic_to_shared(&As[0][ek0][er0]);
        const unsigned sB = (unsigned)__cvta_generic_to_shared(&Bs[0][ek0][er0]);
        constexpr unsigned STGB = DTK * DTB * sizeof(float), EIGHTB = 8 * DTB * sizeof(float);
        unsigned soff = 0;
        auto issue = [&](int cq) {
            if (cq < nchunk) {
                cp_async16_sd(sA + soff, pa);
                cp_async16_sd(sA + soff + EIGHTB, pa + 8 * a.ldc);
                cp_async16_sd(sB + soff, pb);
                cp_async16_sd(sB + soff + EIGHTB, pb + 8 * a.ldcol);
                pa += (int64_t)DTK * a.ldc;
                pb += (int64_t)DTK * a.ldcol;
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            soff = (soff == (DTNS - 1) * STGB) ? 0u : soff + STGB;
        };
        issue(0);
        issue(1);
        if (tid < DTB) {
            rmap[tid] = (tid < mpr) ? a.map[row0 + tid] : -1;
        } else {
            const int q = tid - DTB;
            cmap[q] = (q < mpc) ? a.cmapL[col0 + q] : -1;
            cpos[q] = (q < mpc) ? a.nlpos[col0 + q] : 0x7FFFFFFF;
        }
        __syncthreads();
        float2 acc[8][4];
        // an interior tile (full, every row at or below every column's position): all 64
        // seeds exist, unmasked gathers (as in k_trailing_c)
        if (mpr == DTB && mpc == DTB && row0 >= cpos[DTB - 1]) {
            int32_t rm[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) rm[q] = rmap[RR(q)];
            const float *vold = a.Vold;
            const int64_t ldp = a.ldp;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float *c0p = vold + (int64_t)cmap[CC(2 * j)] * ldp;
                const float *c1p = vold + (int64_t)cmap[CC(2 * j + 1)] * ldp;
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
                for (int hh = 0; hh < 2; ++hh) {
                    const int cl = CC(2 * j + hh);
                    const int32_t cm = cmap[cl];
                    const int32_t cp = cpos[cl];
                    const float *colp = a.Vold + (int64_t)(cm >= 0 ? cm : 0) * a.ldp;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const bool ok = cm >= 0 && rm[q] >= 0 && row0 + RR(q) >= cp;
                        const float v = ok ? __ldg(colp + rm[q]) : 0.f;
                        if (hh) acc[q][j].y = v;
                        else acc[q][j].x = v;
                    }
                }
            }
        }
        int st = 0;
        for (int cq = 0; cq < nchunk; ++cq, st = (st == DTNS - 1) ? 0 : st + 1) {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
            issue(cq + 2);
            const int kmax = min(DTK, a.nbp - cq * DTK);
            if (kmax == DTK) {
#pragma unroll
                for (int kk = 0; kk < DTK; ++kk) {
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
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        // fully below the diagonal band (every row at or below every column's position)
        const bool full = mpr == DTB && mpc == DTB && row0 >= cpos[DTB - 1] && (a.ldp & 3) == 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int cl = CC(2 * j + hh);
                float *colp = a.Vnew + (col0 + cl) * a.ldp + row0;
                if (full) {
                    *reinterpret_cast<float4 *>(colp + tx * 4) =
                        hh ? make_float4(acc[0][j].y, acc[1][j].y, acc[2][j].y, acc[3][j].y)
                           : make_float4(acc[0][j].x, acc[1][j].x, acc[2][j].x, acc[3][j].x);
                    *reinterpret_cast<float4 *>(colp + 64 + tx * 4) =
                        hh ? make_float4(acc[4][j].y, acc[5][j].y, acc[6][j].y, acc[7][j].y)
                           : make_float4(acc[4][j].x, acc[5][j].x, acc[6][j].x, acc[7][j].x);
                } else if (cl < mpc) {
                    const int32_t cp = cpos[cl];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int rl = RR(q);
                        if (rl < mpr && row0 + rl >= cp) colp[rl] = hh ? acc[q][j].y : acc[q][j].x;
                    }
                }
            }
        }
        if (tid == 0) next = after;   // read by everyone after the barrier at the loop top
    }
#undef RR
#undef CC
}

// Lfac[a + k ldf] = L_{pivorig[a], k} from the rank owning row pivorig[a]
__global__ void k_dgather_L(int64_t N, int G, const DRank *rp, int h, int64_t ldl, float *__restrict__ Lfac,
                            int64_t ldf) {
    const int32_t *pivorig = rp[h].pivorig;
    for (int64_t k = blockIdx.x; k < N; k += gridDim.x) {
        float *dst = Lfac + k * ldf;
        for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
            float v = 0.f;
            if (r == k) v = 1.f;
            else if (r > k) {
                const int32_t o = pivorig[r];
                v = rp[owner_of(o, G)].Lorig[o + k * ldl];
            }
            dst[r] = v;
        }
    }
}

// cross-rank barrier (real ranks): every rank adds 1 to every rank's counter
// (release, system scope), then waits until its own counter reaches G * epoch
__global__ void k_xbar(const DRank *rp, int G, int h, int which, unsigned int epoch, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    for (int q = 0; q < G; ++q) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(rp[q].bar + which) : "memory");
    const unsigned long long deadline = gtime() + timeout_ns;
    const unsigned int want = (unsigned int)G * epoch;
    unsigned int v;
    unsigned spins = 0;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(rp[h].bar + which) : "memory");
        if (v >= want) break;
        if ((++spins & 1023u) == 0 && gtime() > deadline) {
            rp[h].status[3] = 1;
            break;
        }
    }
}

}  // namespace

// ------------------------------------------------------------------ host driver
struct DistBufs {
    DBuf<float> V[2], S[2], DG[2], sigma[2], Sc, Snc, Scol, Dk;
    DBuf<int32_t> lpos[2], lorig[2], pivpos[2], orig[2], nloc, cmapL, pivorig, status, map, tiles;
    DBuf<unsigned long long> slots, mbox;
    DBuf<unsigned int> bar;
};

// trailing: one FMA per lower-triangle entry per pivot (the same algorithmic count as
// one GPU: every pair is stored on exactly one rank)
static double dtrail_flops_total(int64_t mp, int nbp) { return (double)mp * (double)(mp + 1) * nbp; }
// "<cls>@<rank>": per-rank kernel classes of the emulation (tools/dist_model.py)
static const char *rank_class(const char *cls, int h) {
    static std::vector<std::string> names[2];
    const int w = cls[0] == 't' ? 0 : 1;
    auto &v = names[w];
    if (v.capacity() < 64) v.reserve(64);   // c_str() pointers stay valid (G <= 64)
    while ((int)v.size() <= h) v.push_back(std::string(cls) + "@" + std::to_string(v.size()));
    return v[h].c_str();
}

void lowprec_factor_dist(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                         hf_lowfactor *lf, int nparts) {
    cudaStream_t st = ctx->stream;
    const int nsm = ctx->num_sms;
    lf->L = L;
    lf->stream = st;
    if (L == 0) {
        lf->N = lf->Ntau = lf->n2 = 0;
        return;
    }
    // real ranks: a multi-GPU context, or a one-rank NCCL context asked for one partition
    // (the real-rank code path -- IPC handles over NCCL, device barrier, system-scope
    // exchange -- on a single GPU, for the tests; there are no peers to map)
    bool real = ctx->nranks > 1;
#ifdef HF_WITH_NCCL
    if (ctx->comm && ctx->nranks == 1 && nparts == 1) real = true;
#endif
    const int G = real ? ctx->nranks : nparts;
    HF_REQUIRE(L <= (int64_t)DPOS_MAX - 1, "L too large for the 17-bit position key");
    HF_REQUIRE(G >= 1 && G <= 64, "stage-1 ranks out of range (1..64)");
    HF_REQUIRE(L <= ((int64_t)1 << 20), "L too large for the 20-bit local column field");
    const int lo = real ? ctx->rank : 0, hi = real ? ctx->rank + 1 : G;
    std::vector<int64_t> ncols(G, 0);
    for (int64_t j = 0; j < L; ++j) ncols[(j / DCB) % G]++;
    int64_t ncmax = 1;
    for (auto c : ncols) ncmax = std::max(ncmax, c);
    // lookahead (HF_DIST_LOOKAHEAD=1: the chain of panel p+1 runs while panel p's trailing
    // update runs on a second stream, on the SMs the chain leaves free).  Off by default:
    // measured on one B200 the chain runs 1.57x slower beside the concurrent update and
    // the time model then projects the serial schedule faster at every G
    // (profiles/dist_lookahead_c2_r02.log, profiles/dist_model_c4_r02.json).
    // (=2: the lookahead chain with everything on one stream -- the time model's
    // measurement of the lookahead chain's own cost, no concurrency)
    bool look = false;
    int look_mode = 0;
    if (const char *e = getenv("HF_DIST_LOOKAHEAD")) look_mode = atoi(e);
    look = look_mode != 0;

    // chain geometry: Cper CTAs per rank, R rows each, the panel's values of own rows in
    // shared memory (R x nb floats, twice with lookahead); about one GPU's worth of slots
    // in total (G x Cper ~ #SMs) -- the same per-rank geometry for real and emulated ranks,
    // so the emulation measures the real per-rank chain up to the NVLink latency
    int maxsmem = 0;
    HF_CUDA(cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    cudaFuncAttributes fa, fb;
    HF_CUDA(cudaFuncGetAttributes(&fa, k_chain_d<false>));
    HF_CUDA(cudaFuncGetAttributes(&fb, k_chain_d<true>));
    maxsmem -= (int)std::max(fa.sharedSizeBytes, fb.sharedSizeBytes) + 64;
    const int cmax_sm = real ? nsm : std::max(1, nsm / G);
    // as few CTAs as the panel's shared memory allows (fewer CTAs: a cheaper exchange; the
    // one-GPU chain's measured optimum is 64 CTAs at C2), at least 64 over all ranks
    const int nf0 = look ? 2 : 1;
    const int64_t rows_fit = std::max<int64_t>(32, (int64_t)(maxsmem / 4) / (nf0 * 128 + 4));
    int cper_def = (int)std::min<int64_t>(cmax_sm, std::max<int64_t>(cdiv(64, G), cdiv(ncmax, rows_fit)));
    if (const char *e = getenv("HF_DIST_CTAS")) cper_def = std::max(1, std::min(cmax_sm, atoi(e)));
    int Cmax = std::max(cper_def, (int)std::min<int64_t>(cmax_sm, cdiv(ncmax, 1024)));
    int64_t R0 = cdiv(ncmax, Cmax);
    const int nf = look ? 2 : 1;
    auto fits = [&](int nbx, int64_t R) { return (int64_t)(nf * nbx * R + 4 * nbx + 16) * 4 <= (int64_t)maxsmem; };
    int nb = o.nb > 0 ? o.nb : 128;
    while (nb > 16 && !fits(nb, R0)) nb -= 16;
    while (nb > 8 && !fits(nb, R0)) nb /= 2;
    while (!fits(nb, R0) && Cmax < cmax_sm) {   // more CTAs if the panel does not fit even at nb = 8
        ++Cmax;
        R0 = cdiv(ncmax, Cmax);
    }
    HF_REQUIRE(R0 <= 1024 && fits(nb, R0), "stage 1 (distributed): a rank's rows do not fit its chain CTAs");
    const int64_t ldp = L, lds = L, ldl = L;
    const int64_t ldc = cdiv(L, DTB) * DTB;
    const int64_t ldcol = cdiv(ncmax, DTB) * DTB;
    const int ctmax = (int)cdiv(ncmax, DTB);
    HF_REQUIRE(ctmax <= 1024, "stage 1 (distributed): too many column tiles per rank");
    const int nbpad = (int)cdiv(nb, DTK) * DTK;

    std::vector<DistBufs> B(G);
    DBuf<float> Lorig_all;
    std::vector<DRank> tab(G);
    std::memset(tab.data(), 0, sizeof(DRank) * G);
    for (int h = lo; h < hi; ++h) {
        DistBufs &b = B[h];
        const int64_t nc = std::max<int64_t>(ncols[h], 1);
        DRank &r = tab[h];
        for (int q = 0; q < 2; ++q) {
            b.V[q].alloc((size_t)L * nc, st);
            b.lpos[q].alloc(nc, st);
            b.lorig[q].alloc(nc, st);
            b.orig[q].alloc(L, st);
            b.S[q].alloc((size_t)L * nb, st);
            b.DG[q].alloc(nc, st);
            b.sigma[q].alloc(nb, st);
            b.pivpos[q].alloc(nb, st);
            r.V[q] = b.V[q].p; r.lpos[q] = b.lpos[q].p; r.lorig[q] = b.lorig[q].p; r.orig[q] = b.orig[q].p;
            r.S[q] = b.S[q].p; r.DG[q] = b.DG[q].p; r.sigma[q] = b.sigma[q].p; r.pivpos[q] = b.pivpos[q].p;
        }
        b.Sc.alloc((size_t)ldc * nbpad, st);
        b.Snc.alloc((size_t)ldc * nbpad, st);
        b.Scol.alloc((size_t)ldcol * nbpad, st);
        b.Dk.alloc(L, st);
        b.nloc.alloc(2, st);
        b.cmapL.alloc(nc, st);
        b.pivorig.alloc(L, st);
        b.status.alloc(4, st);
        b.status.zero(st);
        b.map.alloc(L, st);
        b.tiles.alloc((size_t)2 * ctmax + 2, st);
        b.slots.alloc((size_t)2 * G * Cmax * DSLOT, st);
        b.slots.zero(st);
        b.mbox.alloc((size_t)2 * Cmax * (nb + 1), st);
        b.mbox.zero(st);
        b.bar.alloc(2, st);
        b.bar.zero(st);
        r.nloc = b.nloc.p; r.cmapL = b.cmapL.p; r.slots = b.slots.p; r.mbox = b.mbox.p;
        r.Dk = b.Dk.p; r.pivorig = b.pivorig.p; r.status = b.status.p;
        r.map = b.map.p; r.tiles = b.tiles.p; r.Sc = b.Sc.p; r.Snc = b.Snc.p; r.Scol = b.Scol.p; r.bar = b.bar.p;
    }
    if (!real)   // emulated ranks share one slot array (see k_chain_d's publish)
        for (int h = lo; h < hi; ++h) tab[h].slots = B[lo].slots.p;
    // the factor rows by original index: one per rank on a real run, shared when emulated
    Lorig_all.alloc((size_t)L * L, st);
    for (int h = lo; h < hi; ++h) tab[h].Lorig = Lorig_all.p;
    std::vector<void *> opened;
#ifdef HF_WITH_NCCL
    if (real) {
        // peers' V and S (both buffers), slots, mbox, Lorig, barrier counters: CUDA-IPC
        // handles all-gathered over NCCL, opened with peer access (NVLink)
        constexpr int NH = 8;
        const DRank &m0 = tab[ctx->rank];
        void *mine[NH] = {m0.V[0], m0.V[1], m0.S[0], m0.S[1], m0.slots, m0.mbox, m0.Lorig, m0.bar};
        std::vector<cudaIpcMemHandle_t> hm(NH);
        for (int q = 0; q < NH; ++q) HF_CUDA(cudaIpcGetMemHandle(&hm[q], mine[q]));
        const size_t hb = NH * sizeof(cudaIpcMemHandle_t);
        DBuf<char> dh;
        dh.alloc(hb * (G + 1), st);
        HF_CUDA(cudaMemcpyAsync(dh.p, hm.data(), hb, cudaMemcpyHostToDevice, st));
        collective_allgather_bytes(ctx, dh.p, dh.p + hb, hb);
        std::vector<cudaIpcMemHandle_t> all((size_t)NH * G);
        HF_CUDA(cudaMemcpyAsync(all.data(), dh.p + hb, hb * G, cudaMemcpyDeviceToHost, st));
        HF_CUDA(cudaStreamSynchronize(st));
        for (int g = 0; g < G; ++g) {
            if (g == ctx->rank) continue;
            void *pp[NH];
            for (int q = 0; q < NH; ++q) {
                HF_CUDA(cudaIpcOpenMemHandle(&pp[q], all[(size_t)g * NH + q], cudaIpcMemLazyEnablePeerAccess));
                opened.push_back(pp[q]);
            }
            tab[g].V[0] = (float *)pp[0]; tab[g].V[1] = (float *)pp[1];
            tab[g].S[0] = (float *)pp[2]; tab[g].S[1] = (float *)pp[3];
            tab[g].slots = (unsigned long long *)pp[4]; tab[g].mbox = (unsigned long long *)pp[5];
            tab[g].Lorig = (float *)pp[6]; tab[g].bar = (unsigned int *)pp[7];
        }
    }
#else
    HF_REQUIRE(!real, "multi-GPU stage 1 needs NCCL");
#endif
    DBuf<DRank> dtab;
    dtab.alloc(G, st);
    HF_CUDA(cudaMemcpyAsync(dtab.p, tab.data(), sizeof(DRank) * G, cudaMemcpyHostToDevice, st));
    const unsigned long long timeout_ns = 60ull * 1000000000ull;
    cudaStream_t st2 = st;
    if (look && look_mode != 2) {
        if (!ctx->side) {
            HF_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
            for (auto &e : ctx->ev) HF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        st2 = ctx->side;
    }
    unsigned int bar_epoch[2] = {0, 0};
    auto xbar = [&](cudaStream_t s, int which) {   // real ranks only: stream-ordered device barrier
        if (!real) return;
        ++bar_epoch[which];
        k_xbar<<<1, 32, 0, s>>>(dtab.p, G, ctx->rank, which, bar_epoch[which], timeout_ns);
        HF_CHECK_LAUNCH(ctx);
    };
    // per-panel device times of the emulation (HF_DIST_PANEL_TIMES: tools/dist_model.py)
    const bool ptimes = !real && getenv("HF_DIST_PANEL_TIMES") != nullptr;
    std::vector<cudaEvent_t> pev;
    std::vector<int> pkind;   // 0: a chain (2 events), 1: one rank's gather + trailing (3 events)
    auto pevent = [&](cudaStream_t s) {
        if (!ptimes) return;
        cudaEvent_t e;
        HF_CUDA(cudaEventCreate(&e));
        HF_CUDA(cudaEventRecord(e, s));
        pev.push_back(e);
    };

    {
        ClassTimer tm(ctx, "other");
        for (int h = lo; h < hi; ++h) {
            DistBufs &b = B[h];
            k_dcast<<<(unsigned)std::min<int64_t>(std::max<int64_t>(ncols[h], 1), 65535), 256, 0, st>>>(
                L, K, ld, h, G, b.V[0].p, ldp, ncols[h], b.lpos[0].p, b.lorig[0].p);
            HF_CHECK_LAUNCH(ctx);
            k_diota<<<(unsigned)cdiv(L, 256), 256, 0, st>>>(L, b.orig[0].p);
            HF_CHECK_LAUNCH(ctx);
            const int32_t nl0[2] = {(int32_t)ncols[h], 0};
            HF_CUDA(cudaMemcpyAsync(b.nloc.p, nl0, sizeof(nl0), cudaMemcpyHostToDevice, st));
        }
        HF_CUDA(cudaStreamSynchronize(st));   // nl0 dies here
    }
    xbar(st, 0);   // every rank's columns are cast before anyone reads them
    for (void *kf : {(void *)k_chain_d<false>, (void *)k_chain_d<true>, (void *)k_chain_d<false, 256>,
                     (void *)k_chain_d<true, 256>, (void *)k_chain_d<false, 512>, (void *)k_chain_d<true, 512>})
        HF_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_trailing_d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DTRAIL_SMEM));
    int tocc = 0;
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, k_trailing_d, 256, DTRAIL_SMEM));
    const int tgrid = std::max(1, tocc) * nsm;
    if (st2 != st) {
        HF_CUDA(cudaEventRecord(ctx->ev[0], st));   // the side stream starts after the setup
        HF_CUDA(cudaStreamWaitEvent(st2, ctx->ev[0], 0));
    }

    const bool want_dbg = getenv("HF_CHAIN_DEBUG") != nullptr;
    DBuf<unsigned long long> dbgbuf;
    if (want_dbg) {
        dbgbuf.alloc(8, st);
        dbgbuf.zero(st);
    }
    int cur = 0, nbprev = 0;
    int64_t m = L, K0 = 0;
    bool loc_pending = false;   // lookahead: a compaction on st2 the next chain must wait for
    while (m > 0) {
        const int nbp = (int)std::min<int64_t>(nb, m);
        const int nbq = (look && K0 > 0) ? nbprev : 0;
        // rows per rank are at most min(ncols, m): fewer chain CTAs as the matrix shrinks
        const int64_t rows_hi = std::min<int64_t>(ncmax, m);
        const int Cper = (int)std::max<int64_t>(1, std::min<int64_t>(Cmax, cdiv(rows_hi, R0)));
        const int nthr = (int)std::max<int64_t>(64, cdiv(R0, 32) * 32);
        const size_t shm = ((size_t)(nbp + nbq) * R0 + 4 + 3 * (size_t)nbp + nbq + 8) * sizeof(float);
        DChainArgs ca;
        ca.rp = dtab.p; ca.G = G; ca.rank0 = lo; ca.Cper = Cper; ca.R = (int)R0; ca.cur = cur; ca.nbp = nbp;
        ca.nbmax = nb; ca.nbq = nbq; ca.m = m; ca.K0 = K0; ca.ldp = ldp; ca.lds = lds; ca.ldl = ldl; ca.tau = o.tau;
        ca.timeout_ns = timeout_ns;
        ca.dbg = want_dbg ? dbgbuf.p : nullptr;
        if (loc_pending) {   // the previous panel's compaction (and the trailing update before it)
            HF_CUDA(cudaStreamWaitEvent(st, ctx->ev[1], 0));
            loc_pending = false;
        }
        if (ptimes) pkind.push_back(0);
        pevent(st);
        {
            double cf = 0.0;
            for (int t = 0; t < nbp; ++t) cf += 2.0 * (double)(m - t) * (t + nbq);
            ClassTimer tm(ctx, "chain", st, cf, 16.0 * ((double)m * nbp - 0.5 * (double)nbp * (nbp - 1)));
            void *args[] = {&ca};
            const int lb = std::max(nthr, getenv("HF_CHAIN_LB") ? atoi(getenv("HF_CHAIN_LB")) : 0);
            void *kf = real ? (lb <= 256 ? (void *)k_chain_d<true, 256> : lb <= 512 ? (void *)k_chain_d<true, 512>
                                                                               : (void *)k_chain_d<true>)
                            : (lb <= 256 ? (void *)k_chain_d<false, 256> : lb <= 512 ? (void *)k_chain_d<false, 512>
                                                                                : (void *)k_chain_d<false>);
            HF_CUDA(cudaLaunchCooperativeKernel(kf, dim3((unsigned)((hi - lo) * Cper)), dim3(nthr), args, shm, st));
            HF_CHECK_LAUNCH(ctx);
        }
        pevent(st);
        xbar(st, 0);   // every rank's S of this panel is written before it is gathered
        const int64_t mp = m - nbp;
        if (mp > 0) {
            if (st2 != st) {   // the side stream waits for this chain
                HF_CUDA(cudaEventRecord(ctx->ev[2], st));
                HF_CUDA(cudaStreamWaitEvent(st2, ctx->ev[2], 0));
            }
            for (int h = lo; h < hi; ++h) {   // compaction of this panel (global and own columns)
                DistBufs &b = B[h];
                ClassTimer tm(ctx, "other", st2);
                ClassTimer tr(ctx, rank_class("gather", h), st2);
                k_dcompact<<<(unsigned)std::min<int64_t>(cdiv(m, 256), 4096), 256, 0, st2>>>(
                    m, nbp, b.pivpos[cur].p, b.orig[cur].p, b.map.p, b.orig[cur ^ 1].p, b.status.p);
                HF_CHECK_LAUNCH(ctx);
                k_dlocal<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(ncols[h], 256), 1024)), 256, 0, st2>>>(
                    h, G, nbp, b.pivpos[cur].p, b.orig[cur].p, b.lpos[cur].p, b.lorig[cur].p, b.lpos[cur ^ 1].p,
                    b.lorig[cur ^ 1].p, b.cmapL.p, b.nloc.p, cur, b.status.p);
                HF_CHECK_LAUNCH(ctx);
            }
            if (st2 != st) {   // the next chain waits for this compaction (and what precedes it on st2)
                HF_CUDA(cudaEventRecord(ctx->ev[1], st2));
                loc_pending = true;
            }
            for (int h = lo; h < hi; ++h) {
                DistBufs &b = B[h];
                if (ptimes) pkind.push_back(1);
                pevent(st2);
                {
                    ClassTimer tm(ctx, "other", st2);
                    ClassTimer tr(ctx, rank_class("gather", h), st2);
                    DGatherArgs ga;
                    ga.rp = dtab.p; ga.h = h; ga.G = G; ga.nbp = nbp; ga.cur = cur; ga.mp = mp; ga.lds = lds; ga.ldc = ldc;
                    k_dgather<<<dim3((unsigned)cdiv(mp, 256), (unsigned)cdiv(nbp, 16)), 256, 0, st2>>>(ga);
                    HF_CHECK_LAUNCH(ctx);
                    k_dcols<<<(unsigned)(1 + cdiv(ldcol, 256)), 256, 0, st2>>>(nbp, mp, b.Sc.p, ldc, b.lpos[cur ^ 1].p,
                                                                             b.nloc.p, cur ^ 1, b.Scol.p, ldcol,
                                                                             b.tiles.p, ctmax, b.status.p);
                    HF_CHECK_LAUNCH(ctx);
                }
                pevent(st2);
                DTrailArgs ta;
                ta.mp = mp; ta.nbp = nbp; ta.ctmax = ctmax; ta.Vold = b.V[cur].p; ta.Vnew = b.V[cur ^ 1].p;
                ta.ldp = ldp; ta.map = b.map.p; ta.cmapL = b.cmapL.p; ta.nlpos = b.lpos[cur ^ 1].p; ta.nloc = b.nloc.p;
                ta.nxt = cur ^ 1; ta.tiles = b.tiles.p; ta.Snc = b.Snc.p; ta.Scol = b.Scol.p; ta.ldc = ldc;
                ta.ldcol = ldcol; ta.status = b.status.p;
                // real ranks with lookahead: leave the chain's SMs free (the next chain
                // launches while this update runs); the emulation's chain spans every SM
                // (G = 1: one GPU, the lookahead is real there too)
                ta.reserve = (look && st2 != st && (real || G == 1)) ? Cmax : 0;
                ClassTimer tm(ctx, "trailing", st2, dtrail_flops_total(mp, nbp) / G, 0.0);
                ClassTimer tr(ctx, rank_class("trailing", h), st2);   // per rank (the time model)
                k_trailing_d<<<(unsigned)tgrid, 256, DTRAIL_SMEM, st2>>>(ta);
                HF_CHECK_LAUNCH(ctx);
                pevent(st2);
            }
            xbar(st2, 1);   // every rank's columns of the next-but-one chain's matrix are updated
            cur ^= 1;
        }
        nbprev = nbp;
        K0 += nbp;
        m = mp;
    }
    if (st2 != st) {   // join the side stream
        HF_CUDA(cudaEventRecord(ctx->ev[3], st2));
        HF_CUDA(cudaStreamWaitEvent(st, ctx->ev[3], 0));
    }
    if (ptimes) {   // per panel: chain ms; per rank: gather ms and trailing ms
        HF_CUDA(cudaStreamSynchronize(st));
        std::string line = "[";
        size_t q = 0;
        for (size_t pi = 0; pi < pkind.size(); ++pi) {
            if (pkind[pi] == 0) {   // chain start / end
                float ch = 0.f;
                cudaEventElapsedTime(&ch, pev[q], pev[q + 1]);
                line += std::string(pi ? "]},{" : "{") + "\"chain\":" + std::to_string(ch) + ",\"ranks\":[";
                q += 2;
            } else {                // gather start / trailing start / trailing end of one rank
                float g = 0.f, t = 0.f;
                cudaEventElapsedTime(&g, pev[q], pev[q + 1]);
                cudaEventElapsedTime(&t, pev[q + 1], pev[q + 2]);
                line += std::string(pkind[pi - 1] == 0 ? "" : ",") + "[" + std::to_string(g) + "," + std::to_string(t) + "]";
                q += 3;
            }
        }
        line += pkind.empty() ? "]" : "]}]";
        fprintf(stderr, "[hf dist panels] %s\n", line.c_str());
        for (auto e : pev) cudaEventDestroy(e);
    }
    if (want_dbg) {
        unsigned long long hd[8];
        HF_CUDA(cudaMemcpy(hd, dbgbuf.p, sizeof(hd), cudaMemcpyDeviceToHost));
        const double np = hd[5] ? (double)hd[5] : 1.0;
        fprintf(stderr, "[hf dchain] steps %llu  us/step: argmax %.3f  publish %.3f  exchange %.3f  fetch %.3f  compute %.3f\n",
                hd[5], hd[4] / np * 1e-3, hd[0] / np * 1e-3, hd[1] / np * 1e-3, hd[2] / np * 1e-3, hd[3] / np * 1e-3);
    }
    // outputs: every rank holds the pivots, D and the status; the factor rows come
    // from their owners
    const int me = lo;
    lowprec_outputs(ctx, L, o, lf, B[me].status.p, B[me].pivorig.p, B[me].Dk.p);
    if (lf->N > 0) {
        ClassTimer tm(ctx, "other");
        k_dgather_L<<<(unsigned)std::min<int64_t>(lf->N, 65535), 256, 0, st>>>(lf->N, G, dtab.p, me, ldl, lf->Lfac.p,
                                                                              lf->N);
        HF_CHECK_LAUNCH(ctx);
    }
    xbar(st, 0);   // nobody reads a peer's buffers any more
    HF_CUDA(cudaStreamSynchronize(st));
    int32_t hs[4];
    HF_CUDA(cudaMemcpy(hs, B[me].status.p, sizeof(hs), cudaMemcpyDeviceToHost));
    for (void *p : opened) cudaIpcCloseMemHandle(p);
    if (hs[3] != 0) throw Error{HF_ERR_NCCL, "stage 1: a peer did not answer within the exchange timeout (multi-GPU chain)"};
}

}  // namespace hf
