// k_lowprec64.cu -- NEXT-1, the lower precision of the paper's
// (double, double-double) pair: stage 1 of Alg. 1 in FP64 -- the same
// symmetric max-|diag| pivoting with threshold postponing
// and the same canonical arithmetic [R2]-[R10] with T = double (fma, sqrt and
// division in IEEE double), bitwise against the oracle's FP64 variant
// (oracle_factor_f64).  Same structure as k_lowprec.cu (blocked left-looking
// panels, lazy diagonal, stable compaction, one cooperative chain launch per
// panel, canonical trailing update), with these FP64 differences:
//  * the pivot key does not fit 64 bits (|d| takes 63): every exchanged value
//    travels as "LL" words of 32-bit payload + 32-bit step tag (the key as
//    three words |d| hi, |d| lo, position/sign; mailbox values as two), so a
//    reader validates each word by its tag with no fences;
//  * the trailing update is DFMA on 64 x 64 tiles (4 x 4 per thread).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>

#include "hf_internal.cuh"

namespace hf {
namespace {

constexpr uint32_t POS_MAX64 = 0x1FFFF;
constexpr int SLOT_WORDS = 32;   // 256 B per CTA slot (one L2 line each)

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// key = (|d| bits, (POS_MAX - pos) << 1 | sign): lexicographic max = [R3]
struct Key64 {
    unsigned long long ab;
    uint32_t pi;
};
__device__ __forceinline__ bool key_gt(const Key64 &x, const Key64 &y) {
    return x.ab > y.ab || (x.ab == y.ab && x.pi > y.pi);
}
__device__ __forceinline__ Key64 warp_max_key(Key64 k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Key64 y{__shfl_xor_sync(0xffffffffu, k.ab, o), __shfl_xor_sync(0xffffffffu, k.pi, o)};
        if (key_gt(y, k)) k = y;
    }
    return k;
}

__global__ void k_copy_lower64(int64_t L, const double *__restrict__ K, int64_t ldk, double *__restrict__ V,
                               int64_t ldv) {
    for (int64_t j = blockIdx.x; j < L; j += gridDim.x)
        for (int64_t i = j + threadIdx.x; i < L; i += blockDim.x) V[i + j * ldv] = K[i + j * ldk];
}

__global__ void k_iota32_64(int64_t n, int32_t *a) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

struct Chain64Args {
    int64_t m, K0;
    int nbp, R;
    double tau;
    const double *V;
    int64_t ldv;
    const int32_t *orig;
    double *S, *Sn;
    int64_t lds;
    int32_t *pivpos;
    double *Lorig;
    int64_t ldl;
    double *Dk;
    int32_t *pivorig;
    unsigned long long *slots;   // [2][G][SLOT_WORDS]
    unsigned long long *mbox;    // [2][G][2 nb]
    int32_t *status;
};

// MAXT: the launch bound, as k_chain's (a 256 / 512 bound lifts the 64-register cap)
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_chain64(Chain64Args a) {
    extern __shared__ double smem64[];
    __shared__ unsigned long long rab[32];
    __shared__ uint32_t rpi[32];
    __shared__ Key64 bkey;
    if (*(volatile int32_t *)&a.status[2]) return;
    const int G = gridDim.x;
    const int tid = threadIdx.x, nthr = blockDim.x, nwarp = nthr >> 5, lane = tid & 31, wid = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * a.R;
    const int64_t nown = max((int64_t)0, min((int64_t)a.R, a.m - r0));
    const int nb = a.nbp;
    double *sneg = smem64;                     // [nbp][R]
    double *sp = smem64 + (size_t)nb * a.R;    // [nbp]
    double *sgm = sp + nb;                     // [nbp]
    const bool has = tid < nown;
    const int64_t i = r0 + tid;
    const int32_t oi = has ? a.orig[i] : 0;
    double dg = has ? a.V[i + i * a.ldv] : 0.0;
    bool piv = !has;
    double dprev = a.K0 > 0 ? a.Dk[a.K0 - 1] : 0.0;
    bool pend = false;
    double ps = 0.0, pn = 0.0, pl = 0.0;
    int t = 0;
    bool stopped = false;
    for (; t < nb; ++t) {
        const int64_t k = a.K0 + t;
        const unsigned long long tag = (unsigned long long)(uint32_t)(k + 1);
        // ---- local argmax [R3]
        Key64 key{0ull, 0u};
        if (!piv) key = Key64{(unsigned long long)__double_as_longlong(fabs(dg)),
                              ((POS_MAX64 - (uint32_t)i) << 1) | (dg < 0.0 ? 1u : 0u)};
        key = warp_max_key(key);
        if (lane == 0) {
            rab[wid] = key.ab;
            rpi[wid] = key.pi;
        }
        __syncthreads();
        // ---- publish: warp 0 the key words, warp 1 the candidate row's panel values
        if (wid < 2) {
            Key64 v = (lane < nwarp) ? Key64{rab[lane], rpi[lane]} : Key64{0ull, 0u};
            v = warp_max_key(v);
            if (wid == 0 && lane == 0) {
                unsigned long long *slot = a.slots + ((size_t)(t & 1) * G + blockIdx.x) * SLOT_WORDS;
                st_relaxed_u64(slot + 0, ((v.ab >> 32) << 32) | tag);
                st_relaxed_u64(slot + 1, ((v.ab & 0xFFFFFFFFull) << 32) | tag);
                st_relaxed_u64(slot + 2, ((unsigned long long)v.pi << 32) | tag);
            } else if (wid == 1 && v.pi) {
                unsigned long long *mb = a.mbox + ((size_t)(t & 1) * G + blockIdx.x) * (2 * nb);
                const int lr = (int)((int64_t)(POS_MAX64 - (v.pi >> 1)) - r0);
                for (int u = lane; u < t; u += 32) {
                    const unsigned long long bits = (unsigned long long)__double_as_longlong(sneg[(size_t)u * a.R + lr]);
                    st_relaxed_u64(&mb[2 * u], ((bits >> 32) << 32) | tag);
                    st_relaxed_u64(&mb[2 * u + 1], ((bits & 0xFFFFFFFFull) << 32) | tag);
                }
            }
        }
        if (pend) {
            a.S[i + (int64_t)(t - 1) * a.lds] = ps;
            a.Sn[i + (int64_t)(t - 1) * a.lds] = pn;
            a.Lorig[(int64_t)oi + (k - 1) * a.ldl] = pl;
            pend = false;
        }
        // ---- exchange: warp 0 reads every slot of this step
        if (wid == 0) {
            const unsigned long long *sl = a.slots + (size_t)(t & 1) * G * SLOT_WORDS;
            Key64 mx;
            for (;;) {
                bool ok = true;
                mx = Key64{0ull, 0u};
                for (int g = lane; g < G; g += 32) {
                    const unsigned long long w0 = ld_relaxed_u64(&sl[(size_t)g * SLOT_WORDS + 0]);
                    const unsigned long long w1 = ld_relaxed_u64(&sl[(size_t)g * SLOT_WORDS + 1]);
                    const unsigned long long w2 = ld_relaxed_u64(&sl[(size_t)g * SLOT_WORDS + 2]);
                    ok &= ((w0 & 0xFFFFFFFFull) == tag) && ((w1 & 0xFFFFFFFFull) == tag) &&
                          ((w2 & 0xFFFFFFFFull) == tag);
                    const Key64 c{((w0 >> 32) << 32) | (w1 >> 32), (uint32_t)(w2 >> 32)};
                    if (key_gt(c, mx)) mx = c;
                }
                if (__all_sync(0xffffffffu, ok)) break;
            }
            mx = warp_max_key(mx);
            if (lane == 0) bkey = mx;
        }
        __syncthreads();
        const Key64 bk = bkey;
        const double absd = __longlong_as_double((long long)bk.ab);
        const int64_t P = (int64_t)(POS_MAX64 - (bk.pi >> 1));
        const double d = (bk.pi & 1u) ? -absd : absd;
        // ---- [R4] stop test, strict, in FP64
        const bool stop = (k == 0) ? (absd == 0.0) : (absd < __dmul_rn(a.tau, fabs(dprev)));
        if (stop) {
            if (blockIdx.x == 0 && tid == 0) {
                a.status[0] = (int32_t)k;
                a.status[1] = t;
                a.status[2] = 1;
            }
            stopped = true;
            break;
        }
        const double sg = d > 0.0 ? 1.0 : -1.0;
        {
            const int owner = (int)(P / a.R);
            const unsigned long long *mb = a.mbox + ((size_t)(t & 1) * G + owner) * (2 * nb);
            for (int u = tid; u < t; u += nthr) {
                unsigned long long h, l;
                do {
                    h = ld_relaxed_u64(&mb[2 * u]);
                } while ((h & 0xFFFFFFFFull) != tag);
                do {
                    l = ld_relaxed_u64(&mb[2 * u + 1]);
                } while ((l & 0xFFFFFFFFull) != tag);
                const double val = __longlong_as_double((long long)(((h >> 32) << 32) | (l >> 32)));
                sp[u] = -sgm[u] * val;   // s_P^u (exact sign flip)
            }
            if (tid == 0) sgm[t] = sg;
        }
        double v = 0.0;
        if (!piv && i != P) v = (i >= P) ? a.V[i + P * a.ldv] : a.V[P + i * a.ldv];
        __syncthreads();
        const double r = __dsqrt_rn(absd);   // [R7]
        if (has && i == P) {
            piv = true;
            a.Dk[k] = d;
            a.pivorig[k] = oi;
            a.pivpos[t] = (int32_t)P;
        } else if (!piv) {
            double c = v;
            const double *sn = sneg + tid;
            for (int u = 0; u < t; ++u) c = __fma_rn(sn[(size_t)u * a.R], sp[u], c);   // [R8] in order
            const double sv = __ddiv_rn(c, r);
            const double ns = -sg * sv;
            sneg[(size_t)t * a.R + tid] = ns;
            ps = sv;
            pn = ns;
            pl = __ddiv_rn(c, d);   // [R10] L = c / d
            pend = true;
            dg = __fma_rn(ns, sv, dg);
        }
        dprev = d;
    }
    if (pend) {
        a.S[i + (int64_t)(t - 1) * a.lds] = ps;
        a.Sn[i + (int64_t)(t - 1) * a.lds] = pn;
        a.Lorig[(int64_t)oi + (a.K0 + t - 1) * a.ldl] = pl;
    }
    if (!stopped && blockIdx.x == 0 && tid == 0) a.status[1] = t;
}

__global__ void k_compact64(int64_t m, int nbp, const int32_t *__restrict__ pivpos, const int32_t *__restrict__ orig,
                            int32_t *__restrict__ map, int32_t *__restrict__ norig, const int32_t *status) {
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
        int lo = 0, hi = nbp;
        while (lo < hi) {
            int md = (lo + hi) >> 1;
            if (srt[md] < p) lo = md + 1; else hi = md;
        }
        if (!(lo < nbp && srt[lo] == p)) {
            map[p - lo] = (int32_t)p;
            norig[p - lo] = orig[p];
        }
    }
}

// symmetric rank-nbp update of the trailing lower triangle, DFMA, 64 x 64 tiles,
// 256 threads x (4 x 4); one fma per entry per pivot, in order [R8]
constexpr int TB64 = 64, TK64 = 16;
struct Trail64Args {
    int64_t mp;
    int nbp;
    const double *Vold;
    double *Vnew;
    int64_t ldv;
    const int32_t *map;
    const double *S, *Sn;
    int64_t lds;
    const int32_t *status;
};

__global__ void __launch_bounds__(256) k_trailing64(Trail64Args a) {
    if (a.status[2]) return;
    __shared__ __align__(16) double As[TK64][TB64];
    __shared__ __align__(16) double Bs[TK64][TB64];
    __shared__ int32_t rmap[TB64], cmap[TB64];
    const int64_t t = blockIdx.x;
    int64_t bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int64_t bj = t - bi * (bi + 1) / 2;
    const int64_t row0 = bi * TB64, col0 = bj * TB64;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;   // rows tx*4.., cols ty*4..
    if (tid < TB64) {
        rmap[tid] = (row0 + tid < a.mp) ? a.map[row0 + tid] : -1;
        cmap[tid] = (col0 + tid < a.mp) ? a.map[col0 + tid] : -1;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int32_t rm = rmap[tx * 4 + i], cm = cmap[ty * 4 + j];
            acc[i][j] = (cm >= 0 && rm >= cm) ? a.Vold[(int64_t)rm + (int64_t)cm * a.ldv] : 0.0;
        }
    const int lr = tid & 63, lk = tid >> 6;   // 4 k-rows per pass
    const int32_t arow = rmap[lr], bcol = cmap[lr];
    for (int t0 = 0; t0 < a.nbp; t0 += TK64) {
        const int kmax = min(TK64, a.nbp - t0);
#pragma unroll
        for (int q = 0; q < TK64 / 4; ++q) {
            const int kk = lk + 4 * q, tt = t0 + kk;
            As[kk][lr] = (kk < kmax && arow >= 0) ? a.Sn[arow + (int64_t)tt * a.lds] : 0.0;
            Bs[kk][lr] = (kk < kmax && bcol >= 0) ? a.S[bcol + (int64_t)tt * a.lds] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kmax; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][tx * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][ty * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t r = row0 + tx * 4 + i, c = col0 + ty * 4 + j;
            if (r < a.mp && c < a.mp && r >= c) a.Vnew[r + c * a.ldv] = acc[i][j];
        }
}

__global__ void k_gather_L64(int64_t N, const int32_t *__restrict__ pivorig, const double *__restrict__ Lorig,
                             int64_t ldl, double *__restrict__ Lfac, int64_t ldf) {
    for (int64_t k = blockIdx.x; k < N; k += gridDim.x) {
        const double *src = Lorig + k * ldl;
        double *dst = Lfac + k * ldf;
        for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
            double v = 0.0;
            if (r == k) v = 1.0;
            else if (r > k) v = src[pivorig[r]];
            dst[r] = v;
        }
    }
}

}  // namespace

// FP64 stage 1 (prec = 64): same outputs as lowprec_factor in lf->Lfac64 / D64
// (h_D holds the FP32-rounded pivots only for reporting d_ref; h_D64 is exact).
void lowprec_factor64(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                      hf_lowfactor *lf) {
    cudaStream_t st = ctx->stream;
    const int nsm = ctx->num_sms;
    lf->L = L;
    lf->stream = st;
    lf->prec = 64;
    if (L == 0) {
        lf->N = lf->Ntau = lf->n2 = 0;
        return;
    }
    HF_REQUIRE(L <= (int64_t)POS_MAX64 - 1, "L too large for the 17-bit position key");
    int maxsmem = 0;
    HF_CUDA(cudaDeviceGetAttribute(&maxsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    cudaFuncAttributes fa;
    HF_CUDA(cudaFuncGetAttributes(&fa, k_chain64<1024>));
    maxsmem -= (int)fa.sharedSizeBytes;
    const int nb_def = 64;
    const int gmax = (int)std::min<int64_t>(nsm, std::max<int64_t>(64, cdiv(L, (int64_t)(maxsmem / 8 / (nb_def + 2)))));
    const int64_t G0 = std::min<int64_t>(gmax, std::max<int64_t>(1, cdiv(L, 32)));
    const int64_t R0 = cdiv(L, G0);
    HF_REQUIRE(R0 <= 1024, "L too large for one chain CTA per SM (R > 1024)");
    int nb = o.nb > 0 ? std::min<int>(o.nb, 256) : nb_def;
    while (nb > 8 && (int64_t)(nb * R0 + 2 * nb) * 8 > (int64_t)maxsmem) nb /= 2;

    DBuf<double> V[2], S, Sn, Lorig, Dk;
    V[0].alloc((size_t)L * L, st);
    V[1].alloc((size_t)L * L, st);
    S.alloc((size_t)L * nb, st);
    Sn.alloc((size_t)L * nb, st);
    Lorig.alloc((size_t)L * L, st);
    Dk.alloc(L, st);
    DBuf<int32_t> orig[2], map, pivpos, pivorig, status;
    orig[0].alloc(L, st);
    orig[1].alloc(L, st);
    map.alloc(L, st);
    pivpos.alloc(nb, st);
    pivorig.alloc(L, st);
    status.alloc(4, st);
    DBuf<unsigned long long> slots, mbox;
    slots.alloc((size_t)2 * nsm * SLOT_WORDS, st);
    slots.zero(st);
    mbox.alloc((size_t)2 * nsm * 2 * nb, st);
    mbox.zero(st);
    HF_CUDA(cudaMemsetAsync(status.p, 0, 4 * sizeof(int32_t), st));
    {
        ClassTimer tm(ctx, "other");
        k_copy_lower64<<<(unsigned)std::min<int64_t>(L, 65535), 256, 0, st>>>(L, K, ld, V[0].p, L);
        HF_CHECK_LAUNCH(ctx);
        k_iota32_64<<<(unsigned)cdiv(L, 256), 256, 0, st>>>(L, orig[0].p);
        HF_CHECK_LAUNCH(ctx);
    }
    HF_CUDA(cudaFuncSetAttribute(k_chain64<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_chain64<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    HF_CUDA(cudaFuncSetAttribute(k_chain64<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem));
    int cur = 0;
    int64_t m = L, K0 = 0;
    while (m > 0) {
        const int nbp = (int)std::min<int64_t>(nb, m);
        const int64_t G = std::min<int64_t>(gmax, std::max<int64_t>(1, cdiv(m, 32)));
        const int64_t R = cdiv(m, G);
        const int nthr = (int)std::max<int64_t>(64, cdiv(R, 32) * 32);
        const size_t shm = ((size_t)nbp * R + 2 * nbp) * sizeof(double);
        Chain64Args ca{m, K0, nbp, (int)R, o.tau, V[cur].p, L, orig[cur].p, S.p, Sn.p, L, pivpos.p,
                       Lorig.p, L, Dk.p, pivorig.p, slots.p, mbox.p, status.p};
        {
            ClassTimer tm(ctx, "chain");
            void *args[] = {&ca};
            const int lb = std::max(nthr, getenv("HF_CHAIN_LB") ? atoi(getenv("HF_CHAIN_LB")) : 0);
            void *kf = lb <= 256 ? (void *)k_chain64<256> : lb <= 512 ? (void *)k_chain64<512> : (void *)k_chain64<1024>;
            HF_CUDA(cudaLaunchCooperativeKernel(kf, dim3((unsigned)G), dim3(nthr), args, shm, st));
            HF_CHECK_LAUNCH(ctx);
        }
        const int64_t mp = m - nbp;
        if (mp > 0) {
            {
                ClassTimer tm(ctx, "other");
                k_compact64<<<(unsigned)std::min<int64_t>(cdiv(m, 256), 4096), 256, 0, st>>>(
                    m, nbp, pivpos.p, orig[cur].p, map.p, orig[cur ^ 1].p, status.p);
                HF_CHECK_LAUNCH(ctx);
            }
            Trail64Args ta{mp, nbp, V[cur].p, V[cur ^ 1].p, L, map.p, S.p, Sn.p, L, status.p};
            const int64_t T = cdiv(mp, TB64);
            ClassTimer tm(ctx, "trailing");
            k_trailing64<<<(unsigned)(T * (T + 1) / 2), 256, 0, st>>>(ta);
            HF_CHECK_LAUNCH(ctx);
            cur ^= 1;
        }
        K0 += nbp;
        m = mp;
    }
    int32_t hs[4];
    HF_CUDA(cudaMemcpyAsync(hs, status.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    const int64_t Ntau = hs[2] ? hs[0] : L;
    int64_t N = Ntau;   // [R5] floor, [R9] enlargement
    if (L - o.n_min < N) N = std::max<int64_t>(0, L - o.n_min);
    if (N < L) N = std::max<int64_t>(0, N - o.n_extra);
    lf->Ntau = Ntau;
    lf->N = N;
    lf->n2 = L - N;
    std::vector<int32_t> po(std::max<int64_t>(N, 1));
    if (N > 0) HF_CUDA(cudaMemcpyAsync(po.data(), pivorig.p, N * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    lf->h_D64.assign(std::max<int64_t>(N, 1), 0.0);
    if (N > 0) HF_CUDA(cudaMemcpyAsync(lf->h_D64.data(), Dk.p, N * sizeof(double), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    lf->h_D64.resize(N);
    lf->h_D.assign(N, 0.f);
    for (int64_t k = 0; k < N; ++k) lf->h_D[k] = (float)lf->h_D64[k];
    std::vector<int32_t> rank(L, -1);
    lf->h_perm.resize(L);
    for (int64_t k = 0; k < N; ++k) {
        lf->h_perm[k] = po[k];
        rank[po[k]] = (int32_t)k;
    }
    int64_t w = N;
    for (int64_t q = 0; q < L; ++q)
        if (rank[q] < 0) lf->h_perm[w++] = q;
    lf->perm.alloc(L, st);
    lf->pos1.alloc(L, st);
    HF_CUDA(cudaMemcpyAsync(lf->perm.p, lf->h_perm.data(), L * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    HF_CUDA(cudaMemcpyAsync(lf->pos1.p, rank.data(), L * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    lf->D64.alloc(std::max<int64_t>(N, 1), st);
    if (N > 0) HF_CUDA(cudaMemcpyAsync(lf->D64.p, Dk.p, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    V[0].release();
    V[1].release();
    lf->Lfac64.alloc((size_t)std::max<int64_t>(N, 1) * std::max<int64_t>(N, 1), st);
    if (N > 0) {
        ClassTimer tm(ctx, "other");
        k_gather_L64<<<(unsigned)std::min<int64_t>(N, 65535), 256, 0, st>>>(N, pivorig.p, Lorig.p, L, lf->Lfac64.p, N);
        HF_CHECK_LAUNCH(ctx);
    }
    HF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hf
