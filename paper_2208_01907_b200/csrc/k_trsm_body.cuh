// k_trsm_body.cuh -- the preconditioner solves of k_trsm.cu, written once for
// the element type T (included twice by k_trsm.cu: T = float, the paper's FP32
// preconditioner [R12]; T = double, the FP64 one of the (double, dd) pair).
// Everything here lives in a per-precision namespace of k_trsm.cu.
constexpr int EPC = 16 / (int)sizeof(T);   // elements per 16-byte cp.async chunk

// ------------------------------------------------------------------ setup kernels
// Lp (Np x Np, ld Np) = Lfac (N x N, ld N) padded with the identity; Up = Lp^T.
// 32x32 tiles through shared memory so both the read and the transposed write
// are coalesced.  Only the lower tiles of Lp (and so the upper tiles of Up) are
// written: nothing reads the other triangle (the diagonal-block inverses use the
// strictly lower entries, the solves the off-diagonal blocks below / above).
__global__ void __launch_bounds__(256) k_pad_transpose(int64_t N, int64_t Np, const T *__restrict__ Lf,
                                                       T *__restrict__ Lp, T *__restrict__ Up) {
    __shared__ T t[32][33];
    if (blockIdx.x < blockIdx.y) return;   // a tile strictly above the diagonal
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int q = ty; q < 32; q += 8) {
        const int64_t i = i0 + tx, j = j0 + q;
        T v;
        if (i < N && j < N) v = Lf[i + j * N];
        else v = (i == j) ? T(1) : T(0);
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
__global__ void __launch_bounds__(64) k_diag_inv(int64_t Np, const T *__restrict__ Lp, T *__restrict__ LinvF,
                                                 T *__restrict__ LinvB) {
    extern __shared__ __align__(16) unsigned char dsm_[];   // 2 x 64 x 65 elements (dynamic)
    T (*Ls)[TBS + 1] = reinterpret_cast<T (*)[TBS + 1]>(dsm_);
    T (*Xs)[TBS + 1] = Ls + TBS;
    const int64_t r0 = (int64_t)blockIdx.x * TBS;
    const int j = threadIdx.x;
    for (int i = 0; i < TBS; ++i) Ls[i][j] = Lp[(r0 + i) + (r0 + j) * Np];
    __syncthreads();
    // column j of the inverse: x_i = delta_ij - sum_{j<=k<i} L_ik x_k
    for (int i = 0; i < TBS; ++i) {
        T s = (i == j) ? T(1) : T(0);
        if (i > j)
            for (int k = j; k < i; ++k) s = fma_rn(-Ls[i][k], Xs[k][j], s);
        Xs[i][j] = (i < j) ? T(0) : s;
    }
    __syncthreads();
    T *F = LinvF + (size_t)blockIdx.x * TILE;
    T *B = LinvB + (size_t)blockIdx.x * TILE;
    for (int k = 0; k < TBS; ++k) {
        F[k * TBS + j] = Xs[j][k];
        B[k * TBS + j] = Xs[k][j];
    }
}

struct TrsmArgs {
    int64_t N, Np;
    int ncol, ncolp, nch, nblk, seg;
    const int4 *items;   // [nitems] (logical block j, chunk, q_lo | q_hi << 16, slot >= 0: PARTIAL | < 0: EARLY)
    const int4 *pinfo;   // [nblk] block j: (first slot, #bulk slots, #near slots, tail q_lo); base slot last
    int npw;             // P-worker CTAs per chunk (block j -> worker j % npw)
    int nitems;
    int h48;             // helper PARTIAL items in the 4 x 8 k-split form (FP32)
    T *part;         // partial sums [slot][chunk][64 x CW] (row-major)
    T *P;            // P_j, row-major Np x ncolp (by physical row)
    int *pflags;         // [2][nslots*nch]
    int *aflags;         // [2][nblk*nch]   P_j ready
    int nslots;
    const T *Lp;     // forward operand  (Np x Np, col-major)
    const T *Up;     // backward operand (Np x Np, col-major) = Lp^T
    const T *LinvF;  // [nblk][64][64] tile layout of Dinv (forward)
    const T *LinvB;  // (backward)
    const T *D;      // [N]
    const int64_t *perm; // [L] pivot order -> original index
    const double *R;     // input, original row order (L x ncol, ldr)
    int64_t ldr;
    T *Y;            // forward result, row-major Np x ncolp
    T *Xb;           // backward result, row-major Np x ncolp
    int *flags;          // [2][nblk*nch]   chain released Y_j
    int *counter;        // [2]
    unsigned *smids;     // [2 dir][owner | role + 2][TRSM_MAXSM] role assignment by SM
    int epoch;
    unsigned long long *dbg;   // optional chain phase timers (HF_TRSM_DEBUG)
};


// acc[i][j] (+|-)= sum_k As[k][tr*4+i] * Bs[k][tc*4+j]; FP32: FFMA2 with a broadcast
// scalar (half the issue slots of scalar FFMA), the pairs along j kept in float2
template <bool NEG>
__device__ __forceinline__ void tile_prod(T (&acc)[4][4], const T *As, const T *Bs, int tr, int tc, int k0 = 0,
                                          int k1 = TBS) {
    if constexpr (sizeof(T) == 4) {
        float2 c2[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            c2[i][0] = make_float2(acc[i][0], acc[i][1]);
            c2[i][1] = make_float2(acc[i][2], acc[i][3]);
        }
        // software pipelined: the fragments of the next 4 k are loaded while the current 4
        // are used (the chain CTA runs this with only 2 warps per SM sub-partition)
        V4<T> fa[2][4], fy[2][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            fa[0][u] = ld4(&As[(k0 + u) * TBS + tr * 4]);
            fy[0][u] = ld4(&Bs[(k0 + u) * CW + tc * 4]);
        }
#pragma unroll
        for (int kb = 0; kb < TBS; kb += 4) {
            const int cur = (kb >> 2) & 1;
            if (k0 + kb >= k1) break;
            if (k0 + kb + 4 < k1) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    fa[cur ^ 1][u] = ld4(&As[(k0 + kb + 4 + u) * TBS + tr * 4]);
                    fy[cur ^ 1][u] = ld4(&Bs[(k0 + kb + 4 + u) * CW + tc * 4]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const V4<T> a = fa[cur][u], y = fy[cur][u];
                const T av[4] = {NEG ? -a.x : a.x, NEG ? -a.y : a.y, NEG ? -a.z : a.z, NEG ? -a.w : a.w};
                const float2 y01 = make_float2(y.x, y.y), y23 = make_float2(y.z, y.w);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    c2[i][0] = __ffma2_rn(make_float2(av[i], av[i]), y01, c2[i][0]);
                    c2[i][1] = __ffma2_rn(make_float2(av[i], av[i]), y23, c2[i][1]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc[i][0] = c2[i][0].x;
            acc[i][1] = c2[i][0].y;
            acc[i][2] = c2[i][1].x;
            acc[i][3] = c2[i][1].y;
        }
    } else {
#pragma unroll 8
        for (int k = k0; k < k1; ++k) {
            const V4<T> a = ld4(&As[k * TBS + tr * 4]);
            const V4<T> y = ld4(&Bs[k * CW + tc * 4]);
            const T av[4] = {NEG ? -a.x : a.x, NEG ? -a.y : a.y, NEG ? -a.z : a.z, NEG ? -a.w : a.w};
            const T yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma_rn(av[i], yv[j], acc[i][j]);
        }
    }
}
__device__ __forceinline__ void tile_fma(T (&acc)[4][4], const T *As, const T *Bs, int tr, int tc, int k0 = 0,
                                         int k1 = TBS) {
    tile_prod<false>(acc, As, Bs, tr, tc, k0, k1);
}
__device__ __forceinline__ void tile_fms(T (&acc)[4][4], const T *As, const T *Bs, int tr, int tc, int k0 = 0,
                                         int k1 = TBS) {
    tile_prod<true>(acc, As, Bs, tr, tc, k0, k1);
}

// Helper PARTIAL items (FP32): a 4 x 8 output block per thread over HALF the k range of
// each tile (two k groups of 128 threads, reduced once per item), so a k step costs three
// shared loads for 16 FFMA2 instead of two for 8.  A warp covers 8 row groups x 4 column
// groups: one 128-B wavefront per operand load.
__device__ __forceinline__ void tile_prod48(float2 (&c2)[4][4], const float *As, const float *Bs, int r4, int c8,
                                            int k0) {
#pragma unroll 8
    for (int k = k0; k < k0 + TBS / 2; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(&As[k * TBS + r4]);
        const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[k * CW + c8]);
        const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[k * CW + c8 + 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float2 y[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                             make_float2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) c2[i][jp] = __ffma2_rn(make_float2(av[i], av[i]), y[jp], c2[i][jp]);
    }
}

// ------------------------------------------------------------------ setup: G = Dinv Op
// In place, one 64x64 tile per CTA: Op(b-block, q-block) <- Dinv_b Op(b, q) for
// every dependency block q of b (forward: q < b on Lp; backward: q > b on Up).
// The tile is read coalesced (column-major) and transposed through shared
// memory into the [k][c] operand layout.
template <bool BWD>
__global__ void __launch_bounds__(256) k_scale_op(int nblk, int64_t Np, T *__restrict__ Op,
                                                  const T *__restrict__ Linv) {
    const int b = blockIdx.x, q = blockIdx.y;
    if (BWD ? !(q > b) : !(q < b)) return;
    extern __shared__ __align__(16) unsigned char dsm_[];   // Ts[c][k] (padded) / Dinv tile, then Bs
    T *buf = reinterpret_cast<T *>(dsm_);
    T *Bs = buf + TBS * (TBS + 1) + 4;
    T *As = buf;
    const int tid = threadIdx.x, tr = tid & 15, tc = tid >> 4;
    const int64_t r0 = (int64_t)b * TBS, q0 = (int64_t)q * TBS;
    for (int e = tid; e < TILE; e += 256) {
        const int r = e & 63, c = e >> 6;
        buf[c * (TBS + 1) + r] = Op[(r0 + r) + (q0 + c) * Np];      // Ts[c][k] = Op(r0+k, q0+c)
    }
    __syncthreads();
    for (int e = tid; e < TILE; e += 256) {
        const int k = e >> 6, c = e & 63;
        Bs[k * CW + c] = buf[c * (TBS + 1) + k];
    }
    __syncthreads();
    for (int e = tid; e < TILE; e += 256) As[e] = Linv[(size_t)b * TILE + e];
    __syncthreads();
    T acc[4][4] = {};
    tile_fma(acc, As, Bs, tr, tc);                     // Dinv_b Op_bq
    // column jj of the thread's 4x4 block: 4 consecutive rows -> one 16-byte (FP32) store
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
        st4(&Op[(r0 + tr * 4) + (q0 + tc * 4 + jj) * Np], acc[0][jj], acc[1][jj], acc[2][jj], acc[3][jj]);
}

// W (original row order, ldw) = lift(Xb) on Lambda_1 rows, 0 on Lambda_2 rows
__global__ void k_lift_scatter(int64_t L, int ncol, int ncolp, const int32_t *__restrict__ pos1,
                               const T *__restrict__ Xb, double *__restrict__ W, int64_t ldw) {
    for (int c = blockIdx.y; c < ncol; c += gridDim.y)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (int64_t)gridDim.x * blockDim.x) {
            const int32_t r = pos1[i];
            W[i + (int64_t)c * ldw] = r >= 0 ? (double)Xb[(int64_t)r * ncolp + c] : 0.0;
        }
}

constexpr int NTHR = 320;                 // 8 compute warps + 2 store warps (chain); helpers use 256
constexpr int NCOMP = 256;
constexpr int TRSM_MAXSM = 256;           // SM id table size of the role assignment
constexpr int SMEM_ELEMS = 7 * TILE;     // 112 KB: chain = Yring[3] + M[2 stages][2]; helper = 3 x (A + B)

template <bool BWD>
__global__ void __launch_bounds__(NTHR, 2) k_trsm(TrsmArgs a) {
    extern __shared__ __align__(16) T sm[];
    __shared__ int item_s;
    // thread -> 4x4 output block: a warp covers 8 row groups x 4 column groups, so each
    // k step's operand loads are one 128-B A wavefront and one 64-B B wavefront
    const int tid = threadIdx.x, tr = (tid & 7) | (((tid >> 5) & 1) << 3), tc = ((tid >> 3) & 3) | (((tid >> 6) & 3) << 2);
    int *flags = a.flags + (BWD ? a.nblk * a.nch : 0);
    int *pflags = a.pflags + (BWD ? a.nslots * a.nch : 0);
    int *aflags = a.aflags + (BWD ? a.nblk * a.nch : 0);
    int *counter = a.counter + (BWD ? 1 : 0);
    // role by SM: the first CTA to arrive on an SM claims it and takes the next role
    // ticket (chain chunks, then P-workers); a CTA that finds its SM owned by a role
    // leaves, so chain CTAs and P-workers each have an SM to themselves
    unsigned *smrole = a.smids + (BWD ? 2 * TRSM_MAXSM : 0);   // [owner | role + 2] per SM
    int *role_ctr = a.counter + 2 + (BWD ? 1 : 0);
    const int nroles = a.nch * (1 + a.npw);
    __shared__ int role_s;
    if (tid == 0) {
        const unsigned me = smid() % TRSM_MAXSM;
        int role = -1;   // -1: helper, -2: leave
        if (atomicCAS(&smrole[me], 0u, 1u) == 0u) {
            const int r = atomicAdd(role_ctr, 1);
            role = r < nroles ? r : -1;
            atomicExch(&smrole[TRSM_MAXSM + me], (unsigned)(role + 2));
        } else {
            unsigned v;
            while ((v = *(volatile unsigned *)&smrole[TRSM_MAXSM + me]) == 0u) __nanosleep(32);
            role = v >= 2u ? -2 : -1;
        }
        role_s = role;
    }
    __syncthreads();
    const int role = role_s;
    if (role == -2) return;
    const T *Op = BWD ? a.Up : a.Lp;
    T *Yout = BWD ? a.Xb : a.Y;
    const T *Dinv = BWD ? a.LinvB : a.LinvF;
    auto phys = [&](int j) { return BWD ? (a.nblk - 1 - j) : j; };

    if (role >= 0 && role < a.nch) {
        // =================================================== CHAIN (chunk cc)
        const int cc = role, c0 = cc * CW;
        T *Yr = sm;               // [3][TILE] ring: Y_j in slot j % 3
        T *Mb = sm + 3 * TILE;    // [2 stages][G_{j,j-1}, G_{j,j-2}]
        if (tid >= NCOMP) {
            // ---- store warps: slot j -> global, fence, release
            const int st = tid - NCOMP;
            for (int j = 0; j < a.nblk; ++j) {
                bar_sync(1 + j % 3, NTHR);                // FULL(slot j % 3)
                const T *ys = Yr + (j % 3) * TILE;
                const int64_t r0 = (int64_t)phys(j) * TBS;
#pragma unroll 4
                for (int u = 0; u < 16; ++u) {
                    const int e = st + u * 64;            // 1024 float4 = 64 rows x 16
                    const int r = e >> 4, c4 = (e & 15) * 4;
                    st4v(&Yout[(r0 + r) * a.ncolp + c0 + c4], ld4(&ys[r * CW + c4]));
                }
                bar_sync(9, NTHR - NCOMP);
                if (st == 0) {
                    __threadfence();
                    st_release32(&flags[j * a.nch + cc], a.epoch);
                }
                bar_arrive(6 + j % 3, NTHR);              // EMPTY(slot j % 3): may be reused
            }
            return;
        }
        // ---- compute warps
        // G_{j,j-1}, G_{j,j-2} tiles of the scaled operator, layout [k][r] = G(r0+r, q0+k)
        auto load_m = [&](int j) {
            T *dst = Mb + (j & 1) * 2 * TILE;
            const int64_t r0 = (int64_t)phys(j) * TBS;
#pragma unroll
            for (int lag = 1; lag <= 2; ++lag) {
                if (j - lag < 0) continue;
                const int64_t q0 = (int64_t)phys(j - lag) * TBS;
                T *d = dst + (lag - 1) * TILE;
#pragma unroll
                for (int u = 0; u < TILE / EPC / NCOMP; ++u) {
                    const int e = (tid + u * NCOMP) * EPC;
                    const int k = e >> 6, r4 = e & 63;
                    cp_async16(&d[k * TBS + r4], Op + (r0 + r4) + (q0 + k) * a.Np);
                }
            }
            cp_commit();
        };
        load_m(0);
        const bool dbg = a.dbg && cc == 0 && tid == 0;
        unsigned long long ph[4] = {0, 0, 0, 0}, tp = dbg ? gtimer() : 0;
#define PH(q) if (dbg) { unsigned long long n_ = gtimer(); ph[q] += n_ - tp; tp = n_; }
        for (int j = 0; j < a.nblk; ++j) {
            if (j + 1 < a.nblk) load_m(j + 1);
            const int64_t r0 = (int64_t)phys(j) * TBS;
            if (tid == 0) wait_epoch(&aflags[j * a.nch + cc], a.epoch);
            bar_sync(4, NCOMP);
            PH(0)
            T acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const V4<T> v = ld4(&a.P[(r0 + tr * 4 + i) * a.ncolp + c0 + tc * 4]);
                acc[i][0] = v.x; acc[i][1] = v.y; acc[i][2] = v.z; acc[i][3] = v.w;
            }
            if (j + 1 < a.nblk) cp_wait_1(); else cp_wait_all();
            bar_sync(4, NCOMP);
            PH(1)
            const T *M = Mb + (j & 1) * 2 * TILE;
            if (j >= 1) tile_fms(acc, M, Yr + ((j - 1) % 3) * TILE, tr, tc);
            if (j >= 2) tile_fms(acc, M + TILE, Yr + ((j - 2) % 3) * TILE, tr, tc);
            PH(2)
            if (j >= 3) bar_sync(6 + j % 3, NTHR);       // EMPTY: store warps are done with Y_{j-3}
            T *ys = Yr + (j % 3) * TILE;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                st4(&ys[(tr * 4 + i) * CW + tc * 4], acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            bar_sync(4, NCOMP);                           // slot complete for the compute warps ...
            bar_arrive(1 + j % 3, NTHR);                  // ... FULL: handed to the store warps
            PH(3)
        }
        for (int j = (a.nblk > 3 ? a.nblk - 3 : 0); j < a.nblk; ++j) bar_sync(6 + j % 3, NTHR);   // drain
        if (dbg)
            for (int q = 0; q < 4; ++q) atomicAdd(&a.dbg[(BWD ? 4 : 0) + q], ph[q]);
#undef PH
        return;
    }

    // ============================================ P-WORKERS and HELPERS (NCOMP threads)
    if (tid >= NCOMP) return;
    const bool worker = role >= a.nch;
    const T *src = Yout;
    auto load_dep = [&](int s, int64_t r0, int64_t q0, int c0) {
        T *As = sm + s * 2 * TILE;
        T *Bs = As + TILE;
#pragma unroll
        for (int u = 0; u < TILE / EPC / NCOMP; ++u) {
            const int e = (tid + u * NCOMP) * EPC;   // 16-byte chunks of the tile
            const int k = e >> 6, r4 = e & 63;
            cp_async16(&As[k * TBS + r4], Op + (r0 + r4) + (q0 + k) * a.Np);
            cp_async16(&Bs[k * CW + r4], src + (q0 + k) * a.ncolp + c0 + r4);
        }
    };
    // t += sum over logical dependency blocks [q_lo, q_hi) of Op_bq Y_q, three stages of
    // cp.async in flight.  Released flags are checked eight at a time (independent loads,
    // one round trip), so old dependencies cost no poll each.
    __shared__ int rdy_s;
    // h2 != null (helpers, FP32): the 4 x 8 k-split form of tile_prod48 into h2 instead of t
    const int kg = tid >> 7, t7 = tid & 127;
    const int r4h = ((t7 & 7) | (((t7 >> 5) & 1) << 3)) * 4, c8h = (((t7 >> 3) & 3) | ((t7 >> 6) << 2)) * 8;
    auto accumulate = [&](T (&t)[4][4], int64_t r0, int c0, int cc, int q_lo, int q_hi, float2 (*h2)[4] = nullptr) {
        const int ndep = q_hi - q_lo;
        if (ndep <= 0) return;
        int ready = 0;   // blocks [q_lo, q_lo + ready) known released (uniform)
        auto ensure = [&](int dq) {
            if (dq < ready) return;
            if (tid < 32) {   // warp 0: up to 32 flags in one round trip, ready prefix by ballot
                const int *f = flags + (size_t)(q_lo + dq) * a.nch + cc;
                const int nchk = min(32, ndep - dq);
                const bool ok = tid < nchk && ld_relaxed32(f + (size_t)tid * a.nch) == a.epoch;
                const unsigned bad = ~__ballot_sync(0xffffffffu, ok);
                int n = __ffs(bad) - 1;   // bad != 0: lane nchk.. are never ok
                if (n > nchk) n = nchk;
                if (n == 0) {
                    if (tid == 0)
                        while (ld_relaxed32(f) != a.epoch) __nanosleep(20);
                    n = 1;
                }
                if (tid == 0) {
                    fence_acquire();
                    rdy_s = dq + n;
                }
            }
            bar_sync(5, NCOMP);
            ready = rdy_s;
        };
        ensure(0);
        load_dep(0, r0, (int64_t)phys(q_lo) * TBS, c0);
        cp_commit();
        if (ndep > 1) {
            ensure(1);
            load_dep(1, r0, (int64_t)phys(q_lo + 1) * TBS, c0);
            cp_commit();
        }
        // one barrier per tile: it publishes stage dq and frees stage (dq + 2) % 3 (read in
        // the previous iteration), which is refilled right after it
        for (int dq = 0; dq < ndep; ++dq) {
            if (dq + 1 < ndep) cp_wait_1();
            else cp_wait_all();
            bar_sync(5, NCOMP);
            if (dq + 2 < ndep) {
                ensure(dq + 2);
                load_dep((dq + 2) % 3, r0, (int64_t)phys(q_lo + dq + 2) * TBS, c0);
                cp_commit();
            }
            const T *As = sm + (dq % 3) * 2 * TILE;
            if constexpr (sizeof(T) == 4) {
                if (h2) tile_prod48(*reinterpret_cast<float2 (*)[4][4]>(h2), reinterpret_cast<const float *>(As),
                                    reinterpret_cast<const float *>(As + TILE), r4h, c8h, kg * (TBS / 2));
                else tile_fma(t, As, As + TILE, tr, tc);
            } else {
                tile_fma(t, As, As + TILE, tr, tc);
            }
        }
        bar_sync(5, NCOMP);   // the stage buffers are free for the caller
    };
    // out = Dinv_j RHS_j (no dependency): forward truncates R (FP64, original order)
    // to FP32, backward starts from z = D^{-1} y
    auto dinv_rhs = [&](T (&out)[4][4], int b, int64_t r0, int c0) {
        T rhs[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t r = r0 + tr * 4 + i;
            if (!BWD) {
                const int64_t pr = r < a.N ? a.perm[r] : 0;
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int c = c0 + tc * 4 + jj;
                    rhs[i][jj] = (r < a.N && c < a.ncol) ? cvt_down(a.R[pr + (int64_t)c * a.ldr], T()) : T(0);
                }
            } else {
                const V4<T> y = ld4(&a.Y[r * a.ncolp + c0 + tc * 4]);
                const T d = r < a.N ? a.D[r] : T(1);
                rhs[i][0] = div_rn(y.x, d);
                rhs[i][1] = div_rn(y.y, d);
                rhs[i][2] = div_rn(y.z, d);
                rhs[i][3] = div_rn(y.w, d);
            }
        }
        T *As = sm, *Bs = sm + TILE;
        const T *Li = Dinv + (size_t)b * TILE;
#pragma unroll
        for (int u = 0; u < TILE / EPC / NCOMP; ++u) {
            const int e = (tid + u * NCOMP) * EPC;
            cp_async16(&As[e], Li + e);
        }
        cp_commit();
#pragma unroll
        for (int i = 0; i < 4; ++i)
            st4(&Bs[(tr * 4 + i) * CW + tc * 4], rhs[i][0], rhs[i][1], rhs[i][2], rhs[i][3]);
        cp_wait_all();
        bar_sync(5, NCOMP);
        tile_fma(out, As, Bs, tr, tc);
        bar_sync(5, NCOMP);   // the stage-0 buffers are reused by accumulate()
    };
    // acc += slots [s_lo, s_hi) of chunk cc in increasing order, in batches: tid 0 waits
    // for the next slot and takes every consecutive slot already released with it, then
    // all threads stream the batch (two slots' loads in flight)
    auto sum_slots = [&](T (&acc)[4][4], int cc, int s_lo, int s_hi) {
        for (int s2 = s_lo; s2 < s_hi;) {
            if (tid == 0) {
                const int *pf = pflags + cc;
                if (ld_relaxed32(pf + (size_t)s2 * a.nch) != a.epoch)
                    while (ld_relaxed32(pf + (size_t)s2 * a.nch) != a.epoch) __nanosleep(20);
                int e = s2 + 1;
                while (e < s_hi && ld_relaxed32(pf + (size_t)e * a.nch) == a.epoch) ++e;
                fence_acquire();
                item_s = e;
            }
            bar_sync(5, NCOMP);
            const int e = item_s;
            bar_sync(5, NCOMP);   // item_s is rewritten by the next batch / item fetch
            const T *pp = a.part + ((size_t)s2 * a.nch + cc) * (TBS * CW) + (tr * 4) * CW + tc * 4;
            const size_t sstride = (size_t)a.nch * TBS * CW;
            V4<T> cur[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) cur[i] = ld4(pp + i * CW);
            for (int q = s2; q < e; ++q) {
                V4<T> nxt[4];
                if (q + 1 < e) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) nxt[i] = ld4(pp + (size_t)(q + 1 - s2) * sstride + i * CW);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[i][0] += cur[i].x;
                    acc[i][1] += cur[i].y;
                    acc[i][2] += cur[i].z;
                    acc[i][3] += cur[i].w;
                }
                if (q + 1 < e) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) cur[i] = nxt[i];
                }
            }
            s2 = e;
        }
    };
    auto store_slot = [&](const T (&v)[4][4], int cc, int sl) {
        T *pp = a.part + ((size_t)sl * a.nch + cc) * (TBS * CW);
#pragma unroll
        for (int i = 0; i < 4; ++i) st4(&pp[(tr * 4 + i) * CW + tc * 4], v[i][0], v[i][1], v[i][2], v[i][3]);
        bar_sync(5, NCOMP);
        if (tid == 0) {
            __threadfence();
            st_release32(&pflags[sl * a.nch + cc], a.epoch);
        }
    };

    if (worker) {
        // ------------------------------------------------ P-WORKER (chunk cc, blocks j = w mod npw)
        // P_j = base_j - (near slots, in order) - tail [tail_lo, j-2), alone on its SM so the
        // few short sums between Y_{j-3} and P_j run at full speed (base_j = Dinv_j RHS_j -
        // bulk slots comes from an EARLY item of the helpers).
        const int wi = role - a.nch, cc = wi / a.npw, w = wi % a.npw;
        const int c0 = cc * CW;
        const bool wdbg = a.dbg && tid == 0 && cc == 0;
        unsigned long long wph[4] = {0, 0, 0, 0}, wtp = wdbg ? gtimer() : 0;
#define WPH(q) if (wdbg) { unsigned long long n_ = gtimer(); wph[q] += n_ - wtp; wtp = n_; }
        for (int j = w; j < a.nblk; j += a.npw) {
            const int4 pi = a.pinfo[j];   // (first slot, #bulk, #near, tail_lo)
            const int64_t r0 = (int64_t)phys(j) * TBS;
            const int sbase = pi.x + pi.y + pi.z;
            T base[4][4] = {}, t[4][4] = {};
            WPH(3)
            sum_slots(base, cc, sbase, sbase + 1);
            WPH(0)
            sum_slots(t, cc, pi.x + pi.y, sbase);
            WPH(1)
            accumulate(t, r0, c0, cc, pi.w, j > 2 ? j - 2 : 0);
            WPH(2)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                st4(&a.P[(r0 + tr * 4 + i) * a.ncolp + c0 + tc * 4], base[i][0] - t[i][0], base[i][1] - t[i][1],
                    base[i][2] - t[i][2], base[i][3] - t[i][3]);
            bar_sync(5, NCOMP);
            if (tid == 0) {
                __threadfence();
                st_release32(&aflags[j * a.nch + cc], a.epoch);
            }
        }
        if (wdbg)
            for (int q = 0; q < 4; ++q) atomicAdd(&a.dbg[8 + (BWD ? 4 : 0) + q], wph[q]);
#undef WPH
        return;
    }

    // ------------------------------------------- HELPERS: PARTIAL and EARLY items in table order
    for (;;) {
        if (tid == 0) item_s = atomicAdd(counter, 1);
        bar_sync(5, NCOMP);
        const int idx = item_s;
        bar_sync(5, NCOMP);   // item_s is reused by sum_slots
        if (idx >= a.nitems) return;
        const int4 it = a.items[idx];
        const int j = it.x, cc = it.y, slot = it.w;
        const int b = phys(j);
        const int64_t r0 = (int64_t)b * TBS;
        const int c0 = cc * CW;
        T t[4][4] = {};
        if (slot >= 0) {
            // PARTIAL: t = sum over the segment [q_lo, q_hi) of Op_bq Y_q -> slot
            if constexpr (sizeof(T) == 4) {
                if (!a.h48) {
                    accumulate(t, r0, c0, cc, it.z & 0xFFFF, it.z >> 16);
                    store_slot(t, cc, slot);
                    continue;
                }
                float2 h2[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp) h2[i][jp] = make_float2(0.f, 0.f);
                accumulate(t, r0, c0, cc, it.z & 0xFFFF, it.z >> 16, h2);
                // k group 1 -> shared (stage buffers are free after the last barrier), group 0 adds
                // and stores the slot in its [64][CW] layout
                T *red = sm;
                if (kg == 1) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        st4(&red[(r4h + i) * CW + c8h], T(h2[i][0].x), T(h2[i][0].y), T(h2[i][1].x), T(h2[i][1].y));
                        st4(&red[(r4h + i) * CW + c8h + 4], T(h2[i][2].x), T(h2[i][2].y), T(h2[i][3].x), T(h2[i][3].y));
                    }
                }
                bar_sync(5, NCOMP);
                if (kg == 0) {
                    T *pp = a.part + ((size_t)slot * a.nch + cc) * (TBS * CW);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const V4<T> u0 = ld4(&red[(r4h + i) * CW + c8h]), u1 = ld4(&red[(r4h + i) * CW + c8h + 4]);
                        st4(&pp[(r4h + i) * CW + c8h], T(h2[i][0].x) + u0.x, T(h2[i][0].y) + u0.y,
                            T(h2[i][1].x) + u0.z, T(h2[i][1].y) + u0.w);
                        st4(&pp[(r4h + i) * CW + c8h + 4], T(h2[i][2].x) + u1.x, T(h2[i][2].y) + u1.y,
                            T(h2[i][3].x) + u1.z, T(h2[i][3].y) + u1.w);
                    }
                }
                bar_sync(5, NCOMP);
                if (tid == 0) {
                    __threadfence();
                    st_release32(&pflags[slot * a.nch + cc], a.epoch);
                }
            } else {
                accumulate(t, r0, c0, cc, it.z & 0xFFFF, it.z >> 16);
                store_slot(t, cc, slot);
            }
        } else {
            // EARLY: base_j = Dinv_j RHS_j - (bulk slots, in order) -> the base slot
            const int4 pi = a.pinfo[j];
            T out[4][4] = {};
            dinv_rhs(out, b, r0, c0);
            sum_slots(t, cc, pi.x, pi.x + pi.y);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) out[i][jj] -= t[i][jj];
            store_slot(out, cc, pi.x + pi.y + pi.z);
        }
    }
}

// ------------------------------------------------------------------ host side
// Ufac != null (NEXT-3, nonsymmetric LDU): the backward operator is U = Ufac^T
// instead of L^T, and its diagonal-block inverses come from Ufac.
void precond_setup_t(hf_ctx *ctx, PrecondT<T> &p, int64_t N, int64_t L, const T *Lfac, const T *D,
                   const int64_t *perm, const int32_t *pos1, const T *Ufac = nullptr) {
    p.N = N;
    p.L = L;
    p.Lfac = Lfac;
    p.D = D;
    p.perm = perm;
    p.pos1 = pos1;
    if (N == 0) return;
    cudaStream_t st = ctx->stream;
    const int64_t nblk = cdiv(N, TBS);
    p.Np = nblk * TBS;
    p.Lp.alloc((size_t)p.Np * p.Np, st);
    p.Up.alloc((size_t)p.Np * p.Np, st);
    p.LinvF.alloc((size_t)nblk * TILE, st);
    p.LinvB.alloc((size_t)nblk * TILE, st);
    ClassTimer tm(ctx, "trsm_setup");
    dim3 g((unsigned)(p.Np / 32), (unsigned)(p.Np / 32));
    DBuf<T> Ulp, Ltr, scr;   // nonsymmetric only: Ufac padded, a discarded transpose / inverse
    if (!Ufac) {
        k_pad_transpose<<<g, 256, 0, st>>>(N, p.Np, Lfac, p.Lp.p, p.Up.p);
        HF_CHECK_LAUNCH(ctx);
    } else {
        Ulp.alloc((size_t)p.Np * p.Np, st);
        Ltr.alloc((size_t)p.Np * p.Np, st);
        k_pad_transpose<<<g, 256, 0, st>>>(N, p.Np, Lfac, p.Lp.p, Ltr.p);
        HF_CHECK_LAUNCH(ctx);
        k_pad_transpose<<<g, 256, 0, st>>>(N, p.Np, Ufac, Ulp.p, p.Up.p);   // Up = Ufac^T = U
        HF_CHECK_LAUNCH(ctx);
        Ltr.release();
    }
    const size_t sm_inv = (size_t)2 * TBS * (TBS + 1) * sizeof(T);
    const size_t sm_sc = ((size_t)TBS * (TBS + 1) + 4 + TILE) * sizeof(T);
    static DevState attr_setup_dev(0);
    int &attr_setup = attr_setup_dev[ctx->device];
    if (!attr_setup) {
        HF_CUDA(cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_inv));
        HF_CUDA(cudaFuncSetAttribute(k_scale_op<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc));
        HF_CUDA(cudaFuncSetAttribute(k_scale_op<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc));
        attr_setup = 1;
    }
    if (!Ufac) {
        k_diag_inv<<<(unsigned)nblk, TBS, sm_inv, st>>>(p.Np, p.Lp.p, p.LinvF.p, p.LinvB.p);
        HF_CHECK_LAUNCH(ctx);
    } else {
        scr.alloc((size_t)nblk * TILE, st);
        k_diag_inv<<<(unsigned)nblk, TBS, sm_inv, st>>>(p.Np, p.Lp.p, p.LinvF.p, scr.p);
        HF_CHECK_LAUNCH(ctx);
        k_diag_inv<<<(unsigned)nblk, TBS, sm_inv, st>>>(p.Np, Ulp.p, scr.p, p.LinvB.p);   // (U_bb)^{-1}
        HF_CHECK_LAUNCH(ctx);
    }
    // G = Dinv Op in place (after the diagonal inverses, which read the diagonal blocks only)
    dim3 gs((unsigned)nblk, (unsigned)nblk);
    k_scale_op<false><<<gs, 256, sm_sc, st>>>((int)nblk, p.Np, p.Lp.p, p.LinvF.p);
    HF_CHECK_LAUNCH(ctx);
    k_scale_op<true><<<gs, 256, sm_sc, st>>>((int)nblk, p.Np, p.Up.p, p.LinvB.p);
    HF_CHECK_LAUNCH(ctx);
}

// Work decomposition of P_j = Dinv_j RHS_j - sum_{q < j-2} G_jq Y_q (logical
// blocks j: forward j = b, backward j = nblk-1-b).  The dependency range is cut
// into segments whose sizes grow GEOMETRICALLY away from the diagonal: a TAIL
// that the P-worker sums itself once Y_{j-3} is out, NEAR partial segments of
// 1, 2, 4, ... < SEG blocks and BULK partial segments of SEG blocks back to
// q = 0.  A segment ending at q_hi can run once Y_{q_hi-1} is out; the sizes
// keep every near segment's work below the chain time left until P_j is
// needed.  The helpers' table holds, in topological order, PARTIAL items
// (placed at chain stage max(q_hi - 1, j - 3 - LA), LA = lookahead, so bulk
// work is queued just ahead of the chain instead of in front of it) and one
// EARLY item per block and chunk, base_j = Dinv_j RHS_j - (bulk slots), placed
// ELAG stages after its last bulk segment's gate (at most j - 3).  The
// P-worker of (j, chunk) computes P_j = base_j - (near slots) - tail.  Every
// table item depends only on earlier items and on chain stages <= its own,
// and a P-worker only on items and chain stages before its block, so the
// persistent CTAs cannot deadlock.  Slot layout of block j: [bulk..., near...,
// base]; slots are summed in increasing q order (deterministic).
static void build_items(int nblk, int nch, int seg, std::vector<int4> &items, std::vector<int4> &pinfo, int &nslots) {
    int LA = 24;   // HF_TRSM_LA: tuning
    if (const char *e = getenv("HF_TRSM_LA")) LA = std::max(0, atoi(e));
    int TAIL = 1;  // HF_TRSM_TAIL: tuning (1 / 2 / 4: 7.06 / 7.17 / 7.72 ms per C2 apply)
    if (const char *e = getenv("HF_TRSM_TAIL")) TAIL = std::max(1, atoi(e));
    int ELAG = 8;  // HF_TRSM_ELAG: stages between the last bulk segment's gate and its EARLY item
    const bool GEO = !(getenv("HF_TRSM_GEO") && atoi(getenv("HF_TRSM_GEO")) == 0);   // geometric near segments
    if (const char *e = getenv("HF_TRSM_ELAG")) ELAG = std::max(0, atoi(e));
    pinfo.assign(nblk, make_int4(0, 0, 0, 0));
    nslots = 0;
    std::vector<std::vector<int4>> stage(nblk + 2);   // stage s -> index s+1 (stage -1 first)
    std::vector<std::pair<int, int>> segs;
    for (int j = 0; j < nblk; ++j) {
        const int nq = j > 2 ? j - 2 : 0;
        segs.clear();
        const int tail_lo = std::max(0, nq - TAIL);
        int hi = tail_lo, sz = GEO ? 1 : seg, nnear = 0;
        while (hi > 0) {
            const int lo = std::max(0, hi - sz);
            segs.push_back({lo, hi});
            if (sz < seg) ++nnear;
            hi = lo;
            sz = std::min(seg, 2 * sz);
        }
        std::reverse(segs.begin(), segs.end());      // increasing q: bulk first, then near
        const int nbulk = (int)segs.size() - nnear;
        pinfo[j] = make_int4(nslots, nbulk, nnear, tail_lo);
        int st_e = -1;
        for (int s2 = 0; s2 < (int)segs.size(); ++s2) {
            const int lo = segs[s2].first, h2 = segs[s2].second;
            const int sst = std::max(h2 - 1, j - 3 - LA);
            if (s2 < nbulk) st_e = std::max(st_e, std::max(sst, h2 - 1 + ELAG));
            for (int c = 0; c < nch; ++c) stage[sst + 1].push_back(make_int4(j, c, lo | (h2 << 16), nslots + s2));
        }
        st_e = std::max(-1, std::min(st_e, j - 3));   // before the P-worker needs it, after its bulk partials
        for (int c = 0; c < nch; ++c) stage[st_e + 1].push_back(make_int4(j, c, 0, -1 - nbulk));
        nslots += (int)segs.size() + 1;     // + the base slot
    }
    items.clear();
    for (auto &v : stage)
        for (auto &x : v) items.push_back(x);
}

void precond_apply_t(hf_ctx *ctx, PrecondT<T> &p, int64_t ncol, const double *R, int64_t ldr, double *W, int64_t ldw) {
    cudaStream_t st = ctx->stream;
    if (ncol == 0) return;
    if (p.N == 0) {
        HF_CUDA(cudaMemset2DAsync(W, ldw * sizeof(double), 0, p.L * sizeof(double), ncol, st));
        return;
    }
    const int nblk = (int)(p.Np / TBS);
    const int nch = (int)cdiv(ncol, CW);
    const int ncolp = nch * CW;
    int seg = std::max(16, (int)cdiv(nblk, 32));   // HF_TRSM_SEG: tuning (8 / 16 / 32: 7.6 / 7.2 / 7.1-7.5 ms per C2 apply)
    if (const char *e = getenv("HF_TRSM_SEG")) seg = std::max(2, atoi(e));
    p.Y.alloc((size_t)p.Np * ncolp, st);
    p.Xb.alloc((size_t)p.Np * ncolp, st);
    p.P.alloc((size_t)p.Np * ncolp, st);
    // the item table lives in the context's cache: look it up again whenever the shape,
    // the segment or the context differs (a hybrid may be solved through another context)
    if (p.tab_nblk != nblk || p.tab_nch != nch || p.tab_seg != seg || p.tab_ctx != ctx->serial) {
        auto key = std::make_pair(nblk, nch * 1000 + seg);
        auto it = ctx->trsm_tables.find(key);
        if (it == ctx->trsm_tables.end()) {
            std::vector<int4> items, pinfo;
            TrsmTable t;
            build_items(nblk, nch, seg, items, pinfo, t.nslots);
            t.items.alloc(std::max<size_t>(items.size(), 1), st);
            t.pinfo.alloc(pinfo.size(), st);
            if (!items.empty())
                HF_CUDA(cudaMemcpyAsync(t.items.p, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
            HF_CUDA(cudaMemcpyAsync(t.pinfo.p, pinfo.data(), pinfo.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
            HF_CUDA(cudaStreamSynchronize(st));   // host vectors die here (once per shape and context)
            t.nitems = (int)items.size();
            it = ctx->trsm_tables.emplace(key, std::move(t)).first;
        }
        p.items = it->second.items.p;
        p.pinfo = it->second.pinfo.p;
        p.nitems = it->second.nitems;
        p.nslots = it->second.nslots;
        p.tab_nblk = nblk;
        p.tab_nch = nch;
        p.tab_seg = seg;
        p.tab_ctx = ctx->serial;
        p.part.alloc((size_t)std::max(p.nslots, 1) * nch * TBS * CW, st);
        p.pflags.alloc((size_t)2 * std::max(p.nslots, 1) * nch, st);
        p.pflags.zero(st);
        p.flags.alloc((size_t)4 * nblk * nch, st);   // [chain flags x2 | P flags x2]
        p.flags.zero(st);
        p.epoch = 0;
    }
    const int h48 = !(getenv("HF_TRSM_H48") && atoi(getenv("HF_TRSM_H48")) == 0);
    int npw = 2;   // HF_TRSM_PW: P-worker CTAs per chunk
    if (const char *e = getenv("HF_TRSM_PW")) npw = std::max(1, atoi(e));
    const int nroles = nch * (1 + npw);
    // [2 item counters | 2 role tickets | 2 directions x (owner[MAXSM] | role[MAXSM])]
    const size_t ncnt = 4 + 4 * (size_t)TRSM_MAXSM;
    p.counter.alloc(ncnt, st);
    HF_CUDA(cudaMemsetAsync(p.counter.p, 0, ncnt * sizeof(int), st));
    p.epoch += 1;
    TrsmArgs a;
    a.N = p.N; a.Np = p.Np; a.ncol = (int)ncol; a.ncolp = ncolp; a.nch = nch; a.nblk = nblk; a.seg = seg;
    a.items = p.items; a.pinfo = p.pinfo; a.npw = npw; a.nitems = p.nitems; a.h48 = h48; a.part = p.part.p; a.P = p.P.p;
    a.pflags = p.pflags.p; a.aflags = p.flags.p + 2 * nblk * nch; a.nslots = p.nslots; a.Lp = p.Lp.p; a.Up = p.Up.p;
    a.LinvF = p.LinvF.p; a.LinvB = p.LinvB.p; a.D = p.D; a.perm = p.perm; a.R = R; a.ldr = ldr; a.Y = p.Y.p;
    a.Xb = p.Xb.p; a.flags = p.flags.p; a.counter = p.counter.p;
    a.smids = reinterpret_cast<unsigned *>(p.counter.p + 4); a.epoch = p.epoch; a.dbg = nullptr;
    const bool want_dbg = getenv("HF_TRSM_DEBUG") != nullptr;
    if (want_dbg) {
        p.dbg.alloc(16, st);
        p.dbg.zero(st);
        a.dbg = p.dbg.p;
    }
    const size_t shm = (size_t)SMEM_ELEMS * sizeof(T);
    static DevState per_sm_dev(0);
    int &per_sm = per_sm_dev[ctx->device];
    if (!per_sm) {
        HF_CUDA(cudaFuncSetAttribute(k_trsm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        HF_CUDA(cudaFuncSetAttribute(k_trsm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        int a0 = 0, a1 = 0;
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a0, k_trsm<false>, NTHR, shm));
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a1, k_trsm<true>, NTHR, shm));
        per_sm = std::max(1, std::min(a0, a1));
    }
    // roles by SM (chain CTAs, P-workers), then helpers; CTAs sharing an SM with a
    // role leave, so launch enough that helpers remain
    const int grid = std::min(std::max(nroles * per_sm + 1, nroles + p.nitems + per_sm), ctx->num_sms * per_sm);
    HF_REQUIRE(grid >= nroles * per_sm + 1, "preconditioner: too many RHS chunks for one launch");
    // algorithmic work of one application (forward + backward): N^2 ncol FMAs, the two
    // triangles of the factor (sizeof(T) N^2 / 2 each) and the right-hand sides in/out
    const double nn = (double)p.N * (double)p.N;
    ClassTimer tm(ctx, "trsm", st, 2.0 * nn * (double)ncol,
                  (double)sizeof(T) * nn + 16.0 * (double)p.N * (double)ncol);
    void *args[] = {&a};
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_trsm<false>, dim3(grid), dim3(NTHR), args, shm, st));
    HF_CHECK_LAUNCH(ctx);
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_trsm<true>, dim3(grid), dim3(NTHR), args, shm, st));
    HF_CHECK_LAUNCH(ctx);
    dim3 gl((unsigned)std::min<int64_t>(cdiv(p.L, 256), 1024), (unsigned)std::min<int64_t>(ncol, 1024));
    k_lift_scatter<<<gl, 256, 0, st>>>(p.L, (int)ncol, ncolp, p.pos1, p.Xb.p, W, ldw);
    HF_CHECK_LAUNCH(ctx);
    if (want_dbg) {
        unsigned long long h[16];
        HF_CUDA(cudaMemcpyAsync(h, p.dbg.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        HF_CUDA(cudaStreamSynchronize(st));
        for (int d = 0; d < 2; ++d) {
            fprintf(stderr, "[hf trsm %s] nblk %d nch %d grid %d items %d | us/link: wait-P %.3f  load %.3f  compute %.3f  store %.3f\n",
                    d ? "bwd" : "fwd", nblk, nch, grid, p.nitems, h[4 * d] / 1e3 / nblk, h[4 * d + 1] / 1e3 / nblk,
                    h[4 * d + 2] / 1e3 / nblk, h[4 * d + 3] / 1e3 / nblk);
            fprintf(stderr, "[hf trsm %s] P-workers (chunk 0), us per block: base %.3f  near slots %.3f  tail %.3f  store+next %.3f\n",
                    d ? "bwd" : "fwd", h[8 + 4 * d] / 1e3 / nblk, h[9 + 4 * d] / 1e3 / nblk, h[10 + 4 * d] / 1e3 / nblk,
                    h[11 + 4 * d] / 1e3 / nblk);
        }
    }
}

