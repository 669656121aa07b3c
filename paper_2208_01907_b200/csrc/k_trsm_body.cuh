// k_trsm_body.cuh -- the preconditioner solves of k_trsm.cu, written once for
// the element type T (included twice by k_trsm.cu: T = float, the paper's FP32
// preconditioner [R12]; T = double, the FP64 one of the (double, dd) pair).
// Everything here lives in a per-precision namespace of k_trsm.cu.
constexpr int EPC = 16 / (int)sizeof(T);   // elements per 16-byte cp.async chunk

// ------------------------------------------------------------------ setup kernels
// Lp (Np x Np, ld Np) = Lfac (N x N, ld N) padded with the identity; Up = Lp^T.
// 32x32 tiles through shared memory so both the read and the transposed write
// are coalesced.
__global__ void __launch_bounds__(256) k_pad_transpose(int64_t N, int64_t Np, const T *__restrict__ Lf,
                                                       T *__restrict__ Lp, T *__restrict__ Up) {
    __shared__ T t[32][33];
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
    const int4 *items;   // [nitems] (logical block j, chunk, segment or -1, slot)
    int nitems;
    const int *pbase;    // [nblk] first partial slot of logical block j
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
    unsigned *smids;     // [2][nch] SM of each chain CTA (+1; 0 = not yet published)
    int epoch;
    unsigned long long *dbg;   // optional chain phase timers (HF_TRSM_DEBUG)
};


// acc[i][j] (+|-)= sum_k As[k][tr*4+i] * Bs[k][tc*4+j]; FP32: FFMA2 with a broadcast
// scalar (half the issue slots of scalar FFMA), the pairs along j kept in float2
template <bool NEG>
__device__ __forceinline__ void tile_prod(T (&acc)[4][4], const T *As, const T *Bs, int tr, int tc) {
    if constexpr (sizeof(T) == 4) {
        float2 c2[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            c2[i][0] = make_float2(acc[i][0], acc[i][1]);
            c2[i][1] = make_float2(acc[i][2], acc[i][3]);
        }
#pragma unroll 16
        for (int k = 0; k < TBS; ++k) {
            const V4<T> a = ld4(&As[k * TBS + tr * 4]);
            const V4<T> y = ld4(&Bs[k * CW + tc * 4]);
            const T av[4] = {NEG ? -a.x : a.x, NEG ? -a.y : a.y, NEG ? -a.z : a.z, NEG ? -a.w : a.w};
            const float2 y01 = make_float2(y.x, y.y), y23 = make_float2(y.z, y.w);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                c2[i][0] = __ffma2_rn(make_float2(av[i], av[i]), y01, c2[i][0]);
                c2[i][1] = __ffma2_rn(make_float2(av[i], av[i]), y23, c2[i][1]);
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
        for (int k = 0; k < TBS; ++k) {
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
__device__ __forceinline__ void tile_fma(T (&acc)[4][4], const T *As, const T *Bs, int tr, int tc) {
    tile_prod<false>(acc, As, Bs, tr, tc);
}
__device__ __forceinline__ void tile_fms(T (&acc)[4][4], const T *As, const T *Bs, int tr, int tc) {
    tile_prod<true>(acc, As, Bs, tr, tc);
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
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) Op[(r0 + tr * 4 + i) + (q0 + tc * 4 + jj) * Np] = acc[i][jj];
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
constexpr int SMEM_ELEMS = 7 * TILE;     // 112 KB: chain = Yring[3] + M[2 stages][2]; helper = 2 x (A + B)

template <bool BWD>
__global__ void __launch_bounds__(NTHR, 2) k_trsm(TrsmArgs a) {
    extern __shared__ __align__(16) T sm[];
    __shared__ int item_s;
    const int tid = threadIdx.x, tr = tid & 15, tc = (tid >> 4) & 15;
    int *flags = a.flags + (BWD ? a.nblk * a.nch : 0);
    int *pflags = a.pflags + (BWD ? a.nslots * a.nch : 0);
    int *aflags = a.aflags + (BWD ? a.nblk * a.nch : 0);
    int *counter = a.counter + (BWD ? 1 : 0);
    unsigned *smids = a.smids + (BWD ? a.nch : 0);
    const T *Op = BWD ? a.Up : a.Lp;
    T *Yout = BWD ? a.Xb : a.Y;
    const T *Dinv = BWD ? a.LinvB : a.LinvF;
    auto phys = [&](int j) { return BWD ? (a.nblk - 1 - j) : j; };

    if ((int)blockIdx.x < a.nch) {
        // =================================================== CHAIN (chunk cc)
        const int cc = blockIdx.x, c0 = cc * CW;
        if (tid == 0) atomicExch(&smids[cc], smid() + 1u);
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

    // ======================================================= HELPERS (256 threads)
    if (tid >= NCOMP) return;
    {
        // leave the chain CTAs' SMs to them
        __shared__ int leave;
        if (tid == 0) {
            const unsigned me = smid() + 1u;
            int l = 0;
            for (int c = 0; c < a.nch; ++c) {
                unsigned v;
                while ((v = *(volatile unsigned *)&smids[c]) == 0u) __nanosleep(64);
                l |= (v == me);
            }
            leave = l;
        }
        bar_sync(5, NCOMP);
        if (leave) return;
    }
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
    auto wait_flag = [&](const int *f) {
        if (tid == 0) wait_epoch(f, a.epoch);
        bar_sync(5, NCOMP);
    };
    // t += sum over logical dependency blocks [q_lo, q_hi) of Op_bq Y_q, double buffered
    auto accumulate = [&](T (&t)[4][4], int64_t r0, int c0, int cc, int q_lo, int q_hi) {
        const int ndep = q_hi - q_lo;
        if (ndep <= 0) return;
        wait_flag(&flags[q_lo * a.nch + cc]);
        load_dep(0, r0, (int64_t)phys(q_lo) * TBS, c0);
        cp_commit();
        for (int dq = 0; dq < ndep; ++dq) {
            if (dq + 1 < ndep) {
                wait_flag(&flags[(q_lo + dq + 1) * a.nch + cc]);
                load_dep((dq + 1) & 1, r0, (int64_t)phys(q_lo + dq + 1) * TBS, c0);
                cp_commit();
                cp_wait_1();
            } else {
                cp_wait_all();
            }
            bar_sync(5, NCOMP);
            const T *As = sm + (dq & 1) * 2 * TILE;
            tile_fma(t, As, As + TILE, tr, tc);
            bar_sync(5, NCOMP);
        }
    };

    for (;;) {
        if (tid == 0) item_s = atomicAdd(counter, 1);
        bar_sync(5, NCOMP);
        const int idx = item_s;
        if (idx >= a.nitems) return;
        const int4 it = a.items[idx];
        const int j = it.x, cc = it.y, sg = it.z, slot = it.w;
        const int b = phys(j);
        const int64_t r0 = (int64_t)b * TBS;
        const int c0 = cc * CW;
        T t[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) t[i][jj] = T(0);
        if (sg >= 0) {
            // ---- PARTIAL item: t = sum over segment sg of Op_bq Y_q -> slot
            accumulate(t, r0, c0, cc, sg * a.seg, (sg + 1) * a.seg);
            T *pp = a.part + ((size_t)slot * a.nch + cc) * (TBS * CW);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                st4(&pp[(tr * 4 + i) * CW + tc * 4], t[i][0], t[i][1], t[i][2], t[i][3]);
            bar_sync(5, NCOMP);
            if (tid == 0) {
                __threadfence();
                st_release32(&pflags[slot * a.nch + cc], a.epoch);
            }
            continue;
        }
        // ---- P-item.  First Dinv_j RHS_j (no dependency): forward truncates R
        //      (FP64, original order) to FP32, backward starts from z = D^{-1} y
        T out[4][4] = {};
        {
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
        }
        // then t = partial slots in fixed order + the last segment (up to j-3)
        const int nq = j > 2 ? j - 2 : 0;
        const int nseg = (nq + a.seg - 1) / a.seg;
        for (int s2 = 0; s2 + 1 < nseg; ++s2) {
            const int sl = a.pbase[j] + s2;
            wait_flag(&pflags[sl * a.nch + cc]);
            const T *pp = a.part + ((size_t)sl * a.nch + cc) * (TBS * CW);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const V4<T> v = ld4(&pp[(tr * 4 + i) * CW + tc * 4]);
                t[i][0] += v.x;
                t[i][1] += v.y;
                t[i][2] += v.z;
                t[i][3] += v.w;
            }
        }
        accumulate(t, r0, c0, cc, nseg > 0 ? (nseg - 1) * a.seg : 0, nq);
        // P_j = Dinv_j RHS_j - t
#pragma unroll
        for (int i = 0; i < 4; ++i)
            st4(&a.P[(r0 + tr * 4 + i) * a.ncolp + c0 + tc * 4], out[i][0] - t[i][0], out[i][1] - t[i][1], out[i][2] - t[i][2], out[i][3] - t[i][3]);
        bar_sync(5, NCOMP);
        if (tid == 0) {
            __threadfence();
            st_release32(&aflags[j * a.nch + cc], a.epoch);
        }
    }
}

// ------------------------------------------------------------------ host side
void precond_setup_t(hf_ctx *ctx, PrecondT<T> &p, int64_t N, int64_t L, const T *Lfac, const T *D,
                   const int64_t *perm, const int32_t *pos1) {
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
    ClassTimer tm(ctx, "trsm");
    dim3 g((unsigned)(p.Np / 32), (unsigned)(p.Np / 32));
    k_pad_transpose<<<g, 256, 0, st>>>(N, p.Np, Lfac, p.Lp.p, p.Up.p);
    HF_CHECK_LAUNCH(ctx);
    const size_t sm_inv = (size_t)2 * TBS * (TBS + 1) * sizeof(T);
    const size_t sm_sc = ((size_t)TBS * (TBS + 1) + 4 + TILE) * sizeof(T);
    static bool attr_setup = false;
    if (!attr_setup) {
        HF_CUDA(cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_inv));
        HF_CUDA(cudaFuncSetAttribute(k_scale_op<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc));
        HF_CUDA(cudaFuncSetAttribute(k_scale_op<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc));
        attr_setup = true;
    }
    k_diag_inv<<<(unsigned)nblk, TBS, sm_inv, st>>>(p.Np, p.Lp.p, p.LinvF.p, p.LinvB.p);
    HF_CHECK_LAUNCH(ctx);
    // G = Dinv Op in place (after the diagonal inverses, which read the diagonal blocks only)
    dim3 gs((unsigned)nblk, (unsigned)nblk);
    k_scale_op<false><<<gs, 256, sm_sc, st>>>((int)nblk, p.Np, p.Lp.p, p.LinvF.p);
    HF_CHECK_LAUNCH(ctx);
    k_scale_op<true><<<gs, 256, sm_sc, st>>>((int)nblk, p.Np, p.Up.p, p.LinvB.p);
    HF_CHECK_LAUNCH(ctx);
}

// Helper item table in topological order.  Logical blocks j (forward j = b,
// backward j = nblk-1-b); P_j depends on chain outputs 0..j-3 and on its
// partial slots.  Items are placed by the chain stage after which they can
// run: P-item(j) at stage j-3; PARTIAL(j, s) (segment [s*seg, (s+1)*seg) of
// the dependency range [0, j-2), all but its last segment) at stage
// max((s+1)*seg - 1, j-3-LA), LA = lookahead, so bulk work is queued just
// ahead of the chain instead of in front of it.  Within a stage: P-items
// first.  Every item depends only on earlier items and on chain stages <=
// its own stage, so persistent CTAs taking items in order cannot deadlock.
static void build_items(int nblk, int nch, int seg, std::vector<int4> &items, std::vector<int> &pbase, int &nslots) {
    int LA = 24;   // HF_TRSM_LA: tuning
    if (const char *e = getenv("HF_TRSM_LA")) LA = std::max(0, atoi(e));
    pbase.assign(nblk, 0);
    nslots = 0;
    std::vector<std::vector<int4>> stage(nblk + 2);   // stage s -> index s+1 (stage -1 first)
    for (int j = 0; j < nblk; ++j) {
        pbase[j] = nslots;
        const int nq = j > 2 ? j - 2 : 0;
        const int nseg = (nq + seg - 1) / seg;
        nslots += std::max(0, nseg - 1);
    }
    for (int j = 0; j < nblk; ++j) {
        const int st = std::max(-1, j - 3);
        for (int c = 0; c < nch; ++c) stage[st + 1].push_back(make_int4(j, c, -1, -1));
    }
    for (int j = 0; j < nblk; ++j) {
        const int nq = j > 2 ? j - 2 : 0;
        const int nseg = (nq + seg - 1) / seg;
        for (int s = 0; s + 1 < nseg; ++s) {
            const int st = std::max((s + 1) * seg - 1, j - 3 - LA);
            for (int c = 0; c < nch; ++c) stage[st + 1].push_back(make_int4(j, c, s, pbase[j] + s));
        }
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
    if (p.tab_nblk != nblk || p.tab_nch != nch) {
        auto key = std::make_pair(nblk, nch * 1000 + seg);
        auto it = ctx->trsm_tables.find(key);
        if (it == ctx->trsm_tables.end()) {
            std::vector<int4> items;
            std::vector<int> pbase;
            TrsmTable t;
            build_items(nblk, nch, seg, items, pbase, t.nslots);
            t.items.alloc(items.size(), st);
            t.pbase.alloc(pbase.size(), st);
            HF_CUDA(cudaMemcpyAsync(t.items.p, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
            HF_CUDA(cudaMemcpyAsync(t.pbase.p, pbase.data(), pbase.size() * sizeof(int), cudaMemcpyHostToDevice, st));
            HF_CUDA(cudaStreamSynchronize(st));   // host vectors die here (once per shape and context)
            t.nitems = (int)items.size();
            it = ctx->trsm_tables.emplace(key, std::move(t)).first;
        }
        p.items = it->second.items.p;
        p.pbase = it->second.pbase.p;
        p.nitems = it->second.nitems;
        p.nslots = it->second.nslots;
        p.tab_nblk = nblk;
        p.tab_nch = nch;
        p.part.alloc((size_t)std::max(p.nslots, 1) * nch * TBS * CW, st);
        p.pflags.alloc((size_t)2 * std::max(p.nslots, 1) * nch, st);
        p.pflags.zero(st);
        p.flags.alloc((size_t)4 * nblk * nch, st);   // [chain flags x2 | P flags x2]
        p.flags.zero(st);
        p.epoch = 0;
    }
    p.counter.alloc(2 + 2 * (size_t)nch, st);      // [2 counters | 2 x nch SM ids]
    HF_CUDA(cudaMemsetAsync(p.counter.p, 0, (2 + 2 * (size_t)nch) * sizeof(int), st));
    p.epoch += 1;
    TrsmArgs a{p.N, p.Np, (int)ncol, ncolp, nch, nblk, seg, p.items, p.nitems, p.pbase, p.part.p,
               p.P.p, p.pflags.p, p.flags.p + 2 * nblk * nch, p.nslots, p.Lp.p, p.Up.p, p.LinvF.p, p.LinvB.p,
               p.D, p.perm, R, ldr, p.Y.p, p.Xb.p, p.flags.p, p.counter.p,
               reinterpret_cast<unsigned *>(p.counter.p + 2), p.epoch, nullptr};
    const bool want_dbg = getenv("HF_TRSM_DEBUG") != nullptr;
    if (want_dbg) {
        p.dbg.alloc(8, st);
        p.dbg.zero(st);
        a.dbg = p.dbg.p;
    }
    const size_t shm = (size_t)SMEM_ELEMS * sizeof(T);
    static int per_sm = 0;
    if (!per_sm) {
        HF_CUDA(cudaFuncSetAttribute(k_trsm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        HF_CUDA(cudaFuncSetAttribute(k_trsm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        int a0 = 0, a1 = 0;
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a0, k_trsm<false>, NTHR, shm));
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a1, k_trsm<true>, NTHR, shm));
        per_sm = std::max(1, std::min(a0, a1));
    }
    // helpers that share an SM with a chain CTA leave, so launch more than 2 nch
    const int grid = std::min(std::max(2 * nch + 1, nch + p.nitems + per_sm), ctx->num_sms * per_sm);
    HF_REQUIRE(grid >= 2 * nch + 1, "preconditioner: too many RHS chunks for one launch");
    ClassTimer tm(ctx, "trsm");
    void *args[] = {&a};
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_trsm<false>, dim3(grid), dim3(NTHR), args, shm, st));
    HF_CHECK_LAUNCH(ctx);
    HF_CUDA(cudaLaunchCooperativeKernel((void *)k_trsm<true>, dim3(grid), dim3(NTHR), args, shm, st));
    HF_CHECK_LAUNCH(ctx);
    dim3 gl((unsigned)std::min<int64_t>(cdiv(p.L, 256), 1024), (unsigned)std::min<int64_t>(ncol, 1024));
    k_lift_scatter<<<gl, 256, 0, st>>>(p.L, (int)ncol, ncolp, p.pos1, p.Xb.p, W, ldw);
    HF_CHECK_LAUNCH(ctx);
    if (want_dbg) {
        unsigned long long h[8];
        HF_CUDA(cudaMemcpyAsync(h, p.dbg.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        HF_CUDA(cudaStreamSynchronize(st));
        for (int d = 0; d < 2; ++d)
            fprintf(stderr, "[hf trsm %s] nblk %d nch %d grid %d items %d | us/link: wait-P %.3f  load %.3f  compute %.3f  store %.3f\n",
                    d ? "bwd" : "fwd", nblk, nch, grid, p.nitems, h[4 * d] / 1e3 / nblk, h[4 * d + 1] / 1e3 / nblk,
                    h[4 * d + 2] / 1e3 / nblk, h[4 * d + 3] / 1e3 / nblk);
    }
}

