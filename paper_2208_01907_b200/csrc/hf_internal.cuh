// hf_internal.cuh -- private definitions of libhf (B200 / sm_100a).
// Nothing here is shared with oracle/ (test infrastructure).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/hf.h"

#ifdef HF_WITH_NCCL
#include <nccl.h>
#endif

namespace hf {

// ----------------------------------------------------------------- errors
struct Error {
    hf_status st;
    std::string msg;
};

#define HF_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            throw ::hf::Error{e_ == cudaErrorMemoryAllocation ? HF_ERR_OOM : HF_ERR_CUDA, \
                              std::string(#call) + ": " + cudaGetErrorString(e_) +     \
                                  " (" __FILE__ ":" + std::to_string(__LINE__) + ")"}; \
    } while (0)

#define HF_CHECK_LAUNCH(ctx)                                                           \
    do {                                                                               \
        cudaError_t e_ = cudaGetLastError();                                           \
        if (e_ != cudaSuccess)                                                         \
            throw ::hf::Error{HF_ERR_CUDA, std::string("kernel launch: ") +            \
                                               cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                                               std::to_string(__LINE__) + ")"};        \
        (ctx)->launches++;                                                             \
    } while (0)

#define HF_REQUIRE(cond, msg)                                                          \
    do {                                                                               \
        if (!(cond)) throw ::hf::Error{HF_ERR_INVALID_ARG, std::string(msg)};          \
    } while (0)

// ----------------------------------------------------------------- device buffers
// device-memory cache (alloc.cu): stream-ordered reuse of freed blocks
void *dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void *p, cudaStream_t s);
size_t cached_free_bytes(int dev);

template <typename T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept { *this = std::move(o); }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void release() {
        if (p) dev_free(p, s);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count, cudaStream_t stream) {
        if (count <= n && p) return;
        release();
        s = stream;
        size_t bytes = (count ? count : 1) * sizeof(T);
        p = static_cast<T *>(dev_alloc(bytes, stream));
        n = count;
    }
    void zero(cudaStream_t stream) {
        if (p) HF_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), stream));
    }
};

// ----------------------------------------------------------------- context
struct KStat {
    double ms = 0.0;
    int64_t launches = 0;
};
// algorithmic work of one kernel class (flops, bytes), summed while profiling
struct KWork {
    double flops = 0.0, bytes = 0.0;
};

// one-time per-device state (kernel attributes such as the dynamic shared-memory
// limit apply per device context, so a process with contexts on several devices
// sets them once per device)
constexpr int HF_MAX_DEV = 64;
struct DevState {
    int v[HF_MAX_DEV];
    explicit DevState(int init) {
        for (int &x : v) x = init;
    }
    int &operator[](int dev) { return v[((dev % HF_MAX_DEV) + HF_MAX_DEV) % HF_MAX_DEV]; }
};

}  // namespace hf

namespace hf {
// dataflow item table of the preconditioner solves (k_trsm.cu), per shape
struct TrsmTable {
    int nitems = 0, nslots = 0;
    DBuf<int4> items;     // PARTIAL items
    DBuf<int4> pinfo;     // per block: (first slot, #slots, tail q_lo, tail q_hi)
};
}  // namespace hf

struct hf_ctx {
    uint64_t serial = 0;               // unique per context (never reused): owner tag of cached tables
    int device = 0;
    cudaStream_t stream = 0;
    int num_sms = 148;
    int rank = 0, nranks = 1;
    int vrank = 0, vnranks = 0;        // single-GPU emulation of one rank (hf_set_virtual_rank)
    int s1parts = 0;                   // stage-1 column partitions emulated on this GPU (0: off)
#ifdef HF_WITH_NCCL
    ncclComm_t comm = nullptr;
#endif
    std::string last_error;
    int64_t launches = 0;
    bool profiling = false;
    // pending (start, stop) event pairs per class; resolved lazily
    std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::map<std::string, hf::KStat> stats;
    std::map<std::string, hf::KWork> work;   // algorithmic flops / bytes per class (hf_kernel_work)
    std::vector<cudaEvent_t> event_pool;
    std::map<std::pair<int, int>, hf::TrsmTable> trsm_tables;   // (nblk, nch) -> table
    cudaStream_t side = nullptr;       // second stream (stage-1 lookahead: trailing updates), lazily created
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // hf_upload_lower: host -> device copies on their own stream (lazily created); the
    // event marks the last one, and hf_scale / hf_scale_host order the context stream after it
    cudaStream_t up = nullptr;
    cudaEvent_t up_ev = nullptr;
    bool up_pending = false;
    // the blocked preconditioner's two helper streams (k_trsm_blk.cu), lazily created
    cudaStream_t aux[2] = {nullptr, nullptr};
    // the automatic mat-vec choice's memory check per (L, n) (gcr.cu): made once, since
    // cudaMemGetInfo waits on the device and the choice then stays the same for every solve
    std::map<std::pair<int64_t, int64_t>, bool> matvec_room;
};

namespace hf {

// switches to the context's device for the duration of a call and restores the
// caller's current device (every launch and kernel attribute of a call then
// targets ctx->device whatever device the caller has current)
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const hf_ctx *ctx) {
        if (!ctx) return;
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            return;
        }
        if (prev != ctx->device) cudaSetDevice(ctx->device);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// RAII timer around launches of one kernel class (only when profiling).
// flops / bytes: the ALGORITHMIC work of the launches it brackets (what the method
// must compute, e.g. only the lower-triangle entries of a trailing update), summed
// per class for hf_kernel_work while profiling; 0 where nobody reports it.
struct ClassTimer {
    hf_ctx *ctx;
    const char *cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    double fl = 0.0, by = 0.0;
    ClassTimer(hf_ctx *c, const char *k, cudaStream_t on = nullptr, double flops = 0.0, double bytes = 0.0)
        : ctx(c), cls(k), s(on ? on : c->stream), fl(flops), by(bytes) {
        if (!ctx->profiling) return;
        a = take(); b = take();
        cudaEventRecord(a, s);
    }
    ~ClassTimer() {
        if (!ctx->profiling || !a) return;
        cudaEventRecord(b, s);
        ctx->pending[cls].push_back({a, b});
        auto &w = ctx->work[cls];
        w.flops += fl;
        w.bytes += by;
    }
    cudaEvent_t take() {
        if (!ctx->event_pool.empty()) {
            cudaEvent_t e = ctx->event_pool.back();
            ctx->event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// host-side pacing diagnostics (HF_TRACE_HOST=<ms>): prints the host time since the previous
// trace point when it exceeds the threshold
void host_trace(const char *where);

}  // namespace hf

// preconditioner state (k_trsm.cu): T = float (FP32 factor) or double (FP64, NEXT-1)
namespace hf {
template <typename T>
struct PrecondT {
    int64_t N = 0, L = 0;
    const T *Lfac = nullptr;       // N x N unit lower, pivot order
    const T *D = nullptr;          // [N]
    const int64_t *perm = nullptr; // [L] pivot order -> original index
    const int32_t *pos1 = nullptr; // [L] original index -> pivot rank, -1 on Lambda_2
    int64_t Np = 0;                // N rounded up to the 64-row block
    DBuf<T> Lp, Up;            // Np x Np: L padded with the identity, and L^T, each block row
                                   // scaled in place by its diagonal-block inverse (G = Dinv Op)
    DBuf<T> LinvF, LinvB;      // inverses of the 64x64 diagonal blocks (tile layouts)
    DBuf<T> P;                 // Np x ncolp: P_j of the chain recurrence (row-major)
    DBuf<T> Y;                 // Np x ncolp workspace (FP32, row-major)
    DBuf<T> Xb;                // Np x ncolp workspace (FP32, row-major)
    DBuf<int> flags;
    DBuf<int> counter;
    int epoch = 0;
    // dataflow workspaces (k_trsm.cu), re-sized when the block/chunk counts change
    int tab_nblk = -1, tab_nch = -1, tab_seg = -1, nitems = 0, nslots = 0;
    uint64_t tab_ctx = 0;          // serial of the context whose table cache owns items / pinfo
    const int4 *items = nullptr;   // owned by the context's table cache
    const int4 *pinfo = nullptr;
    DBuf<T> part;
    DBuf<int> pflags;
    DBuf<unsigned long long> dbg;
};
// the blocked tensor-core form of the FP32 preconditioner (k_trsm_blk.cu)
struct PrecondBlk {
    int64_t N = 0, L = 0, Nb = 0, BS = 0;
    int nb = 0;
    const float *D = nullptr;
    const int64_t *perm = nullptr;
    const int32_t *pos1 = nullptr;
    DBuf<uint16_t> Lc, Lr;         // the strictly lower blocks of L as three exact bfloat16 parts,
                                   // packed by block column (parts side by side) / block row
                                   // (parts stacked): k_trsm_blk.cu lc_off / lr_off
    DBuf<uint16_t> Ic, It;         // Linv_j, six-part concatenations (BS x 6BS / 6BS x BS) per block
    DBuf<uint16_t> Gc, Ht;         // G_j = L_{j+1,j} Linv_j (BS x 6BS), H_j = Linv_{j+1} L_{j+1,j} (6BS x BS)
    DBuf<float> Xa, Xb, Y;         // Nb x ncp FP32 workspaces (column-major)
    DBuf<float> P6a, P6c;          // 6 x BS x ncp part-product partials of the small products (streams A, C)
    DBuf<uint16_t> S6, SB;         // per block: 6BS x ncp part stacks of its right-hand side / solution
    DBuf<uint16_t> SC;             // few columns: per block the 3BS x 3ncp part matrix of the bulk update
    DBuf<float> TB;                // few columns: Nb x 3ncp partials of the bulk update
    std::vector<cudaEvent_t> ev;   // per-block events of the three-stream schedule
    PrecondBlk() = default;
    PrecondBlk(const PrecondBlk &) = delete;
    PrecondBlk &operator=(const PrecondBlk &) = delete;
    ~PrecondBlk() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};
struct Precond {
    int prec = 32;
    bool blk = false;              // FP32, symmetric: the blocked tensor-core solve
    PrecondT<float> f;
    PrecondT<double> d;
    PrecondBlk b;
};
}  // namespace hf

// ----------------------------------------------------------------- handles
struct hf_lowfactor {
    int64_t L = 0, N = 0, Ntau = 0, n2 = 0;
    int prec = 32;                     // 32: FP32 factor (the north_star); 64: FP64 (NEXT-1)
    std::vector<double> h_D64;         // prec 64: D (host copy, exact)
    hf::DBuf<double> D64, Lfac64;      // prec 64: D and the N x N unit lower factor
    std::vector<int64_t> h_perm;       // Pi (host copy)
    std::vector<float> h_D;            // D (host copy)
    hf::DBuf<int64_t> perm;            // Pi (device)
    hf::DBuf<int32_t> pos1;            // original index -> pivot rank (Lambda_1) or -1
    hf::DBuf<float> D;                 // [N]
    hf::DBuf<float> Lfac;              // N x N unit lower, pivot order, ld = N
    bool nonsym = false;               // NEXT-3: LDU of a general matrix; U = Ufac^T
    hf::DBuf<float> Ufac;              // N x N: column k = row k of the unit upper U
    cudaStream_t stream = 0;
};

struct hf_hybrid {
    const double *K = nullptr;         // borrowed scaled K
    int64_t ld = 0, L = 0, N = 0, n2 = 0;
    const hf_lowfactor *lf = nullptr;  // borrowed
    hf::DBuf<double> X;                // L x n2, original row order, zero on Lambda_2 rows
    hf::DBuf<double> B;                // L x n2: K12 (original row order, zero on Lambda_2 rows)
    hf::DBuf<double> S22;              // n2 x n2, Lambda_2 ascending
    bool dd = false;                   // NEXT-1: X and S22 in double-double (hi in X / S22, lo below)
    bool nonsym = false;               // NEXT-3: general K: B2 = K21^T, S22 by LU with complete pivoting
    hf::DBuf<double> B2;               // L x n2: K21^T (original row order, zero on Lambda_2 rows)
    hf::DBuf<double> LUh;              // n2 x n2: [L \ U] of P S22 Q
    hf::DBuf<int32_t> pcol2;           // [n2] column pivot labels (perm2 holds the row labels)
    hf::DBuf<double> Xlo, S22lo, Lhlo, Dhlo;   // dd: lo parts (Lh / Dh hold the hi parts)
    hf::DBuf<int64_t> lam2;            // [n2] original indices (ascending)
    hf::DBuf<uint8_t> mask1;           // [L] 1 on Lambda_1 rows
    // stage 3
    bool hard_done = false;
    int64_t rank = 0, kernel_dim = 0;
    hf::DBuf<double> Lh;               // n2 x n2 unit lower (pivoted positions)
    hf::DBuf<double> Dh;               // n2 x n2 block diagonal
    hf::DBuf<int32_t> perm2;           // [n2]
    hf::DBuf<int32_t> blocks;          // [n2]
    mutable hf::Precond pc;            // FP32 preconditioner (workspaces reused by hf_solve)
    cudaStream_t stream = 0;
    int num_sms = 148;
};

// ----------------------------------------------------------------- launchers
namespace hf {
void launch_scale(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q, int *bad_flag);
void launch_scale_full(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q, int *bad_flag);   // NEXT-3
void lowprec_factor(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                    hf_lowfactor *lf, const int32_t *blk_host = nullptr, int nblk = 0);
double chain_exchange_floor(hf_ctx *ctx, int nctas, int nthreads, int steps);
void lowprec_outputs(hf_ctx *ctx, int64_t L, const hf_lowprec_opts &o, hf_lowfactor *lf, const int32_t *status,
                     const int32_t *pivorig, const float *Dk);
void lowprec_factor_dist(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                         hf_lowfactor *lf, int nranks_emulated);
void lowprec_factor64(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                      hf_lowfactor *lf);
void lowprec_factor_ns(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts &o,
                       hf_lowfactor *lf);   // NEXT-3
// NEXT-4: nested-dissection blocks of the symmetric pattern of K (nd.cu)
void nd_blocks(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, int levels, int min_size, int32_t *blk_host,
               int32_t *nblk_host);
void schur_gcr(hf_ctx *ctx, hf_hybrid *hy, const hf_gcr_opts &o, hf_gcr_info *info);
void factor_hard(hf_ctx *ctx, hf_hybrid *hy, double eps_ker);
void schur_gcr_dd(hf_ctx *ctx, hf_hybrid *hy, const hf_gcr_opts &o, hf_gcr_info *info);   // gcr_dd.cu
void factor_hard_dd(hf_ctx *ctx, hf_hybrid *hy, double eps_ker);
void hybrid_solve_dd(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *xh, double *xl,
                     const hf_gcr_opts &o, hf_gcr_info *info);
void hybrid_solve(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *x, const hf_gcr_opts &o,
                  hf_gcr_info *info);
// multi-GPU plumbing (dist.cu)
void shard_cols(int64_t n2, int nranks, int rank, int64_t *c0, int64_t *c1);
#ifdef HF_WITH_NCCL
void collective_begin(hf_ctx *ctx);
void collective_end(hf_ctx *ctx);
void collective_bcast(hf_ctx *ctx, double *buf, size_t count, int root);
void collective_max(hf_ctx *ctx, double *buf, size_t count);
void collective_allgather_bytes(hf_ctx *ctx, const void *send, void *recv, size_t bytes);
void collective_barrier(hf_ctx *ctx, int *dev_int);
#endif
}  // namespace hf
