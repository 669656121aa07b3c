// api.cu -- extern "C" entry points of libhf (include/hf.h).  Argument checks,
// status/error plumbing and handle lifetime; every step of the path runs in
// the kernels of k_*.cu.
#include <math.h>

#include <atomic>
#include <cstring>
#include <memory>

#include "hf_internal.cuh"
#include "k_dgemm.cuh"
#include "k_small.cuh"
#include "lt.cuh"
#include "ozaki.cuh"

namespace {

thread_local std::string g_noctx_error;
std::atomic<uint64_t> g_ctx_serial{0};

using hf::DeviceGuard;

template <typename F>
hf_status guarded(hf_ctx *ctx, F &&f) {
    DeviceGuard dg(ctx);
    try {
        hf::host_trace("api call");
        f();
        hf::host_trace("api return");
        if (ctx) ctx->last_error.clear();
        return HF_OK;
    } catch (const hf::Error &e) {
        if (ctx) ctx->last_error = e.msg;
        else g_noctx_error = e.msg;
        return e.st;
    } catch (const std::bad_alloc &) {
        if (ctx) ctx->last_error = "host allocation failed";
        return HF_ERR_OOM;
    } catch (const std::exception &e) {
        if (ctx) ctx->last_error = e.what();
        return HF_ERR_CUDA;
    }
}

void resolve_stats(hf_ctx *ctx) {
    for (auto &kv : ctx->pending) {
        auto &st = ctx->stats[kv.first];
        for (auto &pr : kv.second) {
            float ms = 0.f;
            if (cudaEventSynchronize(pr.second) == cudaSuccess &&
                cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess)
                st.ms += ms;
            st.launches += 1;
            ctx->event_pool.push_back(pr.first);
            ctx->event_pool.push_back(pr.second);
        }
        kv.second.clear();
    }
}

}  // namespace

extern "C" {

hf_status hf_create(int device, void *cuda_stream, hf_ctx **out) {
    if (!out) return HF_ERR_INVALID_ARG;
    *out = nullptr;
    std::unique_ptr<hf_ctx> c(new (std::nothrow) hf_ctx());
    if (!c) return HF_ERR_OOM;
    hf_status s = guarded(nullptr, [&] {
        HF_CUDA(cudaSetDevice(device));
        cudaDeviceProp p;
        HF_CUDA(cudaGetDeviceProperties(&p, device));
        HF_REQUIRE(p.major >= 10, "libhf is built for sm_100a (B200); device is sm_" +
                                      std::to_string(p.major) + std::to_string(p.minor));
        c->device = device;
        c->num_sms = p.multiProcessorCount;
        c->stream = (cudaStream_t)cuda_stream;
        c->serial = ++g_ctx_serial;
        // (libhf's workspaces come from its own cache, alloc.cu; the device's default
        // stream-ordered pool, which other libraries in the process use, is left alone)
    });
    if (s != HF_OK) return s;
    *out = c.release();
    return HF_OK;
}

hf_status hf_destroy(hf_ctx *ctx) {
    if (!ctx) return HF_OK;
    DeviceGuard dg(ctx);
    cudaStreamSynchronize(ctx->stream);
    for (auto &kv : ctx->pending)
        for (auto &pr : kv.second) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    for (auto e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->up) {
        cudaStreamSynchronize(ctx->up);
        cudaStreamDestroy(ctx->up);
    }
    for (auto a : ctx->aux)
        if (a) {
            cudaStreamSynchronize(a);
            try {
                hf::lt_release_stream(ctx, a);
            } catch (...) {
            }
            cudaStreamDestroy(a);
        }
    if (ctx->up_ev) cudaEventDestroy(ctx->up_ev);
#ifdef HF_WITH_NCCL
    if (ctx->comm) ncclCommDestroy(ctx->comm);
#endif
    delete ctx;
    return HF_OK;
}

const char *hf_last_error(const hf_ctx *ctx) {
    return ctx ? ctx->last_error.c_str() : g_noctx_error.c_str();
}

hf_status hf_set_profiling(hf_ctx *ctx, int enable) {
    if (!ctx) return HF_ERR_INVALID_ARG;
    ctx->profiling = enable != 0;
    // pre-create the timing events: creating thousands of them inside a timed
    // region stalls the launch stream when the driver grows its event storage
    if (ctx->profiling)
        while (ctx->event_pool.size() < 16384) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) break;
            ctx->event_pool.push_back(e);
        }
    return HF_OK;
}

hf_status hf_kernel_stats(hf_ctx *ctx, const char *cls, double *ms_host, int64_t *launches_host) {
    if (!ctx || !cls) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        resolve_stats(ctx);
        auto it = ctx->stats.find(cls);
        double ms = 0.0;
        int64_t n = 0;
        if (it != ctx->stats.end()) {
            ms = it->second.ms;
            n = it->second.launches;
        }
        if (ms_host) *ms_host = ms;
        if (launches_host) *launches_host = n;
    });
}

hf_status hf_kernel_work(hf_ctx *ctx, const char *cls, double *flops_host, double *bytes_host) {
    if (!ctx || !cls) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        auto it = ctx->work.find(cls);
        if (flops_host) *flops_host = it != ctx->work.end() ? it->second.flops : 0.0;
        if (bytes_host) *bytes_host = it != ctx->work.end() ? it->second.bytes : 0.0;
    });
}

hf_status hf_chain_exchange_floor(hf_ctx *ctx, int nctas, int nthreads, int steps, double *us_per_step_host) {
    if (!ctx || !us_per_step_host || nctas < 1 || steps < 1) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] { *us_per_step_host = hf::chain_exchange_floor(ctx, nctas, nthreads, steps); });
}

hf_status hf_launch_count(const hf_ctx *ctx, int64_t *launches_host) {
    if (!ctx || !launches_host) return HF_ERR_INVALID_ARG;
    *launches_host = ctx->launches;
    return HF_OK;
}

// ------------------------------------------------------------------ a1
// The lower triangle of a host Kbar moves in column panels of 256: one 2D copy per panel
// (rows j0..L-1 of columns j0..j0+255), so the bytes on the host link are L^2/2 x 8 plus the
// panels' diagonal blocks; the upper triangle, which hf_scale never reads, stays on the host.
static int64_t copy_lower_panels(cudaStream_t st, int64_t L, const double *Kh, int64_t ldh, double *K, int64_t ld) {
    constexpr int64_t W = 256;
    int64_t bytes = 0;
    for (int64_t j0 = 0; j0 < L; j0 += W) {
        const int64_t w = std::min<int64_t>(W, L - j0);
        HF_CUDA(cudaMemcpy2DAsync(K + j0 + j0 * ld, (size_t)ld * sizeof(double), Kh + j0 + j0 * ldh,
                                  (size_t)ldh * sizeof(double), (size_t)(L - j0) * sizeof(double), (size_t)w,
                                  cudaMemcpyHostToDevice, st));
        bytes += (L - j0) * w * (int64_t)sizeof(double);
    }
    return bytes;
}

// the context stream waits for the uploads issued so far (hf_upload_lower)
static void order_after_uploads(hf_ctx *ctx) {
    if (!ctx->up_pending) return;
    HF_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->up_ev, 0));
    ctx->up_pending = false;
}

static void scale_checked(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q, const char *who) {
    hf::DBuf<int> bad;
    bad.alloc(1, ctx->stream);
    bad.zero(ctx->stream);
    hf::launch_scale(ctx, L, K, ld, q, bad.p);
    int hb = 0;
    HF_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    HF_CUDA(cudaStreamSynchronize(ctx->stream));
    HF_REQUIRE(!hb, std::string(who) + ": K holds NaN or Inf");
}

hf_status hf_scale(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q) {
    if (!ctx) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ld >= L && (L == 0 || (K && q)), "hf_scale: bad arguments");
        if (L == 0) return;
        order_after_uploads(ctx);
        scale_checked(ctx, L, K, ld, q, "hf_scale");
    });
}

hf_status hf_scale_host(hf_ctx *ctx, int64_t L, const double *Kbar_host, int64_t ldh, double *K, int64_t ld,
                        double *q, int64_t *h2d_bytes_host) {
    if (!ctx) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ldh >= L && ld >= L && (L == 0 || (Kbar_host && K && q)), "hf_scale_host: bad arguments");
        if (h2d_bytes_host) *h2d_bytes_host = 0;
        if (L == 0) return;
        order_after_uploads(ctx);
        const int64_t bytes = copy_lower_panels(ctx->stream, L, Kbar_host, ldh, K, ld);
        scale_checked(ctx, L, K, ld, q, "hf_scale_host");
        if (h2d_bytes_host) *h2d_bytes_host = bytes;
    });
}

hf_status hf_upload_lower(hf_ctx *ctx, int64_t L, const double *Kbar_host, int64_t ldh, double *K, int64_t ld,
                          int64_t *h2d_bytes_host) {
    if (!ctx) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ldh >= L && ld >= L && (L == 0 || (Kbar_host && K)), "hf_upload_lower: bad arguments");
        if (h2d_bytes_host) *h2d_bytes_host = 0;
        if (L == 0) return;
        if (!ctx->up) {
            HF_CUDA(cudaStreamCreateWithFlags(&ctx->up, cudaStreamNonBlocking));
            HF_CUDA(cudaEventCreateWithFlags(&ctx->up_ev, cudaEventDisableTiming));
        }
        const int64_t bytes = copy_lower_panels(ctx->up, L, Kbar_host, ldh, K, ld);
        HF_CUDA(cudaEventRecord(ctx->up_ev, ctx->up));
        ctx->up_pending = true;
        if (h2d_bytes_host) *h2d_bytes_host = bytes;
    });
}

hf_status hf_matvec(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const double *W, int64_t ldw, int64_t n,
                    double *Z, int64_t ldz, int32_t matvec, int32_t slices) {
    if (!ctx) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && n >= 0 && ld >= L && ldw >= L && ldz >= L && matvec >= 1 && matvec <= 3 &&
                       (slices == 0 || (slices >= 2 && slices <= 9)) && (L == 0 || n == 0 || (K && W && Z)),
                   "hf_matvec: bad arguments");
        if (L == 0 || n == 0) return;
        if (matvec == 1) {
            hf::DBuf<double> work;
            hf::dgemm(ctx, false, L, n, L, 1.0, K, ld, W, ldw, 0.0, Z, ldz, nullptr, &work);
        } else if (matvec == 2) {
            hf::Ozaki oz;
            hf::ozaki_prepare(ctx, oz, K, ld, L, nullptr, slices > 0 ? slices : hf::ozaki_slices(), n);
            hf::ozaki_matvec(ctx, oz, W, ldw, n, Z, ldz, 0.0, 1.0);
        } else {
            hf::Ozaki2 oz;
            hf::ozaki2_prepare(ctx, oz, K, ld, L, nullptr, n);
            hf::ozaki2_matvec(ctx, oz, W, ldw, n, Z, ldz, 0.0, 1.0);
        }
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

hf_status hf_scale_full(hf_ctx *ctx, int64_t L, double *K, int64_t ld, double *q) {
    if (!ctx) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ld >= L && (L == 0 || (K && q)), "hf_scale_full: bad arguments");
        if (L == 0) return;
        hf::DBuf<int> bad;
        bad.alloc(1, ctx->stream);
        bad.zero(ctx->stream);
        hf::launch_scale_full(ctx, L, K, ld, q, bad.p);
        int hb = 0;
        HF_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
        HF_REQUIRE(!hb, "hf_scale_full: K holds NaN or Inf");
    });
}

// ------------------------------------------------------------------ a2-a3
hf_status hf_factor_lowprec(hf_ctx *ctx, int64_t L, const double *K, int64_t ld,
                            const hf_lowprec_opts *opts, hf_lowfactor **out, int64_t *N_host,
                            int64_t *n2_host, int64_t *n2_tau_only_host) {
    if (!ctx || !out) return HF_ERR_INVALID_ARG;
    *out = nullptr;
    hf_lowprec_opts o{1e-2, 0, 0, 0, 32, 0};
    if (opts) o = *opts;
    if (o.prec == 0) o.prec = 32;
    std::unique_ptr<hf_lowfactor> lf(new hf_lowfactor());
    hf_status s = guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ld >= L && (L == 0 || K), "hf_factor_lowprec: bad arguments");
        HF_REQUIRE(o.tau > 0.0 && o.tau < 1.0, "hf_factor_lowprec: tau must lie in (0,1)");
        HF_REQUIRE(o.n_extra >= 0 && o.n_min >= 0, "hf_factor_lowprec: n_extra/n_min < 0");
        HF_REQUIRE(o.nb >= 0 && o.nb <= 256 && o.nb % 8 == 0, "hf_factor_lowprec: nb in {0, 8..256, multiple of 8}");
        HF_REQUIRE(o.prec == 32 || o.prec == 64, "hf_factor_lowprec: prec must be 32 or 64");
        if (o.nonsym) {
            HF_REQUIRE(o.prec == 32, "hf_factor_lowprec: the nonsymmetric LDU is FP32 only");
            HF_REQUIRE(ctx->nranks == 1 && ctx->s1parts == 0, "hf_factor_lowprec: the nonsymmetric LDU is single-GPU");
            hf::lowprec_factor_ns(ctx, L, K, ld, o, lf.get());
        } else if (o.prec == 64) {
            HF_REQUIRE(ctx->nranks == 1 && ctx->s1parts == 0, "hf_factor_lowprec: prec 64 is single-GPU");
            hf::lowprec_factor64(ctx, L, K, ld, o, lf.get());
        } else if (ctx->nranks > 1) hf::lowprec_factor_dist(ctx, L, K, ld, o, lf.get(), ctx->nranks);
        else if (ctx->s1parts > 0) hf::lowprec_factor_dist(ctx, L, K, ld, o, lf.get(), ctx->s1parts);
        else hf::lowprec_factor(ctx, L, K, ld, o, lf.get());
    });
    if (s != HF_OK) return s;
    if (N_host) *N_host = lf->N;
    if (n2_host) *n2_host = lf->n2;
    if (n2_tau_only_host) *n2_tau_only_host = lf->L - lf->Ntau;
    *out = lf.release();
    return HF_OK;
}

hf_status hf_lowfactor_export(hf_ctx *ctx, const hf_lowfactor *lf, int64_t *perm_host, float *D_host,
                              float *Lfac, int64_t ldl) {
    if (!ctx || !lf) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        if (perm_host && lf->L) std::memcpy(perm_host, lf->h_perm.data(), lf->L * sizeof(int64_t));
        if (D_host && lf->N) std::memcpy(D_host, lf->h_D.data(), lf->N * sizeof(float));
        if (Lfac && lf->N) {
            HF_REQUIRE(ldl >= lf->N, "hf_lowfactor_export: ldl < N");
            HF_CUDA(cudaMemcpy2DAsync(Lfac, ldl * sizeof(float), lf->Lfac.p, lf->N * sizeof(float),
                                      lf->N * sizeof(float), lf->N, cudaMemcpyDeviceToDevice, ctx->stream));
        }
    });
}

hf_status hf_nd_blocks(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, int32_t levels, int32_t min_size,
                       int32_t *blk_host, int32_t *nblk_host) {
    if (!ctx || !blk_host || !nblk_host) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ld >= L && (L == 0 || K) && levels >= 1 && levels <= 30 && min_size >= 1,
                   "hf_nd_blocks: bad arguments");
        hf::nd_blocks(ctx, L, K, ld, levels, min_size, blk_host, nblk_host);
    });
}

hf_status hf_factor_lowprec_blocks(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, const hf_lowprec_opts *opts,
                                   const int32_t *blk_host, int32_t nblk, hf_lowfactor **out, int64_t *N_host,
                                   int64_t *n2_host, int64_t *n2_tau_only_host) {
    if (!ctx || !out || (L > 0 && !blk_host)) return HF_ERR_INVALID_ARG;
    *out = nullptr;
    hf_lowprec_opts o{1e-2, 0, 0, 0, 32, 0};
    if (opts) o = *opts;
    if (o.prec == 0) o.prec = 32;
    std::unique_ptr<hf_lowfactor> lf(new hf_lowfactor());
    hf_status s = guarded(ctx, [&] {
        HF_REQUIRE(L >= 0 && ld >= L && (L == 0 || K), "hf_factor_lowprec_blocks: bad arguments");
        HF_REQUIRE(o.tau > 0.0 && o.tau < 1.0, "hf_factor_lowprec_blocks: tau must lie in (0,1)");
        HF_REQUIRE(o.n_extra >= 0 && o.n_min >= 0, "hf_factor_lowprec_blocks: n_extra/n_min < 0");
        HF_REQUIRE(o.nb >= 0 && o.nb <= 256 && o.nb % 8 == 0, "hf_factor_lowprec_blocks: nb in {0, 8..256, multiple of 8}");
        HF_REQUIRE(o.prec == 32 && !o.nonsym, "hf_factor_lowprec_blocks: FP32 symmetric only");
        HF_REQUIRE(ctx->nranks == 1 && ctx->s1parts == 0, "hf_factor_lowprec_blocks: single-GPU");
        HF_REQUIRE(nblk >= 0, "hf_factor_lowprec_blocks: nblk < 0");
        for (int64_t i = 0; i < L; ++i)
            HF_REQUIRE(blk_host[i] >= 0 && blk_host[i] < std::max(nblk, 1), "hf_factor_lowprec_blocks: block id out of range");
        hf::lowprec_factor(ctx, L, K, ld, o, lf.get(), blk_host, nblk);
    });
    if (s != HF_OK) return s;
    if (N_host) *N_host = lf->N;
    if (n2_host) *n2_host = lf->n2;
    if (n2_tau_only_host) *n2_tau_only_host = lf->L - lf->Ntau;
    *out = lf.release();
    return HF_OK;
}

hf_status hf_lowfactor_export_u(hf_ctx *ctx, const hf_lowfactor *lf, float *Ufac, int64_t ldu) {
    if (!ctx || !lf) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        if (!lf->nonsym) throw hf::Error{HF_ERR_STATE, "hf_lowfactor_export_u: not a nonsymmetric (LDU) factor"};
        if (Ufac && lf->N) {
            HF_REQUIRE(ldu >= lf->N, "hf_lowfactor_export_u: ldu < N");
            HF_CUDA(cudaMemcpy2DAsync(Ufac, ldu * sizeof(float), lf->Ufac.p, lf->N * sizeof(float),
                                      lf->N * sizeof(float), lf->N, cudaMemcpyDeviceToDevice, ctx->stream));
            HF_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    });
}

hf_status hf_lowfactor_export64(hf_ctx *ctx, const hf_lowfactor *lf, int64_t *perm_host, double *D_host,
                                double *Lfac, int64_t ldl) {
    if (!ctx || !lf) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        if (lf->prec != 64) throw hf::Error{HF_ERR_STATE, "hf_lowfactor_export64: not a prec-64 factor"};
        if (perm_host && lf->L) std::memcpy(perm_host, lf->h_perm.data(), lf->L * sizeof(int64_t));
        if (D_host && lf->N) std::memcpy(D_host, lf->h_D64.data(), lf->N * sizeof(double));
        if (Lfac && lf->N) {
            HF_REQUIRE(ldl >= lf->N, "hf_lowfactor_export64: ldl < N");
            HF_CUDA(cudaMemcpy2DAsync(Lfac, ldl * sizeof(double), lf->Lfac64.p, lf->N * sizeof(double),
                                      lf->N * sizeof(double), lf->N, cudaMemcpyDeviceToDevice, ctx->stream));
            HF_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    });
}

hf_status hf_lowfactor_destroy(hf_lowfactor *lf) {
    if (lf) {
        cudaStreamSynchronize(lf->stream);
        delete lf;
    }
    return HF_OK;
}

// ------------------------------------------------------------------ a5 preconditioner
hf_status hf_precond_apply(hf_ctx *ctx, const hf_lowfactor *lf, int64_t ncol, const double *R, int64_t ldr,
                           double *W, int64_t ldw) {
    if (!ctx || !lf) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(ncol >= 0 && ldr >= lf->L && ldw >= lf->L && (ncol == 0 || lf->L == 0 || (R && W)),
                   "hf_precond_apply: bad arguments");
        if (ncol == 0 || lf->L == 0) return;
        hf::Precond pc;
        hf::precond_setup(ctx, pc, lf);
        hf::precond_apply(ctx, pc, ncol, R, ldr, W, ldw);
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

hf_status hf_gram_inverse(hf_ctx *ctx, int64_t n, const double *M, int64_t ldm, double *Minv,
                          int32_t *breakdown_host) {
    if (!ctx || !breakdown_host) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(n >= 0 && ldm >= std::max<int64_t>(n, 1) && (n == 0 || (M && Minv)), "hf_gram_inverse: bad arguments");
        *breakdown_host = 0;
        if (n == 0) return;
        hf::DBuf<double> wk, dg;
        hf::DBuf<int> st;
        st.alloc(1, ctx->stream);
        st.zero(ctx->stream);
        hf::spd_inverse(ctx, n, M, ldm, Minv, wk, dg, st.p);
        int h = 0;
        HF_CUDA(cudaMemcpyAsync(&h, st.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
        *breakdown_host = h ? 1 : 0;
    });
}

// ------------------------------------------------------------------ a4-a6
hf_status hf_schur_gcr(hf_ctx *ctx, const double *K, int64_t ld, const hf_lowfactor *lf,
                       const hf_gcr_opts *opts, hf_hybrid **out, double *S22_host_or_null,
                       hf_gcr_info *info_host) {
    if (!ctx || !lf || !out) return HF_ERR_INVALID_ARG;
    *out = nullptr;
    hf_gcr_opts o{1e-14, 100, 0, 0};
    if (opts) o = *opts;
    hf_gcr_info info{0, 0.0, 0.0, 0};
    std::unique_ptr<hf_hybrid> hy(new hf_hybrid());
    hf_status s = guarded(ctx, [&] {
        HF_REQUIRE(ld >= lf->L && (lf->L == 0 || K), "hf_schur_gcr: bad arguments");

        HF_REQUIRE(o.tol > 0.0 && o.max_iter >= 1, "hf_schur_gcr: tol > 0, max_iter >= 1");
        HF_REQUIRE(o.matvec >= 0 && o.matvec <= 3 && (o.slices == 0 || (o.slices >= 2 && o.slices <= 9)),
                   "hf_schur_gcr: matvec in 0..3, slices 0 or 2..9");
        hy->K = K;
        hy->ld = ld;
        hy->L = lf->L;
        hy->N = lf->N;
        hy->n2 = lf->n2;
        hy->lf = lf;
        hy->stream = ctx->stream;
        hy->num_sms = ctx->num_sms;
        hf::schur_gcr(ctx, hy.get(), o, &info);
        if (S22_host_or_null && hy->n2 > 0) {
            HF_CUDA(cudaMemcpyAsync(S22_host_or_null, hy->S22.p, hy->n2 * hy->n2 * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            HF_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    });
    if (info_host) *info_host = info;
    if (s == HF_OK || s == HF_ERR_NOT_CONVERGED || s == HF_ERR_BREAKDOWN) *out = hy.release();
    return s;
}

hf_status hf_hybrid_export(hf_ctx *ctx, const hf_hybrid *hy, double *X, int64_t ldx, double *S22,
                           int64_t lds);

hf_status hf_schur_gcr_dd(hf_ctx *ctx, const double *K, int64_t ld, const hf_lowfactor *lf,
                          const hf_gcr_opts *opts, hf_hybrid **out, double *S22hi_host_or_null,
                          double *S22lo_host_or_null, hf_gcr_info *info_host) {
    if (!ctx || !lf || !out) return HF_ERR_INVALID_ARG;
    *out = nullptr;
    hf_gcr_opts o{1e-28, 100, 0, 0};
    if (opts) o = *opts;
    hf_gcr_info info{0, 0.0, 0.0, 0};
    std::unique_ptr<hf_hybrid> hy(new hf_hybrid());
    hf_status s = guarded(ctx, [&] {
        HF_REQUIRE(ld >= lf->L && (lf->L == 0 || K), "hf_schur_gcr_dd: bad arguments");
        HF_REQUIRE(o.tol > 0.0 && o.max_iter >= 1, "hf_schur_gcr_dd: tol > 0, max_iter >= 1");
        HF_REQUIRE(lf->prec == 64, "hf_schur_gcr_dd: the factor must be FP64 (hf_factor_lowprec with prec 64)");
        HF_REQUIRE(ctx->nranks <= 1 && ctx->vnranks == 0, "hf_schur_gcr_dd: single-rank only");
        hy->K = K;
        hy->ld = ld;
        hy->L = lf->L;
        hy->N = lf->N;
        hy->n2 = lf->n2;
        hy->lf = lf;
        hy->stream = ctx->stream;
        hy->num_sms = ctx->num_sms;
        hf::schur_gcr_dd(ctx, hy.get(), o, &info);
        const size_t bytes = (size_t)hy->n2 * hy->n2 * sizeof(double);
        if (S22hi_host_or_null && hy->n2 > 0)
            HF_CUDA(cudaMemcpyAsync(S22hi_host_or_null, hy->S22.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        if (S22lo_host_or_null && hy->n2 > 0)
            HF_CUDA(cudaMemcpyAsync(S22lo_host_or_null, hy->S22lo.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
    });
    if (info_host) *info_host = info;
    if (s == HF_OK || s == HF_ERR_NOT_CONVERGED || s == HF_ERR_BREAKDOWN) *out = hy.release();
    return s;
}

hf_status hf_solve_dd(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *xhi, double *xlo,
                      hf_gcr_info *info_host) {
    if (!ctx || !hy || !b || !xhi || !xlo) return HF_ERR_INVALID_ARG;
    hf_gcr_info info{0, 0.0, 0.0, 0};
    hf_status s = guarded(ctx, [&] {
        if (!hy->dd) throw hf::Error{HF_ERR_STATE, "hf_solve_dd: not a double-double hybrid"};
        if (!hy->hard_done && hy->n2 > 0) throw hf::Error{HF_ERR_STATE, "hf_solve_dd: call hf_factor_hard first"};
        hf_gcr_opts o{1e-28, 100, 0, 0};
        hf::hybrid_solve_dd(ctx, hy, b, xhi, xlo, o, &info);
    });
    if (info_host) *info_host = info;
    return s;
}

hf_status hf_hybrid_export_dd(hf_ctx *ctx, const hf_hybrid *hy, double *Xhi, double *Xlo, int64_t ldx,
                              double *S22hi, double *S22lo, int64_t lds) {
    if (!ctx || !hy) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        if (!hy->dd) throw hf::Error{HF_ERR_STATE, "hf_hybrid_export_dd: not a double-double hybrid"};
        const int64_t L = hy->L, n2 = hy->n2;
        HF_REQUIRE(ldx >= L && lds >= n2, "hf_hybrid_export_dd: leading dimensions");
        if (n2 == 0) return;
        cudaStream_t st = ctx->stream;
        if (Xhi) HF_CUDA(cudaMemcpy2DAsync(Xhi, ldx * 8, hy->X.p, L * 8, L * 8, n2, cudaMemcpyDeviceToDevice, st));
        if (Xlo) HF_CUDA(cudaMemcpy2DAsync(Xlo, ldx * 8, hy->Xlo.p, L * 8, L * 8, n2, cudaMemcpyDeviceToDevice, st));
        if (S22hi) HF_CUDA(cudaMemcpy2DAsync(S22hi, lds * 8, hy->S22.p, n2 * 8, n2 * 8, n2, cudaMemcpyDeviceToDevice, st));
        if (S22lo) HF_CUDA(cudaMemcpy2DAsync(S22lo, lds * 8, hy->S22lo.p, n2 * 8, n2 * 8, n2, cudaMemcpyDeviceToDevice, st));
        HF_CUDA(cudaStreamSynchronize(st));
    });
}

hf_status hf_factor_hard(hf_ctx *ctx, hf_hybrid *hy, double eps_ker, int64_t *kernel_dim_host) {
    if (!ctx || !hy) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        HF_REQUIRE(eps_ker >= 0.0, "hf_factor_hard: eps_ker < 0");
        if (hy->dd) hf::factor_hard_dd(ctx, hy, eps_ker);
        else hf::factor_hard(ctx, hy, eps_ker);
        if (kernel_dim_host) *kernel_dim_host = hy->kernel_dim;
    });
}

hf_status hf_hard_export(hf_ctx *ctx, const hf_hybrid *hy, int64_t *perm2_host, int32_t *blocks_host,
                         int64_t *rank_host) {
    if (!ctx || !hy) return HF_ERR_INVALID_ARG;
    return guarded(ctx, [&] {
        if (!hy->hard_done) throw hf::Error{HF_ERR_STATE, "hf_hard_export: call hf_factor_hard first"};
        const int64_t n2 = hy->n2;
        if (rank_host) *rank_host = hy->rank;
        if (n2 == 0) return;
        std::vector<int32_t> p(n2), b(n2);
        HF_CUDA(cudaMemcpyAsync(p.data(), hy->perm2.p, n2 * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        HF_CUDA(cudaMemcpyAsync(b.data(), hy->blocks.p, n2 * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        HF_CUDA(cudaStreamSynchronize(ctx->stream));
        if (perm2_host)
            for (int64_t i = 0; i < n2; ++i) perm2_host[i] = p[i];
        if (blocks_host) std::memcpy(blocks_host, b.data(), n2 * sizeof(int32_t));
    });
}

hf_status hf_solve(hf_ctx *ctx, const hf_hybrid *hy, const double *b, double *x, hf_gcr_info *info_host) {
    if (!ctx || !hy || !b || !x) return HF_ERR_INVALID_ARG;
    hf_gcr_info info{0, 0.0, 0.0, 0};
    hf_status s = guarded(ctx, [&] {
        if (!hy->hard_done && hy->n2 > 0)
            throw hf::Error{HF_ERR_STATE, "hf_solve: call hf_factor_hard first"};
        if (hy->dd) throw hf::Error{HF_ERR_STATE, "hf_solve: a double-double hybrid is solved by hf_solve_dd"};
        hf_gcr_opts o{1e-14, 100, 0, 0};
        hf::hybrid_solve(ctx, hy, b, x, o, &info);
    });
    if (info_host) *info_host = info;
    return s;
}

hf_status hf_hybrid_destroy(hf_hybrid *hy) {
    if (hy) {
        cudaStreamSynchronize(hy->stream);
        delete hy;
    }
    return HF_OK;
}

}  // extern "C"
