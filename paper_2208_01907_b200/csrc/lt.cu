// lt.cu -- cuBLASLt plumbing of libhf (see lt.cuh).
#include <cublasLt.h>

#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "lt.cuh"

namespace hf {
namespace {

#define HF_CUBLAS(x)                                                                                   \
    do {                                                                                               \
        cublasStatus_t s_ = (x);                                                                       \
        if (s_ != CUBLAS_STATUS_SUCCESS)                                                               \
            throw Error{HF_ERR_CUDA, std::string(#x) + ": cublasLt status " + std::to_string((int)s_)}; \
    } while (0)

struct LtPlan {
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
    cublasLtMatmulAlgo_t algo;
};

// one cuBLASLt handle, workspace and plan cache per device, created on first use and
// kept for the process (never destroyed: no teardown ordering against the CUDA context)
struct LtState {
    cublasLtHandle_t h = nullptr;
    std::map<cudaStream_t, void *> ws;   // one workspace per stream: concurrent GEMMs never share one
    std::map<std::array<int64_t, 14>, LtPlan> plans;
    std::mutex mu;   // guards plans and ws
    void *workspace(cudaStream_t s);
};
constexpr size_t LT_WS = (size_t)32 << 20;

LtState &lt_state(hf_ctx *ctx) {
    static std::mutex mu;
    static LtState *st[256] = {};
    std::lock_guard<std::mutex> g(mu);
    LtState *&s = st[ctx->device % 256];
    if (!s) {
        std::unique_ptr<LtState> n(new LtState());
        HF_CUBLAS(cublasLtCreate(&n->h));
        s = n.release();
    }
    return *s;
}

void *LtState::workspace(cudaStream_t s) {
    auto it = ws.find(s);
    if (it != ws.end()) return it->second;
    void *p = nullptr;
    HF_CUDA(cudaMalloc(&p, LT_WS));
    ws.emplace(s, p);
    return p;
}

cublasLtMatrixLayout_t layout(cudaDataType_t t, int64_t rows, int64_t cols, int64_t ld, int batch, int64_t stride) {
    cublasLtMatrixLayout_t l;
    HF_CUBLAS(cublasLtMatrixLayoutCreate(&l, t, (uint64_t)rows, (uint64_t)cols, ld));
    if (batch > 1) {
        const int32_t b = batch;
        HF_CUBLAS(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &b, sizeof(b)));
        HF_CUBLAS(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &stride,
                                                   sizeof(stride)));
    }
    return l;
}

// plan for key (kind, tA, tB, m, n, k, lda, ldb, ldc, batch, sA, sB, sC, tf32)
const LtPlan &plan(LtState &lt, const std::array<int64_t, 14> &key) {
    auto it = lt.plans.find(key);
    if (it != lt.plans.end()) return it->second;
    const bool imma = key[0] == 1, bf16 = key[0] == 3;
    const bool tA = key[1], tB = key[2];
    const int64_t m = key[3], n = key[4], k = key[5], lda = key[6], ldb = key[7], ldc = key[8];
    const int batch = (int)key[9];
    LtPlan pl;
    if (imma) {
        HF_CUBLAS(cublasLtMatmulDescCreate(&pl.op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
    } else if (bf16) {
        HF_CUBLAS(cublasLtMatmulDescCreate(&pl.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    } else {
        HF_CUBLAS(cublasLtMatmulDescCreate(&pl.op, key[13] ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F_PEDANTIC,
                                           CUDA_R_32F));
    }
    const cublasOperation_t oa = tA ? CUBLAS_OP_T : CUBLAS_OP_N, ob = tB ? CUBLAS_OP_T : CUBLAS_OP_N;
    HF_CUBLAS(cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSA, &oa, sizeof(oa)));
    HF_CUBLAS(cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSB, &ob, sizeof(ob)));
    const cudaDataType_t ti = imma ? CUDA_R_8I : (bf16 ? CUDA_R_16BF : CUDA_R_32F), to = imma ? CUDA_R_32I : CUDA_R_32F;
    pl.la = layout(ti, tA ? k : m, tA ? m : k, lda, batch, key[10]);
    pl.lb = layout(ti, tB ? n : k, tB ? k : n, ldb, batch, key[11]);
    pl.lc = layout(to, m, n, ldc, batch, key[12]);
    cublasLtMatmulPreference_t pref;
    HF_CUBLAS(cublasLtMatmulPreferenceCreate(&pref));
    const size_t wsb = LT_WS;
    HF_CUBLAS(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)));
    cublasLtMatmulHeuristicResult_t res;
    int nres = 0;
    HF_CUBLAS(cublasLtMatmulAlgoGetHeuristic(lt.h, pl.op, pl.la, pl.lb, pl.lc, pl.lc, pref, 1, &res, &nres));
    cublasLtMatmulPreferenceDestroy(pref);
    HF_REQUIRE(nres > 0, "cuBLASLt: no algorithm for this GEMM shape");
    pl.algo = res.algo;
    return lt.plans.emplace(key, pl).first->second;
}

}  // namespace

// the workspace of a stream that is about to be destroyed (hf_destroy: the context's helper
// streams, after they are synchronised); a later stream with the same handle gets a new one
void lt_release_stream(hf_ctx *ctx, cudaStream_t s) {
    LtState &lt = lt_state(ctx);
    std::lock_guard<std::mutex> g(lt.mu);
    auto it = lt.ws.find(s);
    if (it == lt.ws.end()) return;
    cudaFree(it->second);
    lt.ws.erase(it);
}

// library kernels: not counted in ctx->launches (libhf's own launches)
void lt_imma(hf_ctx *ctx, int64_t rows, int64_t cols, int64_t k, const int8_t *A, int64_t lda, const int8_t *B,
             int64_t ldb, int32_t *D, int64_t ldd, int batch, int64_t sA, int64_t sB, int64_t sD) {
    if (rows == 0 || cols == 0 || batch == 0) return;
    LtState &lt = lt_state(ctx);
    std::lock_guard<std::mutex> g(lt.mu);
    const LtPlan &pl = plan(lt, {1, 1, 0, rows, cols, k, lda, ldb, ldd, batch, batch > 1 ? sA : 0,
                                 batch > 1 ? sB : 0, batch > 1 ? sD : 0, 0});
    const int32_t one = 1, zero = 0;
    HF_CUBLAS(cublasLtMatmul(lt.h, pl.op, &one, A, pl.la, B, pl.lb, &zero, D, pl.lc, D, pl.lc, &pl.algo,
                             lt.workspace(ctx->stream), LT_WS, ctx->stream));
}

void lt_sgemm(hf_ctx *ctx, bool tA, bool tB, int64_t m, int64_t n, int64_t k, float alpha, const float *A,
              int64_t lda, int64_t sA, const float *B, int64_t ldb, int64_t sB, float beta, float *C, int64_t ldc,
              int64_t sC, int batch, bool tf32) {
    if (m == 0 || n == 0 || batch == 0) return;
    LtState &lt = lt_state(ctx);
    std::lock_guard<std::mutex> g(lt.mu);
    const LtPlan &pl = plan(lt, {2, tA, tB, m, n, k, lda, ldb, ldc, batch, batch > 1 ? sA : 0,
                                 batch > 1 ? sB : 0, batch > 1 ? sC : 0, tf32 ? 1 : 0});
    HF_CUBLAS(cublasLtMatmul(lt.h, pl.op, &alpha, A, pl.la, B, pl.lb, &beta, C, pl.lc, C, pl.lc, &pl.algo,
                             lt.workspace(ctx->stream), LT_WS, ctx->stream));
}

void lt_bgemm(hf_ctx *ctx, bool tA, int64_t m, int64_t n, int64_t k, float alpha, const __nv_bfloat16 *A,
              int64_t lda, const __nv_bfloat16 *B, int64_t ldb, float beta, float *C, int64_t ldc,
              cudaStream_t st, int batch, int64_t sA, int64_t sB, int64_t sC) {
    if (m == 0 || n == 0 || batch == 0) return;
    if (!st) st = ctx->stream;
    LtState &lt = lt_state(ctx);
    std::lock_guard<std::mutex> g(lt.mu);
    const LtPlan &pl = plan(lt, {3, tA, 0, m, n, k, lda, ldb, ldc, batch, batch > 1 ? sA : 0, batch > 1 ? sB : 0,
                                 batch > 1 ? sC : 0, 0});
    HF_CUBLAS(cublasLtMatmul(lt.h, pl.op, &alpha, A, pl.la, B, pl.lb, &beta, C, pl.lc, C, pl.lc, &pl.algo,
                             lt.workspace(st), LT_WS, st));
}

}  // namespace hf
