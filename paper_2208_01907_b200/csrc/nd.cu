// nd.cu -- NEXT-4: the nested-dissection ordering of the
// multi-block postponing of sec. 2.2 ("Lambda is decomposed into
// 2^m - 1 sub-indices with m-level bi-section tree").
//
// The symmetric sparsity pattern of K (device, column-major, symmetric) is
// extracted on the GPU as CSR rows (one warp per row, ballot compaction, so
// every row's columns come out in ascending order) and copied to the host;
// the bisection is a plain host graph algorithm (the library's "graph
// builder"):
//   for a block S (ascending original indices) at depth < m - 1 with
//   |S| > min_size: BFS in the graph restricted to S from its smallest index;
//   u = the smallest index of the last BFS level; the levels V_0..V_h of a BFS
//   from u.  h < 2: leaf.  Otherwise separator V_mid, mid = (h + 1) / 2,
//   S1 = V_0 .. V_{mid-1}, S2 = the rest of S (later levels and every index
//   the BFS did not reach).  Blocks numbered in post-order: S1's, S2's, then
//   the separator.
// (Written from the paper's description, independently of the oracle's
// Python version; tests compare the two index for index.)
#include <algorithm>
#include <functional>
#include <vector>

#include "hf_internal.cuh"

namespace hf {
namespace {

// count the off-diagonal nonzeros of every row (one warp per row)
__global__ void k_row_nnz(int64_t L, const double *__restrict__ K, int64_t ld, int32_t *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= L) return;
    int c = 0;
    for (int64_t j = lane; j < L; j += 32) c += (j != row && K[row + j * ld] != 0.0) ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[row] = c;
}

// write the columns of every row in ascending order (warp ballot compaction)
__global__ void k_row_cols(int64_t L, const double *__restrict__ K, int64_t ld, const int64_t *__restrict__ rowptr,
                           int32_t *__restrict__ col) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= L) return;
    int64_t w = rowptr[row];
    for (int64_t j0 = 0; j0 < L; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool nz = j < L && j != row && K[row + j * ld] != 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, nz);
        if (nz) col[w + __popc(m & ((1u << lane) - 1u))] = (int32_t)j;
        w += __popc(m);
    }
}

}  // namespace

void nd_blocks(hf_ctx *ctx, int64_t L, const double *K, int64_t ld, int levels, int min_size, int32_t *blk_host,
               int32_t *nblk_host) {
    cudaStream_t st = ctx->stream;
    if (L == 0) {
        *nblk_host = 0;
        return;
    }
    DBuf<int32_t> cnt;
    cnt.alloc(L, st);
    const unsigned grid = (unsigned)cdiv(L, 8);   // 8 warps per CTA
    k_row_nnz<<<grid, 256, 0, st>>>(L, K, ld, cnt.p);
    HF_CHECK_LAUNCH(ctx);
    std::vector<int32_t> hc(L);
    HF_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, L * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> rowptr(L + 1, 0);
    for (int64_t i = 0; i < L; ++i) rowptr[i + 1] = rowptr[i] + hc[i];
    const int64_t nnz = rowptr[L];
    DBuf<int64_t> rp;
    rp.alloc(L + 1, st);
    DBuf<int32_t> cols;
    cols.alloc(std::max<int64_t>(nnz, 1), st);
    HF_CUDA(cudaMemcpyAsync(rp.p, rowptr.data(), (L + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    k_row_cols<<<grid, 256, 0, st>>>(L, K, ld, rp.p, cols.p);
    HF_CHECK_LAUNCH(ctx);
    std::vector<int32_t> col(std::max<int64_t>(nnz, 1));
    HF_CUDA(cudaMemcpyAsync(col.data(), cols.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HF_CUDA(cudaStreamSynchronize(st));

    // recursive level-structure bisection
    std::vector<int32_t> blk(L, -1), mark(L, 0), dist(L, -1);
    int32_t counter = 0, epoch = 0;
    auto emit = [&](const std::vector<int32_t> &S) {
        for (int32_t i : S) blk[i] = counter;
        ++counter;
    };
    // BFS within the members marked with the current epoch; returns the levels
    auto bfs = [&](int32_t start, int ep, std::vector<std::vector<int32_t>> &lv) {
        lv.clear();
        std::vector<int32_t> front{start}, touched{start};
        dist[start] = 0;
        while (!front.empty()) {
            std::sort(front.begin(), front.end());
            lv.push_back(front);
            std::vector<int32_t> nxt;
            for (int32_t v : front)
                for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
                    const int32_t w = col[e];
                    if (mark[w] == ep && dist[w] < 0) {
                        dist[w] = (int32_t)lv.size();
                        nxt.push_back(w);
                        touched.push_back(w);
                    }
                }
            front.swap(nxt);
        }
        for (int32_t v : touched) dist[v] = -1;
    };
    std::function<void(std::vector<int32_t> &, int)> rec = [&](std::vector<int32_t> &S, int depth) {
        if (depth >= levels - 1 || (int64_t)S.size() <= min_size) {
            emit(S);
            return;
        }
        const int ep = ++epoch;
        for (int32_t i : S) mark[i] = ep;
        std::vector<std::vector<int32_t>> lv;
        bfs(S[0], ep, lv);
        const int32_t u = lv.back()[0];
        bfs(u, ep, lv);
        const int h = (int)lv.size() - 1;
        if (h < 2) {
            emit(S);
            return;
        }
        const int mid = (h + 1) / 2;
        std::vector<int32_t> sep = lv[mid], S1, S2;
        const int ep2 = ++epoch;   // "seen" marks
        for (int q = 0; q <= h; ++q)
            for (int32_t v : lv[q]) mark[v] = ep2;
        for (int q = 0; q < mid; ++q) S1.insert(S1.end(), lv[q].begin(), lv[q].end());
        for (int q = mid + 1; q <= h; ++q) S2.insert(S2.end(), lv[q].begin(), lv[q].end());
        for (int32_t v : S)
            if (mark[v] != ep2) S2.push_back(v);
        std::sort(S1.begin(), S1.end());
        std::sort(S2.begin(), S2.end());
        rec(S1, depth + 1);
        if (!S2.empty()) rec(S2, depth + 1);
        emit(sep);
    };
    std::vector<int32_t> all(L);
    for (int64_t i = 0; i < L; ++i) all[i] = (int32_t)i;
    rec(all, 0);
    for (int64_t i = 0; i < L; ++i) blk_host[i] = blk[i];
    *nblk_host = counter;
}

}  // namespace hf
