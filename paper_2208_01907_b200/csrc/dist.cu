// dist.cu -- NCCL bootstrap for multi-GPU contexts (one process per GPU).
#include <cstring>
#include <memory>

#include "hf_internal.cuh"

#define HF_NCCL(call)                                                                      \
    do {                                                                                   \
        ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess)                                                             \
            throw ::hf::Error{HF_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
    } while (0)

namespace hf {

// contiguous balanced column slices: rank r owns [r n2 / G, (r+1) n2 / G)
void shard_cols(int64_t n2, int nranks, int rank, int64_t *c0, int64_t *c1) {
    if (nranks <= 1) {
        *c0 = 0;
        *c1 = n2;
        return;
    }
    *c0 = (n2 * rank) / nranks;
    *c1 = (n2 * (rank + 1)) / nranks;
}

#ifdef HF_WITH_NCCL
void collective_begin(hf_ctx *) { HF_NCCL(ncclGroupStart()); }
void collective_end(hf_ctx *) { HF_NCCL(ncclGroupEnd()); }
void collective_bcast(hf_ctx *ctx, double *buf, size_t count, int root) {
    HF_NCCL(ncclBroadcast(buf, buf, count, ncclDouble, root, ctx->comm, ctx->stream));
}
void collective_max(hf_ctx *ctx, double *buf, size_t count) {
    HF_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclMax, ctx->comm, ctx->stream));
}
void collective_allgather_bytes(hf_ctx *ctx, const void *send, void *recv, size_t bytes) {
    HF_NCCL(ncclAllGather(send, recv, bytes, ncclChar, ctx->comm, ctx->stream));
}
// stream-ordered barrier over the ranks (a 1-int all-reduce)
void collective_barrier(hf_ctx *ctx, int *dev_int) {
    HF_NCCL(ncclAllReduce(dev_int, dev_int, 1, ncclInt, ncclSum, ctx->comm, ctx->stream));
}
#endif

}  // namespace hf

extern "C" {

hf_status hf_shard_cols(int64_t n2, int nranks, int rank, int64_t *c0_host, int64_t *c1_host) {
    if (n2 < 0 || nranks < 1 || rank < 0 || rank >= nranks || !c0_host || !c1_host) return HF_ERR_INVALID_ARG;
    hf::shard_cols(n2, nranks, rank, c0_host, c1_host);
    return HF_OK;
}

hf_status hf_set_virtual_rank(hf_ctx *ctx, int rank, int nranks) {
    if (!ctx || nranks < 0 || (nranks > 0 && (rank < 0 || rank >= nranks))) return HF_ERR_INVALID_ARG;
    ctx->vrank = nranks > 0 ? rank : 0;
    ctx->vnranks = nranks;
    return HF_OK;
}

hf_status hf_stage1_partition(int64_t L, int nparts, int part, int64_t *ncols_host, int64_t *cols_host) {
    if (L < 0 || nparts < 1 || part < 0 || part >= nparts || !ncols_host) return HF_ERR_INVALID_ARG;
    const int64_t CB = 128;   // column block of the partitioned factorization (k_lowprec.cu)
    int64_t n = 0;
    for (int64_t j = 0; j < L; ++j)
        if ((j / CB) % nparts == part) {
            if (cols_host) cols_host[n] = j;
            ++n;
        }
    *ncols_host = n;
    return HF_OK;
}

hf_status hf_set_stage1_partitions(hf_ctx *ctx, int nparts) {
    if (!ctx || nparts < 0 || nparts > 1024) return HF_ERR_INVALID_ARG;
    ctx->s1parts = nparts;
    return HF_OK;
}

hf_status hf_nccl_unique_id(void *id128_host) {
    if (!id128_host) return HF_ERR_INVALID_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return HF_ERR_NCCL;
    std::memcpy(id128_host, &id, sizeof(id));
    return HF_OK;
}

hf_status hf_create_dist(int device, void *cuda_stream, const void *nccl_unique_id128, int rank,
                         int nranks, hf_ctx **out) {
    if (!out || !nccl_unique_id128 || nranks < 1 || rank < 0 || rank >= nranks) return HF_ERR_INVALID_ARG;
    hf_status s = hf_create(device, cuda_stream, out);
    if (s != HF_OK) return s;
    hf_ctx *c = *out;
    try {
        ncclUniqueId id;
        std::memcpy(&id, nccl_unique_id128, sizeof(id));
        HF_NCCL(ncclCommInitRank(&c->comm, nranks, id, rank));
        c->rank = rank;
        c->nranks = nranks;
    } catch (const hf::Error &e) {
        c->last_error = e.msg;
        return e.st;
    }
    return HF_OK;
}

}  // extern "C"
