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

extern "C" {

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
