// alloc.cu -- the library's device-memory cache.
//
// Every workspace and handle buffer of libhf (DBuf) comes from here.  Freed
// blocks are kept per (device, stream) and handed out again, in stream order,
// to later requests of (nearly) the same size, so a repeated factorization
// maps no new memory: at C2 one step touches ~10 GB of workspaces, and
// re-mapping that through cudaMalloc / the driver pool on every call cost more
// than the factorization itself.  On cudaErrorMemoryAllocation the cache is
// trimmed (device synchronised, cached blocks freed) and the request retried
// once.  At most HF_CACHE_FRACTION (default 0.4) of the device is kept
// cached, so the caller's own allocator (torch) keeps room; hf_trim_cache()
// (include/hf.h) releases everything cached.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "hf_internal.cuh"

namespace hf {
namespace {

struct Live {
    size_t bytes;
    int dev;
};

struct Cache {
    std::mutex mu;
    std::map<int, size_t> cap;   // per device: max bytes kept cached (HF_CACHE_FRACTION of the device, 0.4)
    std::map<std::pair<int, cudaStream_t>, std::multimap<size_t, void *>> free_;
    std::unordered_map<void *, Live> live;
    size_t cached_bytes = 0;
};

Cache &cache() {
    static Cache *c = new Cache();   // never destroyed: frees may run at process exit
    return *c;
}

size_t round_bytes(size_t b) {
    if (b == 0) b = 1;
    if (b < ((size_t)1 << 20)) return (b + 511) & ~(size_t)511;
    return (b + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
}

void trim_device(int dev) {
    Cache &c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    for (auto it = c.free_.begin(); it != c.free_.end();) {
        if (it->first.first == dev) {
            for (auto &kv : it->second) {
                cudaFree(kv.second);
                c.cached_bytes -= kv.first;
            }
            it = c.free_.erase(it);
        } else {
            ++it;
        }
    }
    cudaSetDevice(cur);
}

}  // namespace

void host_trace(const char *where) {
    static const double thr = getenv("HF_TRACE_HOST") ? atof(getenv("HF_TRACE_HOST")) : -1.0;
    if (thr < 0.0) return;
    static auto last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - last).count();
    if (ms > thr) fprintf(stderr, "[hf host] %.3f ms before %s\n", ms, where);
    last = now;
}

void *dev_alloc(size_t bytes, cudaStream_t s) {
    int dev = 0;
    HF_CUDA(cudaGetDevice(&dev));
    const size_t want = round_bytes(bytes);
    Cache &c = cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto f = c.free_.find({dev, s});
        if (f != c.free_.end()) {
            auto it = f->second.lower_bound(want);
            // best fit, at most 25% (or 2 MB) larger than asked
            if (it != f->second.end() && it->first <= want + std::max(want / 4, ((size_t)2 << 20))) {
                void *p = it->second;
                c.cached_bytes -= it->first;
                c.live[p] = Live{it->first, dev};
                f->second.erase(it);
                return p;
            }
        }
    }
    void *p = nullptr;
    static const bool dbg = getenv("HF_ALLOC_DEBUG") != nullptr;
    if (dbg) fprintf(stderr, "[hf alloc] cudaMalloc %zu bytes (cached %zu)\n", want, c.cached_bytes);
    host_trace("cudaMalloc call");
    cudaError_t e = cudaMalloc(&p, want);
    host_trace("cudaMalloc");
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        trim_device(dev);
        e = cudaMalloc(&p, want);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error{e == cudaErrorMemoryAllocation ? HF_ERR_OOM : HF_ERR_CUDA,
                    std::string("device allocation of ") + std::to_string(want) + " bytes: " + cudaGetErrorString(e)};
    }
    std::lock_guard<std::mutex> g(c.mu);
    c.live[p] = Live{want, dev};
    return p;
}

void dev_free(void *p, cudaStream_t s) {
    if (!p) return;
    Cache &c = cache();
    std::unique_lock<std::mutex> g(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;
    const Live l = it->second;
    c.live.erase(it);
    auto ci = c.cap.find(l.dev);
    if (ci == c.cap.end()) {
        size_t fr = 0, tot = 0;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(l.dev);
        cudaMemGetInfo(&fr, &tot);
        cudaSetDevice(cur);
        double f = 0.4;
        if (const char *e = getenv("HF_CACHE_FRACTION")) f = atof(e);
        ci = c.cap.emplace(l.dev, (size_t)(f * (double)tot)).first;
    }
    if (c.cached_bytes + l.bytes > ci->second) {
        // over the cap: give the block back (cudaFree synchronises; only past the cap)
        g.unlock();
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(l.dev);
        host_trace("over-cap free");
        cudaStreamSynchronize(s);
        cudaFree(p);
        host_trace("over-cap free done");
        cudaSetDevice(cur);
        return;
    }
    c.free_[{l.dev, s}].insert({l.bytes, p});
    c.cached_bytes += l.bytes;
}

// bytes the cache holds free (reusable, or returned to the driver on an OOM retry) on a device
size_t cached_free_bytes(int dev) {
    Cache &c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    size_t b = 0;
    for (auto &kv : c.free_)
        if (kv.first.first == dev)
            for (auto &e : kv.second) b += e.first;
    return b;
}

}  // namespace hf

extern "C" hf_status hf_trim_cache(int device) {
    hf::trim_device(device);
    return cudaGetLastError() == cudaSuccess ? HF_OK : HF_ERR_CUDA;
}
