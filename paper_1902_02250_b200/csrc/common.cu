// common.cu -- error plumbing and stream-ordered buffers of libkitc.so.
#include <cstdio>
#include <atomic>
#include <cstring>

#include "kitc_internal.cuh"

namespace kitc {

static thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};

kitc_status set_error(kitc_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

kitc_status check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return KITC_OK;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return set_error(KITC_ENOMEM, std::string("CUDA out of memory in ") + what);
    }
    return set_error(KITC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Keep freed pool memory cached so per-step rebuilds do not return memory to
// the driver (stream-ordered allocator, default pool of the current device).
static void retain_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

kitc_status DevBuf::ensure(size_t need, cudaStream_t s, bool keep) {
    if (need <= bytes) return KITC_OK;
    retain_pool();
    size_t nb = need + need / 4 + 256;
    void* np = nullptr;
    KITC_CUDA(cudaMallocAsync(&np, nb, s));
    if (keep && p && bytes) KITC_CUDA(cudaMemcpyAsync(np, p, bytes, cudaMemcpyDeviceToDevice, s));
    if (p) KITC_CUDA(cudaFreeAsync(p, s));
    p = np;
    bytes = nb;
    return KITC_OK;
}

void DevBuf::release(cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
}

kitc_status HostBuf::ensure(size_t need) {
    if (need <= bytes) return KITC_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    size_t nb = need + need / 2 + 4096;
    KITC_CUDA(cudaMallocHost(&p, nb));
    bytes = nb;
    return KITC_OK;
}

void HostBuf::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
}

}  // namespace kitc

extern "C" const char* kitc_last_error(void) { return kitc::g_last_error.c_str(); }

extern "C" uint64_t kitc_launch_count(void) { return kitc::g_launches.load(); }
