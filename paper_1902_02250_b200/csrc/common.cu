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

// Buffers are retained by their handle across rebuilds and only reallocated when
// they must grow (by 25% + 256 B), so steady-state steps allocate nothing.
size_t dev_alloc_bytes(size_t need) { return (need + need / 4 + 256 + 255) / 256 * 256; }

kitc_status DevBuf::ensure(size_t need, cudaStream_t s, bool keep) {
    if (need <= bytes) return KITC_OK;
    size_t nb = dev_alloc_bytes(need);
    void* np = nullptr;
    if (al && al->alloc) {
        np = al->alloc(nb, (void*)s, al->ctx);
        if (!np) return set_error(KITC_ENOMEM, "kitc_allocator: allocation of " + std::to_string(nb) + " bytes failed");
        if (reinterpret_cast<uintptr_t>(np) % 16) {
            al->release(np, (void*)s, al->ctx);
            return set_error(KITC_EINVAL, "kitc_allocator: pointer not 16-byte aligned");
        }
    } else {
        KITC_CUDA(cudaMallocAsync(&np, nb, s));
    }
    if (keep && p && bytes) KITC_CUDA(cudaMemcpyAsync(np, p, bytes, cudaMemcpyDeviceToDevice, s));
    release(s);
    p = np;
    bytes = nb;
    return KITC_OK;
}

void DevBuf::release(cudaStream_t s) {
    if (p) {
        if (al && al->alloc)
            al->release(p, (void*)s, al->ctx);
        else
            cudaFreeAsync(p, s);
    }
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

extern "C" uint32_t kitc_build_flags(void) {
#ifdef KITC_CHECKS
    return KITC_BUILD_CHECKS;
#else
    return 0;
#endif
}
