// ez_util.cpp — error reporting and small library-level entry points.
#include <cstdint>
#include <mutex>
#include <string>

#include "ez_common.h"

namespace ez {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int32_t fail(int32_t status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

int32_t cuda_fail(cudaError_t err, const char* what, const char* file, int line) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(err) + " (" +
                   cudaGetErrorString(err) + ") at " + file + ":" + std::to_string(line);
    return EZ_CUDA_ERROR;
}

// The library's short-lived scratch comes from the device's default
// stream-ordered pool.  With the default release threshold (0) the pool
// hands memory back at every synchronisation and the next cudaMallocAsync
// maps it again (measured 3-7 ms per call on B200); keep it cached instead.
int32_t retain_async_pool() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail(cudaGetLastError(), "cudaGetDevice", __FILE__, __LINE__);
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev & 63]) return EZ_OK;
    cudaMemPool_t pool;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, dev);
    uint64_t keep = UINT64_MAX;
    if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e != cudaSuccess) return cuda_fail(e, "default mem pool release threshold", __FILE__, __LINE__);
    done[dev & 63] = true;
    return EZ_OK;
}

}  // namespace ez

extern "C" {

int32_t ez_abi_version(void) { return EZ_ABI_VERSION; }

const char* ez_last_error(void) { return ez::g_last_error.c_str(); }

int32_t ez_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // extern "C"
