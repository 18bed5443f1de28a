// ez_util.cpp — error reporting and small library-level entry points.
#include <immintrin.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

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

// ---------------------------------------------------------------------------
// host_parallel: a small persistent pool for host-side byte moves (pageable
// batches are copied into the pinned staging ring by several threads; one
// thread's memcpy from pageable memory is far below the PCIe rate).
// ---------------------------------------------------------------------------
namespace {
class HostPool {
  public:
    explicit HostPool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
        for (auto& t : th_) t.detach();  // lives for the process (never destroyed)
    }
    int size() const { return static_cast<int>(th_.size()) + 1; }
    void run(int parts, const std::function<void(int)>& f) {
        std::lock_guard<std::mutex> one(run_mu_);  // one job at a time
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &f;
        parts_ = parts;
        next_ = 0;
        remaining_ = parts;
        ++gen_;
        cv_.notify_all();
        drain(lk);  // the caller works too
        done_.wait(lk, [&] { return remaining_ == 0; });
        job_ = nullptr;
    }

  private:
    void drain(std::unique_lock<std::mutex>& lk) {
        while (next_ < parts_) {
            const int i = next_++;
            const std::function<void(int)>* f = job_;
            lk.unlock();
            (*f)(i);
            lk.lock();
            if (--remaining_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            drain(lk);
        }
    }
    std::vector<std::thread> th_;
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    int parts_ = 0, next_ = 0, remaining_ = 0;
    uint64_t gen_ = 0;
};

HostPool& host_pool() {
    // EZ_HOST_THREADS overrides the size (default: the host's hardware threads, at most 16)
    static HostPool* p = [] {
        int n = std::min(16, static_cast<int>(std::thread::hardware_concurrency()));
        if (const char* e = getenv("EZ_HOST_THREADS")) n = atoi(e);
        return new HostPool(std::max(1, n) - 1);
    }();
    return *p;
}
}  // namespace

// Copy into write-combined pinned memory with non-temporal 64-byte stores
// (AVX-512 when the host has it): streaming stores neither read the
// destination lines nor pollute the caches, so the staging copy of pageable
// rows runs closer to the host's read bandwidth.
__attribute__((target("avx512f"))) static void copy_stream_avx512(char* dst, const char* src, size_t n) {
    size_t i = 0;
    const size_t head = (64 - (reinterpret_cast<uintptr_t>(dst) & 63)) & 63;
    if (head) {
        std::memcpy(dst, src, std::min(head, n));
        i = std::min(head, n);
    }
    for (; i + 64 <= n; i += 64)
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), _mm512_loadu_si512(src + i));
    if (i < n) std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}

void copy_to_staging(void* dst, const void* src, size_t n) {
    static const bool avx512 = __builtin_cpu_supports("avx512f") && !getenv("EZ_HOST_NO_NT");
    if (avx512 && n >= 4096) copy_stream_avx512(static_cast<char*>(dst), static_cast<const char*>(src), n);
    else std::memcpy(dst, src, n);
}

void host_parallel(int64_t n, int64_t min_per_part, const std::function<void(int64_t, int64_t)>& fn) {
    if (n <= 0) return;
    const int parts = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(host_pool().size(), n / std::max<int64_t>(1, min_per_part))));
    if (parts == 1) {
        fn(0, n);
        return;
    }
    host_pool().run(parts, [&](int i) { fn(n * i / parts, n * (i + 1) / parts); });
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
