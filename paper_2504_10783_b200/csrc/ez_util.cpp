// ez_util.cpp — error reporting and small library-level entry points.
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
