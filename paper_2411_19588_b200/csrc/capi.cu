// C-ABI meta entry points: version string and thread-local error message.
#include <atomic>
#include <cstdio>
#include <string>

#include "common.cuh"

namespace uws {

static thread_local std::string g_last_error;

static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

void count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int cuda_fail(cudaError_t e, const char* what) {
    char buf[512];
    snprintf(buf, sizeof(buf), "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    g_last_error = buf;
    return UWS_ECUDA;
}

__global__ void k_zero_words(uint32_t* __restrict__ p, size_t words) {
    pdl_entry();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += (size_t)gridDim.x * blockDim.x)
        p[i] = 0u;
}

cudaError_t zero_async(void* ptr, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return cudaSuccess;
    if (((uintptr_t)ptr | bytes) % 4 != 0) return cudaErrorInvalidValue;
    const size_t words = bytes / 4;
    const unsigned blocks = (unsigned)(words < (size_t)148 * 4 * 256 ? ceil_div((int64_t)words, 256)
                                                                     : 148 * 4);
    launch(k_zero_words, dim3(blocks), dim3(256), 0, st, (uint32_t*)ptr, words);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace uws

extern "C" const char* uws_version(void) { return "uwsplat_b200 0.1.0 (sm_100a)"; }

extern "C" const char* uws_last_error(void) { return uws::g_last_error.c_str(); }

extern "C" uint64_t uws_kernel_launches(void) { return uws::g_launches.load(); }
