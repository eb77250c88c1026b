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

// two ranges in one launch (the chains that zero a small and a large buffer back to back)
__global__ void k_zero_words2(uint32_t* __restrict__ p, size_t words, uint32_t* __restrict__ q,
                              size_t qwords) {
    pdl_entry();
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words + qwords; i += stride) {
        if (i < words) p[i] = 0u;
        else q[i - words] = 0u;
    }
}

cudaError_t zero_async2(void* p, size_t pbytes, void* q, size_t qbytes, cudaStream_t st) {
    if (pbytes == 0 || p == nullptr) return zero_async(q, qbytes, st);
    if (qbytes == 0 || q == nullptr) return zero_async(p, pbytes, st);
    if (((uintptr_t)p | pbytes | (uintptr_t)q | qbytes) % 4 != 0) return cudaErrorInvalidValue;
    const size_t words = pbytes / 4, qwords = qbytes / 4, total = words + qwords;
    const unsigned blocks = (unsigned)(total < (size_t)148 * 4 * 256 ? ceil_div((int64_t)total, 256)
                                                                     : 148 * 4);
    launch(k_zero_words2, dim3(blocks), dim3(256), 0, st, (uint32_t*)p, words, (uint32_t*)q, qwords);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace uws

extern "C" const char* uws_version(void) { return "uwsplat_b200 0.1.0 (sm_100a)"; }

extern "C" const char* uws_last_error(void) { return uws::g_last_error.c_str(); }

extern "C" uint64_t uws_kernel_launches(void) { return uws::g_launches.load(); }
