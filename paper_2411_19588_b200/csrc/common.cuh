// Shared helpers for the sm_100a kernels: error plumbing, constants, small
// device utilities.  Every constant cites the reference line it mirrors.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/uwsplat_b200.h"

namespace uws {

// projection.py:21-26
constexpr int kTile = 16;
constexpr double kDilation = 0.3;
constexpr double kFloor = 1.0 / 255.0;
constexpr double kMinSigma2 = 9.0;
// rasterizer.py:27-29
constexpr double kClamp = 0.99;
constexpr double kTStop = 1e-4;
constexpr double kWeightEps = 1e-8;
// scene.py:22
constexpr double kSH_C0 = 0.28209479177387814;
// medium.py:23
constexpr double kLogisticRate = 0.1;

// float32 gates.  The reference decides in float64; the float32 kernels
// decide with these thresholds and re-evaluate in float64 inside a guard band
// (|rel| < kGuard) where float32 rounding could flip the decision.
constexpr float kFloorF = 0.003921568859368563f;       // (float)(1/255)
constexpr float kGuard = 3e-5f;
constexpr float kFloorLo = kFloorF * (1.0f - kGuard);
constexpr float kFloorHi = kFloorF * (1.0f + kGuard);
constexpr float kClampF = 0.99f;
constexpr float kClampLo = 0.99f * (1.0f - kGuard);
constexpr float kClampHi = 0.99f * (1.0f + kGuard);
// smallest float >= 1e-4 (double): T_f >= 1e-4  <=>  T_f >= kTStopF
constexpr float kTStopF = 1.00000004749745130539e-04f;
// uws_raster_out.tile_nrows flag: the stored rows are the tile's whole list
constexpr int kRowsComplete = 1 << 30;

void set_error(const std::string& msg);
void count_launches(int n);
int cuda_fail(cudaError_t e, const char* what);

#define UWS_CHECK_LAUNCH(what)                                   \
    do {                                                         \
        ::uws::count_launches(1);                                \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return ::uws::cuda_fail(_e, what); \
    } while (0)

#define UWS_CUDA(call)                                            \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::uws::cuda_fail(_e, #call); \
    } while (0)

#define UWS_REQUIRE(cond, msg)          \
    do {                                \
        if (!(cond)) {                  \
            ::uws::set_error(msg);      \
            return UWS_EINVAL;          \
        }                               \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch.  Kernels launched with launch() (programmatic
// stream serialization) start with pdl_entry(): it lets the NEXT kernel in the
// stream be launched as soon as all of this grid's CTAs are resident (its CTAs
// fill the SMs this grid's tail frees), and blocks until the PREVIOUS grid has
// completed and its writes are visible.  Because every such kernel waits before
// it reads anything, completion stays transitive along the stream (kernel N+1
// starts its work only after N, which started only after N-1, ...).
// The wait does not drop L1 lines that the previous grid's CTAs loaded on this SM
// while this CTA was already resident (e.g. a counter line that other CTAs then
// changed with atomics: measured stale), hence the acquire fence, which
// invalidates the SM's L1 (CCTL.IVALL) after the wait.
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("fence.acquire.gpu;" ::: "memory");
}

template <bool PDL, typename... P, typename... A>
inline void launch_ex(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      A&&... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = PDL ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);  // errors: cudaGetLastError
}

template <typename... P, typename... A>
inline void launch(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   A&&... args) {
    launch_ex<true>(kernel, grid, block, smem, st, std::forward<A>(args)...);
}

// Zero `bytes` bytes at `ptr` (4-byte aligned) on the device.  Used instead of
// cudaMemsetAsync inside the launch chains: a memset between two programmatically
// serialized kernels does not order the second one after it (a kernel launched
// right after a memset could run before the memset had landed).
cudaError_t zero_async(void* ptr, size_t bytes, cudaStream_t st);
cudaError_t zero_async2(void* p, size_t pbytes, void* q, size_t qbytes, cudaStream_t st);

// Launch after the previous grid has fully drained: for a kernel that depends on
// the L1 / shared-memory split its SMs are configured with (an early-launched
// grid inherits the previous kernel's carveout on SMs that never go idle).
template <typename... P, typename... A>
inline void launch_serial(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, A&&... args) {
    launch_ex<false>(kernel, grid, block, smem, st, std::forward<A>(args)...);
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Workspace {
    char* base;
    size_t size;
    size_t used = 0;
    bool dry;  // size query only
    Workspace(void* b, size_t s, bool dry_run = false) : base((char*)b), size(s), dry(dry_run) {}
    template <typename T>
    T* take(size_t count) {
        size_t off = used;
        used = align_up(used + count * sizeof(T));
        if (dry) return nullptr;
        return (T*)(base + off);
    }
    bool ok() const { return dry || used <= size; }
};

inline cudaStream_t as_stream(void* s) { return (cudaStream_t)s; }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// a / b (b > 0, normal) and sqrt(x) as IEEE round-to-nearest, with a zero
// operand answered directly: a zero in any lane otherwise sends the whole warp
// down the out-of-line special-operand path of the division / square root.
// The empty asm keeps the substituted operand opaque to the optimiser.
__device__ __forceinline__ double div_pos_nz(double a, double b) {
    double as = a == 0.0 ? 1.0 : a;
    asm("" : "+d"(as));
    const double q = __ddiv_rn(as, b);
    return a == 0.0 ? a : q;  // +-0 / b = +-0
}
__device__ __forceinline__ double sqrt_nz(double x) {
    double xs = x == 0.0 ? 1.0 : x;
    asm("" : "+d"(xs));
    const double r = __dsqrt_rn(xs);
    return x == 0.0 ? x : r;  // sqrt(+-0) = +-0
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace uws
