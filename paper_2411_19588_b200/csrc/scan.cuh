// Single-pass prefix primitives: block-level scans and decoupled look-back
// across blocks (tile ids handed out by an atomic ticket so every
// predecessor of a block is already resident -> forward progress).
#pragma once

#include "common.cuh"

namespace uws {

// 64-bit look-back status word: [flag:2 | value:62]
constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbInc = 2ull << 62;
constexpr unsigned long long kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    return *(const volatile unsigned long long*)p;
}
__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
    *(volatile unsigned long long*)p = v;
}
__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) { return *(const volatile unsigned*)p; }
__device__ __forceinline__ void st_volatile(unsigned* p, unsigned v) { *(volatile unsigned*)p = v; }

// Called by ALL lanes of ONE warp of block `tile`: publishes the block aggregate,
// walks back over the predecessors 32 at a time (lane l reads tile - 1 - l - 32k)
// and returns the exclusive prefix of this block in every lane.  A window is
// consumed up to its first inclusive prefix, or up to its first unpublished
// predecessor (then re-polled from there).
__device__ __forceinline__ unsigned long long lookback_exclusive(unsigned long long* status, int tile,
                                                                 unsigned long long aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_volatile(&status[0], kLbInc | aggregate);
        return 0;
    }
    if (lane == 0) st_volatile(&status[tile], kLbAgg | aggregate);
    unsigned long long excl = 0;
    int j = tile - 1;  // newest predecessor not yet summed
    while (true) {
        const int k = j - lane;
        const unsigned long long s = k >= 0 ? ld_volatile(&status[k]) : kLbInc;  // before tile 0: 0
        const unsigned flag = (unsigned)(s >> 62);
        const unsigned inc = __ballot_sync(0xffffffffu, flag == 2);
        const unsigned nready = __ballot_sync(0xffffffffu, flag == 0);
        const int m = inc ? __ffs(inc) - 1 : 31;                   // last lane of the window
        const unsigned win = m == 31 ? 0xffffffffu : ((2u << m) - 1u);
        const int take = (nready & win) ? __ffs(nready & win) - 1 : m + 1;  // lanes [0, take)
        unsigned long long v = lane < take ? (s & kLbMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (take == m + 1 && inc) break;
        j -= take;
    }
    if (lane == 0) st_volatile(&status[tile], kLbInc | (excl + aggregate));
    return excl;
}

// Block-wide exclusive sum of one value per thread.  `smem` needs
// (THREADS/32 + 1) slots.  Returns the exclusive prefix; *total = block sum.
template <int THREADS, typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* smem, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    if (warp == 0) {
        constexpr int W = THREADS / 32;
        T w = lane < W ? smem[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < W) smem[lane] = w;  // inclusive over warps
        if (lane == W - 1) smem[W] = w;
    }
    __syncthreads();
    T warp_excl = warp > 0 ? smem[warp - 1] : T(0);
    *total = smem[THREADS / 32];
    return warp_excl + x - v;
}

}  // namespace uws
