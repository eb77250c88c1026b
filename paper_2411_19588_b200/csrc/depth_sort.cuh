// Depth order of the visible rows: (float64 depth, source row), stable.
//
// The reference orders by lexsort((source, depth, tile)) (rasterizer.py:79);
// the depth-major part is a stable sort of the rows by their float64 depth.
// Positive doubles order like their bit patterns, so the full key is 64 bits
// (8 radix passes).  Here the rows are radix-sorted by the HIGH 32 bits only
// (sign, exponent, 20 mantissa bits: 4 passes, fewer after the
// trivial top digits of the keys made relative to their minimum are skipped) and the rare runs of equal
// high words -- depths within ~1e-6 relative of each other -- are then put in
// (low word, row) order:
//   * runs of <= kShortRun rows: one thread, odd-even transposition network in
//     registers (stable: adjacent swaps on strictly greater keys, max-key padding);
//   * runs of up to 32 rows: one warp, bitonic sort on (low word << 32 | row)
//     (unique keys, so the order equals the stable one);
//   * longer runs (pathological: many Gaussians at almost the same depth): one
//     CTA per run, a stable 4-pass LSD counting sort on the low word.
// Rows enter the sort in ascending order, so every stage is stable and the
// result equals the 64-bit sort bit for bit.
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace uws {
namespace depth_sort {

constexpr int kShortRun = 8;
constexpr int kWarpRun = 32;
constexpr int kLongThreads = 256;

// High 32 bits of the depth's bit pattern, and their minimum as ~min into the
// (zeroed) neg_min word: the radix sort makes the keys relative to it, so the
// top digit of one scene's depths (a few exponent steps) is trivial and skipped.
// Zeroes the run counters.
__global__ void __launch_bounds__(256) k_depth_hi(const uint64_t* __restrict__ depth_bits,
                                                  const uint32_t* __restrict__ n_dev, uint32_t n_cap,
                                                  uint32_t* __restrict__ keys, uint32_t* long_cnt,
                                                  uint32_t* neg_min) {
    pdl_entry();
    __shared__ uint32_t s_min[8];
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 2) long_cnt[i] = 0;  // [0] runs > kShortRun, [1] runs > kWarpRun
    const uint32_t n = min(*n_dev, n_cap);
    uint32_t k = 0xffffffffu;
    if (i < n) {
        k = (uint32_t)(depth_bits[i] >> 32);
        keys[i] = k;
    }
    k = __reduce_min_sync(0xffffffffu, k);
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x < 32) {  // one atomic per block
        k = __reduce_min_sync(0xffffffffu, threadIdx.x < 8 ? s_min[threadIdx.x] : 0xffffffffu);
        if (threadIdx.x == 0 && k != 0xffffffffu) atomicMax(neg_min, ~k);
    }
}

// one thread per sorted position; run starts fix their run
__global__ void k_tie_fix(const uint32_t* __restrict__ keys, uint32_t* __restrict__ rows,
                          const uint64_t* __restrict__ depth_bits, const uint32_t* __restrict__ n_dev,
                          uint32_t n_cap, uint32_t* __restrict__ long_cnt,
                          uint32_t* __restrict__ long_list) {
    pdl_entry();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = min(*n_dev, n_cap);
    if (i >= n) return;
    const uint32_t k = keys[i];
    if (i > 0 && keys[i - 1] == k) return;      // not the first of its run
    if (i + 1 >= n || keys[i + 1] != k) return;  // no tie
    uint32_t len = 2;
    while (len <= (uint32_t)kShortRun && i + len < n && keys[i + len] == k) ++len;
    if (len > (uint32_t)kShortRun) {
        long_list[atomicAdd(long_cnt, 1u)] = i;
        return;
    }
    if (len == 2) {  // the common tie: one compare-exchange
        const uint32_t r0 = rows[i], r1 = rows[i + 1];
        if ((uint32_t)depth_bits[r0] > (uint32_t)depth_bits[r1]) {
            rows[i] = r1;
            rows[i + 1] = r0;
        }
        return;
    }
    uint32_t r[kShortRun], lo[kShortRun];
#pragma unroll
    for (int j = 0; j < kShortRun; ++j) {
        r[j] = (uint32_t)j < len ? rows[i + j] : 0xffffffffu;
        lo[j] = (uint32_t)j < len ? (uint32_t)depth_bits[r[j]] : 0xffffffffu;
    }
#pragma unroll
    for (int round = 0; round < kShortRun; ++round) {
#pragma unroll
        for (int j = round & 1; j + 1 < kShortRun; j += 2) {
            const bool sw = lo[j] > lo[j + 1];
            const uint32_t a = lo[j], b = lo[j + 1], ra = r[j], rb = r[j + 1];
            lo[j] = sw ? b : a;
            lo[j + 1] = sw ? a : b;
            r[j] = sw ? rb : ra;
            r[j + 1] = sw ? ra : rb;
        }
    }
#pragma unroll
    for (int j = 0; j < kShortRun; ++j)
        if ((uint32_t)j < len) rows[i + j] = r[j];
}

// One warp per run of kShortRun < len: runs of up to 32 rows are sorted in
// registers by a warp bitonic network on (low word << 32 | row); longer runs
// are passed on to k_tie_fix_long.
__global__ void __launch_bounds__(256) k_tie_fix_warp(
    const uint32_t* __restrict__ keys, uint32_t* __restrict__ rows,
    const uint64_t* __restrict__ depth_bits, const uint32_t* __restrict__ n_dev, uint32_t n_cap,
    uint32_t* __restrict__ cnt, const uint32_t* __restrict__ list, uint32_t* __restrict__ huge) {
    pdl_entry();
    const uint32_t n = min(*n_dev, n_cap);
    const uint32_t runs = cnt[0];
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
    for (uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < runs; r += nwarps) {
        const uint32_t start = list[r];
        const uint32_t k = keys[start];
        const uint32_t j = start + lane;
        const bool in = j < n && keys[j] == k;
        const unsigned ball = __ballot_sync(0xffffffffu, in);
        // run length within this window: contiguous from lane 0
        const int len = __popc(~ball) == 0 ? 32 : __ffs(~ball) - 1;
        if (len == 32 && start + 32 < n && keys[start + 32] == k) {  // longer than a warp
            if (lane == 0) huge[atomicAdd(&cnt[1], 1u)] = start;
            continue;
        }
        const uint32_t row = lane < len ? rows[j] : 0u;
        unsigned long long key =
            lane < len ? ((unsigned long long)(uint32_t)depth_bits[row] << 32) | row : ~0ull;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, jj);
                const bool up = (lane & kk) == 0;       // ascending sub-sequence
                const bool lower = (lane & jj) == 0;    // this lane holds the smaller slot
                const bool take_min = up == lower;
                key = take_min ? (other < key ? other : key) : (other > key ? other : key);
            }
        }
        if (lane < len) rows[j] = (uint32_t)key;
    }
}

// One CTA per long run: find its end, then 4 stable counting-sort passes on the
// low word (8 bits each), chunk by chunk in order, ping-ponging with tmp.
__global__ void __launch_bounds__(kLongThreads) k_tie_fix_long(
    const uint32_t* __restrict__ keys, uint32_t* __restrict__ rows,
    const uint64_t* __restrict__ depth_bits, const uint32_t* __restrict__ n_dev, uint32_t n_cap,
    const uint32_t* __restrict__ long_cnt, const uint32_t* __restrict__ long_list,  // runs > 32
    uint32_t* __restrict__ tmp) {
    pdl_entry();
    constexpr int W = kLongThreads / 32;
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_wc[W][257];
    __shared__ uint32_t s_tmp[W + 1];
    __shared__ uint32_t s_end;
    const uint32_t n = min(*n_dev, n_cap);
    const uint32_t cnt = long_cnt[1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t run = blockIdx.x; run < cnt; run += gridDim.x) {
        const uint32_t start = long_list[run];
        const uint32_t k = keys[start];
        // end of the run: first position past start whose key differs
        if (tid == 0) s_end = n;
        __syncthreads();
        for (uint32_t c0 = start; c0 < n; c0 += kLongThreads) {
            const uint32_t j = c0 + tid;
            if (j < n && keys[j] != k) atomicMin(&s_end, j);
            __syncthreads();
            if (s_end != n) break;
            __syncthreads();
        }
        const uint32_t len = s_end - start;
        __syncthreads();
        uint32_t* src = rows + start;
        uint32_t* dst = tmp + start;
        for (int pass = 0; pass < 4; ++pass) {
            const int shift = 8 * pass;
            s_base[tid] = 0;
            __syncthreads();
            for (uint32_t j = tid; j < len; j += kLongThreads)
                atomicAdd(&s_base[((uint32_t)depth_bits[src[j]] >> shift) & 0xFF], 1u);
            __syncthreads();
            {
                uint32_t tot;
                const uint32_t v = s_base[tid];
                const uint32_t ex = block_exclusive_sum<kLongThreads, uint32_t>(v, s_tmp, &tot);
                __syncthreads();
                s_base[tid] = ex;
            }
            __syncthreads();
            for (uint32_t c0 = 0; c0 < len; c0 += kLongThreads) {
                for (int q = tid; q < W * 257; q += kLongThreads) (&s_wc[0][0])[q] = 0;
                __syncthreads();
                const uint32_t j = c0 + tid;
                const bool valid = j < len;
                const uint32_t row = valid ? src[j] : 0u;
                const unsigned d = valid ? (((uint32_t)depth_bits[row] >> shift) & 0xFF) : 256u;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                const unsigned below = __popc(peers & lanemask_lt());
                if (valid && below == 0) s_wc[warp][d] = __popc(peers);
                __syncthreads();
                if (valid) {
                    uint32_t pre = 0;
                    for (int w = 0; w < warp; ++w) pre += s_wc[w][d];
                    dst[s_base[d] + pre + below] = row;
                }
                __syncthreads();
                {
                    uint32_t add = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) add += s_wc[w][tid];
                    s_base[tid] += add;
                }
                __syncthreads();
            }
            uint32_t* t = src;
            src = dst;
            dst = t;
        }
        // 4 passes: the result is back in rows
        __syncthreads();
    }
}

}  // namespace depth_sort
}  // namespace uws
