// Depth order of the visible rows by bucketing: (float64 depth, source row).
//
// The reference orders by lexsort((source, depth, tile)) (rasterizer.py:79); its
// depth-major part is the order of the rows by (float64 depth, row).  Positive
// doubles order like their bit patterns, so the key is the 64-bit pattern with
// the row as the final tie-break.
//
// One scene's visible depths span a few exponent steps, so the HIGH 32 bits of
// the keys, made relative to their minimum, fit in ~22 bits.  They are cut into
// kBuckets = 2^20 equal buckets (bucket = (hi - min) >> shift, shift chosen on
// the device from the span): count, exclusive scan, scatter the rows into their
// bucket's slots (atomic cursor: any order inside a bucket), then sort every
// bucket by (64-bit key, row) -- one thread for <= kThreadRun rows (register
// network), one warp for <= 32 (bitonic), one CTA beyond (shared-memory bitonic
// up to kCtaRun rows, else a 12-pass stable LSD counting sort on the row and the
// key).  At 1M Gaussians/1080p a bucket holds ~1-3 rows; the total order equals
// the reference's exactly, whatever the distribution.
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace uws {
namespace depth_bucket {

#ifndef UWS_LOG_BUCKETS
#define UWS_LOG_BUCKETS 20
#endif
constexpr int kLogBuckets = UWS_LOG_BUCKETS;  // measured at C3: 2^19 and 2^21 are slower
constexpr uint32_t kBuckets = 1u << kLogBuckets;
constexpr int kThreadRun = 8;
constexpr int kCtaThreads = 256;
constexpr int kCtaRun = 2048;  // shared-memory bitonic limit

// meta block (zeroed before every sort): [0] ~min hi word, [1] max hi word,
// [2] rows in warp-sorted buckets, [3] rows in CTA-sorted buckets, then counts
struct Meta {
    uint32_t neg_min, max, n_warp, n_cta;
};

// range = {~min, max} of the keys' high words (Meta's first two fields, or the
// preprocess kernel's uws_projected.depth_range)
__device__ __forceinline__ uint32_t bucket_shift(const uint32_t* range) {
    const uint32_t span = range[1] - ~range[0];
    const int bits = span ? 32 - __clz(span) : 0;
    return bits > kLogBuckets ? (uint32_t)(bits - kLogBuckets) : 0u;
}

__device__ __forceinline__ bool key_less(uint64_t ka, uint32_t ra, uint64_t kb, uint32_t rb) {
    return ka < kb || (ka == kb && ra < rb);
}

// high words of the keys and their min / max
__global__ void __launch_bounds__(256) k_hi_minmax(const uint64_t* __restrict__ depth_bits,
                                                   const uint32_t* __restrict__ n_dev,
                                                   uint32_t n_cap, Meta* meta) {
    pdl_entry();
    __shared__ uint32_t s_lo[8], s_hi[8];
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = min(*n_dev, n_cap);
    uint32_t lo = 0xffffffffu, hi = 0u;
    if (i < n) {
        lo = hi = (uint32_t)(depth_bits[i] >> 32);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const bool ok = threadIdx.x < blockDim.x / 32;
        lo = __reduce_min_sync(0xffffffffu, ok ? s_lo[threadIdx.x] : 0xffffffffu);
        hi = __reduce_max_sync(0xffffffffu, ok ? s_hi[threadIdx.x] : 0u);
        if (threadIdx.x == 0 && lo != 0xffffffffu) {
            atomicMax(&meta->neg_min, ~lo);
            atomicMax(&meta->max, hi);
        }
    }
}

__device__ __forceinline__ uint32_t key_hi(const uint64_t* depth_bits, uint32_t i) {
    return (uint32_t)(depth_bits[i] >> 32);
}

__global__ void __launch_bounds__(256) k_bucket_count(const uint64_t* __restrict__ depth_bits,
                                                      const uint32_t* __restrict__ n_dev,
                                                      uint32_t n_cap, const uint32_t* __restrict__ range,
                                                      uint32_t* __restrict__ count) {
    pdl_entry();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = min(*n_dev, n_cap);
    if (i >= n) return;
    const uint32_t kmin = ~range[0], sh = bucket_shift(range);
    atomicAdd(&count[min((key_hi(depth_bits, i) - kmin) >> sh, kBuckets - 1)], 1u);
}

// start[] = exclusive bucket starts on entry, bucket ends on exit
__global__ void __launch_bounds__(256) k_bucket_scatter(const uint64_t* __restrict__ depth_bits,
                                                        const uint32_t* __restrict__ n_dev,
                                                        uint32_t n_cap, const uint32_t* __restrict__ range,
                                                        uint32_t* __restrict__ start,
                                                        uint32_t* __restrict__ rows) {
    pdl_entry();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = min(*n_dev, n_cap);
    if (i >= n) return;
    const uint32_t kmin = ~range[0], sh = bucket_shift(range);
    rows[atomicAdd(&start[min((key_hi(depth_bits, i) - kmin) >> sh, kBuckets - 1)], 1u)] = i;
}

// One thread per bucket: short buckets sorted in registers, longer ones listed.
__global__ void __launch_bounds__(256) k_bucket_fix(const uint32_t* __restrict__ ends,
                                                    const uint64_t* __restrict__ depth_bits,
                                                    uint32_t* __restrict__ rows, Meta* meta,
                                                    uint32_t* __restrict__ warp_list,
                                                    uint32_t* __restrict__ cta_list) {
    pdl_entry();
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= kBuckets) return;
    const uint32_t hi = ends[b], lo = b ? ends[b - 1] : 0u;
    const uint32_t len = hi - lo;
    if (len <= 1) return;
    if (len > (uint32_t)kThreadRun) {
        if (len <= 32u) warp_list[atomicAdd(&meta->n_warp, 1u)] = b;
        else cta_list[atomicAdd(&meta->n_cta, 1u)] = b;
        return;
    }
    if (len == 2) {  // the common non-trivial case (~1-3 rows per bucket): one exchange
        const uint32_t r0 = rows[lo], r1 = rows[lo + 1];
        if (key_less(depth_bits[r1], r1, depth_bits[r0], r0)) {
            rows[lo] = r1;
            rows[lo + 1] = r0;
        }
        return;
    }
    uint32_t r[kThreadRun];
    uint64_t k[kThreadRun];
#pragma unroll
    for (int j = 0; j < kThreadRun; ++j) {
        r[j] = (uint32_t)j < len ? rows[lo + j] : 0xffffffffu;
        k[j] = (uint32_t)j < len ? depth_bits[r[j]] : ~0ull;
    }
    // odd-even transposition network (padding sorts last)
#pragma unroll
    for (int round = 0; round < kThreadRun; ++round) {
#pragma unroll
        for (int j = round & 1; j + 1 < kThreadRun; j += 2) {
            const bool sw = key_less(k[j + 1], r[j + 1], k[j], r[j]);
            const uint64_t ka = k[j], kb = k[j + 1];
            const uint32_t ra = r[j], rb = r[j + 1];
            k[j] = sw ? kb : ka;
            k[j + 1] = sw ? ka : kb;
            r[j] = sw ? rb : ra;
            r[j + 1] = sw ? ra : rb;
        }
    }
#pragma unroll
    for (int j = 0; j < kThreadRun; ++j)
        if ((uint32_t)j < len) rows[lo + j] = r[j];
}

// One warp per listed bucket of 9..32 rows: bitonic sort on (key, row).
__global__ void __launch_bounds__(256) k_bucket_warp(const uint32_t* __restrict__ ends,
                                                     const uint64_t* __restrict__ depth_bits,
                                                     uint32_t* __restrict__ rows,
                                                     const Meta* __restrict__ meta,
                                                     const uint32_t* __restrict__ list) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const uint32_t nlist = meta->n_warp;
    const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
    for (uint32_t w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); w < nlist; w += nwarps) {
        const uint32_t b = list[w];
        const uint32_t hi = ends[b], lo = b ? ends[b - 1] : 0u;
        const uint32_t len = hi - lo;
        uint32_t r = (uint32_t)lane < len ? rows[lo + lane] : 0xffffffffu;
        uint64_t k = (uint32_t)lane < len ? depth_bits[r] : ~0ull;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const uint64_t ko = __shfl_xor_sync(0xffffffffu, k, jj);
                const uint32_t ro = __shfl_xor_sync(0xffffffffu, r, jj);
                const bool up = (lane & kk) == 0;      // ascending sub-sequence
                const bool lower = (lane & jj) == 0;   // this lane keeps the smaller
                const bool other_less = key_less(ko, ro, k, r);
                const bool take = (up == lower) ? other_less : !other_less;
                k = take ? ko : k;
                r = take ? ro : r;
            }
        }
        if ((uint32_t)lane < len) rows[lo + lane] = r;
    }
}

// One CTA per listed bucket of > 32 rows.
__global__ void __launch_bounds__(kCtaThreads) k_bucket_cta(const uint32_t* __restrict__ ends,
                                                            const uint64_t* __restrict__ depth_bits,
                                                            uint32_t* __restrict__ rows,
                                                            const Meta* __restrict__ meta,
                                                            const uint32_t* __restrict__ list,
                                                            uint32_t* __restrict__ tmp) {
    pdl_entry();
    constexpr int W = kCtaThreads / 32;
    __shared__ uint64_t s_key[kCtaRun];
    __shared__ uint32_t s_row[kCtaRun];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_wc[W][257];
    __shared__ uint32_t s_tmp[W + 1];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t nlist = meta->n_cta;
    for (uint32_t w = blockIdx.x; w < nlist; w += gridDim.x) {
        const uint32_t b = list[w];
        const uint32_t hi = ends[b], lo = b ? ends[b - 1] : 0u;
        const uint32_t len = hi - lo;
        if (len <= (uint32_t)kCtaRun) {
            uint32_t p2 = 64;
            while (p2 < len) p2 <<= 1;
            for (uint32_t j = tid; j < p2; j += kCtaThreads) {
                const uint32_t r = j < len ? rows[lo + j] : 0xffffffffu;
                s_row[j] = r;
                s_key[j] = j < len ? depth_bits[r] : ~0ull;
            }
            __syncthreads();
            for (uint32_t kk = 2; kk <= p2; kk <<= 1) {
                for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
                    for (uint32_t i = tid; i < p2; i += kCtaThreads) {
                        const uint32_t o = i ^ jj;
                        if (o > i) {
                            const bool up = (i & kk) == 0;
                            const bool gt = key_less(s_key[o], s_row[o], s_key[i], s_row[i]);
                            if (gt == up) {  // out of order for this direction: swap
                                const uint64_t tk = s_key[i];
                                s_key[i] = s_key[o];
                                s_key[o] = tk;
                                const uint32_t tr = s_row[i];
                                s_row[i] = s_row[o];
                                s_row[o] = tr;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (uint32_t j = tid; j < len; j += kCtaThreads) rows[lo + j] = s_row[j];
            __syncthreads();
            continue;
        }
        // long bucket: stable LSD counting sort, 8-bit digits of the row (4 passes)
        // and of the 64-bit key (8 passes): row order first, then key order
        uint32_t* src = rows + lo;
        uint32_t* dst = tmp + lo;
        for (int pass = 0; pass < 12; ++pass) {
            const int shift = 8 * (pass & 3);
            s_base[tid] = 0;
            __syncthreads();
            auto digit = [&](uint32_t r) -> unsigned {
                if (pass < 4) return (r >> shift) & 0xFFu;
                const uint64_t k = depth_bits[r];
                return (unsigned)(k >> (8 * (pass - 4))) & 0xFFu;
            };
            for (uint32_t j = tid; j < len; j += kCtaThreads) atomicAdd(&s_base[digit(src[j])], 1u);
            __syncthreads();
            {
                uint32_t tot;
                const uint32_t v = s_base[tid];
                const uint32_t ex = block_exclusive_sum<kCtaThreads, uint32_t>(v, s_tmp, &tot);
                __syncthreads();
                s_base[tid] = ex;
            }
            __syncthreads();
            for (uint32_t c0 = 0; c0 < len; c0 += kCtaThreads) {
                for (int q = tid; q < W * 257; q += kCtaThreads) (&s_wc[0][0])[q] = 0;
                __syncthreads();
                const uint32_t j = c0 + tid;
                const bool valid = j < len;
                const uint32_t row = valid ? src[j] : 0u;
                const unsigned d = valid ? digit(row) : 256u;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                const unsigned below = __popc(peers & lanemask_lt());
                if (valid && below == 0) s_wc[warp][d] = __popc(peers);
                __syncthreads();
                if (valid) {
                    uint32_t pre = 0;
                    for (int q = 0; q < warp; ++q) pre += s_wc[q][d];
                    dst[s_base[d] + pre + below] = row;
                }
                __syncthreads();
                {
                    uint32_t add = 0;
#pragma unroll
                    for (int q = 0; q < W; ++q) add += s_wc[q][tid];
                    s_base[tid] += add;
                }
                __syncthreads();
            }
            uint32_t* t = src;
            src = dst;
            dst = t;
        }
        // 12 passes: the result is back in rows
        __syncthreads();
    }
}

}  // namespace depth_bucket
}  // namespace uws
