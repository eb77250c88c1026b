// Stable LSD radix sort of (key, uint32 value) pairs, 8-bit digits, one
// kernel per digit pass in the "onesweep" style: a single up-front global
// histogram for all passes, then per pass each tile ranks its keys in
// registers/shared memory (warp match + per-warp counters, stable in input
// order), resolves its global per-digit base by decoupled look-back over the
// preceding tiles, reorders in shared memory and writes digit runs coalesced.
// Every key is read once and written once per pass.
//
// Passes whose digit is the same for every key are identity permutations; the
// histogram shows them before any pass runs, so their kernels exit at once and
// the remaining passes pick their ping-pong buffers from the per-pass flags so
// that the last executed pass still lands in the output.
#pragma once

#include "scan.cuh"

namespace uws {
namespace radix {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 256;

// status word per (tile, bin): [flag:2 | count:30]
constexpr unsigned kStAgg = 1u << 30;
constexpr unsigned kStInc = 2u << 30;
constexpr unsigned kStMask = (1u << 30) - 1;

template <typename K>
struct Cfg;
template <>
struct Cfg<uint64_t> {
    static constexpr int kIpt = 12;
};
template <>
struct Cfg<uint32_t> {
    static constexpr int kIpt = 16;
};

template <typename K>
constexpr int tile_items() {
    return kThreads * Cfg<K>::kIpt;
}

__device__ __forceinline__ uint32_t dev_count(const uint32_t* n_dev, uint32_t n_cap) {
    if (!n_dev) return n_cap;
    uint32_t n = *n_dev;
    return n < n_cap ? n : n_cap;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) k_histogram(const K* __restrict__ keys, uint32_t n_cap,
                                                       const uint32_t* n_dev, int begin_bit,
                                                       int passes, uint32_t* __restrict__ hist) {
    pdl_entry();
    __shared__ uint32_t h[8 * kBins];
    for (int i = threadIdx.x; i < passes * kBins; i += kThreads) h[i] = 0;
    __syncthreads();
    const uint32_t n = dev_count(n_dev, n_cap);
    const unsigned lt = lanemask_lt();
    const uint32_t stride = gridDim.x * kThreads;
    for (uint32_t base = blockIdx.x * kThreads; base < n; base += stride) {
        uint32_t i = base + threadIdx.x;
        bool valid = i < n;
        K key = valid ? keys[i] : K(0);
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        if (vmask == 0) continue;  // whole warp past the end (lane 0 would index bin 256)
        for (int p = 0; p < passes; ++p) {
            unsigned d = valid ? unsigned((key >> (begin_bit + 8 * p)) & 0xFF) : 0x100u;
            unsigned d0 = __shfl_sync(0xffffffffu, d, __ffs(vmask) - 1);
            if (__all_sync(0xffffffffu, d == d0 || !valid)) {
                // common for the high digits of nearby keys: one atomic per warp
                if ((threadIdx.x & 31) == 0) atomicAdd(&h[p * kBins + d0], __popc(vmask));
            } else if (valid) {
                atomicAdd(&h[p * kBins + d], 1u);
            }
        }
    }
    (void)lt;
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kBins; i += kThreads)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// exclusive scan of each pass's 256-bin histogram, in place (one block per pass);
// trivial[p] = 1 when one digit holds every key (the pass is the identity)
static __global__ void __launch_bounds__(kBins) k_scan_hist(uint32_t* hist, int passes,
                                                            const uint32_t* n_dev, uint32_t n_cap,
                                                            uint32_t* trivial) {
    pdl_entry();
    __shared__ uint32_t tmp[kBins / 32 + 1];
    const int p = blockIdx.x;
    const uint32_t n = dev_count(n_dev, n_cap);
    uint32_t v = hist[p * kBins + threadIdx.x];
    const int all = __syncthreads_or(v == n);
    uint32_t tot;
    uint32_t ex = block_exclusive_sum<kBins>(v, tmp, &tot);
    hist[p * kBins + threadIdx.x] = ex;
    if (threadIdx.x == 0) trivial[p] = all ? 1u : 0u;
}

template <typename K>
struct PassArgs {
    const K* keys_in;          // pass input (vals_in NULL: the identity 0..n-1)
    const uint32_t* vals_in;
    K* keys_out;               // where the last executed pass writes
    uint32_t* vals_out;
    K* keys_tmp;               // the other ping-pong buffer
    uint32_t* vals_tmp;
    const uint32_t* trivial;   // [passes] from k_scan_hist
    int pass, passes;
};

template <typename K>
__global__ void __launch_bounds__(kThreads) k_onesweep(PassArgs<K> pa, uint32_t n_cap,
                                                      const uint32_t* n_dev, int shift,
                                                      const uint32_t* __restrict__ bin_base,
                                                      uint32_t* status, uint32_t* ticket) {
    pdl_entry();
    constexpr int IPT = Cfg<K>::kIpt;
    constexpr int TILE = kThreads * IPT;
    // executed passes before this one (j) and in total (m); the data after e executed
    // passes lives in keys_out when m - e is even, else in keys_tmp
    int j = 0, m = 0;
    for (int q = 0; q < pa.passes; ++q) {
        const bool run = pa.trivial[q] == 0u;
        m += run;
        if (q < pa.pass) j += run;
    }
    const uint32_t n = dev_count(n_dev, n_cap);
    if (pa.trivial[pa.pass]) {
        if (m == 0 && pa.pass == pa.passes - 1) {  // every pass trivial: the sort is a copy
            for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) {
                pa.keys_out[i] = pa.keys_in[i];
                pa.vals_out[i] = pa.vals_in ? pa.vals_in[i] : i;
            }
        }
        return;
    }
    const K* __restrict__ keys_in = j == 0 ? pa.keys_in : ((m - j) % 2 == 0 ? pa.keys_out : pa.keys_tmp);
    const uint32_t* __restrict__ vals_in =
        j == 0 ? pa.vals_in : ((m - j) % 2 == 0 ? pa.vals_out : pa.vals_tmp);
    K* __restrict__ keys_out = (m - j - 1) % 2 == 0 ? pa.keys_out : pa.keys_tmp;
    uint32_t* __restrict__ vals_out = (m - j - 1) % 2 == 0 ? pa.vals_out : pa.vals_tmp;
    __shared__ K s_keys[TILE];
    __shared__ uint32_t s_vals[TILE];
    __shared__ uint32_t s_warp[kWarps][kBins];
    __shared__ uint32_t s_local[kBins];
    __shared__ uint32_t s_global[kBins];
    __shared__ uint32_t s_tmp[kBins / 32 + 1];
    __shared__ int s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (int)atomicAdd(ticket, 1u);
    for (int i = tid; i < kWarps * kBins; i += kThreads) (&s_warp[0][0])[i] = 0;
    __syncthreads();
    const int tile = s_tile;
    const uint32_t base = (uint32_t)tile * TILE;

    K key[IPT];
    uint32_t val[IPT];
    uint32_t rank[IPT];
    const unsigned lt = lanemask_lt();
    // warp-striped: warp w owns [w*IPT*32, (w+1)*IPT*32) of the tile
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        uint32_t idx = base + (uint32_t)(warp * IPT + i) * 32u + lane;
        bool valid = idx < n;
        key[i] = valid ? keys_in[idx] : K(0);
        val[i] = valid ? (vals_in ? vals_in[idx] : idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        uint32_t idx = base + (uint32_t)(warp * IPT + i) * 32u + lane;
        bool valid = idx < n;
        unsigned d = valid ? unsigned((key[i] >> shift) & 0xFF) : 0x100u;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = valid ? s_warp[warp][d] : 0u;
        rank[i] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) s_warp[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per bin: exclusive prefix over warps, block count, look-back
    {
        const int b = tid;  // kThreads == kBins
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            uint32_t c = s_warp[w][b];
            s_warp[w][b] = run;
            run += c;
        }
        uint32_t cnt = run;
        uint32_t excl = 0;
        if (tile == 0) {
            st_volatile(&status[b], kStInc | cnt);
        } else {
            st_volatile(&status[(size_t)tile * kBins + b], kStAgg | cnt);
            // look back kLook predecessors per round trip: sum aggregates up to
            // the nearest inclusive prefix, re-poll from the first unpublished one
            // (16 and 32 measured no faster at 777k keys)
            constexpr int kLook = 8;
            int j = tile - 1;
            while (true) {
                uint32_t sv[kLook];
#pragma unroll
                for (int q = 0; q < kLook; ++q)
                    sv[q] = j - q >= 0 ? ld_volatile(&status[(size_t)(j - q) * kBins + b]) : kStInc;
                int used = 0;
                bool done = false;
#pragma unroll
                for (int q = 0; q < kLook; ++q) {
                    if (done || used < q) break;  // stop at the first gap
                    const uint32_t f = sv[q] >> 30;
                    if (f == 0) break;
                    excl += sv[q] & kStMask;
                    used = q + 1;
                    if (f == 2) done = true;
                }
                if (done) break;
                j -= used;
            }
            st_volatile(&status[(size_t)tile * kBins + b], kStInc | (excl + cnt));
        }
        s_global[b] = bin_base[b] + excl;
        uint32_t tot;
        uint32_t loc = block_exclusive_sum<kThreads>(cnt, s_tmp, &tot);
        s_local[b] = loc;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        uint32_t idx = base + (uint32_t)(warp * IPT + i) * 32u + lane;
        if (idx < n) {
            unsigned d = unsigned((key[i] >> shift) & 0xFF);
            uint32_t pos = s_local[d] + s_warp[warp][d] + rank[i];
            s_keys[pos] = key[i];
            s_vals[pos] = val[i];
        }
    }
    __syncthreads();
    uint32_t count = base >= n ? 0u : (n - base < (uint32_t)TILE ? n - base : (uint32_t)TILE);
    for (uint32_t j = tid; j < count; j += kThreads) {
        K k = s_keys[j];
        unsigned d = unsigned((k >> shift) & 0xFF);
        uint32_t o = s_global[d] + (j - s_local[d]);
        keys_out[o] = k;
        vals_out[o] = s_vals[j];
    }
}

// Workspace for sorting n pairs over `passes` 8-bit digits.  hist .. trivial is
// one contiguous block ("meta", meta_bytes long) that must be zero when a sort starts.
template <typename K>
struct Plan {
    K* k_tmp;
    uint32_t* v_tmp;
    uint32_t *hist, *status, *tickets, *trivial;
    size_t meta_bytes;
    int passes;
};

template <typename K>
inline void plan(Workspace& ws, uint32_t n, int passes, Plan<K>& p) {
    int tiles = (int)ceil_div(n > 0 ? n : 1, tile_items<K>());
    p.passes = passes;
    p.k_tmp = ws.take<K>(n);
    p.v_tmp = ws.take<uint32_t>(n);
    p.hist = ws.take<uint32_t>((size_t)passes * kBins);
    p.status = ws.take<uint32_t>((size_t)passes * tiles * kBins);
    p.tickets = ws.take<uint32_t>(passes);
    p.trivial = ws.take<uint32_t>(passes);
    p.meta_bytes = (size_t)((char*)(p.trivial + passes) - (char*)p.hist);
}

// Sort (keys_in, vals_in or identity if NULL) by bits [begin_bit, begin_bit+8*passes).
// n_cap sizes the grids; the actual count is *n_dev when n_dev != NULL.
// The result lands in (keys_out, vals_out); keys_in/vals_in are not modified.
template <typename K>
inline cudaError_t sort_pairs(const Plan<K>& p, const K* keys_in, const uint32_t* vals_in,
                              K* keys_out, uint32_t* vals_out, uint32_t n_cap,
                              const uint32_t* n_dev, int begin_bit, cudaStream_t st) {
    if (n_cap == 0) return cudaSuccess;
    cudaError_t e = zero_async(p.hist, p.meta_bytes, st);
    if (e != cudaSuccess) return e;
    int hist_blocks = (int)ceil_div(n_cap, kThreads * 8);
    if (hist_blocks > 1184) hist_blocks = 1184;
    launch(k_histogram<K>, dim3(hist_blocks), dim3(kThreads), 0, st, keys_in, n_cap, n_dev, begin_bit, p.passes,
                                                     p.hist);
    launch(k_scan_hist, dim3(p.passes), dim3(kBins), 0, st, p.hist, p.passes, n_dev, n_cap, p.trivial);
    const int tiles = (int)ceil_div(n_cap, tile_items<K>());
    PassArgs<K> pa{keys_in, vals_in, keys_out, vals_out, p.k_tmp, p.v_tmp, p.trivial, 0, p.passes};
    for (int q = 0; q < p.passes; ++q) {
        pa.pass = q;
        launch(k_onesweep<K>, dim3(tiles), dim3(kThreads), 0, st, pa, n_cap, n_dev, begin_bit + 8 * q,
                                                  p.hist + q * kBins,
                                                  p.status + (size_t)q * tiles * kBins,
                                                  p.tickets + q);
    }
    count_launches(2 + p.passes);
    return cudaGetLastError();
}

}  // namespace radix
}  // namespace uws
