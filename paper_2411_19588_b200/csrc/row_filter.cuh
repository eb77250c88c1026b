// On-the-fly tile lists from tile-ROW lists (training / render path).
//
// The binning's first level produces, for every tile row, the depth-ordered
// list of rows (visible Gaussians) whose tile rectangle spans that row.  The
// list of tile (ty, tx) is exactly the subsequence of row ty's list whose
// column span contains tx -- the reference's (tile, depth, source) order is
// preserved by construction.  A compositing CTA therefore filters its row
// list in chunks of 256 items with an order-preserving block compaction, and
// because every pixel of a tile stops at T < 1e-4, it only ever walks the
// consumed prefix (~2-3% of the full list at 1M Gaussians / 1080p) instead
// of a materialised E-entry list.
#pragma once

#include "common.cuh"

namespace uws {

constexpr int kChunk = 1024;  // row-list items examined per filter step

// Examine row-list items [cur, min(cur + 1024, end)) and append the rows whose
// column span covers tx, in list order, to dst[base ...]; only positions in
// [0, cap) are written (a negative base skips leading matches, cap 0 only
// counts).  Returns the number of matches; every
// thread of the block must call it (two __syncthreads inside).
template <int THREADS>
__device__ __forceinline__ int filter_chunk(const uint2* __restrict__ items, int cur, int end,
                                            int tx, int* dst, int base, int cap, int* s_scan) {
    constexpr int IPT = kChunk / THREADS;
    constexpr int WARPS = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int rows[IPT];
    unsigned m = 0;
    const int first = cur + threadIdx.x * IPT;  // blocked: thread order == list order
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const uint2 it = first + i < end ? __ldg(items + first + i) : make_uint2(0u, 0xffffu);
        rows[i] = (int)it.x;
        // packed inclusive column span x0 | x1 << 16 (an empty sentinel never matches)
        if ((int)(it.y & 0xffffu) <= tx && tx <= (int)(it.y >> 16)) m |= 1u << i;
    }
    const int c = __popc(m);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_scan[warp] = x;
    __syncthreads();
    int woff = 0, total = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        const int t = s_scan[w];
        woff += w < warp ? t : 0;
        total += t;
    }
    int pos = base + woff + x - c;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if (m & (1u << i)) {
            if (pos >= 0 && pos < cap) dst[pos] = rows[i];
            ++pos;
        }
    }
    __syncthreads();  // s_scan reuse + dst visibility
    return total;
}

}  // namespace uws
