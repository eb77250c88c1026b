// K2-K5 binning: tile-key duplication, (tile, depth) ordering, tile ranges.
//
// Replaces rasterizer.bin_and_sort (rasterizer.py:50-85), whose order is
// lexsort((source_index, depth, tile_id)): tile ascending, then float64
// depth ascending, then source index.
//
// Design: instead of radix-sorting the E (tile, depth) keys, the lists are
// produced by two levels of STABLE bucketing of the depth-sorted rows, so
// every tile entry is written exactly once and no E-sized key is ever read
// back:
//   0. order of the K visible rows by (bit pattern of their float64 depth,
//      row) -- positive doubles order like their bits, and the row is the
//      reference's source-index tie-break: the high words are bucketed, then
//      every bucket is sorted (depth_bucket.cuh);
//   1. rank order -> tile-ROW lists (kBand = 1 tile row per band): each
//      Gaussian is appended, in rank order, to the list of every tile row its
//      rectangle touches, as an 8-byte item (row, column span).  The training
//      and render kernels filter these row lists per tile on the fly;
//   2. (API path only) row lists -> tile lists: each (Gaussian, row) item is
//      appended, in list order, to the tiles of its span.
// A stable append needs, per (block of items, bucket), the number of earlier
// items in the same bucket.  Each block is cut into 8 warp sub-blocks; a warp
// builds its bucket histogram with shared-memory difference arrays and a warp
// scan, block totals are scanned across blocks (decoupled look-back), and each
// warp then appends its items 32 at a time, bucket by bucket: the lanes whose
// span covers the bucket write consecutive slots from its cursor in list
// order -- deterministic, no global atomics, bit-identical to the reference
// order given the same depths and rectangles.  Level-2 blocks stage their
// entries in shared memory so each tile run leaves the SM as coalesced stores.
#include <algorithm>

#include "depth_bucket.cuh"

namespace uws {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpsB = kThreads / 32;
constexpr int kBand = 1;                       // tile rows per band
constexpr int kMaxGX = 256;                    // max tile columns (4096 px)
constexpr int kMaxBands = 256 / kBand;         // max bands (4096 px tall)
constexpr int kPerWarp = 128;                  // level 1: ranks per warp sub-block
constexpr int kBlockItems = kWarpsB * kPerWarp;  // 1024
constexpr int kRankChunks = kPerWarp / 32;
constexpr int kSegPerWarp = 64;                // level 2: items per warp sub-block
constexpr int kSegBlock = kWarpsB * kSegPerWarp;  // 512
constexpr int kSegChunks = kSegPerWarp / 32;
constexpr int kXS = kMaxGX + 1;                // cursor row stride (room for x1+1)
constexpr int kStageCap = 12288;               // entries staged in shared memory per block
#ifndef UWS_SCAN_IPT
#define UWS_SCAN_IPT 8
#endif
constexpr int kScanIpt = UWS_SCAN_IPT;

__device__ __forceinline__ int rect_nx(short4 r) { return (int)r.z - (int)r.x + 1; }
__device__ __forceinline__ int rect_ny(short4 r) { return (int)r.w - (int)r.y + 1; }
__device__ __forceinline__ bool rect_ok(short4 r) { return rect_nx(r) > 0 && rect_ny(r) > 0; }

// ---------------------------------------------------------------------------
// generic single-pass exclusive scan (u32 in, u32 out, total to *total)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_scan_u32(const uint32_t* __restrict__ in,
                                                       uint32_t* __restrict__ out, uint32_t n,
                                                       uint32_t* total,
                                                       unsigned long long* status,
                                                       unsigned* ticket) {
    pdl_entry();
    __shared__ int s_tile;
    __shared__ unsigned long long s_scan[kThreads / 32 + 1];
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int tile = s_tile;
    const uint32_t first = (uint32_t)tile * kThreads * kScanIpt + threadIdx.x * kScanIpt;
    uint32_t v[kScanIpt];
    unsigned long long sum = 0;
    // a full run of kScanIpt from 16-byte-aligned buffers: vector loads and stores
    const bool full = first + kScanIpt <= n &&
                      ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (full) {
#pragma unroll
        for (int j = 0; j < kScanIpt; j += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(in + first + j);
            v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kScanIpt; ++j) v[j] = first + j < n ? in[first + j] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) sum += v[j];
    unsigned long long tot;
    unsigned long long ex = block_exclusive_sum<kThreads, unsigned long long>(sum, s_scan, &tot);
    if (threadIdx.x < 32) {
        const unsigned long long b = lookback_exclusive(status, tile, tot);
        if (threadIdx.x == 0) s_base = b;
    }
    __syncthreads();
    unsigned long long run = s_base + ex;
    uint32_t o[kScanIpt];
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) {
        o[j] = (uint32_t)run;
        run += v[j];
    }
    if (full) {
#pragma unroll
        for (int j = 0; j < kScanIpt; j += 4)
            *reinterpret_cast<uint4*>(out + first + j) = make_uint4(o[j], o[j + 1], o[j + 2], o[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < kScanIpt; ++j)
            if (first + j < n) out[first + j] = o[j];
    }
    if (tile == (int)gridDim.x - 1 && threadIdx.x == kThreads - 1 && total)
        *total = (uint32_t)(s_base + tot);
}

// in-place inclusive scan of one warp's histogram row (nbins <= 256; 8 per lane)
__device__ __forceinline__ void warp_scan_row(int* d, int lane, int nbins) {
    const int b0 = lane * 8;
    int loc[8];
    int s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        loc[i] = (b0 + i < nbins) ? d[b0 + i] : 0;
        s += loc[i];
    }
    int x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    int run = x - s;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        run += loc[i];
        if (b0 + i < nbins) d[b0 + i] = run;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// level 1: rank order -> band lists
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rank_load(const uint32_t* sorted_rows, const short4* rect,
                                          uint32_t k, uint32_t first, int lane,
                                          uint32_t (&row)[kRankChunks], short4 (&rc)[kRankChunks]) {
#pragma unroll
    for (int i = 0; i < kRankChunks; ++i) {
        uint32_t r = first + i * 32 + lane;
        row[i] = r < k ? __ldg(sorted_rows + r) : 0xffffffffu;
    }
#pragma unroll
    for (int i = 0; i < kRankChunks; ++i)
        rc[i] = row[i] != 0xffffffffu ? __ldg(rect + row[i]) : make_short4(0, 0, -1, -1);
}

// band histogram of this warp's ranks (difference array + warp scan)
__device__ __forceinline__ void rank_band_hist(const short4 (&rc)[kRankChunks], int* d, int lane,
                                               int nbands, unsigned long long* e_sum,
                                               unsigned long long* s_sum) {
    unsigned long long e = 0, s = 0;
#pragma unroll
    for (int i = 0; i < kRankChunks; ++i) {
        if (rect_ok(rc[i])) {
            const int b0 = rc[i].y / kBand, b1 = rc[i].w / kBand;
            atomicAdd(&d[b0], 1);
            atomicAdd(&d[b1 + 1], -1);
            e += (unsigned long long)(rect_nx(rc[i]) * rect_ny(rc[i]));
            s += (unsigned long long)(b1 - b0 + 1);
        }
    }
    __syncwarp();
    warp_scan_row(d, lane, nbands);
    if (e_sum) {
        *e_sum = e;
        *s_sum = s;
    }
}

// L1a: per 2048-rank block, items per band -> m_band[band * nblk + b]; totals E, S
__global__ void __launch_bounds__(kThreads) k_band_count(const uint32_t* __restrict__ sorted_rows,
                                                         const short4* __restrict__ rect,
                                                         const int32_t* __restrict__ k_dev,
                                                         int nbands, uint32_t nblk,
                                                         uint32_t* __restrict__ m_band,
                                                         unsigned long long* totals) {
    pdl_entry();
    __shared__ int diff[kWarpsB][kMaxBands + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t k = (uint32_t)*k_dev;
    for (int i = threadIdx.x; i < kWarpsB * (kMaxBands + 1); i += kThreads) (&diff[0][0])[i] = 0;
    __syncthreads();
    uint32_t rowv[kRankChunks];
    short4 rcv[kRankChunks];
    rank_load(sorted_rows, rect, k, blockIdx.x * kBlockItems + warp * kPerWarp, lane, rowv, rcv);
    unsigned long long e, s;
    rank_band_hist(rcv, diff[warp], lane, nbands, &e, &s);
    e = warp_sum(e);
    s = warp_sum(s);
    if (lane == 0) {
        atomicAdd(&totals[0], e);
        atomicAdd(&totals[1], s);
    }
    __syncthreads();
    for (int y = threadIdx.x; y < nbands; y += kThreads) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < kWarpsB; ++w) t += diff[w][y];
        m_band[(size_t)y * nblk + blockIdx.x] = (uint32_t)t;
    }
}

// The warp's kRankChunks x 32 items (chunk-major, lane order == list order)
// appended to the bands [lo, hi] they cover: band by band, the covering items
// of all chunks write consecutive slots from the band's cursor (coalesced runs,
// no per-item serial chain).  Each band is visited once per warp, so the
// cursor is read once and never written back (the warp owns cur[] and consumes
// it here).
__device__ __forceinline__ void warp_append_bands(const int (&lo)[kRankChunks],
                                                  const int (&hi)[kRankChunks],
                                                  const uint2 (&val)[kRankChunks],
                                                  const int* cur, uint2* out, int lane) {
    int l = lo[0], h = hi[0];
#pragma unroll
    for (int i = 1; i < kRankChunks; ++i) {
        l = min(l, lo[i]);
        h = max(h, hi[i]);
    }
    const int umin = __reduce_min_sync(0xffffffffu, l);
    const int umax = __reduce_max_sync(0xffffffffu, h);
    const unsigned lt = lanemask_lt();
    for (int b = umin; b <= umax; ++b) {
        bool in[kRankChunks];
        unsigned m[kRankChunks], any = 0u;
#pragma unroll
        for (int i = 0; i < kRankChunks; ++i) {
            in[i] = lo[i] <= b && b <= hi[i];
            m[i] = __ballot_sync(0xffffffffu, in[i]);
            any |= m[i];
        }
        if (any == 0u) continue;
        int base = cur[b];
#pragma unroll
        for (int i = 0; i < kRankChunks; ++i) {
            if (in[i]) out[base + __popc(m[i] & lt)] = val[i];
            base += __popc(m[i]);
        }
    }
}

// row-list item: the row and its inclusive tile-column span packed in 16+16 bits
__device__ __forceinline__ uint2 row_item(uint32_t row, short4 rc) {
    return make_uint2(row, (uint32_t)(uint16_t)rc.x | ((uint32_t)(uint16_t)rc.z << 16));
}

// L1c: stable scatter of each rank's row into the band lists
__global__ void __launch_bounds__(kThreads) k_band_scatter(const uint32_t* __restrict__ sorted_rows,
                                                           const short4* __restrict__ rect,
                                                           const int32_t* __restrict__ k_dev,
                                                           int nbands, uint32_t nblk,
                                                           const uint32_t* __restrict__ m_band_base,
                                                           const int32_t* __restrict__ overflow,
                                                           uint2* __restrict__ seg) {
    pdl_entry();
    __shared__ int diff[kWarpsB][kMaxBands + 1];
    if (*overflow) return;
    const uint32_t k = (uint32_t)*k_dev;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarpsB * (kMaxBands + 1); i += kThreads) (&diff[0][0])[i] = 0;
    __syncthreads();
    uint32_t rowv[kRankChunks];
    short4 rcv[kRankChunks];
    rank_load(sorted_rows, rect, k, blockIdx.x * kBlockItems + warp * kPerWarp, lane, rowv, rcv);
    rank_band_hist(rcv, diff[warp], lane, nbands, nullptr, nullptr);
    __syncthreads();
    // cursors: block base of the band + counts of the earlier warps
    for (int y = threadIdx.x; y < nbands; y += kThreads) {
        int run = (int)m_band_base[(size_t)y * nblk + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kWarpsB; ++w) {
            int c = diff[w][y];
            diff[w][y] = run;
            run += c;
        }
    }
    __syncthreads();
    int b0[kRankChunks], b1[kRankChunks];
    uint2 val[kRankChunks];
#pragma unroll
    for (int i = 0; i < kRankChunks; ++i) {
        const short4 rc = rcv[i];
        const bool ok = rect_ok(rc);
        b0[i] = ok ? rc.y / kBand : (1 << 30);
        b1[i] = ok ? rc.w / kBand : -1;
        val[i] = row_item(rowv[i], rc);
    }
    warp_append_bands(b0, b1, val, diff[warp], seg, lane);
}

// capacity check: E <= e_cap and S <= s_cap, else every later stage is a no-op
__global__ void k_bin_guard(const unsigned long long* __restrict__ totals, uint64_t e_cap,
                            uint64_t s_cap, int32_t* __restrict__ overflow,
                            float* __restrict__ skip_counter) {
    pdl_entry();
    if (threadIdx.x == 0) {
        const bool ovf = totals[0] > e_cap || totals[1] > s_cap;
        *overflow = ovf ? 1 : 0;
        // skip_counter = {non-finite count, overflow count}: the overflow has
        // its own slot so that, after the gradient all-reduce, every rank can
        // tell "some rank must re-run" from a non-finite skip whatever the
        // non-finite count
        if (ovf && skip_counter) atomicAdd(skip_counter + 1, 1.0f);
    }
}

// row-list starts (row-list path): row_start[y] = scanned m_band[y][0], [gy] = S
__global__ void k_row_starts(const uint32_t* __restrict__ band_base, int nbands, uint32_t nblk_r,
                             const unsigned long long* __restrict__ totals,
                             const int32_t* __restrict__ overflow, int32_t* __restrict__ row_start) {
    pdl_entry();
    const bool ovf = *overflow != 0;
    for (int y = threadIdx.x; y <= nbands; y += blockDim.x)
        row_start[y] = ovf ? 0 : (y < nbands ? (int32_t)band_base[(size_t)y * nblk_r]
                                             : (int32_t)totals[1]);
}

// block table of the band lists: level-2 blocks never cross bands
__global__ void __launch_bounds__(kThreads) k_seg_blocks(const uint32_t* __restrict__ band_base,
                                                         int nbands, uint32_t nblk_r,
                                                         const unsigned long long* __restrict__ totals,
                                                         const int32_t* __restrict__ overflow,
                                                         uint32_t* __restrict__ blk_start,
                                                         uint32_t* __restrict__ blk_band,
                                                         uint32_t* __restrict__ band_seg_start) {
    pdl_entry();
    __shared__ uint32_t s_tmp[kThreads / 32 + 1];
    const int y = threadIdx.x;
    const bool ovf = *overflow != 0;
    const uint32_t s_total = ovf ? 0u : (uint32_t)totals[1];
    uint32_t beg = 0, nb = 0;
    if (y < nbands && !ovf) {
        beg = band_base[(size_t)y * nblk_r];
        const uint32_t end = (y + 1 < nbands) ? band_base[(size_t)(y + 1) * nblk_r] : s_total;
        nb = (end - beg + kSegBlock - 1) / kSegBlock;
    }
    uint32_t tot;
    const uint32_t ex = block_exclusive_sum<kThreads, uint32_t>(nb, s_tmp, &tot);
    if (y < nbands) {
        blk_start[y] = ex;
        band_seg_start[y] = ovf ? 0u : beg;
        for (uint32_t j = 0; j < nb; ++j) blk_band[ex + j] = (uint32_t)y;
    }
    if (y == 0) {
        blk_start[nbands] = tot;
        band_seg_start[nbands] = s_total;
    }
}

// ---------------------------------------------------------------------------
// level 2: band lists -> tile lists
// ---------------------------------------------------------------------------
struct SegRange {
    int band;
    uint32_t s0, s1;
};

__device__ __forceinline__ SegRange seg_range(uint32_t b, const uint32_t* blk_start,
                                              const uint32_t* blk_band,
                                              const uint32_t* band_seg_start) {
    SegRange r;
    r.band = (int)blk_band[b];
    const uint32_t beg = band_seg_start[r.band], end = band_seg_start[r.band + 1];
    r.s0 = beg + (b - blk_start[r.band]) * kSegBlock;
    r.s1 = min(end, r.s0 + kSegBlock);
    return r;
}

// an item's cells inside the band: local rows [r0, r0+nr), columns [x0, x0+nx)
struct Cells {
    int r0, nr, x0, nx;
};

__device__ __forceinline__ void seg_load(const uint2* seg, const short4* rect, SegRange sr,
                                         int warp, int lane, uint32_t (&rw)[kSegChunks],
                                         Cells (&cl)[kSegChunks]) {
    static_assert(kBand == 1, "row items carry columns only");
    (void)rect;
    const uint32_t first = sr.s0 + warp * kSegPerWarp;
#pragma unroll
    for (int i = 0; i < kSegChunks; ++i) {
        const uint32_t s = first + i * 32 + lane;
        const uint2 it = s < sr.s1 ? __ldg(seg + s) : make_uint2(0xffffffffu, 0u);
        rw[i] = it.x;
        const int x0 = (int)(it.y & 0xffffu), x1 = (int)(it.y >> 16);
        Cells c;
        c.r0 = 0;
        c.nr = it.x != 0xffffffffu ? 1 : 0;
        c.x0 = x0;
        c.nx = c.nr ? x1 - x0 + 1 : 0;
        if (c.nx <= 0) c.nr = c.nx = 0;
        cl[i] = c;
    }
}

// per-warp cell histogram: one difference array row per band row
__device__ __forceinline__ void seg_cell_hist(const Cells (&cl)[kSegChunks], int* d, int lane,
                                              int gx) {
#pragma unroll
    for (int i = 0; i < kSegChunks; ++i) {
        const Cells c = cl[i];
        for (int r = 0; r < c.nr; ++r) {
            atomicAdd(&d[(c.r0 + r) * kXS + c.x0], 1);
            atomicAdd(&d[(c.r0 + r) * kXS + c.x0 + c.nx], -1);
        }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kBand; ++r) warp_scan_row(d + r * kXS, lane, gx);
}

// L2a: per block, entries per (band row, column) -> m_cell[b * 4gx + r*gx + x]
__global__ void __launch_bounds__(kThreads) k_cell_count(const uint2* __restrict__ seg,
                                                         const short4* __restrict__ rect, int gx,
                                                         const uint32_t* __restrict__ blk_start,
                                                         const uint32_t* __restrict__ blk_band,
                                                         const uint32_t* __restrict__ band_seg_start,
                                                         int nbands, uint32_t* __restrict__ m_cell) {
    pdl_entry();
    __shared__ int diff[kWarpsB][kBand * kXS];
    const uint32_t nblocks = blk_start[nbands];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ncell = kBand * gx;
    for (uint32_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        for (int i = threadIdx.x; i < kWarpsB * kBand * kXS; i += kThreads) (&diff[0][0])[i] = 0;
        __syncthreads();
        const SegRange sr = seg_range(b, blk_start, blk_band, band_seg_start);
        uint32_t rw[kSegChunks];
        Cells cl[kSegChunks];
        seg_load(seg, rect, sr, warp, lane, rw, cl);
        seg_cell_hist(cl, diff[warp], lane, gx);
        __syncthreads();
        for (int i = threadIdx.x; i < ncell; i += kThreads) {
            const int r = i / gx, x = i - r * gx;
            int t = 0;
#pragma unroll
            for (int w = 0; w < kWarpsB; ++w) t += diff[w][r * kXS + x];
            m_cell[(size_t)b * ncell + i] = (uint32_t)t;
        }
        __syncthreads();
    }
}

// L2b: per band, exclusive prefix of the cell counts over its blocks (in
// place) and the per-tile totals (tile = (4*band + r) * gx + x)
__global__ void __launch_bounds__(kThreads) k_cell_bandscan(uint32_t* __restrict__ m_cell, int gx,
                                                            int gy,
                                                            const uint32_t* __restrict__ blk_start,
                                                            uint32_t* __restrict__ tile_count) {
    pdl_entry();
    const int band = blockIdx.x;
    const uint32_t b0 = blk_start[band], b1 = blk_start[band + 1];
    const int ncell = kBand * gx;
    for (int i = threadIdx.x; i < ncell; i += kThreads) {
        uint32_t run = 0;
        uint32_t b = b0;
        for (; b + 8 <= b1; b += 8) {
            uint32_t t[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) t[j] = m_cell[(size_t)(b + j) * ncell + i];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                m_cell[(size_t)(b + j) * ncell + i] = run;
                run += t[j];
            }
        }
        for (; b < b1; ++b) {
            const uint32_t t = m_cell[(size_t)b * ncell + i];
            m_cell[(size_t)b * ncell + i] = run;
            run += t;
        }
        const int y = band * kBand + i / gx;
        if (y < gy) tile_count[y * gx + (i % gx)] = run;
    }
}

// L2c: stable scatter of each item's row into the tile lists, staged in shared
// memory grouped by cell so each tile run is written with coalesced stores
__global__ void __launch_bounds__(kThreads) k_cell_scatter(const uint2* __restrict__ seg,
                                                           const short4* __restrict__ rect, int gx,
                                                           int gy,
                                                           const uint32_t* __restrict__ blk_start,
                                                           const uint32_t* __restrict__ blk_band,
                                                           const uint32_t* __restrict__ band_seg_start,
                                                           int nbands,
                                                           const uint32_t* __restrict__ m_cell,
                                                           const int32_t* __restrict__ offsets,
                                                           int32_t* __restrict__ entries) {
    pdl_entry();
    __shared__ int diff[kWarpsB][kBand * kXS];
    __shared__ int s_loc[kBand * kMaxGX + 1];   // local run start per cell
    __shared__ int s_dst[kBand * kMaxGX];       // global run start per cell
    __shared__ int s_tmp[kThreads / 32 + 1];
    extern __shared__ int32_t s_stage[];
    const uint32_t nblocks = blk_start[nbands];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ncell = kBand * gx;
    constexpr int kCellsPerThread = kBand * kMaxGX / kThreads;  // 4
    for (uint32_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        for (int i = threadIdx.x; i < kWarpsB * kBand * kXS; i += kThreads) (&diff[0][0])[i] = 0;
        __syncthreads();
        const SegRange sr = seg_range(b, blk_start, blk_band, band_seg_start);
        uint32_t rw[kSegChunks];
        Cells cl[kSegChunks];
        seg_load(seg, rect, sr, warp, lane, rw, cl);
        seg_cell_hist(cl, diff[warp], lane, gx);
        __syncthreads();
        // per-cell block totals -> local run starts (4 consecutive cells per thread)
        int tot[kCellsPerThread];
        int my = 0;
#pragma unroll
        for (int j = 0; j < kCellsPerThread; ++j) {
            const int i = threadIdx.x * kCellsPerThread + j;
            tot[j] = 0;
            if (i < ncell) {
                const int r = i / gx, x = i - r * gx;
#pragma unroll
                for (int w = 0; w < kWarpsB; ++w) tot[j] += diff[w][r * kXS + x];
            }
            my += tot[j];
        }
        int block_total;
        int loc = block_exclusive_sum<kThreads, int>(my, s_tmp, &block_total);
        const bool staged = block_total <= kStageCap;
#pragma unroll
        for (int j = 0; j < kCellsPerThread; ++j) {
            const int i = threadIdx.x * kCellsPerThread + j;
            if (i < ncell) {
                const int r = i / gx, x = i - r * gx;
                const int y = sr.band * kBand + r;
                const int dst = y < gy ? offsets[y * gx + x] + (int)m_cell[(size_t)b * ncell + i] : 0;
                s_loc[i] = loc;
                s_dst[i] = dst;
                int run = staged ? loc : dst;
#pragma unroll
                for (int w = 0; w < kWarpsB; ++w) {
                    const int c = diff[w][r * kXS + x];
                    diff[w][r * kXS + x] = run;
                    run += c;
                }
            }
            loc += tot[j];
        }
        if (threadIdx.x == 0) s_loc[ncell] = block_total;
        __syncthreads();
        int32_t* out = staged ? s_stage : entries;
        int* cur = diff[warp];
#pragma unroll
        for (int i = 0; i < kSegChunks; ++i) {
            const Cells c = cl[i];
            const int cells = c.nr * c.nx;
            unsigned any = __ballot_sync(0xffffffffu, cells > 0);
            while (any) {
                const int j = __ffs(any) - 1;
                any &= any - 1;
                const int r0 = __shfl_sync(0xffffffffu, c.r0, j);
                const int x0 = __shfl_sync(0xffffffffu, c.x0, j);
                const int nx = __shfl_sync(0xffffffffu, c.nx, j);
                const int n = __shfl_sync(0xffffffffu, cells, j);
                const int32_t v = (int32_t)__shfl_sync(0xffffffffu, rw[i], j);
                const float rnx = __fdividef(1.0f, (float)nx);
                for (int l = lane; l < n; l += 32) {
                    const int r = (int)(((float)l + 0.5f) * rnx);  // l / nx, exact for l < 1024
                    const int bkt = (r0 + r) * kXS + x0 + (l - r * nx);
                    const int pos = cur[bkt];
                    cur[bkt] = pos + 1;
                    out[pos] = v;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (staged) {
            // one warp per cell run: coalesced copy-out
            for (int r = 0; r < kBand && sr.band * kBand + r < gy; ++r) {
                for (int x = warp; x < gx; x += kWarpsB) {
                    const int i = r * gx + x;
                    const int l0 = s_loc[i], n = s_loc[i + 1] - l0, d0 = s_dst[i];
                    for (int j = lane; j < n; j += 32) entries[d0 + j] = s_stage[l0 + j];
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// workspace plans
// ---------------------------------------------------------------------------
struct CountPlan {
    uint32_t* sorted_rows;        // rows in (depth, row) order
    uint32_t* tmp;                // scratch rows (long-bucket counting sort)
    depth_bucket::Meta* meta;     // -- zeroed per call: meta, scan status, bucket counts --
    unsigned* bticket;
    unsigned long long* bstat;
    uint32_t* bcount;             // [kBuckets]
    uint32_t* bstart;             // [kBuckets] starts, then ends
    uint32_t* wlist;              // buckets sorted by a warp / by a CTA
    uint32_t* clist;
    uint32_t* m_band;             // [nbands][nblk_r] counts, scanned in place
    unsigned long long* rstat;    // look-back status of the band scan (row-list path)
    unsigned* rticket;
    uint32_t nblk_r;
};

constexpr uint32_t kBucketScanTiles = depth_bucket::kBuckets / (kThreads * kScanIpt);
static_assert(depth_bucket::kBuckets % (kThreads * kScanIpt) == 0, "bucket scan tiling");

void plan_count(Workspace& ws, uint32_t k, int nbands, CountPlan& p) {
    const uint32_t kk = k > 0 ? k : 1;
    p.nblk_r = (uint32_t)ceil_div(kk, kBlockItems);
    p.sorted_rows = ws.take<uint32_t>(kk);
    p.tmp = ws.take<uint32_t>(kk);
    p.meta = ws.take<depth_bucket::Meta>(1);
    p.bticket = ws.take<unsigned>(1);
    p.bstat = ws.take<unsigned long long>(kBucketScanTiles);
    p.bcount = ws.take<uint32_t>(depth_bucket::kBuckets);
    p.bstart = ws.take<uint32_t>(depth_bucket::kBuckets);
    p.wlist = ws.take<uint32_t>(kk / (depth_bucket::kThreadRun + 1) + 1);
    p.clist = ws.take<uint32_t>(kk / 33 + 1);
    p.m_band = ws.take<uint32_t>((size_t)nbands * p.nblk_r);
    p.rstat = ws.take<unsigned long long>(ceil_div((size_t)nbands * p.nblk_r, kThreads * kScanIpt));
    p.rticket = ws.take<unsigned>(1);
}

struct EmitPlan {
    uint2* seg;
    uint32_t *blk_start, *blk_band, *band_seg_start;
    uint32_t* m_cell;
    uint32_t* tile_count;
    unsigned long long* status;  // scan look-back (band scan, tile scan)
    unsigned* tickets;
    uint32_t max_blocks;
};

void plan_emit(Workspace& ws, uint32_t s_cap, int gx, int gy, int nbands, uint32_t nblk_r,
               EmitPlan& p) {
    const uint32_t ss = s_cap > 0 ? s_cap : 1;
    p.max_blocks = (uint32_t)ceil_div(ss, kSegBlock) + (uint32_t)nbands;
    p.seg = ws.take<uint2>(ss);
    p.blk_start = ws.take<uint32_t>(nbands + 1);
    p.blk_band = ws.take<uint32_t>(p.max_blocks);
    p.band_seg_start = ws.take<uint32_t>(nbands + 1);
    p.m_cell = ws.take<uint32_t>((size_t)p.max_blocks * kBand * gx);
    p.tile_count = ws.take<uint32_t>((size_t)gx * gy);
    const size_t n1 = (size_t)nbands * nblk_r, n2 = (size_t)gx * gy;
    const size_t t1 = ceil_div(n1, kThreads * kScanIpt), t2 = ceil_div(n2, kThreads * kScanIpt);
    p.status = ws.take<unsigned long long>(t1 + t2);
    p.tickets = ws.take<unsigned>(2);
}

inline void grid_of(const uws_camera* cam, int* gx, int* gy, int* nbands) {
    *gx = (int)ceil_div(cam->width, kTile);
    *gy = (int)ceil_div(cam->height, kTile);
    *nbands = (int)ceil_div(*gy, kBand);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_bin_workspace_size(int64_t k, int64_t s, int32_t n_tiles_x, int32_t n_tiles_y,
                                      size_t* count_bytes, size_t* emit_bytes) {
    UWS_REQUIRE(k >= 0 && s >= 0 && n_tiles_x > 0 && n_tiles_y > 0,
                "uws_bin_workspace_size: bad argument");
    UWS_REQUIRE(k < (1ll << 31) && s < (1ll << 31), "uws_bin_workspace_size: size out of range");
    const int nbands = (int)ceil_div(n_tiles_y, kBand);
    Workspace w1(nullptr, 0, true);
    CountPlan cp;
    plan_count(w1, (uint32_t)k, nbands, cp);
    Workspace w2(nullptr, 0, true);
    EmitPlan ep;
    plan_emit(w2, (uint32_t)s, n_tiles_x, n_tiles_y, nbands, cp.nblk_r, ep);
    if (count_bytes) *count_bytes = w1.used;
    if (emit_bytes) *emit_bytes = w2.used;
    return UWS_OK;
}

extern "C" int uws_bin_count(const uws_projected* proj, int64_t k_cap, const uws_camera* cam,
                             int64_t* totals, void* count_ws, size_t count_bytes, void* stream) {
    UWS_REQUIRE(proj && cam && totals && proj->num_visible, "uws_bin_count: null argument");
    UWS_REQUIRE(k_cap >= 0 && k_cap < (1ll << 31), "uws_bin_count: k out of range");
    int gx, gy, nbands;
    grid_of(cam, &gx, &gy, &nbands);
    UWS_REQUIRE(gx <= kMaxGX && nbands <= kMaxBands, "uws_bin_count: image larger than 4096 px");
    cudaStream_t st = as_stream(stream);
    if (k_cap == 0) {
        UWS_CUDA(zero_async(totals, 2 * sizeof(int64_t), st));
        return UWS_OK;
    }
    Workspace ws(count_ws, count_bytes);
    CountPlan p;
    plan_count(ws, (uint32_t)k_cap, nbands, p);
    UWS_REQUIRE(ws.ok(), "uws_bin_count: workspace too small");
    namespace db = depth_bucket;
    // totals and the bucket sort's meta + counts, in one launch
    UWS_CUDA(zero_async2(totals, 2 * sizeof(int64_t), p.meta,
                         (char*)(p.bcount + db::kBuckets) - (char*)p.meta, st));
    const uint32_t kc = (uint32_t)k_cap;
    const uint32_t* k_dev = (const uint32_t*)proj->num_visible;
    // 0. order of the rows by (float64 depth bits, row): bucket the high words,
    //    then sort each bucket (depth_bucket.cuh)
    const uint64_t* dbits = (const uint64_t*)proj->depth;
    const unsigned kb = (unsigned)ceil_div(kc, 256);
    // the visible depths' high-word range: from the preprocess kernel when it wrote it
    const uint32_t* range = proj->depth_range;
    if (!range) {
        launch(db::k_hi_minmax, dim3(kb), dim3(256), 0, st, dbits, k_dev, kc, p.meta);
        UWS_CHECK_LAUNCH("k_hi_minmax");
        range = &p.meta->neg_min;
    }
    launch(db::k_bucket_count, dim3(kb), dim3(256), 0, st, dbits, k_dev, kc, range, p.bcount);
    UWS_CHECK_LAUNCH("k_bucket_count");
    launch(k_scan_u32, dim3(kBucketScanTiles), dim3(kThreads), 0, st, (const uint32_t*)p.bcount,
           p.bstart, db::kBuckets, (uint32_t*)nullptr, p.bstat, p.bticket);
    UWS_CHECK_LAUNCH("k_scan_u32");
    launch(db::k_bucket_scatter, dim3(kb), dim3(256), 0, st, dbits, k_dev, kc, range, p.bstart,
           p.sorted_rows);
    UWS_CHECK_LAUNCH("k_bucket_scatter");
    launch(db::k_bucket_fix, dim3(db::kBuckets / 256), dim3(256), 0, st, (const uint32_t*)p.bstart,
           dbits, p.sorted_rows, p.meta, p.wlist, p.clist);
    UWS_CHECK_LAUNCH("k_bucket_fix");
    launch(db::k_bucket_warp, dim3(148), dim3(256), 0, st, (const uint32_t*)p.bstart, dbits,
           p.sorted_rows, (const db::Meta*)p.meta, (const uint32_t*)p.wlist);
    UWS_CHECK_LAUNCH("k_bucket_warp");
    launch(db::k_bucket_cta, dim3(64), dim3(db::kCtaThreads), 0, st, (const uint32_t*)p.bstart, dbits,
           p.sorted_rows, (const db::Meta*)p.meta, (const uint32_t*)p.clist, p.tmp);
    UWS_CHECK_LAUNCH("k_bucket_cta");
    // 1a. per-block band histograms + totals (E entries, S band items)
    launch(k_band_count, dim3(p.nblk_r), dim3(kThreads), 0, st, p.sorted_rows, (const short4*)proj->rect,
                                                proj->num_visible, nbands, p.nblk_r, p.m_band,
                                                (unsigned long long*)totals);
    UWS_CHECK_LAUNCH("k_band_count");
    return UWS_OK;
}

extern "C" int uws_bin_emit(const uws_projected* proj, int64_t k_cap, int64_t e_cap, int64_t s_cap,
                            const uws_camera* cam, const int64_t* totals, int32_t* offsets,
                            int32_t* entries, int32_t* overflow, float* skip_counter,
                            void* count_ws, size_t count_bytes, void* emit_ws, size_t emit_bytes,
                            void* stream) {
    UWS_REQUIRE(proj && cam && offsets && totals && overflow, "uws_bin_emit: null argument");
    UWS_REQUIRE(k_cap >= 0 && e_cap >= 0 && e_cap < (1ll << 31) && s_cap >= 0 && s_cap < (1ll << 31),
                "uws_bin_emit: capacity out of range");
    cudaStream_t st = as_stream(stream);
    int gx, gy, nbands;
    grid_of(cam, &gx, &gy, &nbands);
    const int n_tiles = gx * gy;
    if (k_cap == 0) {
        UWS_CUDA(zero_async(offsets, sizeof(int32_t) * (n_tiles + 1), st));
        UWS_CUDA(zero_async(overflow, sizeof(int32_t), st));
        return UWS_OK;
    }
    Workspace w1(count_ws, count_bytes);
    CountPlan cp;
    plan_count(w1, (uint32_t)k_cap, nbands, cp);
    UWS_REQUIRE(w1.ok(), "uws_bin_emit: count workspace too small");
    Workspace w2(emit_ws, emit_bytes);
    EmitPlan ep;
    plan_emit(w2, (uint32_t)s_cap, gx, gy, nbands, cp.nblk_r, ep);
    UWS_REQUIRE(w2.ok(), "uws_bin_emit: emit workspace too small");
    const unsigned long long* tot = (const unsigned long long*)totals;
    const size_t n1 = (size_t)nbands * cp.nblk_r, n2 = (size_t)n_tiles;
    const size_t t1 = ceil_div(n1, kThreads * kScanIpt), t2 = ceil_div(n2, kThreads * kScanIpt);
    UWS_CUDA(zero_async(ep.status, (char*)(ep.tickets + 2) - (char*)ep.status, st));
    launch(k_bin_guard, dim3(1), dim3(32), 0, st, tot, (uint64_t)e_cap, (uint64_t)s_cap, overflow, skip_counter);
    UWS_CHECK_LAUNCH("k_bin_guard");
    // 1b. band-list bases: exclusive scan of m_band in (band, block) order
    launch(k_scan_u32, dim3((unsigned)t1), dim3(kThreads), 0, st, cp.m_band, cp.m_band, (uint32_t)n1, nullptr,
                                                  ep.status, ep.tickets);
    UWS_CHECK_LAUNCH("k_scan_u32(bands)");
    // 1c. stable scatter rank order -> band lists
    launch(k_band_scatter, dim3(cp.nblk_r), dim3(kThreads), 0, st, cp.sorted_rows, (const short4*)proj->rect,
                                                   proj->num_visible, nbands, cp.nblk_r, cp.m_band,
                                                   overflow, ep.seg);
    UWS_CHECK_LAUNCH("k_band_scatter");
    // 2a. block table of the band lists (all zero on overflow: later stages no-op)
    launch(k_seg_blocks, dim3(1), dim3(kThreads), 0, st, cp.m_band, nbands, cp.nblk_r, tot, overflow, ep.blk_start,
                                         ep.blk_band, ep.band_seg_start);
    UWS_CHECK_LAUNCH("k_seg_blocks");
    // level-2 kernels loop over blocks (count known only on the device):
    // launch a persistent grid instead of one CTA per possible block
    int n_sm = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned grid2 = (unsigned)std::min<uint32_t>(ep.max_blocks, (uint32_t)n_sm * 4u);
    launch(k_cell_count, dim3(grid2), dim3(kThreads), 0, st, ep.seg, (const short4*)proj->rect, gx, ep.blk_start,
                                             ep.blk_band, ep.band_seg_start, nbands, ep.m_cell);
    UWS_CHECK_LAUNCH("k_cell_count");
    launch(k_cell_bandscan, dim3(nbands), dim3(kThreads), 0, st, ep.m_cell, gx, gy, ep.blk_start, ep.tile_count);
    UWS_CHECK_LAUNCH("k_cell_bandscan");
    // 2b. CSR ranges = exclusive scan of the per-tile counts (tile = ty*gx + tx)
    launch(k_scan_u32, dim3((unsigned)t2), dim3(kThreads), 0, st, ep.tile_count, (uint32_t*)offsets, (uint32_t)n2,
                                                  (uint32_t*)offsets + n2, ep.status + t1,
                                                  ep.tickets + 1);
    UWS_CHECK_LAUNCH("k_scan_u32(tiles)");
    // 2c. stable scatter band lists -> tile lists
    static bool attr_set = false;
    if (!attr_set) {
        UWS_CUDA(cudaFuncSetAttribute(k_cell_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kStageCap * (int)sizeof(int32_t)));
        attr_set = true;
    }
    launch(k_cell_scatter, dim3(grid2), dim3(kThreads), kStageCap * sizeof(int32_t), st, 
        ep.seg, (const short4*)proj->rect, gx, gy, ep.blk_start, ep.blk_band, ep.band_seg_start,
        nbands, ep.m_cell, offsets, entries);
    UWS_CHECK_LAUNCH("k_cell_scatter");
    return UWS_OK;
}

extern "C" int uws_bin_rows(const uws_projected* proj, int64_t k_cap, int64_t s_cap,
                            const uws_camera* cam, const int64_t* totals, int32_t* row_start,
                            void* row_items_v, int32_t* overflow, float* skip_counter,
                            void* count_ws, size_t count_bytes, void* stream) {
    uint2* row_items = (uint2*)row_items_v;
    UWS_REQUIRE(proj && cam && totals && row_start && overflow, "uws_bin_rows: null argument");
    UWS_REQUIRE(k_cap >= 0 && s_cap >= 0 && s_cap < (1ll << 31), "uws_bin_rows: capacity out of range");
    static_assert(kBand == 1, "row lists need one tile row per band");
    cudaStream_t st = as_stream(stream);
    int gx, gy, nbands;
    grid_of(cam, &gx, &gy, &nbands);
    if (k_cap == 0) {
        UWS_CUDA(zero_async(row_start, sizeof(int32_t) * (gy + 1), st));
        UWS_CUDA(zero_async(overflow, sizeof(int32_t), st));
        return UWS_OK;
    }
    UWS_REQUIRE(row_items != nullptr, "uws_bin_rows: row_items is required");
    Workspace w1(count_ws, count_bytes);
    CountPlan cp;
    plan_count(w1, (uint32_t)k_cap, nbands, cp);
    UWS_REQUIRE(w1.ok(), "uws_bin_rows: count workspace too small");
    const unsigned long long* tot = (const unsigned long long*)totals;
    const size_t n1 = (size_t)nbands * cp.nblk_r;
    const size_t t1 = ceil_div(n1, kThreads * kScanIpt);
    UWS_CUDA(zero_async(cp.rstat, (char*)(cp.rticket + 1) - (char*)cp.rstat, st));
    // E is irrelevant here (no tile lists are materialised): only S is checked
    launch(k_bin_guard, dim3(1), dim3(32), 0, st, tot, ~0ull, (uint64_t)s_cap, overflow, skip_counter);
    UWS_CHECK_LAUNCH("k_bin_guard");
    launch(k_scan_u32, dim3((unsigned)t1), dim3(kThreads), 0, st, cp.m_band, cp.m_band, (uint32_t)n1, nullptr,
                                                  cp.rstat, cp.rticket);
    UWS_CHECK_LAUNCH("k_scan_u32(rows)");
    launch(k_band_scatter, dim3(cp.nblk_r), dim3(kThreads), 0, st, cp.sorted_rows, (const short4*)proj->rect,
                                                   proj->num_visible, nbands, cp.nblk_r, cp.m_band,
                                                   overflow, row_items);
    UWS_CHECK_LAUNCH("k_band_scatter");
    launch(k_row_starts, dim3(1), dim3(256), 0, st, cp.m_band, nbands, cp.nblk_r, tot, overflow, row_start);
    UWS_CHECK_LAUNCH("k_row_starts");
    return UWS_OK;
}
