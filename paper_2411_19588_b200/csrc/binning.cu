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
//   0. stable radix sort of the K visible rows by the bit pattern of their
//      float64 depth (positive doubles order like their bits; rows are in
//      source order, so stability yields the source-index tie-break);
//   1. rank order -> tile-ROW lists: each Gaussian is appended, in rank
//      order, to the list of every tile row its rectangle spans;
//   2. tile-row lists -> tile lists: each row segment is appended, in list
//      order, to every tile column it spans.
// A stable append needs, per (block of inputs, bucket), the number of earlier
// items in the same bucket.  Each 2048-item block is cut into 8 warp
// sub-blocks; a warp builds its interval histogram with two shared-memory
// atomics per item (difference array) and a warp scan, block totals are
// scanned across blocks (decoupled look-back), and each warp then walks its
// items IN ORDER, its lanes covering the item's buckets with private
// shared-memory cursors -- deterministic, no global atomics, bit-identical to
// the reference order given the same depths and rectangles.
#include "radix.cuh"

namespace uws {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpsB = kThreads / 32;
constexpr int kPerWarp = 256;                 // items per warp sub-block
constexpr int kBlockItems = kWarpsB * kPerWarp;  // 2048
constexpr int kMaxBins = 256;                 // max tile rows / tile columns
constexpr int kSegPerWarp = 128;              // T stage: segments per warp sub-block
constexpr int kSegBlock = kWarpsB * kSegPerWarp;  // 1024 segments per block
constexpr int kStageCap = 12288;              // entries staged in shared memory per block
constexpr int kScanIpt = 8;

__device__ __forceinline__ int rect_nx(short4 r) { return (int)r.z - (int)r.x + 1; }
__device__ __forceinline__ int rect_ny(short4 r) { return (int)r.w - (int)r.y + 1; }

// ---------------------------------------------------------------------------
// generic single-pass exclusive scan (u32 in, u32 out, total to *total)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_scan_u32(const uint32_t* __restrict__ in,
                                                       uint32_t* __restrict__ out, uint32_t n,
                                                       uint32_t* total,
                                                       unsigned long long* status,
                                                       unsigned* ticket) {
    __shared__ int s_tile;
    __shared__ unsigned long long s_scan[kThreads / 32 + 1];
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int tile = s_tile;
    const uint32_t first = (uint32_t)tile * kThreads * kScanIpt + threadIdx.x * kScanIpt;
    uint32_t v[kScanIpt];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) {
        v[j] = first + j < n ? in[first + j] : 0u;
        sum += v[j];
    }
    unsigned long long tot;
    unsigned long long ex = block_exclusive_sum<kThreads, unsigned long long>(sum, s_scan, &tot);
    if (threadIdx.x == 0) s_base = lookback_exclusive(status, tile, tot);
    __syncthreads();
    unsigned long long run = s_base + ex;
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) {
        if (first + j < n) out[first + j] = (uint32_t)run;
        run += v[j];
    }
    if (tile == (int)gridDim.x - 1 && threadIdx.x == kThreads - 1 && total)
        *total = (uint32_t)(s_base + tot);
}

// per-warp interval histogram: diff[w][lo] += 1, diff[w][hi+1] -= 1, then an
// in-place inclusive warp scan turns it into per-bucket counts of warp w
__device__ __forceinline__ void warp_hist_scan(int (*diff)[kMaxBins + 1], int warp, int lane,
                                               int nbins) {
    // each lane owns 8 consecutive bins (nbins <= 256)
    int* d = diff[warp];
    int b0 = lane * 8;
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
// stage 1: rank order -> tile-row lists
// ---------------------------------------------------------------------------
struct RankItem {
    uint32_t row;
    short4 rc;
};

__device__ __forceinline__ RankItem load_rank(const uint32_t* sorted_rows, const short4* rect,
                                              uint32_t r, uint32_t k) {
    RankItem it;
    if (r < k) {
        it.row = sorted_rows[r];
        it.rc = rect[it.row];
    } else {
        it.row = 0;
        it.rc = make_short4(0, 0, -1, -1);
    }
    return it;
}

constexpr int kRankChunks = kPerWarp / 32;

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

__device__ __forceinline__ void rank_warp_hist(const short4 (&rc)[kRankChunks], int warp,
                                               int (*diff)[kMaxBins + 1],
                                               unsigned long long* e_sum, unsigned long long* s_sum) {
    unsigned long long e = 0, s = 0;
#pragma unroll
    for (int i = 0; i < kRankChunks; ++i) {
        int nx = rect_nx(rc[i]), ny = rect_ny(rc[i]);
        if (nx > 0 && ny > 0) {
            atomicAdd(&diff[warp][rc[i].y], 1);
            atomicAdd(&diff[warp][rc[i].w + 1], -1);
            e += (unsigned long long)(nx * ny);
            s += (unsigned long long)ny;
        }
    }
    if (e_sum) {
        *e_sum = e;
        *s_sum = s;
    }
}

// R1: per 2048-rank block, entries per tile row -> m_row[y * nblk + b]; totals E, S
__global__ void __launch_bounds__(kThreads) k_rows_count(const uint32_t* __restrict__ sorted_rows,
                                                         const short4* __restrict__ rect,
                                                         const int32_t* __restrict__ k_dev,
                                                         int gy, uint32_t nblk,
                                                         uint32_t* __restrict__ m_row,
                                                         unsigned long long* totals) {
    __shared__ int diff[kWarpsB][kMaxBins + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t k = (uint32_t)*k_dev;
    for (int i = threadIdx.x; i < kWarpsB * (kMaxBins + 1); i += kThreads) (&diff[0][0])[i] = 0;
    __syncthreads();
    const uint32_t first = blockIdx.x * kBlockItems + warp * kPerWarp;
    unsigned long long e, s;
    uint32_t rowv[kRankChunks];
    short4 rcv[kRankChunks];
    rank_load(sorted_rows, rect, k, first, lane, rowv, rcv);
    rank_warp_hist(rcv, warp, diff, &e, &s);
    e = warp_sum(e);
    s = warp_sum(s);
    if (lane == 0) {
        atomicAdd(&totals[0], e);
        atomicAdd(&totals[1], s);
    }
    __syncthreads();
    warp_hist_scan(diff, warp, lane, gy);
    __syncthreads();
    for (int y = threadIdx.x; y < gy; y += kThreads) {
        int t = 0;
#pragma unroll
        for (int w = 0; w < kWarpsB; ++w) t += diff[w][y];
        m_row[(size_t)y * nblk + blockIdx.x] = (uint32_t)t;
    }
}

// R3: stable scatter of each rank's row into the tile-row lists
__global__ void __launch_bounds__(kThreads) k_rows_scatter(const uint32_t* __restrict__ sorted_rows,
                                                           const short4* __restrict__ rect,
                                                           const int32_t* __restrict__ k_dev,
                                                           int gy, uint32_t nblk,
                                                           const uint32_t* __restrict__ m_row_base,
                                                           const int32_t* __restrict__ overflow,
                                                           uint32_t* __restrict__ seg) {
    __shared__ int diff[kWarpsB][kMaxBins + 1];
    if (*overflow) return;
    const uint32_t k = (uint32_t)*k_dev;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarpsB * (kMaxBins + 1); i += kThreads) (&diff[0][0])[i] = 0;
    __syncthreads();
    const uint32_t first = blockIdx.x * kBlockItems + warp * kPerWarp;
    uint32_t rowv[kRankChunks];
    short4 rcv[kRankChunks];
    rank_load(sorted_rows, rect, k, first, lane, rowv, rcv);
    rank_warp_hist(rcv, warp, diff, nullptr, nullptr);
    __syncthreads();
    warp_hist_scan(diff, warp, lane, gy);
    __syncthreads();
    // cursors: block base of the row + counts of the earlier warps
    for (int y = threadIdx.x; y < gy; y += kThreads) {
        int run = (int)m_row_base[(size_t)y * nblk + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kWarpsB; ++w) {
            int c = diff[w][y];
            diff[w][y] = run;
            run += c;
        }
    }
    __syncthreads();
    int* cur = diff[warp];
#pragma unroll
    for (int i = 0; i < kRankChunks; ++i) {
        RankItem it;
        it.row = rowv[i];
        it.rc = rcv[i];
        int ny = rect_ny(it.rc), nx = rect_nx(it.rc);
        if (nx <= 0) ny = 0;
        unsigned any = __ballot_sync(0xffffffffu, ny > 0);
        while (any) {
            int j = __ffs(any) - 1;
            any &= any - 1;
            int y0 = __shfl_sync(0xffffffffu, (int)it.rc.y, j);
            int n = __shfl_sync(0xffffffffu, ny, j);
            uint32_t rw = __shfl_sync(0xffffffffu, it.row, j);
            for (int l = lane; l < n; l += 32) {
                int y = y0 + l;
                int pos = cur[y];
                cur[y] = pos + 1;
                seg[pos] = rw;
            }
            __syncwarp();
        }
    }
}

// capacity check: E <= e_cap and S <= s_cap, else every later stage is a no-op
__global__ void k_bin_guard(const unsigned long long* __restrict__ totals, uint64_t e_cap,
                            uint64_t s_cap, int32_t* __restrict__ overflow,
                            float* __restrict__ skip_counter) {
    if (threadIdx.x == 0) {
        const bool ovf = totals[0] > e_cap || totals[1] > s_cap;
        *overflow = ovf ? 1 : 0;
        // overflow is counted in units of 65536 so that, after the gradient
        // all-reduce, every rank can tell "some rank must re-run" from a
        // plain non-finite skip (which adds 1)
        if (ovf && skip_counter) atomicAdd(skip_counter, 65536.0f);
    }
}

// block table of the tile-row lists: blocks of 2048 segments never cross rows
__global__ void __launch_bounds__(kThreads) k_seg_blocks(const uint32_t* __restrict__ row_base,
                                                         int gy, uint32_t nblk_r,
                                                         const unsigned long long* __restrict__ totals,
                                                         const int32_t* __restrict__ overflow,
                                                         uint32_t* __restrict__ blk_start,
                                                         uint32_t* __restrict__ blk_row,
                                                         uint32_t* __restrict__ row_seg_start) {
    __shared__ uint32_t s_tmp[kThreads / 32 + 1];
    __shared__ uint32_t s_start[kMaxBins + 1];
    const int y = threadIdx.x;
    const bool ovf = *overflow != 0;
    const uint32_t s_total = ovf ? 0u : (uint32_t)totals[1];
    uint32_t beg = 0, len = 0, nb = 0;
    if (y < gy && !ovf) {
        beg = row_base[(size_t)y * nblk_r];
        uint32_t end = (y + 1 < gy) ? row_base[(size_t)(y + 1) * nblk_r] : s_total;
        len = end - beg;
        nb = (len + kSegBlock - 1) / kSegBlock;
        row_seg_start[y] = beg;
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_sum<kThreads, uint32_t>(nb, s_tmp, &tot);
    if (y < gy) {
        blk_start[y] = ex;
        s_start[y] = ex;
        if (ovf) row_seg_start[y] = 0;
    }
    if (y == 0) {
        blk_start[gy] = tot;
        row_seg_start[gy] = s_total;
    }
    __syncthreads();
    if (y < gy)
        for (uint32_t j = 0; j < nb; ++j) blk_row[ex + j] = (uint32_t)y;
}

// ---------------------------------------------------------------------------
// stage 2: tile-row lists -> tile lists
// ---------------------------------------------------------------------------
struct SegRange {
    int y;
    uint32_t s0, s1;  // segment range of this block
};

__device__ __forceinline__ SegRange seg_range(uint32_t b, const uint32_t* blk_start,
                                              const uint32_t* blk_row, const uint32_t* row_seg_start) {
    SegRange r;
    r.y = (int)blk_row[b];
    uint32_t local = b - blk_start[r.y];
    uint32_t beg = row_seg_start[r.y], end = row_seg_start[r.y + 1];
    r.s0 = beg + local * kSegBlock;
    r.s1 = min(end, r.s0 + kSegBlock);
    return r;
}

constexpr int kSegChunks = kSegPerWarp / 32;

// load this warp's segments (all chunks issued before use: memory-level parallelism)
__device__ __forceinline__ void seg_load(const uint32_t* seg, const short4* rect, SegRange sr,
                                         int warp, int lane, uint32_t (&rw)[kSegChunks],
                                         short4 (&rc)[kSegChunks]) {
    const uint32_t first = sr.s0 + warp * kSegPerWarp;
#pragma unroll
    for (int i = 0; i < kSegChunks; ++i) {
        uint32_t s = first + i * 32 + lane;
        rw[i] = s < sr.s1 ? __ldg(seg + s) : 0xffffffffu;
    }
#pragma unroll
    for (int i = 0; i < kSegChunks; ++i)
        rc[i] = rw[i] != 0xffffffffu ? __ldg(rect + rw[i]) : make_short4(0, 0, -1, 0);
}

__device__ __forceinline__ void seg_warp_hist(const short4 (&rc)[kSegChunks], int warp,
                                              int (*diff)[kMaxBins + 1]) {
#pragma unroll
    for (int i = 0; i < kSegChunks; ++i) {
        if (rc[i].z >= rc[i].x) {
            atomicAdd(&diff[warp][rc[i].x], 1);
            atomicAdd(&diff[warp][rc[i].z + 1], -1);
        }
    }
}

// T1: per block, entries per tile column -> m_col[b * gx + x]
__global__ void __launch_bounds__(kThreads) k_cols_count(const uint32_t* __restrict__ seg,
                                                         const short4* __restrict__ rect, int gx,
                                                         const uint32_t* __restrict__ blk_start,
                                                         const uint32_t* __restrict__ blk_row,
                                                         const uint32_t* __restrict__ row_seg_start,
                                                         int gy, uint32_t* __restrict__ m_col) {
    __shared__ int diff[kWarpsB][kMaxBins + 1];
    const uint32_t nblocks = blk_start[gy];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        for (int i = threadIdx.x; i < kWarpsB * (kMaxBins + 1); i += kThreads) (&diff[0][0])[i] = 0;
        __syncthreads();
        SegRange sr = seg_range(b, blk_start, blk_row, row_seg_start);
        uint32_t rw[kSegChunks];
        short4 rc[kSegChunks];
        seg_load(seg, rect, sr, warp, lane, rw, rc);
        seg_warp_hist(rc, warp, diff);
        __syncthreads();
        warp_hist_scan(diff, warp, lane, gx);
        __syncthreads();
        for (int x = threadIdx.x; x < gx; x += kThreads) {
            int t = 0;
#pragma unroll
            for (int w = 0; w < kWarpsB; ++w) t += diff[w][x];
            m_col[(size_t)b * gx + x] = (uint32_t)t;
        }
        __syncthreads();
    }
}

// T2a: per tile row, exclusive prefix of the column counts over its blocks
// (in place) and the per-tile totals
__global__ void __launch_bounds__(kThreads) k_cols_rowscan(uint32_t* __restrict__ m_col, int gx,
                                                           const uint32_t* __restrict__ blk_start,
                                                           uint32_t* __restrict__ tile_count) {
    const int y = blockIdx.x;
    const uint32_t b0 = blk_start[y], b1 = blk_start[y + 1];
    for (int x = threadIdx.x; x < gx; x += kThreads) {
        uint32_t run = 0;
        uint32_t b = b0;
        for (; b + 8 <= b1; b += 8) {
            uint32_t t[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = m_col[(size_t)(b + i) * gx + x];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                m_col[(size_t)(b + i) * gx + x] = run;
                run += t[i];
            }
        }
        for (; b < b1; ++b) {
            uint32_t t = m_col[(size_t)b * gx + x];
            m_col[(size_t)b * gx + x] = run;
            run += t;
        }
        tile_count[y * gx + x] = run;
    }
}

// T3: stable scatter of each segment's row into the tile lists.  The block's
// entries are first placed in shared memory grouped by tile column, then each
// column's run is written to HBM with coalesced stores (a block contributes
// one contiguous run to each tile list of its row).  Blocks whose entries do
// not fit the staging buffer scatter directly.
__global__ void __launch_bounds__(kThreads) k_cols_scatter(const uint32_t* __restrict__ seg,
                                                           const short4* __restrict__ rect, int gx,
                                                           const uint32_t* __restrict__ blk_start,
                                                           const uint32_t* __restrict__ blk_row,
                                                           const uint32_t* __restrict__ row_seg_start,
                                                           int gy, const uint32_t* __restrict__ m_col,
                                                           const int32_t* __restrict__ offsets,
                                                           int32_t* __restrict__ entries) {
    __shared__ int diff[kWarpsB][kMaxBins + 1];
    __shared__ int s_loc[kMaxBins + 1];    // local run start per column
    __shared__ int s_dst[kMaxBins];        // global run start per column
    __shared__ int s_tmp[kThreads / 32 + 1];
    extern __shared__ int32_t s_stage[];
    const uint32_t nblocks = blk_start[gy];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        for (int i = threadIdx.x; i < kWarpsB * (kMaxBins + 1); i += kThreads) (&diff[0][0])[i] = 0;
        __syncthreads();
        SegRange sr = seg_range(b, blk_start, blk_row, row_seg_start);
        uint32_t rwv[kSegChunks];
        short4 rcv[kSegChunks];
        seg_load(seg, rect, sr, warp, lane, rwv, rcv);
        seg_warp_hist(rcv, warp, diff);
        __syncthreads();
        warp_hist_scan(diff, warp, lane, gx);
        __syncthreads();
        // column totals of this block -> local run starts (one column per thread)
        int tot = 0;
        const int x = threadIdx.x;  // kThreads == kMaxBins
        if (x < gx) {
#pragma unroll
            for (int w = 0; w < kWarpsB; ++w) tot += diff[w][x];
        }
        int block_total;
        int loc = block_exclusive_sum<kThreads, int>(tot, s_tmp, &block_total);
        const bool staged = block_total <= kStageCap;
        if (x < gx) {
            const int dst = offsets[sr.y * gx + x] + (int)m_col[(size_t)b * gx + x];
            s_loc[x] = loc;
            s_dst[x] = dst;
            int run = staged ? loc : dst;
#pragma unroll
            for (int w = 0; w < kWarpsB; ++w) {
                int c = diff[w][x];
                diff[w][x] = run;
                run += c;
            }
        }
        if (x == 0) s_loc[gx] = block_total;
        __syncthreads();
        int32_t* out = staged ? s_stage : entries;
        int* cur = diff[warp];
#pragma unroll
        for (int i = 0; i < kSegChunks; ++i) {
            const uint32_t rw = rwv[i];
            const short4 rc = rcv[i];
            int nx = rect_nx(rc);
            unsigned any = __ballot_sync(0xffffffffu, nx > 0);
            while (any) {
                int j = __ffs(any) - 1;
                any &= any - 1;
                int x0 = __shfl_sync(0xffffffffu, (int)rc.x, j);
                int n = __shfl_sync(0xffffffffu, nx, j);
                uint32_t r = __shfl_sync(0xffffffffu, rw, j);
                for (int l = lane; l < n; l += 32) {
                    int xx = x0 + l;
                    int pos = cur[xx];
                    cur[xx] = pos + 1;
                    out[pos] = (int32_t)r;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (staged) {
            // one warp per column run: coalesced copy-out
            for (int xx = warp; xx < gx; xx += kWarpsB) {
                const int l0 = s_loc[xx], n = s_loc[xx + 1] - l0, d0 = s_dst[xx];
                for (int j = lane; j < n; j += 32) entries[d0 + j] = s_stage[l0 + j];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// workspace plans
// ---------------------------------------------------------------------------
struct CountPlan {
    uint64_t* depth_keys_sorted;
    uint32_t* sorted_rows;
    uint32_t* m_row;        // [gy][nblk_r] counts, scanned in place
    unsigned long long* totals;  // E, S
    uint64_t *k_alt, *k_tmp;
    uint32_t *v_alt, *v_tmp, *hist, *rstatus, *rtickets;
    uint32_t nblk_r;
};

void plan_count(Workspace& ws, uint32_t k, int gy, CountPlan& p) {
    uint32_t kk = k > 0 ? k : 1;
    p.nblk_r = (uint32_t)ceil_div(kk, kBlockItems);
    p.depth_keys_sorted = ws.take<uint64_t>(kk);
    p.sorted_rows = ws.take<uint32_t>(kk);
    p.m_row = ws.take<uint32_t>((size_t)gy * p.nblk_r);
    p.totals = ws.take<unsigned long long>(2);
    radix::plan<uint64_t>(ws, kk, 8, &p.k_alt, &p.v_alt, &p.k_tmp, &p.v_tmp, &p.hist, &p.rstatus,
                          &p.rtickets);
}

struct EmitPlan {
    uint32_t* seg;
    uint32_t *blk_start, *blk_row, *row_seg_start;
    uint32_t* m_col;
    uint32_t* tile_count;
    uint32_t* scan_total;
    unsigned long long* status;  // scan look-back (m_row scan, tile scan)
    unsigned* tickets;
    uint32_t max_blocks;
};

void plan_emit(Workspace& ws, uint32_t s_total, int gx, int gy, uint32_t nblk_r, EmitPlan& p) {
    uint32_t ss = s_total > 0 ? s_total : 1;
    p.max_blocks = (uint32_t)ceil_div(ss, kSegBlock) + (uint32_t)gy;
    p.seg = ws.take<uint32_t>(ss);
    p.blk_start = ws.take<uint32_t>(gy + 1);
    p.blk_row = ws.take<uint32_t>(p.max_blocks);
    p.row_seg_start = ws.take<uint32_t>(gy + 1);
    p.m_col = ws.take<uint32_t>((size_t)p.max_blocks * gx);
    p.tile_count = ws.take<uint32_t>((size_t)gx * gy);
    p.scan_total = ws.take<uint32_t>(2);
    size_t n1 = (size_t)gy * nblk_r, n2 = (size_t)gx * gy;
    size_t t1 = ceil_div(n1, kThreads * kScanIpt), t2 = ceil_div(n2, kThreads * kScanIpt);
    p.status = ws.take<unsigned long long>(t1 + t2);
    p.tickets = ws.take<unsigned>(2);
}

inline void grid_of(const uws_camera* cam, int* gx, int* gy) {
    *gx = (int)ceil_div(cam->width, kTile);
    *gy = (int)ceil_div(cam->height, kTile);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_bin_workspace_size(int64_t k, int64_t s, int32_t n_tiles_x, int32_t n_tiles_y,
                                      size_t* count_bytes, size_t* emit_bytes) {
    UWS_REQUIRE(k >= 0 && s >= 0 && n_tiles_x > 0 && n_tiles_y > 0,
                "uws_bin_workspace_size: bad argument");
    UWS_REQUIRE(k < (1ll << 31) && s < (1ll << 31), "uws_bin_workspace_size: size out of range");
    Workspace w1(nullptr, 0, true);
    CountPlan cp;
    plan_count(w1, (uint32_t)k, n_tiles_y, cp);
    Workspace w2(nullptr, 0, true);
    EmitPlan ep;
    plan_emit(w2, (uint32_t)s, n_tiles_x, n_tiles_y, cp.nblk_r, ep);
    if (count_bytes) *count_bytes = w1.used;
    if (emit_bytes) *emit_bytes = w2.used;
    return UWS_OK;
}

extern "C" int uws_bin_count(const uws_projected* proj, int64_t k_cap, const uws_camera* cam,
                             int64_t* totals, void* count_ws, size_t count_bytes, void* stream) {
    UWS_REQUIRE(proj && cam && totals && proj->num_visible, "uws_bin_count: null argument");
    UWS_REQUIRE(k_cap >= 0 && k_cap < (1ll << 31), "uws_bin_count: k out of range");
    int gx, gy;
    grid_of(cam, &gx, &gy);
    UWS_REQUIRE(gx <= kMaxBins && gy <= kMaxBins, "uws_bin_count: image wider/taller than 4096 px");
    cudaStream_t st = as_stream(stream);
    UWS_CUDA(cudaMemsetAsync(totals, 0, 2 * sizeof(int64_t), st));
    if (k_cap == 0) return UWS_OK;
    Workspace ws(count_ws, count_bytes);
    CountPlan p;
    plan_count(ws, (uint32_t)k_cap, gy, p);
    UWS_REQUIRE(ws.ok(), "uws_bin_count: workspace too small");
    const uint32_t kc = (uint32_t)k_cap;
    const uint32_t* k_dev = (const uint32_t*)proj->num_visible;
    // 0. stable sort of rows by float64 depth bits (8 digit passes)
    size_t meta = (char*)(p.rtickets + 8) - (char*)p.hist;
    UWS_CUDA(radix::sort_pairs<uint64_t>((const uint64_t*)proj->depth, nullptr, p.depth_keys_sorted,
                                         p.sorted_rows, kc, k_dev, 0, 8, p.k_tmp, p.v_tmp, p.hist,
                                         p.rstatus, p.rtickets, meta, st));
    // 1a. per-block tile-row histograms + totals (E entries, S row segments)
    k_rows_count<<<p.nblk_r, kThreads, 0, st>>>(p.sorted_rows, (const short4*)proj->rect,
                                                proj->num_visible, gy, p.nblk_r, p.m_row,
                                                (unsigned long long*)totals);
    UWS_CHECK_LAUNCH("k_rows_count");
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
    int gx, gy;
    grid_of(cam, &gx, &gy);
    const int n_tiles = gx * gy;
    if (k_cap == 0) {
        UWS_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (n_tiles + 1), st));
        UWS_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int32_t), st));
        return UWS_OK;
    }
    Workspace w1(count_ws, count_bytes);
    CountPlan cp;
    plan_count(w1, (uint32_t)k_cap, gy, cp);
    UWS_REQUIRE(w1.ok(), "uws_bin_emit: count workspace too small");
    Workspace w2(emit_ws, emit_bytes);
    EmitPlan ep;
    plan_emit(w2, (uint32_t)s_cap, gx, gy, cp.nblk_r, ep);
    UWS_REQUIRE(w2.ok(), "uws_bin_emit: emit workspace too small");
    const unsigned long long* tot = (const unsigned long long*)totals;
    const size_t n1 = (size_t)gy * cp.nblk_r, n2 = (size_t)n_tiles;
    const size_t t1 = ceil_div(n1, kThreads * kScanIpt), t2 = ceil_div(n2, kThreads * kScanIpt);
    UWS_CUDA(cudaMemsetAsync(ep.status, 0, (char*)(ep.tickets + 2) - (char*)ep.status, st));
    k_bin_guard<<<1, 32, 0, st>>>(tot, (uint64_t)e_cap, (uint64_t)s_cap, overflow, skip_counter);
    UWS_CHECK_LAUNCH("k_bin_guard");
    // 1b. row-list bases: exclusive scan of m_row in (row, block) order
    k_scan_u32<<<(unsigned)t1, kThreads, 0, st>>>(cp.m_row, cp.m_row, (uint32_t)n1, nullptr,
                                                  ep.status, ep.tickets);
    UWS_CHECK_LAUNCH("k_scan_u32(rows)");
    // 1c. stable scatter rank order -> tile-row lists
    k_rows_scatter<<<cp.nblk_r, kThreads, 0, st>>>(cp.sorted_rows, (const short4*)proj->rect,
                                                   proj->num_visible, gy, cp.nblk_r, cp.m_row,
                                                   overflow, ep.seg);
    UWS_CHECK_LAUNCH("k_rows_scatter");
    // 2a. block table of the row lists (all zero on overflow: later stages no-op)
    k_seg_blocks<<<1, kThreads, 0, st>>>(cp.m_row, gy, cp.nblk_r, tot, overflow, ep.blk_start,
                                         ep.blk_row, ep.row_seg_start);
    UWS_CHECK_LAUNCH("k_seg_blocks");
    const unsigned grid2 = ep.max_blocks;
    k_cols_count<<<grid2, kThreads, 0, st>>>(ep.seg, (const short4*)proj->rect, gx, ep.blk_start,
                                             ep.blk_row, ep.row_seg_start, gy, ep.m_col);
    UWS_CHECK_LAUNCH("k_cols_count");
    k_cols_rowscan<<<gy, kThreads, 0, st>>>(ep.m_col, gx, ep.blk_start, ep.tile_count);
    UWS_CHECK_LAUNCH("k_cols_rowscan");
    // 2b. CSR ranges = exclusive scan of the per-tile counts (tile = ty*gx + tx)
    k_scan_u32<<<(unsigned)t2, kThreads, 0, st>>>(ep.tile_count, (uint32_t*)offsets, (uint32_t)n2,
                                                  (uint32_t*)offsets + n2, ep.status + t1,
                                                  ep.tickets + 1);
    UWS_CHECK_LAUNCH("k_scan_u32(tiles)");
    // 2c. stable scatter tile-row lists -> tile lists
    static bool attr_set = false;
    if (!attr_set) {
        UWS_CUDA(cudaFuncSetAttribute(k_cols_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kStageCap * (int)sizeof(int32_t)));
        attr_set = true;
    }
    k_cols_scatter<<<grid2, kThreads, kStageCap * sizeof(int32_t), st>>>(
        ep.seg, (const short4*)proj->rect, gx, ep.blk_start, ep.blk_row, ep.row_seg_start, gy,
        ep.m_col, offsets, entries);
    UWS_CHECK_LAUNCH("k_cols_scatter");
    return UWS_OK;
}
