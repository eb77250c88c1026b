// K2-K5 binning: tile-key duplication, (tile, depth) ordering, tile ranges.
//
// Replaces rasterizer.bin_and_sort (rasterizer.py:50-85), whose order is
// lexsort((source_index, depth, tile_id)): tile ascending, then float64
// depth ascending, then source index.  Factorised into
//   1. a stable radix sort of the K visible rows by the bit pattern of their
//      float64 depth (positive doubles order like their bits; rows are in
//      source order, so stability gives the source-index tie-break),
//   2. per-rank tile counts + an exclusive scan (E on device),
//   3. emission of (tile, row) pairs in depth-rank order (warp-cooperative,
//      coalesced writes),
//   4. a stable radix sort of those pairs by tile id (depth order survives),
//   5. CSR tile ranges from the sorted tile ids.
// Every step is integer work, so the result is bit-identical to the
// reference given the same depths and rectangles.
#include "radix.cuh"

namespace uws {
namespace {

constexpr int kThreads = 256;
constexpr int kScanIpt = 8;

__device__ __forceinline__ uint32_t rect_count(short4 r) {
    int nx = (int)r.z - (int)r.x + 1, ny = (int)r.w - (int)r.y + 1;
    return (nx > 0 && ny > 0) ? (uint32_t)(nx * ny) : 0u;
}

// counts per depth rank + exclusive scan (decoupled look-back) -> emit offsets
__global__ void __launch_bounds__(kThreads) k_count_scan(const uint32_t* __restrict__ sorted_rows,
                                                         const short4* __restrict__ rect, uint32_t k,
                                                         uint64_t* __restrict__ emit_off,
                                                         int64_t* total_entries,
                                                         unsigned long long* status,
                                                         unsigned* ticket) {
    __shared__ int s_tile;
    __shared__ unsigned long long s_scan[kThreads / 32 + 1];
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int tile = s_tile;
    const uint32_t first = (uint32_t)tile * kThreads * kScanIpt + threadIdx.x * kScanIpt;
    uint32_t c[kScanIpt];
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) {
        uint32_t r = first + j;
        c[j] = r < k ? rect_count(rect[sorted_rows[r]]) : 0u;
        sum += c[j];
    }
    unsigned long long tot;
    unsigned long long ex = block_exclusive_sum<kThreads, unsigned long long>(sum, s_scan, &tot);
    if (threadIdx.x == 0) s_base = lookback_exclusive(status, tile, tot);
    __syncthreads();
    unsigned long long run = s_base + ex;
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) {
        uint32_t r = first + j;
        if (r < k) emit_off[r] = run;
        run += c[j];
    }
    if (tile == (int)gridDim.x - 1 && threadIdx.x == kThreads - 1)
        *total_entries = (int64_t)(s_base + tot);
}

// one warp handles 32 consecutive depth ranks; for each rank, the lanes write
// its rectangle's tiles (row-major, as the reference enumerates them)
__global__ void __launch_bounds__(kThreads) k_emit(const uint32_t* __restrict__ sorted_rows,
                                                   const short4* __restrict__ rect,
                                                   const uint64_t* __restrict__ emit_off, uint32_t k,
                                                   int gx, uint32_t* __restrict__ keys,
                                                   uint32_t* __restrict__ vals) {
    const int lane = threadIdx.x & 31;
    const uint32_t r = (blockIdx.x * kThreads + threadIdx.x);
    uint32_t row = 0, cnt = 0;
    uint64_t off = 0;
    short4 rc = make_short4(0, 0, -1, -1);
    if (r < k) {
        row = sorted_rows[r];
        rc = rect[row];
        cnt = rect_count(rc);
        off = emit_off[r];
    }
    for (int j = 0; j < 32; ++j) {
        uint32_t c = __shfl_sync(0xffffffffu, cnt, j);
        if (c == 0) continue;
        uint32_t rw = __shfl_sync(0xffffffffu, row, j);
        uint64_t o = __shfl_sync(0xffffffffu, off, j);
        int x0 = __shfl_sync(0xffffffffu, (int)rc.x, j);
        int y0 = __shfl_sync(0xffffffffu, (int)rc.y, j);
        int nx = __shfl_sync(0xffffffffu, (int)rc.z, j) - x0 + 1;
        for (uint32_t e = lane; e < c; e += 32) {
            uint32_t dy = e / (uint32_t)nx, dx = e - dy * (uint32_t)nx;
            keys[o + e] = (uint32_t)((y0 + (int)dy) * gx + x0 + (int)dx);
            vals[o + e] = rw;
        }
    }
}

// offsets[t] = first index whose tile >= t
__global__ void __launch_bounds__(kThreads) k_ranges(const uint32_t* __restrict__ tiles, uint32_t e,
                                                     int n_tiles, int32_t* __restrict__ offsets) {
    uint32_t i = blockIdx.x * kThreads + threadIdx.x;
    if (i > e) return;
    int cur = i < e ? (int)tiles[i] : n_tiles;
    int prev = i > 0 ? (int)tiles[i - 1] : -1;
    for (int t = prev + 1; t <= cur; ++t) offsets[t] = (int32_t)i;
}

struct CountPlan {
    uint64_t* depth_keys_sorted;
    uint32_t* sorted_rows;
    uint64_t* emit_off;
    unsigned long long* status;
    unsigned* ticket;
    uint64_t *k_alt, *k_tmp;
    uint32_t *v_alt, *v_tmp, *hist, *rstatus, *rtickets;
};

void plan_count(Workspace& ws, uint32_t k, CountPlan& p) {
    uint32_t kk = k > 0 ? k : 1;
    p.depth_keys_sorted = ws.take<uint64_t>(kk);
    p.sorted_rows = ws.take<uint32_t>(kk);
    p.emit_off = ws.take<uint64_t>(kk);
    int64_t scan_tiles = ceil_div(kk, kThreads * kScanIpt);
    p.status = ws.take<unsigned long long>(scan_tiles);
    p.ticket = ws.take<unsigned>(1);
    radix::plan<uint64_t>(ws, kk, 8, &p.k_alt, &p.v_alt, &p.k_tmp, &p.v_tmp, &p.hist, &p.rstatus,
                          &p.rtickets);
}

struct EmitPlan {
    uint32_t *keys, *keys_sorted, *vals;
    uint32_t *k_alt, *k_tmp, *v_alt, *v_tmp, *hist, *rstatus, *rtickets;
};

int tile_passes(int n_tiles) {
    int bits = 1;
    while ((1 << bits) < n_tiles) ++bits;
    return (bits + 7) / 8;
}

void plan_emit(Workspace& ws, uint32_t e, int n_tiles, EmitPlan& p) {
    uint32_t ee = e > 0 ? e : 1;
    p.keys = ws.take<uint32_t>(ee);
    p.vals = ws.take<uint32_t>(ee);
    p.keys_sorted = ws.take<uint32_t>(ee);
    radix::plan<uint32_t>(ws, ee, tile_passes(n_tiles), &p.k_alt, &p.v_alt, &p.k_tmp, &p.v_tmp,
                          &p.hist, &p.rstatus, &p.rtickets);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_bin_workspace_size(int64_t k, int64_t e, int32_t n_tiles, size_t* count_bytes,
                                      size_t* emit_bytes) {
    UWS_REQUIRE(k >= 0 && e >= 0 && n_tiles > 0, "uws_bin_workspace_size: bad argument");
    UWS_REQUIRE(k < (1ll << 31) && e < (1ll << 31), "uws_bin_workspace_size: size out of range");
    Workspace w1(nullptr, 0, true);
    CountPlan cp;
    plan_count(w1, (uint32_t)k, cp);
    Workspace w2(nullptr, 0, true);
    EmitPlan ep;
    plan_emit(w2, (uint32_t)e, n_tiles, ep);
    if (count_bytes) *count_bytes = w1.used;
    if (emit_bytes) *emit_bytes = w2.used;
    return UWS_OK;
}

extern "C" int uws_bin_count(const uws_projected* proj, int64_t k, const uws_camera* cam,
                             int64_t* total_entries, void* count_ws, size_t count_bytes,
                             void* stream) {
    UWS_REQUIRE(proj && cam && total_entries, "uws_bin_count: null argument");
    UWS_REQUIRE(k >= 0 && k < (1ll << 31), "uws_bin_count: k out of range");
    cudaStream_t st = as_stream(stream);
    if (k == 0) {
        UWS_CUDA(cudaMemsetAsync(total_entries, 0, sizeof(int64_t), st));
        return UWS_OK;
    }
    Workspace ws(count_ws, count_bytes);
    CountPlan p;
    plan_count(ws, (uint32_t)k, p);
    UWS_REQUIRE(ws.ok(), "uws_bin_count: workspace too small");
    const uint32_t kk = (uint32_t)k;
    // 1. stable sort of rows by float64 depth bits (8 digit passes)
    size_t meta = (char*)(p.rtickets + 8) - (char*)p.hist;
    UWS_CUDA(radix::sort_pairs<uint64_t>((const uint64_t*)proj->depth, nullptr, p.depth_keys_sorted,
                                         p.sorted_rows, kk, 0, 8, p.k_tmp, p.v_tmp, p.hist,
                                         p.rstatus, p.rtickets, meta, st));
    // 2. per-rank tile counts + scan
    int64_t scan_tiles = ceil_div(kk, kThreads * kScanIpt);
    UWS_CUDA(cudaMemsetAsync(p.status, 0, (char*)(p.ticket + 1) - (char*)p.status, st));
    k_count_scan<<<(unsigned)scan_tiles, kThreads, 0, st>>>(p.sorted_rows, (const short4*)proj->rect,
                                                            kk, p.emit_off, total_entries, p.status,
                                                            p.ticket);
    UWS_CHECK_LAUNCH("k_count_scan");
    return UWS_OK;
}

extern "C" int uws_bin_emit(const uws_projected* proj, int64_t k, int64_t e, const uws_camera* cam,
                            int32_t* offsets, int32_t* entries, void* count_ws, size_t count_bytes,
                            void* emit_ws, size_t emit_bytes, void* stream) {
    UWS_REQUIRE(proj && cam && offsets, "uws_bin_emit: null argument");
    UWS_REQUIRE(k >= 0 && e >= 0 && e < (1ll << 31), "uws_bin_emit: size out of range");
    cudaStream_t st = as_stream(stream);
    const int gx = (int)ceil_div(cam->width, kTile), gy = (int)ceil_div(cam->height, kTile);
    const int n_tiles = gx * gy;
    if (e == 0 || k == 0) {
        UWS_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (n_tiles + 1), st));
        return UWS_OK;
    }
    UWS_REQUIRE(entries != nullptr, "uws_bin_emit: entries is required");
    Workspace w1(count_ws, count_bytes);
    CountPlan cp;
    plan_count(w1, (uint32_t)k, cp);
    UWS_REQUIRE(w1.ok(), "uws_bin_emit: count workspace too small");
    Workspace w2(emit_ws, emit_bytes);
    EmitPlan ep;
    plan_emit(w2, (uint32_t)e, n_tiles, ep);
    UWS_REQUIRE(w2.ok(), "uws_bin_emit: emit workspace too small");
    const uint32_t kk = (uint32_t)k, ee = (uint32_t)e;
    k_emit<<<(unsigned)ceil_div(kk, kThreads), kThreads, 0, st>>>(
        cp.sorted_rows, (const short4*)proj->rect, cp.emit_off, kk, gx, ep.keys, ep.vals);
    UWS_CHECK_LAUNCH("k_emit");
    const int passes = tile_passes(n_tiles);
    size_t meta = (char*)(ep.rtickets + passes) - (char*)ep.hist;
    UWS_CUDA(radix::sort_pairs<uint32_t>(ep.keys, ep.vals, ep.keys_sorted, (uint32_t*)entries, ee, 0,
                                         passes, ep.k_tmp, ep.v_tmp, ep.hist, ep.rstatus,
                                         ep.rtickets, meta, st));
    k_ranges<<<(unsigned)ceil_div(ee + 1, kThreads), kThreads, 0, st>>>(ep.keys_sorted, ee, n_tiles,
                                                                        offsets);
    UWS_CHECK_LAUNCH("k_ranges");
    return UWS_OK;
}
