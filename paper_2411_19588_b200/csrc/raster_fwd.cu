// K6 forward compositing with the underwater medium epilogue.
//
// Replaces the tile loop of rasterizer.render (rasterizer.py:188-241), the
// per-tile blend _composite_block (:148-178) and apply_water (:244-251) with
// logistic_remap (medium.py:26-29).
//
// One CTA per 16x16 tile, PIX vertically strided pixels per thread.  The
// tile's depth-sorted list is streamed through shared memory in batches of
// 256 records; every thread walks the batch front to back.  The walk is a
// tight loop that only leaves to a slow path when a pair's alpha lands in
// the float64 guard band of the 1/255 floor (rare), so the hot loop carries
// no float64 code.  A pixel stops once its transmittance drops below 1e-4 --
// the contributor that crosses the threshold is still blended, as in the
// reference -- and the CTA leaves as soon as all its pixels are done.  The
// per-pixel consumed-prefix length is written out so the backward kernel
// visits exactly the same pairs.
#include <cstdlib>

#include "raster_common.cuh"
#include "row_filter.cuh"

namespace uws {
namespace {

constexpr int kBatch = 256;

struct FwdArgs {
    const uws_splat* splat;
    const double* exact;
    const int32_t* offsets;      // tile lists (full binning) ...
    const int32_t* entries;
    const int32_t* row_start;    // ... or tile-row lists filtered on the fly
    const uint2* row_items;
    int width, height, gx;
    float far_plane;
    const float* medium;  // NULL = clean
    uws_raster_out out;
};

struct PixState {
    float T, cr, cg, cb, dsum, wsum;
    int count, last;
    bool done;
};

__device__ __forceinline__ void blend(PixState& s, float araw, const float4& c, float depth,
                                      int idx) {
    const float alpha = fminf(araw, kClampF);
    const float w = alpha * s.T;
    s.cr = fmaf(w, c.x, s.cr);
    s.cg = fmaf(w, c.y, s.cg);
    s.cb = fmaf(w, c.z, s.cb);
    s.dsum = fmaf(w, depth, s.dsum);
    s.wsum += w;
    s.T = s.T * (1.0f - alpha);
    ++s.count;
    s.last = idx;
    if (!(s.T >= kTStopF)) s.done = true;
}

template <int PIX, bool ROWS>
__global__ void __launch_bounds__(kRasterThreads / PIX, (PIX == 1 ? 3 : 4 * PIX / 2)) k_raster_fwd(FwdArgs a) {
    constexpr int THREADS = kRasterThreads / PIX;
    constexpr int ROWSTEP = kTile / PIX;
    static_assert(!ROWS || THREADS == kBatch, "row-list source needs one thread per batch slot");
    __shared__ float4 sP0[kBatch];  // mx, my, A, B
    __shared__ float4 sP1[kBatch];  // C, op, skip, depth
    __shared__ float4 sP2[kBatch];  // r, g, b, row
    __shared__ int sRow[ROWS ? kBatch + kChunk : 1];
    __shared__ int sScan[THREADS / 32];

    const int tile = blockIdx.x;
    const int ty = tile / a.gx, tx = tile - ty * a.gx;
    const int ox = tx * kTile, oy = ty * kTile;
    const int lx = threadIdx.x & (kTile - 1), ly0 = threadIdx.x / kTile;
    const float fx = (float)lx + 0.5f;

    PixState ps[PIX];
    float fy[PIX];
    bool inside[PIX];
    bool all_done = true;
#pragma unroll
    for (int p = 0; p < PIX; ++p) {
        const int ly = ly0 + p * ROWSTEP;
        fy[p] = (float)ly + 0.5f;
        inside[p] = (ox + lx) < a.width && (oy + ly) < a.height;
        ps[p] = PixState{1.0f, 0.f, 0.f, 0.f, 0.f, 0.f, 0, 0, !inside[p]};
        all_done &= ps[p].done;
    }

    int start = 0, end = 0, cur = 0, nst = 0;
    if (ROWS) {
        cur = a.row_start[ty];
        end = a.row_start[ty + 1];
    } else {
        start = a.offsets[tile];
        end = a.offsets[tile + 1];
    }
    int base = 0;  // tile-list entries consumed so far
    while (true) {
        if (__syncthreads_count(all_done) == THREADS) break;
        int n;
        if (ROWS) {
            // fill the staging list with >= 256 rows of this tile (or all that remain)
            while (nst < kBatch && cur < end) {
                nst += filter_chunk<THREADS>(a.row_items, cur, end, tx, sRow, nst,
                                             kBatch + kChunk, sScan);
                cur += kChunk;
            }
            n = min(nst, kBatch);
            if (n == 0) break;
            if (threadIdx.x < n) {
                StageA sa;
                StageB sb;
                StageC sc;
                stage_entry(a.splat, sRow[threadIdx.x], ox, oy, sa, sb, sc);
                sP0[threadIdx.x] = make_float4(sa.mx, sa.my, sa.A, sa.B);
                sP1[threadIdx.x] = make_float4(sb.C, sb.op, sb.skip, sb.depth);
                sP2[threadIdx.x] = make_float4(sc.r, sc.g, sc.b, __int_as_float(sc.row));
            }
        } else {
            if (start + base >= end) break;
            n = min(kBatch, end - start - base);
#pragma unroll
            for (int s = 0; s < kBatch / THREADS; ++s) {
                const int i = threadIdx.x + s * THREADS;
                if (i < n) {
                    StageA sa;
                    StageB sb;
                    StageC sc;
                    stage_entry(a.splat, a.entries[start + base + i], ox, oy, sa, sb, sc);
                    sP0[i] = make_float4(sa.mx, sa.my, sa.A, sa.B);
                    sP1[i] = make_float4(sb.C, sb.op, sb.skip, sb.depth);
                    sP2[i] = make_float4(sc.r, sc.g, sc.b, __int_as_float(sc.row));
                }
            }
        }
        __syncthreads();
        if (!all_done) {
            const int rel = base + 1;
#pragma unroll
            for (int p = 0; p < PIX; ++p) {
                PixState& s = ps[p];
                int k = 0;
                while (!s.done && k < n) {
                    // hot loop: float32 only
                    for (; k < n; ++k) {
                        const float4 p0 = sP0[k];
                        const float4 p1 = sP1[k];
                        const float dx = fx - p0.x, dy = fy[p] - p0.y;
                        const float power = dx * fmaf(p0.w, dy, p0.z * dx) + p1.x * dy * dy;
                        if (power < p1.z) continue;
                        const float araw = p1.y * ex2_ftz(power);
                        if (araw < kFloorHi) {
                            if (araw >= kFloorLo) break;  // guard band -> slow path
                            continue;
                        }
                        blend(s, araw, sP2[k], p1.w, rel + k);
                        if (s.done) break;
                    }
                    if (s.done || k >= n) break;
                    // slow path: float64 decision of alpha_raw >= 1/255 for entry k
                    const float4 p0 = sP0[k];
                    const float4 p1 = sP1[k];
                    const float4 p2 = sP2[k];
                    const float dx = fx - p0.x, dy = fy[p] - p0.y;
                    const float araw =
                        p1.y * ex2_ftz(dx * fmaf(p0.w, dy, p0.z * dx) + p1.x * dy * dy);
                    if (alpha_raw_f64(a.splat, a.exact, __float_as_int(p2.w), ox + lx,
                                      oy + ly0 + p * ROWSTEP) >= kFloor)
                        blend(s, araw, p2, p1.w, rel + k);
                    ++k;
                }
            }
            all_done = true;
#pragma unroll
            for (int p = 0; p < PIX; ++p) all_done &= ps[p].done;
        }
        base += n;
        if (ROWS) {
            // keep the staged rows beyond this batch for the next one
            __syncthreads();
            const int rem = nst - n;
            constexpr int KEEP = (kBatch + kChunk) / THREADS;
            int keep[KEEP];
#pragma unroll
            for (int q = 0; q < KEEP; ++q) {
                const int i = threadIdx.x + q * THREADS;
                keep[q] = i < rem ? sRow[n + i] : 0;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < KEEP; ++q) {
                const int i = threadIdx.x + q * THREADS;
                if (i < rem) sRow[i] = keep[q];
            }
            nst = rem;
        }
    }
#pragma unroll
    for (int p = 0; p < PIX; ++p) {
        if (!inside[p]) continue;
        const PixState& s = ps[p];
        const int pix = (oy + ly0 + p * ROWSTEP) * a.width + ox + lx;
        const float depth = s.count > 0 ? s.dsum / s.wsum : a.far_plane;
        a.out.depth[pix] = depth;
        a.out.weight[pix] = s.wsum;
        a.out.final_T[pix] = s.T;
        a.out.count[pix] = s.count;
        if (a.out.last) a.out.last[pix] = s.last;
        const float c3[3] = {s.cr, s.cg, s.cb};
        if (a.medium == nullptr) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                a.out.color[3 * pix + ch] = c3[ch];
                if (a.out.color_clean) a.out.color_clean[3 * pix + ch] = c3[ch];
            }
            continue;
        }
        // underwater epilogue: z = logistic(depth); C*exp(-Bd z) + Binf (1 - exp(-Bb z))
        const float z = 2.0f / (1.0f + expf(-(float)kLogisticRate * depth)) - 1.0f;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float att = expf(-a.medium[ch] * z);
            const float bs = a.medium[3 + ch] * (1.0f - expf(-a.medium[6 + ch] * z));
            a.out.color[3 * pix + ch] = c3[ch] * att + bs;
            a.out.color_clean[3 * pix + ch] = c3[ch];
            if (a.out.attenuation) a.out.attenuation[3 * pix + ch] = att;
            if (a.out.backscatter) a.out.backscatter[3 * pix + ch] = bs;
        }
    }
}

int fwd_pix() {
    static int pix = [] {
        const char* e = getenv("UWS_FWD_PIX");
        int v = e ? atoi(e) : 1;
        return (v == 2 || v == 4) ? v : 1;
    }();
    return pix;
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_raster_fwd(const uws_projected* proj, const int32_t* offsets,
                              const int32_t* entries, const uws_camera* cam, const float* medium,
                              uws_raster_out* out, void* stream) {
    UWS_REQUIRE(proj && offsets && cam && out, "uws_raster_fwd: null argument");
    UWS_REQUIRE(out->color && out->depth && out->weight && out->final_T && out->count,
                "uws_raster_fwd: missing output buffer");
    UWS_REQUIRE(medium == nullptr || out->color_clean != nullptr,
                "uws_raster_fwd: underwater mode needs color_clean");
    FwdArgs a;
    a.splat = proj->splat;
    a.exact = proj->exact;
    a.offsets = offsets;
    a.entries = entries;
    a.row_start = nullptr;
    a.row_items = nullptr;
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.far_plane = (float)cam->far_plane;
    a.medium = medium;
    a.out = *out;
    cudaStream_t st = as_stream(stream);
    switch (fwd_pix()) {
        case 2: k_raster_fwd<2, false><<<a.gx * gy, kRasterThreads / 2, 0, st>>>(a); break;
        case 4: k_raster_fwd<4, false><<<a.gx * gy, kRasterThreads / 4, 0, st>>>(a); break;
        default: k_raster_fwd<1, false><<<a.gx * gy, kRasterThreads, 0, st>>>(a); break;
    }
    UWS_CHECK_LAUNCH("k_raster_fwd");
    return UWS_OK;
}

extern "C" int uws_raster_fwd_rows(const uws_projected* proj, const int32_t* row_start,
                                   const void* row_items, const uws_camera* cam,
                                   const float* medium, uws_raster_out* out, void* stream) {
    UWS_REQUIRE(proj && row_start && cam && out, "uws_raster_fwd_rows: null argument");
    UWS_REQUIRE(out->color && out->depth && out->weight && out->final_T && out->count,
                "uws_raster_fwd_rows: missing output buffer");
    UWS_REQUIRE(medium == nullptr || out->color_clean != nullptr,
                "uws_raster_fwd_rows: underwater mode needs color_clean");
    FwdArgs a;
    a.splat = proj->splat;
    a.exact = proj->exact;
    a.offsets = nullptr;
    a.entries = nullptr;
    a.row_start = row_start;
    a.row_items = (const uint2*)row_items;
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.far_plane = (float)cam->far_plane;
    a.medium = medium;
    a.out = *out;
    k_raster_fwd<1, true><<<a.gx * gy, kRasterThreads, 0, as_stream(stream)>>>(a);
    UWS_CHECK_LAUNCH("k_raster_fwd_rows");
    return UWS_OK;
}
