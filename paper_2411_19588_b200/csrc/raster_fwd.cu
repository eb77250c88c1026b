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
#include "raster_common.cuh"
#include "row_filter.cuh"
#include "scan.cuh"

namespace uws {
namespace {

constexpr int kBatch = 256;
constexpr int kFirstFill = 128;
constexpr int kListPad = 4;                    // per-warp lists are walked 4 entries at a time
constexpr int kFwdPx = 2;                      // pixels per thread (measured: 1 and 4 are slower)
constexpr int kFixBlocks = 148 * 3;            // float64 fix-up pass: 8 warps per block

#ifdef UWS_FIX_STATS
__device__ float g_dbg_eb[3840 * 2160];   // per pixel sum alpha/(1-alpha) of the float32 walk
__device__ float g_dbg_t32[3840 * 2160];  // float32 final T
__device__ int g_dbg_cnt32[3840 * 2160];
__device__ unsigned char g_dbg_flag[3840 * 2160];  // the adaptive band would re-walk the pixel
// max rel err, max rel / adaptive band, #count mismatches the adaptive band misses,
// #re-walked (the debug build re-walks the wide +-2e-3 band), #count mismatches
__device__ unsigned g_dbg_max[5];
__device__ unsigned long long g_dbg_ph2[2];   // pixels entering phase 2, phase-2 chunks scanned
#endif

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
    const double* depth64;  // float64 view depths (fix-up pass)
    uws_raster_out out;
};

// Transmittance band in which the float32 walk's T >= 1e-4 decision may differ
// from the reference's float64 one.  The float32 T carries a relative error of
// about c * sum_i alpha_i / (1 - alpha_i) over its blends (each factor 1 - alpha
// inherits alpha's relative error amplified by alpha / (1 - alpha)); measured
// with -DUWS_FIX_STATS (tools/dbg_fix2.py, ~1M re-walked pixels at C2, C3, C4
// and 1M @ 4K): c <= 1.65e-7 and max |T32 - T64| / T64 = 1.9e-6.  Near the
// threshold T ~ 1e-4 the sum is bounded a priori: alpha <= 0.99 gives
// alpha / (1 - alpha) <= 21.5 (-ln(1 - alpha)), and sum -ln(1 - alpha) = -ln T
// ~ 9.2, so the sum is <= 198 and the error <= 3.3e-5.  The band is +-1e-4 (3x
// that bound).  A pixel whose final T, or whose T before its last blend, lands
// in the band is re-walked in float64 by k_raster_fix (~0.1 % of the pixels;
// each blend lowers T by >= 0.39 %, so a walk visits the band at most once and
// that value is the final T or the T before the last blend).
constexpr float kTBandLo = 1e-4f * (1.0f - 1e-4f);
constexpr float kTBandHi = 1e-4f * (1.0f + 1e-4f);

__device__ __forceinline__ bool t_ambiguous(float t) { return t >= kTBandLo && t <= kTBandHi; }

#ifndef UWS_ADAPTIVE_BAND
#define UWS_ADAPTIVE_BAND 0
#endif
// Optional per-pixel band (-DUWS_ADAPTIVE_BAND=1): the walk accumulates eb = sum
// alpha / (1 - alpha) over its blends (one MUFU.RCP + FFMA per blend) and the band is
// +-(5e-7 eb + 2e-6) relative instead of the a-priori +-1e-4.  Validated with
// -DUWS_FIX_STATS on 1.5M re-walked pixels incl. opaque scenes (the error never
// exceeds 0.24 of that band, no count mismatch outside it) and ~10x fewer re-walks,
// but measured slower overall: the forward gains 47 us (spills, extra MUFU) for the
// ~20 us the smaller fix-up saves.
[[maybe_unused]] __device__ __forceinline__ bool t_ambiguous_eb(float t, float eb) {
    const float d = fmaf(5e-7f, eb, 2e-6f) * 1e-4f;
    return fabsf(t - 1e-4f) <= d;
}

// Write one pixel's forward outputs, with the underwater epilogue:
// z = logistic(depth); C exp(-Bd z) + Binf (1 - exp(-Bb z)) (rasterizer.py:244-251)
__device__ __forceinline__ void store_pixel(const FwdArgs& a, int pix, const float c3[3],
                                            float depth, float weight, float T, int count,
                                            int last) {
    a.out.depth[pix] = depth;
    a.out.weight[pix] = weight;
    a.out.final_T[pix] = T;
    a.out.count[pix] = count;
    if (a.out.last) a.out.last[pix] = last;
    if (a.medium == nullptr) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            a.out.color[3 * pix + ch] = c3[ch];
            if (a.out.color_clean) a.out.color_clean[3 * pix + ch] = c3[ch];
        }
        return;
    }
    const float z = 2.0f / (1.0f + __expf(-(float)kLogisticRate * depth)) - 1.0f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float att = __expf(-a.medium[ch] * z);
        const float bs = a.medium[3 + ch] * (1.0f - __expf(-a.medium[6 + ch] * z));
        a.out.color[3 * pix + ch] = c3[ch] * att + bs;
        a.out.color_clean[3 * pix + ch] = c3[ch];
        if (a.out.attenuation) a.out.attenuation[3 * pix + ch] = att;
        if (a.out.backscatter) a.out.backscatter[3 * pix + ch] = bs;
    }
}

// Bit b set <=> the staged box [ylo, yhi] reaches a pixel centre of band b
// (band b = rows R*b .. R*b + R - 1, nb bands).
template <int R, int NB>
__device__ __forceinline__ unsigned band_mask(float ylo, float yhi) {
    const float lo = fmaxf(ceilf((ylo - ((float)R - 0.5f)) * (1.0f / R)), 0.f);
    const float hi = fminf(floorf((yhi - 0.5f) * (1.0f / R)), (float)(NB - 1));
    if (!(lo <= hi)) return (ylo != ylo || yhi != yhi) ? ((1u << NB) - 1u) : 0u;  // NaN: no filter
    const unsigned l = (unsigned)lo, h = (unsigned)hi;
    return ((2u << h) - 1u) & ~((1u << l) - 1u);
}

// PX horizontally adjacent pixels per thread (1 or 2); a warp owns a band of
// 32*PX/16 rows.  The PX pixels of a thread share the record loads, dy and the
// C*dy*dy term; each pixel's power is the same float expression as in K8.
#ifndef UWS_FWD_MINB  // CTAs per SM (6 and 7 measured slower than 8 at PX = 2)
#define UWS_FWD_MINB(PX) (4 * (PX))
#endif
template <bool ROWS, int PX>
__global__ void __launch_bounds__(kRasterThreads / PX, UWS_FWD_MINB(PX)) k_raster_fwd(FwdArgs a) {
    // launched serially (no pdl_entry): the per-CTA L1 invalidation costs more here
    constexpr int kThreads = kRasterThreads / PX;
    constexpr int kWarps = kThreads / 32;
    constexpr int kBandRows = kTile / kWarps;
    constexpr int kLanesPerRow = kTile / PX;
    // staged records, 3 x float4 each (+1: a sentinel that never passes):
    //   [mx, my, A, B] [C, op, hi, depth] [r, g, b, row]
    __shared__ float4 sRec[3 * (kBatch + 1)];
    __shared__ unsigned char sMask[kBatch];
    __shared__ __align__(8) unsigned short sList[kWarps][kBatch + kListPad];
    __shared__ int sRow[ROWS ? kBatch + kChunk : 1];
    __shared__ int sScan[kWarps];

    const int tile = a.out.tile_order ? __ldg(a.out.tile_order + blockIdx.x) : (int)blockIdx.x;
    const int ty = tile / a.gx, tx = tile - ty * a.gx;
    const int ox = tx * kTile, oy = ty * kTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx0 = (lane % kLanesPerRow) * PX, ly = warp * kBandRows + lane / kLanesPerRow;
    const float fy = (float)ly + 0.5f;
    const int py = oy + ly;

    // pixel state; T = 0 marks a pixel outside the image as finished
    // (the blend weight sum is not accumulated: sum_i alpha_i T_i = 1 - T_final exactly,
    // and 1 - T_final is the more accurate float32 value of it)
    float fx[PX], T[PX], cr[PX], cg[PX], cb[PX], dsum[PX];
    float oml[PX];  // 1 - alpha of the last blend: T before it = T / oml (fix-up band test)
#if UWS_ADAPTIVE_BAND || defined(UWS_FIX_STATS)
    float eb[PX] = {};  // sum alpha / (1 - alpha) of the blends (float32 T error scale)
#endif
    int count[PX], last[PX];
    bool inside[PX];
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        fx[j] = (float)(lx0 + j) + 0.5f;
        inside[j] = ox + lx0 + j < a.width && py < a.height;
        T[j] = inside[j] ? 1.0f : 0.0f;
        cr[j] = cg[j] = cb[j] = dsum[j] = 0.f;
        oml[j] = 1.0f;
        count[j] = last[j] = 0;
    }
    auto alive = [&]() {
        bool any = false;
#pragma unroll
        for (int j = 0; j < PX; ++j) any |= T[j] >= kTStopF;
        return any;
    };
    if (threadIdx.x == 0) {
        sRec[3 * kBatch + 0] = make_float4(0.f, 0.f, 0.f, 0.f);
        sRec[3 * kBatch + 1] = make_float4(0.f, __int_as_float(0xff800000), __int_as_float(0x7f800000), 0.f);  // lg2(op) = -inf
        sRec[3 * kBatch + 2] = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    // 32-bit shared-window address of the record array, kept in one register
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sRec);
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
        if (__syncthreads_count(!alive()) == kThreads) break;
        int n;
        if (ROWS) {
            // fill the staging list with >= kFirstFill rows of this tile for the first
            // batch (most tiles saturate within ~150 entries: less filtering), then
            // >= kBatch rows (or all that remain)
            const int fill = base == 0 ? kFirstFill : kBatch;
            while (nst < fill && cur < end) {
                nst += filter_chunk<kThreads>(a.row_items, cur, end, tx, sRow, nst,
                                              kBatch + kChunk, sScan);
                cur += kChunk;
            }
            n = min(nst, kBatch);
            if (n == 0) break;
        } else {
            if (start + base >= end) break;
            n = min(kBatch, end - start - base);
        }
#pragma unroll
        for (int s = 0; s < kBatch / kThreads; ++s) {
            const int i = threadIdx.x + s * kThreads;
            if (i < n) {
                const int row = ROWS ? sRow[i] : a.entries[start + base + i];
                if (ROWS && a.out.tile_rows && base + i < a.out.tile_rows_cap)
                    a.out.tile_rows[(size_t)tile * a.out.tile_rows_cap + base + i] = row;
                StageA sa;
                StageB sb;
                StageC sc;
                stage_entry(a.splat, row, ox, oy, sa, sb, sc);
                sRec[3 * i + 0] = make_float4(sa.mx, sa.my, sa.A, sa.B);
                sRec[3 * i + 1] = make_float4(sb.C, sb.lop, sb.hi, sb.depth);
                sRec[3 * i + 2] = make_float4(sc.r, sc.g, sc.b, __int_as_float(sc.row));
                // bands whose rows the pass region reaches within the tile's columns
                PassRegion pr;
                pr.init(sa, sb);
                unsigned msk = 0u;
#pragma unroll
                for (int bnd = 0; bnd < kWarps; ++bnd) {
                    const float2 xr = pr.xrange((float)(bnd * kBandRows) + 0.5f,
                                                (float)(bnd * kBandRows + kBandRows) - 0.5f);
                    if (xr.y >= 0.5f && xr.x <= (float)kTile - 0.5f) msk |= 1u << bnd;
                }
                sMask[i] = (unsigned char)msk;
            }
        }
        __syncthreads();
        // this warp's entries: those whose box reaches its band, in list order
        int m = 0;
        if (__any_sync(0xffffffffu, alive())) {
            for (int c = 0; c < n; c += 32) {
                const int i = c + lane;
                const bool keep = i < n && ((sMask[i] >> warp) & 1u);
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (keep)  // index of the staged record
                    sList[warp][m + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)i;
                m += __popc(bal);
            }
            if (lane < kListPad) sList[warp][m + lane] = (unsigned short)kBatch;  // sentinel
            __syncwarp();
        }
        const int rel = base + 1;
#pragma unroll 1
        for (int jl = 0; jl < m && alive(); jl += kListPad) {
            const ushort4 q = *reinterpret_cast<const ushort4*>(&sList[warp][jl]);
            const int idx[kListPad] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int u = 0; u < kListPad; ++u) {
                const uint32_t ra = sbase + 48u * (uint32_t)idx[u];
                const float4 p0 = lds128(ra);
                const float4 p1 = lds128(ra + 16u);
                const float dy = fy - p0.y;
                const float qy = fmaf(p1.x * dy, dy, p1.y);  // + lg2(opacity)
                const float4 c = lds128(ra + 32u);
#pragma unroll
                for (int j = 0; j < PX; ++j) {
                    const float dx = fx[j] - p0.x;
                    // bitwise K8's expression: the forward and backward gate decisions agree
                    // even where float32 cancellation makes both differ from float64
                    // (thin, long ellipses far from their centre)
                    const float power = dx * fmaf(p0.w, dy, p0.z * dx) + qy;
                    auto blend = [&](float araw) {
                        const float alpha = fminf(araw, kClampF);
                        const float w = alpha * T[j];
                        cr[j] = fmaf(w, c.x, cr[j]);
                        cg[j] = fmaf(w, c.y, cg[j]);
                        cb[j] = fmaf(w, c.z, cb[j]);
                        dsum[j] = fmaf(w, p1.w, dsum[j]);
                        const float om = 1.0f - alpha;
                        oml[j] = om;
#if UWS_ADAPTIVE_BAND || defined(UWS_FIX_STATS)
                        eb[j] = fmaf(alpha, rcp_ftz(om), eb[j]);
#endif
                        T[j] = T[j] * om;
                        ++count[j];
                        last[j] = rel + idx[u];
                    };
                    // the sure pass first: one test on the common path
                    const bool live = T[j] >= kTStopF;
                    if (power >= kPassLg2 && live) {
                        blend(ex2_ftz(power));
                    } else if (power >= kSkipLg2 && live) {
                        // near the 1/255 floor (rare): float64 in the guard band
                        const float araw = ex2_ftz(power);
                        if (araw >= kFloorHi ||
                            (araw >= kFloorLo &&
                             alpha_raw_f64_cold(a.splat, a.exact, __float_as_int(c.w),
                                                ox + lx0 + j, py) >= kFloor))
                            blend(araw);
                    }
                }
            }
        }
        base += n;
        if (ROWS) {
            // keep the staged rows beyond this batch for the next one
            __syncthreads();
            const int rem = nst - n;
            constexpr int KEEP = (kBatch + kChunk) / kThreads;
            int keep[KEEP];
#pragma unroll
            for (int q = 0; q < KEEP; ++q) {
                const int i = threadIdx.x + q * kThreads;
                keep[q] = i < rem ? sRow[n + i] : 0;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < KEEP; ++q) {
                const int i = threadIdx.x + q * kThreads;
                if (i < rem) sRow[i] = keep[q];
            }
            nst = rem;
        }
    }
    // stored row count, flagged when it is the tile's whole list (nothing past it
    // for the fix-up pass to look for)
    if (ROWS && a.out.tile_rows && threadIdx.x == 0)
        a.out.tile_nrows[tile] = min(base, a.out.tile_rows_cap) |
                                 ((cur >= end && nst == 0 && base <= a.out.tile_rows_cap)
                                      ? kRowsComplete : 0);
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        if (!inside[j]) continue;
        const int pix = py * a.width + ox + lx0 + j;
        const float tbj = T[j] / oml[j];  // within ~1 ulp of the float32 T before the last blend
        const float wsum = 1.0f - T[j];
        const float depth = count[j] > 0 ? dsum[j] / wsum : a.far_plane;
        const float c3[3] = {cr[j], cg[j], cb[j]};
        store_pixel(a, pix, c3, depth, wsum, T[j], count[j], last[j]);
#ifdef UWS_FIX_STATS
        g_dbg_eb[pix] = eb[j];
        g_dbg_t32[pix] = T[j];
        g_dbg_cnt32[pix] = count[j];
#endif
#if defined(UWS_FIX_STATS)
        g_dbg_flag[pix] = t_ambiguous_eb(T[j], eb[j]) || t_ambiguous_eb(tbj, eb[j]);
        const bool amb = fabsf(T[j] - 1e-4f) <= 2e-7f || fabsf(tbj - 1e-4f) <= 2e-7f;
#elif UWS_ADAPTIVE_BAND
        const bool amb = t_ambiguous_eb(T[j], eb[j]) || t_ambiguous_eb(tbj, eb[j]);
#else
        const bool amb = t_ambiguous(T[j]) || t_ambiguous(tbj);
#endif
        if (a.out.fix_pixels && amb) {
            const int slot = atomicAdd(a.out.fix_count, 1);
            a.out.fix_pixels[slot] = pix;   // capacity H*W: one slot per pixel at most
        }
    }
}

// Float64 re-walk of the pixels whose float32 T >= 1e-4 decision was ambiguous
// (rasterizer.py:166-178 exactly: live_i = T_i >= 1e-4, alpha = min(raw, 0.99),
// raw < 1/255 -> 0): one warp per pixel, 32 list entries per step.  Every lane
// evaluates its entry's float64 alpha and loads its colour and depth; only the
// transmittance recurrence T_{i+1} = T_i (1 - alpha_i) -- the product the
// reference forms with cumprod, in the same order -- runs serially over the
// passing lanes, each lane keeping the T it was blended with; the weighted sums
// are then lane-parallel and reduced across the warp once at the end (the
// reference forms them as a BLAS product, in no particular order either).  The
// tile's list comes from the CSR tile lists, or the rows the forward stored per
// tile, or -- past what was stored -- from filtering the tile-row list.
// fix_count = {count, ticket}: the last block resets both, so the buffer is zero
// for the next call.
// One list entry as a lane sees it in the float64 re-walk.
struct FixEntry {
    double al;       // min(alpha_raw, 0.99) in float64
    double d;        // float64 view depth
    float r, g, b;   // colour
    bool ok;         // row present and alpha_raw >= 1/255
};

__device__ __forceinline__ FixEntry fix_load(const FwdArgs& a, int row, int px, int py) {
    FixEntry e;
    const double ar = row >= 0 ? alpha_raw_f64(a.splat, a.exact, row, px, py) : 0.0;
    e.ok = row >= 0 && ar >= kFloor;
    e.al = fmin(ar, kClamp);
    e.r = e.g = e.b = 0.f;
    e.d = 0.0;
    if (e.ok) {
        const float4 c = *reinterpret_cast<const float4*>(&a.splat[row].r);
        e.r = c.x; e.g = c.y; e.b = c.z;
        e.d = a.depth64[row];
    }
    return e;
}

struct FixWalk {
    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, dn = 0.0, ws = 0.0;  // c*/dn/ws: lane partials
    int count = 0, last = 0;
    bool done = false;

    // 32 list entries (lane entry e at list position pos), in list order
    __device__ __forceinline__ void step(const FixEntry& e, int pos, int lane) {
        unsigned pass = __ballot_sync(0xffffffffu, e.ok);
        if (!pass || done) return;
        double myT = 0.0;  // T this lane's entry is blended with (0: not blended)
        unsigned blended = 0u;
        while (pass) {
            const int s = __ffs(pass) - 1;
            pass &= pass - 1;
            if (T < kTStop) { done = true; break; }
            const double als = __shfl_sync(0xffffffffu, e.al, s);
            if (lane == s) myT = T;
            T *= 1.0 - als;
            blended |= 1u << s;
        }
        if (blended) {
            const int hi = 31 - __clz(blended);
            count += __popc(blended);
            last = __shfl_sync(0xffffffffu, pos, hi) + 1;
        }
        const double w = e.al * myT;
        c0 += w * (double)e.r;
        c1 += w * (double)e.g;
        c2 += w * (double)e.b;
        dn += w * e.d;
        ws += w;
    }
};

constexpr int kFixUnroll = 4;  // list chunks of 32 whose loads are in flight together

template <bool ROWS>
__global__ void __launch_bounds__(256) k_raster_fix(FwdArgs a) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int n = *(volatile int*)a.out.fix_count;
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nwarps) {
        const int pix = a.out.fix_pixels[i];
        const int py = pix / a.width, px = pix - py * a.width;
        const int ty = py / kTile, tx = px / kTile, tile = ty * a.gx + tx;
        // list source: [0, nlist) direct; then (ROWS) the row-list filter
        const int32_t* list;
        int nlist;
        bool complete = true;
        if (ROWS) {
            list = a.out.tile_rows ? a.out.tile_rows + (size_t)tile * a.out.tile_rows_cap : nullptr;
            const int nr = a.out.tile_rows ? a.out.tile_nrows[tile] : 0;
            nlist = nr & ~kRowsComplete;
            complete = (nr & kRowsComplete) != 0;
        } else {
            list = a.entries + a.offsets[tile];
            nlist = a.offsets[tile + 1] - a.offsets[tile];
        }
        FixWalk fw;
        // phase 1: the directly listed entries, kFixUnroll chunks of 32 at a time (the
        // dependent list -> record loads are latency-bound)
        for (int k0 = 0; k0 < nlist && !fw.done; k0 += 32 * kFixUnroll) {
            int row[kFixUnroll];
#pragma unroll
            for (int u = 0; u < kFixUnroll; ++u) {
                const int k = k0 + 32 * u + lane;
                row[u] = k < nlist ? list[k] : -1;
            }
            FixEntry e[kFixUnroll];
#pragma unroll
            for (int u = 0; u < kFixUnroll; ++u) e[u] = fix_load(a, row[u], px, py);
#pragma unroll
            for (int u = 0; u < kFixUnroll; ++u) fw.step(e[u], k0 + 32 * u + lane, lane);
        }
        // phase 2 (row lists, rare): the tile's entries past the stored ones
        if (ROWS && !complete && !fw.done && fw.T >= kTStop) {
            int seen = 0;  // matches of this tile so far, in list order
            const int rend = a.row_start[ty + 1];
#ifdef UWS_FIX_STATS
            if (lane == 0) atomicAdd(&g_dbg_ph2[0], 1ull);
#endif
            for (int c = a.row_start[ty]; c < rend && !fw.done; c += 32) {
#ifdef UWS_FIX_STATS
                if (lane == 0) atomicAdd(&g_dbg_ph2[1], 1ull);
#endif
                const int q = c + lane;
                const uint2 it = q < rend ? __ldg(a.row_items + q) : make_uint2(0u, 0xffffu);
                const bool m = (int)(it.y & 0xffffu) <= tx && tx <= (int)(it.y >> 16);
                const unsigned bal = __ballot_sync(0xffffffffu, m);
                const int pos = seen + __popc(bal & lanemask_lt());  // list position if m
                seen += __popc(bal);
                fw.step(fix_load(a, (m && pos >= nlist) ? (int)it.x : -1, px, py), pos, lane);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            fw.c0 += __shfl_xor_sync(0xffffffffu, fw.c0, o);
            fw.c1 += __shfl_xor_sync(0xffffffffu, fw.c1, o);
            fw.c2 += __shfl_xor_sync(0xffffffffu, fw.c2, o);
            fw.dn += __shfl_xor_sync(0xffffffffu, fw.dn, o);
            fw.ws += __shfl_xor_sync(0xffffffffu, fw.ws, o);
        }
#ifdef UWS_FIX_STATS
        if (lane == 0) {
            atomicAdd(&g_dbg_max[3], 1u);
            if (g_dbg_cnt32[pix] == fw.count) {
                const float rel = (float)(fabs((double)g_dbg_t32[pix] - fw.T) / fw.T);
                atomicMax(&g_dbg_max[0], __float_as_uint(rel));
                atomicMax(&g_dbg_max[1], __float_as_uint(rel / fmaf(5e-7f, g_dbg_eb[pix], 2e-6f)));
            } else {
                atomicAdd(&g_dbg_max[4], 1u);
                if (!g_dbg_flag[pix]) atomicAdd(&g_dbg_max[2], 1u);
            }
        }
#endif
        if (lane == 0) {
            const float c3[3] = {(float)fw.c0, (float)fw.c1, (float)fw.c2};
            const float depth = fw.ws > kWeightEps ? (float)(fw.dn / fw.ws) : a.far_plane;
            store_pixel(a, pix, c3, depth, (float)fw.ws, (float)fw.T, fw.count, fw.last);
        }
    }
    // reset {count, ticket} once every block has read the count
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.out.fix_count + 1, 1) == (int)gridDim.x - 1) {
            a.out.fix_count[2] = a.out.fix_count[0];  // pixels re-walked (diagnostic)
            a.out.fix_count[0] = 0;
            a.out.fix_count[1] = 0;
        }
    }
}

// Compositing schedule: the tiles by descending consumed-prefix length (the forward's
// tile_nrows / 8, capped at 127), by a one-CTA counting sort.  Tiles are independent, so
// any permutation gives the same images and gradients; launching the heaviest tiles
// first keeps a few long tiles from running alone at the end of the grid (measured:
// the forward's SMs were busy only ~79 % of its duration in raster order).
constexpr int kOrderThreads = 1024, kOrderIpt = 8;  // tiles per thread per chunk (8160 at 1080p)
constexpr int kOrderBuckets = 128;                    // cost / 8, capped

__device__ __forceinline__ void order_costs(const int32_t* __restrict__ nrows, int n, int c0,
                                            int (&bkt)[kOrderIpt]) {
    // a chunk's costs loaded up front: one global latency per chunk, not one per tile;
    // slot = bucket * 32 + lane (descending cost): a lane never shares a counter with
    // another lane of its warp (neighbouring tiles often cost the same: one counter per
    // bucket serialised the warp's shared atomics, ~10 us)
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < kOrderIpt; ++q) {
        const int i = c0 + (int)threadIdx.x + q * kOrderThreads;
        const int c = i < n ? min(__ldg(nrows + i) & ~kRowsComplete, 8 * kOrderBuckets - 1) : 0;
        bkt[q] = i < n ? (kOrderBuckets - 1 - (c >> 3)) * 32 + lane : -1;
    }
}

__global__ void __launch_bounds__(kOrderThreads) k_tile_order(const int32_t* __restrict__ nrows,
                                                              int n, int32_t* __restrict__ order) {
    pdl_entry();
    constexpr int kChunk = kOrderThreads * kOrderIpt;
    constexpr int kSlots = kOrderBuckets * 32;
    constexpr int kPer = kSlots / kOrderThreads;  // consecutive slots scanned per thread
    __shared__ int hist[kSlots];
    __shared__ int sred[kOrderThreads / 32 + 1];
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < kPer; ++k) hist[t + k * kOrderThreads] = 0;
    __syncthreads();
    int bkt[kOrderIpt];
    for (int c0 = 0; c0 < n; c0 += kChunk) {
        order_costs(nrows, n, c0, bkt);
#pragma unroll
        for (int q = 0; q < kOrderIpt; ++q)
            if (bkt[q] >= 0) atomicAdd(&hist[bkt[q]], 1);
    }
    __syncthreads();
    int v[kPer], run = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        v[k] = run;
        run += hist[t * kPer + k];
    }
    int total;
    const int ex = block_exclusive_sum<kOrderThreads, int>(run, sred, &total);
#pragma unroll
    for (int k = 0; k < kPer; ++k) hist[t * kPer + k] = ex + v[k];  // (own slots, read above)
    __syncthreads();
    for (int c0 = 0; c0 < n; c0 += kChunk) {
        if (c0 > 0 || n > kChunk) order_costs(nrows, n, c0, bkt);
#pragma unroll
        for (int q = 0; q < kOrderIpt; ++q)
            if (bkt[q] >= 0)
                order[atomicAdd(&hist[bkt[q]], 1)] = c0 + t + q * kOrderThreads;
    }
}

}  // namespace
}  // namespace uws

using namespace uws;

#ifdef UWS_FIX_STATS
extern "C" int uws_debug_ph2_stats(unsigned long long* out2) {
    cudaMemcpyFromSymbol(out2, g_dbg_ph2, sizeof(unsigned long long) * 2);
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_dbg_ph2, z, sizeof(z));
    return 0;
}
extern "C" int uws_debug_fix_stats(unsigned* out5) {
    cudaMemcpyFromSymbol(out5, g_dbg_max, sizeof(unsigned) * 5);
    unsigned z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_dbg_max, z, sizeof(z));
    return 0;
}
#endif

extern "C" int uws_raster_fwd(const uws_projected* proj, const int32_t* offsets,
                              const int32_t* entries, const uws_camera* cam, const float* medium,
                              uws_raster_out* out, void* stream) {
    UWS_REQUIRE(proj && offsets && cam && out, "uws_raster_fwd: null argument");
    UWS_REQUIRE(out->color && out->depth && out->weight && out->final_T && out->count,
                "uws_raster_fwd: missing output buffer");
    UWS_REQUIRE(medium == nullptr || out->color_clean != nullptr,
                "uws_raster_fwd: underwater mode needs color_clean");
    UWS_REQUIRE(out->fix_pixels == nullptr || out->fix_count != nullptr,
                "uws_raster_fwd: fix_pixels needs fix_count");
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
    a.depth64 = proj->depth;
    a.out = *out;
    launch_serial(k_raster_fwd<false, kFwdPx>, dim3(a.gx * gy), dim3(kRasterThreads / kFwdPx), 0, as_stream(stream), a);
    UWS_CHECK_LAUNCH("k_raster_fwd");
    if (out->fix_pixels) {
        launch(k_raster_fix<false>, dim3(kFixBlocks), dim3(256), 0, as_stream(stream), a);
        UWS_CHECK_LAUNCH("k_raster_fix");
    }
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
    UWS_REQUIRE(out->fix_pixels == nullptr || out->fix_count != nullptr,
                "uws_raster_fwd_rows: fix_pixels needs fix_count");
    UWS_REQUIRE(out->tile_rows == nullptr || (out->tile_nrows && out->tile_rows_cap > 0),
                "uws_raster_fwd_rows: tile_rows needs tile_nrows and a positive cap");
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
    a.depth64 = proj->depth;
    a.out = *out;
    launch_serial(k_raster_fwd<true, kFwdPx>, dim3(a.gx * gy), dim3(kRasterThreads / kFwdPx), 0, as_stream(stream), a);
    UWS_CHECK_LAUNCH("k_raster_fwd_rows");
    if (out->fix_pixels) {
        launch(k_raster_fix<true>, dim3(kFixBlocks), dim3(256), 0, as_stream(stream), a);
        UWS_CHECK_LAUNCH("k_raster_fix_rows");
    }
    return UWS_OK;
}

extern "C" int uws_tile_order(const int32_t* tile_nrows, int32_t n_tiles, int32_t* order,
                              void* stream) {
    UWS_REQUIRE(tile_nrows && order && n_tiles >= 0, "uws_tile_order: bad argument");
    if (n_tiles == 0) return UWS_OK;
    launch(k_tile_order, dim3(1), dim3(kOrderThreads), 0, as_stream(stream), tile_nrows, (int)n_tiles,
           order);
    UWS_CHECK_LAUNCH("k_tile_order");
    return UWS_OK;
}
