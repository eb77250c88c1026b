// Shared pieces of the forward and backward compositing kernels.
//
// Per-pair arithmetic is float32.  The three discontinuous gates of the
// reference (alpha_raw >= 1/255, alpha_raw < 0.99, T >= 1e-4;
// rasterizer.py:163-169, backward.py:151) are decided with float32 and, when
// alpha_raw falls inside a +-kGuard relative band around a threshold,
// re-decided from the float64 record exactly as the reference computes it.
//
// Staged record layout (per tile-list entry, shared memory): the conic is
// pre-scaled by -0.5*log2(e) (and -log2(e) for the cross term) and the opacity
// is staged as its log2, so that
//     alpha_raw = 2^(dx*(A*dx + B*dy) + (C*dy*dy + lg2(opacity)))
// costs 2 FADD + 4 FMUL/FFMA + 1 MUFU.EX2 per pair (the C*dy*dy + lg2 term is
// one FFMA shared by the pixels of a row), and the mean is stored relative to
// the tile origin (computed in float64 -> exact local offsets).  Folding the
// opacity into the exponent adds at most half an ulp of |power| <= 8 to the
// exponent (3.3e-7 relative in alpha_raw), two orders below the guard band.
#pragma once

#include "common.cuh"

namespace uws {

constexpr int kRasterThreads = kTile * kTile;  // pixels per tile
constexpr float kLog2e = 1.4426950408889634f;

struct __align__(16) StageA {
    float mx, my, A, B;  // tile-local mean; -0.5*ca*log2e, -cb*log2e
};
struct __align__(16) StageB {
    // -0.5*cc*log2e, lg2(opacity), sure-pass threshold of the power WITHOUT the
    // opacity term (kPassLg2 - lop: used by the pass-region pre-filter), depth
    float C, lop, hi, depth;
};

// power >= hi       : alpha_raw is certainly >= kFloorHi (passes the 1/255 floor)
// power <  hi - kSkipDelta : alpha_raw is certainly <  kFloorLo (rejected)
// in between (a ~0.3% band of alpha_raw around 1/255): decide from alpha_raw as
// before, with the float64 re-evaluation inside the guard band.
// hi = lg2(kFloorHi/op) + 2e-3 and the old reject threshold lg2(kFloorLo/op) - 2e-3
// differ by log2(kFloorHi/kFloorLo) + 4e-3 = 0.0040866; the constant rounds up.
constexpr float kSkipDelta = 0.0041f;
// The same thresholds on the folded exponent power + lg2(opacity):
// lg2(kFloorHi) + 2e-3 = -7.99231 (rounded up), and below kSkipLg2 alpha_raw is
// certainly < kFloorLo (lg2(kFloorLo) = -7.99440).
constexpr float kPassLg2 = -7.9923f;
constexpr float kSkipLg2 = kPassLg2 - kSkipDelta;
// lg2(opacity) below this: alpha_raw <= opacity stays below the clamp guard
// band (lg2(kClampLo) - 1e-3 = -0.015543, rounded down)
constexpr float kLopClampLo = -0.0156f;
struct __align__(16) StageC {
    float r, g, b;
    int row;
};

__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2_ftz(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16-byte shared-memory load from a 32-bit shared-window address (keeps the
// base of a record array in one register instead of rematerialising it)
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// float64 alpha_raw exactly as the reference evaluates it (rasterizer.py:159-163)
__device__ __forceinline__ double alpha_raw_f64(const uws_splat* __restrict__ splat,
                                             const double* __restrict__ exact, int row, int px,
                                             int py) {
    const double mx = splat[row].mx, my = splat[row].my;
    const double4 e = reinterpret_cast<const double4*>(exact)[row];
    double dx = __dsub_rn((double)px + 0.5, mx);
    double dy = __dsub_rn((double)py + 0.5, my);
    double q = __dadd_rn(__dmul_rn(__dmul_rn(e.x, dx), dx), __dmul_rn(__dmul_rn(e.z, dy), dy));
    double power = __dsub_rn(__dmul_rn(-0.5, q), __dmul_rn(__dmul_rn(e.y, dx), dy));
    return __dmul_rn(e.w, exp(power));
}

// Out-of-line copy for loops that must stay free of float64 code.
static __device__ __noinline__ double alpha_raw_f64_cold(const uws_splat* __restrict__ splat,
                                                         const double* __restrict__ exact, int row,
                                                         int px, int py) {
    return alpha_raw_f64(splat, exact, row, px, py);
}

// Gate decision for alpha_raw >= 1/255 given the float32 estimate.
__device__ __forceinline__ bool floor_pass(float araw, const uws_splat* splat, const double* exact,
                                           int row, int px, int py) {
    if (araw >= kFloorHi) return true;
    if (araw < kFloorLo) return false;
    return alpha_raw_f64_cold(splat, exact, row, px, py) >= kFloor;
}

// Gate decision for alpha_raw < 0.99 (backward mask).
__device__ __forceinline__ bool below_clamp(float araw, const uws_splat* splat, const double* exact,
                                            int row, int px, int py) {
    if (araw < kClampLo) return true;
    if (araw >= kClampHi) return false;
    return alpha_raw_f64_cold(splat, exact, row, px, py) < kClamp;
}

__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Conservative tile-local box {ylo, yhi, xlo, xhi} of the region where the
// staged pair test `power >= hi - kSkipDelta` can hold: for the positive-definite form
// q = a dx^2 + b dx dy + c dy^2 <= Q (a = -A, b = -B, c = -C, Q = kSkipDelta - hi) the
// extents are |dy| <= sqrt(4aQ / (4ac - b^2)), |dx| <= sqrt(4cQ / (4ac - b^2)).
// A relative + absolute margin keeps it a strict superset of what the float32
// per-pixel test accepts; it is only a pre-filter.
__device__ __forceinline__ float4 stage_extent(const StageA& s, const StageB& t) {
    const float a = -s.A, b = -s.B, c = -t.C, Q = -(t.hi - kSkipDelta);
    if (Q < 0.f) return make_float4(1e30f, -1e30f, 1e30f, -1e30f);  // nothing passes
    const float det4 = 4.f * a * c - b * b;
    if (!(det4 > 0.f) || !(a > 0.f) || !(c > 0.f) || !(Q >= 0.f))
        return make_float4(-1e30f, 1e30f, -1e30f, 1e30f);  // degenerate/NaN: no pre-filter
    const float ey = sqrtf(4.f * a * Q / det4) * 1.001f + 0.01f;
    const float ex = sqrtf(4.f * c * Q / det4) * 1.001f + 0.01f;
    return make_float4(s.my - ey, s.my + ey, s.mx - ex, s.mx + ex);
}

// Exact x-range {xlo, xhi} (tile-local pixel-centre coordinates) of the region
// where `power >= hi - kSkipDelta` can hold, restricted to the pixel-centre rows
// y in [y0, y1]; empty (xlo > xhi) when the region misses those rows.  The
// region is the ellipse q = a dx^2 + b dx dy + c dy^2 <= Q of stage_extent,
// enlarged by 0.2% (+1e-3) so that it stays a superset of what the float32
// per-pixel test accepts.  Its rightmost point (ex, -b ex / 2c) and leftmost
// point (-ex, b ex / 2c) bound the range when their row lies in the strip;
// otherwise the range ends on the strip's boundary rows (the boundary x(dy)
// curves are concave / convex).
struct PassRegion {
    float mx, my, b, fourAQ, det4, ey, ex, yr, inv2a;
    int mode;  // 0: ellipse, 1: nothing passes, 2: no pre-filter (degenerate / NaN)

    __device__ __forceinline__ void init(const StageA& s, const StageB& t) {
        const float a = -s.A, c = -t.C;
        b = -s.B;
        mx = s.mx;
        my = s.my;
        const float Q = fmaf(-(t.hi - kSkipDelta), 1.002f, 1e-3f);
        det4 = 4.f * a * c - b * b;
        mode = 0;
        if (!(t.hi - kSkipDelta <= 0.f)) mode = 1;
        else if (!(det4 > 0.f) || !(a > 0.f) || !(c > 0.f) || !(Q >= 0.f)) mode = 2;
        fourAQ = 4.f * a * Q;
        ey = sqrtf(fourAQ / det4);
        ex = sqrtf(4.f * c * Q / det4);
        yr = -b * ex / (2.f * c);  // row of the rightmost point; the leftmost is at -yr
        inv2a = 0.5f / a;
    }

    __device__ __forceinline__ float2 xrange(float y0, float y1) const {
        if (mode == 1) return make_float2(1e30f, -1e30f);
        if (mode == 2) return make_float2(-1e30f, 1e30f);
        const float lo = fmaxf(y0 - my, -ey), hi = fminf(y1 - my, ey);
        if (lo > hi) return make_float2(1e30f, -1e30f);
        // boundary abscissae at the two (clipped) strip rows
        const float dl = sqrtf(fmaxf(fourAQ - det4 * lo * lo, 0.f));
        const float dh = sqrtf(fmaxf(fourAQ - det4 * hi * hi, 0.f));
        const float xmax = (yr >= lo && yr <= hi)
                               ? ex
                               : fmaxf((-b * lo + dl) * inv2a, (-b * hi + dh) * inv2a);
        const float xmin = (-yr >= lo && -yr <= hi)
                               ? -ex
                               : fminf((-b * lo - dl) * inv2a, (-b * hi - dh) * inv2a);
        return make_float2(mx + xmin - fmaf(1e-3f, fabsf(xmin), 0.01f),
                           mx + xmax + fmaf(1e-3f, fabsf(xmax), 0.01f));
    }
};

__device__ __forceinline__ float2 band_xrange(const StageA& s, const StageB& t, float y0, float y1) {
    PassRegion r;
    r.init(s, t);
    return r.xrange(y0, y1);
}

// Stage entry `row` of a tile whose origin is (ox, oy).
__device__ __forceinline__ void stage_entry(const uws_splat* __restrict__ splat, int row, int ox,
                                            int oy, StageA& a, StageB& b, StageC& c) {
    const float4* p = reinterpret_cast<const float4*>(splat + row);
    float4 w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2);
    double mx = __hiloint2double(__float_as_int(w0.y), __float_as_int(w0.x));
    double my = __hiloint2double(__float_as_int(w0.w), __float_as_int(w0.z));
    a.mx = (float)(mx - (double)ox);
    a.my = (float)(my - (double)oy);
    a.A = (-0.5f * kLog2e) * w1.x;
    a.B = (-kLog2e) * w1.y;
    b.C = (-0.5f * kLog2e) * w1.z;
    b.lop = lg2_ftz(w1.w);
    // alpha_raw >= floor_hi  <=  power + lop >= log2(floor_hi) + margin; the
    // margin (0.14% of alpha_raw) dwarfs the float32 lg2/ex2 error
    b.hi = kPassLg2 - b.lop;
    b.depth = w2.w;
    c.r = w2.x;
    c.g = w2.y;
    c.b = w2.z;
    c.row = row;
}

}  // namespace uws
