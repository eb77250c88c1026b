// Shared pieces of the forward and backward compositing kernels.
//
// Per-pair arithmetic is float32.  The three discontinuous gates of the
// reference (alpha_raw >= 1/255, alpha_raw < 0.99, T >= 1e-4;
// rasterizer.py:163-169, backward.py:151) are decided with float32 and, when
// alpha_raw falls inside a +-kGuard relative band around a threshold,
// re-decided from the float64 record exactly as the reference computes it.
#pragma once

#include "common.cuh"

namespace uws {

constexpr int kRasterThreads = kTile * kTile;  // one thread per pixel

// Staged record of one tile-list entry (tile-local mean for exact offsets).
struct __align__(16) StageA {
    float mx, my, ca, cb;  // mean relative to the tile origin, conic a, b
};
struct __align__(16) StageB {
    float cc, op, skip, r;  // conic c, opacity, log-threshold for early reject, red
};
struct __align__(8) StageC {
    float g, b;
};

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

// Gate decision for alpha_raw >= 1/255 given the float32 estimate.
__device__ __forceinline__ bool floor_pass(float araw, const uws_splat* splat, const double* exact,
                                           int row, int px, int py) {
    if (araw >= kFloorHi) return true;
    if (araw < kFloorLo) return false;
    return alpha_raw_f64(splat, exact, row, px, py) >= kFloor;
}

// Gate decision for alpha_raw < 0.99 (backward mask).
__device__ __forceinline__ bool below_clamp(float araw, const uws_splat* splat, const double* exact,
                                            int row, int px, int py) {
    if (araw < kClampLo) return true;
    if (araw >= kClampHi) return false;
    return alpha_raw_f64(splat, exact, row, px, py) < kClamp;
}

// Stage entry `row` of a tile whose origin is (ox, oy).
__device__ __forceinline__ void stage_entry(const uws_splat* __restrict__ splat, int row, int ox,
                                            int oy, StageA& a, StageB& b, StageC& c, float& depth) {
    const float4* p = reinterpret_cast<const float4*>(splat + row);
    float4 w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2);
    double mx, my;
    mx = __hiloint2double(__float_as_int(w0.y), __float_as_int(w0.x));
    my = __hiloint2double(__float_as_int(w0.w), __float_as_int(w0.z));
    a.mx = (float)(mx - (double)ox);
    a.my = (float)(my - (double)oy);
    a.ca = w1.x;
    a.cb = w1.y;
    b.cc = w1.z;
    b.op = w1.w;
    // alpha_raw < floor_lo  <=>  power < log(floor_lo / op); keep a margin so
    // float32 log/exp error can only send borderline pairs to the full test
    b.skip = __logf(kFloorLo / w1.w) - 1e-3f;
    b.r = w2.x;
    c.g = w2.y;
    c.b = w2.z;
    depth = w2.w;
}

}  // namespace uws
