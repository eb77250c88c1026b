// K8 backward compositing + medium-parameter gradients.
//
// Replaces backward._backward_block (backward.py:124-163), the per-tile loop
// and fixed-order merge of backward_render (:278-344), and backward_medium
// (:261-275).
//
// One CTA per tile, one thread per pixel, walking the tile list BACK to
// front over exactly the prefix the forward consumed (per-pixel `last`).
// Transmittance is recovered as T_i = T_{i+1} / (1 - alpha_i) from the
// stored final transmittance, and the suffix sum_{j>i} w_j (G . c_j) of the
// reference's reverse cumsum (:149) is carried as one scalar per pixel, so no
// per-pair state is stored.  Alpha and its gates are recomputed with the
// forward's exact arithmetic, hence identical decisions.
//
// The 9 per-(pixel, Gaussian) partials (dpower, dpower*dx, dpower*dy,
// dpower*dx^2, dpower*dx*dy, dpower*dy^2, w*G) are reduced across the warp
// with a transposed butterfly (14 shuffles instead of 45), accumulated over
// the CTA's 8 warps in shared memory, chained through the conic once per
// (tile, Gaussian) and only then sent to HBM with 9 atomics.
#include "raster_common.cuh"

namespace uws {
namespace {

constexpr int kWarps = kRasterThreads / 32;

struct BwdArgs {
    const uws_splat* splat;
    const double* exact;
    const int32_t* offsets;
    const int32_t* entries;
    int width, height, gx;
    const float* medium;
    const float* color_clean;
    const float* depth;
    const float* final_T;
    const int32_t* last;
    const float* dL;
    float* screen;       // [K][9]
    double* medium_acc;  // [9]
};

// Reduce v[0..7] across the warp; returns the full sum of value index
// ((lane>>4)&1)*4 + ((lane>>3)&1)*2 + ((lane>>2)&1) (valid in every lane).
__device__ __forceinline__ float butterfly8(float v[8], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    float h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float send = b4 ? v[i] : v[i + 4];
        float keep = b4 ? v[i + 4] : v[i];
        h[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float q[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        float send = b3 ? h[i] : h[i + 2];
        float keep = b3 ? h[i + 2] : h[i];
        q[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float send = b2 ? q[0] : q[1];
    float r = (b2 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

__global__ void __launch_bounds__(kRasterThreads, 3) k_raster_bwd(BwdArgs a) {
    __shared__ StageA sA[kRasterThreads];
    __shared__ StageB sB[kRasterThreads];
    __shared__ StageC sC[kRasterThreads];
    __shared__ int sRow[kRasterThreads];
    __shared__ float sAcc[9][kRasterThreads];
    __shared__ float sMed[kWarps][9];
    __shared__ int sMaxLast;

    const int tile = blockIdx.x;
    const int ty = tile / a.gx, tx = tile - ty * a.gx;
    const int ox = tx * kTile, oy = ty * kTile;
    const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x / kTile;
    const int px = ox + lx, py = oy + ly;
    const bool inside = px < a.width && py < a.height;
    const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int start = a.offsets[tile], end = a.offsets[tile + 1];

    if (threadIdx.x == 0) sMaxLast = 0;
#pragma unroll
    for (int v = 0; v < 9; ++v) sAcc[v][threadIdx.x] = 0.f;

    float G[3] = {0.f, 0.f, 0.f};
    float med[9];
#pragma unroll
    for (int v = 0; v < 9; ++v) med[v] = 0.f;
    float T = 1.f;
    int mylast = 0;
    if (inside) {
        const int pix = py * a.width + px;
        T = a.final_T[pix];
        mylast = a.last[pix];
        if (a.medium) {
            const float d = a.depth[pix];
            const float z = 2.0f / (1.0f + expf(-(float)kLogisticRate * d)) - 1.0f;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const float dl = a.dL[3 * pix + ch];
                const float att = expf(-a.medium[ch] * z);
                const float ebs = expf(-a.medium[6 + ch] * z);
                G[ch] = dl * att;
                med[ch] = dl * a.color_clean[3 * pix + ch] * (-z) * att;   // d attenuation
                med[3 + ch] = dl * (1.0f - ebs);                             // d water_color
                med[6 + ch] = dl * a.medium[3 + ch] * z * ebs;               // d backscatter
            }
        } else {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) G[ch] = a.dL[3 * pix + ch];
        }
    }
    if (a.medium) {
#pragma unroll
        for (int v = 0; v < 9; ++v) {
            float s = warp_sum(med[v]);
            if (lane == 0) sMed[warp][v] = s;
        }
    }
    __syncthreads();
    if (mylast > 0) atomicMax(&sMaxLast, mylast);
    if (a.medium && threadIdx.x < 9) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += sMed[w][threadIdx.x];
        atomicAdd(&a.medium_acc[threadIdx.x], (double)s);
    }
    __syncthreads();
    const int maxlast = sMaxLast;

    float S = 0.f;  // sum over later contributors of w_j (G . c_j)
    for (int bend = start + maxlast; bend > start; bend -= kRasterThreads) {
        const int bstart = max(start, bend - kRasterThreads);
        const int nb = bend - bstart;
        __syncthreads();
        if (threadIdx.x < nb) {
            const int row = a.entries[bstart + threadIdx.x];
            float dep;
            stage_entry(a.splat, row, ox, oy, sA[threadIdx.x], sB[threadIdx.x], sC[threadIdx.x], dep);
            sRow[threadIdx.x] = row;
        }
        __syncthreads();
        for (int k = nb - 1; k >= 0; --k) {
            const int jrel = bstart - start + k;
            float v[9];
            bool hit = false;
            if (jrel < mylast) {
                const StageA A = sA[k];
                const StageB B = sB[k];
                const float dx = fx - A.mx, dy = fy - A.my;
                const float power = -0.5f * (A.ca * dx * dx + B.cc * dy * dy) - A.cb * dx * dy;
                if (power >= B.skip) {
                    const float araw = B.op * __expf(power);
                    if (araw >= kFloorHi || floor_pass(araw, a.splat, a.exact, sRow[k], px, py)) {
                        hit = true;
                        const float alpha = fminf(araw, kClampF);
                        const float inv_om = __frcp_rn(1.0f - alpha);
                        const float Ti = T * inv_om;
                        const float w = alpha * Ti;
                        const StageC C = sC[k];
                        const float U = G[0] * B.r + G[1] * C.g + G[2] * C.b;
                        const float dalpha = U * Ti - S * inv_om;
                        S += w * U;
                        T = Ti;
                        const float dp = below_clamp(araw, a.splat, a.exact, sRow[k], px, py)
                                             ? dalpha * araw
                                             : 0.f;
                        v[0] = dp;
                        v[1] = dp * dx;
                        v[2] = dp * dy;
                        v[3] = v[1] * dx;
                        v[4] = v[1] * dy;
                        v[5] = v[2] * dy;
                        v[6] = w * G[0];
                        v[7] = w * G[1];
                        v[8] = w * G[2];
                    }
                }
            }
            if (!__any_sync(0xffffffffu, hit)) continue;
            if (!hit) {
#pragma unroll
                for (int i = 0; i < 9; ++i) v[i] = 0.f;
            }
            const float r8 = butterfly8(v, lane);
            const float r9 = warp_sum(v[8]);
            if ((lane & 3) == 0) {
                const int idx = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                atomicAdd(&sAcc[idx][k], r8);
            }
            if (lane == 0) atomicAdd(&sAcc[8][k], r9);
        }
        __syncthreads();
        if (threadIdx.x < nb) {
            const int k = threadIdx.x;
            float s[9];
            bool any = false;
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                s[i] = sAcc[i][k];
                sAcc[i][k] = 0.f;
                any |= s[i] != 0.f;
            }
            if (any) {
                const StageA A = sA[k];
                const StageB B = sB[k];
                float* g = a.screen + (size_t)sRow[k] * 9;
                atomicAdd(g + 0, s[0]);                          // d_logit (before (1-s))
                atomicAdd(g + 1, A.ca * s[1] + A.cb * s[2]);     // d_mean2d x
                atomicAdd(g + 2, A.cb * s[1] + B.cc * s[2]);     // d_mean2d y
                atomicAdd(g + 3, -0.5f * s[3]);                  // d_conic a
                atomicAdd(g + 4, -s[4]);                         // d_conic b
                atomicAdd(g + 5, -0.5f * s[5]);                  // d_conic c
                atomicAdd(g + 6, s[6]);                          // d_color
                atomicAdd(g + 7, s[7]);
                atomicAdd(g + 8, s[8]);
            }
        }
    }
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_raster_bwd(const uws_projected* proj, const int32_t* offsets,
                              const int32_t* entries, const uws_camera* cam, const float* medium,
                              const uws_raster_out* fwd, const float* dL_dC, float* screen_grads,
                              double* medium_acc, void* stream) {
    UWS_REQUIRE(proj && offsets && cam && fwd && dL_dC && screen_grads,
                "uws_raster_bwd: null argument");
    UWS_REQUIRE(fwd->final_T && fwd->last, "uws_raster_bwd: forward context missing");
    UWS_REQUIRE(medium == nullptr || (fwd->color_clean && fwd->depth && medium_acc),
                "uws_raster_bwd: underwater backward needs color_clean, depth and medium_acc");
    BwdArgs a;
    a.splat = proj->splat;
    a.exact = proj->exact;
    a.offsets = offsets;
    a.entries = entries;
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.medium = medium;
    a.color_clean = fwd->color_clean;
    a.depth = fwd->depth;
    a.final_T = fwd->final_T;
    a.last = fwd->last;
    a.dL = dL_dC;
    a.screen = screen_grads;
    a.medium_acc = medium_acc;
    k_raster_bwd<<<a.gx * gy, kRasterThreads, 0, as_stream(stream)>>>(a);
    UWS_CHECK_LAUNCH("k_raster_bwd");
    return UWS_OK;
}
