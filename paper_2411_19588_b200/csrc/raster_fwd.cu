// K6 forward compositing with the underwater medium epilogue.
//
// Replaces the tile loop of rasterizer.render (rasterizer.py:188-241), the
// per-tile blend _composite_block (:148-178) and apply_water (:244-251) with
// logistic_remap (medium.py:26-29).
//
// One CTA per 16x16 tile, one thread per pixel.  The tile's depth-sorted list
// is streamed through shared memory in batches of 256 records (each thread
// stages one record with three 16-byte loads); every thread then walks the
// batch front to back.  A pixel stops once its transmittance drops below
// 1e-4 -- the contributor that crosses the threshold is still blended, as in
// the reference -- and the CTA leaves as soon as all 256 pixels are done.
// The per-pixel consumed-prefix length is written out so the backward kernel
// visits exactly the same pairs.
#include "raster_common.cuh"

namespace uws {
namespace {

struct FwdArgs {
    const uws_splat* splat;
    const double* exact;
    const int32_t* offsets;
    const int32_t* entries;
    int width, height, gx;
    float far_plane;
    const float* medium;  // NULL = clean
    uws_raster_out out;
};

__global__ void __launch_bounds__(kRasterThreads, 3) k_raster_fwd(FwdArgs a) {
    __shared__ StageA sA[kRasterThreads];
    __shared__ StageB sB[kRasterThreads];
    __shared__ StageC sC[kRasterThreads];
    __shared__ float sD[kRasterThreads];
    __shared__ int sRow[kRasterThreads];

    const int tile = blockIdx.x;
    const int ty = tile / a.gx, tx = tile - ty * a.gx;
    const int ox = tx * kTile, oy = ty * kTile;
    const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x / kTile;
    const int px = ox + lx, py = oy + ly;
    const bool inside = px < a.width && py < a.height;
    const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;

    const int start = a.offsets[tile], end = a.offsets[tile + 1];
    float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f, dsum = 0.f, wsum = 0.f;
    int count = 0, last = 0;
    bool done = !inside;

    for (int base = start; base < end; base += kRasterThreads) {
        if (__syncthreads_count(done) == kRasterThreads) break;
        const int j = base + threadIdx.x;
        if (j < end) {
            const int row = a.entries[j];
            stage_entry(a.splat, row, ox, oy, sA[threadIdx.x], sB[threadIdx.x], sC[threadIdx.x],
                        sD[threadIdx.x]);
            sRow[threadIdx.x] = row;
        }
        __syncthreads();
        const int n = min(kRasterThreads, end - base);
        if (!done) {
            for (int k = 0; k < n; ++k) {
                const StageA A = sA[k];
                const float dx = fx - A.mx, dy = fy - A.my;
                const StageB B = sB[k];
                const float power = -0.5f * (A.ca * dx * dx + B.cc * dy * dy) - A.cb * dx * dy;
                if (power < B.skip) continue;
                const float araw = B.op * __expf(power);
                if (araw < kFloorHi && !floor_pass(araw, a.splat, a.exact, sRow[k], px, py)) continue;
                const float alpha = fminf(araw, kClampF);
                const float w = alpha * T;
                const StageC C = sC[k];
                cr += w * B.r;
                cg += w * C.g;
                cb += w * C.b;
                dsum += w * sD[k];
                wsum += w;
                T = T * (1.0f - alpha);
                ++count;
                last = base - start + k + 1;
                if (!(T >= kTStopF)) {
                    done = true;
                    break;
                }
            }
        }
    }
    if (!inside) return;
    const int pix = py * a.width + px;
    const float depth = count > 0 ? dsum / wsum : a.far_plane;
    a.out.depth[pix] = depth;
    a.out.weight[pix] = wsum;
    a.out.final_T[pix] = T;
    a.out.count[pix] = count;
    if (a.out.last) a.out.last[pix] = last;
    if (a.medium == nullptr) {
        a.out.color[3 * pix + 0] = cr;
        a.out.color[3 * pix + 1] = cg;
        a.out.color[3 * pix + 2] = cb;
        if (a.out.color_clean) {
            a.out.color_clean[3 * pix + 0] = cr;
            a.out.color_clean[3 * pix + 1] = cg;
            a.out.color_clean[3 * pix + 2] = cb;
        }
        return;
    }
    // underwater epilogue: z = logistic(depth); C*exp(-Bd z) + Binf (1 - exp(-Bb z))
    const float z = 2.0f / (1.0f + expf(-(float)kLogisticRate * depth)) - 1.0f;
    const float c3[3] = {cr, cg, cb};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float att = expf(-a.medium[ch] * z);
        const float bs = a.medium[3 + ch] * (1.0f - expf(-a.medium[6 + ch] * z));
        a.out.color[3 * pix + ch] = c3[ch] * att + bs;
        if (a.out.color_clean) a.out.color_clean[3 * pix + ch] = c3[ch];
        if (a.out.attenuation) a.out.attenuation[3 * pix + ch] = att;
        if (a.out.backscatter) a.out.backscatter[3 * pix + ch] = bs;
    }
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
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.far_plane = (float)cam->far_plane;
    a.medium = medium;
    a.out = *out;
    k_raster_fwd<<<a.gx * gy, kRasterThreads, 0, as_stream(stream)>>>(a);
    UWS_CHECK_LAUNCH("k_raster_fwd");
    return UWS_OK;
}
