// K1 preprocess: per-Gaussian EWA projection, degree-0 colour, opacity-aware
// radius, tile rectangle and stream compaction of the visible set.
//
// Replaces projection.project_cloud (projection.py:100-199),
// footprint_radius (:89-97) and _spans_for (:229-249).
//
// Arithmetic is float64 and this translation unit is compiled with
// -fmad=false, so every expression maps 1:1 onto the IEEE operation numpy
// performs.  Where numpy's matmul (OpenBLAS / numpy SIMD loops) fuses, the
// code fuses explicitly with __fma_rn in the same order:
//     dot3(a, b) = fma(a2, b2, fma(a1, b1, a0 * b0)).
// Hence mean2d, depth and radius -- the inputs of every integer decision
// downstream (culling, tile rectangles, depth order) -- match the reference
// up to the last-ulp differences of exp/log between libm and CUDA.
//
// One thread per Gaussian; the visible rows are compacted in source order
// with a single-pass decoupled look-back scan.
#include "project_math.cuh"
#include "scan.cuh"

namespace uws {
namespace {

#ifndef UWS_PRE_IPT
#define UWS_PRE_IPT 2
#endif
#ifndef UWS_PRE_MINB
#define UWS_PRE_MINB 6
#endif
#ifndef UWS_PRE_THREADS
#define UWS_PRE_THREADS 128
#endif
constexpr int kThreads = UWS_PRE_THREADS;
constexpr int kIpt = UWS_PRE_IPT;
constexpr int kMinBlocks = UWS_PRE_MINB;

struct Proj {
    double mx, my, depth, a, b, c, radius, k0, k1, k2, s;
    float r, g, bl;
    int16_t x0, y0, x1, y1;
};

__device__ __forceinline__ bool project_one(const uws_cloud& cl, const uws_camera& cam,
                                            const FrustumLim& lim, int64_t i, int gx, int gy,
                                            Proj& o) {
    Geo G;
    geo_view(cl, cam, i, G);                                                  // :112
    const double vz = G.vz;
    if (!(vz > cam.near_plane) || !(vz < cam.far_plane)) return false;      // :114
    double logit = cl.opacity_logits[i];
    double s = 1.0 / (1.0 + exp(-logit));                                      // expit, :116
    if (!(s >= kFloor)) return false;                                          // :117
    geo_shape(cl, cam, i, lim, G);                                              // :126-153
    const double* T = G.T;
    const double* S = G.S;
    const double u = G.u, v = G.v;
    // cov2d = (T S) T^T (:154)
    double A[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            A[3 * r + c] = dot3f(T[3 * r], T[3 * r + 1], T[3 * r + 2], S[c], S[3 + c], S[6 + c]);
    double C00 = dot3f(A[0], A[1], A[2], T[0], T[1], T[2]);
    double C01 = dot3f(A[0], A[1], A[2], T[3], T[4], T[5]);
    double C10 = dot3f(A[3], A[4], A[5], T[0], T[1], T[2]);
    double C11 = dot3f(A[3], A[4], A[5], T[3], T[4], T[5]);
    double a = C00 + kDilation;
    double b = 0.5 * (C01 + C10);
    double c = C11 + kDilation;

    double mx = cam.fx * u + cam.cx;                                            // :160
    double my = cam.fy * v + cam.cy;
    // footprint_radius (:89-97)
    double mid = 0.5 * (a + c);
    double det = a * c - b * b;
    double lam = mid + sqrt(fmax(mid * mid - det, 0.0));
    double reach = 2.0 * log(fmax(255.0 * s, 1.0));
    double rad = sqrt(fmax(reach, kMinSigma2) * lam);
    // on-image cull (:164-169)
    if (!(mx + rad >= -0.5) || !(mx - rad <= cam.width + 0.5) || !(my + rad >= -0.5) ||
        !(my - rad <= cam.height + 0.5))
        return false;

    o.mx = mx; o.my = my; o.depth = vz;
    o.a = a; o.b = b; o.c = c; o.radius = rad; o.s = s;
    const double rdet = __drcp_rn(det);                                       // :174-175
    o.k0 = div_rcp(c, det, rdet); o.k1 = div_rcp(-b, det, rdet); o.k2 = div_rcp(a, det, rdet);
    // colour: max(f * C0 + 0.5, 0) (scene.py:136-139)
    o.r = (float)fmax((double)cl.sh_coeffs[3 * i + 0] * kSH_C0 + 0.5, 0.0);
    o.g = (float)fmax((double)cl.sh_coeffs[3 * i + 1] * kSH_C0 + 0.5, 0.0);
    o.bl = (float)fmax((double)cl.sh_coeffs[3 * i + 2] * kSH_C0 + 0.5, 0.0);
    // tile rectangle (_spans_for, :229-249)
    double ix0 = ceil(((mx - rad) - 0.5) - 1e-9);
    double ix1 = floor(((mx + rad) - 0.5) + 1e-9);
    double iy0 = ceil(((my - rad) - 0.5) - 1e-9);
    double iy1 = floor(((my + rad) - 0.5) + 1e-9);
    double tx0 = floor(ix0 / kTile), tx1 = floor(ix1 / kTile);
    double ty0 = floor(iy0 / kTile), ty1 = floor(iy1 / kTile);
    tx0 = fmin(fmax(tx0, 0.0), (double)(gx - 1));
    ty0 = fmin(fmax(ty0, 0.0), (double)(gy - 1));
    tx1 = fmin(fmax(tx1, -1.0), (double)(gx - 1));
    ty1 = fmin(fmax(ty1, -1.0), (double)(gy - 1));
    tx1 = fmax(tx1, tx0 - 1.0);
    ty1 = fmax(ty1, ty0 - 1.0);
    o.x0 = (int16_t)tx0; o.y0 = (int16_t)ty0; o.x1 = (int16_t)tx1; o.y1 = (int16_t)ty1;
    return true;
}

// writes one visible row
__device__ __forceinline__ void emit_row(uws_projected& out, unsigned long long row, int64_t i,
                                         const Proj& p) {
    out.source_index[row] = (int32_t)i;
    uws_splat sp;
    sp.mx = p.mx; sp.my = p.my;
    sp.ca = (float)p.k0; sp.cb = (float)p.k1; sp.cc = (float)p.k2; sp.opacity = (float)p.s;
    sp.r = p.r; sp.g = p.g; sp.b = p.bl; sp.depth = (float)p.depth;
    out.splat[row] = sp;
    double4 ex4 = make_double4(p.k0, p.k1, p.k2, p.s);
    reinterpret_cast<double4*>(out.exact)[row] = ex4;
    out.depth[row] = p.depth;
    short4 rc = make_short4(p.x0, p.y0, p.x1, p.y1);
    reinterpret_cast<short4*>(out.rect)[row] = rc;
    if (out.cov2d) {
        out.cov2d[3 * row + 0] = p.a;
        out.cov2d[3 * row + 1] = p.b;
        out.cov2d[3 * row + 2] = p.c;
    }
    if (out.radius) out.radius[row] = p.radius;
}

// kIpt consecutive Gaussians per thread (independent float64 chains the
// scheduler can interleave); a block covers kThreads * kIpt Gaussians.
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_preprocess(uws_cloud cl, uws_camera cam,
                                                                     FrustumLim lim,
                                                                     uws_projected out, int gx,
                                                                     int gy,
                                                                     unsigned long long* status,
                                                                     unsigned* ticket) {
    // launched serially (no pdl_entry): the per-CTA L1 invalidation costs more here
    __shared__ int s_tile;
    __shared__ unsigned long long s_scan[kThreads / 32 + 1];
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int tile = s_tile;
    const int64_t i0 = ((int64_t)tile * kThreads + threadIdx.x) * kIpt;
    Proj p[kIpt];
    bool vis[kIpt];
    unsigned cnt = 0;
#pragma unroll
    for (int q = 0; q < kIpt; ++q) {
        vis[q] = i0 + q < cl.n && project_one(cl, cam, lim, i0 + q, gx, gy, p[q]);
        cnt += vis[q];
    }
    unsigned long long total;
    unsigned long long ex = block_exclusive_sum<kThreads, unsigned long long>(cnt, s_scan, &total);
    if (threadIdx.x < 32) {
        const unsigned long long b = lookback_exclusive(status, tile, total);
        if (threadIdx.x == 0) s_base = b;
    }
    __syncthreads();
    unsigned long long row = s_base + ex;
    uint32_t dlo = 0xffffffffu, dhi = 0u;  // high words of the visible depths (binning's range)
#pragma unroll
    for (int q = 0; q < kIpt; ++q)
        if (vis[q]) {
            emit_row(out, row++, i0 + q, p[q]);
            const uint32_t h = (uint32_t)(__double_as_longlong(p[q].depth) >> 32);
            dlo = min(dlo, h);
            dhi = max(dhi, h);
        }
    if (out.depth_range) {
        dlo = __reduce_min_sync(0xffffffffu, dlo);
        dhi = __reduce_max_sync(0xffffffffu, dhi);
        if ((threadIdx.x & 31) == 0) {
            s_scan[threadIdx.x >> 5] = ((unsigned long long)dhi << 32) | (~dlo);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t nlo = 0u, hi = 0u;
#pragma unroll
            for (int w = 0; w < kThreads / 32; ++w) {
                nlo = max(nlo, (uint32_t)s_scan[w]);
                hi = max(hi, (uint32_t)(s_scan[w] >> 32));
            }
            if (nlo != 0u) {   // some visible row in the block
                atomicMax(&out.depth_range[0], nlo);
                atomicMax(&out.depth_range[1], hi);
            }
        }
    }
    if (tile == (int)gridDim.x - 1 && threadIdx.x == kThreads - 1)
        *out.num_visible = (int32_t)(s_base + total);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_preprocess_workspace_size(int64_t n, size_t* bytes) {
    UWS_REQUIRE(bytes != nullptr && n >= 0, "uws_preprocess_workspace_size: bad argument");
    int64_t blocks = ceil_div(n > 0 ? n : 1, kThreads * kIpt);
    Workspace ws(nullptr, 0, true);
    ws.take<unsigned long long>(blocks);
    ws.take<unsigned>(1);
    *bytes = ws.used;
    return UWS_OK;
}

extern "C" int uws_preprocess_fwd(const uws_cloud* cloud, const uws_camera* cam, uws_projected* out,
                                  void* workspace, size_t workspace_bytes, void* stream) {
    UWS_REQUIRE(cloud && cam && out, "uws_preprocess_fwd: null argument");
    UWS_REQUIRE(cloud->n >= 0 && cloud->n < (1ll << 31), "uws_preprocess_fwd: n out of range");
    UWS_REQUIRE(cam->width > 0 && cam->height > 0, "uws_preprocess_fwd: empty image");
    UWS_REQUIRE(out->num_visible != nullptr, "uws_preprocess_fwd: num_visible is required");
    cudaStream_t st = as_stream(stream);
    if (cloud->n == 0) {
        UWS_CUDA(zero_async(out->num_visible, sizeof(int32_t), st));
        return UWS_OK;
    }
    int gx = (int)ceil_div(cam->width, kTile), gy = (int)ceil_div(cam->height, kTile);
    UWS_REQUIRE(gx < 32768 && gy < 32768, "uws_preprocess_fwd: image too large for int16 tile ids");
    int64_t blocks = ceil_div(cloud->n, kThreads * kIpt);
    Workspace ws(workspace, workspace_bytes);
    auto* status = ws.take<unsigned long long>(blocks);
    auto* ticket = ws.take<unsigned>(1);
    UWS_REQUIRE(ws.ok(), "uws_preprocess_fwd: workspace too small");
    UWS_CUDA(zero_async2(status, (char*)(ticket + 1) - (char*)status, out->depth_range,
                         out->depth_range ? 2 * sizeof(uint32_t) : 0, st));
    launch_serial(k_preprocess, dim3((unsigned)blocks), dim3(kThreads), 0, st, *cloud, *cam, frustum_lim(*cam), *out, gx, gy, status, ticket);
    UWS_CHECK_LAUNCH("k_preprocess");
    return UWS_OK;
}
