// K7 training objective: L1 + D-SSIM with its analytic image gradient.
//
// Replaces losses.total_loss (losses.py:140-160) with l1_loss (:40-49),
// d_ssim_loss (:83-123; 11x11 Gaussian sigma 1.5, valid windows only,
// C1 = 0.01^2, C2 = 0.03^2, adjoint of the valid filter :68-74) and
// guidance_loss (:126-137).
//
// Two tiled passes, each staging a (16+10) x (32+10) halo patch in shared
// memory and filtering separably: (1) window moments -> SSIM map partial sums
// and the three per-window derivative maps; (2) the adjoint filter of those
// maps fused with the L1 subgradient -> dL/dC.  Partial sums are reduced in
// a fixed order (deterministic) by a one-block finalize kernel.
#include "common.cuh"

namespace uws {
namespace {

constexpr int kOW = 32, kOH = 16, kR = 5, kN = 11;
constexpr int kPW = kOW + 2 * kR, kPH = kOH + 2 * kR;
constexpr int kThreads = 256;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ float c_taps[kN];

__device__ __forceinline__ float block_sum_f(float v, float* sred) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    float s = 0.f;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) s += sred[w];
    return s;
}

__global__ void __launch_bounds__(kThreads) k_ssim_moments(const float* __restrict__ img_a,
                                                           const float* __restrict__ img_b, int H,
                                                           int W, int C, float* __restrict__ t_mu,
                                                           float* __restrict__ t_aa,
                                                           float* __restrict__ t_ab,
                                                           double* __restrict__ part_s) {
    __shared__ float sa[kPH][kPW + 1], sb[kPH][kPW + 1];
    __shared__ float hs[5][kPH][kOW + 1];
    __shared__ float sred[kThreads / 32];
    const int ch = blockIdx.z;
    const int x0 = blockIdx.x * kOW, y0 = blockIdx.y * kOH;  // valid-window origin == image pixel
    const int VW = W - 2 * kR, VH = H - 2 * kR;
    for (int i = threadIdx.x; i < kPH * kPW; i += kThreads) {
        int r = i / kPW, c = i - r * kPW;
        int gy = y0 + r, gx = x0 + c;
        bool ok = gy < H && gx < W;
        size_t o = ((size_t)gy * W + gx) * C + ch;
        sa[r][c] = ok ? img_a[o] : 0.f;
        sb[r][c] = ok ? img_b[o] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kPH * kOW; i += kThreads) {
        int r = i / kOW, c = i - r * kOW;
        float m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
        for (int t = 0; t < kN; ++t) {
            float w = c_taps[t], xa = sa[r][c + t], xb = sb[r][c + t];
            m0 += w * xa;
            m1 += w * xb;
            m2 += w * xa * xa;
            m3 += w * xb * xb;
            m4 += w * xa * xb;
        }
        hs[0][r][c] = m0; hs[1][r][c] = m1; hs[2][r][c] = m2; hs[3][r][c] = m3; hs[4][r][c] = m4;
    }
    __syncthreads();
    float ssum = 0.f;
    for (int i = threadIdx.x; i < kOH * kOW; i += kThreads) {
        int r = i / kOW, c = i - r * kOW;
        int oy = y0 + r, ox = x0 + c;
        if (oy >= VH || ox >= VW) continue;
        float u1 = 0, u2 = 0, v1 = 0, v2 = 0, v12 = 0;
#pragma unroll
        for (int t = 0; t < kN; ++t) {
            float w = c_taps[t];
            u1 += w * hs[0][r + t][c];
            u2 += w * hs[1][r + t][c];
            v1 += w * hs[2][r + t][c];
            v2 += w * hs[3][r + t][c];
            v12 += w * hs[4][r + t][c];
        }
        const float A1 = 2.0f * u1 * u2 + (float)kC1;
        const float A2 = 2.0f * (v12 - u1 * u2) + (float)kC2;
        const float B1 = u1 * u1 + u2 * u2 + (float)kC1;
        const float B2 = (v1 - u1 * u1) + (v2 - u2 * u2) + (float)kC2;
        const float inv = 1.0f / (B1 * B2);
        const float S = A1 * A2 * inv;
        ssum += S;
        size_t o = ((size_t)oy * VW + ox) * C + ch;
        t_mu[o] = 2.0f * u2 * (A2 - A1) * inv - 2.0f * u1 * S * (1.0f / B1 - 1.0f / B2);
        t_aa[o] = -S / B2;
        t_ab[o] = 2.0f * A1 * inv;
    }
    float bs = block_sum_f(ssum, sred);
    if (threadIdx.x == 0)
        part_s[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = (double)bs;
}

__global__ void __launch_bounds__(kThreads) k_ssim_grad(const float* __restrict__ img_a,
                                                        const float* __restrict__ img_b, int H, int W,
                                                        int C, const float* __restrict__ t_mu,
                                                        const float* __restrict__ t_aa,
                                                        const float* __restrict__ t_ab,
                                                        float k_ssim, float k_l1,
                                                        float* __restrict__ grad,
                                                        double* __restrict__ part_l1) {
    __shared__ float sm[3][kPH][kPW + 1];
    __shared__ float hs[3][kPH][kOW + 1];
    __shared__ float sred[kThreads / 32];
    const int ch = blockIdx.z;
    const int x0 = blockIdx.x * kOW, y0 = blockIdx.y * kOH;
    const int VW = W - 2 * kR, VH = H - 2 * kR;
    // adj[y][x] = sum_{u,v} w_u w_v M[y+u-2R][x+v-2R], M zero outside the valid grid
    for (int i = threadIdx.x; i < kPH * kPW; i += kThreads) {
        int r = i / kPW, c = i - r * kPW;
        int my = y0 + r - 2 * kR, mx = x0 + c - 2 * kR;
        bool ok = my >= 0 && my < VH && mx >= 0 && mx < VW;
        size_t o = ((size_t)my * VW + mx) * C + ch;
        sm[0][r][c] = ok ? t_mu[o] : 0.f;
        sm[1][r][c] = ok ? t_aa[o] : 0.f;
        sm[2][r][c] = ok ? t_ab[o] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kPH * kOW; i += kThreads) {
        int r = i / kOW, c = i - r * kOW;
        float m0 = 0, m1 = 0, m2 = 0;
#pragma unroll
        for (int t = 0; t < kN; ++t) {
            float w = c_taps[t];
            m0 += w * sm[0][r][c + t];
            m1 += w * sm[1][r][c + t];
            m2 += w * sm[2][r][c + t];
        }
        hs[0][r][c] = m0; hs[1][r][c] = m1; hs[2][r][c] = m2;
    }
    __syncthreads();
    float l1sum = 0.f;
    for (int i = threadIdx.x; i < kOH * kOW; i += kThreads) {
        int r = i / kOW, c = i - r * kOW;
        int y = y0 + r, x = x0 + c;
        if (y >= H || x >= W) continue;
        float g0 = 0, g1 = 0, g2 = 0;
#pragma unroll
        for (int t = 0; t < kN; ++t) {
            float w = c_taps[t];
            g0 += w * hs[0][r + t][c];
            g1 += w * hs[1][r + t][c];
            g2 += w * hs[2][r + t][c];
        }
        size_t o = ((size_t)y * W + x) * C + ch;
        float a = img_a[o], b = img_b[o];
        float d = a - b;
        float sg = (d > 0.f) ? 1.f : ((d < 0.f) ? -1.f : 0.f);
        l1sum += fabsf(d);
        grad[o] = k_ssim * (g0 + 2.0f * a * g1 + b * g2) + k_l1 * sg;
    }
    float bs = block_sum_f(l1sum, sred);
    if (threadIdx.x == 0)
        part_l1[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = (double)bs;
}

__global__ void __launch_bounds__(kThreads) k_loss_finalize(const double* __restrict__ part_s,
                                                            int n_s, const double* __restrict__ part_l1,
                                                            int n_l1, double n_px, double n_win,
                                                            const float* medium, int has_guidance,
                                                            double lam_s, double lam_g,
                                                            double* result, float* nonfinite) {
    __shared__ double rs[kThreads], rl[kThreads];
    double s = 0, l = 0;
    for (int i = threadIdx.x; i < n_s; i += kThreads) s += part_s[i];
    for (int i = threadIdx.x; i < n_l1; i += kThreads) l += part_l1[i];
    rs[threadIdx.x] = s;
    rl[threadIdx.x] = l;
    __syncthreads();
    for (int o = kThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            rs[threadIdx.x] += rs[threadIdx.x + o];
            rl[threadIdx.x] += rl[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double l1 = rl[0] / n_px;
        double ds = 1.0 - rs[0] / n_win;
        double lb = 0.0;
        if (medium && has_guidance) {
            for (int c = 0; c < 3; ++c) {
                lb += fabs((double)medium[3 + c] - (double)medium[9 + c]);
                lb += fabs((double)medium[6 + c] - (double)medium[12 + c]);
            }
        }
        double total = (1.0 - lam_s) * l1 + lam_s * ds + lam_g * lb;
        result[0] = l1;
        result[1] = ds;
        result[2] = lb;
        result[3] = total;
        result[4] = isfinite(total) ? 1.0 : 0.0;
        result[5] = 0.0;
        if (!isfinite(total) && nonfinite) atomicAdd(nonfinite, 1.0f);
    }
}

bool g_taps_ready = false;

int ensure_taps() {
    if (g_taps_ready) return UWS_OK;
    double k[kN], s = 0;
    for (int i = 0; i < kN; ++i) {
        double x = i - (kN - 1) / 2.0;
        k[i] = exp(-0.5 * (x / 1.5) * (x / 1.5));
        s += k[i];
    }
    float f[kN];
    for (int i = 0; i < kN; ++i) f[i] = (float)(k[i] / s);
    UWS_CUDA(cudaMemcpyToSymbol(c_taps, f, sizeof(f)));
    g_taps_ready = true;
    return UWS_OK;
}

struct LossPlan {
    float *t_mu, *t_aa, *t_ab;
    double *part_s, *part_l1;
    int n_s, n_l1;
};

void plan_loss(Workspace& ws, int h, int w, int c, LossPlan& p) {
    int vh = h - 2 * kR > 0 ? h - 2 * kR : 1, vw = w - 2 * kR > 0 ? w - 2 * kR : 1;
    size_t nv = (size_t)vh * vw * c;
    p.t_mu = ws.take<float>(nv);
    p.t_aa = ws.take<float>(nv);
    p.t_ab = ws.take<float>(nv);
    p.n_s = (int)(ceil_div(vw, kOW) * ceil_div(vh, kOH) * c);
    p.n_l1 = (int)(ceil_div(w, kOW) * ceil_div(h, kOH) * c);
    p.part_s = ws.take<double>(p.n_s);
    p.part_l1 = ws.take<double>(p.n_l1);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_loss_workspace_size(int32_t h, int32_t w, int32_t c, size_t* bytes) {
    UWS_REQUIRE(bytes && h > 0 && w > 0 && c > 0, "uws_loss_workspace_size: bad argument");
    Workspace ws(nullptr, 0, true);
    LossPlan p;
    plan_loss(ws, h, w, c, p);
    *bytes = ws.used;
    return UWS_OK;
}

extern "C" int uws_loss_fwd_bwd(const float* rendered, const float* gt, int32_t h, int32_t w,
                                int32_t c, const float* medium, int32_t has_guidance,
                                double lambda_ssim, double lambda_guide, float* dL_dC,
                                double* result, float* nonfinite, void* workspace,
                                size_t workspace_bytes, void* stream) {
    UWS_REQUIRE(rendered && gt && dL_dC && result, "uws_loss_fwd_bwd: null argument");
    UWS_REQUIRE(h >= kN && w >= kN, "uws_loss_fwd_bwd: image smaller than the 11x11 window");
    UWS_REQUIRE(c >= 1, "uws_loss_fwd_bwd: bad channel count");
    int rc = ensure_taps();
    if (rc != UWS_OK) return rc;
    Workspace ws(workspace, workspace_bytes);
    LossPlan p;
    plan_loss(ws, h, w, c, p);
    UWS_REQUIRE(ws.ok(), "uws_loss_fwd_bwd: workspace too small");
    cudaStream_t st = as_stream(stream);
    const int vh = h - 2 * kR, vw = w - 2 * kR;
    const double n_px = (double)h * w * c, n_win = (double)vh * vw * c;
    dim3 g1((unsigned)ceil_div(vw, kOW), (unsigned)ceil_div(vh, kOH), (unsigned)c);
    k_ssim_moments<<<g1, kThreads, 0, st>>>(rendered, gt, h, w, c, p.t_mu, p.t_aa, p.t_ab, p.part_s);
    UWS_CHECK_LAUNCH("k_ssim_moments");
    dim3 g2((unsigned)ceil_div(w, kOW), (unsigned)ceil_div(h, kOH), (unsigned)c);
    const float k_ssim = (float)(lambda_ssim * (-1.0 / n_win));
    const float k_l1 = (float)((1.0 - lambda_ssim) / n_px);
    k_ssim_grad<<<g2, kThreads, 0, st>>>(rendered, gt, h, w, c, p.t_mu, p.t_aa, p.t_ab, k_ssim, k_l1,
                                         dL_dC, p.part_l1);
    UWS_CHECK_LAUNCH("k_ssim_grad");
    k_loss_finalize<<<1, kThreads, 0, st>>>(p.part_s, p.n_s, p.part_l1, p.n_l1, n_px, n_win, medium,
                                            has_guidance, lambda_ssim, lambda_guide, result,
                                            nonfinite);
    UWS_CHECK_LAUNCH("k_loss_finalize");
    return UWS_OK;
}
