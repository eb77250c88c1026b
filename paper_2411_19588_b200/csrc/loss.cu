// K7 training objective: L1 + D-SSIM with its analytic image gradient.
//
// Replaces losses.total_loss (losses.py:140-160) with l1_loss (:40-49),
// d_ssim_loss (:83-123; 11x11 Gaussian sigma 1.5, valid windows only,
// C1 = 0.01^2, C2 = 0.03^2, adjoint of the valid filter :68-74) and
// guidance_loss (:126-137).
//
// Two tiled passes over 32x32 tiles with a 10-pixel halo staged in shared
// memory, each filtering separably with register-blocked sliding sums (8
// outputs per horizontal item, 4 per vertical item, taps in the constant
// bank): (1) window moments -> SSIM map partial sums and the three
// per-window derivative maps (planar, one plane per map and channel); (2) the
// adjoint filter of those maps fused with the L1 subgradient -> dL/dC.  Partial
// sums are reduced in a fixed order (deterministic) by a one-block finalize
// kernel.
#include "common.cuh"

namespace uws {
namespace {

constexpr int kR = 5, kN = 11;
constexpr int kT = 32;               // output tile edge
constexpr int kP = kT + 2 * kR;      // staged patch edge (42)
constexpr int kHR = 8;               // horizontal outputs per item
constexpr int kVR = 4;               // vertical outputs per item
constexpr int kThreads = 256;
constexpr int kMaxC = 4;             // channels staged at once by the moments pass
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ float c_taps[kN];
__constant__ float2 c_taps2[kN];  // (w, w): the tap for both lanes of an FFMA2

// c + a * b on two float lanes with one FFMA2 (sm_100): per lane the same
// IEEE fma as fmaf, so results are bitwise those of two FFMAs
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)),
          "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<unsigned long long*>(&a)),
          "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 4-byte asynchronous global -> shared copy; ok = false writes a zero
__device__ __forceinline__ void cp_async4(float* sdst, const float* gsrc, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gsrc),
                 "r"(ok ? 4 : 0)
                 : "memory");
}
// 16-byte asynchronous global -> shared copy; ok = false writes zeros
__device__ __forceinline__ void cp_async16(float* sdst, const float* gsrc, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc),
                 "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Derivative-map planes are stored with kMapPad zero columns on the left (window x at
// column x + kMapPad) and zero columns up to the row pitch on the right, so the grad
// pass stages each block's 42-column window as 11 aligned 16-byte chunks per row
// (x0 - 2R + kMapPad = x0: 16-byte aligned since x0 is a multiple of 32).
constexpr int kMapPad = 2 * kR;
constexpr int kMP = 44;              // staged window row: 42 columns rounded up to 16 bytes
constexpr size_t kGradSmem = (size_t)(2 * 3 * kP * kMP + 3 * kP * (kT + 1)) * sizeof(float);

__host__ __device__ constexpr int map_pitch(int w) {  // floats per map row
    return kT * ((w + kT - 1) / kT) + 12;
}

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

// Pass 1.  Block = 32x32 valid windows (all channels); dynamic smem holds the
// interleaved (a, b) patch [2][kP][kP*C + 1] and the horizontal moments
// [4][kP][kT + 1] of the channel in flight.
template <int CT>  // compile-time channel count (0: runtime C)
__global__ void __launch_bounds__(kThreads, 3) k_ssim_moments(const float* __restrict__ img_a,
                                                              const float* __restrict__ img_b,
                                                              int H, int W, int C_,
                                                              float* __restrict__ maps,
                                                              double* __restrict__ part_s) {
    // launched serially (no pdl_entry): the per-CTA L1 invalidation costs more here
    const int C = CT > 0 ? CT : C_;
    extern __shared__ float smem[];
    const int pitch = kP * C + 1;
    float* sa = smem;
    float* sb = sa + kP * pitch;
    float* hs = sb + kP * pitch;  // [4][kP][kT + 1]
    __shared__ float sred[kThreads / 32];
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;  // valid-window origin == image pixel
    const int VW = W - 2 * kR, VH = H - 2 * kR;
    const int MPW = map_pitch(W);
    const size_t plane = (size_t)VH * MPW;
    // zero pad columns of this block's map rows: the left pad [0, kMapPad) in the first
    // column of blocks, everything right of the valid windows [VW + kMapPad, MPW) in the last
    {
        const int left = blockIdx.x == 0 ? kMapPad : 0;
        const int rfirst = VW + kMapPad;
        const int right = blockIdx.x == gridDim.x - 1 ? MPW - rfirst : 0;
        const int per_row = left + right;
        for (int i = threadIdx.x; i < kT * 3 * C * per_row; i += kThreads) {
            const int k = i % per_row, rest = i / per_row;
            const int r = rest % kT, m = rest / kT;
            const int col = k < left ? k : rfirst + (k - left);
            const int oy = y0 + r;
            if (oy < VH) maps[(size_t)m * plane + (size_t)oy * MPW + col] = 0.f;
        }
    }
    // stage rows of kP*C contiguous floats (coalesced): one warp per row, every
    // copy asynchronous so all of the patch's loads are in flight at once
    {
        const int rowlen = kP * C;
        const int lane = threadIdx.x & 31;
        const int qmax = min(rowlen, (W - x0) * C);  // columns inside the image
        for (int r = threadIdx.x >> 5; r < kP; r += kThreads / 32) {
            const int gy = y0 + r;
            const float* ra = img_a + ((size_t)min(gy, H - 1) * W + x0) * C;
            const float* rb = img_b + ((size_t)min(gy, H - 1) * W + x0) * C;
            const bool rok = gy < H;
            for (int q = lane; q < rowlen; q += 32) {
                const bool ok = rok && q < qmax;
                cp_async4(&sa[r * pitch + q], ok ? ra + q : img_a, ok);
                cp_async4(&sb[r * pitch + q], ok ? rb + q : img_b, ok);
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
    }
    __syncthreads();
    float ssum = 0.f;
    for (int ch = 0; ch < C; ++ch) {
        // horizontal: item = (row, group of 8 columns)
        for (int it = threadIdx.x; it < kP * (kT / kHR); it += kThreads) {
            const int r = it >> 2, c0 = (it & 3) * kHR;
            // (mu_a, mu_b) and (E[a^2] + E[b^2], E[ab]) accumulate in FFMA2 pairs: SSIM
            // uses sigma_a^2 and sigma_b^2 only through their sum (B2) and its
            // derivative coefficient is shared, so four moments suffice
            float2 m01[kHR], m23[kHR];
#pragma unroll
            for (int j = 0; j < kHR; ++j) m01[j] = m23[j] = make_float2(0.f, 0.f);
            const float* pa = sa + r * pitch + c0 * C + ch;
            const float* pb = sb + r * pitch + c0 * C + ch;
#pragma unroll
            for (int q = 0; q < kHR + kN - 1; ++q) {
                const float2 x01 = make_float2(pa[q * C], pb[q * C]);
                const float2 sq = mul2(x01, x01);
                const float2 x23 = make_float2(sq.x + sq.y, x01.x * x01.y);
#pragma unroll
                for (int j = 0; j < kHR; ++j) {
                    const int t = q - j;
                    if (t < 0 || t >= kN) continue;
                    const float2 w2 = c_taps2[t];
                    m01[j] = fma2(w2, x01, m01[j]);
                    m23[j] = fma2(w2, x23, m23[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < kHR; ++j) {
                hs[(0 * kP + r) * (kT + 1) + c0 + j] = m01[j].x;
                hs[(1 * kP + r) * (kT + 1) + c0 + j] = m01[j].y;
                hs[(2 * kP + r) * (kT + 1) + c0 + j] = m23[j].x;
                hs[(3 * kP + r) * (kT + 1) + c0 + j] = m23[j].y;
            }
        }
        __syncthreads();
        // vertical: item = (column, group of 4 rows)
        {
            const int c = threadIdx.x & (kT - 1), r0 = (threadIdx.x >> 5) * kVR;
            float2 u01[kVR], u23[kVR];
#pragma unroll
            for (int j = 0; j < kVR; ++j) u01[j] = u23[j] = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < kVR + kN - 1; ++q) {
                const float* hq = hs + (r0 + q) * (kT + 1) + c;
                const float2 h01 = make_float2(hq[0 * kP * (kT + 1)], hq[1 * kP * (kT + 1)]);
                const float2 h23 = make_float2(hq[2 * kP * (kT + 1)], hq[3 * kP * (kT + 1)]);
#pragma unroll
                for (int j = 0; j < kVR; ++j) {
                    const int t = q - j;
                    if (t < 0 || t >= kN) continue;
                    const float2 w2 = c_taps2[t];
                    u01[j] = fma2(w2, h01, u01[j]);
                    u23[j] = fma2(w2, h23, u23[j]);
                }
            }
            const int ox = x0 + c;
#pragma unroll
            for (int j = 0; j < kVR; ++j) {
                const int oy = y0 + r0 + j;
                if (oy >= VH || ox >= VW) continue;
                const float u1 = u01[j].x, u2 = u01[j].y, vs = u23[j].x, v12 = u23[j].y;
                const float A1 = 2.0f * u1 * u2 + (float)kC1;
                const float A2 = 2.0f * (v12 - u1 * u2) + (float)kC2;
                const float uu = u1 * u1 + u2 * u2;
                const float B1 = uu + (float)kC1;
                const float B2 = (vs - uu) + (float)kC2;
                // B1 >= C1 and B2 >= C2 (> 0): approximate reciprocals (rel. error ~2^-22)
                const float r1 = rcp_approx(B1), r2 = rcp_approx(B2);
                const float inv = r1 * r2;
                const float S = A1 * A2 * inv;
                ssum += S;
                const size_t o = (size_t)oy * MPW + ox + kMapPad;
                maps[(0 * C + ch) * plane + o] = 2.0f * u2 * (A2 - A1) * inv - 2.0f * u1 * S * (r1 - r2);
                maps[(1 * C + ch) * plane + o] = -S * r2;
                maps[(2 * C + ch) * plane + o] = 2.0f * A1 * inv;
            }
        }
        __syncthreads();  // hs reuse by the next channel
    }
    float bs = block_sum_f(ssum, sred);
    if (threadIdx.x == 0) part_s[blockIdx.y * gridDim.x + blockIdx.x] = (double)bs;
}

// Pass 2.  Block = 32x32 image pixels; per channel the three derivative maps
// are staged with a 2R halo (zero outside the valid grid) and filtered by the
// adjoint (= the same symmetric) window.
template <int CT>
__global__ void __launch_bounds__(kThreads, 3) k_ssim_grad(const float* __restrict__ img_a,
                                                           const float* __restrict__ img_b, int H,
                                                           int W, int C_,
                                                           const float* __restrict__ maps,
                                                           float k_ssim, float k_l1,
                                                           float* __restrict__ grad,
                                                           double* __restrict__ part_l1) {
    // launched serially (no pdl_entry): measured faster
    // double-buffered derivative-map windows [2][3][kP][kP+1] (cp.async: the next
    // channel's window streams in while this channel is filtered), then hs
    extern __shared__ float smem[];
    typedef float Win[3][kP][kMP];
    Win* sbuf = reinterpret_cast<Win*>(smem);
    float (*hs)[kP][kT + 1] = reinterpret_cast<float (*)[kP][kT + 1]>(smem + 2 * 3 * kP * kMP);
    __shared__ float sred[kThreads / 32];
    const int C = CT > 0 ? CT : C_;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    const int VH = H - 2 * kR;
    const int MPW = map_pitch(W);
    const size_t plane = (size_t)VH * MPW;
    // adj[y][x] = sum_{u,v} w_u w_v M[y+u-2R][x+v-2R], M zero outside the valid grid
    // (zero pad columns in the planes, zero fill for rows outside)
    // chunk i = threadIdx.x + 256 k of [3 maps][kP rows][kMP/4 chunks]: its (map, row, chunk)
    // advance by (0, 23, 3) per step (256 = 23 * 11 + 3), with carries -- no divisions
    constexpr int kCh = kMP / 4;
    static_assert(kThreads == 23 * kCh + 3, "chunk stepping");
    const int c4_0 = threadIdx.x % kCh, r_0 = (threadIdx.x / kCh) % kP;
    auto issue = [&](int ch) {  // 3 maps x 42 rows x 11 aligned 16-byte chunks
        Win& dst = sbuf[ch & 1];
        const float* mp = maps + (size_t)ch * plane + x0;
        int c4 = c4_0, r = r_0, m = 0;
#pragma unroll
        for (int k = 0; k < (3 * kP * kCh + kThreads - 1) / kThreads; ++k) {
            if (m < 3) {
                const int my = y0 + r - 2 * kR;
                const bool ok = my >= 0 && my < VH;
                const float* src = mp + (size_t)m * C * plane + (size_t)(ok ? my : 0) * MPW + 4 * c4;
                cp_async16(&dst[m][r][4 * c4], src, ok);
            }
            c4 += 3;
            r += 23;
            if (c4 >= kCh) {
                c4 -= kCh;
                ++r;
            }
            if (r >= kP) {
                r -= kP;
                ++m;
            }
        }
        cp_async_commit();
    };
    issue(0);
    float l1sum = 0.f;
    for (int ch = 0; ch < C; ++ch) {
        if (ch + 1 < C) {
            issue(ch + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        float (*sm)[kP][kMP] = sbuf[ch & 1];
        for (int it = threadIdx.x; it < kP * (kT / kHR); it += kThreads) {
            const int r = it >> 2, c0 = (it & 3) * kHR;
            float2 g01[kHR];
            float g2[kHR];
#pragma unroll
            for (int j = 0; j < kHR; ++j) {
                g01[j] = make_float2(0.f, 0.f);
                g2[j] = 0.f;
            }
#pragma unroll
            for (int q = 0; q < kHR + kN - 1; ++q) {
                const float2 x01 = make_float2(sm[0][r][c0 + q], sm[1][r][c0 + q]);
                const float x2 = sm[2][r][c0 + q];
#pragma unroll
                for (int j = 0; j < kHR; ++j) {
                    const int t = q - j;
                    if (t < 0 || t >= kN) continue;
                    g01[j] = fma2(c_taps2[t], x01, g01[j]);
                    g2[j] = fmaf(c_taps[t], x2, g2[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < kHR; ++j) {
                hs[0][r][c0 + j] = g01[j].x;
                hs[1][r][c0 + j] = g01[j].y;
                hs[2][r][c0 + j] = g2[j];
            }
        }
        __syncthreads();
        {
            const int c = threadIdx.x & (kT - 1), r0 = (threadIdx.x >> 5) * kVR;
            const int x = x0 + c;
            float pa[kVR], pb[kVR];
#pragma unroll
            for (int j = 0; j < kVR; ++j) {  // issue the image loads before the filter math
                const int y = y0 + r0 + j;
                const bool ok = y < H && x < W;
                const size_t o = ((size_t)y * W + x) * C + ch;
                pa[j] = ok ? __ldg(img_a + o) : 0.f;
                pb[j] = ok ? __ldg(img_b + o) : 0.f;
            }
            float2 g01[kVR];
            float g2[kVR];
#pragma unroll
            for (int j = 0; j < kVR; ++j) {
                g01[j] = make_float2(0.f, 0.f);
                g2[j] = 0.f;
            }
#pragma unroll
            for (int q = 0; q < kVR + kN - 1; ++q) {
                const float2 h01 = make_float2(hs[0][r0 + q][c], hs[1][r0 + q][c]);
                const float h2 = hs[2][r0 + q][c];
#pragma unroll
                for (int j = 0; j < kVR; ++j) {
                    const int t = q - j;
                    if (t < 0 || t >= kN) continue;
                    g01[j] = fma2(c_taps2[t], h01, g01[j]);
                    g2[j] = fmaf(c_taps[t], h2, g2[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < kVR; ++j) {
                const int y = y0 + r0 + j;
                if (y >= H || x >= W) continue;
                const size_t o = ((size_t)y * W + x) * C + ch;
                const float a = pa[j], b = pb[j];
                const float d = a - b;
                const float sg = (d > 0.f) ? 1.f : ((d < 0.f) ? -1.f : 0.f);
                l1sum += fabsf(d);
                grad[o] = k_ssim * (g01[j].x + 2.0f * a * g01[j].y + b * g2[j]) + k_l1 * sg;
            }
        }
        __syncthreads();  // sm / hs reuse by the next channel
    }
    float bs = block_sum_f(l1sum, sred);
    if (threadIdx.x == 0) part_l1[blockIdx.y * gridDim.x + blockIdx.x] = (double)bs;
}

constexpr int kFinThreads = 1024;

__global__ void __launch_bounds__(kFinThreads) k_loss_finalize(const double* __restrict__ part_s,
                                                            int n_s, const double* __restrict__ part_l1,
                                                            int n_l1, double n_px, double n_win,
                                                            const float* medium, int has_guidance,
                                                            double lam_s, double lam_g,
                                                            double* result, float* nonfinite) {
    pdl_entry();
    __shared__ double rs[kFinThreads / 32], rl[kFinThreads / 32];
    // fixed-order (deterministic) sums; each thread's loads are all issued before its adds
    double s = 0, l = 0;
    const int n = max(n_s, n_l1);
    for (int i0 = 0; i0 < n; i0 += 4 * kFinThreads) {
        double a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * kFinThreads + (int)threadIdx.x;
            a[q] = i < n_s ? part_s[i] : 0.0;
            b[q] = i < n_l1 ? part_l1[i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            s += a[q];
            l += b[q];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, o);
        l += __shfl_down_sync(0xffffffffu, l, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        rs[warp] = s;
        rl[warp] = l;
    }
    __syncthreads();
    if (warp == 0) {
        s = rs[lane];
        l = rl[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_down_sync(0xffffffffu, s, o);
            l += __shfl_down_sync(0xffffffffu, l, o);
        }
        if (lane == 0) {
            rs[0] = s;
            rl[0] = l;
        }
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
    float2 f2[kN];
    for (int i = 0; i < kN; ++i) f2[i] = make_float2(f[i], f[i]);
    UWS_CUDA(cudaMemcpyToSymbol(c_taps2, f2, sizeof(f2)));
    g_taps_ready = true;
    return UWS_OK;
}

struct LossPlan {
    float* maps;  // [3 maps][C][VH][map_pitch(W)] (zero-padded rows)
    double *part_s, *part_l1;
    int n_s, n_l1;
};

void plan_loss(Workspace& ws, int h, int w, int c, LossPlan& p) {
    int vh = h - 2 * kR > 0 ? h - 2 * kR : 1, vw = w - 2 * kR > 0 ? w - 2 * kR : 1;
    p.maps = ws.take<float>((size_t)vh * map_pitch(w) * c * 3);
    p.n_s = (int)(ceil_div(vw, kT) * ceil_div(vh, kT));
    p.n_l1 = (int)(ceil_div(w, kT) * ceil_div(h, kT));
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
    UWS_REQUIRE(c >= 1 && c <= kMaxC, "uws_loss_fwd_bwd: channel count must be 1..4");
    int rc = ensure_taps();
    if (rc != UWS_OK) return rc;
    Workspace ws(workspace, workspace_bytes);
    LossPlan p;
    plan_loss(ws, h, w, c, p);
    UWS_REQUIRE(ws.ok(), "uws_loss_fwd_bwd: workspace too small");
    cudaStream_t st = as_stream(stream);
    const int vh = h - 2 * kR, vw = w - 2 * kR;
    const double n_px = (double)h * w * c, n_win = (double)vh * vw * c;
    const size_t smem1 = (size_t)(2 * kP * (kP * c + 1) + 4 * kP * (kT + 1)) * sizeof(float);
    static bool attr_set = false;
    if (!attr_set) {
        const int mx = (int)(2 * kP * (kP * kMaxC + 1) + 4 * kP * (kT + 1)) * (int)sizeof(float);
        UWS_CUDA(cudaFuncSetAttribute(k_ssim_moments<3>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        UWS_CUDA(cudaFuncSetAttribute(k_ssim_moments<0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        UWS_CUDA(cudaFuncSetAttribute(k_ssim_grad<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kGradSmem));
        UWS_CUDA(cudaFuncSetAttribute(k_ssim_grad<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kGradSmem));
        attr_set = true;
    }
    dim3 g1((unsigned)ceil_div(vw, kT), (unsigned)ceil_div(vh, kT));
    if (c == 3)
        launch_serial(k_ssim_moments<3>, dim3(g1), dim3(kThreads), smem1, st, rendered, gt, h, w, c, p.maps, p.part_s);
    else
        launch_serial(k_ssim_moments<0>, dim3(g1), dim3(kThreads), smem1, st, rendered, gt, h, w, c, p.maps, p.part_s);
    UWS_CHECK_LAUNCH("k_ssim_moments");
    dim3 g2((unsigned)ceil_div(w, kT), (unsigned)ceil_div(h, kT));
    const float k_ssim = (float)(lambda_ssim * (-1.0 / n_win));
    const float k_l1 = (float)((1.0 - lambda_ssim) / n_px);
    if (c == 3)
        launch_serial(k_ssim_grad<3>, dim3(g2), dim3(kThreads), kGradSmem, st, rendered, gt, h, w, c, p.maps, k_ssim,
                                                        k_l1, dL_dC, p.part_l1);
    else
        launch_serial(k_ssim_grad<0>, dim3(g2), dim3(kThreads), kGradSmem, st, rendered, gt, h, w, c, p.maps, k_ssim,
                                                        k_l1, dL_dC, p.part_l1);
    UWS_CHECK_LAUNCH("k_ssim_grad");
    launch(k_loss_finalize, dim3(1), dim3(kFinThreads), 0, st, p.part_s, p.n_s, p.part_l1, p.n_l1, n_px, n_win, medium,
                                            has_guidance, lambda_ssim, lambda_guide, result,
                                            nonfinite);
    UWS_CHECK_LAUNCH("k_loss_finalize");
    return UWS_OK;
}
