// K10 fused optimizer step.
//
// Replaces optim.apply_gradients (optim.py:98-120) -> adam_step (:69-83) for
// the five cloud tensors and the three medium triplets, followed by
// GaussianCloud.normalize_rotations (scene.py:132-134) and
// MediumParams.clamp_ (scene.py:174-178).
//
// float64 arithmetic with explicitly rounded intrinsics (no FMA contraction)
// in numpy's operation order; learning rates and bias corrections
// 1 - beta^step come from the host exactly as Python computes them.  Given
// the same float32 gradients the update is therefore bit-identical to the
// reference.  Every scalar's p, m, v are read and written and g read (and
// zeroed): 392 B/Gaussian of HBM traffic, coalesced.
#include "common.cuh"

namespace uws {
namespace {

constexpr int kThreads = 256;

struct AdamK {
    double lr, b1c, b2c, r1, r2;  // r = RN(1 / b) from the host
};

// Correctly rounded a / b for a divisor known up front: q0 = RN(a * r) with
// r = RN(1/b) is within 1 ulp of a/b, the FMA residual a - b*q0 is exact, and
// one FMA correction yields RN(a/b) (Markstein).  Same result as __ddiv_rn
// for the normal-range operands Adam sees, in 3 instead of ~20 FP64 ops.
__device__ __forceinline__ double div_by_const(double a, double b, double r) {
    const double q0 = __dmul_rn(a, r);
    const double e = __fma_rn(-b, q0, a);
    return __fma_rn(e, r, q0);
}

// RN(a / b) from rb = RN(1 / b) (Markstein, as div_by_const); signed zeros kept
// (the FMA residual of a = -0 would give +0)
__device__ __forceinline__ double div_shared(double a, double b, double rb) {
    const double q0 = __dmul_rn(a, rb);
    const double e = __fma_rn(-b, q0, a);
    const double q = __fma_rn(e, rb, q0);
    return a == 0.0 ? a : q;
}

__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, const AdamK& k,
                                      const uws_adam_params& hp) {
    const double gd = (double)g;
    const double mm = __dadd_rn(__dmul_rn(hp.beta1, (double)m), __dmul_rn(hp.one_minus_beta1, gd));
    const double vv = __dadd_rn(__dmul_rn(hp.beta2, (double)v),
                                __dmul_rn(__dmul_rn(hp.one_minus_beta2, gd), gd));
    const double mh = div_by_const(mm, k.b1c, k.r1);
    const double vh = div_by_const(vv, k.b2c, k.r2);
    // Zero moments (Gaussians that never received a gradient) would send
    // sqrt and the division down their out-of-line special-operand paths;
    // their results are known exactly: sqrt(+0) = +0, and (+-0) / den = +-0
    // for den = sqrt(vh) + eps > 0.
    // (The substituted operands keep the unused branch on the inline fast path
    // when the compiler evaluates both sides of the selects.)
    // (The empty asm makes the substituted operands opaque: otherwise the
    // compiler proves them dead and feeds the zeros to sqrt/div after all.)
    const double num = __dmul_rn(k.lr, mh);
    double vs = vh == 0.0 ? 1.0 : vh, ns = num == 0.0 ? 1.0 : num;
    asm("" : "+d"(vs), "+d"(ns));
    const double den = vh == 0.0 ? hp.eps : __dadd_rn(__dsqrt_rn(vs), hp.eps);
    const double q = num == 0.0 ? num : __ddiv_rn(ns, den);
    const double upd = __dsub_rn((double)p, q);
    p = (float)upd;
    m = (float)mm;
    v = (float)vv;
}

struct AdamCtl {
    const float* skip;      // device float[2] {non-finite, overflow}: skip when either > 0
    float* grad_accum;      // densify statistics (pipeline.py:191-192), may be NULL
    int32_t* obs_count;
    int zero_grads;         // leave the gradient buffer zeroed for the next step
};


// Layout of the flat cloud buffers (scene.py field order): positions [0, 3n),
// log_scales [3n, 6n), rotations [6n, 10n), sh [10n, 13n), opacity [13n, 14n);
// the gradient buffer adds the densify statistics at [14n, 15n) and [15n, 16n).
//
// Blocks [0, nb_flat) run the elementwise update of the 10n non-rotation
// scalars, kEpt per thread with every load issued before the FP64 math;
// blocks [nb_flat, ...) take one Gaussian per thread: its quaternion (update +
// normalize_rotations) and its densify statistics.
template <int kEpt, int MINB>  // scalars per thread in the elementwise section; resident blocks
__global__ void __launch_bounds__(kThreads, MINB) k_adam_cloud(float* __restrict__ P, float* __restrict__ M,
                                                         float* __restrict__ V,
                                                         float* __restrict__ Gr, int64_t n,
                                                         int nb_flat, uws_adam_params hp,
                                                         AdamCtl ctl) {
    // launched serially (no pdl_entry): the per-CTA L1 invalidation costs more here
    const bool skip = ctl.skip && (ctl.skip[0] > 0.0f || ctl.skip[1] > 0.0f);
    if ((int)blockIdx.x < nb_flat) {
        const int64_t n10 = 10 * n;
        const int64_t t0 = (int64_t)blockIdx.x * kThreads * kEpt + threadIdx.x;
        int64_t j[kEpt];
        float p[kEpt], m[kEpt], v[kEpt], g[kEpt];
#pragma unroll
        for (int e = 0; e < kEpt; ++e) {
            const int64_t t = t0 + e * kThreads;
            j[e] = t < 6 * n ? t : t + 4 * n;  // skip the rotation block
            if (t < n10 && !skip) {
                p[e] = P[j[e]];
                m[e] = M[j[e]];
                v[e] = V[j[e]];
                g[e] = Gr[j[e]];
            }
        }
#pragma unroll
        for (int e = 0; e < kEpt; ++e) {
            const int64_t t = t0 + e * kThreads;
            if (t >= n10) break;
            if (!skip) {
                const int f = j[e] < 3 * n ? 0 : (j[e] < 6 * n ? 1 : (j[e] < 13 * n ? 3 : 4));
                const AdamK k{hp.lr[f], hp.bias1[f], hp.bias2[f], hp.inv_bias1[f],
                              hp.inv_bias2[f]};
                adam1(p[e], m[e], v[e], g[e], k, hp);
                P[j[e]] = p[e];
                M[j[e]] = m[e];
                V[j[e]] = v[e];
            }
            if (ctl.zero_grads) Gr[j[e]] = 0.f;
        }
        return;
    }
    const int64_t i = (int64_t)(blockIdx.x - nb_flat) * kThreads + threadIdx.x;
    if (i >= n) return;
    if (!skip && ctl.grad_accum) {
        ctl.grad_accum[i] += Gr[14 * n + i];
        ctl.obs_count[i] += (int32_t)Gr[15 * n + i];
    }
    if (ctl.zero_grads) {
        Gr[14 * n + i] = 0.f;
        Gr[15 * n + i] = 0.f;
    }
    const int64_t o = 6 * n + 4 * i;
    if (skip) {
        if (ctl.zero_grads)
#pragma unroll
            for (int c = 0; c < 4; ++c) Gr[o + c] = 0.f;
        return;
    }
    float p[4], m[4], v[4], g[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        p[c] = P[o + c];
        m[c] = M[o + c];
        v[c] = V[o + c];
        g[c] = Gr[o + c];
    }
    const AdamK k{hp.lr[2], hp.bias1[2], hp.bias2[2], hp.inv_bias1[2], hp.inv_bias2[2]};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        adam1(p[c], m[c], v[c], g[c], k, hp);
        M[o + c] = m[c];
        V[o + c] = v[c];
        if (ctl.zero_grads) Gr[o + c] = 0.f;
    }
    // normalize_rotations: q / max(|q|, 1e-12) in float64, stored float32
    const double a = p[0], b = p[1], c = p[2], d = p[3];
    double nr = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)),
                                              __dmul_rn(c, c)),
                                     __dmul_rn(d, d)));
    nr = fmax(nr, 1e-12);
    const double rn = __drcp_rn(nr);  // four quotients by one divisor: RN(x / nr) each
    P[o + 0] = (float)div_shared(a, nr, rn);
    P[o + 1] = (float)div_shared(b, nr, rn);
    P[o + 2] = (float)div_shared(c, nr, rn);
    P[o + 3] = (float)div_shared(d, nr, rn);
}

// Vector form for even n (the rotation block [6n, 10n) is then 16-byte aligned
// and every float4 group holds either one quaternion or four scalars of the
// other fields): 16-byte loads of p, m, v and g; group t < n also folds the
// densify statistics of Gaussian t.  Persistent grid (kAdamBlocksPerSM CTAs per
// SM), software-pipelined: each thread issues the next group's four loads
// before the float64 math of the current one, so HBM stays busy through the
// FP64 phase.
#ifndef UWS_ADAM_MINB
#define UWS_ADAM_MINB 3
#endif
constexpr int kAdamBlocksPerSM = UWS_ADAM_MINB;

__device__ __forceinline__ void adam_group(float* __restrict__ P, float* __restrict__ M,
                                           float* __restrict__ V, float* __restrict__ Gr,
                                           int64_t n, const uws_adam_params& hp,
                                           const AdamCtl& ctl, int64_t t, float4 p4, float4 m4,
                                           float4 v4, float4 g4) {
    float p[4] = {p4.x, p4.y, p4.z, p4.w}, m[4] = {m4.x, m4.y, m4.z, m4.w};
    float v[4] = {v4.x, v4.y, v4.z, v4.w};
    const float g[4] = {g4.x, g4.y, g4.z, g4.w};
    const int64_t j0 = 4 * t;
    const bool rot = j0 >= 6 * n && j0 < 10 * n;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int64_t j = j0 + c;
        const int f = rot ? 2 : (j < 3 * n ? 0 : (j < 6 * n ? 1 : (j < 13 * n ? 3 : 4)));
        const AdamK k{hp.lr[f], hp.bias1[f], hp.bias2[f], hp.inv_bias1[f], hp.inv_bias2[f]};
        adam1(p[c], m[c], v[c], g[c], k, hp);
    }
    if (rot) {
        // normalize_rotations: q / max(|q|, 1e-12) in float64, stored float32
        const double a = p[0], b = p[1], c = p[2], d = p[3];
        double nr = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)),
                                                  __dmul_rn(c, c)),
                                         __dmul_rn(d, d)));
        nr = fmax(nr, 1e-12);
        const double rn = __drcp_rn(nr);  // four quotients by one divisor: RN(x / nr) each
        p[0] = (float)div_shared(a, nr, rn);
        p[1] = (float)div_shared(b, nr, rn);
        p[2] = (float)div_shared(c, nr, rn);
        p[3] = (float)div_shared(d, nr, rn);
    }
    reinterpret_cast<float4*>(P)[t] = make_float4(p[0], p[1], p[2], p[3]);
    reinterpret_cast<float4*>(M)[t] = make_float4(m[0], m[1], m[2], m[3]);
    reinterpret_cast<float4*>(V)[t] = make_float4(v[0], v[1], v[2], v[3]);
    if (ctl.zero_grads) reinterpret_cast<float4*>(Gr)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void __launch_bounds__(kThreads, kAdamBlocksPerSM) k_adam_cloud4(
    float* __restrict__ P, float* __restrict__ M, float* __restrict__ V, float* __restrict__ Gr,
    int64_t n, uws_adam_params hp, AdamCtl ctl, int64_t g_begin, int64_t g_end) {
    // launched serially (no pdl_entry): the per-CTA L1 invalidation costs more here
    // groups [g_begin, g_end) of the 14n/4 (all of them for a whole step)
    const bool skip = ctl.skip && (ctl.skip[0] > 0.0f || ctl.skip[1] > 0.0f);
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    int64_t t = g_begin + (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const float4* P4 = reinterpret_cast<const float4*>(P);
    const float4* M4 = reinterpret_cast<const float4*>(M);
    const float4* V4 = reinterpret_cast<const float4*>(V);
    float4* G4 = reinterpret_cast<float4*>(Gr);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 p4 = z4, m4 = z4, v4 = z4, g4 = z4;
    if (t < g_end && !skip) {
        p4 = P4[t]; m4 = M4[t]; v4 = V4[t]; g4 = G4[t];
    }
    for (; t < g_end; t += stride) {
        const int64_t tn = t + stride;
        float4 pn = z4, mn = z4, vn = z4, gn = z4;
        if (tn < g_end && !skip) {  // next group's loads in flight during this group's math
            pn = P4[tn]; mn = M4[tn]; vn = V4[tn]; gn = G4[tn];
        }
        if (t < n) {
            if (!skip && ctl.grad_accum) {
                ctl.grad_accum[t] += Gr[14 * n + t];
                ctl.obs_count[t] += (int32_t)Gr[15 * n + t];
            }
            if (ctl.zero_grads) {
                Gr[14 * n + t] = 0.f;
                Gr[15 * n + t] = 0.f;
            }
        }
        if (skip) {
            if (ctl.zero_grads) G4[t] = z4;
        } else {
            adam_group(P, M, V, Gr, n, hp, ctl, t, p4, m4, v4, g4);
        }
        p4 = pn; m4 = mn; v4 = vn; g4 = gn;
    }
}

inline unsigned adam_grid(int64_t groups) {
    static int sms = 0;
    if (sms == 0 && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess)
        sms = 148;
    const int64_t need = ceil_div(groups, kThreads);
    const int64_t cap = (int64_t)sms * kAdamBlocksPerSM;
    return (unsigned)(need < cap ? need : cap);
}

__global__ void k_adam_medium(float* __restrict__ P, float* __restrict__ M, float* __restrict__ V,
                              float* __restrict__ Gr, uws_adam_params hp, AdamCtl ctl) {
    pdl_entry();
    const int v = threadIdx.x;
    if (v >= 16) return;
    const bool skip = ctl.skip && (ctl.skip[0] > 0.0f || ctl.skip[1] > 0.0f);
    __syncwarp();
    if (v >= 9 || skip) {
        // slots 9, 10 (skip counters) and the pad 11..15 are left to the host
        // launcher (the counters survive a skip, see uws_adam_step)
        return;
    }
    const int f = 5 + v / 3;
    const AdamK k{hp.lr[f], hp.bias1[f], hp.bias2[f], hp.inv_bias1[f], hp.inv_bias2[f]};
    float p = P[v], m = M[v], vv = V[v];
    adam1(p, m, vv, Gr[v], k, hp);
    // clamp_: attenuation >= 0, water_color in [0,1], backscatter in [0,5]
    if (v < 3) p = fmaxf(p, 0.0f);
    else if (v < 6) p = fminf(fmaxf(p, 0.0f), 1.0f);
    else p = fminf(fmaxf(p, 0.0f), 5.0f);
    P[v] = p;
    M[v] = m;
    V[v] = vv;
    if (ctl.zero_grads) Gr[v] = 0.f;
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_adam_step(float* params, float* exp_avg, float* exp_avg_sq, float* grads,
                             int64_t n, float* medium_params, float* medium_exp_avg,
                             float* medium_exp_avg_sq, float* medium_grads,
                             const uws_adam_params* hp, const float* skip, float* grad_accum,
                             int32_t* obs_count, int32_t zero_grads, void* stream) {
    UWS_REQUIRE(hp != nullptr && n >= 0, "uws_adam_step: bad argument");
    UWS_REQUIRE((grad_accum == nullptr) == (obs_count == nullptr),
                "uws_adam_step: grad_accum and obs_count go together");
    cudaStream_t st = as_stream(stream);
    AdamCtl ctl{skip, grad_accum, obs_count, zero_grads};
    // the medium kernel reads the skip flag before the cloud kernel may zero it
    if (medium_params) {
        UWS_REQUIRE(medium_exp_avg && medium_exp_avg_sq && medium_grads,
                    "uws_adam_step: null medium buffer");
        AdamCtl mctl = ctl;
        mctl.zero_grads = 0;
        // serial launch: after a multi-GPU all-reduce the stream waits on an event
        // right before this kernel, and a programmatic (early) launch must not
        // overtake that wait
        launch_serial(k_adam_medium, dim3(1), dim3(32), 0, st, medium_params, medium_exp_avg,
                      medium_exp_avg_sq, medium_grads, *hp, mctl);
        UWS_CHECK_LAUNCH("k_adam_medium");
    }
    if (n > 0) {
        UWS_REQUIRE(params && exp_avg && exp_avg_sq && grads, "uws_adam_step: null cloud buffer");
        const bool aligned = n % 2 == 0 &&
                             ((uintptr_t)params | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq |
                              (uintptr_t)grads) % 16 == 0;
        if (aligned) {
            launch_serial(k_adam_cloud4, dim3(adam_grid(14 * n / 4)),
                          dim3(kThreads), 0, st, params, exp_avg, exp_avg_sq, grads, n, *hp, ctl,
                          (int64_t)0, 14 * n / 4);
            UWS_CHECK_LAUNCH("k_adam_cloud4");
        } else {
            constexpr int kEpt = 2;
            const int nb_flat = (int)ceil_div(10 * n, kThreads * kEpt);
            const int nb_rot = (int)ceil_div(n, kThreads);
            launch_serial(k_adam_cloud<kEpt, 4>, dim3((unsigned)(nb_flat + nb_rot)), dim3(kThreads), 0, st, 
                params, exp_avg, exp_avg_sq, grads, n, nb_flat, *hp, ctl);
            UWS_CHECK_LAUNCH("k_adam_cloud");
        }
    }
    if (medium_params && zero_grads) {
        // medium slots and pad zeroed after every reader is done; the skip
        // counters (slots 9, 10) are left alone: non-zero they keep skipping
        // later steps until the host has handled the skip and cleared them
        UWS_CUDA(zero_async2(medium_grads, 9 * sizeof(float), medium_grads + 11,
                             5 * sizeof(float), st));
    }
    return UWS_OK;
}

extern "C" int uws_adam_step_range(float* params, float* exp_avg, float* exp_avg_sq, float* grads,
                                   int64_t n, const uws_adam_params* hp, const float* skip,
                                   float* grad_accum, int32_t* obs_count, int32_t zero_grads,
                                   int64_t group_begin, int64_t group_end, void* stream) {
    UWS_REQUIRE(hp != nullptr && n > 0 && n % 2 == 0, "uws_adam_step_range: needs an even n > 0");
    UWS_REQUIRE(params && exp_avg && exp_avg_sq && grads, "uws_adam_step_range: null cloud buffer");
    UWS_REQUIRE(((uintptr_t)params | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq |
                 (uintptr_t)grads) % 16 == 0,
                "uws_adam_step_range: buffers must be 16-byte aligned");
    UWS_REQUIRE((grad_accum == nullptr) == (obs_count == nullptr),
                "uws_adam_step_range: grad_accum and obs_count go together");
    UWS_REQUIRE(0 <= group_begin && group_begin <= group_end && group_end <= 14 * n / 4,
                "uws_adam_step_range: group range out of bounds");
    if (group_end == group_begin) return UWS_OK;
    AdamCtl ctl{skip, grad_accum, obs_count, zero_grads};
    launch_serial(k_adam_cloud4, dim3(adam_grid(group_end - group_begin)),
                  dim3(kThreads), 0, as_stream(stream), params, exp_avg, exp_avg_sq, grads, n, *hp,
                  ctl, group_begin, group_end);
    UWS_CHECK_LAUNCH("k_adam_cloud4");
    return UWS_OK;
}
