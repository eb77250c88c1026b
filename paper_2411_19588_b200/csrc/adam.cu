// K10 fused optimizer step.
//
// Replaces optim.apply_gradients (optim.py:98-120) -> adam_step (:69-83) for
// the five cloud tensors and the three medium triplets, followed by
// GaussianCloud.normalize_rotations (scene.py:165-167) and
// MediumParams.clamp_ (scene.py:207-211).
//
// float64 arithmetic with explicitly rounded intrinsics (no FMA contraction)
// in numpy's operation order; learning rates and bias corrections
// 1 - beta^step come from the host exactly as Python computes them.  Given
// the same float32 gradients the update is therefore bit-identical to the
// reference.  One thread per Gaussian touches its 14 scalars (p, m, v read
// and written, g read): 392 B/Gaussian of HBM traffic, coalesced per field.
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

__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, const AdamK& k,
                                      const uws_adam_params& hp) {
    const double gd = (double)g;
    const double mm = __dadd_rn(__dmul_rn(hp.beta1, (double)m), __dmul_rn(hp.one_minus_beta1, gd));
    const double vv = __dadd_rn(__dmul_rn(hp.beta2, (double)v),
                                __dmul_rn(__dmul_rn(hp.one_minus_beta2, gd), gd));
    const double mh = div_by_const(mm, k.b1c, k.r1);
    const double vh = div_by_const(vv, k.b2c, k.r2);
    const double upd = __dsub_rn((double)p, __ddiv_rn(__dmul_rn(k.lr, mh), __dadd_rn(__dsqrt_rn(vh), hp.eps)));
    p = (float)upd;
    m = (float)mm;
    v = (float)vv;
}

struct AdamCtl {
    const float* skip;      // device: skip the update when *skip > 0 (non-finite count)
    float* grad_accum;      // densify statistics (pipeline.py:191-192), may be NULL
    int32_t* obs_count;
    int zero_grads;         // leave the gradient buffer zeroed for the next step
};

__global__ void __launch_bounds__(kThreads) k_adam_cloud(float* __restrict__ P, float* __restrict__ M,
                                                         float* __restrict__ V,
                                                         float* __restrict__ Gr, int64_t n,
                                                         uws_adam_params hp, AdamCtl ctl) {
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (i >= n) return;
    const bool skip = ctl.skip && *ctl.skip > 0.0f;
    if (skip) {
        if (ctl.zero_grads) {
            const int64_t base[5] = {0, 3 * n, 6 * n, 10 * n, 13 * n};
            const int width[5] = {3, 3, 4, 3, 1};
#pragma unroll
            for (int f = 0; f < 5; ++f)
                for (int c = 0; c < width[f]; ++c) Gr[base[f] + i * width[f] + c] = 0.f;
            Gr[14 * n + i] = 0.f;
            Gr[15 * n + i] = 0.f;
        }
        return;
    }
    if (ctl.grad_accum) {
        ctl.grad_accum[i] += Gr[14 * n + i];
        ctl.obs_count[i] += (int32_t)Gr[15 * n + i];
    }
    if (ctl.zero_grads) {
        Gr[14 * n + i] = 0.f;
        Gr[15 * n + i] = 0.f;
    }
    const int64_t base[5] = {0, 3 * n, 6 * n, 10 * n, 13 * n};
    const int width[5] = {3, 3, 4, 3, 1};
#pragma unroll
    for (int f = 0; f < 5; ++f) {
        const AdamK k{hp.lr[f], hp.bias1[f], hp.bias2[f], hp.inv_bias1[f], hp.inv_bias2[f]};
        float q[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (c >= width[f]) break;
            const int64_t o = base[f] + i * width[f] + c;
            float p = P[o], m = M[o], v = V[o];
            adam1(p, m, v, Gr[o], k, hp);
            if (ctl.zero_grads) Gr[o] = 0.f;
            q[c] = p;
            M[o] = m;
            V[o] = v;
            if (f != 2) P[o] = p;
        }
        if (f == 2) {
            // normalize_rotations: q / max(|q|, 1e-12) in float64, stored float32
            const double a = q[0], b = q[1], c = q[2], d = q[3];
            double nr = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)),
                                                      __dmul_rn(c, c)),
                                             __dmul_rn(d, d)));
            nr = fmax(nr, 1e-12);
            const int64_t o = base[2] + i * 4;
            P[o + 0] = (float)__ddiv_rn(a, nr);
            P[o + 1] = (float)__ddiv_rn(b, nr);
            P[o + 2] = (float)__ddiv_rn(c, nr);
            P[o + 3] = (float)__ddiv_rn(d, nr);
        }
    }
}

__global__ void k_adam_medium(float* __restrict__ P, float* __restrict__ M, float* __restrict__ V,
                              float* __restrict__ Gr, uws_adam_params hp, AdamCtl ctl) {
    const int v = threadIdx.x;
    if (v >= 16) return;
    const bool skip = ctl.skip && *ctl.skip > 0.0f;
    __syncwarp();
    if (v >= 9 || skip) {
        // slots 9..15 (non-finite counter + pad) are reset after every step
        if (ctl.zero_grads) Gr[v] = 0.f;
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
        k_adam_medium<<<1, 32, 0, st>>>(medium_params, medium_exp_avg, medium_exp_avg_sq,
                                        medium_grads, *hp, mctl);
        UWS_CHECK_LAUNCH("k_adam_medium");
    }
    if (n > 0) {
        UWS_REQUIRE(params && exp_avg && exp_avg_sq && grads, "uws_adam_step: null cloud buffer");
        k_adam_cloud<<<(unsigned)ceil_div(n, kThreads), kThreads, 0, st>>>(params, exp_avg, exp_avg_sq,
                                                                           grads, n, *hp, ctl);
        UWS_CHECK_LAUNCH("k_adam_cloud");
    }
    if (medium_params && zero_grads) {
        // medium slots + counter/pad (16 floats) zeroed after every reader is done
        UWS_CUDA(cudaMemsetAsync(medium_grads, 0, 16 * sizeof(float), st));
    }
    return UWS_OK;
}
