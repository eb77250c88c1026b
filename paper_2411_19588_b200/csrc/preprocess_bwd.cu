// K9 projection backward: screen-space gradients -> world parameters.
//
// Replaces backward._project_backward (backward.py:184-258) and
// _quat_backward (:166-181), plus the medium-gradient merge of
// backward_render (:294-302) and the guidance subgradient of
// backward_medium (:270-274).
//
// One thread per visible row.  Instead of storing the reference's backward
// context (t_view, rotmat, cov3d, clamp masks ...; projection.py:187-198)
// the forward geometry is recomputed in float64 from the 56-byte parameter
// record (project_math.cuh) -- cheaper than writing and re-reading ~200 B
// per Gaussian.  Each visible row maps to a distinct source Gaussian, so the
// accumulation into the flat gradient buffer needs no atomics.
#include "project_math.cuh"

namespace uws {
namespace {

constexpr int kThreads = 128;

// Arithmetic type of the chain rule below the recomputed float64 geometry (float64,
// as the reference).  With the projection's divisions by one divisor done as one
// correctly rounded reciprocal + Markstein corrections (project_math.cuh) and every
// record load issued up front, the float64 chain rule is the faster one at C3:
// 0.064 ms vs 0.115 ms for a float32 chain rule (-DUWS_PBWD_F32), whose schedule
// exposes the load latencies (ncu: long_scoreboard 21 cycles per issue).
#ifdef UWS_PBWD_F32
typedef float real;
#else
typedef double real;
#endif

template <bool ACC>  // add into the gradient buffer (else store: it is known to be zero)
__global__ void __launch_bounds__(kThreads, 5) k_preprocess_bwd(uws_cloud cl, uws_camera cam,
                                                             FrustumLim lim,
                                                             const int32_t* __restrict__ src_index,
                                                             const double* __restrict__ exact,
                                                             const int32_t* __restrict__ k_dev,
                                                             float* __restrict__ screen,
                                                             float* __restrict__ grads,
                                                             float* __restrict__ nonfinite) {
    // launched serially (no pdl_entry): measured 1.7x slower with it
    const int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (row >= (int64_t)*k_dev) return;
    const int64_t n = cl.n;
    const int64_t i = src_index[row];
    float* sg = screen + row * 9;
    const real gl = sg[0], dmx = sg[1], dmy = sg[2];
    const real dca = sg[3], dcb = sg[4], dcc = sg[5];
    const real dcol[3] = {sg[6], sg[7], sg[8]};
    // leave the screen-space accumulator zeroed for the next view
#pragma unroll
    for (int v = 0; v < 9; ++v) sg[v] = 0.f;

    const double4 ex = reinterpret_cast<const double4*>(exact)[row];  // conic, opacity
    float sh[3];  // issued with the record loads of geo_view
#pragma unroll
    for (int c = 0; c < 3; ++c) sh[c] = cl.sh_coeffs[3 * i + c];
    Geo G;
    geo_view(cl, cam, i, G);
    geo_shape(cl, cam, i, lim, G);
    // geometry in the chain rule's type (float64 decisions above are kept: xm, ym, signs)
    real GS[9], GRq[9], Gs[3], Gqu[4];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        GS[q] = (real)G.S[q];
        GRq[q] = (real)G.Rq[q];
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) Gs[q] = (real)G.s[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) Gqu[q] = (real)G.qu[q];
    const real fx = (real)cam.fx, fy = (real)cam.fy;
    const real vz = (real)G.vz, xu = (real)G.xu, yu = (real)G.yu, vx = (real)G.vx, vy = (real)G.vy;
    const real k0 = (real)ex.x, k1 = (real)ex.y, k2 = (real)ex.z, sop = (real)ex.w;
    real R[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) R[q] = (real)cam.R[q];

    // conic -> cov2d: dX = -Y dY Y (:192-204)
    const real h = (real)0.5 * dcb;
    const real P00 = k0 * dca + k1 * h, P01 = k0 * h + k1 * dcc;
    const real P10 = k1 * dca + k2 * h, P11 = k1 * h + k2 * dcc;
    const real X00 = -(P00 * k0 + P01 * k1);
    const real X01 = -(P00 * k1 + P01 * k2);
    const real X11 = -(P10 * k1 + P11 * k2);
    const real G2[4] = {X00, X01, X01, X11};

    // dSigma = T^T G2 T ; dT = 2 G2 T Sigma ; dJ = dT R^T (:214-217)
    real T[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) T[q] = (real)G.T[q];
    real GT[6];  // G2 T (2x3)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) GT[3 * r + c] = G2[2 * r] * T[c] + G2[2 * r + 1] * T[3 + c];
    real dS[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) dS[3 * a + b] = T[a] * GT[b] + T[3 + a] * GT[3 + b];
    real dT[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dT[3 * r + c] = (real)2 * (GT[3 * r] * GS[c] + GT[3 * r + 1] * GS[3 + c] + GT[3 * r + 2] * GS[6 + c]);
    real dJ[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dJ[3 * r + c] = dT[3 * r] * R[3 * c] + dT[3 * r + 1] * R[3 * c + 1] + dT[3 * r + 2] * R[3 * c + 2];

    // cov3d = M M^T, M = Rq diag(s): dM = 2 dSigma M (:220-224)
    real M[9], dM[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M[3 * r + c] = GRq[3 * r + c] * Gs[c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dM[3 * r + c] = (real)2 * (dS[3 * r] * M[c] + dS[3 * r + 1] * M[3 + c] + dS[3 * r + 2] * M[6 + c]);
    real dls[3], gR[9];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        dls[c] = (GRq[c] * dM[c] + GRq[3 + c] * dM[3 + c] + GRq[6 + c] * dM[6 + c]) * Gs[c];
#pragma unroll
        for (int r = 0; r < 3; ++r) gR[3 * r + c] = dM[3 * r + c] * Gs[c];
    }
    // rotation matrix -> raw quaternion (:166-181)
    const real w = Gqu[0], x = Gqu[1], y = Gqu[2], z = Gqu[3];
#define g(r, c) gR[3 * (r) + (c)]
    real dq[4];
    dq[0] = 2 * (z * (g(1, 0) - g(0, 1)) + y * (g(0, 2) - g(2, 0)) + x * (g(2, 1) - g(1, 2)));
    dq[1] = 2 * (y * (g(0, 1) + g(1, 0)) + z * (g(0, 2) + g(2, 0)) + w * (g(2, 1) - g(1, 2)) -
                 2 * x * (g(1, 1) + g(2, 2)));
    dq[2] = 2 * (x * (g(0, 1) + g(1, 0)) + w * (g(0, 2) - g(2, 0)) + z * (g(1, 2) + g(2, 1)) -
                 2 * y * (g(0, 0) + g(2, 2)));
    dq[3] = 2 * (w * (g(1, 0) - g(0, 1)) + x * (g(0, 2) + g(2, 0)) + y * (g(1, 2) + g(2, 1)) -
                 2 * z * (g(0, 0) + g(1, 1)));
#undef g
    const real radial = dq[0] * w + dq[1] * x + dq[2] * y + dq[3] * z;

    // view-space point: through J (clamped) and the unclamped mean (:226-248)
    const real rz = (real)1 / vz, rz2 = rz * rz, rz3 = rz2 * rz;
    const real dxu = dJ[2] * (-fx * rz2);
    const real dyu = dJ[5] * (-fy * rz2);
    real dtz = dJ[0] * (-fx * rz2) + dJ[2] * ((real)2 * fx * xu * rz3) +
                 dJ[4] * (-fy * rz2) + dJ[5] * ((real)2 * fy * yu * rz3);
    real dtx = G.xm ? (real)0 : dxu;
    real dty = G.ym ? (real)0 : dyu;
    if (G.xm) dtz += dxu * (real)((G.u > 0 ? 1.0 : (G.u < 0 ? -1.0 : 0.0)) * G.limx);
    if (G.ym) dtz += dyu * (real)((G.v > 0 ? 1.0 : (G.v < 0 ? -1.0 : 0.0)) * G.limy);
    dtx += dmx * fx * rz;
    dty += dmy * fy * rz;
    dtz = dtz - dmx * fx * vx * rz2 - dmy * fy * vy * rz2;

    float* gpos = grads;
    float* gls = grads + 3 * n;
    float* grot = grads + 6 * n;
    float* gsh = grads + 10 * n;
    float* gop = grads + 13 * n;
    float* gnorm = grads + 14 * n;
    float* gobs = grads + 15 * n;
    bool finite = true;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float v = (ACC ? gpos[3 * i + c] : 0.f) + (float)(dtx * R[c] + dty * R[3 + c] + dtz * R[6 + c]);
        gpos[3 * i + c] = v;
        finite &= isfinite(v);
        v = (ACC ? gls[3 * i + c] : 0.f) + (float)dls[c];
        gls[3 * i + c] = v;
        finite &= isfinite(v);
        const double col = (double)sh[c] * kSH_C0 + 0.5;
        v = (ACC ? gsh[3 * i + c] : 0.f) + (col > 0.0 ? (float)((real)kSH_C0 * dcol[c]) : 0.0f);
        gsh[3 * i + c] = v;
        finite &= isfinite(v);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float v = (ACC ? grot[4 * i + c] : 0.f) + (float)div_rcp((double)(dq[c] - Gqu[c] * radial), G.qn, G.rqn);
        grot[4 * i + c] = v;
        finite &= isfinite(v);
    }
    {
        float v = (ACC ? gop[i] : 0.f) + (float)(((real)1 - sop) * gl);
        gop[i] = v;
        finite &= isfinite(v);
    }
    const double nx = (double)dmx * cam.width * 0.5, ny = (double)dmy * cam.height * 0.5;
    gnorm[i] = (ACC ? gnorm[i] : 0.f) + (float)sqrt_nz(nx * nx + ny * ny);
    gobs[i] = (ACC ? gobs[i] : 0.f) + 1.0f;
    if (!finite && nonfinite) atomicAdd(nonfinite, 1.0f);
}

// medium slots: accumulated image sums + lambda * sign(param - guide); the
// accumulator is left zeroed for the next view
__global__ void k_medium_finalize(double* __restrict__ acc, const float* __restrict__ medium,
                                  int has_guidance, double lam, float* __restrict__ gmed,
                                  float* __restrict__ nonfinite) {
    pdl_entry();
    const int v = threadIdx.x;
    if (v >= 9) return;
    double s = acc ? acc[v] : 0.0;
    if (acc) acc[v] = 0.0;
    if (acc && has_guidance && lam != 0.0 && v >= 3) {
        double d = (double)medium[v] - (double)medium[v + 6];
        s += lam * (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0));
    }
    const float r = gmed[v] + (float)s;
    gmed[v] = r;
    if (!isfinite(r) && nonfinite) atomicAdd(nonfinite, 1.0f);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_preprocess_bwd(const uws_cloud* cloud, const uws_camera* cam,
                                  const uws_projected* proj, int64_t k_cap, float* screen_grads,
                                  double* medium_acc, const float* medium, int32_t has_guidance,
                                  double lambda_guide, float* grads, float* nonfinite,
                                  int32_t accumulate, void* stream) {
    UWS_REQUIRE(cloud && cam && proj && grads && proj->num_visible, "uws_preprocess_bwd: null argument");
    UWS_REQUIRE(k_cap >= 0 && k_cap <= cloud->n, "uws_preprocess_bwd: k out of range");
    UWS_REQUIRE(medium_acc == nullptr || medium != nullptr, "uws_preprocess_bwd: medium missing");
    cudaStream_t st = as_stream(stream);
    if (k_cap > 0) {
        UWS_REQUIRE(screen_grads != nullptr, "uws_preprocess_bwd: screen_grads missing");
        const unsigned nb = (unsigned)ceil_div(k_cap, kThreads);
        if (accumulate)
            launch_serial(k_preprocess_bwd<true>, dim3(nb), dim3(kThreads), 0, st, *cloud, *cam, frustum_lim(*cam), proj->source_index,
                                                           proj->exact, proj->num_visible,
                                                           screen_grads, grads, nonfinite);
        else
            launch_serial(k_preprocess_bwd<false>, dim3(nb), dim3(kThreads), 0, st, *cloud, *cam, frustum_lim(*cam), proj->source_index,
                                                            proj->exact, proj->num_visible,
                                                            screen_grads, grads, nonfinite);
        UWS_CHECK_LAUNCH("k_preprocess_bwd");
    }
    if (medium_acc) {
        launch(k_medium_finalize, dim3(1), dim3(32), 0, st, medium_acc, medium, has_guidance, lambda_guide,
                                            grads + 16 * cloud->n, nonfinite);
        UWS_CHECK_LAUNCH("k_medium_finalize");
    }
    return UWS_OK;
}
