// Float64 per-Gaussian projection geometry shared by the preprocess forward
// (preprocess.cu) and backward (preprocess_bwd.cu) kernels.  Both
// translation units are compiled with -fmad=false so the expressions below
// are evaluated exactly as numpy evaluates the reference
// (projection.py:111-158, scene.py:32-48); numpy's fused matmul inner
// products are reproduced with explicit __fma_rn in the same order.
#pragma once

#include "common.cuh"

namespace uws {

__device__ __forceinline__ double dot3f(double a0, double a1, double a2, double b0, double b1,
                                        double b2) {
    return __fma_rn(a2, b2, __fma_rn(a1, b1, a0 * b0));
}

// RN(a / b) from rb = RN(1 / b) (__drcp_rn): q0 = RN(a rb) is within an ulp of a/b,
// the residual a - b q0 is exact as one FMA and the FMA correction rounds to RN(a/b)
// (Markstein), for the normal-range operands of the projection.  Several quotients
// by one divisor then cost one correctly rounded reciprocal plus three FP64 ops each
// instead of a full division each.  A zero dividend keeps its sign (-0 / b = -0).
__device__ __forceinline__ double div_rcp(double a, double b, double rb) {
#ifdef UWS_GEO_PLAINDIV
    return __ddiv_rn(a, b);
#endif
    const double q0 = __dmul_rn(a, rb);
    const double e = __fma_rn(-b, q0, a);
    const double q = __fma_rn(e, rb, q0);
    return a == 0.0 ? a : q;
}

struct Geo {
    double vx, vy, vz;     // view-space mean (projection.py:112)
    double u, v;           // vx/vz, vy/vz (unclamped)
    double xu, yu;         // clamped tx, ty used by the Jacobian (:134-135)
    bool xm, ym;           // frustum clamp active (:132-133)
    double limx, limy;
    float qraw[4], lsraw[3];  // the Gaussian's rotation / log-scale record (loaded with the mean)
    double qn, rqn;        // |q| (:138), RN(1 / |q|)
    double qu[4];          // q/|q| (:139)
    double Rq[9];          // quat_to_rotmat(q/|q|) (normalises again)
    double s[3];           // exp(log_scale)
    double S[9];           // cov3d = M M^T
    double T[6];           // J R_view
};

// view transform only (cheap cull test first)
__device__ __forceinline__ void geo_view(const uws_cloud& cl, const uws_camera& cam, int64_t i,
                                         Geo& g) {
    const double* R = cam.R;
    double p0 = cl.positions[3 * i + 0], p1 = cl.positions[3 * i + 1], p2 = cl.positions[3 * i + 2];
#ifndef UWS_GEO_LATE_LOADS
    // every load of the record issued here, together (their latencies overlap)
#pragma unroll
    for (int c = 0; c < 4; ++c) g.qraw[c] = cl.rotations[4 * i + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) g.lsraw[c] = cl.log_scales[3 * i + c];
#endif
    g.vx = dot3f(p0, p1, p2, R[0], R[1], R[2]) + cam.t[0];
    g.vy = dot3f(p0, p1, p2, R[3], R[4], R[5]) + cam.t[1];
    g.vz = dot3f(p0, p1, p2, R[6], R[7], R[8]) + cam.t[2];
}

// the frustum-clamp limits 1.3 * ((0.5 * width) / fx) (projection.py:132-133), per camera:
// computed once on the host (IEEE double, the same operations)
struct FrustumLim {
    double x, y;
};
inline FrustumLim frustum_lim(const uws_camera& cam) {
    return FrustumLim{1.3 * ((0.5 * cam.width) / cam.fx), 1.3 * ((0.5 * cam.height) / cam.fy)};
}

__device__ __forceinline__ void geo_shape(const uws_cloud& cl, const uws_camera& cam, int64_t i,
                                          const FrustumLim& lim, Geo& g) {
    const double* R = cam.R;
    g.limx = lim.x;
    g.limy = lim.y;
    const double rz = __drcp_rn(g.vz);  // = 1.0 / vz
    g.u = div_rcp(g.vx, g.vz, rz);
    g.v = div_rcp(g.vy, g.vz, rz);
    double uc = fmin(fmax(g.u, -g.limx), g.limx);
    double vc = fmin(fmax(g.v, -g.limy), g.limy);
    g.xm = g.u != uc;
    g.ym = g.v != vc;
    g.xu = uc * g.vz;
    g.yu = vc * g.vz;

#ifdef UWS_GEO_LATE_LOADS
#pragma unroll
    for (int c = 0; c < 4; ++c) g.qraw[c] = cl.rotations[4 * i + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) g.lsraw[c] = cl.log_scales[3 * i + c];
#endif
    double q0 = g.qraw[0], q1 = g.qraw[1], q2 = g.qraw[2], q3 = g.qraw[3];
    g.qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    const double rq = g.rqn = __drcp_rn(g.qn);
    g.qu[0] = div_rcp(q0, g.qn, rq); g.qu[1] = div_rcp(q1, g.qn, rq);
    g.qu[2] = div_rcp(q2, g.qn, rq); g.qu[3] = div_rcp(q3, g.qn, rq);
    double n2 = sqrt(((g.qu[0] * g.qu[0] + g.qu[1] * g.qu[1]) + g.qu[2] * g.qu[2]) + g.qu[3] * g.qu[3]);
    const double rn2 = __drcp_rn(n2);
    double w = div_rcp(g.qu[0], n2, rn2), x = div_rcp(g.qu[1], n2, rn2);
    double y = div_rcp(g.qu[2], n2, rn2), z = div_rcp(g.qu[3], n2, rn2);
    double* Rq = g.Rq;
    Rq[0] = 1 - 2 * (y * y + z * z); Rq[1] = 2 * (x * y - w * z); Rq[2] = 2 * (x * z + w * y);
    Rq[3] = 2 * (x * y + w * z); Rq[4] = 1 - 2 * (x * x + z * z); Rq[5] = 2 * (y * z - w * x);
    Rq[6] = 2 * (x * z - w * y); Rq[7] = 2 * (y * z + w * x); Rq[8] = 1 - 2 * (x * x + y * y);
    g.s[0] = exp((double)g.lsraw[0]);
    g.s[1] = exp((double)g.lsraw[1]);
    g.s[2] = exp((double)g.lsraw[2]);
    double M[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M[3 * r + c] = Rq[3 * r + c] * g.s[c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            g.S[3 * r + c] = dot3f(M[3 * r], M[3 * r + 1], M[3 * r + 2], M[3 * c], M[3 * c + 1], M[3 * c + 2]);

    const double rz2 = rz * rz;
    double J00 = cam.fx * rz, J02 = (-cam.fx * g.xu) * rz2;
    double J11 = cam.fy * rz, J12 = (-cam.fy * g.yu) * rz2;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        g.T[c] = dot3f(J00, 0.0, J02, R[c], R[3 + c], R[6 + c]);
        g.T[3 + c] = dot3f(0.0, J11, J12, R[c], R[3 + c], R[6 + c]);
    }
}

}  // namespace uws
