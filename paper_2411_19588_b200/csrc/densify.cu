// K11 densification on the device: clone / split / prune with stream
// compaction, and the opacity reset.
//
// Replaces optim.densify_and_prune (optim.py:132-198) and reset_opacities
// (optim.py:201-207).  The reference's new cloud is the concatenation
//     [kept rows, in order | clones, in order | split child 0 | split child 1]
// where keep = ~(prune | split), clone = candidate & small & ~prune and
// split = candidate & ~small & ~prune.  Here:
//   1. k_dens_classify: per Gaussian, the three flags in float64 exactly as
//      numpy evaluates them (mean gradient, max exp(log_scale), expit), and
//      per-block counts (2048 Gaussians per block);
//   2. k_dens_scan: one block scans the per-block counts -> block offsets and
//      the totals (n_keep, n_clone, n_split) the host reads to size the new
//      buffers and to draw the split samples with its numpy Generator;
//   3. k_dens_apply: each block re-ranks its Gaussians and writes every
//      output row once: kept rows with their Adam moments, clones and split
//      children with zero moments; split children get
//      position + R(q) (sample * exp(log_scale)) and log_scale - log(factor)
//      in float64 (built with -fmad=false: numpy's operation order, no FMA).
#include "common.cuh"
#include "scan.cuh"

namespace uws {
namespace {

constexpr int kThreads = 256;
constexpr int kIpt = 8;
constexpr int kBlockItems = kThreads * kIpt;  // 2048
constexpr unsigned char kKeep = 1, kClone = 2, kSplit = 4;

// per-Gaussian field offsets in the flat [pos 3n | ls 3n | rot 4n | sh 3n | op n] layout
struct Fields {
    int64_t n;
    __device__ int64_t pos(int64_t i) const { return 3 * i; }
    __device__ int64_t ls(int64_t i) const { return 3 * n + 3 * i; }
    __device__ int64_t rot(int64_t i) const { return 6 * n + 4 * i; }
    __device__ int64_t sh(int64_t i) const { return 10 * n + 3 * i; }
    __device__ int64_t op(int64_t i) const { return 13 * n + i; }
};

__device__ __forceinline__ unsigned long long pack3(unsigned a, unsigned b, unsigned c) {
    return (unsigned long long)a | ((unsigned long long)b << 21) | ((unsigned long long)c << 42);
}
__device__ __forceinline__ unsigned field3(unsigned long long v, int k) {
    return (unsigned)((v >> (21 * k)) & ((1ull << 21) - 1));
}

__global__ void __launch_bounds__(kThreads) k_dens_classify(
    const float* __restrict__ P, int64_t n, const float* __restrict__ grad_accum,
    const int32_t* __restrict__ obs, double grad_thr, double size_thr, double min_opacity,
    unsigned char* __restrict__ codes, unsigned long long* __restrict__ blk_counts) {
    pdl_entry();
    __shared__ unsigned long long s_tmp[kThreads / 32 + 1];
    const Fields F{n};
    unsigned keep = 0, clone = 0, split = 0;
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
#pragma unroll
    for (int k = 0; k < kIpt; ++k) {
        const int64_t i = base + k * kThreads + threadIdx.x;
        if (i >= n) break;
        // optim.py:143-145: mean_grad = grad_accum / max(obs, 1) (float64)
        const double cnt = (double)obs[i];
        const double mean_grad = (double)grad_accum[i] / fmax(cnt, 1.0);
        const bool candidate = mean_grad > grad_thr && obs[i] > 0;
        // :147-148: max over axes of exp(log_scale)
        const double s0 = exp((double)P[F.ls(i) + 0]), s1 = exp((double)P[F.ls(i) + 1]),
                     s2 = exp((double)P[F.ls(i) + 2]);
        const double max_scale = fmax(fmax(s0, s1), s2);
        const bool small = max_scale <= size_thr;
        // :153-154: expit (scipy: 1 / (1 + exp(-x)))
        const double opacity = 1.0 / (1.0 + exp(-(double)P[F.op(i)]));
        const bool prune = opacity < min_opacity;
        const bool c = candidate && small && !prune;
        const bool s = candidate && !small && !prune;
        const bool kp = !(prune || s);
        codes[i] = (unsigned char)((kp ? kKeep : 0) | (c ? kClone : 0) | (s ? kSplit : 0));
        keep += kp;
        clone += c;
        split += s;
    }
    unsigned long long tot;
    block_exclusive_sum<kThreads, unsigned long long>(pack3(keep, clone, split), s_tmp, &tot);
    if (threadIdx.x == 0) blk_counts[blockIdx.x] = tot;
}

// one block: exclusive offsets per block (3 x int64) and the totals
__global__ void __launch_bounds__(1024) k_dens_scan(const unsigned long long* __restrict__ blk_counts,
                                                     int nblk, long long* __restrict__ blk_off,
                                                     long long* __restrict__ totals) {
    pdl_entry();
    __shared__ long long s_tmp[3][1024 / 32 + 1];
    long long run[3] = {0, 0, 0};
    for (int c0 = 0; c0 < nblk; c0 += 1024) {
        const int b = c0 + (int)threadIdx.x;
        const unsigned long long v = b < nblk ? blk_counts[b] : 0ull;
        for (int k = 0; k < 3; ++k) {
            long long tot;
            const long long ex =
                block_exclusive_sum<1024, long long>((long long)field3(v, k), s_tmp[k], &tot);
            if (b < nblk) blk_off[3 * b + k] = run[k] + ex;
            run[k] += tot;
            __syncthreads();
        }
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < 3; ++k) totals[k] = run[k];
}

// quat_to_rotmat (scene.py:32-48): normalize by sqrt(((w^2 + x^2) + y^2) + z^2),
// then the textbook matrix, in numpy's evaluation order
__device__ void rotmat(const float* q4, double R[9]) {
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    const double nr = sqrt(((w * w + x * x) + y * y) + z * z);
    w = w / nr;
    x = x / nr;
    y = y / nr;
    z = z / nr;
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
}

__device__ __forceinline__ void copy_row(const float* __restrict__ src, float* __restrict__ dst,
                                         const Fields& A, const Fields& B, int64_t i, int64_t j) {
#pragma unroll
    for (int c = 0; c < 3; ++c) dst[B.pos(j) + c] = src[A.pos(i) + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) dst[B.ls(j) + c] = src[A.ls(i) + c];
#pragma unroll
    for (int c = 0; c < 4; ++c) dst[B.rot(j) + c] = src[A.rot(i) + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) dst[B.sh(j) + c] = src[A.sh(i) + c];
    dst[B.op(j)] = src[A.op(i)];
}

__global__ void __launch_bounds__(kThreads) k_dens_apply(
    const float* __restrict__ P, const float* __restrict__ M, const float* __restrict__ V,
    int64_t n, const unsigned char* __restrict__ codes, const long long* __restrict__ blk_off,
    const double* __restrict__ samples, double log_factor, int64_t n_keep, int64_t n_clone,
    int64_t n_split, float* __restrict__ P2, float* __restrict__ M2, float* __restrict__ V2) {
    pdl_entry();
    __shared__ unsigned long long s_tmp[kThreads / 32 + 1];
    const Fields A{n};
    const Fields B{n_keep + n_clone + 2 * n_split};
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    // blocked ranks: thread t owns items base + t*kIpt .. +kIpt (list order)
    unsigned char cd[kIpt];
    unsigned keep = 0, clone = 0, split = 0;
#pragma unroll
    for (int k = 0; k < kIpt; ++k) {
        const int64_t i = base + (int64_t)threadIdx.x * kIpt + k;
        cd[k] = i < n ? codes[i] : 0;
        keep += (cd[k] & kKeep) != 0;
        clone += (cd[k] & kClone) != 0;
        split += (cd[k] & kSplit) != 0;
    }
    unsigned long long tot;
    const unsigned long long ex =
        block_exclusive_sum<kThreads, unsigned long long>(pack3(keep, clone, split), s_tmp, &tot);
    int64_t rk = blk_off[3 * blockIdx.x + 0] + field3(ex, 0);
    int64_t rc = blk_off[3 * blockIdx.x + 1] + field3(ex, 1);
    int64_t rs = blk_off[3 * blockIdx.x + 2] + field3(ex, 2);
#pragma unroll 1
    for (int k = 0; k < kIpt; ++k) {
        const int64_t i = base + (int64_t)threadIdx.x * kIpt + k;
        if (i >= n) break;
        if (cd[k] & kKeep) {
            copy_row(P, P2, A, B, i, rk);
            copy_row(M, M2, A, B, i, rk);
            copy_row(V, V2, A, B, i, rk);
            ++rk;
        }
        if (cd[k] & kClone) {
            copy_row(P, P2, A, B, i, n_keep + rc);  // moments start at zero
            ++rc;
        }
        if (cd[k] & kSplit) {
            double R[9];
            rotmat(P + A.rot(i), R);
            double s[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) s[c] = exp((double)P[A.ls(i) + c]);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int64_t j = n_keep + n_clone + half * n_split + rs;
                const double* smp = samples + ((int64_t)half * n_split + rs) * 3;
                double v[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) v[c] = smp[c] * s[c];
                copy_row(P, P2, A, B, i, j);
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    // einsum("nij,nj->ni"): ((R0 v0 + R1 v1) + R2 v2)
                    const double off = (R[3 * r] * v[0] + R[3 * r + 1] * v[1]) + R[3 * r + 2] * v[2];
                    P2[B.pos(j) + r] = (float)((double)P[A.pos(i) + r] + off);
                    P2[B.ls(j) + r] = (float)((double)P[A.ls(i) + r] - log_factor);
                }
            }
            ++rs;
        }
    }
}

__global__ void k_reset_opacity(float* __restrict__ P, float* __restrict__ M,
                                float* __restrict__ V, int64_t n, float value) {
    pdl_entry();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    P[13 * n + i] = value;
    M[13 * n + i] = 0.f;
    V[13 * n + i] = 0.f;
}

struct DensPlan {
    unsigned char* codes;
    unsigned long long* blk_counts;
    long long* blk_off;
    int nblk;
};

void plan_dens(Workspace& ws, int64_t n, DensPlan& p) {
    p.nblk = (int)ceil_div(n > 0 ? n : 1, kBlockItems);
    p.codes = ws.take<unsigned char>((size_t)(n > 0 ? n : 1));
    p.blk_counts = ws.take<unsigned long long>((size_t)p.nblk);
    p.blk_off = ws.take<long long>((size_t)p.nblk * 3);
}

}  // namespace
}  // namespace uws

using namespace uws;

extern "C" int uws_densify_workspace_size(int64_t n, size_t* bytes) {
    UWS_REQUIRE(bytes && n >= 0, "uws_densify_workspace_size: bad argument");
    UWS_REQUIRE(n < (1ll << 21) * 2048ll, "uws_densify_workspace_size: n out of range");
    Workspace ws(nullptr, 0, true);
    DensPlan p;
    plan_dens(ws, n, p);
    *bytes = ws.used;
    return UWS_OK;
}

extern "C" int uws_densify_classify(const float* params, int64_t n, const float* grad_accum,
                                    const int32_t* obs_count, double grad_threshold,
                                    double size_threshold, double min_opacity, int64_t* totals,
                                    void* workspace, size_t workspace_bytes, void* stream) {
    UWS_REQUIRE(totals && n >= 0, "uws_densify_classify: bad argument");
    UWS_REQUIRE(n == 0 || (params && grad_accum && obs_count), "uws_densify_classify: null buffer");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        UWS_CUDA(zero_async(totals, 3 * sizeof(int64_t), st));
        return UWS_OK;
    }
    Workspace ws(workspace, workspace_bytes);
    DensPlan p;
    plan_dens(ws, n, p);
    UWS_REQUIRE(ws.ok(), "uws_densify_classify: workspace too small");
    launch(k_dens_classify, dim3(p.nblk), dim3(kThreads), 0, st, params, n, grad_accum, obs_count, grad_threshold,
                                                 size_threshold, min_opacity, p.codes,
                                                 p.blk_counts);
    UWS_CHECK_LAUNCH("k_dens_classify");
    launch(k_dens_scan, dim3(1), dim3(1024), 0, st, p.blk_counts, p.nblk, p.blk_off, (long long*)totals);
    UWS_CHECK_LAUNCH("k_dens_scan");
    return UWS_OK;
}

extern "C" int uws_densify_apply(const float* params, const float* exp_avg,
                                 const float* exp_avg_sq, int64_t n, const void* workspace,
                                 size_t workspace_bytes, const double* samples,
                                 double log_split_factor, int64_t n_keep, int64_t n_clone,
                                 int64_t n_split, float* new_params, float* new_exp_avg,
                                 float* new_exp_avg_sq, void* stream) {
    UWS_REQUIRE(n > 0 && params && exp_avg && exp_avg_sq && workspace,
                "uws_densify_apply: bad argument");
    UWS_REQUIRE(n_keep >= 0 && n_clone >= 0 && n_split >= 0 && n_keep + n_split <= n &&
                    n_clone <= n_keep,
                "uws_densify_apply: inconsistent counts");
    UWS_REQUIRE(n_split == 0 || samples, "uws_densify_apply: split samples missing");
    UWS_REQUIRE(new_params && new_exp_avg && new_exp_avg_sq, "uws_densify_apply: null output");
    Workspace ws(const_cast<void*>(workspace), workspace_bytes);
    DensPlan p;
    plan_dens(ws, n, p);
    UWS_REQUIRE(ws.ok(), "uws_densify_apply: workspace too small");
    launch(k_dens_apply, dim3(p.nblk), dim3(kThreads), 0, as_stream(stream), 
        params, exp_avg, exp_avg_sq, n, p.codes, p.blk_off, samples, log_split_factor, n_keep,
        n_clone, n_split, new_params, new_exp_avg, new_exp_avg_sq);
    UWS_CHECK_LAUNCH("k_dens_apply");
    return UWS_OK;
}

extern "C" int uws_reset_opacities(float* params, float* exp_avg, float* exp_avg_sq, int64_t n,
                                   float value, void* stream) {
    UWS_REQUIRE(n >= 0 && (n == 0 || (params && exp_avg && exp_avg_sq)),
                "uws_reset_opacities: bad argument");
    if (n == 0) return UWS_OK;
    launch(k_reset_opacity, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, as_stream(stream), params, exp_avg,
                                                                               exp_avg_sq, n, value);
    UWS_CHECK_LAUNCH("k_reset_opacity");
    return UWS_OK;
}
