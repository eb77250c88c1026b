// Guidance refresh: the dark-pixel backscatter estimate on the device
// (reference backscatter.py:52-270; called every refit_period iterations by
// pipeline.py:204-208 on the current view's ground truth and remapped depth).
//
//   k_bs_resize    one thread per output pixel: bilinear colour / nearest depth
//                  with half-pixel centres (backscatter.py:52-79), the >= 0
//                  clamps, the RGB sum as the selection key, depth min/max
//   k_bs_label     depth clusters: searchsorted over numpy's linspace edges
//                  (backscatter.py:82-97), cluster sizes
//   radix sorts    stable (sum, pixel) then stable by cluster: cluster-major,
//                  darkest first, raster order on ties (backscatter.py:124-126)
//   k_bs_pick      the ceil(p_dark * size) first of every cluster
//   k_bs_compact   the dark set in raster order (backscatter.py:128-131)
//   k_bs_fit       one CTA: depth intervals, per interval and channel the first
//                  minimum (backscatter.py:251-264), then per channel one warp
//                  per Levenberg-Marquardt start (backscatter.py:142-208)
//
// Compiled with -fmad=false: every float64 expression is evaluated in numpy's
// operation order, so the dark set is bit-identical to the reference's given
// the same inputs.  The fit's sums are warp reductions (numpy hands them to
// BLAS in an unspecified order), so fitted values agree to the solver tolerance.
#include "common.cuh"
#include "radix.cuh"
#include "scan.cuh"

namespace uws {
namespace bsc {

constexpr int kThreads = 256;
constexpr int kMaxEdges = 257;      // edges_num, intervals_num limit (8-bit cluster key)
constexpr int kFitThreads = 1024;   // 32 warps: 3 channels x 10 starts
constexpr int kStarts = 10;
constexpr int kLmIters = 200;       // backscatter.py:30
constexpr double kLmTol = 1e-10;    // backscatter.py:31
constexpr double kBinfHi = 1.0;     // backscatter.py:21
constexpr double kBbHi = 5.0;       // backscatter.py:22
__constant__ double kBbStarts[5] = {0.1, 0.5, 1.0, 2.0, 4.0};  // backscatter.py:29

struct Hdr {
    unsigned long long zmin, zmax;  // canonical bits of the clamped resized depth
    uint32_t degenerate, error, n_dark, pad;
    uint32_t counts[kMaxEdges];
};

// numpy.maximum(x, 0.0) / numpy.clip: NaN propagates, ties keep x
__device__ __forceinline__ double np_max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
    double a = (x >= lo || x != x) ? x : lo;
    return (a <= hi || a != a) ? a : hi;
}
// order-preserving bits of a non-negative double (-0.0 -> +0.0)
__device__ __forceinline__ unsigned long long okey(double x) {
    return (unsigned long long)__double_as_longlong(x == 0.0 ? 0.0 : x);
}
__device__ __forceinline__ double from_key(unsigned long long k) {
    return __longlong_as_double((long long)k);
}

// numpy.linspace(lo, hi, num)[i] (numpy/_core/function_base.py): i*step + lo,
// step = (hi-lo)/(num-1); (i/div)*delta + lo when step underflows to 0; last = hi
__device__ __forceinline__ double linspace_at(double lo, double hi, int num, int i) {
    if (i == num - 1) return hi;
    const double delta = hi - lo;
    const double div = (double)(num - 1);
    const double step = delta / div;
    const double y = step == 0.0 ? ((double)i / div) * delta : (double)i * step;
    return y + lo;
}

// numpy pairwise summation of a contiguous float64 vector (loops_utils.h):
// blocks of <= 128 with 8 accumulators, longer vectors split at n/2 rounded
// down to a multiple of 8.  Written out for n <= 256 (no recursion).
__device__ double np_sum_block(const double* a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += a[i];
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
}

__device__ double np_sum(const double* a, int n) {  // n <= 256
    if (n <= 128) return np_sum_block(a, n);
    int n2 = n / 2;
    n2 -= n2 % 8;  // <= 128
    const int r = n - n2;  // <= 136
    double right;
    if (r <= 128) {
        right = np_sum_block(a + n2, r);
    } else {
        int r2 = r / 2;
        r2 -= r2 % 8;
        right = np_sum_block(a + n2, r2) + np_sum_block(a + n2 + r2, r - r2);
    }
    return np_sum_block(a, n2) + right;
}

__global__ void k_bs_init(Hdr* hdr) {
    pdl_entry();
    for (int i = threadIdx.x; i < kMaxEdges; i += blockDim.x) hdr->counts[i] = 0;
    if (threadIdx.x == 0) {
        hdr->zmin = ~0ull;
        hdr->zmax = 0ull;
        hdr->degenerate = hdr->error = hdr->n_dark = 0;
    }
}

template <bool RAW>
__global__ void __launch_bounds__(kThreads) k_bs_resize(const float* __restrict__ img,
                                                        const void* __restrict__ depth, int h, int w,
                                                        int th, int tw, double* __restrict__ rgb,
                                                        double* __restrict__ zout,
                                                        uint64_t* __restrict__ key, Hdr* hdr) {
    pdl_entry();
    const uint32_t P = (uint32_t)th * (uint32_t)tw;
    const uint32_t p = blockIdx.x * kThreads + threadIdx.x;
    unsigned long long zk_min = ~0ull, zk_max = 0ull;
    if (p < P) {
        const int i = (int)(p / (uint32_t)tw), j = (int)(p % (uint32_t)tw);
        double c[3];
        int di = i, dj = j;
        if (th == h) {  // no resize (backscatter.py:244-245)
            const float* s = img + ((size_t)i * w + j) * 3;
            c[0] = s[0];
            c[1] = s[1];
            c[2] = s[2];
        } else {
            // resize_nearest: min((k + 0.5) * h / th, h - 1) truncated (backscatter.py:52-57)
            di = (int)fmin(((double)i + 0.5) * (double)h / (double)th, (double)(h - 1));
            dj = (int)fmin(((double)j + 0.5) * (double)w / (double)tw, (double)(w - 1));
            // resize_bilinear (backscatter.py:60-79)
            const double ys = np_clip(((double)i + 0.5) * (double)h / (double)th - 0.5, 0.0, (double)(h - 1));
            const double xs = np_clip(((double)j + 0.5) * (double)w / (double)tw - 0.5, 0.0, (double)(w - 1));
            const int y0 = (int)floor(ys), x0 = (int)floor(xs);
            const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
            const double fy = ys - (double)y0, fx = xs - (double)x0;
            const float* r0 = img + (size_t)y0 * w * 3;
            const float* r1 = img + (size_t)y1 * w * 3;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double top = (double)r0[x0 * 3 + k] * (1.0 - fx) + (double)r0[x1 * 3 + k] * fx;
                const double bot = (double)r1[x0 * 3 + k] * (1.0 - fx) + (double)r1[x1 * 3 + k] * fx;
                c[k] = top * (1.0 - fy) + bot * fy;
            }
        }
        double z;
        const size_t dsrc = (size_t)di * w + dj;
        if (RAW) {  // logistic_remap (medium.py:26-29) of the raw render depth
            const double d = (double)((const float*)depth)[dsrc];
            z = 2.0 / (1.0 + exp(-0.1 * d)) - 1.0;
        } else {
            z = ((const double*)depth)[dsrc];
        }
        z = np_max0(z);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c[k] = np_max0(c[k]);
            rgb[(size_t)p * 3 + k] = c[k];
        }
        zout[p] = z;
        key[p] = okey((c[0] + c[1]) + c[2]);  // image.reshape(-1, 3).sum(axis=1)
        zk_min = zk_max = okey(z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, zk_min, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, zk_max, o);
        zk_min = a < zk_min ? a : zk_min;
        zk_max = b > zk_max ? b : zk_max;
    }
    if ((threadIdx.x & 31) == 0 && zk_min != ~0ull) {
        atomicMin(&hdr->zmin, zk_min);
        atomicMax(&hdr->zmax, zk_max);
    }
}

// cluster_range over linspace(min, max, ne) (backscatter.py:82-97, 115-117)
__global__ void __launch_bounds__(kThreads) k_bs_label(const double* __restrict__ z, uint32_t P,
                                                       int ne, Hdr* hdr, uint32_t* __restrict__ lab) {
    pdl_entry();
    __shared__ double edges[kMaxEdges];
    __shared__ uint32_t cnt[kMaxEdges];
    const double lo = from_key(hdr->zmin), hi = from_key(hdr->zmax);
    for (int i = threadIdx.x; i < kMaxEdges; i += kThreads) {
        edges[i] = i < ne ? linspace_at(lo, hi, ne, i) : 0.0;
        cnt[i] = 0;
    }
    __syncthreads();
    const bool degenerate = ne < 2 || !(edges[ne - 1] > edges[0]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        hdr->degenerate = degenerate;
        if (!degenerate)
            for (int i = 1; i < ne; ++i)
                if (!(edges[i] > edges[i - 1])) hdr->error = 1;
    }
    const uint32_t p = blockIdx.x * kThreads + threadIdx.x;
    if (p < P) {
        int l = 0;
        if (!degenerate) {
            // searchsorted(edges, z, side="right") - 1, clipped to [0, ne - 2]
            const double v = z[p];
            int a = 0, b = ne;  // first edge > v
            while (a < b) {
                const int m = (a + b) >> 1;
                if (edges[m] <= v) a = m + 1;
                else b = m;
            }
            l = min(max(a - 1, 0), ne - 2);
        }
        lab[p] = (uint32_t)l;
        atomicAdd(&cnt[l], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kMaxEdges; i += kThreads)
        if (cnt[i]) atomicAdd(&hdr->counts[i], cnt[i]);
}

__global__ void k_bs_gather(const uint32_t* __restrict__ lab, const uint32_t* __restrict__ idx,
                            uint32_t P, uint32_t* __restrict__ out) {
    pdl_entry();
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < P) out[q] = lab[idx[q]];
}

// the first ceil(p_dark * size) (at least 1) of every cluster in (cluster, sum, pixel) order
__global__ void __launch_bounds__(kThreads) k_bs_pick(const uint32_t* __restrict__ lab_sorted,
                                                      const uint32_t* __restrict__ idx, uint32_t P,
                                                      const Hdr* hdr, double p_dark,
                                                      uint32_t* __restrict__ pick) {
    pdl_entry();
    __shared__ uint32_t start[kMaxEdges], quota[kMaxEdges];
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int i = 0; i < kMaxEdges; ++i) {
            const uint32_t c = hdr->counts[i];
            start[i] = s;
            const double q = ceil(p_dark * (double)c);
            quota[i] = q < 1.0 ? 1u : (q >= (double)c ? c : (uint32_t)q);
            s += c;
        }
    }
    __syncthreads();
    const uint32_t q = blockIdx.x * kThreads + threadIdx.x;
    if (q < P) {
        const uint32_t l = lab_sorted[q];
        pick[idx[q]] = (q - start[l] < quota[l]) ? 1u : 0u;
    }
}

// the dark set in raster order (np.sort of the picked pixel indices)
__global__ void __launch_bounds__(1024) k_bs_compact(const uint32_t* __restrict__ pick,
                                                     const double* __restrict__ z,
                                                     const double* __restrict__ rgb, uint32_t P,
                                                     double* __restrict__ dz,
                                                     double* __restrict__ drgb,
                                                     double* __restrict__ dark_out, Hdr* hdr) {
    pdl_entry();
    __shared__ uint32_t tmp[1024 / 32 + 1];
    uint32_t base = 0;
    for (uint32_t c0 = 0; c0 < P; c0 += 1024) {
        const uint32_t p = c0 + threadIdx.x;
        const uint32_t f = p < P ? pick[p] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_sum<1024, uint32_t>(f, tmp, &tot);
        if (f) {
            const uint32_t o = base + ex;
            dz[o] = z[p];
            drgb[3 * o + 0] = rgb[3 * (size_t)p + 0];
            drgb[3 * o + 1] = rgb[3 * (size_t)p + 1];
            drgb[3 * o + 2] = rgb[3 * (size_t)p + 2];
            if (dark_out) {
                dark_out[4 * (size_t)o + 0] = z[p];
                dark_out[4 * (size_t)o + 1] = rgb[3 * (size_t)p + 0];
                dark_out[4 * (size_t)o + 2] = rgb[3 * (size_t)p + 1];
                dark_out[4 * (size_t)o + 3] = rgb[3 * (size_t)p + 2];
            }
        }
        base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) hdr->n_dark = base;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return __shfl_sync(0xffffffffu, v, 0);  // one value for every lane
}

__device__ __forceinline__ double sse_warp(double b_inf, double b_b, const double* z, const double* y,
                                           int m, int lane) {
    double s = 0.0;
    for (int j = lane; j < m; j += 32) {
        const double r = b_inf * (1.0 - exp(-b_b * z[j])) - y[j];
        s += r * r;
    }
    return warp_sum(s);
}

// np.linalg.solve of the damped 2x2 system (LAPACK gesv: partial pivoting,
// the pivot column scaled by the reciprocal); false where the reference's
// solve raises LinAlgError (an exactly zero pivot)
__device__ __forceinline__ bool solve2(double a00, double a01, double a10, double a11, double b0,
                                       double b1, double* x0, double* x1) {
    if (fabs(a10) > fabs(a00)) {
        double t = a00; a00 = a10; a10 = t;
        t = a01; a01 = a11; a11 = t;
        t = b0; b0 = b1; b1 = t;
    }
    if (a00 == 0.0) return false;
    const double l = a10 * (1.0 / a00);
    const double u11 = a11 - l * a01;
    if (u11 == 0.0) return false;
    const double y1 = b1 - l * b0;
    *x1 = y1 / u11;
    *x0 = (b0 - a01 * *x1) / a00;
    return true;
}

// _lm_fit (backscatter.py:142-175), one warp, all lanes in lock step
__device__ void lm_warp(const double* z, const double* y, int m, double s0, double s1, int lane,
                        double* out_p0, double* out_p1, double* out_sse) {
    double p0 = np_clip(s0, 0.0, kBinfHi), p1 = np_clip(s1, 0.0, kBbHi);
    double sse = sse_warp(p0, p1, z, y, m, lane);
    double lam = 1e-3;
    for (int it = 0; it < kLmIters; ++it) {
        double haa = 0.0, hab = 0.0, hbb = 0.0, ga = 0.0, gb = 0.0;
        for (int j = lane; j < m; j += 32) {
            const double e = exp(-p1 * z[j]);
            const double a = 1.0 - e;
            const double b = p0 * z[j] * e;
            const double r = p0 * (1.0 - e) - y[j];
            haa += a * a;
            hab += a * b;
            hbb += b * b;
            ga += a * r;
            gb += b * r;
        }
        haa = warp_sum(haa);
        hab = warp_sum(hab);
        hbb = warp_sum(hbb);
        ga = warp_sum(ga);
        gb = warp_sum(gb);
        bool accepted = false, done = false;
        for (int t = 0; t < 12; ++t) {
            const double d0 = (haa >= 1e-12 || haa != haa) ? haa : 1e-12;
            const double d1 = (hbb >= 1e-12 || hbb != hbb) ? hbb : 1e-12;
            double x0, x1;
            if (!solve2(haa + lam * d0, hab + lam * 0.0, hab + lam * 0.0, hbb + lam * d1, -ga, -gb,
                        &x0, &x1)) {
                lam *= 10.0;
                continue;
            }
            const double c0 = np_clip(p0 + x0, 0.0, kBinfHi), c1 = np_clip(p1 + x1, 0.0, kBbHi);
            const double cs = sse_warp(c0, c1, z, y, m, lane);
            if (cs <= sse) {
                const double dx = c0 - p0, dy = c1 - p1;
                const double moved = sqrt(dx * dx + dy * dy);
                p0 = c0;
                p1 = c1;
                sse = cs;
                lam = fmax(lam / 3.0, 1e-12);
                accepted = true;
                done = moved < kLmTol;
                break;
            }
            lam *= 3.0;
        }
        if (!accepted || done) break;
    }
    *out_p0 = p0;
    *out_p1 = p1;
    *out_sse = sse;
}

__global__ void __launch_bounds__(kFitThreads) k_bs_fit(const double* __restrict__ rgb, uint32_t P,
                                                        const double* __restrict__ dz,
                                                        const double* __restrict__ drgb,
                                                        const Hdr* hdr, int ni,
                                                        double* __restrict__ result,
                                                        float* __restrict__ guide) {
    pdl_entry();
    __shared__ double edges[kMaxEdges];
    __shared__ unsigned long long best_v[kMaxEdges][3];
    __shared__ uint32_t best_j[kMaxEdges][3];
    __shared__ double pz[3][kMaxEdges], py[3][kMaxEdges], r2[3][kMaxEdges];
    __shared__ int pm[3], state[3];
    __shared__ double starts[3][2];
    __shared__ double fit_p0[kStarts * 3], fit_p1[kStarts * 3], fit_sse[kStarts * 3];
    __shared__ unsigned long long red_min[32], red_max[32];
    __shared__ int deg2_s, err_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nd = hdr->n_dark;
    if (hdr->error) {
        if (tid == 0) {
            result[9] = 1.0;
            result[10] = (double)nd;
            result[11] = 1.0;
        }
        return;
    }
    if (nd == 0 || hdr->degenerate) {
        // mean colour of the resized image (numpy's axis-0 reduction: sequential)
        if (tid < 3) {
            double s = 0.0;
            for (uint32_t p = 0; p < P; ++p) s += rgb[3 * (size_t)p + tid];
            result[tid] = np_clip(s / (double)P, 0.0, kBinfHi);
            result[3 + tid] = kBbHi;
            result[6 + tid] = 0.0;
        }
        if (tid == 0) {
            result[9] = 1.0;
            result[10] = (double)nd;
            result[11] = 0.0;
        }
        return;
    }
    // depth intervals over the dark set (backscatter.py:256-257)
    unsigned long long kmin = ~0ull, kmax = 0ull;
    for (uint32_t j = tid; j < nd; j += kFitThreads) {
        const unsigned long long k = okey(dz[j]);
        kmin = k < kmin ? k : kmin;
        kmax = k > kmax ? k : kmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    if (lane == 0) {
        red_min[warp] = kmin;
        red_max[warp] = kmax;
    }
    for (int i = tid; i < kMaxEdges * 3; i += kFitThreads) {
        (&best_v[0][0])[i] = ~0ull;
        (&best_j[0][0])[i] = 0xffffffffu;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < 32; ++w) {
            red_min[0] = red_min[w] < red_min[0] ? red_min[w] : red_min[0];
            red_max[0] = red_max[w] > red_max[0] ? red_max[w] : red_max[0];
        }
    }
    __syncthreads();
    const double lo = from_key(red_min[0]), hi = from_key(red_max[0]);
    for (int i = tid; i < kMaxEdges; i += kFitThreads) edges[i] = i < ni ? linspace_at(lo, hi, ni, i) : 0.0;
    __syncthreads();
    if (tid == 0) {
        const int deg2 = ni < 2 || !(edges[ni - 1] > edges[0]);
        int err = 0;
        if (!deg2)
            for (int i = 1; i < ni; ++i)
                if (!(edges[i] > edges[i - 1])) err = 1;
        deg2_s = deg2;
        err_s = err;
    }
    __syncthreads();
    const int deg2 = deg2_s;
    if (err_s) {
        if (tid == 0) {
            result[9] = 1.0;
            result[10] = (double)nd;
            result[11] = 1.0;
        }
        return;
    }
    // per (interval, channel): the first minimum (np.argmin over the members)
    for (int pass = 0; pass < 2; ++pass) {
        for (uint32_t j = tid; j < nd; j += kFitThreads) {
            int l = 0;
            if (!deg2) {
                const double v = dz[j];
                int a = 0, b = ni;
                while (a < b) {
                    const int m = (a + b) >> 1;
                    if (edges[m] <= v) a = m + 1;
                    else b = m;
                }
                l = min(max(a - 1, 0), ni - 2);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const unsigned long long key = okey(drgb[3 * (size_t)j + k]);
                if (pass == 0) atomicMin(&best_v[l][k], key);
                else if (key == best_v[l][k]) atomicMin(&best_j[l][k], j);
            }
        }
        __syncthreads();
    }
    // fit points in interval order; degenerate / trivial channels settled here
    if (tid < 3) {
        const int k = tid;
        const int nint = deg2 ? 1 : ni - 1;
        int m = 0;
        for (int i = 0; i < nint; ++i) {
            const uint32_t j = best_j[i][k];
            if (j == 0xffffffffu) continue;
            pz[k][m] = dz[j];
            py[k][m] = drgb[3 * (size_t)j + k];
            ++m;
        }
        pm[k] = m;
        bool distinct = false;
        for (int i = 1; i < m; ++i) distinct |= pz[k][i] != pz[k][0];
        double ymax = -INFINITY, amax = 0.0;
        for (int i = 0; i < m; ++i) {
            ymax = fmax(ymax, py[k][i]);
            amax = fmax(amax, fabs(py[k][i]));
        }
        if (m < 3 || !distinct) {  // fit_saturating_exponential's degenerate branch
            const double b_inf = np_clip(m ? np_sum(py[k], m) / (double)m : 0.0, 0.0, kBinfHi);
            for (int i = 0; i < m; ++i) {
                const double r = b_inf * (1.0 - exp(-kBbHi * pz[k][i])) - py[k][i];
                r2[k][i] = r * r;
            }
            result[k] = b_inf;
            result[3 + k] = kBbHi;
            result[6 + k] = m ? sqrt(np_sum(r2[k], m) / (double)m) : 0.0;
            state[k] = 1;  // settled, degenerate
        } else if (amax == 0.0) {
            result[k] = 0.0;
            result[3 + k] = 0.0;
            result[6 + k] = 0.0;
            state[k] = 2;  // settled
        } else {
            starts[k][0] = np_sum(py[k], m) / (double)m;
            starts[k][1] = ymax;
            state[k] = 0;
        }
    }
    __syncthreads();
    if (warp < 3 * kStarts) {
        const int k = warp / kStarts, s = warp % kStarts;
        if (state[k] == 0)
            lm_warp(pz[k], py[k], pm[k], starts[k][s / 5], kBbStarts[s % 5], lane, &fit_p0[warp],
                    &fit_p1[warp], &fit_sse[warp]);
    }
    __syncthreads();
    if (tid < 3 && state[tid] == 0) {
        const int k = tid;
        double bp0 = 0.0, bp1 = 0.0, bs = INFINITY;
        for (int s = 0; s < kStarts; ++s) {
            const double e = fit_sse[k * kStarts + s];
            if (e < bs - 1e-15) {
                bs = e;
                bp0 = fit_p0[k * kStarts + s];
                bp1 = fit_p1[k * kStarts + s];
            }
        }
        result[k] = bp0;
        result[3 + k] = bp1;
        result[6 + k] = sqrt(bs / (double)pm[k]);
    }
    __syncthreads();
    if (tid == 0) {
        const bool degenerate = deg2 || state[0] == 1 || state[1] == 1 || state[2] == 1;
        result[9] = degenerate ? 1.0 : 0.0;
        result[10] = (double)nd;
        result[11] = 0.0;
        if (!degenerate && guide) {  // pipeline.py:206-208, astype(float32)
            for (int k = 0; k < 3; ++k) {
                guide[k] = __double2float_rn(result[k]);
                guide[3 + k] = __double2float_rn(result[3 + k]);
            }
        }
    }
}

struct Plan {
    int th, tw;
    uint32_t P;
    Hdr* hdr;
    double *rgb, *z, *dz, *drgb;
    uint64_t *key, *key_sorted;
    uint32_t *idx_sorted, *lab, *lab_g, *lab_sorted, *idx_final, *pick;
    // radix temporaries (64-bit sums: 8 passes; cluster labels: 1 pass)
    radix::Plan<uint64_t> r64;
    radix::Plan<uint32_t> r32;
};

inline void dims(int h, int w, int rh, int* th, int* tw) {
    *th = rh < h ? rh : h;
    if (*th == h) {
        *tw = w;
    } else {  // max(1, round(w * th / h)): Python true division, round half to even
        const double t = nearbyint((double)((int64_t)w * *th) / (double)h);
        *tw = t < 1.0 ? 1 : (int)t;
    }
}

inline void plan(Workspace& ws, int h, int w, int rh, Plan& p) {
    dims(h, w, rh, &p.th, &p.tw);
    p.P = (uint32_t)p.th * (uint32_t)p.tw;
    const uint32_t n = p.P > 0 ? p.P : 1;
    p.hdr = ws.take<Hdr>(1);
    p.rgb = ws.take<double>((size_t)n * 3);
    p.z = ws.take<double>(n);
    p.dz = ws.take<double>(n);
    p.drgb = ws.take<double>((size_t)n * 3);
    p.key = ws.take<uint64_t>(n);
    p.key_sorted = ws.take<uint64_t>(n);
    p.idx_sorted = ws.take<uint32_t>(n);
    p.lab = ws.take<uint32_t>(n);
    p.lab_g = ws.take<uint32_t>(n);
    p.lab_sorted = ws.take<uint32_t>(n);
    p.idx_final = ws.take<uint32_t>(n);
    p.pick = ws.take<uint32_t>(n);
    radix::plan<uint64_t>(ws, n, 8, p.r64);
    radix::plan<uint32_t>(ws, n, 1, p.r32);
}

}  // namespace bsc
}  // namespace uws

using namespace uws;

static int check_cfg(const uws_backscatter_cfg* cfg, const char* who) {
    (void)who;
    UWS_REQUIRE(cfg, "backscatter: null config");
    UWS_REQUIRE(cfg->resized_height >= 1, "backscatter: resized_height must be >= 1");
    UWS_REQUIRE(cfg->edges_num >= 0 && cfg->edges_num <= bsc::kMaxEdges,
                "backscatter: edges_num must be in [0, 257]");
    UWS_REQUIRE(cfg->intervals_num >= 0 && cfg->intervals_num <= bsc::kMaxEdges,
                "backscatter: intervals_num must be in [0, 257]");
    UWS_REQUIRE(cfg->p_dark == cfg->p_dark, "backscatter: p_dark is NaN");
    return UWS_OK;
}

extern "C" int uws_backscatter_workspace_size(int32_t h, int32_t w, const uws_backscatter_cfg* cfg,
                                              size_t* bytes) {
    UWS_REQUIRE(bytes && h > 0 && w > 0, "uws_backscatter_workspace_size: bad argument");
    if (int rc = check_cfg(cfg, "uws_backscatter_workspace_size")) return rc;
    UWS_REQUIRE((int64_t)h * w < (1ll << 31), "uws_backscatter_workspace_size: image too large");
    Workspace ws(nullptr, 0, true);
    bsc::Plan p;
    bsc::plan(ws, h, w, cfg->resized_height, p);
    *bytes = ws.used;
    return UWS_OK;
}

extern "C" int uws_estimate_backscatter(const float* image, const void* depth, int32_t depth_is_raw,
                                        int32_t h, int32_t w, const uws_backscatter_cfg* cfg,
                                        double* result, float* medium_guide, double* dark,
                                        void* workspace, size_t workspace_bytes, void* stream) {
    UWS_REQUIRE(image && depth && result && workspace && h > 0 && w > 0,
                "uws_estimate_backscatter: bad argument");
    if (int rc = check_cfg(cfg, "uws_estimate_backscatter")) return rc;
    using namespace bsc;
    cudaStream_t st = as_stream(stream);
    Workspace ws(workspace, workspace_bytes);
    Plan p;
    plan(ws, h, w, cfg->resized_height, p);
    UWS_REQUIRE(ws.ok(), "uws_estimate_backscatter: workspace too small");
    const uint32_t P = p.P;
    const int blocks = (int)ceil_div(P, kThreads);
    launch(k_bs_init, dim3(1), dim3(kThreads), 0, st, p.hdr);
    UWS_CHECK_LAUNCH("k_bs_init");
    if (depth_is_raw)
        launch(k_bs_resize<true>, dim3(blocks), dim3(kThreads), 0, st, image, depth, h, w, p.th, p.tw, p.rgb, p.z,
                                                       p.key, p.hdr);
    else
        launch(k_bs_resize<false>, dim3(blocks), dim3(kThreads), 0, st, image, depth, h, w, p.th, p.tw, p.rgb, p.z,
                                                        p.key, p.hdr);
    UWS_CHECK_LAUNCH("k_bs_resize");
    launch(k_bs_label, dim3(blocks), dim3(kThreads), 0, st, p.z, P, cfg->edges_num, p.hdr, p.lab);
    UWS_CHECK_LAUNCH("k_bs_label");
    // stable by RGB sum (pixel order on ties), then stable by cluster
    UWS_CUDA(radix::sort_pairs<uint64_t>(p.r64, p.key, nullptr, p.key_sorted, p.idx_sorted, P,
                                         nullptr, 0, st));
    launch(k_bs_gather, dim3(blocks), dim3(kThreads), 0, st, p.lab, p.idx_sorted, P, p.lab_g);
    UWS_CHECK_LAUNCH("k_bs_gather");
    UWS_CUDA(radix::sort_pairs<uint32_t>(p.r32, p.lab_g, p.idx_sorted, p.lab_sorted, p.idx_final, P,
                                         nullptr, 0, st));
    launch(k_bs_pick, dim3(blocks), dim3(kThreads), 0, st, p.lab_sorted, p.idx_final, P, p.hdr, cfg->p_dark, p.pick);
    UWS_CHECK_LAUNCH("k_bs_pick");
    launch(k_bs_compact, dim3(1), dim3(1024), 0, st, p.pick, p.z, p.rgb, P, p.dz, p.drgb, dark, p.hdr);
    UWS_CHECK_LAUNCH("k_bs_compact");
    launch(k_bs_fit, dim3(1), dim3(kFitThreads), 0, st, p.rgb, P, p.dz, p.drgb, p.hdr, cfg->intervals_num, result,
                                        medium_guide);
    UWS_CHECK_LAUNCH("k_bs_fit");
    return UWS_OK;
}
