// K8 backward compositing + medium-parameter gradients.
//
// Replaces backward._backward_block (backward.py:124-163), the per-tile loop
// and fixed-order merge of backward_render (:278-344), and backward_medium
// (:261-275).
//
// One CTA per tile, kPix vertically strided pixels per thread, walking the
// tile list BACK to front over exactly the prefix the forward consumed
// (per-pixel `last`).  Transmittance is recovered as T_i = T_{i+1}/(1-alpha_i)
// from the stored final transmittance, and the suffix sum_{j>i} w_j (G . c_j)
// of the reference's reverse cumsum (:149) is carried as one scalar per
// pixel, so no per-pair state is stored.  Alpha and its gates are recomputed
// with the forward's exact arithmetic, hence identical decisions.
//
// The 9 per-(pixel, Gaussian) partials (dpower, dpower*dx, dpower*dy,
// dpower*dx^2, dpower*dx*dy, dpower*dy^2, w*G) are first summed over the
// thread's kPix pixels, then across the warp with a transposed butterfly
// (12 shuffles instead of 45), accumulated over the CTA's warps in shared
// memory, chained through the conic once per (tile, Gaussian) and only then
// sent to HBM with 9 atomics.
#include "radix.cuh"
#include "raster_common.cuh"
#include "row_filter.cuh"

namespace uws {
namespace {

#ifndef UWS_BWD_MINB
#define UWS_BWD_MINB 12
#endif
constexpr int kBatch = 128;
constexpr float kLn2 = 0.69314718055994531f;
constexpr int kPix = 4;                          // pixels per thread
constexpr int kThreads = kRasterThreads / kPix;  // 64
constexpr int kWarps = kThreads / 32;            // 2
constexpr int kBandRows = kTile / kWarps;        // each warp owns an 8-row band of the tile
static_assert(kWarps == 2, "one x-range per warp band in Rec::D");
// the clamp guard band as |araw - mid| < half (a slightly wider superset of [kClampLo, kClampHi))
constexpr float kClampMid = 0.5f * (kClampLo + kClampHi);
constexpr float kClampHalf = 0.51f * (kClampHi - kClampLo);

struct BwdArgs {
    const uws_splat* splat;
    const double* exact;
    const int32_t* offsets;      // tile lists (full binning) ...
    const int32_t* entries;
    const int32_t* row_start;    // ... or tile-row lists filtered on the fly
    const uint2* row_items;
    const int32_t* tile_rows;    // the forward's staged rows per tile (optional)
    const int32_t* tile_nrows;
    int tile_rows_cap;
    const int32_t* order;        // CTA b handles tile order[b] (NULL: raster order)
    int width, height, gx;
    const float* medium;
    const float* color_clean;
    const float* depth;
    const float* final_T;
    const int32_t* last;
    const float* dL;
    float* screen;       // [K][9]
    double* medium_acc;  // [9]
    // deterministic mode (DET): the (tile, Gaussian) partials go to slot
    // tile_base[tile] + list position instead of atomics on screen / medium_acc
    const int32_t* tile_base;  // [tiles + 1] exclusive prefix of the consumed prefixes
    float* part;               // [R][9]
    uint32_t* part_row;        // [R] visible row, or none_row when no pixel used it
    uint32_t none_row;
    double* med_part;          // [tiles][9]
};

// Reduce v[0..8] across the warp.  v[0..7] by a transposed butterfly (each stage
// sends half of the values still held, so stages 16/8/4 cost 4+2+1 shuffles),
// v[8] by plain stages 16/8/4, and the last two stages exchange (r, v8-partial)
// transposed: 12 shuffles.  Lanes with (lane & 3) == 0 return the full sum of
// value ((lane>>4)&1)*4 + ((lane>>3)&1)*2 + ((lane>>2)&1); lanes with
// (lane & 3) == 2 the full sum of v[8].
__device__ __forceinline__ float butterfly9(const float v[9], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    float h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float send = b4 ? v[i] : v[i + 4];
        float keep = b4 ? v[i + 4] : v[i];
        h[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float e = v[8] + __shfl_xor_sync(0xffffffffu, v[8], 16);
    float q[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        float send = b3 ? h[i] : h[i + 2];
        float keep = b3 ? h[i + 2] : h[i];
        q[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    e += __shfl_xor_sync(0xffffffffu, e, 8);
    float send = b2 ? q[0] : q[1];
    float r = (b2 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    e += __shfl_xor_sync(0xffffffffu, e, 4);
    send = b1 ? r : e;
    float x = (b1 ? e : r) + __shfl_xor_sync(0xffffffffu, send, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_u8(uint32_t addr, unsigned v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// The float64 records for the guard-band re-decisions, read by the out-of-line
// re-decision from shared memory: the hot loop then passes no pointers to the call
// (passing them made the compiler reload four kernel-parameter words per entry).
__shared__ const uws_splat* s_bwd_splat;
__shared__ const double* s_bwd_exact;
static __device__ __noinline__ double alpha_raw_f64_bwd(int row, int px, int py) {
    return alpha_raw_f64(s_bwd_splat, s_bwd_exact, row, px, py);
}

constexpr int kMaxMarks = 64;   // recorded batch starts per tile (row-list source)

#ifdef UWS_BWD_STATS
// debug build: [0..32] (warp, entry) iterations by number of lanes with a pair,
// [33] pairs, [34] iterations culled by the band test
__device__ unsigned long long g_bwd_hist[35];
#endif

template <bool ROWS, int MINB, bool DET = false>
__global__ void __launch_bounds__(kThreads, MINB) k_raster_bwd(BwdArgs a) {
    // launched serially (no pdl_entry): the per-CTA L1 invalidation costs more here
    __shared__ int sMarkCur[ROWS ? kMaxMarks : 1], sMarkSkip[ROWS ? kMaxMarks : 1];
    __shared__ int sScan[kWarps];
    struct __align__(16) Rec {
        StageA A;
        StageB B;
        StageC C;
        float4 D;  // pre-filter: x-range of the pass region in band 0 and band 1
    };
    __shared__ Rec sRec[kBatch];  // one array: one base address for all four loads
    __shared__ float sAcc[kWarps][9][kBatch + 1];  // per-warp partials; +1: the 8 storing lanes hit distinct banks
    // the batch's rows (filled and consumed by the staging phase) share sAcc's storage: sAcc is
    // written only by the walk that follows and read back before the next batch is staged
    int* const sRow = reinterpret_cast<int*>(&sAcc[0][0][0]);  // (filter writes positions < nb <= kBatch)
    static_assert(kWarps * 9 * (kBatch + 1) >= kBatch, "sRow alias");
    __shared__ unsigned char sHit[kWarps][kBatch];  // sAcc[w][.][k] valid
    __shared__ float sMed[kWarps][9];
    __shared__ int sMaxLast;

    const int tile = a.order ? __ldg(a.order + blockIdx.x) : (int)blockIdx.x;
    const int ty = tile / a.gx, tx = tile - ty * a.gx;
    const int ox = tx * kTile, oy = ty * kTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & (kTile - 1);
    const int ly0 = warp * kBandRows + (lane >> 4);  // pixel p sits on row ly0 + 2p
    const float fx = (float)lx + 0.5f;
    const int start = ROWS ? 0 : a.offsets[tile];

    if (threadIdx.x == 0) {
        sMaxLast = 0;
        s_bwd_splat = a.splat;
        s_bwd_exact = a.exact;
    }
    for (int i = threadIdx.x; i < kWarps * kBatch; i += kThreads) (&sHit[0][0])[i] = 0;

    float G[kPix][3], T[kPix], S[kPix], fy[kPix];
    int mylast[kPix];
    float med[9];
#pragma unroll
    for (int v = 0; v < 9; ++v) med[v] = 0.f;
    int maxl = 0, minl = 0x7fffffff;  // longest / shortest consumed prefix of the thread's pixels
#pragma unroll
    for (int p = 0; p < kPix; ++p) {
        const int ly = ly0 + 2 * p;
        fy[p] = (float)ly + 0.5f;
        asm("" : "+f"(fy[p]));  // keep it in a register (not rematerialised from tid)
        S[p] = 0.f;
        T[p] = 1.f;
        mylast[p] = 0;
        G[p][0] = G[p][1] = G[p][2] = 0.f;
        const int px = ox + lx, py = oy + ly;
        if (!(px < a.width && py < a.height)) minl = 0;
        if (px < a.width && py < a.height) {
            const int pix = py * a.width + px;
            T[p] = a.final_T[pix];
            mylast[p] = a.last[pix];
            maxl = max(maxl, mylast[p]);
            minl = min(minl, mylast[p]);
            if (a.medium) {
                const float d = a.depth[pix];
                const float z = 2.0f / (1.0f + __expf(-(float)kLogisticRate * d)) - 1.0f;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const float dl = a.dL[3 * pix + ch];
                    const float att = __expf(-a.medium[ch] * z);
                    const float ebs = __expf(-a.medium[6 + ch] * z);
                    G[p][ch] = dl * att;
                    med[ch] += dl * a.color_clean[3 * pix + ch] * (-z) * att;   // d attenuation
                    med[3 + ch] += dl * (1.0f - ebs);                            // d water_color
                    med[6 + ch] += dl * a.medium[3 + ch] * z * ebs;              // d backscatter
                }
            } else {
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) G[p][ch] = a.dL[3 * pix + ch];
            }
        }
    }
    if (a.medium) {
#pragma unroll
        for (int v = 0; v < 9; ++v) {
            float s = warp_sum(med[v]);
            if (lane == 0) sMed[warp][v] = s;
        }
    }
    const int wmax = __reduce_max_sync(0xffffffffu, maxl);  // this warp's consumed prefix
    __syncthreads();
    if (lane == 0 && wmax > 0) atomicMax(&sMaxLast, wmax);
    if (a.medium && threadIdx.x < 9) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += sMed[w][threadIdx.x];
        if (DET)
            a.med_part[(size_t)tile * 9 + threadIdx.x] = (double)s;
        else
            atomicAdd(&a.medium_acc[threadIdx.x], (double)s);
    }
    __syncthreads();
    const int maxlast = sMaxLast;

    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sRec);  // 64-byte records
    static_assert(sizeof(Rec) == 64, "record layout");
    const int nbatch = (maxlast + kBatch - 1) / kBatch;
    int rend = 0, stride = 1;
    // the forward stored this tile's consumed prefix: no filtering of the row lists
    const int32_t* saved = (ROWS && a.tile_rows && maxlast <= (a.tile_nrows[tile] & ~kRowsComplete))
                               ? a.tile_rows + (size_t)tile * a.tile_rows_cap
                               : nullptr;
    if (ROWS && nbatch > 0 && !saved) {
        // pass 1 over the row list: where does each batch of tile entries start?
        const int rs = a.row_start[ty];
        rend = a.row_start[ty + 1];
        stride = (nbatch + kMaxMarks - 1) / kMaxMarks;
        int cnt = 0, cur = rs, b = 0;
        if (nbatch == 1) {  // the common case: the whole prefix is one batch from the start
            if (threadIdx.x == 0) {
                sMarkCur[0] = rs;
                sMarkSkip[0] = 0;
            }
            cnt = maxlast;
        }
        while (cnt < maxlast && cur < rend) {
            const int t = filter_chunk<kThreads>(a.row_items, cur, rend, tx, nullptr, 0, 0,
                                                 sScan);
            while (b < nbatch && b * kBatch < cnt + t) {
                if (threadIdx.x == 0) {
                    sMarkCur[b / stride] = cur;
                    sMarkSkip[b / stride] = b * kBatch - cnt;
                }
                b += stride;
            }
            cnt += t;
            cur += kChunk;
        }
        __syncthreads();
    }

    // per-lane shared-memory store slot of the reduced partials: lanes with
    // (lane & 3) == 0 hold butterfly value idx, lane 2 the ninth value; lane 0 the hit flag
    const int accRow = (lane & 3) == 0
                           ? ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)
                           : 8;
    const bool accStore = (lane & 3) == 0 || lane == 2;
    // opaque (kept in registers, not rematerialised from the CTA's shared window per use)
    uint32_t accBase, hitBase;
    asm volatile("mov.u32 %0, %1;" : "=r"(accBase) : "r"((uint32_t)__cvta_generic_to_shared(&sAcc[warp][accRow][0])));
    asm volatile("mov.u32 %0, %1;" : "=r"(hitBase) : "r"((uint32_t)__cvta_generic_to_shared(&sHit[warp][0])));
    const uint32_t dOff = 48u + 8u * (uint32_t)warp;  // this warp's x-range in Rec::D
    for (int bi = nbatch - 1; bi >= 0; --bi) {
        const int lo = bi * kBatch;
        const int nb = min(kBatch, maxlast - lo);
        __syncthreads();
        if (ROWS && !saved) {
            // pass 2: re-collect this batch's rows from its recorded start
            const int mk = bi / stride;
            int cur = sMarkCur[mk];
            int got = -(sMarkSkip[mk] + (bi - mk * stride) * kBatch);
            while (got < nb) {
                got += filter_chunk<kThreads>(a.row_items, cur, rend, tx, sRow, got, nb,
                                              sScan);
                cur += kChunk;
            }
        }
#pragma unroll
        for (int s = 0; s < kBatch / kThreads; ++s) {
            const int i = threadIdx.x + s * kThreads;
            if (i < nb) {
                Rec& r = sRec[i];
                const int row =
                    ROWS ? (saved ? saved[lo + i] : sRow[i]) : a.entries[start + lo + i];
                stage_entry(a.splat, row, ox, oy, r.A, r.B, r.C);
                // exact x-ranges of the pass region within each warp's band rows
                PassRegion pr;
                pr.init(r.A, r.B);
                const float2 x0 = pr.xrange(0.5f, (float)kBandRows - 0.5f);
                const float2 x1 = pr.xrange((float)kBandRows + 0.5f, (float)kTile - 0.5f);
                r.D = make_float4(x0.x, x0.y, x1.x, x1.y);
            }
        }
        __syncthreads();
        // back to front over the entries this warp's pixels consumed
        // one induction variable (this warp's x-range address of entry k); k itself is
        // recovered opaquely (asm) on the non-culled path only, so the compiler keeps no
        // strength-reduced copies of the k-linear addresses alive across the loop
        uint32_t rbeg;
        asm volatile("mov.u32 %0, %1;" : "=r"(rbeg) : "r"(sbase + dOff));
        for (uint32_t rd = rbeg + 64u * (uint32_t)max(min(nb, wmax - lo), 0); rd != rbeg;) {
            rd -= 64u;
            float xlo, xhi;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(xlo), "=f"(xhi) : "r"(rd) : "memory");
            // the pass region misses this warp's band within the tile's columns (uniform)
            if (xhi < 0.5f || xlo > (float)kTile - 0.5f) {
#ifdef UWS_BWD_STATS
                if (lane == 0) atomicAdd(&g_bwd_hist[34], 1ull);
#endif
                continue;
            }
            int k;
            asm("{\n\t.reg .u32 t;\n\tsub.u32 t, %1, %2;\n\tshr.u32 %0, t, 6;\n\t}"
                : "=r"(k) : "r"(rd), "r"(rbeg));
            const uint32_t ra = rd - dOff;
            const int jrel = lo + k;
            // A thread's kPix pixels share one column, hence dx: the dx-weighted
            // partials are formed once after the pixel loop from sum(dp) and sum(dp dy).
            float sdp = 0.f, sdpy = 0.f, sdpyy = 0.f, wg0 = 0.f, wg1 = 0.f, wg2 = 0.f, dx = 0.f;
            bool hit = false;
#ifdef UWS_BWD_STATS
            bool paired = false;
#endif
            if (fx >= xlo && fx <= xhi) {  // column inside the band's range
                hit = true;  // (a lane whose column reaches the pass region; its partials may be 0)
                const float4 a4 = lds128(ra), b4 = lds128(ra + 16u), c4 = lds128(ra + 32u);
                const StageA A{a4.x, a4.y, a4.z, a4.w};
                const StageB B{b4.x, b4.y, b4.z, b4.w};
                const StageC C{c4.x, c4.y, c4.z, __float_as_int(c4.w)};
                dx = fx - A.mx;
                const float tA = A.A * dx;
                // one pair's contribution: alpha = min(araw, 0.99), d power masked by the clamp
                auto pair = [&](int p, float dy, float araw, bool unclamped, bool clampfree) {
#ifdef UWS_BWD_STATS
                    atomicAdd(&g_bwd_hist[33], 1ull);
                    paired = true;
#endif
                    // clampfree: alpha_raw <= opacity < the clamp band (the fast path)
                    const float alpha = clampfree ? araw : fminf(araw, kClampF);
                    const float inv_om = rcp_ftz(1.0f - alpha);
                    const float Ti = T[p] * inv_om;
                    const float w = alpha * Ti;
                    const float U = G[p][0] * C.r + G[p][1] * C.g + G[p][2] * C.b;
                    const float dalpha = U * Ti - S[p] * inv_om;
                    S[p] = fmaf(w, U, S[p]);
                    T[p] = Ti;
                    const float dp = unclamped ? dalpha * araw : 0.f;
                    // moments about the first pixel's row: dy = dy0 + 2p
                    sdp += dp;
                    if (p > 0) {
                        sdpy = fmaf(2.0f * p, dp, sdpy);         // sum 2p dp
                        sdpyy = fmaf(4.0f * p * p, dp, sdpyy);   // sum 4p^2 dp
                    }
                    wg0 = fmaf(w, G[p][0], wg0);
                    wg1 = fmaf(w, G[p][1], wg1);
                    wg2 = fmaf(w, G[p][2], wg2);
                };
                if (jrel < minl && B.lop < kLopClampLo) {
                    // every pixel of the thread still consumes this entry and alpha_raw
                    // <= opacity stays below the clamp band: only the floor gate remains
#pragma unroll
                    for (int p = 0; p < kPix; ++p) {
                        const float dy = fy[p] - A.my;
                        const float power = dx * fmaf(A.B, dy, tA) + fmaf(B.C * dy, dy, B.lop);
                        // the sure pass first: one test on the common path
                        if (power >= kPassLg2) {
                            pair(p, dy, ex2_ftz(power), true, true);
                            continue;
                        }
                        if (power < kSkipLg2) continue;
                        const float araw = ex2_ftz(power);
                        if (araw < kFloorLo) continue;
                        if (araw < kFloorHi &&
                            !(alpha_raw_f64_bwd(C.row, ox + lx,
                                                 oy + ly0 + 2 * p) >= kFloor))
                            continue;
                        pair(p, dy, araw, true, true);
                    }
                } else {
#pragma unroll
                    for (int p = 0; p < kPix; ++p) {
                        if (jrel >= mylast[p]) continue;
                        const float dy = fy[p] - A.my;
                        const float power = dx * fmaf(A.B, dy, tA) + fmaf(B.C * dy, dy, B.lop);
                        if (power < kSkipLg2) continue;
                        const float araw = ex2_ftz(power);
                        bool unclamped = araw < kClampLo;
                        if (power < kPassLg2 || fabsf(araw - kClampMid) < kClampHalf) {
                            // near a gate (rare): the full decision from alpha_raw, with
                            // both gates re-decided from the float64 record in the guard bands
                            if (araw < kFloorLo) continue;
                            if (araw < kFloorHi || fabsf(araw - kClampMid) < kClampHalf) {
                                const double e = alpha_raw_f64_bwd(C.row,
                                                                    ox + lx, oy + ly0 + 2 * p);
                                if (!(e >= kFloor)) continue;
                                unclamped = e < kClamp;
                            }
                        }
                        pair(p, dy, araw, unclamped, false);
                    }
                }
                {
                    const float dy0 = fy[0] - A.my;
                    const float y1 = fmaf(dy0, sdp, sdpy);        // sum dp dy
                    sdpyy = fmaf(dy0, y1 + sdpy, sdpyy);          // sum dp dy^2
                    sdpy = y1;
                }
            }
            const float sdpx = sdp * dx;
            float v[9] = {sdp, sdpx, sdpy, sdpx * dx, sdpy * dx, sdpyy, wg0, wg1, wg2};
#ifdef UWS_BWD_STATS
            {
                const unsigned hb = __ballot_sync(0xffffffffu, paired);
                if (lane == 0) atomicAdd(&g_bwd_hist[__popc(hb)], 1ull);
            }
#endif
            if (!__any_sync(0xffffffffu, hit)) continue;
            const float r = butterfly9(v, lane);
            if (accStore) sts_f32(accBase + 4u * (uint32_t)k, r);
            if (lane == 0) sts_u8(hitBase + (uint32_t)k, 1u);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < nb; k += kThreads) {
            float s[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) s[i] = 0.f;
            bool any = false;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {  // fixed order: deterministic per tile
                if (sHit[w][k]) {
                    any = true;
                    sHit[w][k] = 0;
#pragma unroll
                    for (int i = 0; i < 9; ++i) s[i] += sAcc[w][i][k];
                }
            }
            if (DET) {
                // every consumed slot is written (row = none when no pixel used it)
                const size_t slot = (size_t)a.tile_base[tile] + lo + k;
                const float ca = sRec[k].A.A * (-2.0f * kLn2);
                const float cb = sRec[k].A.B * (-kLn2);
                const float cc = sRec[k].B.C * (-2.0f * kLn2);
                float* g = a.part + slot * 9;
                g[0] = s[0];
                g[1] = ca * s[1] + cb * s[2];
                g[2] = cb * s[1] + cc * s[2];
                g[3] = -0.5f * s[3];
                g[4] = -s[4];
                g[5] = -0.5f * s[5];
                g[6] = s[6];
                g[7] = s[7];
                g[8] = s[8];
                a.part_row[slot] = any ? (uint32_t)sRec[k].C.row : a.none_row;
            } else if (any) {
                // natural-units conic from the log2-scaled staged values
                const float ca = sRec[k].A.A * (-2.0f * kLn2);
                const float cb = sRec[k].A.B * (-kLn2);
                const float cc = sRec[k].B.C * (-2.0f * kLn2);
                float* g = a.screen + (size_t)sRec[k].C.row * 9;
                atomicAdd(g + 0, s[0]);                      // d_logit (before (1-s))
                atomicAdd(g + 1, ca * s[1] + cb * s[2]);     // d_mean2d x
                atomicAdd(g + 2, cb * s[1] + cc * s[2]);     // d_mean2d y
                atomicAdd(g + 3, -0.5f * s[3]);              // d_conic a
                atomicAdd(g + 4, -s[4]);                     // d_conic b
                atomicAdd(g + 5, -0.5f * s[5]);              // d_conic c
                atomicAdd(g + 6, s[6]);                      // d_color
                atomicAdd(g + 7, s[7]);
                atomicAdd(g + 8, s[8]);
            }
        }
    }
}

// ---- deterministic mode ---------------------------------------------------
// Per tile: the consumed list prefix = max over its pixels of `last` (what the
// backward walks), written to count[tile].
__global__ void __launch_bounds__(256) k_tile_consumed(const int32_t* __restrict__ last, int width,
                                                       int height, int gx, int32_t* count) {
    pdl_entry();
    const int tile = blockIdx.x;
    const int ty = tile / gx, tx = tile - ty * gx;
    const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
    int v = (px < width && py < height) ? last[py * width + px] : 0;
    v = __reduce_max_sync(0xffffffffu, v);
    __shared__ int sm[8];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int m = 0;
        for (int w = 0; w < 8; ++w) m = max(m, sm[w]);
        count[tile] = m;
    }
}

// Exclusive scan of count[0..n) into base[0..n], one block (n = tiles <= a few 1e4).
__global__ void __launch_bounds__(1024) k_tile_scan(const int32_t* __restrict__ count, int n,
                                                    int32_t* base) {
    pdl_entry();
    __shared__ int32_t sm[33];
    int32_t carry = 0;
    for (int c = 0; c < n; c += 1024) {
        const int i = c + threadIdx.x;
        const int32_t v = i < n ? count[i] : 0;
        int32_t tot;
        const int32_t ex = block_exclusive_sum<1024, int32_t>(v, sm, &tot);
        if (i < n) base[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) base[n] = carry;
}

// One thread per run of equal rows in the row-sorted slots: the run's partials
// summed in slot order (tile order, as backward.py:334-341 merges), stored.
__global__ void __launch_bounds__(256) k_part_reduce(const uint32_t* __restrict__ rows,
                                                     const uint32_t* __restrict__ slots,
                                                     const float* __restrict__ part,
                                                     const int32_t* __restrict__ n_dev,
                                                     uint32_t none_row, float* screen) {
    pdl_entry();
    const int n = *n_dev;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t r = rows[i];
        if (r == none_row || (i > 0 && rows[i - 1] == r)) continue;
        float acc[9];
#pragma unroll
        for (int v = 0; v < 9; ++v) acc[v] = 0.f;
        for (int j = i; j < n && rows[j] == r; ++j) {
            const float* g = part + (size_t)slots[j] * 9;
#pragma unroll
            for (int v = 0; v < 9; ++v) acc[v] += g[v];
        }
        float* o = screen + (size_t)r * 9;
#pragma unroll
        for (int v = 0; v < 9; ++v) o[v] += acc[v];
    }
}

// medium_acc += per-tile medium partials summed in tile order (thread v = slot v).
__global__ void __launch_bounds__(32) k_med_reduce(const double* __restrict__ med_part, int tiles,
                                                   double* medium_acc) {
    pdl_entry();
    if (threadIdx.x >= 9) return;
    double s = 0.0;
    for (int t = 0; t < tiles; ++t) s += med_part[(size_t)t * 9 + threadIdx.x];
    medium_acc[threadIdx.x] += s;
}

struct DetPlan {
    float* part;
    uint32_t *part_row, *rows_sorted, *slots_sorted;
    double* med_part;
    radix::Plan<uint32_t> sort;
};

inline void det_plan(Workspace& ws, int tiles, int64_t r, int64_t k, DetPlan& p) {
    const uint32_t n = (uint32_t)(r > 0 ? r : 1);
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= (uint64_t)k) ++bits;  // keys 0..k (k = none)
    p.part = ws.take<float>((size_t)n * 9);
    p.part_row = ws.take<uint32_t>(n);
    p.rows_sorted = ws.take<uint32_t>(n);
    p.slots_sorted = ws.take<uint32_t>(n);
    p.med_part = ws.take<double>((size_t)tiles * 9);
    radix::plan<uint32_t>(ws, n, (bits + 7) / 8, p.sort);
}

}  // namespace
}  // namespace uws

using namespace uws;

#ifdef UWS_BWD_STATS
extern "C" int uws_debug_bwd_stats(unsigned long long* out35) {
    cudaMemcpyFromSymbol(out35, g_bwd_hist, sizeof(unsigned long long) * 35);
    unsigned long long z[35] = {};
    cudaMemcpyToSymbol(g_bwd_hist, z, sizeof(z));
    return 0;
}
#endif

extern "C" int uws_raster_bwd_det_prefix(const uws_camera* cam, const uws_raster_out* fwd,
                                         int32_t* tile_count, int32_t* tile_base, void* stream) {
    UWS_REQUIRE(cam && fwd && fwd->last && tile_count && tile_base,
                "uws_raster_bwd_det_prefix: null argument");
    const int gx = (int)ceil_div(cam->width, kTile), gy = (int)ceil_div(cam->height, kTile);
    launch(k_tile_consumed, dim3(gx * gy), dim3(256), 0, as_stream(stream), fwd->last, cam->width,
           cam->height, gx, tile_count);
    launch(k_tile_scan, dim3(1), dim3(1024), 0, as_stream(stream), (const int32_t*)tile_count,
           gx * gy, tile_base);
    count_launches(1);
    UWS_CHECK_LAUNCH("k_tile_scan");
    return UWS_OK;
}

extern "C" int uws_raster_bwd_det_workspace_size(int32_t tiles, int64_t r, int64_t k,
                                                 size_t* bytes) {
    UWS_REQUIRE(bytes && tiles >= 0 && r >= 0 && k >= 0,
                "uws_raster_bwd_det_workspace_size: bad argument");
    Workspace ws(nullptr, 0, true);
    DetPlan p;
    det_plan(ws, tiles, r, k, p);
    *bytes = ws.used;
    return UWS_OK;
}

extern "C" int uws_raster_bwd(const uws_projected* proj, const int32_t* offsets,
                              const int32_t* entries, const uws_camera* cam, const float* medium,
                              const uws_raster_out* fwd, const float* dL_dC, float* screen_grads,
                              double* medium_acc, void* stream) {
    UWS_REQUIRE(proj && offsets && cam && fwd && dL_dC && screen_grads,
                "uws_raster_bwd: null argument");
    UWS_REQUIRE(fwd->final_T && fwd->last, "uws_raster_bwd: forward context missing");
    UWS_REQUIRE(medium == nullptr || (fwd->color_clean && fwd->depth && medium_acc),
                "uws_raster_bwd: underwater backward needs color_clean, depth and medium_acc");
    BwdArgs a;
    a.splat = proj->splat;
    a.exact = proj->exact;
    a.offsets = offsets;
    a.entries = entries;
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.medium = medium;
    a.color_clean = fwd->color_clean;
    a.depth = fwd->depth;
    a.final_T = fwd->final_T;
    a.last = fwd->last;
    a.dL = dL_dC;
    a.screen = screen_grads;
    a.medium_acc = medium_acc;
    a.row_start = nullptr;
    a.row_items = nullptr;
    a.tile_rows = nullptr;
    a.tile_nrows = nullptr;
    a.tile_rows_cap = 0;
    a.order = fwd->tile_order;
    launch_serial(k_raster_bwd<false, UWS_BWD_MINB>, dim3(a.gx * gy), dim3(kThreads), 0, as_stream(stream), a);
    UWS_CHECK_LAUNCH("k_raster_bwd");
    return UWS_OK;
}

extern "C" int uws_raster_bwd_rows(const uws_projected* proj, const int32_t* row_start,
                                   const void* row_items, const uws_camera* cam,
                                   const float* medium, const uws_raster_out* fwd,
                                   const float* dL_dC, float* screen_grads, double* medium_acc,
                                   void* stream) {
    UWS_REQUIRE(proj && row_start && cam && fwd && dL_dC && screen_grads,
                "uws_raster_bwd_rows: null argument");
    UWS_REQUIRE(fwd->final_T && fwd->last, "uws_raster_bwd_rows: forward context missing");
    UWS_REQUIRE(medium == nullptr || (fwd->color_clean && fwd->depth && medium_acc),
                "uws_raster_bwd_rows: underwater backward needs color_clean, depth and medium_acc");
    BwdArgs a;
    a.splat = proj->splat;
    a.exact = proj->exact;
    a.offsets = nullptr;
    a.entries = nullptr;
    a.row_start = row_start;
    a.row_items = (const uint2*)row_items;
    a.tile_rows = fwd->tile_rows;
    a.tile_nrows = fwd->tile_nrows;
    a.tile_rows_cap = fwd->tile_rows_cap;
    a.order = fwd->tile_order;
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.medium = medium;
    a.color_clean = fwd->color_clean;
    a.depth = fwd->depth;
    a.final_T = fwd->final_T;
    a.last = fwd->last;
    a.dL = dL_dC;
    a.screen = screen_grads;
    a.medium_acc = medium_acc;
    launch_serial(k_raster_bwd<true, UWS_BWD_MINB>, dim3(a.gx * gy), dim3(kThreads), 0, as_stream(stream), a);
    UWS_CHECK_LAUNCH("k_raster_bwd_rows");
    return UWS_OK;
}

// Deterministic form of uws_raster_bwd / uws_raster_bwd_rows: the same kernel
// writes each (tile, Gaussian) partial to its slot, the slots are stably sorted
// by row and every row's partials are summed in tile order.
template <bool ROWS>
static int bwd_det(BwdArgs a, int gy, const int32_t* tile_base, int64_t r, int64_t k,
                   void* workspace, size_t workspace_bytes, cudaStream_t st) {
    const int tiles = a.gx * gy;
    Workspace ws(workspace, workspace_bytes);
    DetPlan p;
    det_plan(ws, tiles, r, k, p);
    UWS_REQUIRE(ws.ok(), "uws_raster_bwd_det: workspace too small");
    a.tile_base = tile_base;
    a.part = p.part;
    a.part_row = p.part_row;
    a.none_row = (uint32_t)k;
    a.med_part = p.med_part;
    launch_serial(k_raster_bwd<ROWS, UWS_BWD_MINB, true>, dim3(tiles), dim3(kThreads), 0, st, a);
    UWS_CHECK_LAUNCH("k_raster_bwd_det");
    if (r > 0) {
        UWS_CUDA(radix::sort_pairs<uint32_t>(p.sort, p.part_row, nullptr, p.rows_sorted,
                                             p.slots_sorted, (uint32_t)r, nullptr, 0, st));
        const int64_t nb = (int64_t)ceil_div(r, 256);
        const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
        launch(k_part_reduce, dim3(blocks), dim3(256), 0, st, (const uint32_t*)p.rows_sorted,
               (const uint32_t*)p.slots_sorted, (const float*)p.part, tile_base + tiles,
               (uint32_t)k, a.screen);
        UWS_CHECK_LAUNCH("k_part_reduce");
    }
    if (a.medium) {
        launch(k_med_reduce, dim3(1), dim3(32), 0, st, (const double*)p.med_part, tiles,
               a.medium_acc);
        UWS_CHECK_LAUNCH("k_med_reduce");
    }
    return UWS_OK;
}

extern "C" int uws_raster_bwd_det(const uws_projected* proj, const int32_t* offsets,
                                  const int32_t* entries, const int32_t* row_start,
                                  const void* row_items, const uws_camera* cam,
                                  const float* medium, const uws_raster_out* fwd,
                                  const float* dL_dC, float* screen_grads, double* medium_acc,
                                  const int32_t* tile_base, int64_t r, int64_t k, void* workspace,
                                  size_t workspace_bytes, void* stream) {
    UWS_REQUIRE(proj && cam && fwd && dL_dC && screen_grads && tile_base,
                "uws_raster_bwd_det: null argument");
    UWS_REQUIRE((offsets != nullptr) != (row_start != nullptr),
                "uws_raster_bwd_det: give either tile lists or row lists");
    UWS_REQUIRE(fwd->final_T && fwd->last, "uws_raster_bwd_det: forward context missing");
    UWS_REQUIRE(medium == nullptr || (fwd->color_clean && fwd->depth && medium_acc),
                "uws_raster_bwd_det: underwater backward needs color_clean, depth and medium_acc");
    UWS_REQUIRE(r >= 0 && k >= 0 && k < 0xffffffffll, "uws_raster_bwd_det: bad sizes");
    BwdArgs a = {};
    a.splat = proj->splat;
    a.exact = proj->exact;
    a.offsets = offsets;
    a.entries = entries;
    a.row_start = row_start;
    a.row_items = (const uint2*)row_items;
    if (row_start) {
        a.tile_rows = fwd->tile_rows;
        a.tile_nrows = fwd->tile_nrows;
        a.tile_rows_cap = fwd->tile_rows_cap;
    }
    a.order = fwd->tile_order;
    a.width = cam->width;
    a.height = cam->height;
    a.gx = (int)ceil_div(cam->width, kTile);
    const int gy = (int)ceil_div(cam->height, kTile);
    a.medium = medium;
    a.color_clean = fwd->color_clean;
    a.depth = fwd->depth;
    a.final_T = fwd->final_T;
    a.last = fwd->last;
    a.dL = dL_dC;
    a.screen = screen_grads;
    a.medium_acc = medium_acc;
    return row_start ? bwd_det<true>(a, gy, tile_base, r, k, workspace, workspace_bytes,
                                     as_stream(stream))
                     : bwd_det<false>(a, gy, tile_base, r, k, workspace, workspace_bytes,
                                      as_stream(stream));
}
