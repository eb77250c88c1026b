/*
 * uwsplat_b200.h -- C ABI of the B200 (sm_100a) underwater-splatting hot path.
 *
 * A drop-in device backend for the reference package `uwsplat` 0.1.0 (pure
 * Python; it ships no FFI of its own).  Each entry point below replaces one
 * stage of the reference's CPU path; the Python shim
 * `paper_2411_19588_b200` binds them with ctypes and keeps the reference's
 * public function names, arguments and exceptions.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors) unless the name says `host_`.  Nothing here allocates memory:
 *     scratch space is sized by the matching *_workspace_size() call and
 *     passed in by the caller.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it.  Calls are thread-safe for distinct streams + workspaces.
 *   - Every call returns UWS_OK (0) or an error code and records a message
 *     retrievable with uws_last_error() (thread-local).
 *   - Per-Gaussian parameters are float32 structure-of-arrays exactly as the
 *     reference GaussianCloud stores them (scene.py:90-147).
 */
#ifndef UWSPLAT_B200_H
#define UWSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UWS_OK 0
#define UWS_EINVAL 1      /* bad argument (maps to ValueError / DataError) */
#define UWS_ECUDA 2       /* CUDA runtime error */
#define UWS_ECAPACITY 3   /* caller-provided capacity too small */

#define UWS_TILE 16

/* Pinhole camera (reference: scene.py:190-245, Camera).  R is row-major
 * world->view, x_view = R x + t.  tan_fov = 0.5*width/fx. */
typedef struct uws_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    double near_plane, far_plane;
} uws_camera;

/* GaussianCloud fields (scene.py:97-105), float32 SoA, device pointers. */
typedef struct uws_cloud {
    const float* positions;       /* [n][3] */
    const float* log_scales;      /* [n][3] */
    const float* rotations;       /* [n][4] wxyz */
    const float* sh_coeffs;       /* [n][1][3] degree-0 features */
    const float* opacity_logits;  /* [n] */
    int64_t n;
} uws_cloud;

/* Raster record of one visible Gaussian (48 bytes, 16-byte aligned).
 * mean2d is kept in float64 so tile-local pixel offsets are exact. */
typedef struct uws_splat {
    double mx, my;                 /* mean2d, pixels (unclamped, projection.py:160) */
    float ca, cb, cc, opacity;     /* conic [c,-b,a]/det (projection.py:174-175), sigmoid(logit) */
    float r, g, b, depth;          /* clamped degree-0 colour, view depth */
} uws_splat;

/* ProjectedCloud (projection.py:40-86) in device form.  Rows are the
 * visible Gaussians in ascending source order; capacity = cloud n. */
typedef struct uws_projected {
    int32_t* source_index;   /* [K] */
    uws_splat* splat;        /* [K] */
    double* exact;           /* [K][4] conic a,b,c + opacity in float64 (gate re-evaluation) */
    double* depth;           /* [K] float64 view depth (sort key) */
    int16_t* rect;           /* [K][4] inclusive tile rect x0,y0,x1,y1, grid-clipped (projection.py:229-249) */
    double* cov2d;           /* optional [K][3] packed a,b,c (NULL to skip) */
    double* radius;          /* optional [K] footprint radius (NULL to skip) */
    int32_t* num_visible;    /* [1] K, written by uws_preprocess_fwd */
    uint32_t* depth_range;   /* optional [2] {~min, max} of the visible depths' high 32 bits,
                                written by uws_preprocess_fwd for uws_bin_count (NULL: the
                                binning finds them itself) */
} uws_projected;

/* Per-pixel forward outputs (RenderOutput, rasterizer.py:132-145).  All
 * [H][W] (x3 for colours) float32 unless noted; optional ones may be NULL. */
typedef struct uws_raster_out {
    float* color;          /* [H][W][3] underwater (or clean) colour */
    float* color_clean;    /* [H][W][3] clean composite; required when medium != NULL */
    float* depth;          /* [H][W] raw weighted depth, far where empty */
    float* weight;         /* [H][W] sum alpha_i T_i */
    float* final_T;        /* [H][W] final transmittance */
    int32_t* count;        /* [H][W] blended contributors */
    int32_t* last;         /* [H][W] consumed prefix length of the tile list (backward context) */
    float* attenuation;    /* optional [H][W][3] exp(-B_d z) */
    float* backscatter;    /* optional [H][W][3] B_inf (1 - exp(-B_b z)) */
    /* optional (row-list path): the first tile_rows_cap rows each tile staged, in
     * list order, so the backward reads its consumed prefix instead of filtering
     * the row lists again; NULL to skip.  tile_rows [tiles][tile_rows_cap],
     * tile_nrows [tiles] = rows stored (written by uws_raster_fwd_rows), with bit 30
     * set when the stored rows are the tile's whole list. */
    int32_t* tile_rows;
    int32_t* tile_nrows;
    int32_t tile_rows_cap;
    /* optional exact-transmittance pass: the float32 walk decides T >= 1e-4
     * (rasterizer.py:169) in float32; pixels whose T lands within +-0.2 % of
     * 1e-4 are listed in fix_pixels [H*W] and re-walked in float64, so count,
     * last and the T decision equal the reference's.  fix_count: device
     * int32[3]; [0] and [1] zero on entry and left zero on exit, [2] set to the
     * number of pixels re-walked.  NULL to skip. */
    int32_t* fix_pixels;
    int32_t* fix_count;
    /* optional [tiles] permutation of the tiles: CTA b of the forward and of the
     * backward composites tile tile_order[b].  A schedule only (tiles are
     * independent): heaviest tiles first shortens the kernels' tails.  NULL =
     * raster order.  uws_tile_order computes it from a forward's tile_nrows. */
    const int32_t* tile_order;
} uws_raster_out;

/* Adam hyper-parameters for one apply_gradients call (optim.py:69-120).
 * Index order: positions, log_scales, rotations, sh_coeffs, opacity_logits,
 * attenuation, water_color, backscatter.  bias1/bias2 = 1 - beta^step and
 * the learning rates are computed on the host exactly as the reference does. */
typedef struct uws_adam_params {
    double lr[8];
    double bias1[8];
    double bias2[8];
    double inv_bias1[8];   /* RN(1 / bias1): exact-division helper */
    double inv_bias2[8];
    double beta1, beta2, one_minus_beta1, one_minus_beta2, eps;
} uws_adam_params;

/* ---- meta ------------------------------------------------------------ */
const char* uws_version(void);
const char* uws_last_error(void);
/* number of kernels this library has launched in the process (monotonic) */
uint64_t uws_kernel_launches(void);

/* ---- preprocess (replaces projection.project_cloud, projection.py:100-199,
 *      footprint_radius :89-97 and _spans_for :229-249) ------------------ */
int uws_preprocess_workspace_size(int64_t n, size_t* bytes);
int uws_preprocess_fwd(const uws_cloud* cloud, const uws_camera* cam, uws_projected* out,
                       void* workspace, size_t workspace_bytes, void* stream);

/* ---- binning (replaces rasterizer.bin_and_sort, rasterizer.py:50-85).
 *      Sizes live on the device so a training step needs no host sync:
 *      K is read from proj->num_visible (k_cap only sizes grids/workspace).
 *      uws_bin_count stable-sorts the visible rows by float64 depth and
 *      counts, per tile row, the entries of each 2048-rank block; it writes
 *      totals[0] = E (tile entries) and totals[1] = S (row segments).
 *      uws_bin_emit builds the tile lists by two levels of stable bucketing
 *      -- rank order -> tile-row lists -> tile lists -- and the CSR ranges.
 *      If E > e_cap or S > s_cap it sets *overflow = 1, writes all-zero
 *      offsets (empty lists) and nothing else -- and, if skip_counter (device
 *      float[2] = {non-finite count, overflow count}, the gradient buffer's
 *      slots 16n+9, 16n+10) is given, adds 1 to skip_counter[1] so a
 *      following uws_adam_step is a no-op; the
 *      caller grows its buffers to the totals and re-runs.  count_ws is sized with (k_cap, 0) and must
 *      be the same buffer in both calls; emit_ws with (k_cap, s_cap). */
int uws_bin_workspace_size(int64_t k_cap, int64_t s_cap, int32_t n_tiles_x, int32_t n_tiles_y,
                           size_t* count_bytes, size_t* emit_bytes);
int uws_bin_count(const uws_projected* proj, int64_t k_cap, const uws_camera* cam,
                  int64_t* totals /* device [2]: E, S */, void* count_ws, size_t count_bytes,
                  void* stream);
int uws_bin_emit(const uws_projected* proj, int64_t k_cap, int64_t e_cap, int64_t s_cap,
                 const uws_camera* cam, const int64_t* totals /* device, from uws_bin_count */,
                 int32_t* offsets /* [tiles+1] */, int32_t* entries /* [e_cap] rows */,
                 int32_t* overflow /* device flag */, float* skip_counter /* optional */,
                 void* count_ws, size_t count_bytes, void* emit_ws, size_t emit_bytes,
                 void* stream);

/* Row-list variant for the training/render hot path: after uws_bin_count,
 * builds only the first level -- for every tile row, the depth-ordered rows
 * whose rectangle spans it (row_start [tiles_y+1], row_items [s_cap]) --
 * and no E-sized tile lists.  The *_rows compositing kernels derive each
 * tile's list from its row list on the fly and stop at saturation.  Only
 * S <= s_cap is checked (overflow / skip_counter as above). */
int uws_bin_rows(const uws_projected* proj, int64_t k_cap, int64_t s_cap, const uws_camera* cam,
                 const int64_t* totals, int32_t* row_start,
                 void* row_items /* [s_cap] x 8 B: row, tile x0 | x1 << 16 */,
                 int32_t* overflow, float* skip_counter, void* count_ws, size_t count_bytes,
                 void* stream);

/* ---- forward compositing + medium epilogue (replaces rasterizer.render's
 *      tile loop / _composite_block :148-178 / apply_water :244-251).
 *      medium: device float[9] = attenuation[3], water_color[3],
 *      backscatter[3]; NULL selects clean mode. ---------------------------- */
int uws_raster_fwd(const uws_projected* proj, const int32_t* offsets, const int32_t* entries,
                   const uws_camera* cam, const float* medium, uws_raster_out* out, void* stream);
/* Schedule for the next compositing launches over the same view and buffers:
 * the tiles by descending consumed-prefix length (tile_nrows of a forward,
 * low 30 bits / 8, capped at 127), written to order [n_tiles].  One CTA, async on
 * stream.  (No reference counterpart: the reference composites tiles in a
 * worker pool, rasterizer.py:186-241.) */
int uws_tile_order(const int32_t* tile_nrows, int32_t n_tiles, int32_t* order, void* stream);
int uws_raster_fwd_rows(const uws_projected* proj, const int32_t* row_start,
                        const void* row_items, const uws_camera* cam, const float* medium,
                        uws_raster_out* out, void* stream);

/* ---- loss (replaces losses.total_loss :140-160 incl. l1 :40-49 and
 *      d_ssim :83-123).  rendered/gt: [H][W][C] float32.  medium: device
 *      float[15] (9 params + water_color_guide[3] + backscatter_guide[3]) or
 *      NULL.  result: device double[6] = l1, d_ssim, l_bs, total,
 *      finite flag (1.0/0.0), reserved.  nonfinite (optional device float):
 *      incremented when the total is not finite (pipeline.py:182-184). ---- */
int uws_loss_workspace_size(int32_t h, int32_t w, int32_t c, size_t* bytes);
int uws_loss_fwd_bwd(const float* rendered, const float* gt, int32_t h, int32_t w, int32_t c,
                     const float* medium, int32_t has_guidance, double lambda_ssim,
                     double lambda_guide, float* dL_dC, double* result, float* nonfinite,
                     void* workspace, size_t workspace_bytes, void* stream);

/* ---- backward compositing (replaces backward._backward_block :124-163 and
 *      backward_medium :261-275).  screen_grads: [K][9] float32 accumulated
 *      (+=) per visible row: d_logit_raw, d_mean2d x,y, d_conic a,b,c,
 *      d_color r,g,b.  medium_acc: device double[9] accumulated (+=). ----- */
int uws_raster_bwd(const uws_projected* proj, const int32_t* offsets, const int32_t* entries,
                   const uws_camera* cam, const float* medium, const uws_raster_out* fwd,
                   const float* dL_dC, float* screen_grads, double* medium_acc, void* stream);
/* _rows variant: reads each tile's consumed prefix from fwd->tile_rows when the
 * forward stored it (tile_rows != NULL and the prefix fits the cap), else
 * filters the row lists again. */
int uws_raster_bwd_rows(const uws_projected* proj, const int32_t* row_start,
                        const void* row_items, const uws_camera* cam, const float* medium,
                        const uws_raster_out* fwd, const float* dL_dC, float* screen_grads,
                        double* medium_acc, void* stream);

/* Deterministic backward (opt-in): gradients bit-identical from run to run,
 * like the reference, which merges per-tile partials in tile order
 * (backward.py:334-341).  uws_raster_bwd_det_prefix writes each
 * tile's consumed list prefix (max of fwd->last over its pixels) to
 * tile_count [tiles] and their exclusive prefix to tile_base [tiles+1]
 * (tile_base[tiles] = R, the slot count).  uws_raster_bwd_det then runs the
 * backward kernel writing every (tile, Gaussian) partial to its own slot,
 * sorts the slots by row (stable) and sums each row's partials in tile order
 * into screen_grads (+=); the per-tile medium partials are summed in tile
 * order into medium_acc (+=).  Exactly one of offsets/entries (tile lists) or
 * row_start/row_items (row lists) is given; k = visible rows (proj->num_visible). */
int uws_raster_bwd_det_prefix(const uws_camera* cam, const uws_raster_out* fwd,
                              int32_t* tile_count, int32_t* tile_base, void* stream);
int uws_raster_bwd_det_workspace_size(int32_t tiles, int64_t r, int64_t k, size_t* bytes);
int uws_raster_bwd_det(const uws_projected* proj, const int32_t* offsets, const int32_t* entries,
                       const int32_t* row_start, const void* row_items, const uws_camera* cam,
                       const float* medium, const uws_raster_out* fwd, const float* dL_dC,
                       float* screen_grads, double* medium_acc, const int32_t* tile_base,
                       int64_t r, int64_t k, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ---- projection backward (replaces backward._project_backward :184-258 and
 *      _quat_backward :166-181).  grads: float32 flat buffer laid out as
 *      [positions 3n | log_scales 3n | rotations 4n | sh 3n | opacity n |
 *       mean2d_grad_norm n | observed n | medium 9 | non-finite counter |
 *       overflow counter | pad 5], accumulated (+=); K is read from proj->num_visible.
 *      screen_grads and medium_acc are consumed and left zeroed.  The
 *      guidance subgradient lambda_guide*sign(.) is added into the medium
 *      slots (backward.py:270-274).  nonfinite (optional device float) is
 *      incremented when an accumulated gradient is not finite
 *      (GradientBuffer.all_finite, backward.py:66-69).  accumulate = 0
 *      stores the visible rows' parameter gradients instead of adding them
 *      (first view into a buffer known to be zero: saves the read). ------ */
int uws_preprocess_bwd(const uws_cloud* cloud, const uws_camera* cam, const uws_projected* proj,
                       int64_t k_cap, float* screen_grads, double* medium_acc,
                       const float* medium, int32_t has_guidance, double lambda_guide,
                       float* grads, float* nonfinite, int32_t accumulate, void* stream);

/* ---- optimizer (replaces optim.apply_gradients :98-120 / adam_step :69-83,
 *      GaussianCloud.normalize_rotations scene.py:132-134 and
 *      MediumParams.clamp_ scene.py:174-178).  params/m/v: 14n floats in the
 *      field layout above; grads: the flat gradient buffer; medium_*: 9
 *      floats (medium_grads = grads + 16n).  Optional step control for the
 *      device-resident training loop (pipeline.py:182-192): skip (device
 *      float[2] = {non-finite count, overflow count}) with either > 0 turns
 *      the update into a no-op; grad_accum/obs_count receive the
 *      densification statistics; zero_grads leaves the gradient buffer
 *      zeroed for the next step except the skip counters (medium_grads[9],
 *      [10]), which stay set after a skip so that steps already queued
 *      behind it skip as well, until the caller clears them. ------ */
int uws_adam_step(float* params, float* exp_avg, float* exp_avg_sq, float* grads, int64_t n,
                  float* medium_params, float* medium_exp_avg, float* medium_exp_avg_sq,
                  float* medium_grads, const uws_adam_params* hp, const float* skip,
                  float* grad_accum, int32_t* obs_count, int32_t zero_grads, void* stream);
/* The cloud part of uws_adam_step for the float4 groups [group_begin, group_end)
 * of the 14n parameter scalars (even n, 16-byte aligned buffers), so an update
 * can follow a gradient all-reduce chunk by chunk; the densification statistics
 * of Gaussian t are folded by the range holding group t.  The medium part is
 * uws_adam_step with n = 0. */
int uws_adam_step_range(float* params, float* exp_avg, float* exp_avg_sq, float* grads, int64_t n,
                        const uws_adam_params* hp, const float* skip, float* grad_accum,
                        int32_t* obs_count, int32_t zero_grads, int64_t group_begin,
                        int64_t group_end, void* stream);

/* ---- densification (replaces optim.densify_and_prune :132-198 and
 *      reset_opacities :201-207).  Two phases around one host read: classify
 *      writes totals[3] = {n_keep, n_clone, n_split} (device int64) so the
 *      caller can size the new buffers and draw the split samples
 *      ([2][n_split][3] float64, standard normal, from its own generator, in
 *      the reference's order); apply writes the new cloud / moments
 *      (n_keep + n_clone + 2 n_split rows; moment buffers must be zeroed by the
 *      caller: only kept rows are written).  Same workspace for both. ---- */
int uws_densify_workspace_size(int64_t n, size_t* bytes);
int uws_densify_classify(const float* params, int64_t n, const float* grad_accum,
                         const int32_t* obs_count, double grad_threshold, double size_threshold,
                         double min_opacity, int64_t* totals, void* workspace,
                         size_t workspace_bytes, void* stream);
int uws_densify_apply(const float* params, const float* exp_avg, const float* exp_avg_sq,
                      int64_t n, const void* workspace, size_t workspace_bytes,
                      const double* samples, double log_split_factor, int64_t n_keep,
                      int64_t n_clone, int64_t n_split, float* new_params, float* new_exp_avg,
                      float* new_exp_avg_sq, void* stream);
int uws_reset_opacities(float* params, float* exp_avg, float* exp_avg_sq, int64_t n, float value,
                        void* stream);

/* ---- guidance refresh (replaces backscatter.estimate_backscatter :211-270,
 *      called every refit_period iterations by pipeline.py:204-208).
 *      image: (h, w, 3) float32; depth: (h, w), either the remapped float64
 *      depth (depth_is_raw = 0, the reference's argument) or the raw float32
 *      render depth (depth_is_raw = 1: logistic_remap, medium.py:26-29, is
 *      applied inside, as pipeline.py:205 does before the call).
 *      Resize to min(resized_height, h) rows (bilinear colour, nearest depth),
 *      per depth cluster the ceil(p_dark*size) darkest pixels (stable), the
 *      per-interval per-channel minima, and a box-constrained multi-start
 *      Levenberg-Marquardt fit of v(z) = b_inf (1 - exp(-b_b z)) per channel.
 *      result[12] (device float64): water_color_est[3], backscatter_est[3],
 *      residual[3], degenerate (0/1), number of dark pixels, error (1: cluster
 *      edges not strictly increasing, the reference's DataError).
 *      medium_guide (optional, device float32[6] = medium slots 9..14): set to
 *      the float32 estimate when it is not degenerate (pipeline.py:206-208).
 *      dark (optional, device float64 [4 * pixels]): the dark set as
 *      (z, r, g, b) rows in raster order.  edges_num and intervals_num <= 257. */
typedef struct uws_backscatter_cfg {
    double p_dark;          /* 0.01 */
    int32_t intervals_num;  /* 25 */
    int32_t resized_height; /* 300 */
    int32_t edges_num;      /* 10 */
    int32_t pad;
} uws_backscatter_cfg;

int uws_backscatter_workspace_size(int32_t h, int32_t w, const uws_backscatter_cfg* cfg,
                                   size_t* bytes);
int uws_estimate_backscatter(const float* image, const void* depth, int32_t depth_is_raw,
                             int32_t h, int32_t w, const uws_backscatter_cfg* cfg,
                             double* result, float* medium_guide, double* dark,
                             void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* UWSPLAT_B200_H */
