/*
 * splat_b200.h -- C ABI of the B200-native Splat-LOAM hot path.
 *
 * Plain pointers and sizes only (no torch types).  All device pointers are
 * CUDA device memory owned by the caller unless stated otherwise; every call
 * is stream-ordered on the given cudaStream_t (passed as void*) and never
 * aborts: it returns an ss_status code which the Python host layer maps onto
 * the reference's exception classes (splatscan/errors.py:8-25).
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference tree, pkg/src/splatscan/):
 *   ss_render_forward        rasterizer.py:455-499  rasterize_forward
 *   ss_records_*             rasterizer.py:136-148  BlendRecords
 *   ss_render_backward       rasterizer.py:534-701  rasterize_backward
 *   ss_render_backward_blend rasterizer.py:556-684  (its per-tile accumulation loop)
 *   ss_render_finalize       rasterizer.py:686-701  (its per-splat gradient mapping)
 *                            (+ splats.py:133-163 tangent_raw_gradients and the
 *                             raw-space chain rule of mapping.py:479-494 when
 *                             raw_space = 1)
 *   ss_mapping_loss          mapping.py:128-196     range/normal/opacity losses
 *   ss_scale_loss            mapping.py:166-178     scale hinge
 *   ss_adam_step             mapping.py:367-379     Adam of refine (+ :495-496 clamp)
 *   ss_render_finalize_adam_dev  the finalize fused with the refine step's Adam
 *   ss_reg_anchors           registration.py:190-213 sample_model (+ :430 thinning)
 *   ss_range_image           geometry.py:252-268     build_range_image
 *   ss_smooth_range_image    geometry.py:271-287     smooth_range_image (size 3)
 *   ss_range_image_normals   geometry.py:290-338     range_image_normals
 *   ss_photo_system          registration.py:316-362 _photo_system (+ Huber and
 *                            the H/b accumulation of registration.py:470-477,
 *                            objective of registration.py:379-384)
 *   ss_leaf_tree_build       registration.py:98-164  build_leaf_tree
 *   ss_spawn_weights, ss_densify_mask, ss_spawn_splats, ss_prune_*
 *                            mapping.py:202-311, 412-438 map growth
 *   ss_reg_solve             registration.py:437-524 the GN/LM loop of register
 *   ss_reg_solve_async       the same, enqueued only (batches of frames, one stream each)
 *                            (every mode) + _geo_system :231-274, se3.py:121-150
 */
#ifndef SPLAT_B200_H
#define SPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (host layer maps them to splatscan.errors) ---------- */
typedef enum {
  SS_OK = 0,
  SS_ERR_INVALID_ARGUMENT = 1, /* GeometryError: bad sizes / camera / config   */
  SS_ERR_STALE_RECORDS = 2,    /* GeometryError: records do not match model    */
  SS_ERR_UNSUPPORTED = 3,      /* GeometryError: e.g. tile_size not 8 or 16    */
  SS_ERR_CUDA = 4,             /* RuntimeError: CUDA launch / allocation error */
  SS_ERR_CAPACITY = 5,         /* internal: pair capacity exceeded, retry      */
  SS_ERR_DEGENERATE = 6,       /* GeometryError: zero / parallel raw tangents  */
  SS_ERR_REGISTRATION = 7      /* RegistrationError: too few residuals survive */
} ss_status;

/* SphericalCamera (geometry.py:68-115) */
typedef struct {
  int32_t width, height;
  double az_min, az_max, el_min, el_max;
} ss_camera;

/* RasterConfig (rasterizer.py:69-78) */
typedef struct {
  int32_t tile_size;  /* 8 (reference default) or 16 */
  int32_t chunk_size; /* accepted for API parity; output-neutral */
  double alpha_cutoff, alpha_clamp, min_transmittance, denom_eps, cutoff_sigma, bbox_pad_px;
} ss_raster_cfg;

/* SplatModel raw storage (splats.py:166-212), float32 device arrays */
typedef struct {
  int32_t n;
  const float* centers;       /* n x 3 */
  const float* raw_t_alpha;   /* n x 3 */
  const float* raw_t_beta;    /* n x 3 */
  const float* log_scales;    /* n x 2 */
  const float* logit_opacity; /* n     */
} ss_splats;

/* Opaque records of one forward render (tile lists, per-pixel blend state).
 * Owns its device buffers (stream-ordered allocations). */
typedef struct ss_records ss_records;

ss_records* ss_records_create(void);
void ss_records_destroy(ss_records* rec, void* stream);

/* Forward render.  pose_Rt = row-major R (9) then t (3), sensor-in-world
 * (se3.py:3-7).  Outputs (device, float32): range H*W, normal H*W*3,
 * opacity H*W.  Fills `rec` for ss_render_backward.  Fully stream-ordered
 * (no host synchronisation, CUDA-graph capturable): the (tile, splat) pair
 * buffers are sized speculatively, so completion must be confirmed with
 * ss_records_check before host use of the results. */
int ss_render_forward(const ss_camera* cam, const double* pose_Rt, const ss_splats* splats,
                      const ss_raster_cfg* cfg, float* out_range, float* out_normal,
                      float* out_opacity, ss_records* rec, void* stream);

/* Confirm a forward: wait = 1 blocks until it finished; wait = 0 polls.
 * Returns SS_ERR_CAPACITY when the speculative pair capacity was exceeded
 * (outputs invalid; the next ss_render_forward on `rec` allocates enough,
 * so re-run), or the device-side status (e.g. SS_ERR_DEGENERATE). */
int ss_records_check(ss_records* rec, int wait);

/* Deterministic gradient reduction for the backward passes of these records
 * (default off): every (tile, splat) entry is reduced across the warp in a
 * fixed order and stored at its list position, then summed per splat over
 * its tiles in row-major order -- bit-identical gradients run to run, at the
 * cost of ~64 B per tile pair of extra traffic.  Without it the per-splat
 * sums use float atomics (order-dependent rounding, ~1e-7 relative). */
int ss_records_set_deterministic(ss_records* rec, int32_t deterministic);

/* Buffer generation of `rec`: incremented whenever a forward or backward had
 * to reallocate any of the records' device buffers.  A CUDA graph captured
 * over `rec` is only valid while the generation it was captured at holds. */
int ss_records_generation(const ss_records* rec, uint64_t* generation);

/* Reserve pair capacity for the next forwards on `rec` (at least n_pairs). */
int ss_records_reserve(ss_records* rec, int64_t n_pairs);

/* *sticky = 1 (device int) if the last forward on `rec` overflowed its pair
 * capacity: lets a CUDA-graph replay loop detect an overflow after the fact. */
int ss_records_sticky_overflow(const ss_records* rec, int32_t* sticky, void* stream);

/* Number of (tile, splat) pairs and tiles of a finished forward. */
int ss_records_counts(const ss_records* rec, int64_t* n_pairs, int32_t* tiles_x, int32_t* tiles_y);
/* Copy tile_ptr (tiles+1) and pair_splats (n_pairs) into caller device
 * buffers as int64, matching BlendRecords (rasterizer.py:145-146). */
int ss_records_export(const ss_records* rec, int64_t* tile_ptr, int64_t* pair_splats, void* stream);

/* Per-pixel blend state of a finished forward into caller device buffers (W x H
 * each, either may be NULL): the transmittance left after the tile list
 * (_chunk_transmittance's carried-out value, rasterizer.py:402-414) and the
 * 1-based list position of the last contributing entry (0: none). */
int ss_records_pixel_state(const ss_records* rec, float* final_T, int32_t* last, void* stream);

/* Work counts of a finished forward for the roofline: evaluations E =
 * sum over tiles of pixels x list length, contributions U = (pixel, splat)
 * pairs with nonzero blend weight.  Synchronises the stream. */
int ss_records_work(const ss_records* rec, int64_t* evaluations, int64_t* contributions, void* stream);

/* Optional CUDA-event timing of every kernel stage launched with `rec`
 * (0 preprocess, 1 emit, 2 bucket, 3 tile_sort, 4 unused, 5 forward,
 * 6 backward, 7 finalize).  ss_records_stage_times waits for the events,
 * returns summed milliseconds and launch counts per stage and resets. */
int ss_records_profile(ss_records* rec, int enable);
int ss_records_stage_times(ss_records* rec, double* ms, int32_t* launches, int32_t n_stages);

/* Backward.  dD: H*W, dN: H*W*3, dO: H*W float32 pixel gradients
 * (PixelGradients, rasterizer.py:90-96).
 * raw_space = 0: grads = n x 15 plain-space SplatGradients
 *   [d_centers 3 | d_t_alpha 3 | d_t_beta 3 | d_normal 3 | d_scales 2 | d_opacity 1]
 * raw_space = 1: grads = n x 12 raw-parameter gradients
 *   [centers 3 | raw_t_alpha 3 | raw_t_beta 3 | log_scales 2 | logit_opacity 1]
 *   d_scales_extra (n x 2, may be NULL) adds the scale-loss gradient first
 *   (mapping.py:492). */
int ss_render_backward(const ss_records* rec, const ss_splats* splats, const float* dD,
                       const float* dN, const float* dO, const float* d_scales_extra,
                       float* grads, int raw_space, void* stream);

/* ss_render_backward in two halves, so that a caller can overlap the per-splat
 * finalize with a collective over the finished rows (shared-map multi-GPU
 * training): ss_render_backward_blend runs the blend backward
 * into the records' per-splat accumulators; ss_render_finalize turns the
 * accumulators of splats [begin, end) into rows begin..end-1 of `grads`
 * (same layout as above; begin a multiple of 128) and clears them.  Calling
 * blend once and finalize over a partition of [0, n) equals ss_render_backward. */
int ss_render_backward_blend(const ss_records* rec, const ss_splats* splats, const float* dD,
                             const float* dN, const float* dO, void* stream);
int ss_render_finalize(const ss_records* rec, const ss_splats* splats, const float* d_scales_extra,
                       float* grads, int raw_space, int32_t begin, int32_t end, void* stream);

/* Mapping loss of one keyframe (mapping.py:128-196) on device images.
 * kf_range/kf_valid: target range image; kf_normal/kf_nvalid: target normals.
 * Writes pixel gradients dD, dN, dO and accumulates the four loss parts
 * [range, opacity, normal, unused] into parts4 (float64, device, zeroed by
 * the caller). */
int ss_mapping_loss(int32_t width, int32_t height, const float* range, const float* normal,
                    const float* opacity, const float* kf_range, const uint8_t* kf_valid,
                    const float* kf_normal, const uint8_t* kf_nvalid, double w_opacity,
                    double w_normal, double range_floor, float* dD, float* dN, float* dO,
                    double* parts4, void* stream);

/* Scale hinge of the mapping loss (mapping.py:166-178): writes the n x 2
 * log-scale-space input d_scales_extra for ss_render_backward (w_scale on the
 * larger axis of splats above `cap`) and adds the hinge sum to *loss_out
 * (device float64). */
int ss_scale_loss(const float* log_scales, int32_t n, double cap, double w_scale, float* d_scales_extra,
                  double* loss_out, void* stream);

/* One Adam step of refine (mapping.py:367-379, 495-496) on the five raw
 * parameter arrays (in place) from the packed n x 12 raw gradient; m, v:
 * n x 12 moments; t: step count after increment; lrs5: learning rates of
 * (centers, raw_t_alpha, raw_t_beta, log_scales, logit_opacity); log scales
 * are clamped to [log_scale_lo, log_scale_hi] afterwards. */
int ss_adam_step(float* centers, float* raw_t_alpha, float* raw_t_beta, float* log_scales, float* logit_opacity,
                 const float* grads, float* m, float* v, int32_t n, int32_t t, const double* lrs5, double beta1,
                 double beta2, double eps, double log_scale_lo, double log_scale_hi, void* stream);

/* The same Adam step with the step counter on the device (t_dev += 1, bias
 * corrections computed there into bias_ws[2]): no per-step host argument, so
 * the whole refine step replays as one CUDA graph. */
int ss_adam_step_dev(float* centers, float* raw_t_alpha, float* raw_t_beta, float* log_scales, float* logit_opacity,
                     const float* grads, float* m, float* v, int32_t n, int32_t* t_dev, float* bias_ws,
                     const double* lrs5, double beta1, double beta2, double eps, double log_scale_lo,
                     double log_scale_hi, void* stream);
/* The finalize of ss_render_finalize (all rows, raw space, d_scales_extra the scale-hinge
 * gradient) fused with ss_adam_step_dev: the raw gradient of each splat goes straight into
 * the Adam step (mapping.py:479-496) on the splats' own parameter arrays (updated in place,
 * the const of ss_splats notwithstanding) and the moments m, v; no gradient array.  Runs
 * after ss_render_backward_blend; t_dev / bias_ws as for ss_adam_step_dev.  scale_loss !=
 * NULL: the scale hinge (mapping.py:166-178, ss_scale_loss) is evaluated here too, its
 * loss added to *scale_loss, and d_scales_extra is ignored. */
int ss_render_finalize_adam_dev(const ss_records* rec, const ss_splats* splats, const float* d_scales_extra,
                                float* m, float* v, int32_t* t_dev, float* bias_ws, const double* lrs5,
                                double beta1, double beta2, double eps, double log_scale_lo, double log_scale_hi,
                                double scale_cap, double w_scale, double* scale_loss, void* stream);

/* history[*it_dev] = parts4 (the four mapping-loss parts of a step), *it_dev += 1. */
int ss_store_loss_parts(const double* parts4, double* history, int32_t* it_dev, int32_t cap, void* stream);

/* ---- photometric registration (registration.py:170-384) -------------- */
typedef struct {
  double huber_photo, trim_factor, spread_gate;
} ss_reg_cfg;

/* Anchors of sample_model (registration.py:190-213, 430): from a render of
 * the model at pose_Rt on geo_cam (range D, opacity O, float32 device),
 * pixels with O > vis_opacity and D > 0, minus range jumps > spread_gate,
 * back-projected at depth D/O and mapped to the world; every `thin`-th kept
 * pixel (row-major) becomes an anchor.  X_out: cap x 3 float64 (device).
 * counts_out (host): [kept pixels, anchors].  Synchronises the stream.
 * workspace: ss_anchor_workspace_bytes(width, height) bytes of device memory. */
size_t ss_anchor_workspace_bytes(int32_t width, int32_t height);
int ss_reg_anchors(const ss_camera* geo_cam, const float* D, const float* O, const double* pose_Rt,
                   double vis_opacity, double spread_gate, int32_t thin, double* X_out, int32_t cap,
                   int32_t* counts_out, void* workspace, void* stream);

/* build_range_image (geometry.py:252-268): sensor-frame points (n x 3
 * float64, device) -> nearest range per pixel (float64 H*W) and valid mask. */
int ss_range_image(const ss_camera* cam, const double* pts, int32_t n, double* range_out, uint8_t* valid_out,
                   void* stream);

/* Map growth (mapping.py:202-311, 412-438).
 * ss_spawn_weights: _range_gradient_weights (float64 H*W) of a keyframe range image.
 * ss_densify_mask: densify_mask = valid & (rendered opacity <= densify_opacity |
 *   |rendered range - keyframe range| >= densify_range_err).
 * ss_spawn_splats: spawn_splats' splat construction for m drawn pixel indices
 *   (row-major int64; the weighted draw itself is numpy's on the host), written
 *   as float32 raw parameters at the given device pointers.
 * ss_prune_flags + ss_prune_compact: SplatModel.prune / _Adam.prune -- keep splats
 *   with sigmoid(logit) >= prune_opacity; flags and offsets live in `workspace`
 *   (ss_prune_workspace_bytes(n)), then each per-splat array (rows of `width`
 *   floats) is compacted stably into `dst`. */
int ss_spawn_weights(int32_t width, int32_t height, int32_t wrap, const double* range, const uint8_t* valid,
                     double* w_out, void* stream);
int ss_densify_mask(int32_t n_pixels, const double* kf_range, const uint8_t* kf_valid, const float* render_range,
                    const float* render_opacity, double densify_opacity, double densify_range_err, uint8_t* mask_out,
                    void* stream);
int ss_spawn_splats(const ss_camera* cam, const double* kf_range, const double* kf_normal, const uint8_t* kf_nvalid,
                    const double* pose_Rt, const int64_t* pixels, int32_t m, double footprint_gain,
                    double scale_floor, double opacity_init, float* centers, float* raw_t_alpha, float* raw_t_beta,
                    float* log_scales, float* logit_opacity, void* stream);
size_t ss_prune_workspace_bytes(int32_t n);
int ss_prune_flags(int32_t n, const float* logit_opacity, double prune_opacity, int32_t* n_keep_out, void* workspace,
                   void* stream);
int ss_prune_compact(int32_t n, int32_t width, const float* src, float* dst, const void* workspace, void* stream);

/* smooth_range_image (geometry.py:271-287), size 3: 3x3 median of the valid
 * ranges (invalid pixels count as +inf; columns wrap when `wrap`, else both
 * axes clamp), pixels whose median is +inf keep their range.  range/out:
 * H*W float64, valid: H*W bytes, all device.  Bit-exact. */
int ss_smooth_range_image(int32_t width, int32_t height, int32_t wrap, const double* range, const uint8_t* valid,
                          double* out, void* stream);

/* range_image_normals (geometry.py:290-338): central-difference unit normals
 * (H*W*3 float64) oriented toward the sensor and their mask (four valid
 * neighbours, azimuth seam wrapped for full-circle cameras). */
int ss_range_image_normals(const ss_camera* cam, const double* range, const uint8_t* valid, double* normal_out,
                           uint8_t* ok_out, void* stream);

/* One evaluation of _photo_system (registration.py:316-362) with Huber
 * weights: residuals of anchors X_w (M x 3 float64) against the scan range
 * image at pose T (row-major R then t), trimmed at
 * max(trim_factor * median|r|, trim_floor), reduced into out30 (host):
 *   [0:21] sum w J^T J (upper triangle, row-major), [21:27] sum w J^T r,
 *   [27] sum Huber(r), [28] kept count m, [29] sum r^2   (unnormalised).
 * objective_only = 1 skips the Jacobian (trial poses of the LM loop).
 * workspace: ss_photo_workspace_bytes(M) bytes.  Synchronises the stream. */
size_t ss_photo_workspace_bytes(int32_t M);
int ss_photo_system(const double* X_w, int32_t M, const double* scan_range, const uint8_t* scan_valid,
                    const ss_camera* cam, const double* T_Rt, double trim_floor, const ss_reg_cfg* cfg,
                    int32_t objective_only, double* out30, void* workspace, void* stream);

/* build_leaf_tree (registration.py:98-164) of n device points (float64 n x 3):
 * planar leaves of recursive PCA median splits, level-parallel on the device.
 * Leaf arrays (host, capacity max_leaves): centroids, normals oriented toward
 * viewpoint3 (zero when unusable), sizes, usable flags; point_leaf_out
 * (device, n) maps every point to its leaf.  workspace:
 * ss_leaf_tree_workspace_bytes(n).  Synchronises the stream (one small
 * read-back per tree level). */
size_t ss_leaf_tree_workspace_bytes(int32_t n);
int ss_leaf_tree_build(const double* pts, int32_t n, const double* viewpoint3, int32_t leaf_size, double tau,
                       int32_t max_leaves, double* centroids_out, double* normals_out, int32_t* sizes_out,
                       uint8_t* usable_out, int32_t* point_leaf_out, int32_t* n_leaves_out, void* workspace,
                       void* stream);

/* RegistrationConfig fields of the GN/LM loop (registration.py:41-61);
 * mode: 0 photometric, 1 geometric, 2 joint, 3 sequential. */
typedef struct {
  double huber_photo, huber_geo, trim_factor, spread_gate, assoc_gate, trim_floor_photo, trim_floor_geo, tol,
      damping_init, damping_max;
  int32_t max_iters, min_residuals, assoc_k, mode;
} ss_reg_solve_cfg;

/* The whole Gauss-Newton / Levenberg loop of register() (registration.py:
 * 437-524) on the device, one cooperative kernel, every mode: per
 * evaluation the geometric system (k nearest usable leaves within
 * assoc_gate -- found through a hash grid of gate-sized cells built on the
 * stream first --, closest plane, median trim; registration.py:231-274) and / or
 * the photometric one (_photo_system, :316-362), Huber-weighted 6x6 normal
 * equations, the damped solve, T <- T exp(delta), acceptance with the
 * reference's positional pairing of residual families and frozen terms
 * (:379-384), damping and trim-floor schedules, sequential phases.
 * Geometric inputs: usable leaf centroids / normals (n_leaves x 3 float64)
 * and the subsampled scan (n_geo_scan x 3, sensor frame); photometric:
 * world anchors X_w (M x 3) and the scan range image.  All device.
 * Returns the final pose (before the host's SVD re-orthonormalisation),
 * info6 = {iterations, converged, n_geo, n_photo, evaluations, status},
 * r2_out2 = sum r^2 of the last geometric / photometric systems.
 * SS_ERR_REGISTRATION when fewer than min_residuals residuals survive.
 * workspace: ss_reg_solve_workspace_bytes(n_leaves, n_geo_scan, M).  Synchronises. */
size_t ss_reg_solve_workspace_bytes(int32_t n_leaves, int32_t n_geo_scan, int32_t M);

/* Result record of one loop: final pose (row-major R | t, before the host's SVD
 * re-orthonormalisation), sum r^2 of the last geometric / photometric systems,
 * info = {iterations, converged, n_geo, n_photo, evaluations, status (!= 0: too few
 * residuals, the reference's RegistrationError)}. */
typedef struct {
  double T[12];
  double r2[2];
  int32_t info[6];
} ss_reg_out;

/* ss_reg_solve without the host synchronisation, for running several independent
 * registrations at once (frame batches, one stream each): the loop runs on `stream`
 * with at most max_blocks cooperative blocks (0: one per SM; with B concurrent loops,
 * num_SMs / B each, the grid barriers then span fewer blocks) and its ss_reg_out is
 * copied to out_host (pinned host memory; valid once the stream is synchronised).
 * Each concurrent call needs its own workspace. */
int ss_reg_solve_async(const double* leaf_centroids, const double* leaf_normals, int32_t n_leaves,
                       const double* geo_scan, int32_t n_geo_scan, const double* X_w, int32_t M,
                       const double* scan_range, const uint8_t* scan_valid, const ss_camera* cam,
                       const double* T0_Rt, const ss_reg_solve_cfg* cfg, int32_t max_blocks,
                       ss_reg_out* out_host, void* workspace, void* stream);

/* B photometric registrations against one model, each register(mode="photometric")
 * (registration.py:387-524, sample_model :190-213 with the [::thin] anchor subsample of
 * :430), enqueued from C with no host work between the frames: on streams[b], the model
 * render at geo_cam from poses0_Rt[12 b ...] (records recs[b]) and the range image of
 * scan b (scan_pts rows scan_offsets[b] .. scan_offsets[b+1], device, ready); then every
 * frame's anchors (waiting for its own render); then the B loops back to back, max_blocks
 * cooperative blocks each (they run concurrently), results to out_host[b] (pinned; info[5] = 2: too few confident
 * pixels).  Per-frame device buffers: render_buf (5 geo pixels floats), scan_range /
 * scan_valid (cam pixels), anchors (anchor_cap x 3), anchor_ws / solve_ws (the strides:
 * ss_anchor_workspace_bytes(geo), ss_reg_solve_workspace_bytes(0, 0, anchor_cap)).
 * Synchronises every stream before returning. */
int ss_register_photo_batch(int32_t B, const ss_camera* geo_cam, const ss_camera* cam, const ss_splats* splats,
                            const ss_raster_cfg* rcfg, ss_records* const* recs, void* const* streams,
                            const double* poses0_Rt, const double* scan_pts, const int32_t* scan_offsets,
                            int32_t thin, double vis_opacity, double spread_gate, const ss_reg_solve_cfg* cfg,
                            int32_t max_blocks, float* render_buf, double* scan_range, uint8_t* scan_valid,
                            double* anchors, int32_t anchor_cap, void* anchor_ws, size_t anchor_ws_stride,
                            void* solve_ws, size_t solve_ws_stride, ss_reg_out* out_host);
int ss_reg_solve(const double* leaf_centroids, const double* leaf_normals, int32_t n_leaves, const double* geo_scan,
                 int32_t n_geo_scan, const double* X_w, int32_t M, const double* scan_range,
                 const uint8_t* scan_valid, const ss_camera* cam, const double* T0_Rt, const ss_reg_solve_cfg* cfg,
                 double* T_out_Rt, int32_t* info6, double* r2_out2, void* workspace, void* stream);

/* Host-side staging of a float64 parameter array for upload (no GPU work): copies n values
 * from src into dst -- as float64, or rounded to nearest float32 when dst_f32 is non-zero
 * (the rounding the kernels' float32 parameters need; NULL dst: fingerprint only) -- and, unless
 * fp is NULL (conversion only; not both NULL), writes their content
 * fingerprint, a position-weighted wrapping sum whose weights depend on the global index
 * base + k, so chunks processed on different host threads add up.  Replaces the float32
 * conversion the drop-in does per call instead of the reference's direct use of the host
 * arrays (rasterizer.py:223-241 _splat_camera_arrays reads model.centers etc. each call). */
int ss_host_stage_f64(const double* src, void* dst, int32_t dst_f32, int64_t n, int64_t base, uint64_t* fp);

/* Measured FP32 FMA throughput of the current device (TFLOP/s), the roofline
 * denominator of the FP32-bound blend kernels.  Synchronises the stream. */
int ss_fp32_peak_tflops(double* tflops, void* stream);

const char* ss_version(void);

#ifdef __cplusplus
}
#endif
#endif
