/*
 * splat_b200.h -- C ABI of the B200 (sm_100a) differentiable Gaussian
 * splatting hot path (libsplat_b200.so).
 *
 * The reference (`splatgrad`, pure Python + numpy) exposes this path as
 * Python functions; there is no reference FFI.  Each entry point below is
 * the batched, device-side replacement of one reference function and cites
 * it (paths under /root/reference/pkg/src/splatgrad, "sg/").  The Python
 * package paper_2312_02121_b200 binds these with ctypes and re-exposes the
 * reference's own API names on top.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless marked [host].  The library
 *    never allocates device memory and never synchronizes the device; every
 *    call is stream-ordered on `stream` and reentrant.
 *  - Return value: 0 on success, -1 on a launch/argument error whose text is
 *    available from gs_last_error() (thread-local).
 *  - Per-element input errors of the reference (ValueError raised by
 *    sg/core.py:160-163,189-191, sg/projection.py:54-55,108-109) do not abort
 *    a kernel: they are folded into a device status word with atomicMin of
 *    ((uint64)index << 8 | code), initialised by the caller to
 *    GS_STATUS_OK (all ones).  The host wrapper raises ValueError naming the
 *    first offending Gaussian, as the reference does.
 *  - Float4 arrays must be 16-byte aligned.
 */
#ifndef SPLAT_B200_H
#define SPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gs_stream_t;

#define GS_TILE_SIZE 16 /* sg/binning.py:8 TILE_SIZE */
#define GS_STATUS_OK 0xFFFFFFFFFFFFFFFFull

enum gs_error_code {
    GS_OK = 0,
    GS_ERR_SCALE = 1,   /* sg/core.py:189-191 "scale components must be positive" */
    GS_ERR_QUAT = 2,    /* sg/core.py:160-163 "quaternion norm is too small ..." */
    GS_ERR_HOMOG = 3,   /* sg/projection.py:54-55 "degenerate projection ..." */
    GS_ERR_COV2D = 4,   /* sg/projection.py:108-109 "2d covariance must be positive definite" */
    GS_ERR_BEHIND = 5,  /* sg/projection.py:75-76 "point is behind the camera" */
};

/* Pinhole camera, the fields of sg/core.py:59-129 Camera (view row-major,
 * world->camera).  Passed by host pointer; copied into kernel parameters. */
typedef struct gs_camera {
    float view[16];
    float fx, fy, cx, cy;
    int32_t width, height;
    float near_plane, far_plane;
} gs_camera;

const char* gs_last_error(void);
int gs_version(void);
/* Process-wide tuning options.  "binning": the frame path's tile binning,
 * 0 = auto (direct for n <= 400000 Gaussians on <= 4096 tiles, scatter for
 * other n <= 400000, else depth-first),
 * 1 = depth-first (global stable depth sort, then tile sort of pairs emitted
 * in depth order), 2 = scatter (per-tile counts from the projection, pairs
 * written into their tile ranges through atomic cursors, each range sorted
 * by (depth, index)), 3 = direct (the projection writes every pair into its
 * tile's fixed-stride bin through an atomic slot counter; the raster
 * forward sorts each bin).  Both give sg/binning.py:50-65's (depth,
 * source_index) lists bit for bit.  "fuse_sort" (scatter binning): 1
 * (default) sorts each tile's range at the top of the raster forward CTA
 * that composites it, 0 in a separate per-tile sort kernel; same lists.
 * "tile_emit" (depth-first binning): 1 (default) writes every pair straight
 * to its slot in its tile's list (per-tile counts from the projection, one
 * stable counting pass over the depth-ordered Gaussians) when the tile count
 * fits its shared-memory tables (<= 9800 tiles), 0 emits the pairs and sorts
 * them by tile with onesweep passes; same lists. */
int gs_set_option(const char* name, int value);
/* Current value of an option of gs_set_option (-1 and gs_last_error for an
 * unknown name). */
int gs_get_option(const char* name);
/* Number of SMs of the current device (0 when no device). */
int gs_device_sm_count(void);

/* ---- Stage 1: projection ------------------------------------------------
 * Replaces sg/projection.py:115-145 project_gaussian as batched by
 * sg/raster_forward.py:246-252 _project_scene, plus the conic of
 * sg/raster_forward.py:86-92 _cov2d_inverse_terms.
 *   means3 (n,3), scales3 (n,3), quats4 (n,4) (w,x,y,z), opacities (n)
 * Outputs (n rows, culled rows have tiles_touched = 0 and radius 0):
 *   out_xydr4     (n,4): mean2d.x, mean2d.y, depth (camera z), radius (int bits)
 *   out_conic4    (n,4): A, B, C (inverse of cov2d), opacity
 *   out_tiles     (n)  : number of 16x16 tiles the bbox square touches
 *   out_cov3      (n,3): cov2d a, b, c (optional, may be NULL)
 *   status        (1)  : uint64 status word (see above)                     */
int gs_project_fwd(const float* means3, const float* scales3, const float* quats4,
                   const float* opacities, int64_t n, const gs_camera* cam /*[host]*/,
                   float* out_xydr4, float* out_conic4, uint32_t* out_tiles, float* out_cov3,
                   unsigned long long* status, gs_stream_t stream);

/* ---- Stage 2: tile binning + depth sort ---------------------------------
 * Together these replace sg/binning.py:27-47 assign_tiles and
 * sg/binning.py:50-65 sort_bins.
 * gs_scan_tiles: exclusive scan of tiles_touched -> offsets, total (uint64)
 * (single-pass decoupled look-back).                                        */
size_t gs_scan_workspace_bytes(int64_t n);
int gs_scan_tiles(const uint32_t* tiles, uint32_t* offsets, int64_t n, void* ws, size_t ws_bytes,
                  unsigned long long* total, gs_stream_t stream);

/* gs_emit_keys: for every visible Gaussian i (in index order) and every tile
 * (ty, tx) of its rectangle (row-major), writes
 *   key = (uint64)(ty*tiles_x+tx) << 32 | float_bits(depth), value = i
 * at offsets[i] + k.  Emission is in Gaussian-index order so a STABLE sort on
 * the key reproduces the reference's (depth, source_index) tie-break. */
int gs_emit_keys(const float* xydr4, const uint32_t* offsets, const uint32_t* tiles, int64_t n,
                 int32_t width, int32_t height, unsigned long long* keys, uint32_t* vals,
                 gs_stream_t stream);

/* gs_sort_pairs: stable LSD radix sort (8-bit digits, onesweep: one upfront
 * histogram + one chained-scan scatter per pass) of bits [0, end_bit).
 * Result lands in (keys, vals) if *selector == 0 else in (keys_alt,
 * vals_alt); *selector is written on the host, deterministically. */
size_t gs_sort_workspace_bytes(int64_t n, int end_bit);
int gs_sort_pairs(unsigned long long* keys, unsigned long long* keys_alt, uint32_t* vals,
                  uint32_t* vals_alt, int64_t n, int end_bit, void* ws, size_t ws_bytes,
                  int* selector /*[host]*/, gs_stream_t stream);

/* gs_tile_counts: tiles touched by arbitrary (mean2d, radius) squares given
 * as xydr4 rows (the input of sg/binning.py:27-47 assign_tiles when the
 * projected list comes from the caller rather than gs_project_fwd). */
int gs_tile_counts(const float* xydr4, int64_t n, int32_t width, int32_t height, uint32_t* out_tiles,
                   gs_stream_t stream);

/* gs_tile_ranges: per tile [start, end) into the sorted list (uint32 x 2,
 * zero-filled by the call for empty tiles). */
int gs_tile_ranges(const unsigned long long* sorted_keys, int64_t n, uint32_t* ranges2,
                   int32_t n_tiles, gs_stream_t stream);

/* ---- Stage 3: rasterize forward -----------------------------------------
 * Replaces sg/raster_forward.py:116-154 _composite_tile over the tiles of
 * sg/raster_forward.py:157-172,222-243.  Outputs HWC image (H,W,3), final_T
 * (H,W) and n_contrib (H,W) int32 (sg/raster_forward.py:43-55).
 * counts (optional, may be NULL; uint64[4], accumulated):
 *   E_f, E_f_sigma, E_f_alpha, E_f_commit                    */
int gs_raster_fwd(const uint32_t* ranges2, const uint32_t* sorted_vals, const float* xydr4,
                  const float* conic4, const float* colors3, const float* background3 /*[host]*/,
                  int32_t width, int32_t height, int early_termination, float* out_image,
                  float* out_final_T, int32_t* out_n_contrib, unsigned long long* counts,
                  gs_stream_t stream);

/* ---- Stage 4: rasterize backward ----------------------------------------
 * Replaces sg/raster_backward.py:47-108 _backward_tile summed as in
 * sg/raster_backward.py:166-205 accumulate_image_backward.  Accumulates
 * (atomically; buffers must be zeroed by the caller) per scene Gaussian:
 *   d_rgbo4 (n,4): d_color r, g, b, d_opacity
 *   d_geo4  (n,4): d_mean2d x, y, d_cov2d[0][0], d_cov2d[0][1] (= [1][0])
 *   d_c11   (n)  : d_cov2d[1][1]
 * counts (optional, uint64[3]): E_b, E_b_sigma, E_b_contrib.               */
int gs_raster_bwd(const uint32_t* ranges2, const uint32_t* sorted_vals, const float* xydr4,
                  const float* conic4, const float* colors3, const float* background3 /*[host]*/,
                  int32_t width, int32_t height, const float* final_T, const int32_t* n_contrib,
                  const float* d_image, float* d_rgbo4, float* d_geo4, float* d_c11,
                  unsigned long long* counts, gs_stream_t stream);

/* ---- Stage 5: projection backward ---------------------------------------
 * Replaces the per-Gaussian loop of sg/proj_backward.py:178-223
 * scene_backward (mean2d_backward :53-77, cov2d_backward :88-121,
 * world_backward :124-136, covariance3d_backward :151-175, view rotation
 * path :218-222).  Rows with tiles == 0 (culled) are written as exact 0.
 * d_view16 (4x4 row-major) is fully written (not accumulated); the sum over
 * Gaussians is deterministic (fixed-order block partials in ws).            */
size_t gs_project_bwd_workspace_bytes(int64_t n);
int gs_project_bwd(const float* means3, const float* scales3, const float* quats4, int64_t n,
                   const gs_camera* cam /*[host]*/, const uint32_t* tiles, const float* d_geo4,
                   const float* d_c11, float* d_means3, float* d_scales3, float* d_quats4,
                   float* d_view16, void* ws, size_t ws_bytes, gs_stream_t stream);

/* ---- Whole frame (sync-free orchestration of stages 1-5) ----------------
 * The production path.  Stage 2 is "depth-first": the Gaussians are sorted
 * once by depth (4 onesweep passes over N 32-bit keys), their tile pairs are
 * emitted in that order and stably sorted by tile id (1-2 passes over I
 * 32-bit keys) -- the same per-tile (depth, source_index) order as the
 * 64-bit keys above, with ~3-4x less sort traffic.
 * No host synchronisation, no allocation: intersections go into a caller-
 * chosen capacity; meta (device, 4 words) reports [0] the status word, [1]
 * the true total, [2] the capacity needed when it exceeds the total (direct
 * binning: every tile owns capacity / tiles slots, so tiles x the longest
 * list) and [3] the direct-binning tile stride (0: compact bins).  If
 * max(meta[1], meta[2]) > capacity the caller re-runs with a larger
 * workspace (results are not valid until it does).
 * forward  replaces sg/raster_forward.py:255-271 render;
 * backward replaces sg/proj_backward.py:178-223 scene_backward.          */
typedef struct gs_frame_view {
    float* xydr4;               /* (n,4) as gs_project_fwd out_xydr4 */
    float* conic4;              /* (n,4) as gs_project_fwd out_conic4 */
    uint32_t* tiles;            /* (n)   tiles touched, 0 = culled */
    uint32_t* depth_order;      /* (n)   Gaussian ids by (depth, index) (see depth_order_alt) */
    uint32_t* sorted_tile_keys; /* (capacity) tile id of each sorted pair -- written by scatter
                                   binning and by the depth-first binning with tile_emit 0 only;
                                   otherwise implied by ranges2 */
    uint32_t* sorted_vals;      /* (capacity) Gaussian id of each sorted pair */
    uint32_t* ranges2;          /* (tiles,2) [start, end) */
    unsigned long long* meta;   /* [0] status word, [1] total intersections, [2] capacity needed,
                                   [3] direct-binning tile stride (0: compact bins), [4] the forward
                                   zeroed the backward accumulators, [5,6] visible depth-key bits
                                   min / max, [7] visible Gaussians, [8] depth-sort passes */
    float* d_geo4;              /* (n,4) d_mean2d x,y, d_cov00, d_cov01 (after a backward run with
                                   accumulate bit 1 set; zeros otherwise), row stride 8 floats
                                   (interleaved with d_rgbo) */
    float* d_c11;               /* (n)   d_cov11 (idem) */
    void* bwd_accum;            /* the backward's atomic accumulators (d_rgbo/d_geo rows, d_c11).  Zero
                                   between frames: the projection backward clears every row it
                                   reads; gs_frame_forward zeroes them itself only when the
                                   workspace is not stamped clean for this layout */
    size_t bwd_accum_bytes;
    uint32_t* rec_count;        /* (tiles,4) forward commit records per (tile, 8x8 quadrant warp) */
    uint32_t* depth_order_alt;  /* depth-first binning: the visible Gaussians (meta[7] of them) by
                                   (depth, index) are in depth_order_alt when meta[8] (the depth-sort
                                   pass count) is odd, else in depth_order */
    uint32_t* touched;          /* (ceil(n/32)) bit i: the frame's raster backward added to Gaussian
                                   i's rows (cleared by every gs_frame_forward);
                                   gs_frame_views_project_backward reads only the marked rows.  A
                                   caller that writes the rows itself (e.g. sums them over ranks)
                                   sets every bit first */
} gs_frame_view;

size_t gs_frame_workspace_bytes(int64_t n, int64_t isect_capacity, int32_t width, int32_t height);
/* Mark a freshly allocated (or re-purposed) workspace as not clean: the next
 * gs_frame_forward then zeroes the backward accumulators itself.  Call it
 * once per allocation; a workspace kept across frames of one layout needs
 * nothing more (a stale layout is detected by its signature).              */
int gs_frame_workspace_init(int64_t n, int64_t isect_capacity, int32_t width, int32_t height, void* ws,
                            gs_stream_t stream);
/* The binning gs_frame_forward uses for n Gaussians on a width x height
 * view under the current options: 1 depth-first, 2 scatter, 3 direct. */
int gs_frame_binning(int64_t n, int32_t width, int32_t height);
/* 1 when such a frame's depth-first binning writes its pairs with the
 * tile-sorted emission (option "tile_emit", <= 9800 tiles), else 0. */
int gs_frame_tile_emit(int64_t n, int32_t width, int32_t height);
int gs_frame_view_of(int64_t n, int64_t isect_capacity, int32_t width, int32_t height, void* ws,
                     gs_frame_view* out /*[host]*/);
int gs_frame_forward(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                     const float* colors3, int64_t n, const gs_camera* cam /*[host]*/,
                     const float* background3 /*[host]*/, int early_termination, int64_t isect_capacity,
                     void* ws, size_t ws_bytes, float* out_image, float* out_final_T, int32_t* out_n_contrib,
                     unsigned long long* counts4, void* const* stage_events, gs_stream_t stream);
/* Multi-view steps: the projection of every view (each on its own
 * workspace, all using depth-first binning) in one pass that reads each
 * Gaussian once (40 + 44/n_views instead of 84 bytes per Gaussian and view),
 * then per view gs_frame_forward_projected = gs_frame_forward without its
 * projection (same arguments; no counted pass).  cams / capacities /
 * workspaces / ws_bytes: [host] n_views entries. */
int gs_frames_project(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                      int64_t n, int32_t n_views, const gs_camera* cams /*[host]*/,
                      const int64_t* capacities /*[host]*/, void* const* workspaces /*[host]*/,
                      const size_t* ws_bytes /*[host]*/, gs_stream_t stream);
int gs_frame_forward_projected(const float* means3, const float* scales3, const float* quats4,
                               const float* opacities, const float* colors3, int64_t n,
                               const gs_camera* cam /*[host]*/, const float* background3 /*[host]*/,
                               int early_termination, int64_t isect_capacity, void* ws, size_t ws_bytes,
                               float* out_image, float* out_final_T, int32_t* out_n_contrib,
                               void* const* stage_events, gs_stream_t stream);
/* stage_events (nullable; entries nullable): cudaEvent_t handles recorded
 * on `stream` at stage boundaries, for live per-stage timing.
 *   forward : [0] start [1] projected [2] depth-sorted [3] emitted [4] tile-sorted+ranges [5] rastered
 *   backward: [0] start [1] raster backward done [2] projection backward done
 * d_rgbo4 (n,4) = d_color r,g,b, d_opacity; d_view16 4x4 (always written).
 * accumulate bit 0 clear: d_means3 / d_scales3 / d_quats4 / d_rgbo4 are
 * overwritten; set: this view's gradients are ADDED to them (sum over the
 * views of a step without extra kernels, sg/proj_backward.py:178-223 summed
 * per camera).  Bit 1 set: leave the screen-space gradients readable in the
 * workspace (gs_frame_view d_geo4 / d_c11; the next forward re-zeroes them);
 * clear (default): the projection backward zeroes them as it reads them.
 * Bit 2 set: stage_events has a 4th entry, an event `stream` waits on before
 * the projection backward (a multi-view step serialises only the views'
 * read-modify-write accumulation; their raster backwards may overlap).
 * Bit 3 set: raster backward only -- the screen-space gradients stay in the
 * workspace (gs_frame_view d_geo4 rows + d_c11, d_rgbo in the first half of
 * each row) for a reduction across ranks, then gs_frame_project_backward. */
int gs_frame_backward(const float* means3, const float* scales3, const float* quats4, const float* colors3,
                      int64_t n, const gs_camera* cam /*[host]*/, const float* background3 /*[host]*/,
                      int64_t isect_capacity, void* ws, size_t ws_bytes, const float* final_T,
                      const int32_t* n_contrib, const float* d_image, float* d_means3, float* d_scales3,
                      float* d_quats4, float* d_rgbo4, float* d_view16, int accumulate,
                      unsigned long long* counts3, void* const* stage_events, gs_stream_t stream);

/* The projection backward of a frame (the second half of gs_frame_backward,
 * sg/proj_backward.py:178-223) over the Gaussians [begin, end), from the
 * screen-space gradients in the workspace (after gs_frame_backward with
 * bit 3, possibly summed across ranks in place).  Outputs are indexed by
 * scene Gaussian (rows begin..end-1 written).  flags: bit 0 add into the
 * outputs, bit 1 keep the screen-space rows (else cleared as read), bit 4
 * add this range's d_view into d_view16 (else overwrite), bit 5 treat a
 * Gaussian as visible when its screen-space row is non-zero even if this
 * frame culled it (rows summed over tile bands of one frame).  Ranges let a
 * caller start reducing finished Gaussian buckets while later ones run.   */
int gs_frame_project_backward(const float* means3, const float* scales3, const float* quats4, int64_t n,
                              const gs_camera* cam /*[host]*/, int64_t isect_capacity, void* ws, size_t ws_bytes,
                              int64_t begin, int64_t end, float* d_means3, float* d_scales3, float* d_quats4,
                              float* d_rgbo4, float* d_view16, int flags, gs_stream_t stream);
/* The projection backward of all views of a multi-view step at once
 * (sg/proj_backward.py:178-223 per view, summed over the views): after each
 * view's gs_frame_backward with flag bit 3 (raster backward only; every view
 * on its own workspace), one pass over Gaussians [begin, end) reads the
 * parameters once and every view's screen-space gradient rows that view's
 * raster backward marked (gs_frame_view.touched; unmarked rows are zero), and writes
 * (flag bit 0: adds to) d_means3 / d_scales3 / d_quats4 / d_rgbo4 the sums
 * over the views, and d_views16 (n_views x 16, flag bit 4: added) per view.
 * Adding continues each row's running sum in view order (the row's current
 * value first), so views split over several calls give bit-identical sums.
 * A Gaussian counts as visible in a view iff it is marked there (a culled
 * one is never marked; marked zero rows contribute exactly zero).
 * The rows read are cleared unless flag bit 1 keeps them; the call whose
 * range ends at n stamps each workspace clean (its rows all cleared: calls
 * over earlier ranges must not keep theirs) or, keeping, not clean.  cams / capacities / workspaces / ws_bytes: [host] n_views
 * entries, as given to each view's gs_frame_forward.  Against
 * gs_frame_backward per view it moves ~76 instead of ~224 bytes per visible
 * Gaussian and view (parameters read once, sums written once). */
int gs_frame_views_project_backward(const float* means3, const float* scales3, const float* quats4, int64_t n,
                                    int32_t n_views, const gs_camera* cams /*[host]*/,
                                    const int64_t* capacities /*[host]*/, void* const* workspaces /*[host]*/,
                                    const size_t* ws_bytes /*[host]*/, int64_t begin, int64_t end,
                                    float* d_means3, float* d_scales3, float* d_quats4, float* d_rgbo4,
                                    float* d_views16, int flags, gs_stream_t stream);

/* ---- Training step around the path (sg/optimize.py:96-190 fit) ----------
 * gs_activate : scales = exp(log_scales), opacities = sigmoid(logits)  (:144-145)
 * gs_loss_l2  : d_image = 2 (image - target); *loss += sum (image - target)^2
 *               (fp64 accumulation; :157-158,163)
 * gs_adam_step: chain rule to log/logit space (:167,172), Adam per class
 *               (:84-89) with lrs5 = {mean, scale, quat, opacity, color},
 *               colour clip (:176), and the activated scales/opacities for
 *               the next render.  adam_m14/adam_v14: (n,14) moments, column
 *               order mean 3 | log_scale 3 | quat 4 | logit 1 | color 3.    */
int gs_activate(const float* log_scales3, const float* logits, float* scales3, float* opacities, int64_t n,
                gs_stream_t stream);
int gs_loss_l2(const float* image, const float* target, int64_t n, float* d_image, double* loss,
               gs_stream_t stream);
int gs_adam_step(float* means3, float* log_scales3, float* quats4, float* logits, float* colors3, float* scales3,
                 float* opacities, const float* d_means3, const float* d_scales3, const float* d_quats4,
                 const float* d_rgbo4, float* adam_m14, float* adam_v14, int64_t n, int step,
                 const float* lrs5 /*[host]*/, float beta1, float beta2, float eps, gs_stream_t stream);

/* ---- Per-pixel API -------------------------------
 * Splat arrays are the projection's layout: xydr4 (m,4) (x, y, depth,
 * radius bits; only x, y are read), conic4 (m,4) (A, B, C, opacity),
 * colors3 (m,3).  A query is a pixel centre pix2[q] and, for compositing,
 * its own depth-ordered bin bin_idx[bin_ptr[q] .. bin_ptr[q+1]) of splat
 * indices.  The arithmetic is the tile rasterizers' (bit-identical image /
 * final_T / n_contrib for a rendered pixel's centre and tile bin).
 *
 * gs_conic_from_cov      replaces sg/raster_forward.py:86-92
 *                        _cov2d_inverse_terms: cov3 (m,3) = (a, b, c) of
 *                        the 2d covariance; det <= 0 reports GS_ERR_COV2D
 *                        for the first such row into *status (atomicMin of
 *                        index<<8 | code; initialise to all ones).
 * gs_eval_alpha          replaces sg/raster_forward.py:175-196 eval_alpha
 *                        for n (splat[q], pix2[q]) pairs.
 * gs_composite_pixels    replaces sg/raster_forward.py:199-219
 *                        composite_pixel for n queries.
 * gs_composite_pixels_bwd replaces sg/raster_backward.py:111-135
 *                        composite_pixel_backward (gradients accumulate into
 *                        zeroed d_rgbo4 / d_geo4 / d_c11 rows per splat, the
 *                        gs_raster_bwd layout) and, with t_log != NULL
 *                        (sized like bin_idx), :138-163 transmittance_replay:
 *                        the replayed T before every contributing entry, NaN
 *                        at the others.                                      */
int gs_conic_from_cov(const float* cov3, const float* opacities, int64_t n, float* out_conic4,
                      unsigned long long* status, gs_stream_t stream);
int gs_eval_alpha(const float* xydr4, const float* conic4, const int32_t* splat, const float* pix2, int64_t n,
                  float* out_alpha, float* out_delta2, float* out_sigma, gs_stream_t stream);
int gs_composite_pixels(const float* xydr4, const float* conic4, const float* colors3, const int64_t* bin_ptr,
                        const int32_t* bin_idx, const float* pix2, int64_t n, const float* background3 /*[host]*/,
                        int early_termination, float* out_color3, float* out_final_T, int32_t* out_n_contrib,
                        gs_stream_t stream);
int gs_composite_pixels_bwd(const float* xydr4, const float* conic4, const float* colors3, const int64_t* bin_ptr,
                            const int32_t* bin_idx, const float* pix2, int64_t n,
                            const float* background3 /*[host]*/, const float* final_T, const int32_t* n_contrib,
                            const float* d_pixels3, float* d_rgbo4, float* d_geo4, float* d_c11, float* t_log,
                            gs_stream_t stream);

/* ---- The path in float64 --------------------------
 * For the reference's finite-difference audit (sg/gradcheck.py) and fp64
 * parity: the same stages with every value in double, each following the
 * reference's expression order.  Host-synchronous in one place (the caller
 * reads the intersection total after gs_bin64_count).
 *
 * gs_project64     sg/projection.py:115-145 per Gaussian: mean2d (n,2),
 *                  cov3 (n,3) = (a, b, c), depth, radius, tiles touched
 *                  (0 = culled), depth sort key; errors into *status as
 *                  gs_project_fwd.
 * gs_bin64_count   exclusive scan of tiles -> *out_total (device uint64).
 * gs_bin64_sort    sg/binning.py:27-65: (depth, source_index) order, then
 *                  per-tile lists (ranges2 (n_tiles,2) + *out_vals pointing
 *                  into ws) -- same ws as gs_bin64_count, sized by
 *                  gs_bin64_workspace_bytes(n, n_isect, n_tiles).
 * gs_raster64_fwd  sg/raster_forward.py:116-172 (thread per pixel).
 * gs_raster64_bwd  sg/raster_backward.py:47-108,166-205: d9 (n,9) zeroed,
 *                  accumulates d_color 3, d_opacity, d_mean2d 2, d_cov2d
 *                  00, 01 (= 10), 11 per Gaussian.
 * gs_project64_bwd sg/proj_backward.py:178-223 (d_view16 fixed order).     */
typedef struct gs_camera64 {
    double view[16];
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane, far_plane;
} gs_camera64;

int gs_project64(const double* means3, const double* scales3, const double* quats4, int64_t n,
                 const gs_camera64* cam /*[host]*/, double* out_mean2d, double* out_cov3, double* out_depth,
                 int32_t* out_radius, uint32_t* out_tiles, unsigned long long* out_dkeys,
                 unsigned long long* status, gs_stream_t stream);
size_t gs_bin64_workspace_bytes(int64_t n, int64_t n_isect, int32_t n_tiles);
int gs_bin64_count(const uint32_t* tiles, int64_t n, void* ws, size_t ws_bytes, unsigned long long* out_total,
                   gs_stream_t stream);
int gs_bin64_sort(const double* mean2d, const int32_t* radius, const uint32_t* tiles,
                  const unsigned long long* dkeys, int64_t n, int64_t n_isect, int32_t width, int32_t height,
                  void* ws, size_t ws_bytes, uint32_t* out_ranges2, const uint32_t** out_vals /*[host]*/,
                  gs_stream_t stream);
int gs_raster64_fwd(const uint32_t* ranges2, const uint32_t* vals, const double* mean2d, const double* cov3,
                    const double* opacities, const double* colors3, const double* background3 /*[host]*/,
                    int32_t width, int32_t height, int early_termination, double* out_image, double* out_final_T,
                    int32_t* out_n_contrib, gs_stream_t stream);
int gs_raster64_bwd(const uint32_t* ranges2, const uint32_t* vals, const double* mean2d, const double* cov3,
                    const double* opacities, const double* colors3, const double* background3 /*[host]*/,
                    int32_t width, int32_t height, const double* final_T, const int32_t* n_contrib,
                    const double* d_image, double* d9, gs_stream_t stream);
size_t gs_project64_bwd_workspace_bytes(int64_t n);
int gs_project64_bwd(const double* means3, const double* scales3, const double* quats4, int64_t n,
                     const gs_camera64* cam /*[host]*/, const uint32_t* tiles, const double* d9, double* d_means3,
                     double* d_scales3, double* d_quats4, double* d_view16, void* ws, size_t ws_bytes,
                     gs_stream_t stream);

/* ---- Per-splat helpers in float64 (the rest of sg/__init__.py:64-119) ---
 * gs_op64 runs one helper over n items (one thread each); `in` / `out` are
 * HOST arrays of device pointers, row-major matrices, items contiguous.
 * Errors (degenerate inputs) go to *status as index << 8 | gs_error_code.   */
enum gs_op64_code {
    GS_OP_QUAT_TO_ROTMAT = 1,      /* sg/core.py:146-171        q4 -> R9 */
    GS_OP_COMPOSE_COV3D = 2,       /* sg/core.py:174-195        q4, s3 -> R9, S9, M9, sigma9 */
    GS_OP_FROBENIUS = 3,           /* sg/core.py:198-204        x[cols], y[cols] -> sum x*y */
    GS_OP_WORLD_TO_CAMERA = 4,     /* sg/projection.py:36-42    mean3 -> t4 (camera) */
    GS_OP_CAMERA_TO_PIXEL = 5,     /* sg/projection.py:45-61    t4 -> mean2d2 (camera) */
    GS_OP_PROJECTION_JACOBIAN = 6, /* sg/projection.py:64-82    t4 -> J6 (camera) */
    GS_OP_PROJECT_COVARIANCE = 7,  /* sg/projection.py:85-96    J6, Rcw9, sigma9 -> cov2d4 */
    GS_OP_BOUNDING_RADIUS = 8,     /* sg/projection.py:99-112   cov2d4 -> r (integral double) */
    GS_OP_MEAN2D_BACKWARD = 9,     /* sg/proj_backward.py:53-77  dmean2d2, t4 -> dt4 (camera) */
    GS_OP_COV2D_BACKWARD = 10,     /* sg/proj_backward.py:88-121 G4, T6, sigma9, J6, Rcw9, t4 -> dsigma9, dt4 */
    GS_OP_WORLD_BACKWARD = 11,     /* sg/proj_backward.py:124-136 dt4, mean3 -> dmean3, dview16 (camera) */
    GS_OP_COV3D_BACKWARD = 12,     /* sg/proj_backward.py:151-175 dsigma9, R9, S9, M9, q4 -> dq4, ds3 */
};
int gs_op64(int op, int64_t n, const double* const* in /*[host]*/, double* const* out /*[host]*/, int32_t cols,
            const gs_camera64* cam /*[host], nullable*/, unsigned long long* status, gs_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SPLAT_B200_H */
