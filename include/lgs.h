/*
 * lgs.h -- C ABI of the B200-native LEGO-SLAM splat rasterizer (liblgs.so).
 *
 * Drop-in boundary for the reference renderer, proj/include/legoslam/renderer.hpp:
 *
 *   lego::project_gaussian   renderer.hpp:49-53  -> lgs_debug_projected
 *   lego::render             renderer.hpp:55-56  -> lgs_render_forward
 *   lego::render_backward    renderer.hpp:72-74  -> lgs_render_backward
 *   lego::RenderConfig       renderer.hpp:15-22  -> lgs_render_config
 *   lego::RenderOutput       renderer.hpp:33-45  -> lgs_images (images) + lgs_saved (backward tape)
 *   lego::MapGradients       renderer.hpp:59-68  -> lgs_map_grads
 *   lego::GaussianMap (SoA)  gaussian_map.hpp:57-93 -> lgs_gaussians (reference layouts) / lgs_map (device)
 *   lego::Pose + CameraIntrinsics geometry.hpp:18-29, 43-52 -> lgs_camera
 *
 * The reference ships no C API (proj/src/capi.cpp is a one-line placeholder), so this
 * header is the first C binding of these entry points; INTEGRATION.md shows the C++
 * shim with the exact lego:: signatures and the ctypes binding.
 *
 * Conventions (all mirror the reference):
 *  - Buffers are plain pointers; `memory` says whether they are host or device memory.
 *  - Map layouts: positions [N][3]; rotations [N][4] in Eigen storage order (x,y,z,w);
 *    log_scales [N][3]; opacity_logits [N]; sh [N][K][3] with K = (sh_degree+1)^2, K = 1 being
 *    the reference `colors`; features [d][N] (the column-major N x d Eigen matrix).
 *  - Images are row-major, channel-interleaved HWC (image.hpp:22-34).
 *  - Gradients are dense over the map, zero for culled Gaussians (renderer.cpp:185-186);
 *    rotation gradients are ordered (w,x,y,z) (renderer.hpp:61); feature gradients [d][N].
 *  - A NULL cotangent is the reference's empty image (= zero, renderer.hpp:70-71).
 *  - No exceptions cross the ABI: every call returns an lgs_status.  The reference's only
 *    thrown error, std::invalid_argument on a cotangent shape mismatch (renderer.cpp:176-178),
 *    is LGS_EINVAL.
 *  - All work is enqueued on the context's stream; calls are asynchronous with respect to the
 *    host unless a host buffer is involved (then the call synchronizes before returning).
 *  - Thread safety: one lgs_ctx per host thread / GPU.  Renders are pure w.r.t. the map, so
 *    several contexts may render the same lgs_map concurrently.
 */
#ifndef LGS_H_
#define LGS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define LGS_API __declspec(dllexport)
#else
#define LGS_API __attribute__((visibility("default")))
#endif

typedef enum {
  LGS_OK = 0,
  LGS_EINVAL = 1, /* bad argument / shape mismatch (reference: std::invalid_argument) */
  LGS_ECUDA = 2,  /* CUDA runtime error; see lgs_last_error() */
  LGS_ENOMEM = 3, /* device or host allocation failed */
  LGS_ENODEV = 4, /* no usable sm_100 device */
  LGS_EIO = 5     /* map file error (reference: lego::IoError, errors.hpp:21) */
} lgs_status;

enum { LGS_MEM_HOST = 0, LGS_MEM_DEVICE = 1, LGS_MEM_HOST_MAPPED = 2 };
/* LGS_MEM_HOST_MAPPED (lgs_gaussians only): page-locked host memory (cudaHostAlloc /
 * cudaHostRegister, device-addressable under UVA) that the device reads in place where few rows
 * are needed.  Positions, rotations, scales and opacities are copied as for LGS_MEM_HOST; the SH
 * coefficients and the features are NOT: with the depth-layered binning only the listed Gaussians'
 * rows cross PCIe (their colours and features are fetched where they are first listed).  The
 * caller keeps the buffers alive and unchanged while the map and its tapes are in use (no
 * synchronization at create/update).  Render-only: Adam, download and save reject such a map. */

enum { LGS_TILE = 16, LGS_MAX_FEATURE_DIM = 32, LGS_MAX_SH_DEGREE = 3 };

typedef struct lgs_ctx lgs_ctx;
typedef struct lgs_map lgs_map;
typedef struct lgs_saved lgs_saved;
typedef struct lgs_adam lgs_adam;
typedef struct lgs_plan lgs_plan;

/* renderer.hpp:15-22; defaults from lgs_render_config_default(). */
typedef struct {
  double near_plane;        /* 0.01; must be >= 0 */
  double dilation;          /* 0.3 px^2 */
  double alpha_clamp;       /* 0.99 */
  double alpha_skip;        /* 1/255 */
  double transmittance_min; /* 1e-4 */
  double radius_sigma;      /* 3.0 */
} lgs_render_config;

/* cam_pose is world<-camera (gaussian_map.hpp:30): q = (w,x,y,z), normalized by the callee
 * like Pose(q, t) (geometry.hpp:23). */
typedef struct {
  double q[4];
  double t[3];
  double fx, fy, cx, cy;
  int32_t width, height;
} lgs_camera;

/* The map in the reference's logical layouts. */
typedef struct {
  int64_t n;
  int32_t feature_dim; /* d, 0..LGS_MAX_FEATURE_DIM */
  int32_t sh_degree;   /* 0..3 */
  const float* positions;      /* [N][3] */
  const float* rotations;      /* [N][4] x,y,z,w */
  const float* log_scales;     /* [N][3] */
  const float* opacity_logits; /* [N] */
  const float* sh;             /* [N][K][3] */
  const float* features;       /* [d][N] */
  int32_t memory;              /* LGS_MEM_HOST / LGS_MEM_DEVICE / LGS_MEM_HOST_MAPPED */
} lgs_gaussians;

/* Caller-owned output images, HWC.  Any pointer may be NULL (not written). */
typedef struct {
  float* rgb;   /* [H][W][3] */
  float* depth; /* [H][W], alpha-normalized (renderer.cpp:163-165) */
  float* feat;  /* [H][W][d] */
  float* acc;   /* [H][W] */
  int32_t memory;
} lgs_images;

/* Dense gradients (MapGradients, renderer.hpp:59-68).  NULL members are skipped. */
typedef struct {
  float* position;      /* [N][3] */
  float* rotation;      /* [N][4] w,x,y,z */
  float* log_scale;     /* [N][3] */
  float* opacity_logit; /* [N] */
  float* sh;            /* [N][K][3]; K = 1: the reference colour gradient */
  float* feature;       /* [d][N] */
  int32_t memory;
  int32_t accumulate; /* 0: overwrite (reference semantics); 1: add into (multi-view batches) */
} lgs_map_grads;

/* Optional fused L1 loss: targets HWC; when given to lgs_render_forward the
 * forward also writes the cotangents of L = mean|rgb-T| + mean|depth-T| + mean|feat-T|
 * (sign(0) = 0) into the tape, and lgs_render_backward_l1 consumes them. */
typedef struct {
  const float* rgb;   /* [H][W][3] */
  const float* depth; /* [H][W] */
  const float* feat;  /* [H][W][d] */
  int32_t memory;
} lgs_l1_targets;

/* Per-render counters (parity / roofline bookkeeping). */
typedef struct {
  int64_t visible;        /* V: Gaussians that survived culling */
  int64_t pairs;          /* P: (tile, Gaussian) pairs */
  int64_t tiles;          /* number of 16x16 tiles */
  int64_t max_tile_list;  /* longest per-tile list */
  int64_t listed;         /* entries the tile lists hold: P with complete lists; with the depth-layered
                             binning, saturated tiles keep only the prefix their pixels can reach */
  int64_t active;         /* Gaussians whose gradient rows the backward computes (listed in a traversed
                             tile list; = visible with complete lists); every other row is zero */
  int64_t host_rows;      /* LGS_MEM_HOST_MAPPED maps: Gaussians whose SH row and features this render
                             read in place over PCIe (0 when it copied the SH and feature blocks in bulk:
                             an uncaptured render does when the previous render of the same host map
                             listed more than 1/64 of it, or lists every Gaussian) */
} lgs_render_stats;

/* ---- library / context ---------------------------------------------------------------- */
LGS_API const char* lgs_version(void);
LGS_API const char* lgs_last_error(void); /* thread-local message of the last failure */
LGS_API lgs_render_config lgs_render_config_default(void);

/* One CUDA stream + device arena per context.  `stream` may be NULL (the context creates its
 * own non-blocking stream) or an existing cudaStream_t to enqueue on (e.g. torch's). */
LGS_API lgs_status lgs_ctx_create(int32_t device, void* stream, lgs_ctx** out);
LGS_API lgs_status lgs_ctx_destroy(lgs_ctx* ctx);
/* Binning policy of the context's renders (default 0).  0: depth-layered binning -- the tile lists
 * hold, per tile, the depth-order prefix its pixels can reach before saturating (T < T_min,
 * renderer.cpp:140), completed for tiles that do not saturate; images and gradients are identical.
 * 1: every (tile, Gaussian) pair is listed (parity checks of the complete sorted lists). */
LGS_API lgs_status lgs_ctx_set_full_tile_lists(lgs_ctx* ctx, int32_t full);
/* Context options (the library reads no environment variables):
 *   LGS_OPT_FULL_TILE_LISTS    same as lgs_ctx_set_full_tile_lists;
 *   LGS_OPT_RADIX_DEPTH_ORDER  1: the depth order by a device radix sort over (depth, index) keys
 *                              with complete lists (cross-check of the bucketed order; same result);
 *   LGS_OPT_FUSED_EAGER        1: an uncaptured render with L1 targets runs the fused forward+backward
 *                              kernel of lgs_plan (for profilers that cannot see inside a graph); its
 *                              tape accepts only lgs_render_backward_l1 / _loss (else LGS_EINVAL);
 *   LGS_OPT_HOST_GRAD_DELTA    1: host gradient buffers (lgs_map_grads.memory = LGS_MEM_HOST, not
 *                              accumulating) that the caller passes again unchanged to the next
 *                              backward on this context are rewritten row-sparse: only the rows
 *                              nonzero now cross the link, the rows nonzero last time are zeroed
 *                              on the host; the buffers hold the exact dense MapGradients after
 *                              every call.  The first call (or new buffers) writes densely.  The
 *                              caller must not modify the buffers between calls;
 *   LGS_OPT_SPECULATIVE_PLANS  1 (default): a non-accumulating lgs_plan whose warm-up render
 *                              saturated every tile on its layer-A list is captured without the
 *                              layered binning's second pass (lgs_plan_speculative); 0: always
 *                              with it. */
enum {
  LGS_OPT_FULL_TILE_LISTS = 0,
  LGS_OPT_RADIX_DEPTH_ORDER = 1,
  LGS_OPT_FUSED_EAGER = 2,
  LGS_OPT_HOST_GRAD_DELTA = 3,
  LGS_OPT_SPECULATIVE_PLANS = 4
};
LGS_API lgs_status lgs_ctx_set_option(lgs_ctx* ctx, int32_t option, int64_t value);
LGS_API lgs_status lgs_ctx_set_stream(lgs_ctx* ctx, void* stream);
/* Bytes the context has copied host->device and device->host since creation (map uploads,
 * targets, cotangents, images, gradients; reads of LGS_MEM_HOST_MAPPED memory are not copies). */
LGS_API lgs_status lgs_ctx_transfer_bytes(const lgs_ctx* ctx, int64_t* h2d, int64_t* d2h);
LGS_API lgs_status lgs_ctx_synchronize(lgs_ctx* ctx);
/* Depth-layered binning: layer A of the context's next render takes ~1/div of the (tile, Gaussian)
 * pairs (at most n / (2 div) Gaussians).  div starts at 16 and adapts between uncaptured renders
 * from the previous render's counters: x1/2 when more than a quarter of the tiles needed the
 * second pass, x4 when fewer than 2% did and the tiles consumed less than 1/16 of their lists
 * (views whose near splats cover most tiles).  Results do not depend on it; diagnostics only. */
LGS_API int32_t lgs_ctx_layer_div(const lgs_ctx* ctx);

/* ---- device-resident map (K9 pack: reference layouts -> device SoA) ------------------- */
LGS_API lgs_status lgs_map_create(lgs_ctx* ctx, const lgs_gaussians* src, lgs_map** out);
/* Re-upload attribute values (same n, d, sh_degree). */
LGS_API lgs_status lgs_map_update(lgs_ctx* ctx, lgs_map* map, const lgs_gaussians* src);
LGS_API lgs_status lgs_map_destroy(lgs_map* map);
LGS_API int64_t lgs_map_size(const lgs_map* map);

/* ---- forward (lego::render) ------------------------------------------------------------
 * Renders `map` from `cam`.  `targets` may be NULL.  On success *tape receives a new
 * lgs_saved (free with lgs_saved_destroy) unless tape == NULL. */
LGS_API lgs_status lgs_render_forward(lgs_ctx* ctx, const lgs_map* map, const lgs_camera* cam,
                                      const lgs_render_config* cfg, const lgs_l1_targets* targets,
                                      lgs_images* out, lgs_saved** tape);

/* Convenience drop-in for lego::render(const GaussianMap&, ...): uploads `src` (reference
 * layouts, host or device) into a map owned by the returned tape. */
LGS_API lgs_status lgs_render(lgs_ctx* ctx, const lgs_gaussians* src, const lgs_camera* cam,
                              const lgs_render_config* cfg, lgs_images* out, lgs_saved** tape);

/* ---- backward (lego::render_backward) --------------------------------------------------
 * Cotangents are HWC with the reference's shapes; `cot_memory` says where they live.  Shape
 * checking is by construction (H, W, d come from the tape); pass cot_height/width/channels of
 * the caller's images to reproduce the reference's std::invalid_argument (LGS_EINVAL).
 * `pose_grad` (6 floats, host; NULL = skip) receives dL/dxi at xi = 0 for
 * cam_pose <- compose(se3_exp(xi), cam_pose), xi = (omega, nu). */
typedef struct {
  const float* rgb;   /* [H][W][3] or NULL */
  const float* depth; /* [H][W] or NULL */
  const float* feat;  /* [H][W][d] or NULL */
  int32_t memory;
  int32_t rgb_shape[3];   /* H, W, C of the caller's image (0,0,0 = trust) */
  int32_t depth_shape[3];
  int32_t feat_shape[3];
} lgs_cotangents;

LGS_API lgs_status lgs_render_backward(lgs_ctx* ctx, const lgs_saved* tape, const lgs_cotangents* cot,
                                       lgs_map_grads* grads, float* pose_grad);
/* Backward of the fused L1 loss recorded by lgs_render_forward(targets != NULL). */
LGS_API lgs_status lgs_render_backward_l1(lgs_ctx* ctx, const lgs_saved* tape, lgs_map_grads* grads,
                                          float* pose_grad);
/* L1 loss value of the last forward with targets (host float; synchronizes). */
LGS_API lgs_status lgs_saved_l1_loss(lgs_ctx* ctx, const lgs_saved* tape, double* loss);
LGS_API lgs_status lgs_saved_stats(const lgs_saved* tape, lgs_render_stats* stats);
LGS_API lgs_status lgs_saved_destroy(lgs_saved* tape);

/* ---- parity / debug exports (used by the bit-exact tests) ------------------------------ */
/* Per map index: visible flag, u, v, depth, conic (A, B, C with q = A dx^2 + 2B dx dy + C dy^2),
 * radius, pixel rect (x0, x1, y0, y1), opacity, colour.  Host buffers, each length N (x3/x4). */
LGS_API lgs_status lgs_debug_projected(lgs_ctx* ctx, const lgs_saved* tape, uint8_t* visible, float* u,
                                       float* v, float* depth, float* conic, float* radius, int32_t* bbox,
                                       float* opacity, float* color);
/* Sorted tile key lists, concatenated in tile order: keys = (tile << 32) | f32bits(depth),
 * vals = map index, ranges [tiles][2] = [begin, end).  Host buffers; keys/vals of length
 * lgs_render_stats.listed (= pairs with lgs_ctx_set_full_tile_lists(ctx, 1)). */
LGS_API lgs_status lgs_debug_tile_keys(lgs_ctx* ctx, const lgs_saved* tape, uint64_t* keys, uint32_t* vals,
                                       uint32_t* ranges);
/* Per pixel: final transmittance and contributor-list end (index into the tile list,
 * relative to the tile's begin). Host buffers of H*W. */
LGS_API lgs_status lgs_debug_pixel_state(lgs_ctx* ctx, const lgs_saved* tape, float* final_t,
                                         uint32_t* n_contrib);

/* ---- multi-view helpers ------------------------------------------------------------------
 * Size (floats) of one flat fp32 gradient buffer holding a whole MapGradients back to back in the
 * order position | rotation | log_scale | opacity_logit | sh | feature.  Point an lgs_map_grads
 * into it (accumulate = 1 across the rank's views) and all-reduce it once (NCCL, sum). */
LGS_API int64_t lgs_grads_flat_size(int64_t n, int32_t feature_dim, int32_t sh_degree);

/* Kernel launches issued by this context since creation (for bench bookkeeping). */
LGS_API int64_t lgs_ctx_launch_count(const lgs_ctx* ctx);

/* ---- phase profiling (CUDA events recorded on the context stream around each phase) -------
 * Phases: 0 preprocess, 1 depth sort + scan, 2 key duplication, 3 tile sort + ranges,
 * 4 blend forward, 5 blend backward, 6 preprocess backward, 7 map upload (pack), 8 mapping loss,
 * 9 Adam step, 10 gradient all-reduce, 11 coverage mask, 12 zero rows of the gradient buffers
 * (depth-layered binning: the backward chain writes only the active rows; in a plan this phase
 * runs on a side branch concurrent with the forward). */
enum { LGS_PHASE_COUNT = 13 };
LGS_API const char* lgs_phase_name(int32_t phase);
LGS_API lgs_status lgs_ctx_profile(lgs_ctx* ctx, int32_t enable);
/* Accumulated device milliseconds and launch counts per phase since the last reset
 * (synchronizes on the recorded events). */
LGS_API lgs_status lgs_ctx_phase_times(lgs_ctx* ctx, double* ms, int64_t* counts, int32_t reset);

/* Work counters of a forward: (pixel, Gaussian) pairs that reached the alpha test and pairs
 * that contributed (the reference's pixel_contribs entries, renderer.cpp:157).  Synchronizes.
 * Counted only by forwards run while the context profiles (lgs_ctx_profile); else LGS_EINVAL. */
LGS_API lgs_status lgs_saved_work(const lgs_saved* tape, int64_t* evaluated, int64_t* contributed);

/* ---- mapping losses (SPEC.md:418-426 compute_losses) ------------------
 * l_rgb = w_l1 L1(rgb, kf.rgb) + (1 - w_l1)(1 - SSIM)/2 (11x11 Gaussian window, sigma 1.5, C1 =
 * 0.01^2, C2 = 0.03^2, statistics at the valid window positions, channel-averaged);
 * l_depth = mean |depth - kf.depth| over pixels with a valid measurement (finite, > 0) and
 * rendered acc > 0.5; l_feat = mean |decode(feat) - feat_gt| with the frozen decoder
 * decode(z) = W2 relu(W1 z + b1) + b2 (proj/src/codec.cpp:88-103 apply_net); l_total = l_rgb +
 * w_depth l_depth + w_feat l_feat.  lgs_mapping_loss writes d l_total / d (rgb, depth, feat) into
 * the tape (the decoder chain is codec.cpp:121-143 decode_backward_input), which
 * lgs_render_backward_loss then back-propagates to the map.  New in this layer: the reference
 * specifies these losses but leaves mapping.cpp / metrics.cpp unimplemented. */
typedef struct {
  int32_t high_dim; /* D: teacher feature channels (32 in the reference design) */
  int32_t hidden;   /* hidden width (64) */
  int32_t low_dim;  /* d: must equal the map's feature dim */
  const float* w1;  /* [hidden][d] row-major (codec.hpp wd1_) */
  const float* b1;  /* [hidden] */
  const float* w2;  /* [D][hidden] row-major (wd2_) */
  const float* b2;  /* [D] */
  int32_t memory;
} lgs_decoder;
typedef struct {
  const float* rgb;     /* [H][W][3] */
  const float* depth;   /* [H][W]; a pixel is valid iff finite and > 0 */
  const float* feat_gt; /* [H][W][D] teacher features */
  int32_t memory;
} lgs_keyframe;
typedef struct {
  double w_l1;    /* 0.8: L1 share of l_rgb, D-SSIM gets 1 - w_l1 */
  double w_depth; /* 0.5 */
  double w_feat;  /* 1.0 */
} lgs_loss_weights;
typedef struct {
  double l_rgb, l_depth, l_feat, l_total;
  double ssim;          /* channel-averaged mean SSIM */
  int64_t depth_pixels; /* pixels in the depth mask */
} lgs_loss_breakdown;
LGS_API lgs_loss_weights lgs_loss_weights_default(void);
/* `rendered` = the images lgs_render_forward wrote for `tape` (rgb and feat are read; depth and
 * acc come from the tape).  `out` may be NULL (no host synchronization). */
LGS_API lgs_status lgs_mapping_loss(lgs_ctx* ctx, lgs_saved* tape, const lgs_images* rendered,
                                    const lgs_keyframe* kf, const lgs_decoder* dec, const lgs_loss_weights* w,
                                    lgs_loss_breakdown* out);
/* Debug/parity: copy the tape's cotangents to host HWC buffers (any may be NULL).  Synchronizes. */
LGS_API lgs_status lgs_debug_cotangents(lgs_ctx* ctx, const lgs_saved* tape, float* rgb, float* depth, float* feat);
/* Insertion coverage mask: mask[p] = 1 iff the rendered acc <
 * 0.5 or (the measured depth is valid -- finite, > 0 -- and |rendered depth - measured| >
 * max(0.05 m, 0.05 measured)).  Reads acc / depth from the tape; mask is uint8 [H][W] (host or
 * device); count (may be NULL) receives the number of selected pixels (synchronizes). */
LGS_API lgs_status lgs_coverage_mask(lgs_ctx* ctx, const lgs_saved* tape, const float* measured_depth,
                                     int32_t memory, uint8_t* mask, int32_t mask_memory, int64_t* count);
/* Back-propagates the cotangents stored in the tape (fused L1 or lgs_mapping_loss) to the map. */
LGS_API lgs_status lgs_render_backward_loss(lgs_ctx* ctx, const lgs_saved* tape, lgs_map_grads* grads,
                                            float* pose_grad);
/* Same, fully asynchronous: device gradients only; pose_grad (NULL, device or PINNED host memory)
 * is written in stream order and valid after lgs_ctx_synchronize / an event on the stream. */
LGS_API lgs_status lgs_render_backward_loss_async(lgs_ctx* ctx, const lgs_saved* tape, lgs_map_grads* grads,
                                                  float* pose_grad);

/* ---- Adam step on the resident map (SPEC.md:430 mapping_round) ---------
 * Per-attribute learning rates of SPEC.md:430; standard bias-corrected Adam (beta1 0.9, beta2
 * 0.999, eps 1e-8: the SPEC names only the optimizer).  SH bands above DC use lr_sh_rest
 * (colour lr / 20 by default; SH0 maps are the reference's colour).  Moments live on the device
 * in the map's packed layout; gradients are the dense device lgs_map_grads of a backward (after
 * lgs_allreduce_grads in a multi-GPU batch: every rank then applies the identical update). */
typedef struct {
  double lr_position, lr_rotation, lr_log_scale, lr_opacity, lr_color, lr_sh_rest, lr_feature;
  double beta1, beta2, eps;
} lgs_adam_config;
LGS_API lgs_adam_config lgs_adam_config_default(void);
LGS_API lgs_status lgs_adam_create(lgs_ctx* ctx, const lgs_map* map, const lgs_adam_config* cfg, lgs_adam** out);
LGS_API lgs_status lgs_adam_destroy(lgs_adam* adam);
LGS_API int64_t lgs_adam_steps(const lgs_adam* adam);
LGS_API lgs_status lgs_adam_step(lgs_ctx* ctx, lgs_adam* adam, lgs_map* map, const lgs_map_grads* grads);
/* Copy the resident map back out in the reference layouts (`dst` shape must match; host or
 * device memory; NULL members skipped). */
LGS_API lgs_status lgs_map_download(lgs_ctx* ctx, const lgs_map* map, lgs_gaussians* dst);

/* ---- LEGOMAP1 map files (proj/src/gaussian_map.cpp:196-259) ------------
 * Format: "LEGOMAP1", u32 feature dim (1..4096), u64 count, then per Gaussian f32 position[3],
 * rotation w,x,y,z, log_scale[3], opacity logit, colour[3], feature[d], u64 anchor keyframe id.
 * Colour is SH degree 0 (the format has no higher bands).  Errors are LGS_EIO with the
 * reference's messages ("bad map file magic", "truncated reading ...", "map feature dimension
 * mismatch ...").  On read, a rotation whose norm is off unit by more than 1e-6 is renormalized
 * (GaussianMap::insert, gaussian_map.cpp:21-23); unit ones stay bit-exact. */
LGS_API lgs_status lgs_map_file_info(const char* path, int32_t* feature_dim, int64_t* count);
/* Reads into caller-owned HOST buffers in the reference layouts (dst->n, feature_dim from
 * lgs_map_file_info; sh_degree 0; memory LGS_MEM_HOST).  expected_dim <= 0 accepts any. */
LGS_API lgs_status lgs_map_file_read(const char* path, int32_t expected_dim, lgs_gaussians* dst, uint64_t* anchors);
/* Writes a host or device map in the reference layouts (sh_degree 0); anchors may be NULL (0). */
LGS_API lgs_status lgs_map_file_write(const char* path, const lgs_gaussians* src, const uint64_t* anchors);
/* File <-> resident device map. */
LGS_API lgs_status lgs_map_load(lgs_ctx* ctx, const char* path, int32_t expected_dim, lgs_map** out);
LGS_API lgs_status lgs_map_save(lgs_ctx* ctx, const lgs_map* map, const char* path, const uint64_t* anchors);

/* ---- map pruning (SPEC.md:471-535 [MODULE] pruning) ---------------------
 * The reference's pruning.cpp is a placeholder (proj/src/pruning.cpp:1); these restate the SPEC's
 * operations on the resident map, with the reference's KD-tree KNN order (kdtree.hpp:36-55:
 * ascending (squared distance, index), the live filter applied inside the search).
 *
 * find_language_redundant (Eq. 4): Gaussians visited in ascending index; a live
 *   G_i takes its k_neighbors nearest LIVE others and marks each G_j among them with
 *   |p_i - p_j|^2 < tau_dist^2 and cos(f_i, f_j) > tau_sim; a marked Gaussian is dead at once (it
 *   marks nothing and leaves every later neighbour set).  Distances and cosines in fp64 from the
 *   map's fp32 values: d2 = (dx*dx + dy*dy) + dz*dz, cos = dot / (|f_i| |f_j|) with sequential
 *   channel sums and no fused multiply-adds; a zero-norm feature is similar to nothing, and a map
 *   without features (d = 0) or with fewer than 2 Gaussians marks nothing.
 * find_geometric: sigmoid(opacity logit) < alpha_min OR max_a exp(log_scale_a)
 *   > scale_max, in fp64.
 * Flags are one byte per Gaussian (1 = marked) in host or device memory (`memory`), counts
 * optional.  k_neighbors 1..32, tau_dist > 0, -1 < tau_sim <= 1, else LGS_EINVAL. */
typedef struct {
  int32_t k_neighbors; /* K (default 8) */
  double tau_dist;     /* metres (0.02) */
  double tau_sim;      /* cosine (0.9) */
  double alpha_min;    /* opacity (0.05) */
  double scale_max;    /* metres (0.5) */
} lgs_prune_config;
LGS_API lgs_prune_config lgs_prune_config_default(void);
LGS_API lgs_status lgs_find_language_redundant(lgs_ctx* ctx, const lgs_map* map, const lgs_prune_config* cfg,
                                               uint8_t* flags, int32_t memory, int64_t* count);
LGS_API lgs_status lgs_find_geometric(lgs_ctx* ctx, const lgs_map* map, const lgs_prune_config* cfg, uint8_t* flags,
                                      int32_t memory, int64_t* count);
/* prune: deletes the union of both sets from the map and, when `adam` is given,
 * the same rows of its moments; survivors keep their relative order (so the caller's stable IDs
 * follow by deleting the flagged rows).  The two flag arrays (optional, host or device, OLD
 * indexing) report each rule's set; *kept = the new size.  Tapes and plans made on the map before
 * the call are invalid afterwards (the map changed size): destroy them.  A host-mapped map is
 * rejected (its owner compacts it). */
LGS_API lgs_status lgs_prune(lgs_ctx* ctx, lgs_map* map, lgs_adam* adam, const lgs_prune_config* cfg,
                             uint8_t* removed_language, uint8_t* removed_geometric, int32_t memory, int64_t* kept);
/* Work counters of the last find_language_redundant on this context: Gaussians with a similar
 * neighbour inside tau_dist (the only ones the greedy sweep can touch), dependency rounds of the
 * parallel sweep (csrc/prune.cu). */
LGS_API lgs_status lgs_prune_stats(const lgs_ctx* ctx, int64_t* candidates, int64_t* rounds);

/* ---- captured steps (CUDA graphs) ---------------------------------------------------------------
 * A plan is one forward (fused L1 against device targets) + backward (device gradients, pose
 * gradient to pinned-host / device memory or NULL) on a resident map and a fixed camera,
 * captured once into a CUDA graph and replayed with one launch (no host work inside the step).
 * The tile-list capacity comes from an eager warm-up step; lgs_plan_sync waits for the replay and
 * re-captures + re-runs it if the pair count outgrew the capacity, or if a speculative plan
 * (below) left a tile unsaturated.  Map contents, targets and
 * gradient buffers may change between replays (same pointers); a new camera re-captures.
 * grads->accumulate = 1: each replay adds its gradients into the buffers (the later views of a
 * multi-view batch; an overflowed or missed replay adds nothing before lgs_plan_sync re-runs it;
 * if the batch's first, writing plan is re-run, the accumulating plans replayed before that
 * re-run must be run again -- renderer.sync_plans does this).  The eager
 * warm-up step inside lgs_plan_create also writes (adds into) the gradient buffers. */
LGS_API lgs_status lgs_plan_create(lgs_ctx* ctx, lgs_map* map, const lgs_camera* cam, const lgs_render_config* cfg,
                                   const lgs_l1_targets* targets, const lgs_images* images /* device or NULL */,
                                   lgs_map_grads* grads, float* pose_grad, lgs_plan** out);
LGS_API lgs_status lgs_plan_run(lgs_ctx* ctx, lgs_plan* plan);
LGS_API lgs_status lgs_plan_sync(lgs_ctx* ctx, lgs_plan* plan, int64_t* pairs);
LGS_API lgs_status lgs_plan_set_camera(lgs_ctx* ctx, lgs_plan* plan, const lgs_camera* cam);
/* Device time of the last replay, from events recorded as the graph's first and last nodes. */
LGS_API lgs_status lgs_plan_elapsed_ms(const lgs_plan* plan, float* ms);
/* Profiling plans re-capture with an event-record node around every phase (each costs a few us
 * per replay, so timed plans leave it off).  lgs_plan_phase_times: device ms per phase
 * (LGS_PHASE_COUNT doubles, lgs_ctx_phase_times order) of the last replay; the conditional second
 * pass of the layered binning is not split out. */
LGS_API lgs_status lgs_plan_set_profiling(lgs_ctx* ctx, lgs_plan* plan, int32_t on);
LGS_API lgs_status lgs_plan_phase_times(const lgs_plan* plan, double* ms);
LGS_API int64_t lgs_plan_launches(const lgs_plan* plan);
/* Times lgs_plan_sync re-captured and re-ran the step (tile lists outgrew the capacity, or a
 * speculative replay left a tile unsaturated). */
LGS_API int64_t lgs_plan_recaptures(const lgs_plan* plan);
/* 1: the plan is speculative -- captured without the layered binning's second pass, because the
 * warm-up render saturated every tile on its first-pass (layer-A) list; each replay reports an
 * unsaturated tile through a mapped host word and lgs_plan_sync then re-captures the plan with the
 * second pass (for good) and re-runs the step, so results never depend on the guess (the replay
 * that left a tile unsaturated writes no gradient rows, so an accumulating plan adds nothing
 * before the re-run).  0: not speculative. */
LGS_API int32_t lgs_plan_speculative(const lgs_plan* plan);
LGS_API lgs_status lgs_plan_destroy(lgs_plan* plan);

/* ---- multi-view mapping batches --------------------------------------------
 * New (the reference is single-threaded CPU code with no multi-view path).  Views are sharded
 * over one process per GPU; each rank accumulates its views' gradients (lgs_map_grads.accumulate)
 * and the batch gradient (a sum over views, renderer.cpp:259-353 is linear in the per-pixel
 * cotangents) is one fp32 sum all-reduce over NCCL / NVLink on the context's stream.  NCCL is
 * resolved at run time (libnccl.so.2, the copy the process already loaded if any).
 * Rank 0 calls lgs_comm_unique_id and ships the 128 bytes to the other ranks out of band. */
typedef struct {
  uint8_t bytes[128];
} lgs_comm_id;
LGS_API lgs_status lgs_comm_unique_id(lgs_comm_id* id);
LGS_API lgs_status lgs_comm_init(lgs_ctx* ctx, int32_t world_size, int32_t rank, const lgs_comm_id* id);
LGS_API lgs_status lgs_comm_destroy(lgs_ctx* ctx);
/* In-place sum over ranks of dense device gradients sized by `map` (one call when the six
 * attribute buffers are one flat block, else one grouped NCCL launch). */
LGS_API lgs_status lgs_allreduce_grads(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads);
LGS_API lgs_status lgs_allreduce_f32(lgs_ctx* ctx, float* buf, int64_t count);
/* Same result as lgs_allreduce_grads, exchanging only the rows (Gaussians) with a nonzero
 * gradient on some rank: counts all-gathered (the host waits for them), then (index, row) records
 * all-gathered and summed into every rank's dense buffer in rank order (identical on all ranks).
 * Falls back to the dense all-reduce when the rows are not sparse; *rows_max (optional) = largest
 * per-rank row count, -1 after a dense fallback. */
LGS_API lgs_status lgs_allreduce_grads_sparse(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads,
                                              int64_t* rows_max);
/* The same sum without a host wait inside the step: the row-record blocks are sized by a capacity
 * learnt from earlier exchanges (the first call runs the exact form and sets it to 1.25 x the rows
 * seen).  _async enqueues everything on the context's stream; _wait (after the step) returns once
 * it has completed.  If some rank listed more rows than the capacity, the async exchange changed
 * nothing (the kernels see every rank's count) and _wait re-runs it exactly with a larger capacity,
 * so the result is always the sum over ranks.  *rows_max: the largest per-rank row count. */
LGS_API lgs_status lgs_allreduce_grads_sparse_async(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads);
LGS_API lgs_status lgs_allreduce_grads_sparse_wait(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads,
                                                   int64_t* rows_max);

/* Host waits inside a collective (the sparse exchange's count all-gather) give up after `ms`
 * milliseconds (default 300000) or as soon as NCCL reports an asynchronous error: the communicator
 * is then aborted (ncclCommAbort releases the peers blocked in the collective with an error), the
 * context's communicator is dropped and the call returns LGS_ECUDA. */
LGS_API lgs_status lgs_comm_set_timeout(lgs_ctx* ctx, int64_t ms);

/* Debug/parity: the row-sparse exchange of lgs_allreduce_grads_sparse -- the same scan, pack and
 * apply kernels and the same host logic -- over `world` ranks simulated in one process on this
 * context's GPU (the all-gathers become device copies).  grads[r] are rank r's dense device
 * buffers; on return every one holds the sum over ranks.  LGS_EINVAL when the rows are not sparse
 * enough (the real exchange would take the dense all-reduce).  cap > 0 runs the capacity-speculative
 * form of lgs_allreduce_grads_sparse_async (record blocks of `cap` rows, no host wait): when a rank
 * has more rows, *overflowed = 1 and every buffer is left as it was. */
LGS_API lgs_status lgs_debug_sparse_reduce_simulated(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* const* grads,
                                                     int32_t world, int64_t cap, int64_t* rows_max,
                                                     int32_t* overflowed);

#ifdef __cplusplus
}
#endif
#endif /* LGS_H_ */
