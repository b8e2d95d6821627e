/*
 * hgs.h -- C ABI of libhgs.so, the sm_100a hybrid 2D/3D Gaussian rasterizer.
 *
 * This is the drop-in boundary.  It replaces the reference's native blend seam
 * `hybridsplat.raster._blend_cy` (declared in pkg/setup.py:5-13, bound at
 * raster/render.py:73-80 and grad/backward.py:19-30) -- and, because
 * preprocess and binning are hot too, the whole of
 *   build_frame            raster/project.py:360-379
 *   forward_blend          raster/_blend_py.py:55-123
 *   backward_blend         raster/_blend_py.py:126-242
 *   backward chain rule    grad/backward.py:68-178
 *   exchange_pass          exchange.py:137-155
 * All paths below are relative to /root/reference/pkg/src/hybridsplat.
 *
 * Conventions
 *  - Plain C types only.  Every pointer in hgs_scene / hgs_images / grads is a
 *    DEVICE pointer (cudaMalloc / PyTorch caching allocator); structs passed
 *    by pointer live in HOST memory.
 *  - The library never allocates or frees device memory and keeps no global
 *    state: the caller provides a frame buffer (hgs_frame_bytes) that holds
 *    everything a forward produces and a backward consumes.
 *  - Work is enqueued on the caller's stream (a cudaStream_t passed as void*).
 *    hgs_forward enqueues the whole frame without a host round trip and then
 *    synchronises once to report M, K and the status (HGS_FLAG_ASYNC: never).
 *  - Errors are returned as hgs_status codes; the Python layer maps them to
 *    the reference exception classes (hybridsplat/errors.py).
 */
#ifndef HGS_H_
#define HGS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGS_ABI_VERSION 3

typedef enum hgs_status {
  HGS_OK = 0,
  HGS_ERR_CONFIG = 1,            /* ConfigError: bad camera / settings / shapes  */
  HGS_ERR_INVALID_PARAMETER = 2, /* InvalidParameterError: |q| <= 1e-8 (rotation.py:19-20) */
  HGS_ERR_INTEGRITY = 3,         /* IntegrityError: frame / scene / grad mismatch */
  HGS_ERR_DEGENERATE_SCALE = 4,  /* DegenerateScaleError (exchange.py:67-68)      */
  HGS_ERR_PAIR_CAPACITY = 5,     /* frame buffer too small for K pairs: grow + retry */
  HGS_ERR_CUDA = 6               /* a CUDA launch / copy failed                   */
} hgs_status;

/* Scene in structure-of-arrays layout, float32 (reference: core/types.py:32-50,
 * float64 there).  sh is (n, 3, sh_bases) channel-major; type_spec 0 = 2D surfel,
 * 1 = 3D Gaussian.
 *
 * The four *64 pointers are an optional float64 copy of the geometry (all four
 * or none).  When they are set, every discrete decision of the forward -- depth
 * keys and order, near / singular / quaternion culls, bounding boxes, tile
 * lists and the float64 re-checks of the compositors -- is taken on these exact
 * values, i.e. on the reference's float64 inputs (core/types.py:40-45), and the
 * exported SplatFrame arrays are computed from them.  The float32 fields must
 * then hold their float32 rounding: the compositor records' float32 payload and
 * the chain rule read those.  Without them the float32 fields are the inputs. */
typedef struct hgs_scene {
  int64_t n;
  int32_t sh_bases; /* (degree + 1)^2, degree <= 3 */
  int32_t reserved;
  const float *center;        /* (n, 3) */
  const float *log_scale;     /* (n, 3) */
  const float *rotation;      /* (n, 4) w-first, not necessarily unit */
  const float *opacity_logit; /* (n) */
  const float *sh;            /* (n, 3, sh_bases) */
  const uint8_t *type_spec;   /* (n) */
  const double *center64;        /* (n, 3) nullable [ABI 2] */
  const double *log_scale64;     /* (n, 3) nullable */
  const double *rotation64;      /* (n, 4) nullable */
  const double *opacity_logit64; /* (n)    nullable */
} hgs_scene;

/* Pinhole camera (core/types.py:145-197); pixel (ix, iy) samples (ix+.5, iy+.5). */
typedef struct hgs_camera {
  double fx, fy, cx, cy;
  int32_t width, height;
  double world_to_camera[16]; /* row-major 4x4 */
  double near_plane, far_plane;
} hgs_camera;

/* RenderSettings (raster/project.py:34-45) + mode flags. */
typedef struct hgs_settings {
  float background[3];
  int32_t tile_size; /* 16 (the compositor's tile); see hgs_frame_tile_bins */
  double theta_z, t_z, lambda_z;
  uint32_t flags;
  int32_t n_timing_events;     /* 0, or the length of timing_events            */
  void *const *timing_events;  /* nullable: caller-created cudaEvent_t handles
                                * recorded on the stream at stage boundaries:
                                * forward  [0] start [1] depth keys+sort
                                *          [2] f64 preprocess+scan [3] binning
                                *          [4] composite
                                * backward [0] start [1] composite replay
                                *          [2] chain rule                     */
  /* [ABI 3] nullable: an auxiliary cudaStream_t and two caller-created
   * cudaEvent_t (fork, join).  With all three set, hgs_forward runs the
   * float64 preprocess on aux_stream beside the depth sort and joins it on
   * the main stream before binning (graph capture follows the fork). */
  void *aux_stream;
  void *aux_events[2];
} hgs_settings;

#define HGS_FLAG_NAIVE 0x1u /* render_naive: every splat for every pixel, no tiles, no bbox test (render.py:101-118) */
#define HGS_FLAG_FAST 0x2u  /* skip the float64 re-evaluation of near-threshold decisions */
#define HGS_FLAG_COUNT 0x4u /* count evaluated / contributing pairs per type (hgs_frame_stats) */
#define HGS_FLAG_DETERMINISTIC 0x8u /* backward: fixed-order (sorted-record) gradient reduction instead of
                                     * float atomics -- bitwise reproducible; needs the
                                     * scratch of hgs_backward_det_scratch_bytes */
#define HGS_FLAG_DEFER_ALL 0x10u /* tests: with HGS_FLAG_COUNT, defer every pixel of the forward to the float64
                                    resume kernel (exercises the deferred-pixel path on a whole image) */
#define HGS_FLAG_REPLAY_ONLY 0x20u /* hgs_backward (kg <= 4): the back-to-front replay only; the screen-space
                                      accumulators stay in the scratch for hgs_backward_chain */
#define HGS_FLAG_ACCUMULATE 0x40u  /* hgs_backward / hgs_backward_chain: grads += this view's gradient
                                      (multi-view batches) instead of grads = */
#define HGS_FLAG_ASYNC 0x100u /* [ABI 3] hgs_forward: no host round trip at all (CUDA-graph capturable);
                                * info->m = info->k = -1 until hgs_frame_sync_info, which also reports
                                * the frame's status (bad parameters, pair capacity).  hgs_backward runs
                                * on such a frame directly; the exports need the synced info. */
#define HGS_FLAG_FRAME_ONLY 0x80u /* [ABI 3] hgs_forward: build_frame only (project.py:360-379): depth sort,
                                   * preprocess and binning, no compositing; out may be NULL and the
                                   * frame cannot be back-propagated */

/* Output images (device, row-major).  Any of normal / alpha may be NULL. */
typedef struct hgs_images {
  float *color;         /* (H, W, 3): blend + background * T (render.py:54-61) */
  float *depth;         /* (H, W): sum w * z_center (_blend_py.py:105) */
  float *transmittance; /* (H, W) */
  float *alpha;         /* (H, W): 1 - T                      [extension] */
  float *normal;        /* (H, W, 3): sum w * n_camera         [extension] */
} hgs_images;

/* Filled by hgs_forward, consumed by hgs_backward / hgs_frame_export. */
typedef struct hgs_frame_info {
  int64_t n;          /* Gaussians in the scene */
  int64_t m;          /* splats kept (near + singular-conic cull), SplatFrame.count */
  int64_t k;          /* tile/splat pairs = len(tile_ids) */
  int64_t n_tiles;
  int32_t width, height, tiles_x, tiles_y;
  int64_t pair_capacity;
  int32_t sh_bases;
  uint32_t flags;
  uint32_t internal[4]; /* library bookkeeping (which ping-pong buffer holds the tile lists) */
} hgs_frame_info;

/* Bytes of device memory hgs_forward needs for n Gaussians at W x H and room
 * for pair_capacity tile/splat pairs. */
size_t hgs_frame_bytes(int64_t n, int32_t width, int32_t height, int32_t tile_size, int64_t pair_capacity);

/* render (raster/render.py:83-98): project, depth-sort, bin, composite.
 * Every launch is sized from host-known bounds and reads the data-dependent
 * counts (M, the depth-sort digit plan, K) from the frame on the device; the
 * call ends with one host round trip that fills info->m / info->k and returns
 * the frame's status (none with HGS_FLAG_ASYNC).  HGS_ERR_PAIR_CAPACITY
 * (info->k = required pairs): the frame buffer cannot hold K pairs; the
 * caller grows the buffer and calls again. */
int hgs_forward(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings, void *frame,
                size_t frame_bytes, const hgs_images *out, hgs_frame_info *info, void *stream);

/* [ABI 3] Synchronises the stream, fills info->m, info->k from the frame and
 * returns its status (HGS_OK, HGS_ERR_INVALID_PARAMETER, HGS_ERR_PAIR_CAPACITY
 * with info->k = required pairs, ...). */
int hgs_frame_sync_info(void *frame, hgs_frame_info *info, void *stream);

/* Scratch bytes for hgs_backward with kg stacked upstream gradients. */
size_t hgs_backward_scratch_bytes(int64_t n, int32_t kg);

/* Scratch bytes for a HGS_FLAG_DETERMINISTIC backward with room for `records`
 * per-(splat, warp) / per-(splat, deferred pixel) partial records (about
 * 1.3 x K at KG = 1).  hgs_backward returns HGS_ERR_PAIR_CAPACITY if they do
 * not fit: grow the scratch and call again. */
size_t hgs_backward_det_scratch_bytes(int64_t n, int32_t kg, int64_t records);

/* backward (grad/backward.py:37-181).
 *   pixel_grads  (kg, H, W, 3) dL/dcolor, required
 *   depth_grads  (kg, H, W)    dL/ddepth,  nullable   [extension]
 *   normal_grads (kg, H, W, 3) dL/dnormal, nullable   [extension]
 *   alpha_grads  (kg, H, W)    dL/dalpha,  nullable   [extension]
 *   grads        (kg, n * P) out, P = 11 + 3 * sh_bases, each kg block laid out
 *                field-major: center (n,3) | log_scale (n,3) | rotation (n,4) |
 *                opacity_logit (n) | sh (n,3,B)  (ParamGrads, grad/bundle.py:11-30)
 *   touched      (n) uint8 out, 1 = the Gaussian contributed to some pixel
 * The frame buffer must hold the hgs_forward result for the same scene. */
int hgs_backward(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings, const void *frame,
                 const hgs_frame_info *info, int32_t kg, const float *pixel_grads, const float *depth_grads,
                 const float *normal_grads, const float *alpha_grads, void *scratch, size_t scratch_bytes,
                 float *grads, uint8_t *touched, void *stream);

/* The per-Gaussian chain rule (grad/backward.py:68-178) of the last
 * hgs_backward with HGS_FLAG_REPLAY_ONLY on this scratch (kg <= 4), for the
 * Gaussians [g0, g1) only: grads rows g0..g1-1 of every field are written (or,
 * with HGS_FLAG_ACCUMULATE, added to).  A multi-view step runs it in buckets
 * so each bucket's gradient all-reduce overlaps the next bucket's chain rule. */
int hgs_backward_chain(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings,
                       const void *frame, const hgs_frame_info *info, int32_t kg, const float *depth_grads,
                       const float *normal_grads, const float *alpha_grads, const void *scratch,
                       size_t scratch_bytes, int64_t g0, int64_t g1, float *grads, void *stream);

/* Adaptive type exchange (exchange.py:137-155), in place on log_scale, rotation
 * and type_spec (device).  eranks (n) float out (nullable).  report (host) =
 * {n_3d_to_2d, n_2d_to_3d, n_2d, n_3d, hist[20] over [1, 3]}.  scratch: 256 B. */
typedef struct hgs_exchange_report {
  int64_t n_3d_to_2d, n_2d_to_3d, n_2d, n_3d;
  int64_t erank_hist[20];
} hgs_exchange_report;

int hgs_exchange(int64_t n, float *log_scale, float *rotation, uint8_t *type_spec, double theta_e, float *eranks,
                 void *scratch, hgs_exchange_report *report, void *stream);

/* The same pass on float64 device arrays (the reference's own precision,
 * exchange.py:58-99): host scenes are exchanged through this entry point so
 * that only the flipped rows change and the demoted rows get the float64
 * reparameterisation.  eranks (n) double out (nullable). */
int hgs_exchange_f64(int64_t n, double *log_scale, double *rotation, uint8_t *type_spec, double theta_e,
                     double *eranks, void *scratch, hgs_exchange_report *report, void *stream);

/* Test / API-parity export of the sorted SplatFrame (raster/project.py:60-90)
 * into caller device buffers (each nullable): idx (m) i32, typ (m) u8,
 * depth (m), center2d (m,2), cov2d (m,3), conic (m,3), mrow (m,3,4),
 * alpha_eff (m), color (m,3), bbox (m,4) i32, radius (m), tile_offsets
 * (n_tiles+1) i64, tile_ids (k) i32.  Values are the float64 preprocess
 * results (bit-for-bit what the binning used).  tile_offsets / tile_ids are
 * the COMPOSITOR's 16 x 16 lists (slots, depth order): they omit the
 * (splat, tile) pairs whose support cannot reach the tile, so they are a
 * subset of the reference's bbox lists (project.py:329-357) -- those come
 * from hgs_frame_tile_bins (any tile size, 16 included). */
typedef struct hgs_frame_export {
  int32_t *idx;
  uint8_t *typ;
  double *depth, *center2d, *cov2d, *conic, *mrow, *alpha_eff, *color, *radius, *normal;
  int32_t *bbox;
  int64_t *tile_offsets;
  int32_t *tile_ids;
  int32_t *pixel_count; /* (H, W) blend-log entries per pixel */
  /* [ABI 3] the remaining SplatFrame arrays (project.py:254-257): t_cam (m,3)
   * camera-space centre, alpha (m) sigmoid(opacity_logit) before modulation,
   * view_dir (m,3), cam_dist (m) */
  double *t_cam, *alpha, *view_dir, *cam_dist;
} hgs_frame_export;

int hgs_frame_export_arrays(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings,
                            const void *frame, const hgs_frame_info *info, const hgs_frame_export *out, void *stream);

/* Blend log (raster/render.py:30-51) for small frames: offsets (H*W+1) i64 from
 * the pixel counts, position (total) i32, alpha / u / v (total) float. */
int hgs_blend_log(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings, const void *frame,
                  const hgs_frame_info *info, const int64_t *offsets, int32_t *position, float *alpha, float *u,
                  float *v, void *stream);

/* Diagnostics of the last forward / backward on this frame (synchronous):
 *  [0] float64 pair re-evaluations  [1] float64 transmittance replays
 *  with HGS_FLAG_COUNT: forward [2] 3D pairs evaluated (bbox pass) [3] 2D pairs
 *  evaluated [4] 3D contributing [5] 2D contributing; backward [6] 3D
 *  contributing [7] 2D ray-branch contributing [8] 2D low-pass contributing
 *  [9] pairs evaluated. */
int hgs_frame_stats(const void *frame, const hgs_frame_info *info, uint64_t *out16, void *stream);

/* [ABI 3] The reference's tile lists of a frame (bbox-based, _tile_bins
 * project.py:329-357) at any tile size.  The compositor always bins at
 * 16 x 16 and drops the pairs its support cannot reach; the reference bins
 * every tile of the bbox at settings.tile_size (project.py:37), and only
 * SplatFrame.tile_offsets / tile_ids depend on it (the image does not).
 * tile_size in {8, 16, 32, 64}.  Synchronous:
 * counts the pairs into *k_out and returns HGS_ERR_PAIR_CAPACITY when
 * ids_capacity < *k_out; otherwise writes tile_offsets ((tiles+1) i64) and
 * tile_ids (*k_out i32, sorted slots, ascending within a tile).  scratch:
 * hgs_tile_bins_scratch_bytes(m, W, H, tile_size, ids_capacity). */
size_t hgs_tile_bins_scratch_bytes(int64_t m, int32_t width, int32_t height, int32_t tile_size, int64_t pair_capacity);
int hgs_frame_tile_bins(const void *frame, const hgs_frame_info *info, int32_t tile_size, int64_t *tile_offsets,
                        int32_t *tile_ids, int64_t ids_capacity, void *scratch, size_t scratch_bytes, int64_t *k_out,
                        void *stream);

/* [ABI 3] Batch forms of the reference's public per-primitive helpers, in
 * float64 on the device (hgs_helpers.cu), all pointers device pointers.
 *
 * evaluate_contribution / ray_splat_intersect (raster/project.py:109-152) for n
 * (splat, pixel) pairs: typ (n) u8, center2d (n,2), conic (n,3) = (c00, c01,
 * c11), mrow (n,3,4), opacity (n), pixel (n,2) -> alpha (n) (0 for a degenerate
 * intersection), u / v (n, nullable: the ray/plane coordinates of 2D pairs,
 * (dx, dy) for 3D), flags (n, nullable: bit 0 = |den| < 1e-9, the reference's
 * DegenerateIntersection). */
int hgs_eval_contributions(int64_t n, const uint8_t *typ, const double *center2d, const double *conic,
                           const double *mrow, const double *opacity, const double *pixel, double *alpha, double *u,
                           double *v, int32_t *flags, void *stream);
/* effective_rank (exchange.py:58-73): log_scale (n,3) -> eranks (n).
 * Synchronous; HGS_ERR_DEGENERATE_SCALE if any row's squared scales sum to
 * zero or overflow.  scratch: 256 B of device memory. */
int hgs_effective_rank_f64(int64_t n, const double *log_scale, double *eranks, void *scratch, void *stream);
/* choose_permutation + reparameterize_3d_to_2d (exchange.py:76-99):
 * perm (n) i32 (0 identity, 1 P_x, 2 P_y; nullable), out_log_scale (n,3) /
 * out_rotation (n,4) (both or neither).  Synchronous; HGS_ERR_INVALID_PARAMETER
 * for |q| <= 1e-8.  scratch: 256 B. */
int hgs_reparameterize_f64(int64_t n, const double *log_scale, const double *rotation, double *out_log_scale,
                           double *out_rotation, int32_t *perm, void *scratch, void *stream);
/* modulated_z / modulated_opacity / modulated_opacity_grads (exchange.py:
 * 102-129): opacity (n, the un-modulated alpha; nullable if only sz_star /
 * d_alpha are wanted), log_scale_z (n) -> sz_star, alpha_eff, d_alpha, d_logz
 * (each (n), nullable). */
int hgs_modulation_f64(int64_t n, const double *opacity, const double *log_scale_z, double theta_z, double t_z,
                       double lambda_z, double *sz_star, double *alpha_eff, double *d_alpha, double *d_logz,
                       void *stream);

/* [ABI 3] Host I/O of the reference-facing float64 API (_hostio.py):
 * page-lock an existing host range (cudaHostRegister), and widen n float32
 * device values to float64 in `scratch` (device, 8n bytes, 16-byte aligned)
 * then copy them asynchronously into host memory `dst_host` (registered: the
 * copy is a DMA), so part of each float64 output never touches the host
 * cores. */
int hgs_host_register(void *ptr, size_t bytes);
int hgs_host_unregister(void *ptr);
int hgs_widen_d2h(const float *src, double *dst_host, int64_t n, double *scratch, void *stream);
/* Host-only float32 <-> float64 conversion of n elements (or a plain copy) on `threads` host
 * threads (<= 0: all), destination written with streaming stores (no
 * read-for-ownership of the destination lines).  Synchronous, no CUDA. */
int hgs_host_widen(const float *src, double *dst, int64_t n, int threads);
int hgs_host_narrow(const double *src, float *dst, int64_t n, int threads);
int hgs_host_copy(const void *src, void *dst, int64_t bytes, int threads);
/* Deterministic float64 sums for the host-scene fingerprint: sums[b] = the
 * sum of elements [b B, (b + 1) B) in a fixed order (B = hgs_host_sum_block(),
 * blocks at absolute positions); the caller adds the block sums in order.
 * The copying form also copies src to dst (the upload's staging pass) and
 * yields the same sums. */
/* hgs_host_narrow that also counts the non-finite (inf / NaN) float64
 * inputs into *nonfinite (the reference's upstream-gradient check, on the
 * float64 values, in the same pass). */
int hgs_host_narrow_count(const double *src, float *dst, int64_t n, int threads, int64_t *nonfinite);
int64_t hgs_host_sum_block(void);
int hgs_host_block_sums(const double *src, int64_t n, double *sums, int threads);
int hgs_host_copy_block_sums(const double *src, double *dst, int64_t n, double *sums, int threads);

const char *hgs_status_string(int status);
int hgs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HGS_H_ */
