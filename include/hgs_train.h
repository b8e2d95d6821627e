/*
 * hgs_train.h -- C ABI of the training-step kernels in libhgs.so: the
 * frequency-decoupled loss stack and the per-Gaussian gradient surgery +
 * optimizer step.  These are SURVEY.md section 8(f) "next" rows 1 and 2: the
 * callers on either side of the rasterizer in one training step
 * (render -> L_color, L_low, L_high -> backward with three
 * upstream pixel gradients -> combine_gradients -> optimizer -> quaternion
 * renormalisation).
 *
 * Reference functions replaced (paths relative to
 * /root/reference/pkg/src/hybridsplat):
 *   dwt_level1 / idwt_level1 / dwt_adjoint   freq/dwt.py:55-105
 *   frequency_losses / frequency_loss_grads  freq/dwt.py:108-137
 *   ssim / ssim_grad                          freq/ssim.py:39-74
 *   color_loss / color_loss_grad              freq/ssim.py:77-94
 *   combine_gradients                         freq/surgery.py:55-92
 *   (project_conflicting_gradients           freq/surgery.py:33-52, per Gaussian)
 *   optimizer step + renormalize_rotations    SPEC.md:424-425 (Adam, 3DGS learning rates;
 *                                             no reference code), core/types.py:136-142
 *
 * Same conventions as hgs.h: device pointers for arrays, host pointers for
 * structs, caller-owned memory and scratch, work enqueued on `stream`, no
 * synchronisation unless stated, hgs_status return codes.  Images are
 * row-major (H, W, C) float32; every reduction is in a fixed order, so
 * results are bitwise reproducible run to run.
 */
#ifndef HGS_TRAIN_H_
#define HGS_TRAIN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- losses */

/* LossWeights (freq/surgery.py:19-30): lam = D-SSIM mix inside the colour
 * loss, lambda_low / lambda_high = weights of the frequency losses (Eq. 8). */
typedef struct hgs_loss_weights {
  double lam, lambda_low, lambda_high;
} hgs_loss_weights;

/* losses[] slots written by hgs_image_losses (device float64). */
#define HGS_LOSS_L1 0     /* mean |r - g|                                   (ssim.py:84) */
#define HGS_LOSS_SSIM 1   /* mean SSIM, 11x11 Gaussian window, zero padded  (ssim.py:39-49) */
#define HGS_LOSS_LOW 2    /* MSE over the LL band                           (dwt.py:108-119) */
#define HGS_LOSS_HIGH 3   /* summed MSE over LH, HL, HH                     (dwt.py:108-119) */
#define HGS_LOSS_COLOR 4  /* (1-lam) L1 + lam (1-SSIM)/2, or L1 if lam == 0 (ssim.py:77-87) */
#define HGS_LOSS_COUNT 5

size_t hgs_loss_scratch_bytes(int32_t height, int32_t width, int32_t channels);

/* All image losses of one view and, if pixel_grads is non-NULL, the upstream
 * gradient stack the backward consumes (kg = 3):
 *   pixel_grads[0] = d L_color / dI                       (color_loss_grad, ssim.py:90-94)
 *   pixel_grads[1] = lambda_low  * d L_low  / dI          (frequency_loss_grads, dwt.py:122-137)
 *   pixel_grads[2] = lambda_high * d L_high / dI
 * each (H, W, C).  rendered / gt: (H, W, C), C >= 1.  Odd H / W are edge
 * replicated for the DWT (dwt.py:32-52).  Two fused tile kernels (moments +
 * SSIM map + band sums; blurred partials + gradients) and a fixed-order
 * float64 reduction. */
int hgs_image_losses(int32_t height, int32_t width, int32_t channels, const float *rendered, const float *gt,
                     const hgs_loss_weights *weights, double *losses, float *pixel_grads, void *scratch,
                     size_t scratch_bytes, void *stream);

/* Level-1 orthonormal Haar transform (dwt.py:55-74): image (H, W, C) ->
 * bands (ceil(H/2), ceil(W/2), C) each; odd sizes edge replicated. */
int hgs_dwt_level1(int32_t height, int32_t width, int32_t channels, const float *image, float *ll, float *lh,
                   float *hl, float *hh, void *stream);

/* Inverse (dwt.py:77-93, adjoint = 0) or adjoint (dwt.py:96-105, adjoint = 1)
 * of hgs_dwt_level1: bands -> image (H, W, C).  The inverse crops the padded
 * row / column; the adjoint folds it back onto the edge. */
int hgs_dwt_inverse(int32_t height, int32_t width, int32_t channels, const float *ll, const float *lh,
                    const float *hl, const float *hh, int32_t adjoint, float *image, void *stream);

/* --------------------------------------------- gradient surgery + optimizer */

/* Trainable parameters, float32 SoA, same layout as hgs_scene but mutable. */
typedef struct hgs_params {
  int64_t n;
  int32_t sh_bases;
  int32_t reserved;
  float *center;        /* (n, 3) */
  float *log_scale;     /* (n, 3) */
  float *rotation;      /* (n, 4) w-first; renormalised after every step */
  float *opacity_logit; /* (n) */
  float *sh;            /* (n, 3, sh_bases) */
} hgs_params;

/* combine_gradients modes (freq/surgery.py:15, 55-92) */
#define HGS_COMBINE_PROJECTION 0
#define HGS_COMBINE_NAIVE 1
#define HGS_COMBINE_MASK 2

/* First-order adaptive-moment step (torch.optim.Adam semantics,
 * the optimizer of 3DGS): per parameter group learning rates
 * lr[0..4] = center, log_scale, rotation, opacity_logit, sh. step = the
 * 1-based count of this update (bias correction). */
typedef struct hgs_adam {
  float lr[5];
  float beta1, beta2, eps;
  int64_t step;
} hgs_adam;

/* combine_gradients (freq/surgery.py:55-92): grads are (n * P) field-major
 * ParamGrads blocks as hgs_backward writes them (P = 11 + 3 * sh_bases).
 * Per Gaussian, conflict = g_low . g_high < 0 (float64 dot over all P);
 * projection / mask per type_spec as in surgery.py:80-91.  out = g_color +
 * g_low' + g_high' (may alias g_color).  n_conflicts (device u64) is
 * incremented by the number of conflicted Gaussians. */
int hgs_combine_gradients(int64_t n, int32_t sh_bases, const float *g_color, const float *g_low,
                          const float *g_high, const uint8_t *type_spec, int32_t mode, float *out,
                          unsigned long long *n_conflicts, void *stream);

/* Adam step with gradient `grads` (n * P, field-major), moments exp_avg /
 * exp_avg_sq (n * P, zero-initialised by the caller before step 1), then
 * rotation renormalisation (core/types.py:136-142: |q| <= 1e-8 -> identity). */
int hgs_adam_step(const hgs_params *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                  const hgs_adam *cfg, void *stream);

/* Fused hgs_combine_gradients + hgs_adam_step in one pass over HBM (the
 * single-GPU training step; multi-GPU steps combine, all-reduce, then step). */
int hgs_combine_adam_step(const hgs_params *params, const float *g_color, const float *g_low, const float *g_high,
                          const uint8_t *type_spec, int32_t mode, float *exp_avg, float *exp_avg_sq,
                          const hgs_adam *cfg, unsigned long long *n_conflicts, void *stream);

/* ------------------------------------------------- adaptive density control */
/* SPEC.md:411-419, 425-427 (the reference ships the stats / keep / append
 * helpers, core/types.py:48-49, 110-130, but no densify code). */
typedef struct hgs_densify_config {
  double grad_threshold; /* mean NDC positional-gradient norm above which a Gaussian grows (2e-4) */
  double prune_opacity;  /* sigmoid(opacity_logit) below this is removed (0.005) */
  double split_scale;    /* max scale above this splits, else clones (0.01 * scene extent) */
  double clone_step;     /* clone offset, in units of the max scale, against the centre's Adam moment (0 = copy) */
} hgs_densify_config;

/* After hgs_backward (kg <= 4, same scratch, and the frame it replayed): per
 * Gaussian touched by the view, grad_accum += |NDC-space gradient of the
 * projected centre| summed over the kg stacked losses, obs_count += 1 (3DGS's
 * densification statistics). */
int hgs_densify_stats(const hgs_scene *scene, const hgs_camera *camera, const void *frame,
                      const hgs_frame_info *info, const void *bwd_scratch, int32_t kg, const uint8_t *touched,
                      float *grad_accum, int32_t *obs_count, void *stream);

size_t hgs_densify_scratch_bytes(int64_t n);

/* Decide prune / keep / clone / split per Gaussian and scan the output row
 * counts; synchronises the stream once to return the new count in *n_out and
 * (nullable, host) census[4] = {kept, pruned, cloned, split}.
 * Invariant: n_out = n + clones + 2 splits - splits - pruned. */
int hgs_densify_plan(const hgs_scene *scene, const float *grad_accum, const int32_t *obs_count,
                     const hgs_densify_config *cfg, void *scratch, size_t scratch_bytes, int64_t *n_out,
                     int64_t *census, void *stream);

/* Write the densified scene (out->n = n_out rows, order-preserving: each
 * survivor's rows at its scanned offset).  Split: two children at +-0.5 sigma
 * along the major axis (in-plane for 2D surfels), scales / 1.6.  Clone: the
 * parent and a copy.  Adam moments (nullable) are carried for survivors and
 * zero for new rows.  The caller resets grad_accum / obs_count. */
int hgs_densify_apply(const hgs_scene *scene, const float *exp_avg, const float *exp_avg_sq, const void *scratch,
                      const hgs_densify_config *cfg, const hgs_params *out, uint8_t *out_type_spec,
                      float *out_exp_avg, float *out_exp_avg_sq, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HGS_TRAIN_H_ */
