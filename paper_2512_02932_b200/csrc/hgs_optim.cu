// hgs_optim.cu -- per-Gaussian gradient surgery (freq/surgery.py:55-92) and
// the optimizer step (torch.optim.Adam semantics) over the
// field-major ParamGrads blocks hgs_backward writes (include/hgs_train.h).
//
// One CTA owns G = 64 consecutive Gaussians.  For each of the five fields
// (center 3, log_scale 3, rotation 4, opacity 1, sh 3B) the CTA's slice of a
// field-major array is contiguous, so every global access is a coalesced
// stream; the per-Gaussian transposition the surgery needs (a float64 dot
// product over all P parameters) happens in shared memory (param-major,
// Gaussian-minor, padded stride -> no bank conflicts).  HBM-bound:
//   combine only   : 3 x 4P B read + 4P B written per Gaussian
//   Adam only      : 4P (grad) + 3 x 4P (m, v, p) read, 3 x 4P written
//   combine + Adam : 6 x 4P read + 3 x 4P written (the fused training step)
#include <algorithm>
#include <cmath>

#include "hgs_kernels.cuh"
#include "hgs_nvtx.h"
#include "../../include/hgs_train.h"

namespace hgs {

namespace {

constexpr int kG = 64;           // Gaussians per CTA
constexpr int kOThreads = 256;
constexpr int kStride = kG + 1;  // padded row: (j * 65 + g) % 32 spreads banks

enum : int { kOpCombine = 0, kOpAdam = 1, kOpCombineAdam = 2 };
enum : int { kNone = 0, kProjHigh = 1, kProjLow = 2, kZeroHigh = 3, kZeroLow = 4 };

struct OptArgs {
  int64_t n;
  int B;
  float *field[5];          // parameters (Adam) per field
  const float *gc, *gl, *gh;
  float *out;               // combine only
  float *m, *v;
  const uint8_t *type_spec;
  int mode;
  unsigned long long *n_conflicts;
  float step_size[5];       // lr / (1 - beta1^t) per field group
  float beta1, beta2, eps, bc2_sqrt;
};

__host__ __device__ constexpr int field_width(int f, int B) { return f < 2 ? 3 : (f == 2 ? 4 : (f == 3 ? 1 : 3 * B)); }
__host__ __device__ constexpr int field_j0(int f) { return f == 0 ? 0 : (f == 1 ? 3 : (f == 2 ? 6 : (f == 3 ? 10 : 11))); }
__device__ __forceinline__ int64_t field_off(int f, int64_t n) { return (int64_t)field_j0(f) * n; }

#ifndef HGS_OPT_ZERO_FAST
#define HGS_OPT_ZERO_FAST 1
#endif
#ifndef HGS_OPT_MINB
#define HGS_OPT_MINB 4  // 4 CTAs x 256 threads per SM: 64 registers
#endif

#ifndef HGS_OPT_KU
#define HGS_OPT_KU 4  // elements per thread per step of the element-wise pass (x 4 loads in flight)
#endif
#ifndef HGS_OPT_U1
#define HGS_OPT_U1 4  // unroll of the g_low / g_high staging loop
#endif
constexpr int kU1 = HGS_OPT_U1;

// Templated on the SH basis count so every field width is a compile-time
// constant (index division becomes multiply-shift; loops unroll).
template <int OP, int B>
__global__ void __launch_bounds__(kOThreads, HGS_OPT_MINB) k_optim(OptArgs a) {
  constexpr bool kCombine = OP != kOpAdam;
  constexpr bool kAdam = OP != kOpCombine;
  constexpr int P = 11 + 3 * B;
  __shared__ float sl[kCombine ? P : 1][kStride], sh[kCombine ? P : 1][kStride];
  __shared__ double part[4][kG][3];
  __shared__ float4 surg[kG];
  __shared__ float rot[kG][4];
  __shared__ unsigned int nconf;
  const int64_t g0 = (int64_t)blockIdx.x * kG;
  const int gn = (int)(a.n - g0 < kG ? a.n - g0 : kG);
  const int tid = threadIdx.x;

  if (kCombine) {
    // 1. stage g_low / g_high transposed into shared memory
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      const int fw = field_width(f, B), j0 = field_j0(f);
      const int64_t base = field_off(f, a.n) + g0 * fw;
      const int cnt = gn * fw;
      const float *const glf = a.gl + base, *const ghf = a.gh + base;
      {
#pragma unroll kU1
        for (int e = tid; e < cnt; e += kOThreads) {
          const int g = e / fw, j = j0 + e - g * fw;
          sl[j][g] = __ldg(glf + e);
          sh[j][g] = __ldg(ghf + e);
        }
      }
    }
    if (tid == 0) nconf = 0u;
    __syncthreads();
    // 2. float64 dot / norms per Gaussian: 4 threads per Gaussian, strided j,
    //    combined in a fixed order (bitwise reproducible)
    {
      const int g = tid % kG, q = tid / kG;
      double d = 0.0, nl = 0.0, nh = 0.0;
      if (g < gn)
        for (int j = q; j < P; j += 4) {
          const double x = sl[j][g], y = sh[j][g];
          d += x * y;
          nl += x * x;
          nh += y * y;
        }
      part[q][g][0] = d; part[q][g][1] = nl; part[q][g][2] = nh;
    }
    __syncthreads();
    if (tid < gn) {
      const double d = ((part[0][tid][0] + part[1][tid][0]) + part[2][tid][0]) + part[3][tid][0];
      const double nl = ((part[0][tid][1] + part[1][tid][1]) + part[2][tid][1]) + part[3][tid][1];
      const double nh = ((part[0][tid][2] + part[1][tid][2]) + part[2][tid][2]) + part[3][tid][2];
      const bool conflicted = d < 0.0;  // surgery.py:74-75
      const bool flat = a.type_spec[g0 + tid] == 0;
      int k = kNone;
      float c = 0.f;
      if (conflicted && a.mode == HGS_COMBINE_MASK) {
        k = flat ? kZeroHigh : kZeroLow;  // surgery.py:83-85
      } else if (conflicted && a.mode == HGS_COMBINE_PROJECTION) {
        if (flat && nl > 0.0) { k = kProjHigh; c = (float)(d / nl); }   // Eq. 9, surgery.py:88-89
        if (!flat && nh > 0.0) { k = kProjLow; c = (float)(d / nh); }   // Eq. 10, surgery.py:90-91
      }
      // branch-free form of the five cases (exact: fmaf(-0, x, y) == y, 1 * y == y)
      surg[tid] = make_float4(k == kProjHigh ? c : 0.f, k == kProjLow ? c : 0.f, k == kZeroHigh ? 0.f : 1.f,
                              k == kZeroLow ? 0.f : 1.f);
      if (conflicted) atomicAdd(&nconf, 1u);
    }
    __syncthreads();
    if (tid == 0 && nconf && a.n_conflicts) atomicAdd(a.n_conflicts, (unsigned long long)nconf);
  }

  // 3. element-wise: combined gradient, then (optionally) the Adam update.
  //    kU elements per thread per step, all global loads issued before any
  //    store (the pointers may alias as far as the compiler knows, so it
  //    would otherwise serialise them): kU x 4 loads in flight per thread.
  //    Per-field base pointers + 32-bit indices keep the address arithmetic
  //    to one IMAD.WIDE per access; the surgery is branch-free:
  //    gh' = mh * (gh - ch gl), gl' = ml * (gl - cl gh)  (surgery.py:83-91)
  constexpr int kU = HGS_OPT_KU;
#pragma unroll
  for (int f = 0; f < 5; ++f) {
    const int fw = field_width(f, B), j0 = field_j0(f);
    const int64_t base = field_off(f, a.n) + g0 * fw;
    const int cnt = gn * fw;
    const float *const gcf = a.gc + base;
    float *const mf = kAdam ? a.m + base : nullptr;
    float *const vf = kAdam ? a.v + base : nullptr;
    float *const of = kAdam ? nullptr : a.out + base;
    float *const prm = kAdam ? a.field[f] + g0 * fw : nullptr;
    const float step = kAdam ? a.step_size[f] : 0.f;
    for (int e0 = tid; e0 < cnt; e0 += kOThreads * kU) {
      float gcv[kU], mv[kU], vv[kU], pv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kOThreads;
        if (e < cnt) {
          gcv[u] = __ldcs(gcf + e);
          if (kAdam) {
            mv[u] = __ldcs(mf + e);
            vv[u] = __ldcs(vf + e);
            pv[u] = __ldcs(prm + e);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kOThreads;
        if (e >= cnt) continue;
        const int g = e / fw, j = j0 + e - g * fw;
        float grad = gcv[u];
        if (kCombine) {
          const float gl = sl[j][g], gh = sh[j][g];
          const float4 w = surg[g];  // ch, cl, mh, ml
          grad = (grad + w.w * fmaf(-w.y, gh, gl)) + w.z * fmaf(-w.x, gl, gh);  // surgery.py:92
        }
        if (!kAdam) {
          __stcs(of + e, grad);
          continue;
        }
        float m = mv[u], v = vv[u];
        m = fmaf(1.f - a.beta1, grad - m, m);                // exp_avg.lerp_(grad, 1 - beta1)
        v = fmaf(1.f - a.beta2, grad * grad, v * a.beta2);   // exp_avg_sq.mul_(beta2).addcmul_(g, g, 1 - beta2)
#if HGS_OPT_ZERO_FAST
        // zero moments (untouched Gaussians) bypass the IEEE division and
        // square root, whose slow paths they would take: same results
        // (0 / x = 0, sqrt(0) / b = 0), far fewer instructions
        const float denom = (v == 0.f ? 0.f : sqrtf(v) / a.bc2_sqrt) + a.eps;
        const float pn = m == 0.f ? pv[u] : pv[u] - step * (m / denom);
#else
        const float denom = sqrtf(v) / a.bc2_sqrt + a.eps;
        const float pn = pv[u] - step * (m / denom);
#endif
        __stcs(mf + e, m);
        __stcs(vf + e, v);
        if (f == 2)
          rot[g][e - g * fw] = pn;  // renormalised below
        else
          __stcs(prm + e, pn);
      }
    }
    if (kAdam && f == 2) {  // renormalize_rotations (core/types.py:136-142)
      __syncthreads();
      for (int e = tid; e < gn * 4; e += kOThreads) {
        const int g = e >> 2;
        const double w = rot[g][0], x = rot[g][1], y = rot[g][2], z = rot[g][3];
        const double nrm = sqrt(w * w + x * x + y * y + z * z);
        float q;
        if (nrm <= kQuatMinNorm)
          q = (e & 3) == 0 ? 1.f : 0.f;
        else
          q = (float)((double)rot[g][e & 3] / nrm);
        a.field[2][g0 * 4 + e] = q;
      }
    }
  }
}

template <int B>
void launch_b(int op, OptArgs &a, int blocks, cudaStream_t s) {
  switch (op) {
    case kOpCombine: k_optim<kOpCombine, B><<<blocks, kOThreads, 0, s>>>(a); break;
    case kOpAdam: k_optim<kOpAdam, B><<<blocks, kOThreads, 0, s>>>(a); break;
    default: k_optim<kOpCombineAdam, B><<<blocks, kOThreads, 0, s>>>(a); break;
  }
}

int launch(int op, OptArgs &a, cudaStream_t s) {
  if (a.n <= 0) return HGS_OK;
  const int blocks = (int)((a.n + kG - 1) / kG);
  switch (a.B) {
    case 1: launch_b<1>(op, a, blocks, s); break;
    case 4: launch_b<4>(op, a, blocks, s); break;
    case 9: launch_b<9>(op, a, blocks, s); break;
    default: launch_b<16>(op, a, blocks, s); break;
  }
  return cudaGetLastError() == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

bool sh_ok(int B) { return B == 1 || B == 4 || B == 9 || B == 16; }

int fill_adam(OptArgs &a, const hgs_params *p, const hgs_adam *cfg) {
  if (!p || !cfg || cfg->step < 1 || !(cfg->beta1 >= 0.f && cfg->beta1 < 1.f) ||
      !(cfg->beta2 >= 0.f && cfg->beta2 < 1.f) || !(cfg->eps >= 0.f))
    return HGS_ERR_CONFIG;
  a.field[0] = p->center; a.field[1] = p->log_scale; a.field[2] = p->rotation;
  a.field[3] = p->opacity_logit; a.field[4] = p->sh;
  const double bc1 = 1.0 - std::pow((double)cfg->beta1, (double)cfg->step);
  const double bc2 = 1.0 - std::pow((double)cfg->beta2, (double)cfg->step);
  for (int f = 0; f < 5; ++f) a.step_size[f] = (float)((double)cfg->lr[f] / bc1);
  a.beta1 = cfg->beta1; a.beta2 = cfg->beta2; a.eps = cfg->eps;
  a.bc2_sqrt = (float)std::sqrt(bc2);
  return HGS_OK;
}

}  // namespace
}  // namespace hgs

using namespace hgs;

extern "C" {

int hgs_combine_gradients(int64_t n, int32_t sh_bases, const float *g_color, const float *g_low,
                          const float *g_high, const uint8_t *type_spec, int32_t mode, float *out,
                          unsigned long long *n_conflicts, void *stream) {
  NvtxScope nv("hgs_combine_gradients");
  if (n < 0 || !sh_ok(sh_bases) || mode < 0 || mode > 2) return HGS_ERR_CONFIG;
  if (n > 0 && (!g_color || !g_low || !g_high || !type_spec || !out)) return HGS_ERR_INTEGRITY;
  OptArgs a{};
  a.n = n; a.B = sh_bases;
  a.gc = g_color; a.gl = g_low; a.gh = g_high; a.out = out;
  a.type_spec = type_spec; a.mode = mode; a.n_conflicts = n_conflicts;
  return launch(kOpCombine, a, static_cast<cudaStream_t>(stream));
}

int hgs_adam_step(const hgs_params *params, const float *grads, float *exp_avg, float *exp_avg_sq,
                  const hgs_adam *cfg, void *stream) {
  NvtxScope nv("hgs_adam_step");
  if (!params || params->n < 0 || !sh_ok(params->sh_bases)) return HGS_ERR_CONFIG;
  OptArgs a{};
  a.n = params->n; a.B = params->sh_bases;
  const int rc = fill_adam(a, params, cfg);
  if (rc != HGS_OK) return rc;
  if (a.n > 0 && (!grads || !exp_avg || !exp_avg_sq)) return HGS_ERR_INTEGRITY;
  a.gc = grads; a.m = exp_avg; a.v = exp_avg_sq;
  return launch(kOpAdam, a, static_cast<cudaStream_t>(stream));
}

int hgs_combine_adam_step(const hgs_params *params, const float *g_color, const float *g_low, const float *g_high,
                          const uint8_t *type_spec, int32_t mode, float *exp_avg, float *exp_avg_sq,
                          const hgs_adam *cfg, unsigned long long *n_conflicts, void *stream) {
  NvtxScope nv("hgs_combine_adam_step");
  if (!params || params->n < 0 || !sh_ok(params->sh_bases) || mode < 0 || mode > 2) return HGS_ERR_CONFIG;
  OptArgs a{};
  a.n = params->n; a.B = params->sh_bases;
  const int rc = fill_adam(a, params, cfg);
  if (rc != HGS_OK) return rc;
  if (a.n > 0 && (!g_color || !g_low || !g_high || !type_spec || !exp_avg || !exp_avg_sq)) return HGS_ERR_INTEGRITY;
  a.gc = g_color; a.gl = g_low; a.gh = g_high;
  a.type_spec = type_spec; a.mode = mode; a.n_conflicts = n_conflicts;
  a.m = exp_avg; a.v = exp_avg_sq;
  return launch(kOpCombineAdam, a, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
