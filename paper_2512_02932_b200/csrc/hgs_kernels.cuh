// hgs_kernels.cuh -- kernel argument blocks, frame state, and the per-pair
// evaluation shared by the forward and backward compositors.
#pragma once

#include "hgs_common.cuh"
#include "hgs_sort.cuh"

namespace hgs {

// Small device-side state at the head of the frame buffer.
struct FrameState {
  uint32_t status;
  uint32_t m_count;
  unsigned long long k_total;
  uint32_t tile_counters[24];
  unsigned long long diag[4];  // [0] f64 pair re-checks, [1] f64 T replays
};

struct CompositeArgs {
  // binning
  const SplatRec *recs;
  const uint32_t *tile_off;
  const uint32_t *tile_vals;
  int64_t m;
  int tiles_x, width, height;
  uint32_t flags;
  float bg[3];
  // outputs
  float *color, *depth, *trans, *alpha, *normal;
  float *pix_T;
  uint32_t *pix_last, *pix_count;
  // float64 re-evaluation of near-threshold decisions
  SceneView sc;
  CamD cam;
  ModD mod;
  FrameState *st;
};

// log2 domain constants: at = ex2(arg), arg = log2(alpha_eff) - d * 0.5 log2(e)
constexpr float kHalfLog2e = 0.72134752044448170f;
constexpr float kArgMinAlpha = -7.99435343685885793f;  // log2(1/255)
constexpr float kArgClamp = -0.01449956969511509f;     // log2(0.99)
constexpr float kEps = 5.96046448e-8f;                 // 2^-24

// Result of evaluating one (pixel, splat) pair.
struct PairEval {
  float at;       // clamped alpha
  float dx, dy;   // pixel - centre (pixels)
  float u, v;     // 3D: (dx, dy); 2D: tangent-plane intersection
  float hu0, hu1, hu3, hv0, hv1, hv3, inv_den;  // 2D ray quantities
  float pxl, pyl; // pixel relative to the anchor
  bool ray;       // 2D: ray branch chosen (d_ray <= d_screen)
  bool clamped;   // raw alpha > 0.99 (colour-only gradient)
};

// float64 re-evaluation of one pair exactly as the reference does it
// (_blend_py.py:17-44, 96-100).  Returns false if the pair is skipped.
static __device__ __noinline__ bool pair_f64(const SceneView &sc, const CamD &cam, const ModD &mod, uint32_t idx, int ix,
                                      int iy, double *at_out, bool *ray_out, bool *clamped_out) {
  ProjD o;
  project_d(sc, idx, cam, mod, o);
  const double px = ix + 0.5, py = iy + 0.5;
  const double dx = px - o.ctr[0], dy = py - o.ctr[1];
  double d;
  bool ray = false;
  if (o.typ == 1) {
    d = (o.conic[0] * dx * dx + 2.0 * o.conic[1] * dx * dy) + o.conic[2] * dy * dy;
  } else {
    const double *m = o.mrow;
    double hu0 = px * m[8] - m[0], hu1 = px * m[9] - m[1], hu3 = px * m[11] - m[3];
    double hv0 = py * m[8] - m[4], hv1 = py * m[9] - m[5], hv3 = py * m[11] - m[7];
    double den = hu0 * hv1 - hu1 * hv0;
    if (fabs(den) < kDegenerateDen) return false;
    double u = (hu1 * hv3 - hu3 * hv1) / den, v = (hu3 * hv0 - hu0 * hv3) / den;
    double d_ray = u * u + v * v, d_screen = (dx * dx + dy * dy) * kInvLp2;
    ray = d_ray <= d_screen;
    d = ray ? d_ray : d_screen;
  }
  double raw = o.alpha_eff * exp(-0.5 * d);
  *clamped_out = raw > kAlphaClamp;
  double at = raw > kAlphaClamp ? kAlphaClamp : raw;
  *ray_out = ray;
  *at_out = at;
  return at >= kMinAlpha;
}

// Evaluate a pair in float32.  BWD additionally resolves the backward-only
// decisions (ray branch, clamp) exactly.  Returns false if the pair does not
// contribute.  Decisions whose float32 error bound straddles the threshold
// are re-evaluated in float64 (pair_f64) unless HGS_FLAG_FAST.
template <bool BWD>
__device__ __forceinline__ bool eval_pair(const SplatRec &r, int ix, int iy, const CompositeArgs &a, PairEval &p) {
  const float4 r0 = r.r0;
  const int4 q = r.r5;
  const uint32_t tag = __float_as_uint(r.r4.w);
  const bool is3d = tag >> 31;
  p.pxl = (float)(ix - q.z) + 0.5f;
  p.pyl = (float)(iy - q.w) + 0.5f;
  p.dx = p.pxl - r0.x;
  p.dy = p.pyl - r0.y;
  const bool exact = !(a.flags & HGS_FLAG_FAST);
  bool ambiguous = false;
  float arg = 0.f;
  p.ray = false;
  if (is3d) {
    const float4 cn = r.r1;
    const float t = cn.y * p.dx * p.dy;
    const float d = fmaf(cn.x * p.dx, p.dx, fmaf(cn.z * p.dy, p.dy, 2.f * t));
    p.u = p.dx;
    p.v = p.dy;
    arg = fmaf(d, -kHalfLog2e, r0.w);
    // |d error| <= 16 eps S, S = a dx^2 + c dy^2 + 2|b dx dy| (>= every term)
    const float S = d + 2.f * (fabsf(t) - t);
    const float margin = fmaf(S, 16.f * kEps * kHalfLog2e, 1e-5f);
    if (arg < kArgMinAlpha - margin) return false;  // cheap cull: no ex2
    if (exact && (arg <= kArgMinAlpha + margin || (BWD && fabsf(arg - kArgClamp) <= margin))) ambiguous = true;
  } else {
    const float4 m1 = r.r1, m2 = r.r2;
    const float m23 = r.r3.x;
    // rows re-based at the anchor: hu = pxl m2 - m0', hv = pyl m2 - m1'
    p.hu0 = fmaf(p.pxl, m2.z, -m1.x);
    p.hu1 = fmaf(p.pxl, m2.w, -m1.y);
    p.hu3 = fmaf(p.pxl, m23, -m1.z);
    p.hv0 = fmaf(p.pyl, m2.z, -m1.w);
    p.hv1 = fmaf(p.pyl, m2.w, -m2.x);
    p.hv3 = fmaf(p.pyl, m23, -m2.y);
    const float den = p.hu0 * p.hv1 - p.hu1 * p.hv0;
    const float dmag = fabsf(p.hu0 * p.hv1) + fabsf(p.hu1 * p.hv0);
    if (fabsf(den) <= fmaf(dmag, 1e-4f, (float)kDegenerateDen)) {
      // (near-)degenerate ray/plane intersection (_blend_py.py:36-37)
      if (!exact) {
        if (fabsf(den) < (float)kDegenerateDen) return false;
      } else {
        ambiguous = true;
      }
    }
    if (!ambiguous) {
      p.inv_den = 1.f / den;
      p.u = (p.hu1 * p.hv3 - p.hu3 * p.hv1) * p.inv_den;
      p.v = (p.hu3 * p.hv0 - p.hu0 * p.hv3) * p.inv_den;
      const float dray = fmaf(p.u, p.u, p.v * p.v);
      const float dscr = (p.dx * p.dx + p.dy * p.dy) * 4.f;
      p.ray = dray <= dscr;
      const float d = p.ray ? dray : dscr;
      arg = fmaf(d, -kHalfLog2e, r0.w);
      constexpr float kCoarse = 0.05f;  // log2 units; precise bounds only inside
      if (arg < kArgMinAlpha - kCoarse) return false;
      const bool near = exact && (arg <= kArgMinAlpha + kCoarse ||
                                  (BWD && (fabsf(arg - kArgClamp) <= kCoarse ||
                                           fabsf(dray - dscr) <= 0.02f * (dray + dscr))));
      if (near) {
        // first-order error bounds of the float32 2x2 solve
        const float A0 = fabsf(p.pxl * m2.z) + fabsf(m1.x), A1 = fabsf(p.pxl * m2.w) + fabsf(m1.y);
        const float A3 = fabsf(p.pxl * m23) + fabsf(m1.z);
        const float B0 = fabsf(p.pyl * m2.z) + fabsf(m1.w), B1 = fabsf(p.pyl * m2.w) + fabsf(m2.x);
        const float B3 = fabsf(p.pyl * m23) + fabsf(m2.y);
        const float ad = fabsf(den);
        const float dden = 6.f * kEps * (A0 * B1 + A1 * B0);
        const float du = (6.f * kEps * (A1 * B3 + A3 * B1) + fabsf(p.u) * dden) / ad + 4.f * kEps * fabsf(p.u);
        const float dv = (6.f * kEps * (A3 * B0 + A0 * B3) + fabsf(p.v) * dden) / ad + 4.f * kEps * fabsf(p.v);
        const float e_ray = 2.f * (fabsf(p.u) * du + fabsf(p.v) * dv) + 4.f * kEps * dray;
        const float e_scr = 8.f * kEps * dscr + 1e-6f * (fabsf(p.dx) + fabsf(p.dy));
        const float margin = fmaf(p.ray ? e_ray : e_scr, kHalfLog2e, 1e-5f);
        if (arg < kArgMinAlpha - margin) return false;
        if (arg <= kArgMinAlpha + margin) ambiguous = true;
        if (BWD && (fabsf(arg - kArgClamp) <= margin || fabsf(dray - dscr) <= e_ray + e_scr)) ambiguous = true;
      }
    }
  }
  if (ambiguous) {
    double at64;
    bool ray64, cl64;
    atomicAdd(&a.st->diag[0], 1ull);
    if (!pair_f64(a.sc, a.cam, a.mod, tag & 0x7fffffffu, ix, iy, &at64, &ray64, &cl64)) return false;
    p.at = (float)at64;
    p.clamped = cl64;
    if (!is3d) {
      p.ray = ray64;
      const float den = p.hu0 * p.hv1 - p.hu1 * p.hv0;
      p.inv_den = 1.f / den;
      p.u = (p.hu1 * p.hv3 - p.hu3 * p.hv1) * p.inv_den;
      p.v = (p.hu3 * p.hv0 - p.hu0 * p.hv3) * p.inv_den;
    }
    return true;
  }
  p.clamped = arg > kArgClamp;
  p.at = p.clamped ? 0.99f : ex2_approx(arg);
  return true;
}

// Early-stop decision T < 1e-4 (_blend_py.py:111-113).  Near the threshold
// the pixel's transmittance is replayed in float64 over the tile list.
static __device__ __noinline__ bool replay_T_below(const CompositeArgs &a, int64_t lo, int64_t upto, int ix, int iy,
                                            bool naive) {
  atomicAdd(&a.st->diag[1], 1ull);
  double T = 1.0;
  for (int64_t j = lo; j <= upto; ++j) {
    uint32_t rk = naive ? (uint32_t)j : a.tile_vals[j];
    const SplatRec r = a.recs[rk];
    if (!naive) {
      const int4 q = r.r5;
      const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16);
      const int x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
      if (ix < x0 || ix > x1 || iy < y0 || iy > y1) continue;
    }
    PairEval p;
    if (!eval_pair<false>(r, ix, iy, a, p)) continue;
    double at64;
    bool ray64, cl64;
    if (!pair_f64(a.sc, a.cam, a.mod, __float_as_uint(r.r4.w) & 0x7fffffffu, ix, iy, &at64, &ray64, &cl64))
      continue;
    T *= 1.0 - at64;
  }
  return T < kEarlyStopT;
}

struct FwdGuard {
  const CompositeArgs &a;
  int ix, iy;
  bool exact, naive;
  __device__ FwdGuard(const CompositeArgs &a_, int ix_, int iy_)
      : a(a_), ix(ix_), iy(iy_), exact(!(a_.flags & HGS_FLAG_FAST)), naive(a_.flags & HGS_FLAG_NAIVE) {}
  // Tn = transmittance after the splat at tile-list entry e.
  __device__ __forceinline__ bool early_stop(float Tn, float Tprev, int64_t lo, int64_t e) const {
    const float thr = (float)kEarlyStopT;
    if (exact && fabsf(Tn - thr) <= 2e-5f * thr) return replay_T_below(a, lo, e, ix, iy, naive);
    return Tn < thr;
  }
};

__device__ __forceinline__ bool eval_alpha(const SplatRec &r, int ix, int iy, const FwdGuard &g, float &at) {
  PairEval p;
  if (!eval_pair<false>(r, ix, iy, g.a, p)) return false;
  at = p.at;
  return true;
}

struct BwdArgs {
  CompositeArgs c;          // recs, tile lists, flags, bg, scene / camera for f64 checks
  const float *pix_grad;    // (KG, H, W, 3)
  const float *depth_grad;  // (KG, H, W) or null
  const float *normal_grad; // (KG, H, W, 3) or null
  const float *alpha_grad;  // (KG, H, W) or null
  float *acc;               // (n, KG, 16)
  float *acc_ext;           // (n, KG, 4) or null
  uint8_t *touched_rank;    // (m)
};

struct ChainArgs {
  SceneView sc;
  CamD cam;
  ModD mod;
  const float *acc;      // (n, KG, 16)
  const float *acc_ext;  // (n, KG, 4) or null
  int kg;
  float *grads;          // (KG, n*P) field-major blocks
};

struct ExchangeState {
  unsigned long long counts[4];  // demote, promote, n3 before, degenerate rows
  unsigned long long hist[20];
};

// kernels (defined in hgs_forward.cu / hgs_backward.cu / hgs_exchange.cu)
__global__ void k_depth_keys(SceneView sc, CamD cam, unsigned long long *keys, uint32_t *vals, uint32_t *hist,
                             FrameState *st);
__global__ void k_preprocess(SceneView sc, CamD cam, ModD mod, const uint32_t *sorted_idx, int64_t m, SplatRec *recs,
                             unsigned long long *pair_off, unsigned long long *scan_lb, FrameState *st);
__global__ void k_duplicate(const SplatRec *recs, const unsigned long long *pair_off, int64_t m, int tiles_x,
                            uint32_t *pkeys, uint32_t *pvals, int n_digits, uint32_t *hist);
__global__ void k_tile_ranges(const uint32_t *skeys, int64_t k, int64_t n_tiles, uint32_t *tile_off);
template <bool NAIVE>
__global__ void k_composite_fwd(CompositeArgs a);
template <int KG, bool EXT>
__global__ void k_composite_bwd(BwdArgs b);
__global__ void k_touched_scatter(const SplatRec *recs, const uint8_t *touched_rank, int64_t m, uint8_t *touched);
__global__ void k_chain_rule(ChainArgs c);
__global__ void k_exchange_scan(int64_t n, const float *log_scale, const uint8_t *type_spec, double theta_e,
                                float *eranks, ExchangeState *st);
__global__ void k_exchange_apply(int64_t n, float *log_scale, float *rotation, uint8_t *type_spec, double theta_e);

}  // namespace hgs
