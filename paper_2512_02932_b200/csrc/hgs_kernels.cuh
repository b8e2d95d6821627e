// hgs_kernels.cuh -- kernel argument blocks, frame state, and the per-pair
// evaluation shared by the forward and backward compositors.
#pragma once

#include "hgs_common.cuh"
#include "hgs_sort.cuh"

namespace hgs {

// Device-side state at the head of the frame buffer.  The scene / camera
// copies serve the rare float64 re-evaluation paths, which read them through
// a global pointer instead of (large) kernel parameters.
// The float64 projection of one splat at its depth rank, as the reference
// computes it (project.py:169-258): all a float64 pair re-check needs, so the
// re-checks never re-project the Gaussian from the scene.
struct Rec64 {
  double ctr[2];
  double alpha_eff;
  double g[9];  // 3D: conic (3); 2D: rows (0, 1, 3) x columns (0, 1, 3) of M
};
static_assert(sizeof(Rec64) == 96, "Rec64 is 96 B");

struct FrameState {
  uint32_t status;
  uint32_t m_count;
  unsigned long long k_total;
  uint32_t tile_counters[24];
  uint32_t sort_np;        // depth-sort passes (non-constant digits), set by k_sort_plan
  uint32_t sort_digit[8];  // their digit indices, low to high
  unsigned long long diag[16];  // see hgs_frame_stats in include/hgs.h
  uint32_t n_fix_fwd, n_fix_bwd;  // deferred pixels (worklist lengths)
  SceneView sc;
  CamD cam;
  ModD mod;
  const SplatRec *recs;  // float32 records (by Gaussian index) ...
  const Rec64 *recs64;   // ... and their float64 counterparts
};

// Deferred-exactness worklists.  The hot compositors contain no calls: a lane
// whose next decision is ambiguous in float32 saves its exact state here and
// retires; a fixup kernel resumes the pixel with float64-exact decisions.
struct FwdFix {       // resume the forward walk of one pixel
  uint32_t pix;       // iy * W + ix
  uint32_t entry;     // tile-list position (global index) to resume at
  uint32_t mode;      // 0: pair `entry` is ambiguous (state before it)
                      // 1: early stop after `entry` is ambiguous (state after it)
  uint32_t cnt, last;
  float T, c0, c1, c2, dep, n0, n1, n2;
  uint32_t pad[3];
};
static_assert(sizeof(FwdFix) == 64, "FwdFix is 64 B");

struct BwdFix {       // resume the backward replay of one pixel, going down
  uint32_t pix;
  uint32_t entry;     // tile-list position (global index), inclusive
  float T_run, S0, S1, S2, SD, SN0, SN1, SN2;
  uint32_t pad[6];
};
static_assert(sizeof(BwdFix) == 64, "BwdFix is 64 B");

struct CompositeArgs {
  // binning.  Records are stored by Gaussian index (the preprocess runs
  // before / beside the depth sort); tile_vals holds Gaussian indices, each
  // tile list in depth order.  NAIVE: tile_vals = the depth order itself
  // (rank -> Gaussian), lo = 0, hi = M.
  const SplatRec *recs;
  const uint32_t *tile_off;
  const uint32_t *tile_vals;
  const uint32_t *rank_of;  // Gaussian -> depth rank (SplatFrame slot)
  int64_t m;
  int tiles_x, width, height;
  uint32_t flags;
  float bg[3];
  // outputs
  float *color, *depth, *trans, *alpha, *normal;
  float *pix_T;
  uint32_t *pix_last, *pix_count;
  FrameState *st;  // diagnostics + scene / camera for float64 re-checks
  FwdFix *fwd_fix;  // (H * W) worklist
  BwdFix *bwd_fix;  // (H * W) worklist
  // the forward's exact contribution decisions, replayed by the backward:
  // bit e of word mask_word(lo, tile, c) * 256 + pixel-in-tile is set iff
  // tile-list entry lo + 32 c + e contributed to the pixel (not NAIVE)
  uint32_t *pix_mask;
  const float4 *cull2d;  // per Gaussian, 2 x float4: cull2d_prep of 2D splats
};

// L2 prefetch of one splat record (96 B: at most two 128-B lines).
__device__ __forceinline__ void prefetch_rec(const SplatRec *r) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(r));
  asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char *>(r) + 95));
}

__device__ __forceinline__ size_t mask_word(uint32_t lo, int tile, uint32_t chunk, uint32_t pix_in_tile) {
  return ((size_t)(lo >> 5) + (size_t)tile + chunk) * kBlock + pix_in_tile;
}

// log2 domain constants: at = ex2(arg), arg = log2(alpha_eff) - d * 0.5 log2(e)
constexpr float kHalfLog2e = 0.72134752044448170f;
constexpr float kArgMinAlpha = -7.99435343685885793f;  // log2(1/255)
constexpr float kArgClamp = -0.01449956969511509f;     // log2(0.99)
constexpr float kEps = 5.96046448e-8f;                 // 2^-24
constexpr float kCoarse2D = 0.05f;  // log2 units; 2D precise bounds only inside
#ifndef HGS_EXACT_ENABLED
#define HGS_EXACT_ENABLED 1  // 0: compile the compositors without the float64 re-check paths (experiments)
#endif

enum : int { kSkip = 0, kContrib = 1, kAmbiguous = 2 };  // pair decision outcomes
#ifndef HGS_FIXUP_MINB
#define HGS_FIXUP_MINB 3  // CTAs (of 256) per SM the float64 fixup kernels are register-budgeted for
#endif

__device__ __forceinline__ bool rec_is3d(const SplatRec &r) { return __float_as_uint(r.r4.w) >> 31; }
__device__ __forceinline__ uint32_t rec_idx(const SplatRec &r) { return __float_as_uint(r.r4.w) & 0x7fffffffu; }

// inclusive pixel bbox (raster/_blend_py.py:89-91)
__device__ __forceinline__ bool in_bbox(const int4 q, int ix, int iy) {
  const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16);
  const int x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
  return !(ix < x0 || ix > x1 || iy < y0 || iy > y1);
}

// 32-bit mask of the pixels of an 8 x 4 warp block (lane = row * 8 + col,
// origin (wx0, wy0)) that lie inside the inclusive bbox: bit `lane` is set iff
// in_bbox(q, wx0 + lane % 8, wy0 + lane / 8).
__device__ __forceinline__ uint32_t pixel_mask(const int4 q, int wx0, int wy0) {
  const int x0 = (q.x & 0xffff) - wx0, y0 = (int)((uint32_t)q.x >> 16) - wy0;
  const int x1 = (q.y & 0xffff) - wx0, y1 = (int)((uint32_t)q.y >> 16) - wy0;
  const int c0 = max(x0, 0), c1 = min(x1, 7), r0 = max(y0, 0), r1 = min(y1, 3);
  if (c0 > c1 || r0 > r1) return 0u;
  const uint32_t cols = (0xffu << c0) & (0xffu >> (7 - c1));
  const uint32_t rows = (0xfu << r0) & (0xfu >> (3 - r1));
  const uint32_t spread = (rows & 1u) | ((rows & 2u) << 7) | ((rows & 4u) << 14) | ((rows & 8u) << 21);
  return cols * spread;  // no carries: cols < 256, spread bits 8 apart
}

// Warp-level cull of a 3D splat whose bbox covers part of the warp's 8 x 4
// block (pixel mask pm != 0): true if no pixel centre of the covered
// rectangle can reach the 1/255 cutoff, i.e. the minimum of the conic
// quadratic form over that rectangle exceeds the cutoff distance
// d* = 2 ln(255 alpha_eff) (with a 1e-3 margin, far above float32 error, so
// a pair the evaluation would keep is never culled).  Exact minimum of a
// convex quadratic over a rectangle: 0 if the centre is inside, otherwise
// on the boundary, at the clamped 1D minimiser of each edge.
__device__ __forceinline__ bool cull_3d(const SplatRec &r, uint32_t pm, int wx0, int wy0) {
  const float dstar = (r.r0.w - kArgMinAlpha) * (1.f / kHalfLog2e);
  if (dstar < 0.f) return true;  // alpha_eff < 1/255: never contributes
  // covered rectangle of pixel centres, relative to the splat centre
  const int c0 = __ffs(pm) - 1;  // first covered lane gives the top-left
  const int c1 = 31 - __clz(pm);  // last covered lane gives the bottom-right
  const int4 q = r.r5;
  const float X0 = (float)(wx0 + (c0 & 7) - q.z) + 0.5f - r.r0.x;
  const float X1 = (float)(wx0 + (c1 & 7) - q.z) + 0.5f - r.r0.x;
  const float Y0 = (float)(wy0 + (c0 >> 3) - q.w) + 0.5f - r.r0.y;
  const float Y1 = (float)(wy0 + (c1 >> 3) - q.w) + 0.5f - r.r0.y;
  if (X0 <= 0.f && 0.f <= X1 && Y0 <= 0.f && 0.f <= Y1) return false;
  const float4 e = r.r1;  // (c, s, lambda_p, lambda_q) -> conic (a, b, c)
  const float a = fmaf(e.z * e.x, e.x, e.w * e.y * e.y), b = (e.z - e.w) * e.x * e.y;
  const float c = fmaf(e.z * e.y, e.y, e.w * e.x * e.x);
  const float ia = rcp_approx(a), ic = rcp_approx(c);
  auto qf = [&](float x, float y) { return fmaf(a * x, x, fmaf(2.f * b * x, y, c * y * y)); };
  const float ya = fminf(fmaxf(-b * X0 * ic, Y0), Y1), yb = fminf(fmaxf(-b * X1 * ic, Y0), Y1);
  const float xa = fminf(fmaxf(-b * Y0 * ia, X0), X1), xb = fminf(fmaxf(-b * Y1 * ia, X0), X1);
  const float qmin = fminf(fminf(qf(X0, ya), qf(X1, yb)), fminf(qf(xa, Y0), qf(xb, Y1)));
  return qmin > fmaf(dstar, 1.001f, 1e-3f);
}

// Minimum of the convex quadratic form a X^2 + 2b XY + c Y^2 (a, c > 0,
// ac > b^2) over the rectangle [X0, X1] x [Y0, Y1]: 0 if the origin is inside,
// otherwise on the boundary at the clamped 1D minimiser of each edge.
__device__ __forceinline__ float rect_min_quad(float a, float b, float c, float X0, float X1, float Y0, float Y1) {
  if (X0 <= 0.f && 0.f <= X1 && Y0 <= 0.f && 0.f <= Y1) return 0.f;
  const float ia = rcp_approx(a), ic = rcp_approx(c);
  auto qf = [&](float x, float y) { return fmaf(a * x, x, fmaf(2.f * b * x, y, c * y * y)); };
  const float ya = fminf(fmaxf(-b * X0 * ic, Y0), Y1), yb = fminf(fmaxf(-b * X1 * ic, Y0), Y1);
  const float xa = fminf(fmaxf(-b * Y0 * ia, X0), X1), xb = fminf(fmaxf(-b * Y1 * ia, X0), X1);
  return fminf(fminf(qf(X0, ya), qf(X1, yb)), fminf(qf(xa, Y0), qf(xb, Y1)));
}

// Warp-level cull of a 2D surfel whose bbox covers part of the warp's 8 x 4
// block: true if no covered pixel centre can reach the 1/255 cutoff through
// either branch of d = min(d_ray, d_screen) (_blend_py.py:17-44).
//  * screen branch: 4 |p - c|^2 <= d*  -- a circle of radius sqrt(d*)/2;
//  * ray branch: u^2 + v^2 <= d* with (u, v, 1) ~ adj(H) p, H = [m0'; m1'; m2]
//    the anchor-relative homography of the record -- the image of the disk
//    is the conic p^T adj(H)^T diag(1, 1, -d*) adj(H) p <= 0 (squares: no
//    sign ambiguity of the homogeneous scale).  Used only when that conic is a
//    well-conditioned ellipse; the cull needs both branches out by a 5%
//    margin in d, far above the float32 error of the conic, so a pair the
//    exact evaluation would keep is never culled (degenerate cases keep).
// The ray-branch conic depends only on the splat: cull2d_prep normalises it
// to Qn <= 1, (ca s, cb s, cc s, x0 | y0, valid), once per splat in the
// preprocess; cull_splat_pre runs the per-warp rectangle test for both types.
__device__ __forceinline__ void cull2d_prep(const SplatRec &r, float4 &k0, float4 &k1) {
  k0 = make_float4(0.f, 0.f, 0.f, 0.f);
  k1 = make_float4(0.f, 0.f, 0.f, 0.f);
  const float dstar = (r.r0.w - kArgMinAlpha) * (1.f / kHalfLog2e);
  if (dstar < 0.f) return;
  const float h00 = r.r1.x, h01 = r.r1.y, h02 = r.r1.z;
  const float h10 = r.r1.w, h11 = r.r2.x, h12 = r.r2.y;
  const float h20 = r.r2.z, h21 = r.r2.w, h22 = r.r3.x;
  const float A00 = h11 * h22 - h12 * h21, A01 = h02 * h21 - h01 * h22, A02 = h01 * h12 - h02 * h11;
  const float A10 = h12 * h20 - h10 * h22, A11 = h00 * h22 - h02 * h20, A12 = h02 * h10 - h00 * h12;
  const float A20 = h10 * h21 - h11 * h20, A21 = h01 * h20 - h00 * h21, A22 = h00 * h11 - h01 * h10;
  auto cij = [&](float a0i, float a1i, float a2i, float a0j, float a1j, float a2j) {
    return fmaf(a0i, a0j, fmaf(a1i, a1j, -dstar * a2i * a2j));
  };
  const float ca = cij(A00, A10, A20, A00, A10, A20), cb = cij(A00, A10, A20, A01, A11, A21);
  const float cc = cij(A01, A11, A21, A01, A11, A21), cd = cij(A00, A10, A20, A02, A12, A22);
  const float ce = cij(A01, A11, A21, A02, A12, A22), cf = cij(A02, A12, A22, A02, A12, A22);
  const float det = ca * cc - cb * cb;
  if (!(ca > 0.f) || !(det > 1e-3f * (ca + cc) * (ca + cc) * 0.25f)) return;
  const float idet = 1.f / det;
  const float x0 = (cb * ce - cc * cd) * idet, y0 = (cb * cd - ca * ce) * idet;
  const float fp = cf + cd * x0 + ce * y0;
  if (!(fp < -1e-2f * fabsf(cf))) return;
  const float sc = -1.f / fp;
  k0 = make_float4(ca * sc, cb * sc, cc * sc, x0);
  k1 = make_float4(y0, 1.f, 0.f, 0.f);
}

// The same test on the inclusive pixel rectangle [x0, x1] x [y0, y1]
// (absolute pixel indices, inside the splat's bbox): the warp cull of an 8 x 4
// block and the tile-level cull of the binning (tile lists hold only the
// (splat, tile) pairs some pixel of which can contribute) share it.
__device__ __forceinline__ bool cull_rect(const SplatRec &r, const float4 *c2, int x0, int y0, int x1, int y1) {
  const float dstar = (r.r0.w - kArgMinAlpha) * (1.f / kHalfLog2e);
  if (dstar < 0.f) return true;  // alpha_eff < 1/255: never contributes
  const int4 q = r.r5;
  const float PX0 = (float)(x0 - q.z) + 0.5f, PX1 = (float)(x1 - q.z) + 0.5f;
  const float PY0 = (float)(y0 - q.w) + 0.5f, PY1 = (float)(y1 - q.w) + 0.5f;
  float A, B, C, cx, cy, thr;
  if (rec_is3d(r)) {
    const float4 e = r.r1;  // (c, s, lambda_p, lambda_q) -> conic (A, B, C)
    A = fmaf(e.z * e.x, e.x, e.w * e.y * e.y);
    B = (e.z - e.w) * e.x * e.y;
    C = fmaf(e.z * e.y, e.y, e.w * e.x * e.x);
    cx = r.r0.x; cy = r.r0.y;
    thr = fmaf(dstar, 1.001f, 1e-3f);
  } else {
    const float ex = fmaxf(fmaxf(PX0 - r.r0.x, r.r0.x - PX1), 0.f);
    const float ey = fmaxf(fmaxf(PY0 - r.r0.y, r.r0.y - PY1), 0.f);
    if (4.f * (ex * ex + ey * ey) <= fmaf(dstar, 1.05f, 1e-3f)) return false;  // low-pass circle reaches
    const float4 k0 = c2[0], k1 = c2[1];
    if (!(k1.y > 0.f)) return false;  // no well-conditioned ray conic: keep
    A = k0.x; B = k0.y; C = k0.z;
    cx = k0.w; cy = k1.x;
    thr = 1.05f;
  }
  return rect_min_quad(A, B, C, PX0 - cx, PX1 - cx, PY0 - cy, PY1 - cy) > thr;
}

__device__ __forceinline__ bool cull_splat_pre(const SplatRec &r, const float4 *c2, uint32_t pm, int wx0, int wy0) {
  const int c0 = __ffs(pm) - 1, c1 = 31 - __clz(pm);  // pm is a rectangle (pixel_mask)
  return cull_rect(r, c2, wx0 + (c0 & 7), wy0 + (c0 >> 3), wx0 + (c1 & 7), wy0 + (c1 >> 3));
}

// cull_rect split into its per-splat part (once) and its per-rectangle
// part: the same arithmetic, so the decisions are identical.
struct TileCull {
  float A, B, C, cx, cy, thr, dlow, rcx, rcy;
  int ax, ay;
  bool never, is3d, conic;
};
__device__ __forceinline__ TileCull tile_cull_prep(const SplatRec &r, const float4 *c2) {
  TileCull t;
  const float dstar = (r.r0.w - kArgMinAlpha) * (1.f / kHalfLog2e);
  t.never = dstar < 0.f;
  t.is3d = rec_is3d(r);
  t.ax = r.r5.z;
  t.ay = r.r5.w;
  t.rcx = r.r0.x;
  t.rcy = r.r0.y;
  t.dlow = fmaf(dstar, 1.05f, 1e-3f);
  t.conic = true;
  if (t.is3d) {
    const float4 e = r.r1;
    t.A = fmaf(e.z * e.x, e.x, e.w * e.y * e.y);
    t.B = (e.z - e.w) * e.x * e.y;
    t.C = fmaf(e.z * e.y, e.y, e.w * e.x * e.x);
    t.cx = r.r0.x; t.cy = r.r0.y;
    t.thr = fmaf(dstar, 1.001f, 1e-3f);
  } else {
    const float4 k0 = c2[0], k1 = c2[1];
    t.conic = k1.y > 0.f;
    t.A = k0.x; t.B = k0.y; t.C = k0.z;
    t.cx = k0.w; t.cy = k1.x;
    t.thr = 1.05f;
  }
  return t;
}
// true: no pixel centre of [x0, x1] x [y0, y1] can reach the cutoff
__device__ __forceinline__ bool tile_cull_test(const TileCull &t, int x0, int y0, int x1, int y1) {
  if (t.never) return true;
  const float PX0 = (float)(x0 - t.ax) + 0.5f, PX1 = (float)(x1 - t.ax) + 0.5f;
  const float PY0 = (float)(y0 - t.ay) + 0.5f, PY1 = (float)(y1 - t.ay) + 0.5f;
  if (!t.is3d) {
    const float ex = fmaxf(fmaxf(PX0 - t.rcx, t.rcx - PX1), 0.f);
    const float ey = fmaxf(fmaxf(PY0 - t.rcy, t.rcy - PY1), 0.f);
    if (4.f * (ex * ex + ey * ey) <= t.dlow) return false;  // low-pass circle reaches
    if (!t.conic) return false;                             // no well-conditioned ray conic: keep
  }
  return rect_min_quad(t.A, t.B, t.C, PX0 - t.cx, PX1 - t.cx, PY0 - t.cy, PY1 - t.cy) > t.thr;
}

// Tile-level cull of the binning: splats whose bbox spans at most
// kTileCullMax tiles list only the tiles whose part of the bbox the support
// can reach (35% of the bbox pairs at config 2 have no contributing pixel).
// k_tile_counts decides once per tile (tile_cull_prep / tile_cull_test) and
// k_duplicate emits exactly the kept bits, so counts and pairs agree.
constexpr int kTileCullMax = 32;

#ifndef HGS_CULL_2D
#define HGS_CULL_2D 1
#endif
#ifndef HGS_CULL_PRE
#define HGS_CULL_PRE 1
#endif
#ifndef HGS_STAGED_ORIGIN
#define HGS_STAGED_ORIGIN 1  // compositors stage records with the float block origin
#endif
__device__ __forceinline__ bool cull_splat(const SplatRec &r, uint32_t pm, int wx0, int wy0) {
  if (rec_is3d(r)) return cull_3d(r, pm, wx0, wy0);
  if (!HGS_CULL_2D) return false;
  float4 k[2];
  cull2d_prep(r, k[0], k[1]);  // per warp instead of once per splat (HGS_CULL_PRE = 0)
  return cull_splat_pre(r, k, pm, wx0, wy0);
}

// Staged-record form of the anchor (see eval_fast<..., STAGED>): exact while
// |wx0 - ax| < 2^22, i.e. for every pixel within 4M pixels of the anchor.
__device__ __forceinline__ void stage_block_origin(SplatRec &r, int wx0, int wy0) {
  r.r5.z = __float_as_int(__fadd_rn((float)(wx0 - r.r5.z), 0.5f));
  r.r5.w = __float_as_int(__fadd_rn((float)(wy0 - r.r5.w), 0.5f));
}

// bbox overlaps the pixel rectangle [rx0, rx1] x [ry0, ry1]
__device__ __forceinline__ bool bbox_overlaps(const int4 q, int rx0, int ry0, int rx1, int ry1) {
  const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16);
  const int x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
  return !(x1 < rx0 || x0 > rx1 || y1 < ry0 || y0 > ry1);
}

// Result of evaluating one (pixel, splat) pair.
struct PairEval {
  float at;       // clamped alpha
  float dx, dy;   // pixel - centre (pixels)
  float u, v;     // 3D: (dx, dy); 2D: tangent-plane intersection
  float hu0, hu1, hu3, hv0, hv1, hv3, inv_den;  // 2D ray quantities
  float wp, wq;   // 3D: lambda_p p, lambda_q q (the conic times the offset, in the eigenbasis)
  float pxl, pyl; // pixel relative to the anchor
  bool ray;       // 2D: ray branch chosen (d_ray <= d_screen)
  bool clamped;   // raw alpha > 0.99 (colour-only gradient)
};

// float64 re-evaluation of one pair exactly as the reference does it
// (_blend_py.py:17-44, 96-100), from the splat's stored float64 projection.
// Returns false if the pair is skipped.
static __device__ __noinline__ bool pair_f64(const Rec64 *q, bool is3d, int ix, int iy, double *at_out,
                                             bool *ray_out, bool *clamped_out) {
  const Rec64 o = *q;
  const double px = ix + 0.5, py = iy + 0.5;
  const double dx = px - o.ctr[0], dy = py - o.ctr[1];
  double d;
  bool ray = false;
  if (is3d) {
    d = (o.g[0] * dx * dx + 2.0 * o.g[1] * dx * dy) + o.g[2] * dy * dy;
  } else {
    const double *m = o.g;  // (m00 m01 m03 | m10 m11 m13 | m30 m31 m33)
    double hu0 = px * m[6] - m[0], hu1 = px * m[7] - m[1], hu3 = px * m[8] - m[2];
    double hv0 = py * m[6] - m[3], hv1 = py * m[7] - m[4], hv3 = py * m[8] - m[5];
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

// The float32 pair geometry.  Explicit fmaf / __fmul_rn / __fadd_rn so the
// inline fast path and the out-of-line resolver compute identical bits.
struct Geom {
  float dx, dy, pxl, pyl;
  float d, arg, wp, wq, m;                       // 3D: eigenbasis terms, m = |dx| + |dy|
  float hu0, hu1, hu3, hv0, hv1, hv3, den, dmag;  // 2D
  float inv_den, u, v, dray, dscr;               // 2D
  bool ray;
};

__device__ __forceinline__ void geom_common(const SplatRec &r, int ix, int iy, Geom &g) {
  const int4 q = r.r5;
  g.pxl = __fadd_rn((float)(ix - q.z), 0.5f);
  g.pyl = __fadd_rn((float)(iy - q.w), 0.5f);
  g.dx = __fsub_rn(g.pxl, r.r0.x);
  g.dy = __fsub_rn(g.pyl, r.r0.y);
}

// 3D record: r1 = (c, s, lambda_p, lambda_q), the conic's eigenbasis, r2 =
// (P0, Q0, |P0| + |Q0|, 0) the anchor's rotated offset from the centre
// (write_record).  (p, q) = (P0 + c pxl + s pyl, Q0 + c pyl - s pxl), the
// pixel's rotated offset; d = lambda_p p^2 + lambda_q q^2.
// Float32 error: |p error|, |q error| <= eps (2m + |p|), m = |P0| + |Q0| +
// |pxl| + |pyl|, so |d error| <= eps (6 d + 4 m (lambda_p |p| + lambda_q |q|)).
__device__ __forceinline__ void geom_3d(const SplatRec &r, Geom &g) {
  const float4 e = r.r1, o = r.r2;
  const float p = fmaf(e.x, g.pxl, fmaf(e.y, g.pyl, o.x));
  const float q = fmaf(e.x, g.pyl, fmaf(-e.y, g.pxl, o.y));
  g.wp = __fmul_rn(e.z, p);
  g.wq = __fmul_rn(e.w, q);
  g.d = fmaf(g.wp, p, __fmul_rn(g.wq, q));
  g.arg = fmaf(g.d, -kHalfLog2e, r.r0.w);
  g.m = __fadd_rn(o.z, __fadd_rn(fabsf(g.pxl), fabsf(g.pyl)));
}

// Coarse 3D band (log2 units): inside it the precise bound is formed.  Valid
// while m < kCoarseM3D: with conic eigenvalues <= 1 / 0.3 (the dilation) the
// bound above stays below the band for every d.
constexpr float kCoarse3D = 0.05f;
constexpr float kCoarseM3D = 8192.f;

__device__ __forceinline__ void geom_2d_rows(const SplatRec &r, Geom &g) {
  const float4 m1 = r.r1, m2 = r.r2;
  const float m23 = r.r3.x;
  // rows re-based at the anchor: hu = pxl m2 - m0', hv = pyl m2 - m1'
  g.hu0 = fmaf(g.pxl, m2.z, -m1.x);
  g.hu1 = fmaf(g.pxl, m2.w, -m1.y);
  g.hu3 = fmaf(g.pxl, m23, -m1.z);
  g.hv0 = fmaf(g.pyl, m2.z, -m1.w);
  g.hv1 = fmaf(g.pyl, m2.w, -m2.x);
  g.hv3 = fmaf(g.pyl, m23, -m2.y);
  const float a = __fmul_rn(g.hu0, g.hv1), b = __fmul_rn(g.hu1, g.hv0);
  g.den = __fsub_rn(a, b);
  g.dmag = __fadd_rn(fabsf(a), fabsf(b));
}

__device__ __forceinline__ void geom_2d_solve(const SplatRec &r, Geom &g) {
  g.inv_den = rcp_approx(g.den);  // MUFU.RCP: no out-of-line slow path in the hot loop
  g.u = __fmul_rn(__fsub_rn(__fmul_rn(g.hu1, g.hv3), __fmul_rn(g.hu3, g.hv1)), g.inv_den);
  g.v = __fmul_rn(__fsub_rn(__fmul_rn(g.hu3, g.hv0), __fmul_rn(g.hu0, g.hv3)), g.inv_den);
  g.dray = fmaf(g.u, g.u, __fmul_rn(g.v, g.v));
  g.dscr = __fmul_rn(fmaf(g.dx, g.dx, __fmul_rn(g.dy, g.dy)), 4.f);
  g.ray = g.dray <= g.dscr;
  g.d = g.ray ? g.dray : g.dscr;
  g.arg = fmaf(g.d, -kHalfLog2e, r.r0.w);
}

__device__ __forceinline__ bool near_degenerate(const Geom &g) {
  return fabsf(g.den) <= fmaf(g.dmag, 1e-4f, (float)kDegenerateDen);
}

// Outcome of the out-of-line resolver.
struct Resolved {
  float at;
  uint32_t flags;  // bit0 contributes, bit1 clamped, bit2 ray branch
};

// Out-of-line: exact decisions for a pair the fast path found ambiguous.
// 2D pairs first get a first-order float32 error bound of the 2x2 solve;
// anything still ambiguous is re-evaluated in float64 (pair_f64).
// Precise first-order float32 error bound of a 2D pair that the coarse band
// flagged (pure FP32 arithmetic, no calls: safe on the hot path).  Returns
// kSkip / kContrib when the bound separates every decision, kAmbiguous if not.
__device__ __forceinline__ int refine_2d(const SplatRec &r, const Geom &g, bool bwd, bool known = false) {
  const float4 m1 = r.r1, m2 = r.r2;
  const float m23 = r.r3.x;
  const float A0 = fabsf(g.pxl * m2.z) + fabsf(m1.x), A1 = fabsf(g.pxl * m2.w) + fabsf(m1.y);
  const float A3 = fabsf(g.pxl * m23) + fabsf(m1.z);
  const float B0 = fabsf(g.pyl * m2.z) + fabsf(m1.w), B1 = fabsf(g.pyl * m2.w) + fabsf(m2.x);
  const float B3 = fabsf(g.pyl * m23) + fabsf(m2.y);
  const float ad = fabsf(g.den);
  const float dden = 6.f * kEps * (A0 * B1 + A1 * B0);
  // |den| is only trusted when its error bound is a small fraction of it
  // (near-degenerate pairs: the reciprocal below must not blow up); then
  // |true den| >= ad - dden makes the (u, v) bounds rigorous, not first-order
  if (!(ad > (float)kDegenerateDen + dden) || !(ad > 32.f * dden)) return kAmbiguous;
  const float iad = rcp_approx(ad - dden) * (1.f + 4.f * kEps);
  const float du = (6.f * kEps * (A1 * B3 + A3 * B1) + fabsf(g.u) * dden) * iad + 4.f * kEps * fabsf(g.u);
  const float dv = (6.f * kEps * (A3 * B0 + A0 * B3) + fabsf(g.v) * dden) * iad + 4.f * kEps * fabsf(g.v);
  // (|u| + du)^2 - u^2 = 2|u| du + du^2 (likewise v)
  const float e_ray = fmaf(du, du, dv * dv) + 2.f * (fabsf(g.u) * du + fabsf(g.v) * dv) + 4.f * kEps * g.dray;
  const float e_scr = 8.f * kEps * g.dscr + 1e-6f * (fabsf(g.dx) + fabsf(g.dy));
  const float margin = fmaf(g.ray ? e_ray : e_scr, kHalfLog2e, 1e-5f);
  if (!(margin < kCoarse2D)) return kAmbiguous;
  if (!known) {  // known: the forward's exact decision says the pair contributes
    if (g.arg < kArgMinAlpha - margin) return kSkip;
    if (g.arg <= kArgMinAlpha + margin) return kAmbiguous;
  }
  if (bwd && (fabsf(g.arg - kArgClamp) <= margin || fabsf(g.dray - g.dscr) <= e_ray + e_scr)) return kAmbiguous;
  return kContrib;
}

static __device__ __noinline__ Resolved resolve_pair(const SplatRec *rp, int ix, int iy, FrameState *st, bool bwd) {
  const SplatRec r = *rp;
  Geom g;
  geom_common(r, ix, iy, g);
  Resolved out{0.f, 0u};
  if (!rec_is3d(r)) {
    geom_2d_rows(r, g);
    if (!near_degenerate(g)) {
      geom_2d_solve(r, g);
      const int c = refine_2d(r, g, bwd);
      if (c == kSkip) return out;
      if (c == kContrib) {
        const bool cl = g.arg > kArgClamp;
        out.at = cl ? 0.99f : ex2_approx(g.arg);
        out.flags = 1u | (cl ? 2u : 0u) | (g.ray ? 4u : 0u);
        return out;
      }
    }
  }
  atomicAdd(&st->diag[0], 1ull);
  double at64;
  bool ray64, cl64;
  if (!pair_f64(st->recs64 + (rp - st->recs), rec_is3d(r), ix, iy, &at64, &ray64, &cl64)) return out;
  out.at = (float)at64;
  out.flags = 1u | (cl64 ? 2u : 0u) | (ray64 ? 4u : 0u);
  return out;
}


// Evaluate a pair in float32 (fast path, no calls).  BWD additionally needs
// the backward-only decisions (ray branch, clamp) and the 2D solve
// quantities.  Returns kSkip, kContrib, or kAmbiguous -- the caller then runs
// resolve_pair (out of line) and applies finish_resolved.
// KNOWN (backward with contribution masks): the forward already decided,
// exactly, that the pair contributes -- only the backward-only decisions
// (clamp, ray branch, degenerate solve) are checked.
// STAGED: r is a compositor's shared-memory copy whose r5.z / r5.w hold the
// float anchor-relative centre of the warp block's first pixel,
// (wx0 - ax) + 0.5 (stage_block_origin), and (ox, oy) is the pixel's offset
// in the block: pxl = that + ox is the same exact value as (ix - ax) + 0.5.
// EXM: 1 exact decisions, 0 HGS_FLAG_FAST, 2 read from flags at run time
// (the hot compositors are instantiated per mode: no per-pair flag test).
template <bool BWD, bool KNOWN = false, bool STAGED = false, int EXM = 2>
__device__ __forceinline__ int eval_fast(const SplatRec &r, int ix, int iy, uint32_t flags, PairEval &p,
                                         float ox = 0.f, float oy = 0.f) {
  Geom g;
  if (STAGED) {
    g.pxl = __fadd_rn(__int_as_float(r.r5.z), ox);
    g.pyl = __fadd_rn(__int_as_float(r.r5.w), oy);
    g.dx = __fsub_rn(g.pxl, r.r0.x);
    g.dy = __fsub_rn(g.pyl, r.r0.y);
  } else {
    geom_common(r, ix, iy, g);
  }
  p.dx = g.dx;
  p.dy = g.dy;
  p.pxl = g.pxl;
  p.pyl = g.pyl;
  const bool exact = HGS_EXACT_ENABLED && (EXM == 2 ? !(flags & HGS_FLAG_FAST) : EXM == 1);
  bool amb = false;
  p.ray = false;
  if (rec_is3d(r)) {
    geom_3d(r, g);
    p.u = g.dx;
    p.v = g.dy;
    p.wp = g.wp;
    p.wq = g.wq;
    // cheap cull (no ex2): outside the coarse band no bound is needed
    if (!KNOWN && g.arg < (exact ? kArgMinAlpha - kCoarse3D : kArgMinAlpha) && (!exact || g.m < kCoarseM3D))
      return kSkip;
    if (exact && ((!KNOWN && g.arg <= kArgMinAlpha + kCoarse3D) || (BWD && fabsf(g.arg - kArgClamp) <= kCoarse3D) ||
                  !(g.m < kCoarseM3D))) {
      // |d error| <= eps (6 d + 4 m (|wp| + |wq|)), 25% slack
      const float margin =
          fmaf(fmaf(4.f * g.m, fabsf(g.wp) + fabsf(g.wq), 6.f * g.d), 1.25f * kEps * kHalfLog2e, 1e-5f);
      if (!KNOWN && g.arg < kArgMinAlpha - margin) return kSkip;
      if ((!KNOWN && g.arg <= kArgMinAlpha + margin) || (BWD && fabsf(g.arg - kArgClamp) <= margin)) amb = true;
    }
  } else {
    geom_2d_rows(r, g);
    // (near-)degenerate ray/plane intersection (_blend_py.py:36-37): outside
    // the coarse-band regime, so its decisions always take the precise bound
    // (refine_2d leaves them ambiguous unless |den| clears its error bound)
    const bool nd = near_degenerate(g);
    if (nd && !exact && fabsf(g.den) < (float)kDegenerateDen) return kSkip;
    geom_2d_solve(r, g);
    if ((!nd || !exact) && !KNOWN && g.arg < kArgMinAlpha - (exact ? kCoarse2D : 0.f)) return kSkip;
    if (exact && (nd || (!KNOWN && g.arg <= kArgMinAlpha + kCoarse2D) ||
                  (BWD && (fabsf(g.arg - kArgClamp) <= kCoarse2D ||
                           fabsf(g.dray - g.dscr) <= 0.02f * (g.dray + g.dscr))))) {
      // coarse band hit: the precise bound usually separates the decision
      const int c = refine_2d(r, g, BWD, KNOWN);
      if (c == kSkip) return kSkip;
      amb = c == kAmbiguous;
    }
    p.ray = g.ray;
    if (BWD) {
      p.hu0 = g.hu0; p.hu1 = g.hu1; p.hu3 = g.hu3;
      p.hv0 = g.hv0; p.hv1 = g.hv1; p.hv3 = g.hv3;
      p.inv_den = g.inv_den;
      p.u = g.u;
      p.v = g.v;
    }
  }
  if (amb) return kAmbiguous;
  p.clamped = g.arg > kArgClamp;
  p.at = p.clamped ? 0.99f : ex2_approx(g.arg);
  return kContrib;
}

__device__ __forceinline__ bool finish_resolved(const Resolved rs, PairEval &p) {
  if (!(rs.flags & 1u)) return false;
  p.at = rs.at;
  p.clamped = rs.flags & 2u;
  p.ray = rs.flags & 4u;
  return true;
}

// Convenience form with the call inline (used off the hot loops).
template <bool BWD>
__device__ __forceinline__ bool eval_pair(const SplatRec &r, const SplatRec *rp, int ix, int iy, uint32_t flags,
                                          FrameState *st, PairEval &p) {
  const int c = eval_fast<BWD>(r, ix, iy, flags, p);
  if (c != kAmbiguous) return c == kContrib;
  return finish_resolved(resolve_pair(rp, ix, iy, st, BWD), p);
}

// Early-stop decision T < 1e-4 (_blend_py.py:111-113).  Near the threshold the
// pixel's transmittance is replayed in float64 over its tile list.
// Warp-cooperative: all 32 lanes call it with the same arguments.  32 entries
// per step, each lane evaluates its entry with the exact decisions and the
// float64 alpha; the float64 factors are multiplied across the warp.
#ifndef HGS_REPLAY_E
#define HGS_REPLAY_E 4  // tile-list entries per lane per step of the float64 transmittance replay
#endif
// Float64 transmittance of pixel (ix, iy) after tile-list entries lo..upto,
// exactly as the reference accumulates it (_blend_py.py:104-113).  Each pair's
// contribution decision and alpha come straight from its float64 evaluation
// (pair_f64 -- the decision the float32 path reproduces), 32 x HGS_REPLAY_E
// entries per step so the serial chain of a deep replay is short.
static __device__ __noinline__ bool replay_T_below(const SplatRec *recs, const uint32_t *tile_vals, uint32_t flags,
                                                   FrameState *st, uint32_t lo, uint32_t upto, int ix, int iy) {
  constexpr int E = HGS_REPLAY_E;
  const int lane = threadIdx.x & 31;
  if (lane == 0) atomicAdd(&st->diag[1], 1ull);
  const bool naive = flags & HGS_FLAG_NAIVE;
  double T = 1.0;
  for (uint32_t base = lo; base <= upto; base += 32 * E) {
    double om = 1.0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const uint32_t j = base + (uint32_t)(32 * i + lane);
      if (j <= upto) {
        const uint32_t rk = tile_vals[j];  // NAIVE: the depth order
        const SplatRec *g = recs + rk;
        if (naive || in_bbox(__ldg(&g->r5), ix, iy)) {
          double at64;
          bool ray64, cl64;
          if (pair_f64(st->recs64 + rk, __float_as_uint(__ldg(&g->r4.w)) >> 31, ix, iy, &at64, &ray64, &cl64))
            om *= 1.0 - at64;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) om *= __shfl_xor_sync(0xffffffffu, om, o);
    T *= om;
  }
  return T < kEarlyStopT;
}

// Global per-Gaussian gradient accumulators are float64: a warp's partial
// sums (<= 128 pixels) are float32, but a splat covering the whole image sums
// ~2M contributions of random sign (the upstream pixel gradients) that cancel
// to ~1/sqrt(N) of their absolute sum; float32 atomics then carry errors of
// 1e-3 relative, and the 3D chain rule of a near-camera, far-off-axis Gaussian
// amplifies dL/dcov2d errors ~100x through the cancelling Jacobian terms
// (config-5 orbit view 16: 9% centre-gradient error on two such Gaussians).
using acc_t = double;

struct BwdArgs {
  CompositeArgs c;          // recs, tile lists, flags, bg, state
  const float *pix_grad;    // (KG, H, W, 3)
  const float *depth_grad;  // (KG, H, W) or null
  const float *normal_grad; // (KG, H, W, 3) or null
  const float *alpha_grad;  // (KG, H, W) or null
  acc_t *acc;               // (n, KG, 16)
  acc_t *acc_ext;           // (n, KG, 4) or null
  uint8_t *touched;         // (n) by Gaussian index, zeroed by the caller
  // HGS_FLAG_DETERMINISTIC: per-(splat, warp) / per-(splat, pixel) records
  // instead of atomics; sorted by key and reduced in key order afterwards
  unsigned long long *rec_keys;  // (rec_cap) gidx << 32 | tile << 9 | sub
  uint32_t *rec_vals;            // (rec_cap) record index (the sort's values)
  float *rec_pay;                // (rec_cap, KG * 20): 16 slots + 4 extension slots per kg
  uint32_t *rec_count;
  uint32_t rec_cap;
};

// sub-key of a deterministic-mode record: the warp (main kernel) or 4 + the
// pixel within its tile (fixup kernel) -- unique per (Gaussian, tile)
__device__ __forceinline__ unsigned long long det_key(uint32_t gidx, uint32_t tile, uint32_t sub) {
  return ((unsigned long long)gidx << 32) | ((unsigned long long)tile << 9) | sub;
}

struct ChainArgs {
  SceneView sc;
  CamD cam;
  ModD mod;
  const acc_t *acc;      // (n, KG, 16)
  const acc_t *acc_ext;  // (n, KG, 4) or null
  int kg;
  float *grads;          // (KG, n*P) field-major blocks
  const float2 *eig;     // (n) a 3D splat's float32 eigenbasis (c, s), by Gaussian index
  int64_t g0, g1;        // Gaussian range of this launch
  int accumulate;        // grads += (HGS_FLAG_ACCUMULATE) instead of =
  const uint8_t *touched = nullptr;  // hgs_backward: the replay's touched mask (a superset of the
                                     // Gaussians with a nonzero accumulator), or null: test the slots
};

struct ExchangeState {
  unsigned long long counts[4];  // demote, promote, n3 before, degenerate rows
  unsigned long long hist[20];
};

// kernels (defined in hgs_forward.cu / hgs_backward.cu / hgs_exchange.cu)
__global__ void k_init_state(SceneView sc, CamD cam, ModD mod, const SplatRec *recs, const Rec64 *recs64,
                             FrameState *st);
__global__ void k_init_bwd(SceneView sc, CamD cam, ModD mod, const SplatRec *recs, const Rec64 *recs64,
                           FrameState *st, uint32_t *rec_count, int zero_diag);
cudaError_t launch_depth_keys(const SceneView &sc, const CamD &cam, unsigned long long *keys, uint32_t *vals,
                              uint8_t *kept, uint32_t *hist, FrameState *st, int grid, cudaStream_t s);
__global__ void k_rank_scatter(const uint32_t *vals_a, const uint32_t *vals_b, const FrameState *st, int64_t n,
                               uint32_t *rank_of, uint32_t *order);
cudaError_t launch_preprocess(const SceneView &sc, const CamD &cam, const ModD &mod, const uint8_t *kept,
                              SplatRec *recs, Rec64 *recs64, float4 *cull2d, float2 *eig, uint32_t *counts,
                              cudaStream_t s);
__global__ void k_scan_counts(const uint32_t *counts, const uint32_t *order, int64_t m, unsigned long long *pair_off,
                              unsigned long long *scan_lb, FrameState *st, int64_t cap);
__global__ void k_tile_counts(const SplatRec *recs, const float4 *cull2d, int64_t n, uint32_t *counts,
                              uint32_t *keep);
__global__ void k_rebin_counts(const SplatRec *recs, const uint32_t *order, int64_t m, int tile_shift,
                               uint32_t *counts);
__global__ void k_duplicate(const SplatRec *recs, const uint32_t *order, const unsigned long long *pair_off, int64_t m,
                            const FrameState *st, int tiles_x, int tile_shift, bool emit_rank, bool tile_cull,
                            const uint32_t *keep, uint32_t *pkeys, uint32_t *pvals, int n_digits, uint32_t *hist);
__global__ void k_tile_ranges(const uint32_t *skeys, int64_t k, const FrameState *st, int64_t n_tiles,
                              uint32_t *tile_off);
__global__ void k_sort_plan(const uint32_t *hist, int64_t n, uint32_t *offsets, FrameState *st);
// Host launchers of the template kernels (each instantiated and launched in
// its own translation unit).
cudaError_t launch_composite_fwd(const CompositeArgs &a, int64_t n_tiles, bool naive, bool count, cudaStream_t s);
__global__ void k_fixup_fwd(CompositeArgs a);
__global__ void k_pixel_counts(CompositeArgs a, uint32_t *counts);
// backward compositor (compacted, or naive) + the float64 fixup of deferred pixels
cudaError_t launch_composite_bwd(const BwdArgs &b, int kg, int64_t n_tiles, bool ext, bool det, cudaStream_t s);
__global__ void k_det_reduce(const unsigned long long *keys, const uint32_t *vals, const float *pay, int64_t nrec,
                             int kg, acc_t *acc, acc_t *acc_ext);
cudaError_t launch_chain_rule(const ChainArgs &c, int sh_bases, int grid, size_t smem, cudaStream_t s);
// the frame's per-Gaussian 3D eigenbasis array (hgs_api.cu layout)
const float2 *frame_eig(const void *frame, const hgs_frame_info *info);
template <typename T>
cudaError_t launch_exchange_scan(int64_t n, const T *log_scale, const uint8_t *type_spec, double theta_e, T *eranks,
                                 ExchangeState *st, int grid, cudaStream_t s);
template <typename T>
cudaError_t launch_exchange_apply(int64_t n, T *log_scale, T *rotation, uint8_t *type_spec, double theta_e, int grid,
                                  cudaStream_t s);

}  // namespace hgs
