// hgs_common.cuh -- shared device code for libhgs.so (sm_100a).
//
// Precision plan:
//  * per-Gaussian preprocess runs in float64 (B200 DFMA = 1/2 the FP32 rate,
//    measured 33.8 TFLOP/s), so depth keys, bounding boxes and tile lists are
//    the reference's float64 decisions;
//  * the compositor runs in float32 on a packed per-splat record whose
//    coordinates are stored relative to an integer anchor pixel (no
//    cancellation against absolute pixel coordinates);
//  * near-threshold compositor decisions are re-evaluated in float64 from the
//    scene (project_f64 below) unless HGS_FLAG_FAST is set.
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/hgs.h"

namespace hgs {

// Programmatic dependent launch (Hopper / Blackwell): a kernel launched with
// launch_pdl() may be scheduled while its predecessor on the stream drains
// (each predecessor CTA signals pdl_launch_dependents() when it starts);
// pdl_wait() then blocks until the predecessor has completed and its writes
// are visible.  Every PDL-launched kernel calls pdl_wait() before touching
// global memory, so the ordering is that of a plain launch minus the launch
// gap.  Both are no-ops for kernels launched without the attribute.
#ifndef HGS_PDL
#define HGS_PDL 1
#endif
#ifndef HGS_DEPTH_SORT_TRIGGER
#define HGS_DEPTH_SORT_TRIGGER 0  // early triggers along the depth sort's chain (see hgs_api.cu)
#endif
__device__ __forceinline__ void pdl_launch_dependents() {
#if HGS_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if HGS_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (HGS_PDL && pdl) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
  return launch_ex(true, kernel, grid, block, smem, s, std::forward<Args>(args)...);
}

constexpr int kTile = 16;
constexpr int kTileShift = 4;  // log2(kTile)
constexpr int kBlock = kTile * kTile;  // one thread per pixel of a tile
#ifndef HGS_FIXUP_BLOCKS
#define HGS_FIXUP_BLOCKS (148 * 4)
#endif
constexpr int kFixupBlocks = HGS_FIXUP_BLOCKS;     // persistent fixup grids (one warp per deferred pixel)
constexpr double kAlphaClamp = 0.99;   // raster/project.py:20
constexpr double kMinAlpha = 1.0 / 255.0;
constexpr double kEarlyStopT = 1e-4;
constexpr double kDilation = 0.3;
constexpr double kLowpassSigma = 0.5;
constexpr double kDegenerateDen = 1e-9;
constexpr double kBBoxPad = 1.0;
constexpr double kInvLp2 = 1.0 / (kLowpassSigma * kLowpassSigma);  // _blend_py.py:14
constexpr double kQuatMinNorm = 1e-8;
constexpr double kSupportC = 11.08252709086190;  // 2 ln 255 (project.py:25)

// Scene pointers as kernels see them.
struct SceneView {
  const float *center, *log_scale, *rotation, *opacity_logit, *sh;
  const uint8_t *type_spec;
  int64_t n;
  int sh_bases;
  // optional float64 geometry (hgs.h): the decisions of the forward are taken
  // on these when set (all four or none)
  const double *center64, *log_scale64, *rotation64, *opacity_logit64;
};

// Geometry loads of the float64 preprocess.  G64 = the scene carries the
// float64 copy (the reference's own inputs); otherwise the float32 fields are
// widened.  A template parameter, not a runtime test, so the float32 path's
// code is unchanged.
template <bool G64>
struct SceneGeom {
  static __device__ __forceinline__ double center(const SceneView &sc, int64_t i, int k) {
    return G64 ? sc.center64[3 * i + k] : (double)sc.center[3 * i + k];
  }
  static __device__ __forceinline__ double log_scale(const SceneView &sc, int64_t i, int k) {
    return G64 ? sc.log_scale64[3 * i + k] : (double)sc.log_scale[3 * i + k];
  }
  static __device__ __forceinline__ double rotation(const SceneView &sc, int64_t i, int k) {
    return G64 ? sc.rotation64[4 * i + k] : (double)sc.rotation[4 * i + k];
  }
  static __device__ __forceinline__ double opacity_logit(const SceneView &sc, int64_t i) {
    return G64 ? sc.opacity_logit64[i] : (double)sc.opacity_logit[i];
  }
};

// Camera in float64, precomputed on the host.
struct CamD {
  double V[9];   // world->camera rotation (row-major)
  double tv[3];  // world->camera translation
  double T[16];  // K @ W (types.py:189-197)
  double campos[3];
  double fx, fy, cx, cy, near_plane;
  int width, height, tiles_x, tiles_y;
};

struct ModD {
  double theta_z, t_z, lambda_z;
};

// ---------------------------------------------------------------- records
// Rank-ordered float32 splat record consumed by the compositors, 6 x 16 B.
//  r0 = (lx, ly, depth, log2 alpha_eff) centre relative to anchor pixel
//  r1 = 3D: (c, s, lambda_p, lambda_q) the conic's eigenbasis
//       2D: (m0'0, m0'1, m0'3, m1'0)
//  r2 = 2D: (m1'1, m1'3, m2_0, m2_1)
//       3D: (P0, Q0, |P0| + |Q0|, 0) the anchor's offset from the centre in
//           the eigenbasis (a 3D anchor is clamped to the image)
//  r3 = (m2_3 | 0, red, green, blue)
//  r4 = (nx, ny, nz, bits(idx | typ << 31))
//  r5 = int: (x0 | y0 << 16, x1 | y1 << 16, anchor_x, anchor_y)
// where m0' = M[0] - ax M[3], m1' = M[1] - ay M[3] (rows of the splat->pixel
// map, project.py:234-243, re-based at the anchor in float64).
struct __align__(16) SplatRec {
  float4 r0, r1, r2, r3, r4;
  int4 r5;
};
static_assert(sizeof(SplatRec) == 96, "record must be 96 B");

// ------------------------------------------------------------------ math

__device__ __forceinline__ double expit_d(double x) { return 1.0 / (1.0 + exp(-x)); }

// core/sh.py:32-60
template <typename F>
__device__ __forceinline__ void sh_basis_t(int deg, F x, F y, F z, F *o);

__device__ __forceinline__ void sh_basis_d(int deg, double x, double y, double z, double *o) {
  sh_basis_t<double>(deg, x, y, z, o);
}

template <typename F>
__device__ __forceinline__ void sh_basis_t(int deg, F x, F y, F z, F *o) {
  o[0] = (F)0.28209479177387814;
  if (deg >= 1) {
    o[1] = (F)-0.4886025119029199 * y;
    o[2] = (F)0.4886025119029199 * z;
    o[3] = (F)-0.4886025119029199 * x;
  }
  if (deg >= 2) {
    const F xx = x * x, yy = y * y, zz = z * z;
    o[4] = (F)1.0925484305920792 * x * y;
    o[5] = (F)-1.0925484305920792 * y * z;
    o[6] = (F)0.31539156525252005 * ((F)2.0 * zz - xx - yy);
    o[7] = (F)-1.0925484305920792 * x * z;
    o[8] = (F)0.5462742152960396 * (xx - yy);
  }
  if (deg >= 3) {
    const F xx = x * x, yy = y * y, zz = z * z;
    o[9] = (F)-0.5900435899266435 * y * ((F)3.0 * xx - yy);
    o[10] = (F)2.890611442640554 * x * y * z;
    o[11] = (F)-0.4570457994644658 * y * ((F)4.0 * zz - xx - yy);
    o[12] = (F)0.3731763325901154 * z * ((F)2.0 * zz - (F)3.0 * xx - (F)3.0 * yy);
    o[13] = (F)-0.4570457994644658 * x * ((F)4.0 * zz - xx - yy);
    o[14] = (F)1.445305721320277 * z * (xx - yy);
    o[15] = (F)-0.5900435899266435 * x * (xx - (F)3.0 * yy);
  }
}

// core/rotation.py:24-41; returns false on |q| <= 1e-8
__device__ __forceinline__ bool quat_to_matrix_d(double qw, double qx, double qy, double qz, double *R) {
  double nrm = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
  if (!(nrm > kQuatMinNorm)) return false;
  double w = qw / nrm, x = qx / nrm, y = qy / nrm, z = qz / nrm;
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
  return true;
}

template <bool G64 = false>
__device__ __forceinline__ void load_center_d(const SceneView &sc, int64_t i, double *p) {
  p[0] = SceneGeom<G64>::center(sc, i, 0);
  p[1] = SceneGeom<G64>::center(sc, i, 1);
  p[2] = SceneGeom<G64>::center(sc, i, 2);
}

__device__ __forceinline__ void t_cam_d(const CamD &cam, const double *p, double *t) {
#pragma unroll
  for (int r = 0; r < 3; ++r) t[r] = ((p[0] * cam.V[r * 3] + p[1] * cam.V[r * 3 + 1]) + p[2] * cam.V[r * 3 + 2]) + cam.tv[r];
}

// EWA 2D covariance (a, b, c) incl. dilation for a 3D Gaussian (project.py:209-224).
__device__ __forceinline__ void cov2d_3d(const CamD &cam, const double *t, const double *R, const double *s,
                                         double &a, double &b, double &c) {
  const double z = t[2];
  double J[6] = {cam.fx / z, 0.0, -cam.fx * t[0] / (z * z), 0.0, cam.fy / z, -cam.fy * t[1] / (z * z)};
  double U[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      U[r * 3 + cc] = (J[r * 3] * cam.V[cc] + J[r * 3 + 1] * cam.V[3 + cc]) + J[r * 3 + 2] * cam.V[6 + cc];
  double RS[9], Sig[9], US[6];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) RS[r * 3 + cc] = R[r * 3 + cc] * s[cc];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      Sig[r * 3 + cc] = (RS[r * 3] * RS[cc * 3] + RS[r * 3 + 1] * RS[cc * 3 + 1]) + RS[r * 3 + 2] * RS[cc * 3 + 2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      US[r * 3 + cc] = (U[r * 3] * Sig[cc] + U[r * 3 + 1] * Sig[3 + cc]) + U[r * 3 + 2] * Sig[6 + cc];
  double s00 = (US[0] * U[0] + US[1] * U[1]) + US[2] * U[2];
  double s01 = (US[0] * U[3] + US[1] * U[4]) + US[2] * U[5];
  double s11 = (US[3] * U[3] + US[4] * U[4]) + US[5] * U[5];
  a = s00 + kDilation;
  b = s01;
  c = s11 + kDilation;
}

// det of the dilated 2D covariance, a c - b^2 with both products rounded
// (numpy's order, project.py:223): the singular-conic cull is decided by
// this one expression in k_depth_keys (the depth order / M) and in the
// preprocess (records / tile counts), so the two can never disagree.
__device__ __forceinline__ double conic_det(double a, double b, double c) {
  return __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, b));
}

// Full float64 projection of one Gaussian: everything SplatFrame holds
// (project.py:169-326) plus the extension normal.
struct ProjD {
  double t[3], ctr[2];
  double alpha, alpha_eff;
  double cov[3], conic[3];
  double mrow[12];  // 2D: rows (0, 1, 3) of M, 3 x 4
  double color[3];
  double normal[3];
  double view_dir[3], cam_dist;  // project.py:247-251 (not with GEOM_ONLY)
  double radius;
  double bb[4];  // continuous bbox before floor/ceil
  int bbox[4];   // inclusive pixel box, bbox[2] = -1 when off screen
  int typ;
  bool valid;    // singular-conic cull (project.py:225, 368-371)
  bool quat_ok;
};

// COLOR64 = false evaluates the SH colour in float32 (the record stores a
// float32 colour; the float64 path serves the exports and re-checks).
// GEOM_ONLY skips the colour and the normal (the float64 pair re-checks need
// only the geometry and alpha_eff).
// G64 reads the scene's float64 geometry (SceneView::center64 ...).
template <bool COLOR64 = true, bool GEOM_ONLY = false, bool G64 = false>
__device__ __forceinline__ void project_d(const SceneView &sc, int64_t i, const CamD &cam, const ModD &mod,
                                          ProjD &o, const float *sh_row = nullptr) {
  using G = SceneGeom<G64>;
  double p[3];
  load_center_d<G64>(sc, i, p);
  t_cam_d(cam, p, o.t);
  const double z = o.t[2];
  o.typ = sc.type_spec[i];
  o.ctr[0] = cam.fx * o.t[0] / z + cam.cx;
  o.ctr[1] = cam.fy * o.t[1] / z + cam.cy;
  double R[9];
  o.quat_ok = quat_to_matrix_d(G::rotation(sc, i, 0), G::rotation(sc, i, 1), G::rotation(sc, i, 2),
                               G::rotation(sc, i, 3), R);
  double s[3] = {exp(G::log_scale(sc, i, 0)), exp(G::log_scale(sc, i, 1)), exp(G::log_scale(sc, i, 2))};
  o.alpha = expit_d(G::opacity_logit(sc, i));
  o.alpha_eff = o.alpha;
  o.valid = true;
  o.cov[0] = o.cov[1] = o.cov[2] = 0.0;
  o.conic[0] = o.conic[1] = o.conic[2] = 0.0;
#pragma unroll
  for (int k = 0; k < 12; ++k) o.mrow[k] = 0.0;
  if (o.typ == 1) {
    double a, b, c;
    cov2d_3d(cam, o.t, R, s, a, b, c);
    double det = conic_det(a, b, c);
    bool ok = det > 1e-18;
    double inv = ok ? 1.0 / det : 0.0;
    o.cov[0] = a; o.cov[1] = b; o.cov[2] = c;
    o.conic[0] = c * inv; o.conic[1] = -b * inv; o.conic[2] = a * inv;
    o.valid = ok;
  } else {
    // H columns: s_x R0 | s_y R1 | 0 | mu ; M = T @ H, rows (0, 1, 3)
    double H[12];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      H[r * 4 + 0] = s[0] * R[r * 3 + 0];
      H[r * 4 + 1] = s[1] * R[r * 3 + 1];
      H[r * 4 + 2] = 0.0;
      H[r * 4 + 3] = p[r];
    }
    const int rows[3] = {0, 1, 3};
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) {
      const double *Tr = cam.T + rows[rr] * 4;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        double hw = d == 3 ? 1.0 : 0.0;
        o.mrow[rr * 4 + d] = ((Tr[0] * H[d] + Tr[1] * H[4 + d]) + Tr[2] * H[8 + d]) + Tr[3] * hw;
      }
    }
    // modulated opacity (exchange.py:102-111)
    double sz = s[2];
    double mz = expit_d((sz - mod.theta_z) / mod.t_z) * sz;
    o.alpha_eff = o.alpha * exp(-mod.lambda_z * mz);
  }
  if (GEOM_ONLY) return;
  // view-dependent colour (project.py:248-252, sh.py:110-122)
  double dl[3] = {p[0] - cam.campos[0], p[1] - cam.campos[1], p[2] - cam.campos[2]};
  double dist = sqrt((dl[0] * dl[0] + dl[1] * dl[1]) + dl[2] * dl[2]);
  double den = dist > 1e-12 ? dist : 1e-12;
  double vx = dl[0] / den, vy = dl[1] / den, vz = dl[2] / den;
  o.view_dir[0] = vx; o.view_dir[1] = vy; o.view_dir[2] = vz;
  o.cam_dist = dist;
  const int B = sc.sh_bases;
  const int deg = B == 1 ? 0 : (B == 4 ? 1 : (B == 9 ? 2 : 3));
  const float *shc = sh_row ? sh_row : sc.sh + (int64_t)3 * B * i;  // sh_row: staged copy (shared memory)
  if (COLOR64) {
    double basis[16];
    sh_basis_d(deg, vx, vy, vz, basis);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double acc = 0.0;
      for (int bb = 0; bb < B; ++bb) acc += (double)shc[ch * B + bb] * basis[bb];
      double v = acc + 0.5;
      o.color[ch] = v > 0.0 ? v : 0.0;
    }
  } else {
    float basis[16];
    sh_basis_t<float>(deg, (float)vx, (float)vy, (float)vz, basis);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float acc = 0.f;
#pragma unroll
      for (int bb = 0; bb < 16; ++bb)  // static indices keep basis[] in registers
        if (bb < B) acc = fmaf(shc[ch * B + bb], basis[bb], acc);
      o.color[ch] = fmaxf(acc + 0.5f, 0.f);
    }
  }
  // extension: camera-space normal facing the camera
  int ax = 2;
  if (o.typ == 1) ax = (s[0] <= s[1] && s[0] <= s[2]) ? 0 : (s[1] <= s[2] ? 1 : 2);
  double nw0 = R[ax], nw1 = R[3 + ax], nw2 = R[6 + ax];
  double nc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) nc[r] = (cam.V[r * 3] * nw0 + cam.V[r * 3 + 1] * nw1) + cam.V[r * 3 + 2] * nw2;
  double facing = (nc[0] * o.t[0] + nc[1] * o.t[1]) + nc[2] * o.t[2];
  double sg = facing > 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int r = 0; r < 3; ++r) o.normal[r] = sg * nc[r];
}

// _bboxes (project.py:261-326) for one projected splat.
__device__ __forceinline__ void bbox_d(ProjD &o, int W, int H) {
  const double C = kSupportC;
  double x0, y0, x1, y1;
  if (o.typ == 1) {
    double a = o.cov[0], b = o.cov[1], c = o.cov[2];
    double hx = sqrt(C * a) + kBBoxPad, hy = sqrt(C * c) + kBBoxPad;
    x0 = o.ctr[0] - hx; y0 = o.ctr[1] - hy; x1 = o.ctr[0] + hx; y1 = o.ctr[1] + hy;
    double lam = 0.5 * ((a + c) + sqrt((a - c) * (a - c) + 4.0 * b * b));
    double r3 = 3.0 * sqrt(lam);
    o.radius = isnan(r3) ? r3 : (1.0 < r3 ? r3 : 1.0);
  } else {
    const double *m = o.mrow;
    // A = [m[:,0], m[:,1], m[:,2] + m[:,3]]
    double A[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      A[r * 3] = m[r * 4];
      A[r * 3 + 1] = m[r * 4 + 1];
      A[r * 3 + 2] = m[r * 4 + 2] + m[r * 4 + 3];
    }
    const double sqC = sqrt(C);
    double e = kLowpassSigma * sqC;
    x0 = o.ctr[0] - e - kBBoxPad; y0 = o.ctr[1] - e - kBBoxPad;
    x1 = o.ctr[0] + e + kBBoxPad; y1 = o.ctr[1] + e + kBBoxPad;
    double w_min = A[8] - sqC * hypot(A[6], A[7]);
    bool full = w_min <= 1e-9;
    if (!full) {
      const double dg[3] = {C, C, -1.0};
      double AD[9], Q[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) AD[r * 3 + k] = A[r * 3 + k] * dg[k];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
          Q[r * 3 + cc] = (AD[r * 3] * A[cc * 3] + AD[r * 3 + 1] * A[cc * 3 + 1]) + AD[r * 3 + 2] * A[cc * 3 + 2];
      double dx = Q[2] * Q[2] - Q[0] * Q[8];
      double dy = Q[5] * Q[5] - Q[4] * Q[8];
      if (dx >= 0.0 && dy >= 0.0 && fabs(Q[8]) > 1e-18) {
        double sx = sqrt(dx) / fabs(Q[8]), sy = sqrt(dy) / fabs(Q[8]);
        double mx = Q[2] / Q[8], my = Q[5] / Q[8];
        double v;
        v = mx - sx - kBBoxPad; if (v < x0) x0 = v;
        v = mx + sx + kBBoxPad; if (v > x1) x1 = v;
        v = my - sy - kBBoxPad; if (v < y0) y0 = v;
        v = my + sy + kBBoxPad; if (v > y1) y1 = v;
      } else {
        full = true;
      }
    }
    if (full) { x0 = 0.0; y0 = 0.0; x1 = W - 1.0; y1 = H - 1.0; }
    double hxw = 0.5 * (x1 - x0), hyw = 0.5 * (y1 - y0);
    double rad = 1.0;
    if (hxw > rad) rad = hxw;
    if (hyw > rad) rad = hyw;
    o.radius = rad;
  }
  o.bb[0] = x0; o.bb[1] = y0; o.bb[2] = x1; o.bb[3] = y1;
  auto clip = [](double v, double hi) { return v < 0.0 ? 0.0 : (v > hi ? hi : v); };
  o.bbox[0] = (int)clip(floor(x0), W - 1.0);
  o.bbox[1] = (int)clip(floor(y0), H - 1.0);
  o.bbox[2] = (int)clip(ceil(x1), W - 1.0);
  o.bbox[3] = (int)clip(ceil(y1), H - 1.0);
  if ((x1 < 0) || (x0 > W - 1) || (y1 < 0) || (y0 > H - 1)) o.bbox[2] = -1;
}

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

}  // namespace hgs
