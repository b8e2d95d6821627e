// hgs_helpers.cu -- batch forms of the reference's public per-primitive
// helpers, evaluated on the device in float64 with the same formulas as the
// hot path (include/hgs.h, "[ABI 3] helpers"):
//   evaluate_contribution / ray_splat_intersect   raster/project.py:109-152
//   effective_rank                                exchange.py:58-73
//   choose_permutation / reparameterize_3d_to_2d  exchange.py:76-99
//   modulated_z / modulated_opacity(_grads)       exchange.py:102-129
#include "hgs_kernels.cuh"

namespace hgs {

// One (splat, pixel) pair per thread.  conic = (c00, c01, c11); mrow = the
// 3 x 4 rows (0, 1, 3) of the pixel map, row-major.
__global__ void k_eval_contrib(int64_t n, const uint8_t *__restrict__ typ, const double *__restrict__ center2d,
                               const double *__restrict__ conic, const double *__restrict__ mrow,
                               const double *__restrict__ opacity, const double *__restrict__ pixel,
                               double *__restrict__ alpha, double *__restrict__ u_out, double *__restrict__ v_out,
                               int32_t *__restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double px = pixel[2 * i], py = pixel[2 * i + 1];
    const double dx = px - center2d[2 * i], dy = py - center2d[2 * i + 1];
    double d, u = dx, v = dy;
    int32_t f = 0;
    bool skip = false;
    if (typ[i] == 1) {
      const double *c = conic + 3 * i;
      d = ((c[0] * dx) * dx + ((2.0 * c[1]) * dx) * dy) + (c[2] * dy) * dy;
    } else {
      const double d_screen = (dx * dx + dy * dy) / (kLowpassSigma * kLowpassSigma);
      const double *m = mrow + 12 * i;
      double hu[4], hv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        hu[k] = px * m[8 + k] - m[k];
        hv[k] = py * m[8 + k] - m[4 + k];
      }
      const double den = hu[0] * hv[1] - hu[1] * hv[0];
      if (fabs(den) < kDegenerateDen) {
        f = 1;  // DegenerateIntersection: evaluate_contribution returns 0
        skip = true;
        d = 0.0;
      } else {
        u = (hu[1] * hv[3] - hu[3] * hv[1]) / den;
        v = (hu[3] * hv[0] - hu[0] * hv[3]) / den;
        const double dr = u * u + v * v;
        d = dr < d_screen ? dr : d_screen;
      }
    }
    double a = 0.0;
    if (!skip) {
      a = opacity[i] * exp(-0.5 * d);
      if (a > kAlphaClamp) a = kAlphaClamp;
    }
    alpha[i] = a;
    if (u_out) u_out[i] = u;
    if (v_out) v_out[i] = v;
    if (flags) flags[i] = f;
  }
}

__device__ __forceinline__ bool erank_row(const double *ls, double &er) {
  double q0 = exp(2.0 * ls[0]), q1 = exp(2.0 * ls[1]), q2 = exp(2.0 * ls[2]);
  double tot = (q0 + q1) + q2;
  if (tot == 0.0 || !isfinite(q0) || !isfinite(q1) || !isfinite(q2)) return false;
  double p0 = q0 / tot, p1 = q1 / tot, p2 = q2 / tot;
  double ent = ((p0 > 0.0 ? p0 * log(p0) : 0.0) + (p1 > 0.0 ? p1 * log(p1) : 0.0)) + (p2 > 0.0 ? p2 * log(p2) : 0.0);
  er = exp(-ent);
  return true;
}

__global__ void k_erank(int64_t n, const double *__restrict__ log_scale, double *__restrict__ out,
                        uint32_t *__restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double er;
    if (!erank_row(log_scale + 3 * i, er)) {
      atomicOr(bad, 1u);
      er = nan("");
    }
    out[i] = er;
  }
}

__device__ __forceinline__ void mat_to_quat(const double *m, double *q) {
  double t = (m[0] + m[4]) + m[8];
  if (t > 0) {
    double r = sqrt(1.0 + t), s = 0.5 / r;
    q[0] = 0.5 * r;
    q[1] = (m[7] - m[5]) * s;
    q[2] = (m[2] - m[6]) * s;
    q[3] = (m[3] - m[1]) * s;
  } else {
    int k = 0;
    if (m[4] > m[0]) k = 1;
    if (m[8] > m[k * 4]) k = 2;
    int a = k, b = (k + 1) % 3, c = (k + 2) % 3;
    double r = sqrt(((1.0 + m[a * 4]) - m[b * 4]) - m[c * 4]);
    double s = 0.5 / r;
    q[0] = (m[c * 3 + b] - m[b * 3 + c]) * s;
    q[1 + a] = 0.5 * r;
    q[1 + b] = (m[b * 3 + a] + m[a * 3 + b]) * s;
    q[1 + c] = (m[c * 3 + a] + m[a * 3 + c]) * s;
  }
  if (q[0] < 0) {
    q[0] = -q[0]; q[1] = -q[1]; q[2] = -q[2]; q[3] = -q[3];
  }
}

// perm: 0 identity, 1 P_x, 2 P_y (exchange.py:19-25, 76-88)
__global__ void k_reparam(int64_t n, const double *__restrict__ log_scale, const double *__restrict__ rotation,
                          double *__restrict__ out_ls, double *__restrict__ out_rot, int32_t *__restrict__ perm_out,
                          uint32_t *__restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double *ls = log_scale + 3 * i;
    const double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    const int perm = (s[2] <= s[0] && s[2] <= s[1]) ? 0 : (s[0] <= s[1] ? 1 : 2);
    int src[3];
    if (perm == 0) { src[0] = 0; src[1] = 1; src[2] = 2; }
    else if (perm == 1) { src[0] = 1; src[1] = 2; src[2] = 0; }
    else { src[0] = 2; src[1] = 0; src[2] = 1; }
    if (perm_out) perm_out[i] = perm;
    if (!out_ls && !out_rot) continue;
    const double *q = rotation + 4 * i;
    double R[9];
    if (!quat_to_matrix_d(q[0], q[1], q[2], q[3], R)) {
      atomicOr(bad, 1u);
      continue;
    }
    double RP[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) RP[r * 3 + c] = R[r * 3 + src[c]];
    double qn[4];
    mat_to_quat(RP, qn);
    for (int c = 0; c < 3; ++c) out_ls[3 * i + c] = log(s[src[c]]);
    for (int c = 0; c < 4; ++c) out_rot[4 * i + c] = qn[c];
  }
}

__global__ void k_modulation(int64_t n, const double *__restrict__ opacity, const double *__restrict__ log_scale_z,
                             double theta_z, double t_z, double lambda_z, double *__restrict__ sz_star,
                             double *__restrict__ alpha_eff, double *__restrict__ d_alpha,
                             double *__restrict__ d_logz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double sz = exp(log_scale_z[i]);
    const double gate = expit_d((sz - theta_z) / t_z);
    const double ss = gate * sz;
    const double damp = exp(-lambda_z * ss);
    const double op = opacity ? opacity[i] : 1.0;
    if (sz_star) sz_star[i] = ss;
    if (alpha_eff) alpha_eff[i] = op * damp;
    if (d_alpha) d_alpha[i] = damp;
    if (d_logz) {
      const double dsd = gate + sz * gate * (1.0 - gate) / t_z;
      d_logz[i] = op * damp * (-lambda_z) * dsd * sz;
    }
  }
}

namespace {
int grid_of(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}
}  // namespace

}  // namespace hgs

using namespace hgs;

extern "C" {

int hgs_eval_contributions(int64_t n, const uint8_t *typ, const double *center2d, const double *conic,
                           const double *mrow, const double *opacity, const double *pixel, double *alpha, double *u,
                           double *v, int32_t *flags, void *stream) {
  if (n < 0 || (n > 0 && (!typ || !center2d || !conic || !mrow || !opacity || !pixel || !alpha))) return HGS_ERR_CONFIG;
  if (n == 0) return HGS_OK;
  k_eval_contrib<<<grid_of(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, typ, center2d, conic, mrow, opacity,
                                                                           pixel, alpha, u, v, flags);
  return cudaGetLastError() == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

int hgs_effective_rank_f64(int64_t n, const double *log_scale, double *eranks, void *scratch, void *stream) {
  if (n < 0 || !scratch || (n > 0 && (!log_scale || !eranks))) return HGS_ERR_CONFIG;
  if (n == 0) return HGS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t *bad = static_cast<uint32_t *>(scratch);
  if (cudaMemsetAsync(bad, 0, 4, s) != cudaSuccess) return HGS_ERR_CUDA;
  k_erank<<<grid_of(n), 256, 0, s>>>(n, log_scale, eranks, bad);
  uint32_t h = 0;
  if (cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return HGS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return HGS_ERR_CUDA;
  return h ? HGS_ERR_DEGENERATE_SCALE : HGS_OK;
}

int hgs_reparameterize_f64(int64_t n, const double *log_scale, const double *rotation, double *out_log_scale,
                           double *out_rotation, int32_t *perm, void *scratch, void *stream) {
  if (n < 0 || !scratch || (n > 0 && !log_scale)) return HGS_ERR_CONFIG;
  if ((out_log_scale != nullptr) != (out_rotation != nullptr) || (out_rotation && !rotation)) return HGS_ERR_CONFIG;
  if (n == 0) return HGS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t *bad = static_cast<uint32_t *>(scratch);
  if (cudaMemsetAsync(bad, 0, 4, s) != cudaSuccess) return HGS_ERR_CUDA;
  k_reparam<<<grid_of(n), 256, 0, s>>>(n, log_scale, rotation, out_log_scale, out_rotation, perm, bad);
  uint32_t h = 0;
  if (cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return HGS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return HGS_ERR_CUDA;
  return h ? HGS_ERR_INVALID_PARAMETER : HGS_OK;
}

int hgs_modulation_f64(int64_t n, const double *opacity, const double *log_scale_z, double theta_z, double t_z,
                       double lambda_z, double *sz_star, double *alpha_eff, double *d_alpha, double *d_logz,
                       void *stream) {
  if (n < 0 || !(t_z > 0) || (n > 0 && !log_scale_z)) return HGS_ERR_CONFIG;
  if ((alpha_eff || d_logz) && !opacity) return HGS_ERR_CONFIG;
  if (n == 0) return HGS_OK;
  k_modulation<<<grid_of(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, opacity, log_scale_z, theta_z, t_z,
                                                                         lambda_z, sz_star, alpha_eff, d_alpha, d_logz);
  return cudaGetLastError() == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

}  // extern "C"

// ------------------------------------------------------------ host I/O
// The reference-facing API returns float64 numpy arrays.  Widening on the
// host cores is host-memory bound (~20 B of DRAM traffic per element); a
// share of each output is instead widened on the GPU and DMA'd as float64
// straight into the (registered) destination array, so PCIe and the host
// cores work in parallel (_hostio.download).
namespace hgs {
__global__ void k_widen(const float *__restrict__ src, double *__restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;
  const float4 *s4 = reinterpret_cast<const float4 *>(src);
  double2 *d2 = reinterpret_cast<double2 *>(dst);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = s4[i];
    d2[2 * i] = make_double2(v.x, v.y);
    d2[2 * i + 1] = make_double2(v.z, v.w);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}
}  // namespace hgs

extern "C" {

int hgs_host_register(void *ptr, size_t bytes) {
  if (!ptr || !bytes) return HGS_ERR_CONFIG;
  return cudaHostRegister(ptr, bytes, cudaHostRegisterPortable) == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

int hgs_host_unregister(void *ptr) {
  if (!ptr) return HGS_ERR_CONFIG;
  return cudaHostUnregister(ptr) == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

int hgs_widen_d2h(const float *src, double *dst_host, int64_t n, double *scratch, void *stream) {
  if (n < 0 || (n > 0 && (!src || !dst_host || !scratch))) return HGS_ERR_CONFIG;
  if (((uintptr_t)src & 15u) || ((uintptr_t)scratch & 15u)) return HGS_ERR_CONFIG;
  if (n == 0) return HGS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_widen<<<grid_of(n / 4 + 1), 256, 0, s>>>(src, scratch, n);
  if (cudaGetLastError() != cudaSuccess) return HGS_ERR_CUDA;
  return cudaMemcpyAsync(dst_host, scratch, (size_t)n * 8, cudaMemcpyDeviceToHost, s) == cudaSuccess ? HGS_OK
                                                                                                   : HGS_ERR_CUDA;
}

}  // extern "C"
