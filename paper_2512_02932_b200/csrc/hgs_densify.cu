// hgs_densify.cu -- adaptive density control as GPU stream compaction
// (the reference ships the
// GaussianSet stats / keep / append helpers, core/types.py:48-49, 110-130,
// but no densify code, so the rule set follows the SPEC text):
//
//  k_densify_stats : after a backward, per Gaussian: grad_accum += |NDC-space
//                    gradient of the projected centre| summed over the KG
//                    stacked losses (3DGS's view-space positional gradient),
//                    obs_count += touched.
//  k_densify_decide: prune alpha < prune_opacity; of the rest, mean gradient
//                    (accum / obs) > threshold -> split (max scale >
//                    split_scale) or clone; output rows 0 / 1 / 2.
//  scan            : three-kernel exclusive scan of the row counts.
//  k_densify_write : every Gaussian writes its rows at its scanned offset
//                    (order-preserving compaction): parameters, the Adam
//                    moments (carried for survivors, zero for new rows);
//                    split children sit at +-0.5 sigma along the major axis
//                    with scales / 1.6, clones copy the parent and step
//                    clone_step * sigma_max against the Adam first moment of
//                    the centre.
// HBM-bound: ~ (4P x 3 + stats) bytes read and written per Gaussian.
#include <algorithm>
#include <cmath>

#include "hgs_kernels.cuh"
#include "hgs_nvtx.h"
#include "../../include/hgs_train.h"

namespace hgs {
namespace {

constexpr int kAccD = 16;  // screen-space accumulator slots (hgs_composite_bwd.cu)
constexpr int kDScan = 1024;

enum : uint8_t { kKeep = 0, kPrune = 1, kClone = 2, kSplit = 3 };

__global__ void k_densify_stats(SceneView sc, CamD cam, const acc_t *acc, const float2 *eig, int kg,
                                const uint8_t *touched,
                                float half_w, float half_h, float *grad_accum, int32_t *obs_count) {
  const int64_t n = sc.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!touched[i]) continue;
    float m2[3] = {0.f, 0.f, 0.f};
    const bool is3d = sc.type_spec[i] == 1;
    if (!is3d) {  // depth row of M (columns 0, 1, 3): screen translation moves m0', m1' by delta m2
      const float q0 = sc.rotation[4 * i], q1 = sc.rotation[4 * i + 1], q2 = sc.rotation[4 * i + 2],
                  q3 = sc.rotation[4 * i + 3];
      const float iq = rsqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
      const float w = q0 * iq, x = q1 * iq, y = q2 * iq, z = q3 * iq;
      const float R0[3] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y + w * z), 2.f * (x * z - w * y)};
      const float R1[3] = {2.f * (x * y - w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z + w * x)};
      const float V6 = (float)cam.V[6], V7 = (float)cam.V[7], V8 = (float)cam.V[8];
      m2[0] = expf(sc.log_scale[3 * i]) * (V6 * R0[0] + V7 * R0[1] + V8 * R0[2]);
      m2[1] = expf(sc.log_scale[3 * i + 1]) * (V6 * R1[0] + V7 * R1[1] + V8 * R1[2]);
      m2[2] = (float)(cam.V[6] * sc.center[3 * i] + cam.V[7] * sc.center[3 * i + 1] +
                      cam.V[8] * sc.center[3 * i + 2] + cam.tv[2]);
    }
    float gx = 0.f, gy = 0.f;
    for (int k = 0; k < kg; ++k) {
      const acc_t *A = acc + ((int64_t)i * kg + k) * kAccD;
      if (is3d) {  // eigenbasis sums (hgs_composite_bwd.cu): rotate to pixel axes
        const float2 e = eig[i];
        gx += (float)(e.x * A[4] - e.y * A[5]);
        gy += (float)(e.y * A[4] + e.x * A[5]);
      } else {
        gx += (float)A[4];
        gy += (float)A[5];
        gx += ((float)A[6] * m2[0] + (float)A[7] * m2[1]) + (float)A[8] * m2[2];
        gy += ((float)A[9] * m2[0] + (float)A[10] * m2[1]) + (float)A[11] * m2[2];
      }
    }
    gx *= half_w;  // pixel -> NDC units (3DGS viewspace gradient convention)
    gy *= half_h;
    grad_accum[i] += sqrtf(gx * gx + gy * gy);
    obs_count[i] += 1;
  }
}

__global__ void k_densify_decide(SceneView sc, const float *grad_accum, const int32_t *obs_count, float thr,
                                 float prune_logit, float log_split, uint32_t *counts, uint8_t *mode,
                                 unsigned long long *census) {
  const int64_t n = sc.n;
  // grid-stride loop with a warp-uniform trip count (for the census ballots)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t start = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i0 = start - (threadIdx.x & 31); i0 < n; i0 += stride) {
    const int64_t i = i0 + (threadIdx.x & 31);
    uint8_t md = 0xff;
    if (i < n) {
      md = kKeep;
      if (!(sc.opacity_logit[i] >= prune_logit)) {
        md = kPrune;  // sigmoid(logit) < prune_opacity
      } else {
        const int32_t obs = obs_count[i];
        const float avg = obs > 0 ? grad_accum[i] / (float)obs : 0.f;
        if (avg > thr) {
          const float lmax = fmaxf(fmaxf(sc.log_scale[3 * i], sc.log_scale[3 * i + 1]),
                                   sc.type_spec[i] == 1 ? sc.log_scale[3 * i + 2] : -INFINITY);
          md = lmax > log_split ? kSplit : kClone;
        }
      }
      mode[i] = md;
      counts[i] = md == kPrune ? 0u : (md == kKeep ? 1u : 2u);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t b = __ballot_sync(0xffffffffu, md == c);
      if ((threadIdx.x & 31) == 0 && b) atomicAdd(&census[c], (unsigned long long)__popc(b));
    }
  }
}

// exclusive scan: per-block sums, one-block scan of the sums, per-block scan + offset
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *s_warp, uint32_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  const uint32_t before = w ? s_warp[w - 1] : 0u;
  return before + x - v;
}

__global__ void __launch_bounds__(kDScan) k_scan_block_sums(const uint32_t *counts, int64_t n, uint32_t *sums) {
  __shared__ uint32_t s_warp[32];
  const int64_t i = (int64_t)blockIdx.x * kDScan + threadIdx.x;
  uint32_t tot;
  block_excl_scan(i < n ? counts[i] : 0u, s_warp, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kDScan) k_scan_sums(uint32_t *sums, int nb, unsigned long long *total_out) {
  __shared__ uint32_t s_warp[32];
  __shared__ unsigned long long s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += kDScan) {
    const int b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? sums[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, s_warp, tot);
    if (b < nb) sums[b] = (uint32_t)(s_carry + ex);
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = s_carry;
}

__global__ void __launch_bounds__(kDScan) k_scan_apply(const uint32_t *counts, int64_t n, const uint32_t *sums,
                                                      uint32_t *offsets) {
  __shared__ uint32_t s_warp[32];
  const int64_t i = (int64_t)blockIdx.x * kDScan + threadIdx.x;
  uint32_t tot;
  const uint32_t ex = block_excl_scan(i < n ? counts[i] : 0u, s_warp, tot);
  if (i < n) offsets[i] = sums[blockIdx.x] + ex;
}

struct WriteArgs {
  SceneView src;
  const float *m_src, *v_src;  // (n * P) field-major Adam moments (nullable)
  const uint32_t *off;
  const uint8_t *mode;
  int64_t n_out;
  float *dst[5];               // center, log_scale, rotation, opacity, sh (n_out rows)
  uint8_t *dst_type;
  float *m_dst, *v_dst;        // (n_out * P) field-major (nullable)
  float log_div, clone_step;
};

__device__ __forceinline__ int fwidth(int f, int B) { return f < 2 ? 3 : (f == 2 ? 4 : (f == 3 ? 1 : 3 * B)); }
__device__ __forceinline__ int64_t foff(int f, int64_t n) {
  return (f == 0 ? 0 : (f == 1 ? 3 : (f == 2 ? 6 : (f == 3 ? 10 : 11)))) * n;
}

__global__ void k_densify_write(WriteArgs a) {
  const SceneView &s = a.src;
  const int64_t n = s.n;
  const int B = s.sh_bases;
  const float *srcf[5] = {s.center, s.log_scale, s.rotation, s.opacity_logit, s.sh};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t md = a.mode[i];
    if (md == kPrune) continue;
    const int64_t o = a.off[i];
    const int rows = md == kKeep ? 1 : 2;
    // plain copies of every field into each output row
    for (int r = 0; r < rows; ++r)
      for (int f = 0; f < 5; ++f) {
        const int fw = fwidth(f, B);
        for (int j = 0; j < fw; ++j) a.dst[f][(o + r) * fw + j] = srcf[f][i * fw + j];
      }
    for (int r = 0; r < rows; ++r) a.dst_type[o + r] = s.type_spec[i];
    // Adam moments: survivors keep theirs, new rows start from zero
    if (a.m_dst) {
      for (int f = 0; f < 5; ++f) {
        const int fw = fwidth(f, B);
        for (int j = 0; j < fw; ++j) {
          const int64_t si = foff(f, n) + i * fw + j;
          const int64_t d0 = foff(f, a.n_out) + o * fw + j;
          const bool carry = md == kKeep || md == kClone;  // row o is the parent itself
          a.m_dst[d0] = carry && a.m_src ? a.m_src[si] : 0.f;
          a.v_dst[d0] = carry && a.v_src ? a.v_src[si] : 0.f;
          if (rows == 2) {
            a.m_dst[d0 + fw] = 0.f;
            a.v_dst[d0 + fw] = 0.f;
          }
        }
      }
    }
    if (md == kKeep) continue;
    // geometry of the new rows
    const float q0 = s.rotation[4 * i], q1 = s.rotation[4 * i + 1], q2 = s.rotation[4 * i + 2], q3 = s.rotation[4 * i + 3];
    const float iq = rsqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const float w = q0 * iq, x = q1 * iq, y = q2 * iq, z = q3 * iq;
    const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                        2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                        2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    const float l0 = s.log_scale[3 * i], l1 = s.log_scale[3 * i + 1], l2 = s.log_scale[3 * i + 2];
    const bool is3d = s.type_spec[i] == 1;
    int ax = l1 > l0 ? 1 : 0;  // major axis (in-plane for a 2D surfel)
    if (is3d && l2 > (ax ? l1 : l0)) ax = 2;
    const float sig = expf(ax == 0 ? l0 : (ax == 1 ? l1 : l2));
    if (md == kSplit) {
      const float d = 0.5f * sig;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float sg = r ? -1.f : 1.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a.dst[0][(o + r) * 3 + c] = s.center[3 * i + c] + sg * d * R[c * 3 + ax];
          a.dst[1][(o + r) * 3 + c] = s.log_scale[3 * i + c] - a.log_div;
        }
      }
    } else if (a.clone_step > 0.f && a.m_src) {  // clone: step the copy against the centre's Adam moment
      const float g0 = a.m_src[3 * i], g1 = a.m_src[3 * i + 1], g2 = a.m_src[3 * i + 2];
      const float gn = sqrtf(g0 * g0 + g1 * g1 + g2 * g2);
      if (gn > 0.f) {
        const float t = a.clone_step * sig / gn;
        a.dst[0][(o + 1) * 3 + 0] = s.center[3 * i + 0] - t * g0;
        a.dst[0][(o + 1) * 3 + 1] = s.center[3 * i + 1] - t * g1;
        a.dst[0][(o + 1) * 3 + 2] = s.center[3 * i + 2] - t * g2;
      }
    }
  }
}

SceneView view_of(const hgs_scene &s) {
  SceneView v;
  v.center = s.center; v.log_scale = s.log_scale; v.rotation = s.rotation;
  v.opacity_logit = s.opacity_logit; v.sh = s.sh; v.type_spec = s.type_spec;
  v.n = s.n; v.sh_bases = s.sh_bases;
  return v;
}

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

struct DScratch {
  uint32_t *counts, *offsets, *sums;
  uint8_t *mode;
  unsigned long long *total;  // [0] rows out, [1..4] census keep / prune / clone / split
};

DScratch carve(void *scratch, int64_t n) {
  char *p = static_cast<char *>(scratch);
  auto take = [&](size_t b) { char *q = p; p += (b + 255) & ~(size_t)255; return q; };
  const int64_t nn = std::max<int64_t>(n, 1);
  DScratch d;
  d.counts = reinterpret_cast<uint32_t *>(take(nn * 4));
  d.offsets = reinterpret_cast<uint32_t *>(take(nn * 4));
  d.sums = reinterpret_cast<uint32_t *>(take(((nn + kDScan - 1) / kDScan) * 4));
  d.mode = reinterpret_cast<uint8_t *>(take(nn));
  d.total = reinterpret_cast<unsigned long long *>(take(5 * 8));
  return d;
}

}  // namespace
}  // namespace hgs

using namespace hgs;

extern "C" {

int hgs_densify_stats(const hgs_scene *scene, const hgs_camera *camera, const void *frame,
                      const hgs_frame_info *info, const void *bwd_scratch, int32_t kg, const uint8_t *touched,
                      float *grad_accum, int32_t *obs_count, void *stream) {
  NvtxScope nv("hgs_densify_stats");
  if (!scene || !camera || scene->n < 0 || kg < 1 || kg > 4) return HGS_ERR_CONFIG;
  if (scene->n == 0) return HGS_OK;
  if (!bwd_scratch || !touched || !grad_accum || !obs_count || !frame || !info) return HGS_ERR_INTEGRITY;
  if (info->n != scene->n) return HGS_ERR_INTEGRITY;
  CamD cam;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) cam.V[r * 3 + k] = camera->world_to_camera[r * 4 + k];
    cam.tv[r] = camera->world_to_camera[r * 4 + 3];
  }
  k_densify_stats<<<grid_of(scene->n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of(*scene), cam, static_cast<const acc_t *>(bwd_scratch), frame_eig(frame, info), kg, touched,
      0.5f * (float)camera->width,
      0.5f * (float)camera->height, grad_accum, obs_count);
  return cudaGetLastError() == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

size_t hgs_densify_scratch_bytes(int64_t n) {
  if (n < 0) return 0;
  const int64_t nn = std::max<int64_t>(n, 1);
  return ((nn * 4 + 255) & ~255ll) * 2 + ((((nn + kDScan - 1) / kDScan) * 4 + 255) & ~255ll) + ((nn + 255) & ~255ll) + 256;
}

int hgs_densify_plan(const hgs_scene *scene, const float *grad_accum, const int32_t *obs_count,
                     const hgs_densify_config *cfg, void *scratch, size_t scratch_bytes, int64_t *n_out,
                     int64_t *census, void *stream) {
  NvtxScope nv("hgs_densify_plan");
  if (!scene || !cfg || !n_out || scene->n < 0) return HGS_ERR_CONFIG;
  if (!(cfg->prune_opacity >= 0.0 && cfg->prune_opacity < 1.0) || !(cfg->split_scale > 0.0) ||
      !(cfg->grad_threshold >= 0.0))
    return HGS_ERR_CONFIG;
  *n_out = 0;
  if (census)
    for (int c = 0; c < 4; ++c) census[c] = 0;
  if (scene->n == 0) return HGS_OK;
  if (!grad_accum || !obs_count || !scratch || scratch_bytes < hgs_densify_scratch_bytes(scene->n))
    return HGS_ERR_INTEGRITY;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = scene->n;
  DScratch d = carve(scratch, n);
  const double po = cfg->prune_opacity;
  const float prune_logit = po <= 0.0 ? -INFINITY : (float)std::log(po / (1.0 - po));
  if (cudaMemsetAsync(d.total, 0, 5 * 8, s) != cudaSuccess) return HGS_ERR_CUDA;
  k_densify_decide<<<grid_of(n), 256, 0, s>>>(view_of(*scene), grad_accum, obs_count, (float)cfg->grad_threshold,
                                              prune_logit, (float)std::log(cfg->split_scale), d.counts, d.mode,
                                              d.total + 1);
  const int nb = (int)((n + kDScan - 1) / kDScan);
  k_scan_block_sums<<<nb, kDScan, 0, s>>>(d.counts, n, d.sums);
  k_scan_sums<<<1, kDScan, 0, s>>>(d.sums, nb, d.total);
  k_scan_apply<<<nb, kDScan, 0, s>>>(d.counts, n, d.sums, d.offsets);
  if (cudaGetLastError() != cudaSuccess) return HGS_ERR_CUDA;
  unsigned long long tot[5] = {0, 0, 0, 0, 0};
  if (cudaMemcpyAsync(tot, d.total, sizeof(tot), cudaMemcpyDeviceToHost, s) != cudaSuccess) return HGS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return HGS_ERR_CUDA;
  *n_out = (int64_t)tot[0];
  if (census)
    for (int c = 0; c < 4; ++c) census[c] = (int64_t)tot[1 + c];
  return HGS_OK;
}

int hgs_densify_apply(const hgs_scene *scene, const float *exp_avg, const float *exp_avg_sq, const void *scratch,
                      const hgs_densify_config *cfg, const hgs_params *out, uint8_t *out_type_spec,
                      float *out_exp_avg, float *out_exp_avg_sq, void *stream) {
  NvtxScope nv("hgs_densify_apply");
  if (!scene || !cfg || !out || scene->n < 0 || out->sh_bases != scene->sh_bases) return HGS_ERR_CONFIG;
  if (scene->n == 0 || out->n == 0) return HGS_OK;
  if (!scratch || !out_type_spec || ((out_exp_avg == nullptr) != (out_exp_avg_sq == nullptr)))
    return HGS_ERR_INTEGRITY;
  DScratch d = carve(const_cast<void *>(scratch), scene->n);
  WriteArgs a;
  a.src = view_of(*scene);
  a.m_src = exp_avg;
  a.v_src = exp_avg_sq;
  a.off = d.offsets;
  a.mode = d.mode;
  a.n_out = out->n;
  a.dst[0] = out->center; a.dst[1] = out->log_scale; a.dst[2] = out->rotation;
  a.dst[3] = out->opacity_logit; a.dst[4] = out->sh;
  a.dst_type = out_type_spec;
  a.m_dst = out_exp_avg;
  a.v_dst = out_exp_avg_sq;
  a.log_div = (float)std::log(1.6);
  a.clone_step = (float)cfg->clone_step;
  k_densify_write<<<grid_of(scene->n), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? HGS_OK : HGS_ERR_CUDA;
}

}  // extern "C"
