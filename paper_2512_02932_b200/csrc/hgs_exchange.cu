// hgs_exchange.cu -- Adaptive Type Exchange as per-Gaussian kernels
// (exchange.py:58-99, 137-155).  Two phases so that a DegenerateScaleError
// leaves the scene untouched, like the reference (effective_rank runs over
// every row before any mutation):
//   k_exchange_scan  : erank in float64, demote/promote counts, the 20-bin
//                      histogram over [1, 3] with numpy.histogram's binning,
//                      degenerate-scale flag;
//   k_exchange_apply : covariance-preserving 3D->2D reparameterisation
//                      (permutation of the scale axes, R P^T -> quaternion,
//                      Shepperd with w >= 0) and the type flips.
#include "hgs_kernels.cuh"

namespace hgs {

template <typename T>
__device__ __forceinline__ bool erank_d(const T *ls, double &er) {
  double q0 = exp(2.0 * (double)ls[0]), q1 = exp(2.0 * (double)ls[1]), q2 = exp(2.0 * (double)ls[2]);
  double tot = (q0 + q1) + q2;
  if (tot == 0.0 || !isfinite(q0) || !isfinite(q1) || !isfinite(q2)) return false;
  double p0 = q0 / tot, p1 = q1 / tot, p2 = q2 / tot;
  double ent = ((p0 > 0.0 ? p0 * log(p0) : 0.0) + (p1 > 0.0 ? p1 * log(p1) : 0.0)) + (p2 > 0.0 ? p2 * log(p2) : 0.0);
  er = exp(-ent);
  return true;
}

// numpy.histogram(x, bins=20, range=(1, 3)) bin index, -1 if outside.
__device__ __forceinline__ int hist_bin(double x) {
  const double first = 1.0, last = 3.0, step = (last - first) / 20.0;
  if (!(x >= first && x <= last)) return -1;
  int b = (int)(((x - first) / (last - first)) * 20.0);
  if (b == 20) b -= 1;
  const double lo = b * step + first;
  const double hi = (b + 1 == 20) ? last : (b + 1) * step + first;
  if (x < lo) b -= 1;
  else if (x >= hi && b != 19) b += 1;
  return b;
}

template <typename T>
__global__ void __launch_bounds__(256) k_exchange_scan(int64_t n, const T *__restrict__ log_scale,
                                                       const uint8_t *__restrict__ type_spec, double theta_e,
                                                       T *__restrict__ eranks, ExchangeState *__restrict__ st) {
  __shared__ unsigned int s_hist[20];
  __shared__ unsigned int s_cnt[4];
  if (threadIdx.x < 20) s_hist[threadIdx.x] = 0;
  if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double er;
    if (!erank_d(log_scale + 3 * i, er)) {
      atomicAdd(&s_cnt[3], 1u);
      continue;
    }
    if (eranks) eranks[i] = (T)er;
    const uint8_t t = type_spec[i];
    if (t == 1 && er < theta_e) atomicAdd(&s_cnt[0], 1u);
    if (t == 0 && er > theta_e) atomicAdd(&s_cnt[1], 1u);
    if (t != 0) atomicAdd(&s_cnt[2], 1u);
    const int b = hist_bin(er);
    if (b >= 0) atomicAdd(&s_hist[b], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 20 && s_hist[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], (unsigned long long)s_hist[threadIdx.x]);
  if (threadIdx.x < 4 && s_cnt[threadIdx.x]) atomicAdd(&st->counts[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

// core/rotation.py:44-76 (Shepperd, w >= 0)
__device__ __forceinline__ void matrix_to_quat_d(const double *m, double *q) {
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

template <typename T>
__global__ void __launch_bounds__(256) k_exchange_apply(int64_t n, T *__restrict__ log_scale,
                                                        T *__restrict__ rotation, uint8_t *__restrict__ type_spec,
                                                        double theta_e) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double er;
    if (!erank_d(log_scale + 3 * i, er)) continue;
    const uint8_t t = type_spec[i];
    if (t == 0) {
      if (er > theta_e) type_spec[i] = 1;  // promotion keeps every parameter
      continue;
    }
    if (!(er < theta_e)) continue;
    // choose_permutation (exchange.py:76-88); ties prefer I, then P_x
    const T *ls = log_scale + 3 * i;
    double s[3] = {exp((double)ls[0]), exp((double)ls[1]), exp((double)ls[2])};
    int perm = (s[2] <= s[0] && s[2] <= s[1]) ? 0 : (s[0] <= s[1] ? 1 : 2);
    // new scale diag(P S P^T): P_x -> (s1, s2, s0), P_y -> (s2, s0, s1)
    int src[3];
    if (perm == 0) { src[0] = 0; src[1] = 1; src[2] = 2; }
    else if (perm == 1) { src[0] = 1; src[1] = 2; src[2] = 0; }
    else { src[0] = 2; src[1] = 0; src[2] = 1; }
    double R[9];
    T *q = rotation + 4 * i;
    quat_to_matrix_d(q[0], q[1], q[2], q[3], R);
    // (R P^T)[r][c] = R[r][src[c]]  (P^T column c = e_{src[c]})
    double RP[9];
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) RP[r * 3 + cc] = R[r * 3 + src[cc]];
    double qn[4];
    matrix_to_quat_d(RP, qn);
    const T lsv[3] = {ls[0], ls[1], ls[2]};
    // log(exp(ls)) in float64 (exchange.py:98), stored in T
    T *lw = log_scale + 3 * i;
    for (int cc = 0; cc < 3; ++cc) lw[cc] = (T)log(exp((double)lsv[src[cc]]));
    for (int cc = 0; cc < 4; ++cc) q[cc] = (T)qn[cc];
    type_spec[i] = 0;
  }
}

// Host launchers (the template kernels are instantiated and launched in this
// translation unit).
template <typename T>
cudaError_t launch_exchange_scan(int64_t n, const T *log_scale, const uint8_t *type_spec, double theta_e, T *eranks,
                                 ExchangeState *st, int grid, cudaStream_t s) {
  k_exchange_scan<T><<<grid, 256, 0, s>>>(n, log_scale, type_spec, theta_e, eranks, st);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_exchange_apply(int64_t n, T *log_scale, T *rotation, uint8_t *type_spec, double theta_e, int grid,
                                  cudaStream_t s) {
  k_exchange_apply<T><<<grid, 256, 0, s>>>(n, log_scale, rotation, type_spec, theta_e);
  return cudaGetLastError();
}
template cudaError_t launch_exchange_scan<float>(int64_t, const float *, const uint8_t *, double, float *,
                                                 ExchangeState *, int, cudaStream_t);
template cudaError_t launch_exchange_scan<double>(int64_t, const double *, const uint8_t *, double, double *,
                                                  ExchangeState *, int, cudaStream_t);
template cudaError_t launch_exchange_apply<float>(int64_t, float *, float *, uint8_t *, double, int, cudaStream_t);
template cudaError_t launch_exchange_apply<double>(int64_t, double *, double *, uint8_t *, double, int, cudaStream_t);

}  // namespace hgs
