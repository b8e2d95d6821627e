// hgs_backward.cu -- the per-Gaussian chain rule (grad/backward.py:68-178,
// core/sh.py:125-141, core/rotation.py:79-107, exchange.py:114-129): from
// the screen-space accumulators of k_composite_bwd to ParamGrads.
//
// One thread per Gaussian in original index order (coalesced reads of the
// scene and accumulators, coalesced field-major writes).  Templated on the SH
// degree so every loop unrolls into registers; the geometric chain runs in
// float64 (the 2D anchor un-rebasing cancels ~1e3-pixel terms), the SH
// direction gradient is accumulated on the fly without a basis-gradient table.
#include "hgs_kernels.cuh"

namespace hgs {

constexpr int kAcc = 16;  // accumulator slots per (Gaussian, kg): see hgs_composite_bwd.cu
constexpr int kAccExt = 4;

// sum_b db[b] * dY_b / d(dir)   (core/sh.py:63-107, contracted with db)
template <int DEG>
__device__ __forceinline__ void sh_dir_grad(double x, double y, double z, const double *db, double &gx, double &gy,
                                            double &gz) {
  const double C1 = 0.4886025119029199;
  gx = gy = gz = 0.0;
  if (DEG >= 1) {
    gy += -C1 * db[1];
    gz += C1 * db[2];
    gx += -C1 * db[3];
  }
  if (DEG >= 2) {
    const double A = 1.0925484305920792, Bq = -1.0925484305920792, Cq = 0.31539156525252005,
                 Dq = -1.0925484305920792, Eq = 0.5462742152960396;
    gx += A * y * db[4];
    gy += A * x * db[4];
    gy += Bq * z * db[5];
    gz += Bq * y * db[5];
    gx += Cq * (-2.0 * x) * db[6];
    gy += Cq * (-2.0 * y) * db[6];
    gz += Cq * (4.0 * z) * db[6];
    gx += Dq * z * db[7];
    gz += Dq * x * db[7];
    gx += Eq * (2.0 * x) * db[8];
    gy += Eq * (-2.0 * y) * db[8];
  }
  if (DEG >= 3) {
    const double c0 = -0.5900435899266435, c1 = 2.890611442640554, c2 = -0.4570457994644658,
                 c3 = 0.3731763325901154, c4 = -0.4570457994644658, c5 = 1.445305721320277,
                 c6 = -0.5900435899266435;
    gx += c0 * 6.0 * x * y * db[9];
    gy += c0 * (3.0 * x * x - 3.0 * y * y) * db[9];
    gx += c1 * y * z * db[10];
    gy += c1 * x * z * db[10];
    gz += c1 * x * y * db[10];
    gx += c2 * (-2.0 * x * y) * db[11];
    gy += c2 * (4.0 * z * z - x * x - 3.0 * y * y) * db[11];
    gz += c2 * (8.0 * y * z) * db[11];
    gx += c3 * (-6.0 * x * z) * db[12];
    gy += c3 * (-6.0 * y * z) * db[12];
    gz += c3 * (6.0 * z * z - 3.0 * x * x - 3.0 * y * y) * db[12];
    gx += c4 * (4.0 * z * z - 3.0 * x * x - y * y) * db[13];
    gy += c4 * (-2.0 * x * y) * db[13];
    gz += c4 * (8.0 * x * z) * db[13];
    gx += c5 * (2.0 * x * z) * db[14];
    gy += c5 * (-2.0 * y * z) * db[14];
    gz += c5 * (x * x - y * y) * db[14];
    gx += c6 * (3.0 * x * x - 3.0 * y * y) * db[15];
    gy += c6 * (-6.0 * x * y) * db[15];
  }
}

// One thread per Gaussian.  Gaussians with an all-zero accumulator (culled or
// never composited) get exactly zero gradients (the chain rule is linear).
template <int DEG>
__global__ void __launch_bounds__(128) k_chain_rule_t(ChainArgs c) {
  constexpr int B = (DEG + 1) * (DEG + 1);
  const int64_t n = c.sc.n;
  const int64_t P = 11 + 3 * B;
  const CamD &cam = c.cam;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool any = false;
    for (int k = 0; k < c.kg; ++k) {
      const float4 *a4 = reinterpret_cast<const float4 *>(c.acc + ((int64_t)i * c.kg + k) * kAcc);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float4 x = a4[s];
        any |= (x.x != 0.f) | (x.y != 0.f) | (x.z != 0.f) | (x.w != 0.f);
      }
      if (c.acc_ext) {
        const float4 x = *reinterpret_cast<const float4 *>(c.acc_ext + ((int64_t)i * c.kg + k) * kAccExt);
        any |= (x.x != 0.f) | (x.y != 0.f) | (x.z != 0.f) | (x.w != 0.f);
      }
    }
    if (!any) {
      for (int k = 0; k < c.kg; ++k) {
        float *g = c.grads + (int64_t)k * n * P;
#pragma unroll
        for (int s = 0; s < 3; ++s) { g[3 * i + s] = 0.f; g[3 * n + 3 * i + s] = 0.f; }
#pragma unroll
        for (int s = 0; s < 4; ++s) g[6 * n + 4 * i + s] = 0.f;
        g[10 * n + i] = 0.f;
#pragma unroll
        for (int s = 0; s < 3 * B; ++s) g[11 * n + 3 * B * i + s] = 0.f;
      }
      continue;
    }
    double p[3], t[3];
    load_center_d(c.sc, i, p);
    t_cam_d(cam, p, t);
    const double X = t[0], Y = t[1], Z = t[2];
    const double q0 = c.sc.rotation[4 * i], q1 = c.sc.rotation[4 * i + 1], q2 = c.sc.rotation[4 * i + 2],
                 q3 = c.sc.rotation[4 * i + 3];
    const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    const double qh[4] = {q0 / qn, q1 / qn, q2 / qn, q3 / qn};
    double R[9];
    quat_to_matrix_d(qh[0], qh[1], qh[2], qh[3], R);
    const double sv[3] = {exp((double)c.sc.log_scale[3 * i]), exp((double)c.sc.log_scale[3 * i + 1]),
                          exp((double)c.sc.log_scale[3 * i + 2])};
    const double alpha = expit_d((double)c.sc.opacity_logit[i]);
    const bool is3d = c.sc.type_spec[i] == 1;
    const double fx = cam.fx, fy = cam.fy;
    // view direction, SH basis, raw colour mask (core/sh.py:110-141)
    const double dl0 = p[0] - cam.campos[0], dl1 = p[1] - cam.campos[1], dl2 = p[2] - cam.campos[2];
    const double dist = sqrt((dl0 * dl0 + dl1 * dl1) + dl2 * dl2);
    const double dden = dist > 1e-12 ? dist : 1e-12;
    const double vx = dl0 / dden, vy = dl1 / dden, vz = dl2 / dden;
    double basis[16];
    sh_basis_d(DEG, vx, vy, vz, basis);
    const float *shc = c.sc.sh + (int64_t)3 * B * i;
    double mask[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double raw = 0.0;
#pragma unroll
      for (int bb = 0; bb < B; ++bb) raw += (double)shc[ch * B + bb] * basis[bb];
      mask[ch] = (raw + 0.5) > 0.0 ? 1.0 : 0.0;
    }
    // normal extension: axis and facing sign
    int ax = 2;
    if (is3d) ax = (sv[0] <= sv[1] && sv[0] <= sv[2]) ? 0 : (sv[1] <= sv[2] ? 1 : 2);
    double nc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) nc[r] = (cam.V[r * 3] * R[ax] + cam.V[r * 3 + 1] * R[3 + ax]) + cam.V[r * 3 + 2] * R[6 + ax];
    const double sg = ((nc[0] * X + nc[1] * Y) + nc[2] * Z) > 0.0 ? -1.0 : 1.0;

    for (int k = 0; k < c.kg; ++k) {
      const float *A = c.acc + ((int64_t)i * c.kg + k) * kAcc;
      float *g = c.grads + (int64_t)k * n * P;
      double d_center[3] = {0, 0, 0}, d_ls[3] = {0, 0, 0}, d_R[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      // SH (core/sh.py:125-141)
      const double up0 = A[0] * mask[0], up1 = A[1] * mask[1], up2 = A[2] * mask[2];
      double db[16];
#pragma unroll
      for (int bb = 0; bb < B; ++bb) {
        const double s0 = shc[bb], s1 = shc[B + bb], s2 = shc[2 * B + bb];
        g[11 * n + 3 * B * i + bb] = (float)(up0 * basis[bb]);
        g[11 * n + 3 * B * i + B + bb] = (float)(up1 * basis[bb]);
        g[11 * n + 3 * B * i + 2 * B + bb] = (float)(up2 * basis[bb]);
        db[bb] = (s0 * up0 + s1 * up1) + s2 * up2;
      }
      double gdx, gdy, gdz;
      sh_dir_grad<DEG>(vx, vy, vz, db, gdx, gdy, gdz);
      const double dot = (gdx * vx + gdy * vy) + gdz * vz;
      d_center[0] += (gdx - dot * vx) / dist;
      d_center[1] += (gdy - dot * vy) / dist;
      d_center[2] += (gdz - dot * vz) / dist;
      // opacity: A[3] = dL/dalpha_eff * alpha_eff (exchange.py:114-129 folded in)
      const double Aal = A[3];
      const double d_logit = Aal * (1.0 - alpha);
      // projected centre (backward.py:121-126)
      const double gx = A[4], gy = A[5];
      double dX = gx * fx / Z, dY = gy * fy / Z;
      double dZ = -gx * fx * X / (Z * Z) - gy * fy * Y / (Z * Z);
      if (is3d) {
        // backward.py:128-150
        const double J[6] = {fx / Z, 0.0, -fx * X / (Z * Z), 0.0, fy / Z, -fy * Y / (Z * Z)};
        double U[6];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            U[r * 3 + cc] = (J[r * 3] * cam.V[cc] + J[r * 3 + 1] * cam.V[3 + cc]) + J[r * 3 + 2] * cam.V[6 + cc];
        const double D3[3] = {sv[0] * sv[0], sv[1] * sv[1], sv[2] * sv[2]};
        const double G00 = A[6], G01 = A[7], G11 = A[8];
        // dS = U^T G U (G symmetric)
        double GU[6];
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          GU[l] = G00 * U[l] + G01 * U[3 + l];
          GU[3 + l] = G01 * U[l] + G11 * U[3 + l];
        }
        double dS[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l) dS[a * 3 + l] = U[a] * GU[l] + U[3 + a] * GU[3 + l];
        // dU = (G + G^T) U Sigma = 2 G U Sigma ; Sigma = R D R^T
        double RD[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b2 = 0; b2 < 3; ++b2) RD[a * 3 + b2] = R[a * 3 + b2] * D3[b2];
        double Sig[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l) Sig[a * 3 + l] = (RD[a * 3] * R[l * 3] + RD[a * 3 + 1] * R[l * 3 + 1]) + RD[a * 3 + 2] * R[l * 3 + 2];
        double dU[6];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l)
            dU[a * 3 + l] = 2.0 * ((GU[a * 3] * Sig[l] + GU[a * 3 + 1] * Sig[3 + l]) + GU[a * 3 + 2] * Sig[6 + l]);
        double dJ[6];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            dJ[a * 3 + cc] = (dU[a * 3] * cam.V[cc * 3] + dU[a * 3 + 1] * cam.V[cc * 3 + 1]) + dU[a * 3 + 2] * cam.V[cc * 3 + 2];
        const double z2 = Z * Z, z3 = Z * Z * Z;
        dX += dJ[2] * (-fx / z2);
        dY += dJ[5] * (-fy / z2);
        dZ += ((dJ[0] * (-fx / z2) + dJ[4] * (-fy / z2)) + dJ[2] * (2.0 * fx * X / z3)) + dJ[5] * (2.0 * fy * Y / z3);
        // d_R = (dS + dS^T) R D, d_ls = 2 D diag(R^T dS R)  (dS symmetric here)
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int kk = 0; kk < 3; ++kk)
            d_R[a * 3 + kk] += 2.0 * ((dS[a * 3] * R[kk] + dS[a * 3 + 1] * R[3 + kk]) + dS[a * 3 + 2] * R[6 + kk]) * D3[kk];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double s2 = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) s2 += R[j * 3 + a] * ((dS[j * 3] * R[a] + dS[j * 3 + 1] * R[3 + a]) + dS[j * 3 + 2] * R[6 + a]);
          d_ls[a] += 2.0 * D3[a] * s2;
        }
      } else {
        // 2D: slots 6-14 are dL/d(m0', m1', m3') in anchor-relative pixels;
        // undo the re-basing m0' = M0 - ax M3, m1' = M1 - ay M3 (write_record)
        const double ctr_x = fx * X / Z + cam.cx, ctr_y = fy * Y / Z + cam.cy;
        double axd = fmin(fmax(floor(ctr_x), -1073741824.0), 1073741824.0);
        double ayd = fmin(fmax(floor(ctr_y), -1073741824.0), 1073741824.0);
        if (isnan(axd)) axd = 0.0;
        if (isnan(ayd)) ayd = 0.0;
        const double gm0[4] = {A[6], A[7], 0.0, A[8]};
        const double gm1[4] = {A[9], A[10], 0.0, A[11]};
        double gm3[4] = {A[12], A[13], 0.0, A[14]};
#pragma unroll
        for (int d = 0; d < 4; ++d) gm3[d] -= axd * gm0[d] + ayd * gm1[d];
        // dH = T^T dM over rows (0, 1, 3) of T (backward.py:152-164)
        double dH[12];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int d = 0; d < 4; ++d)
            dH[cc * 4 + d] = (cam.T[0 * 4 + cc] * gm0[d] + cam.T[1 * 4 + cc] * gm1[d]) + cam.T[3 * 4 + cc] * gm3[d];
        const double sx = sv[0], sy = sv[1];
        d_ls[0] += ((R[0] * dH[0] + R[3] * dH[4]) + R[6] * dH[8]) * sx;
        d_ls[1] += ((R[1] * dH[1] + R[4] * dH[5]) + R[7] * dH[9]) * sy;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          d_R[a * 3 + 0] += sx * dH[a * 4 + 0];
          d_R[a * 3 + 1] += sy * dH[a * 4 + 1];
          d_center[a] += dH[a * 4 + 3];
        }
        // modulation (exchange.py:114-129): dL/dls_z = A * (-lambda) (gate + sz gate (1-gate) / T_z) sz
        const double sz = sv[2];
        const double gate = expit_d((sz - c.mod.theta_z) / c.mod.t_z);
        d_ls[2] += Aal * (-c.mod.lambda_z) * (gate + sz * gate * (1.0 - gate) / c.mod.t_z) * sz;
      }
      if (c.acc_ext) {
        const float *E = c.acc_ext + ((int64_t)i * c.kg + k) * kAccExt;
        dZ += E[0];
#pragma unroll
        for (int a = 0; a < 3; ++a)
          d_R[a * 3 + ax] += sg * ((cam.V[a] * E[1] + cam.V[3 + a] * E[2]) + cam.V[6 + a] * E[3]);
      }
      // t_cam -> world centre
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) d_center[cc] += (dX * cam.V[cc] + dY * cam.V[3 + cc]) + dZ * cam.V[6 + cc];
      // quaternion (rotation.py:79-107), then / |q| (backward.py:172)
      const double w = qh[0], x = qh[1], y = qh[2], zq = qh[3];
#define GR(ii, jj) d_R[(ii) * 3 + (jj)]
      const double dw = 2.0 * (((((-zq * GR(0, 1) + y * GR(0, 2)) + zq * GR(1, 0)) - x * GR(1, 2)) - y * GR(2, 0)) + x * GR(2, 1));
      const double dxq = 2.0 * (((((((y * GR(0, 1) + zq * GR(0, 2)) + y * GR(1, 0)) - 2.0 * x * GR(1, 1)) - w * GR(1, 2)) +
                                 zq * GR(2, 0)) + w * GR(2, 1)) - 2.0 * x * GR(2, 2));
      const double dyq = 2.0 * (((((((-2.0 * y * GR(0, 0) + x * GR(0, 1)) + w * GR(0, 2)) + x * GR(1, 0)) + zq * GR(1, 2)) -
                                 w * GR(2, 0)) + zq * GR(2, 1)) - 2.0 * y * GR(2, 2));
      const double dzq = 2.0 * (((((((-2.0 * zq * GR(0, 0) - w * GR(0, 1)) + x * GR(0, 2)) + w * GR(1, 0)) -
                                  2.0 * zq * GR(1, 1)) + y * GR(1, 2)) + x * GR(2, 0)) + y * GR(2, 1));
#undef GR
      const double dotq = ((dw * w + dxq * x) + dyq * y) + dzq * zq;
      g[3 * i + 0] = (float)d_center[0];
      g[3 * i + 1] = (float)d_center[1];
      g[3 * i + 2] = (float)d_center[2];
      g[3 * n + 3 * i + 0] = (float)d_ls[0];
      g[3 * n + 3 * i + 1] = (float)d_ls[1];
      g[3 * n + 3 * i + 2] = (float)d_ls[2];
      g[6 * n + 4 * i + 0] = (float)((dw - dotq * w) / qn);
      g[6 * n + 4 * i + 1] = (float)((dxq - dotq * x) / qn);
      g[6 * n + 4 * i + 2] = (float)((dyq - dotq * y) / qn);
      g[6 * n + 4 * i + 3] = (float)((dzq - dotq * zq) / qn);
      g[10 * n + i] = (float)d_logit;
    }
  }
}

template __global__ void k_chain_rule_t<0>(ChainArgs);
template __global__ void k_chain_rule_t<1>(ChainArgs);
template __global__ void k_chain_rule_t<2>(ChainArgs);
template __global__ void k_chain_rule_t<3>(ChainArgs);

}  // namespace hgs
