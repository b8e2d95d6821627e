// hgs_backward.cu -- backward kernels.
//  k_composite_bwd : back-to-front replay per tile (raster/_blend_py.py:126-242)
//                    with warp transpose-reduction before the atomics.
//  k_chain_rule    : per-Gaussian float64 chain rule (grad/backward.py:68-178,
//                    core/sh.py:125-141, core/rotation.py:79-107,
//                    exchange.py:114-129) writing ParamGrads.
#include "hgs_kernels.cuh"

namespace hgs {

constexpr int kAcc = 16;     // accumulator slots per (Gaussian, kg): see hgs_composite_bwd.cu
constexpr int kAccExt = 4;

// --------------------------------------------------------- chain rule

// core/sh.py:63-107, d basis / d dir, out (B, 3)
__device__ __forceinline__ void sh_basis_grad_d(int deg, double x, double y, double z, double (*g)[3]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) g[i][0] = g[i][1] = g[i][2] = 0.0;
  const double C1 = 0.4886025119029199;
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                        0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                        -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
  if (deg >= 1) {
    g[1][1] = -C1;
    g[2][2] = C1;
    g[3][0] = -C1;
  }
  if (deg >= 2) {
    g[4][0] = C2[0] * y; g[4][1] = C2[0] * x;
    g[5][1] = C2[1] * z; g[5][2] = C2[1] * y;
    g[6][0] = C2[2] * (-2.0 * x); g[6][1] = C2[2] * (-2.0 * y); g[6][2] = C2[2] * (4.0 * z);
    g[7][0] = C2[3] * z; g[7][2] = C2[3] * x;
    g[8][0] = C2[4] * (2.0 * x); g[8][1] = C2[4] * (-2.0 * y);
  }
  if (deg >= 3) {
    g[9][0] = C3[0] * 6.0 * x * y; g[9][1] = C3[0] * (3.0 * x * x - 3.0 * y * y);
    g[10][0] = C3[1] * y * z; g[10][1] = C3[1] * x * z; g[10][2] = C3[1] * x * y;
    g[11][0] = C3[2] * (-2.0 * x * y); g[11][1] = C3[2] * (4.0 * z * z - x * x - 3.0 * y * y);
    g[11][2] = C3[2] * (8.0 * y * z);
    g[12][0] = C3[3] * (-6.0 * x * z); g[12][1] = C3[3] * (-6.0 * y * z);
    g[12][2] = C3[3] * (6.0 * z * z - 3.0 * x * x - 3.0 * y * y);
    g[13][0] = C3[4] * (4.0 * z * z - 3.0 * x * x - y * y); g[13][1] = C3[4] * (-2.0 * x * y);
    g[13][2] = C3[4] * (8.0 * x * z);
    g[14][0] = C3[5] * (2.0 * x * z); g[14][1] = C3[5] * (-2.0 * y * z); g[14][2] = C3[5] * (x * x - y * y);
    g[15][0] = C3[6] * (3.0 * x * x - 3.0 * y * y); g[15][1] = C3[6] * (-6.0 * x * y);
  }
}

// One thread per Gaussian (original index).  Gaussians with an all-zero
// accumulator (culled or never composited) get exactly zero gradients.
__global__ void __launch_bounds__(128) k_chain_rule(ChainArgs c) {
  const int64_t n = c.sc.n;
  const int B = c.sc.sh_bases;
  const int64_t P = 11 + 3 * B;
  const int deg = B == 1 ? 0 : (B == 4 ? 1 : (B == 9 ? 2 : 3));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // does any kg have a non-zero accumulator?
    bool any = false;
    for (int k = 0; k < c.kg; ++k) {
      const float4 *a4 = reinterpret_cast<const float4 *>(c.acc + ((int64_t)i * c.kg + k) * kAcc);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        float4 x = a4[s];
        any |= (x.x != 0.f) | (x.y != 0.f) | (x.z != 0.f) | (x.w != 0.f);
      }
      if (c.acc_ext) {
        float4 x = *reinterpret_cast<const float4 *>(c.acc_ext + ((int64_t)i * c.kg + k) * kAccExt);
        any |= (x.x != 0.f) | (x.y != 0.f) | (x.z != 0.f) | (x.w != 0.f);
      }
    }
    if (!any) {
      for (int k = 0; k < c.kg; ++k) {
        float *g = c.grads + (int64_t)k * n * P;
        for (int s = 0; s < 3; ++s) { g[3 * i + s] = 0.f; g[3 * n + 3 * i + s] = 0.f; }
        for (int s = 0; s < 4; ++s) g[6 * n + 4 * i + s] = 0.f;
        g[10 * n + i] = 0.f;
        for (int s = 0; s < 3 * B; ++s) g[11 * n + 3 * B * i + s] = 0.f;
      }
      continue;
    }
    const CamD &cam = c.cam;
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
    // 3D geometry
    double U[6], D3[3], Sig[9];
    if (is3d) {
      double J[6] = {fx / Z, 0.0, -fx * X / (Z * Z), 0.0, fy / Z, -fy * Y / (Z * Z)};
      for (int r = 0; r < 2; ++r)
        for (int cc = 0; cc < 3; ++cc)
          U[r * 3 + cc] = (J[r * 3] * cam.V[cc] + J[r * 3 + 1] * cam.V[3 + cc]) + J[r * 3 + 2] * cam.V[6 + cc];
      for (int j = 0; j < 3; ++j) D3[j] = sv[j] * sv[j];
      for (int aa = 0; aa < 3; ++aa)
        for (int cc = 0; cc < 3; ++cc)
          Sig[aa * 3 + cc] = (R[aa * 3] * D3[0] * R[cc * 3] + R[aa * 3 + 1] * D3[1] * R[cc * 3 + 1]) +
                             R[aa * 3 + 2] * D3[2] * R[cc * 3 + 2];
    }
    // modulation gradient factor (exchange.py:114-129) times alpha_eff
    double dlz_per_A = 0.0;
    if (!is3d) {
      const double sz = sv[2];
      const double gate = expit_d((sz - c.mod.theta_z) / c.mod.t_z);
      dlz_per_A = (-c.mod.lambda_z) * (gate + sz * gate * (1.0 - gate) / c.mod.t_z) * sz;
    }
    // anchor used by the compositor for 2D rows (write_record)
    const double ctr_x = fx * X / Z + cam.cx, ctr_y = fy * Y / Z + cam.cy;
    double axd = fmin(fmax(floor(ctr_x), -1073741824.0), 1073741824.0);
    double ayd = fmin(fmax(floor(ctr_y), -1073741824.0), 1073741824.0);
    if (isnan(axd)) axd = 0.0;
    if (isnan(ayd)) ayd = 0.0;
    // SH basis, raw colour mask
    double dl[3] = {p[0] - cam.campos[0], p[1] - cam.campos[1], p[2] - cam.campos[2]};
    const double dist = sqrt((dl[0] * dl[0] + dl[1] * dl[1]) + dl[2] * dl[2]);
    const double dden = dist > 1e-12 ? dist : 1e-12;
    const double vd[3] = {dl[0] / dden, dl[1] / dden, dl[2] / dden};
    double basis[16];
    sh_basis_d(deg, vd[0], vd[1], vd[2], basis);
    const float *shc = c.sc.sh + (int64_t)3 * B * i;
    double mask[3];
    for (int ch = 0; ch < 3; ++ch) {
      double acc2 = 0.0;
      for (int bb = 0; bb < B; ++bb) acc2 += (double)shc[ch * B + bb] * basis[bb];
      mask[ch] = (acc2 + 0.5) > 0.0 ? 1.0 : 0.0;
    }
    double bgrad[16][3];
    sh_basis_grad_d(deg, vd[0], vd[1], vd[2], bgrad);
    // normal extension
    int ax = 2;
    if (is3d) ax = (sv[0] <= sv[1] && sv[0] <= sv[2]) ? 0 : (sv[1] <= sv[2] ? 1 : 2);
    double nc[3];
    for (int r = 0; r < 3; ++r) nc[r] = (cam.V[r * 3] * R[ax] + cam.V[r * 3 + 1] * R[3 + ax]) + cam.V[r * 3 + 2] * R[6 + ax];
    const double sg = ((nc[0] * X + nc[1] * Y) + nc[2] * Z) > 0.0 ? -1.0 : 1.0;

    for (int k = 0; k < c.kg; ++k) {
      const float *A = c.acc + ((int64_t)i * c.kg + k) * kAcc;
      float *g = c.grads + (int64_t)k * n * P;
      double d_center[3] = {0, 0, 0}, d_ls[3] = {0, 0, 0}, d_R[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, d_logit;
      // SH (core/sh.py:125-141)
      const double up[3] = {A[0] * mask[0], A[1] * mask[1], A[2] * mask[2]};
      for (int ch = 0; ch < 3; ++ch)
        for (int bb = 0; bb < B; ++bb) g[11 * n + 3 * B * i + ch * B + bb] = (float)(up[ch] * basis[bb]);
      double d_dir[3] = {0, 0, 0};
      for (int bb = 0; bb < B; ++bb) {
        const double db = ((double)shc[bb] * up[0] + (double)shc[B + bb] * up[1]) + (double)shc[2 * B + bb] * up[2];
        d_dir[0] += db * bgrad[bb][0];
        d_dir[1] += db * bgrad[bb][1];
        d_dir[2] += db * bgrad[bb][2];
      }
      const double dot = (d_dir[0] * vd[0] + d_dir[1] * vd[1]) + d_dir[2] * vd[2];
      for (int cc = 0; cc < 3; ++cc) d_center[cc] += (d_dir[cc] - dot * vd[cc]) / dist;
      // opacity: A[3] = g_alpha_eff * alpha_eff
      const double Aal = A[3];
      d_logit = Aal * (1.0 - alpha);
      // projected centre (backward.py:121-126)
      const double gx = A[4], gy = A[5];
      double dX = gx * fx / Z, dY = gy * fy / Z;
      double dZ = -gx * fx * X / (Z * Z) - gy * fy * Y / (Z * Z);
      if (is3d) {
        // backward.py:128-150
        const double Gp[4] = {A[6], A[7], A[7], A[8]};
        double dS[9], dU[6], dJ[6];
        for (int aa = 0; aa < 3; ++aa)
          for (int l = 0; l < 3; ++l) {
            double s2 = 0.0;
            for (int j = 0; j < 2; ++j)
              for (int kk = 0; kk < 2; ++kk) s2 += U[j * 3 + aa] * Gp[j * 2 + kk] * U[kk * 3 + l];
            dS[aa * 3 + l] = s2;
          }
        double GG[4];
        for (int aa = 0; aa < 2; ++aa)
          for (int bb = 0; bb < 2; ++bb) GG[aa * 2 + bb] = Gp[aa * 2 + bb] + Gp[bb * 2 + aa];
        for (int aa = 0; aa < 2; ++aa)
          for (int l = 0; l < 3; ++l) {
            double s2 = 0.0;
            for (int j = 0; j < 2; ++j)
              for (int kk = 0; kk < 3; ++kk) s2 += GG[aa * 2 + j] * U[j * 3 + kk] * Sig[kk * 3 + l];
            dU[aa * 3 + l] = s2;
          }
        for (int aa = 0; aa < 2; ++aa)
          for (int cc = 0; cc < 3; ++cc)
            dJ[aa * 3 + cc] = (dU[aa * 3] * cam.V[cc * 3] + dU[aa * 3 + 1] * cam.V[cc * 3 + 1]) + dU[aa * 3 + 2] * cam.V[cc * 3 + 2];
        const double z2 = Z * Z, z3 = Z * Z * Z;
        dX += dJ[2] * (-fx / z2);
        dY += dJ[5] * (-fy / z2);
        dZ += ((dJ[0] * (-fx / z2) + dJ[4] * (-fy / z2)) + dJ[2] * (2.0 * fx * X / z3)) + dJ[5] * (2.0 * fy * Y / z3);
        double dSs[9];
        for (int aa = 0; aa < 3; ++aa)
          for (int bb = 0; bb < 3; ++bb) dSs[aa * 3 + bb] = dS[aa * 3 + bb] + dS[bb * 3 + aa];
        for (int aa = 0; aa < 3; ++aa)
          for (int kk = 0; kk < 3; ++kk)
            d_R[aa * 3 + kk] += ((dSs[aa * 3] * R[kk] + dSs[aa * 3 + 1] * R[3 + kk]) + dSs[aa * 3 + 2] * R[6 + kk]) * D3[kk];
        for (int aa = 0; aa < 3; ++aa) {
          double s2 = 0.0;
          for (int j = 0; j < 3; ++j)
            for (int kk = 0; kk < 3; ++kk) s2 += R[j * 3 + aa] * dS[j * 3 + kk] * R[kk * 3 + aa];
          d_ls[aa] += 2.0 * D3[aa] * s2;
        }
      } else {
        // 2D: slots 6-14 hold dL/d(m0', m1', m3') in anchor-relative pixels.
        // Undo the re-basing: m0' = M0 - ax M3, m1' = M1 - ay M3.
        const double gm0[4] = {A[6], A[7], 0.0, A[8]};
        const double gm1[4] = {A[9], A[10], 0.0, A[11]};
        double gm3[4] = {A[12], A[13], 0.0, A[14]};
        for (int d = 0; d < 4; ++d) gm3[d] -= axd * gm0[d] + ayd * gm1[d];
        // dH = T^T dM (rows 0, 1, 3 of T), backward.py:152-164
        double dH[12];
        for (int cc = 0; cc < 3; ++cc)
          for (int d = 0; d < 4; ++d)
            dH[cc * 4 + d] = (cam.T[0 * 4 + cc] * gm0[d] + cam.T[1 * 4 + cc] * gm1[d]) + cam.T[3 * 4 + cc] * gm3[d];
        const double sx = sv[0], sy = sv[1];
        d_ls[0] += ((R[0] * dH[0] + R[3] * dH[4]) + R[6] * dH[8]) * sx;
        d_ls[1] += ((R[1] * dH[1] + R[4] * dH[5]) + R[7] * dH[9]) * sy;
        for (int aa = 0; aa < 3; ++aa) {
          d_R[aa * 3 + 0] += sx * dH[aa * 4 + 0];
          d_R[aa * 3 + 1] += sy * dH[aa * 4 + 1];
          d_center[aa] += dH[aa * 4 + 3];
        }
        d_ls[2] += Aal * dlz_per_A;
      }
      if (c.acc_ext) {
        const float *E = c.acc_ext + ((int64_t)i * c.kg + k) * kAccExt;
        dZ += E[0];
        for (int aa = 0; aa < 3; ++aa)
          d_R[aa * 3 + ax] += sg * ((cam.V[aa] * E[1] + cam.V[3 + aa] * E[2]) + cam.V[6 + aa] * E[3]);
      }
      const double dt[3] = {dX, dY, dZ};
      for (int cc = 0; cc < 3; ++cc) d_center[cc] += (dt[0] * cam.V[cc] + dt[1] * cam.V[3 + cc]) + dt[2] * cam.V[6 + cc];
      // quaternion (rotation.py:79-107), then / |q| (backward.py:172)
      const double w = qh[0], x = qh[1], y = qh[2], zq = qh[3];
#define GR(ii, jj) d_R[(ii) * 3 + (jj)]
      double dw = 2.0 * (((((-zq * GR(0, 1) + y * GR(0, 2)) + zq * GR(1, 0)) - x * GR(1, 2)) - y * GR(2, 0)) + x * GR(2, 1));
      double dxq = 2.0 * (((((((y * GR(0, 1) + zq * GR(0, 2)) + y * GR(1, 0)) - 2.0 * x * GR(1, 1)) - w * GR(1, 2)) +
                           zq * GR(2, 0)) + w * GR(2, 1)) - 2.0 * x * GR(2, 2));
      double dyq = 2.0 * (((((((-2.0 * y * GR(0, 0) + x * GR(0, 1)) + w * GR(0, 2)) + x * GR(1, 0)) + zq * GR(1, 2)) -
                           w * GR(2, 0)) + zq * GR(2, 1)) - 2.0 * y * GR(2, 2));
      double dzq = 2.0 * (((((((-2.0 * zq * GR(0, 0) - w * GR(0, 1)) + x * GR(0, 2)) + w * GR(1, 0)) -
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

}  // namespace hgs
