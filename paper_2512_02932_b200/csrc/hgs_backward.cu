// hgs_backward.cu -- the per-Gaussian chain rule (grad/backward.py:68-178,
// core/sh.py:125-141, core/rotation.py:79-107, exchange.py:114-129): from
// the screen-space accumulators of k_composite_bwd to ParamGrads.
//
// One thread per Gaussian in original index order (coalesced reads of the
// scene and accumulators, coalesced field-major writes).  Templated on the SH
// degree so every loop unrolls into registers.  Mixed precision: float32 for
// the 3D covariance chain, SH and quaternion terms; float64 where float32
// would lose the answer -- the 2D anchor un-rebasing and T^T dM (terms of
// ~1e3 pixels cancel), the anchor itself (it must reproduce write_record's
// floor exactly), the steep modulation gate (T_z = 1e-3), and a guarded
// float64 re-evaluation of the colour-clamp mask near raw = 0.
#include "hgs_kernels.cuh"

namespace hgs {

constexpr int kAcc = 16;  // accumulator slots per (Gaussian, kg): see hgs_composite_bwd.cu
constexpr int kAccExt = 4;

// sum_b db[b] * dY_b / d(dir)   (core/sh.py:63-107, contracted with db)
template <int DEG>
__device__ __forceinline__ void sh_dir_grad(float x, float y, float z, const float *db, float &gx, float &gy,
                                            float &gz) {
  const float C1 = 0.4886025119029199f;
  gx = gy = gz = 0.f;
  if (DEG >= 1) {
    gy += -C1 * db[1];
    gz += C1 * db[2];
    gx += -C1 * db[3];
  }
  if (DEG >= 2) {
    const float A = 1.0925484305920792f, Bq = -1.0925484305920792f, Cq = 0.31539156525252005f,
                Dq = -1.0925484305920792f, Eq = 0.5462742152960396f;
    gx += A * y * db[4];
    gy += A * x * db[4];
    gy += Bq * z * db[5];
    gz += Bq * y * db[5];
    gx += Cq * (-2.f * x) * db[6];
    gy += Cq * (-2.f * y) * db[6];
    gz += Cq * (4.f * z) * db[6];
    gx += Dq * z * db[7];
    gz += Dq * x * db[7];
    gx += Eq * (2.f * x) * db[8];
    gy += Eq * (-2.f * y) * db[8];
  }
  if (DEG >= 3) {
    const float c0 = -0.5900435899266435f, c1 = 2.890611442640554f, c2 = -0.4570457994644658f,
                c3 = 0.3731763325901154f, c4 = -0.4570457994644658f, c5 = 1.445305721320277f,
                c6 = -0.5900435899266435f;
    gx += c0 * 6.f * x * y * db[9];
    gy += c0 * (3.f * x * x - 3.f * y * y) * db[9];
    gx += c1 * y * z * db[10];
    gy += c1 * x * z * db[10];
    gz += c1 * x * y * db[10];
    gx += c2 * (-2.f * x * y) * db[11];
    gy += c2 * (4.f * z * z - x * x - 3.f * y * y) * db[11];
    gz += c2 * (8.f * y * z) * db[11];
    gx += c3 * (-6.f * x * z) * db[12];
    gy += c3 * (-6.f * y * z) * db[12];
    gz += c3 * (6.f * z * z - 3.f * x * x - 3.f * y * y) * db[12];
    gx += c4 * (4.f * z * z - 3.f * x * x - y * y) * db[13];
    gy += c4 * (-2.f * x * y) * db[13];
    gz += c4 * (8.f * x * z) * db[13];
    gx += c5 * (2.f * x * z) * db[14];
    gy += c5 * (-2.f * y * z) * db[14];
    gz += c5 * (x * x - y * y) * db[14];
    gx += c6 * (3.f * x * x - 3.f * y * y) * db[15];
    gy += c6 * (-6.f * x * y) * db[15];
  }
}

// raw + 0.5 > 0 for one channel, decided like the reference's float64
// (core/sh.py:134-135): float32 unless within its error bound of 0.
template <int B>
__device__ __forceinline__ float clamp_mask(const float *shc_ch, const float *basis, double vx, double vy, double vz) {
  float raw = 0.5f, mag = 0.5f;
#pragma unroll
  for (int bb = 0; bb < B; ++bb) {
    const float t = shc_ch[bb] * basis[bb];
    raw += t;
    mag += fabsf(t);
  }
  if (fabsf(raw) > 1e-5f * mag) return raw > 0.f ? 1.f : 0.f;
  double bd[16];
  constexpr int deg = B == 1 ? 0 : (B == 4 ? 1 : (B == 9 ? 2 : 3));
  sh_basis_d(deg, vx, vy, vz, bd);
  double r = 0.0;
#pragma unroll
  for (int bb = 0; bb < B; ++bb) r += (double)shc_ch[bb] * bd[bb];
  return (r + 0.5) > 0.0 ? 1.f : 0.f;
}

// One thread per Gaussian, one warp per CTA, 32 consecutive Gaussians per
// warp step.  The SH coefficients (3B floats per Gaussian) are read and the SH
// gradients written through shared memory, as one contiguous, coalesced
// segment per warp step: per-thread rows of 3B floats at a 12B-byte stride
// would issue 3B scalar memory instructions per thread (LSU-throttled).
// Gaussians with an all-zero accumulator (culled or never composited) get
// exactly zero gradients (the chain rule is linear).
constexpr int kChainThreads = 32;
#ifndef HGS_CHAIN_PREFETCH
#define HGS_CHAIN_PREFETCH 1
#endif
#ifndef HGS_CHAIN_TOUCHED
#define HGS_CHAIN_TOUCHED 1
#endif
#ifndef HGS_CHAIN_MINB
#define HGS_CHAIN_MINB 16  // 16 warps per SM: 128 registers
#endif

template <int DEG>
__global__ void __launch_bounds__(kChainThreads, HGS_CHAIN_MINB) k_chain_rule_t(ChainArgs c) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int B = (DEG + 1) * (DEG + 1);
  constexpr int SB = 3 * B, SS = 3 * B + 1;  // row length, padded smem stride
  extern __shared__ float s_chain[];
  float *s_in = s_chain;                     // [32][SS] SH coefficients
  const int64_t n = c.sc.n;
  const int64_t P = 11 + 3 * B;
  const CamD &cam = c.cam;
  const int lane = threadIdx.x;
  const int64_t g_end = c.g1;  // Gaussians [g0, g1) (HGS ranged chain rule); n is the field stride
  for (int64_t base = c.g0 + (int64_t)blockIdx.x * kChainThreads; base < g_end;
       base += (int64_t)gridDim.x * kChainThreads) {
    const int cnt = (int)(g_end - base < kChainThreads ? g_end - base : kChainThreads);
    for (int e = lane; e < cnt * SB; e += kChainThreads) {
      const int r = e / SB;
      s_in[r * SS + (e - r * SB)] = __ldg(c.sc.sh + base * SB + e);
    }
#if HGS_CHAIN_PREFETCH
    {  // next warp step's SH rows, accumulators and scalar fields into L2
      const int64_t nb = base + (int64_t)gridDim.x * kChainThreads;
      if (nb < g_end && c.kg == 1) {  // (measured: a net loss for the 3-gradient training step)
        const int nc = (int)(g_end - nb < kChainThreads ? g_end - nb : kChainThreads);
        const char *sh0 = reinterpret_cast<const char *>(c.sc.sh + nb * SB);
        for (int l = lane; l * 128 < nc * SB * 4; l += kChainThreads)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(sh0 + 128 * l));
        const char *ac0 = reinterpret_cast<const char *>(c.acc + nb * c.kg * kAcc);
        for (int l = lane; l * 128 < nc * c.kg * kAcc * (int)sizeof(acc_t); l += kChainThreads)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(ac0 + 128 * l));
        const char *ptr = nullptr;
        if (lane < 3) ptr = reinterpret_cast<const char *>(c.sc.center + 3 * nb) + 128 * lane;
        else if (lane < 6) ptr = reinterpret_cast<const char *>(c.sc.log_scale + 3 * nb) + 128 * (lane - 3);
        else if (lane < 10) ptr = reinterpret_cast<const char *>(c.sc.rotation + 4 * nb) + 128 * (lane - 6);
        else if (lane == 10) ptr = reinterpret_cast<const char *>(c.sc.opacity_logit + nb);
        else if (lane == 11) ptr = reinterpret_cast<const char *>(c.sc.type_spec + nb);
        if (ptr) asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
      }
    }
#endif
    __syncwarp();
    const int64_t i = base + lane;
    const bool valid = lane < cnt;
    bool any = false;
    if (valid && HGS_CHAIN_TOUCHED && c.touched) {
      any = c.touched[i] != 0;  // one byte instead of the 16 (+ 4) accumulator slots
    } else if (valid) {
      for (int k = 0; k < c.kg; ++k) {
        const double2 *a2 = reinterpret_cast<const double2 *>(c.acc + ((int64_t)i * c.kg + k) * kAcc);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const double2 x = a2[s];
          any |= (x.x != 0.0) | (x.y != 0.0);
        }
        if (c.acc_ext) {
          const double2 *e2 = reinterpret_cast<const double2 *>(c.acc_ext + ((int64_t)i * c.kg + k) * kAccExt);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const double2 x = e2[s];
            any |= (x.x != 0.0) | (x.y != 0.0);
          }
        }
      }
    }
    // per-Gaussian quantities shared by the kg gradient sets
    double pd[3] = {0.0, 0.0, 0.0}, td[3] = {0.0, 0.0, 1.0};
    float X = 0.f, Y = 0.f, Z = 1.f, w = 1.f, x = 0.f, y = 0.f, zq = 0.f, iqn = 1.f;
    float R[9], V[9], basis[16];
    float sv0 = 1.f, sv1 = 1.f, sv2 = 1.f, ls2 = 0.f, alpha = 0.f, vx = 0.f, vy = 0.f, vz = 0.f, dist = 1.f;
    float mask0 = 0.f, mask1 = 0.f, mask2 = 0.f, sg = 1.f;
    bool is3d = false;
    int ax = 2;
    const float fx = (float)cam.fx, fy = (float)cam.fy;
#pragma unroll
    for (int k = 0; k < 9; ++k) V[k] = (float)cam.V[k];
    const float *shc = s_in + lane * SS;
    if (any) {
    load_center_d(c.sc, i, pd);
    t_cam_d(cam, pd, td);
    X = (float)td[0]; Y = (float)td[1]; Z = (float)td[2];
    const float q0 = c.sc.rotation[4 * i], q1 = c.sc.rotation[4 * i + 1], q2 = c.sc.rotation[4 * i + 2],
                q3 = c.sc.rotation[4 * i + 3];
    const float qn = sqrtf(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    iqn = 1.f / qn;
    w = q0 * iqn; x = q1 * iqn; y = q2 * iqn; zq = q3 * iqn;
    R[0] = 1.f - 2.f * (y * y + zq * zq);
    R[1] = 2.f * (x * y - w * zq);
    R[2] = 2.f * (x * zq + w * y);
    R[3] = 2.f * (x * y + w * zq);
    R[4] = 1.f - 2.f * (x * x + zq * zq);
    R[5] = 2.f * (y * zq - w * x);
    R[6] = 2.f * (x * zq - w * y);
    R[7] = 2.f * (y * zq + w * x);
    R[8] = 1.f - 2.f * (x * x + y * y);
    const float ls0 = c.sc.log_scale[3 * i], ls1 = c.sc.log_scale[3 * i + 1];
    ls2 = c.sc.log_scale[3 * i + 2];
    sv0 = expf(ls0); sv1 = expf(ls1); sv2 = expf(ls2);
    alpha = 1.f / (1.f + expf(-c.sc.opacity_logit[i]));
    is3d = c.sc.type_spec[i] == 1;
    // view direction, SH basis, colour-clamp mask (core/sh.py:110-141)
    const double dl0 = pd[0] - cam.campos[0], dl1 = pd[1] - cam.campos[1], dl2 = pd[2] - cam.campos[2];
    const double distd = sqrt((dl0 * dl0 + dl1 * dl1) + dl2 * dl2);
    const double dden = distd > 1e-12 ? distd : 1e-12;
    const double vxd = dl0 / dden, vyd = dl1 / dden, vzd = dl2 / dden;
    vx = (float)vxd; vy = (float)vyd; vz = (float)vzd; dist = (float)distd;
    sh_basis_t<float>(DEG, vx, vy, vz, basis);
    mask0 = clamp_mask<B>(shc, basis, vxd, vyd, vzd);
    mask1 = clamp_mask<B>(shc + B, basis, vxd, vyd, vzd);
    mask2 = clamp_mask<B>(shc + 2 * B, basis, vxd, vyd, vzd);
    // normal extension: axis and facing sign
    // (log-scale order == the forward's float64 scale order; facing sign in float64)
    if (is3d) ax = (ls0 <= ls1 && ls0 <= ls2) ? 0 : (ls1 <= ls2 ? 1 : 2);
    double ncd[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      ncd[r] = (cam.V[r * 3] * (double)R[ax] + cam.V[r * 3 + 1] * (double)R[3 + ax]) + cam.V[r * 3 + 2] * (double)R[6 + ax];
    sg = ((ncd[0] * td[0] + ncd[1] * td[1]) + ncd[2] * td[2]) > 0.0 ? -1.f : 1.f;

    }  // any
    // one gradient set at a time: the SH rows go through one shared buffer
    float *const so = s_chain + kChainThreads * SS + lane * SS;
    for (int k = 0; k < c.kg; ++k) {
      float *g = c.grads + (int64_t)k * n * P;
      if (valid && !any) {
        if (!c.accumulate) {
#pragma unroll
          for (int s = 0; s < 3; ++s) { g[3 * i + s] = 0.f; g[3 * n + 3 * i + s] = 0.f; }
#pragma unroll
          for (int s = 0; s < 4; ++s) g[6 * n + 4 * i + s] = 0.f;
          g[10 * n + i] = 0.f;
        }
#pragma unroll
        for (int s = 0; s < SB; ++s) so[s] = 0.f;
      }
      if (any) {
      const acc_t *A = c.acc + ((int64_t)i * c.kg + k) * kAcc;
      float d_center[3] = {0.f, 0.f, 0.f}, d_ls[3] = {0.f, 0.f, 0.f};
      float d_R[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      // SH (core/sh.py:125-141)
      const float up0 = (float)A[0] * mask0, up1 = (float)A[1] * mask1, up2 = (float)A[2] * mask2;
      float db[16];
#pragma unroll
      for (int bb = 0; bb < B; ++bb) {
        so[bb] = up0 * basis[bb];
        so[B + bb] = up1 * basis[bb];
        so[2 * B + bb] = up2 * basis[bb];
        db[bb] = (shc[bb] * up0 + shc[B + bb] * up1) + shc[2 * B + bb] * up2;
      }
      float gdx, gdy, gdz;
      sh_dir_grad<DEG>(vx, vy, vz, db, gdx, gdy, gdz);
      const float dot = (gdx * vx + gdy * vy) + gdz * vz;
      const float idist = 1.f / dist;
      d_center[0] += (gdx - dot * vx) * idist;
      d_center[1] += (gdy - dot * vy) * idist;
      d_center[2] += (gdz - dot * vz) * idist;
      // opacity: A[3] = dL/dalpha_eff * alpha_eff (exchange.py:114-129 folded in)
      const float Aal = (float)A[3];
      const float d_logit = Aal * (1.f - alpha);
      // projected centre (backward.py:121-126) and, for 3D, the EWA Jacobian
      // chain (backward.py:128-150) in float64: for a near-camera, far
      // off-axis Gaussian the dZ terms of dJ cancel by ~100x, so float32
      // here costs ~1e-3 of the result (the accumulators are float64 too)
      double gx = A[4], gy = A[5];
      double G00 = 0.0, G01 = 0.0, G11 = 0.0;
      if (is3d) {
        // slots 4-8 hold the eigenbasis sums (pair_grads); rotate them with
        // the record's own float32 (c, s) -- the basis the pairs used -- to
        // pixel axes, v = M w with M = [[c, -s], [s, c]], in float64
        const float2 e = __ldg(&c.eig[i]);
        const double cs = e.x, sn = e.y;
        const double Sp = A[4], Sq = A[5], Gpp = A[6], Gpq = A[7], Gqq = A[8];
        gx = cs * Sp - sn * Sq;
        gy = sn * Sp + cs * Sq;
        G00 = (cs * cs * Gpp - 2.0 * cs * sn * Gpq) + sn * sn * Gqq;
        G01 = (cs * sn * Gpp + (cs * cs - sn * sn) * Gpq) - cs * sn * Gqq;
        G11 = (sn * sn * Gpp + 2.0 * cs * sn * Gpq) + cs * cs * Gqq;
      }
      const double Xd = td[0], Yd = td[1], Zd = td[2];
      const double fxd = cam.fx, fyd = cam.fy;
      const double iz = 1.0 / Zd, iz2 = iz * iz;
      double dX = gx * fxd * iz, dY = gy * fyd * iz;
      double dZ = -(gx * fxd * Xd + gy * fyd * Yd) * iz2;
      if (is3d) {
        const double J02 = -fxd * Xd * iz2, J12 = -fyd * Yd * iz2;
        double U[6];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          U[cc] = fxd * iz * cam.V[cc] + J02 * cam.V[6 + cc];
          U[3 + cc] = fyd * iz * cam.V[3 + cc] + J12 * cam.V[6 + cc];
        }
        const double D0 = (double)sv0 * sv0, D1 = (double)sv1 * sv1, D2 = (double)sv2 * sv2;
        double GU[6];
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          GU[l] = G00 * U[l] + G01 * U[3 + l];
          GU[3 + l] = G01 * U[l] + G11 * U[3 + l];
        }
        double dS[9];  // U^T G U
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l) dS[a * 3 + l] = U[a] * GU[l] + U[3 + a] * GU[3 + l];
        double Rd[9];
#pragma unroll
        for (int a = 0; a < 9; ++a) Rd[a] = R[a];
        double Sig[9];  // R D R^T
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int l = 0; l < 3; ++l)
            Sig[a * 3 + l] = (Rd[a * 3] * D0 * Rd[l * 3] + Rd[a * 3 + 1] * D1 * Rd[l * 3 + 1]) + Rd[a * 3 + 2] * D2 * Rd[l * 3 + 2];
        double dJ[6];  // dU V^T, dU = 2 G U Sigma
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          double dU[3];
#pragma unroll
          for (int l = 0; l < 3; ++l)
            dU[l] = 2.0 * ((GU[a * 3] * Sig[l] + GU[a * 3 + 1] * Sig[3 + l]) + GU[a * 3 + 2] * Sig[6 + l]);
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            dJ[a * 3 + cc] = (dU[0] * cam.V[cc * 3] + dU[1] * cam.V[cc * 3 + 1]) + dU[2] * cam.V[cc * 3 + 2];
        }
        const double iz3 = iz2 * iz;
        dX += dJ[2] * (-fxd * iz2);
        dY += dJ[5] * (-fyd * iz2);
        dZ += ((dJ[0] * (-fxd * iz2) + dJ[4] * (-fyd * iz2)) + dJ[2] * (2.0 * fxd * Xd * iz3)) + dJ[5] * (2.0 * fyd * Yd * iz3);
        const double Dv[3] = {D0, D1, D2};
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int kk = 0; kk < 3; ++kk)
            d_R[a * 3 + kk] += (float)(2.0 * ((dS[a * 3] * Rd[kk] + dS[a * 3 + 1] * Rd[3 + kk]) + dS[a * 3 + 2] * Rd[6 + kk]) * Dv[kk]);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double s2 = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) s2 += Rd[j * 3 + a] * ((dS[j * 3] * Rd[a] + dS[j * 3 + 1] * Rd[3 + a]) + dS[j * 3 + 2] * Rd[6 + a]);
          d_ls[a] += (float)(2.0 * Dv[a] * s2);
        }
      } else {
        // 2D: slots 6-14 are dL/d(m0', m1', m3') in anchor-relative pixels;
        // undo the re-basing m0' = M0 - ax M3, m1' = M1 - ay M3 (write_record)
        const double ctr_x = cam.fx * td[0] / td[2] + cam.cx, ctr_y = cam.fy * td[1] / td[2] + cam.cy;
        double axd = fmin(fmax(floor(ctr_x), -1073741824.0), 1073741824.0);
        double ayd = fmin(fmax(floor(ctr_y), -1073741824.0), 1073741824.0);
        if (isnan(axd)) axd = 0.0;
        if (isnan(ayd)) ayd = 0.0;
        const double gm0[3] = {A[6], A[7], A[8]};  // columns 0, 1, 3
        const double gm1[3] = {A[9], A[10], A[11]};
        double gm3[3] = {A[12], A[13], A[14]};
#pragma unroll
        for (int d = 0; d < 3; ++d) gm3[d] -= axd * gm0[d] + ayd * gm1[d];
        // dH = T^T dM over rows (0, 1, 3) of T (backward.py:152-164); columns 0, 1, 3 of H
        float dH[3][3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int d = 0; d < 3; ++d)
            dH[cc][d] = (float)((cam.T[0 * 4 + cc] * gm0[d] + cam.T[1 * 4 + cc] * gm1[d]) + cam.T[3 * 4 + cc] * gm3[d]);
        d_ls[0] += ((R[0] * dH[0][0] + R[3] * dH[1][0]) + R[6] * dH[2][0]) * sv0;
        d_ls[1] += ((R[1] * dH[0][1] + R[4] * dH[1][1]) + R[7] * dH[2][1]) * sv1;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          d_R[a * 3 + 0] += sv0 * dH[a][0];
          d_R[a * 3 + 1] += sv1 * dH[a][1];
          d_center[a] += dH[a][2];
        }
        // modulation (exchange.py:114-129): dL/dls_z = A (-lambda) (gate + sz gate (1-gate) / T_z) sz
        const double sz = exp((double)ls2);
        const double gate = expit_d((sz - c.mod.theta_z) / c.mod.t_z);
        d_ls[2] += (float)((double)Aal * (-c.mod.lambda_z) * (gate + sz * gate * (1.0 - gate) / c.mod.t_z) * sz);
      }
      if (c.acc_ext) {
        const acc_t *E = c.acc_ext + ((int64_t)i * c.kg + k) * kAccExt;
        dZ += E[0];
        const float E1 = (float)E[1], E2 = (float)E[2], E3 = (float)E[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) d_R[a * 3 + ax] += sg * ((V[a] * E1 + V[3 + a] * E2) + V[6 + a] * E3);
      }
      // t_cam -> world centre
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) d_center[cc] += (float)((dX * cam.V[cc] + dY * cam.V[3 + cc]) + dZ * cam.V[6 + cc]);
      // quaternion (rotation.py:79-107), then / |q| (backward.py:172)
#define GR(ii, jj) d_R[(ii) * 3 + (jj)]
      const float dw = 2.f * (((((-zq * GR(0, 1) + y * GR(0, 2)) + zq * GR(1, 0)) - x * GR(1, 2)) - y * GR(2, 0)) + x * GR(2, 1));
      const float dxq = 2.f * (((((((y * GR(0, 1) + zq * GR(0, 2)) + y * GR(1, 0)) - 2.f * x * GR(1, 1)) - w * GR(1, 2)) +
                                zq * GR(2, 0)) + w * GR(2, 1)) - 2.f * x * GR(2, 2));
      const float dyq = 2.f * (((((((-2.f * y * GR(0, 0) + x * GR(0, 1)) + w * GR(0, 2)) + x * GR(1, 0)) + zq * GR(1, 2)) -
                                w * GR(2, 0)) + zq * GR(2, 1)) - 2.f * y * GR(2, 2));
      const float dzq = 2.f * (((((((-2.f * zq * GR(0, 0) - w * GR(0, 1)) + x * GR(0, 2)) + w * GR(1, 0)) -
                                 2.f * zq * GR(1, 1)) + y * GR(1, 2)) + x * GR(2, 0)) + y * GR(2, 1));
#undef GR
      const float dotq = ((dw * w + dxq * x) + dyq * y) + dzq * zq;
      const float gv[11] = {d_center[0], d_center[1], d_center[2], d_ls[0], d_ls[1], d_ls[2],
                            (dw - dotq * w) * iqn, (dxq - dotq * x) * iqn, (dyq - dotq * y) * iqn,
                            (dzq - dotq * zq) * iqn, d_logit};
      float *const gp[11] = {g + 3 * i, g + 3 * i + 1, g + 3 * i + 2, g + 3 * n + 3 * i, g + 3 * n + 3 * i + 1,
                             g + 3 * n + 3 * i + 2, g + 6 * n + 4 * i, g + 6 * n + 4 * i + 1, g + 6 * n + 4 * i + 2,
                             g + 6 * n + 4 * i + 3, g + 10 * n + i};
      if (c.accumulate) {  // multi-view: this view's gradient is added to the running sum
#pragma unroll
        for (int f = 0; f < 11; ++f) *gp[f] += gv[f];
      } else {
#pragma unroll
        for (int f = 0; f < 11; ++f) *gp[f] = gv[f];
      }
      }  // any
      __syncwarp();
      // coalesced SH-gradient segment of this warp step
      float *gs = g + 11 * n + base * SB;
      const float *sk = s_chain + kChainThreads * SS;
      if (c.accumulate) {
        for (int e = lane; e < cnt * SB; e += kChainThreads) {
          const int r = e / SB;
          gs[e] += sk[r * SS + (e - r * SB)];
        }
      } else {
        for (int e = lane; e < cnt * SB; e += kChainThreads) {
          const int r = e / SB;
          gs[e] = sk[r * SS + (e - r * SB)];
        }
      }
      __syncwarp();
    }
  }
}

cudaError_t launch_chain_rule(const ChainArgs &c, int sh_bases, int grid, size_t smem, cudaStream_t s) {
  switch (sh_bases) {
    case 1: return launch_pdl(k_chain_rule_t<0>, dim3(grid), dim3(kChainThreads), smem, s, c);
    case 4: return launch_pdl(k_chain_rule_t<1>, dim3(grid), dim3(kChainThreads), smem, s, c);
    case 9: return launch_pdl(k_chain_rule_t<2>, dim3(grid), dim3(kChainThreads), smem, s, c);
    default: return launch_pdl(k_chain_rule_t<3>, dim3(grid), dim3(kChainThreads), smem, s, c);
  }
  return cudaGetLastError();
}

}  // namespace hgs
