// hgs_loss.cu -- the frequency-decoupled loss stack of one training view
// (include/hgs_train.h; reference freq/dwt.py, freq/ssim.py).
//
// HBM-bound image work, so the design is about passes, not flops:
//  k_loss_moments : one pass over (rendered, gt).  Per 32 x 8 tile and channel
//                   it stages the haloed patch in shared memory, runs the
//                   separable 11-tap window over the five moment images
//                   (x, y, x^2, y^2, xy; ssim.py:31-36) and writes the three
//                   SSIM partial maps the gradient needs (ssim.py:60-72), plus
//                   per-block float64 sums of the SSIM map, |r - g| and the
//                   Haar band energies of (r - g).
//  k_loss_grads   : one pass over the partial maps: blurs them (the adjoint of
//                   the window is the window) and writes the KG = 3 upstream
//                   gradient stack (colour, lambda_low * low, lambda_high *
//                   high) that hgs_backward consumes; the Haar adjoint of a
//                   2 x 2 block is closed form.
//  k_loss_reduce  : one block sums the per-block partials in a fixed order.
// Algorithmic traffic per pixel and channel: 8 B in + 12 B out (moments),
// 20 B in + 12 B out (grads): 52 B / (pixel, channel).
#include <algorithm>
#include <cmath>

#include "hgs_kernels.cuh"
#include "hgs_nvtx.h"
#include "../../include/hgs_train.h"

namespace hgs {

namespace {

constexpr int kLTX = 32, kLTY = 32;      // output tile (tall: the 10-row halo is amortised over 32 rows)
constexpr int kHalo = 5;                  // 11-tap window
constexpr int kPW = kLTX + 2 * kHalo;     // 42
constexpr int kPH = kLTY + 2 * kHalo;     // 42
constexpr int kLThreads = 256;            // 32 x 8 threads, 4 output rows each
constexpr int kRowsPer = kLTY / (kLThreads / kLTX);
constexpr int kNSums = 4;                 // ssim, l1, ll^2, detail^2

struct LossArgs {
  int H, W, C;
  const float *r, *g;
  float *mA, *mB, *mC;   // SSIM partial maps (H, W, C)
  double *part;          // (blocks, kNSums)
  double lam, lam_low, lam_high;
  float *out;            // (3, H, W, C) or null
  double *losses;
  float win[11];         // normalised 11-tap Gaussian window, sigma 1.5 (ssim.py:19-24)
};

constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;  // ssim.py:15-16

__device__ __forceinline__ double block_sum(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kLThreads / 32; ++i) s += red[i];  // fixed order
  return s;
}

// Load the haloed patch of one channel of `src` (zero outside the image:
// the window is zero padded, ssim.py:26-29).
__device__ __forceinline__ void load_patch(const float *src, int H, int W, int C, int c, int x0, int y0,
                                           float (*p)[kPW]) {
  for (int k = threadIdx.x; k < kPH * kPW; k += kLThreads) {
    const int py = k / kPW, px = k % kPW;
    const int y = y0 - kHalo + py, x = x0 - kHalo + px;
    p[py][px] = (y >= 0 && y < H && x >= 0 && x < W) ? __ldg(src + ((size_t)y * W + x) * C + c) : 0.f;
  }
}

__global__ void __launch_bounds__(kLThreads) k_loss_moments(LossArgs a) {
  __shared__ float sx[kPH][kPW], sy[kPH][kPW];
  __shared__ float h[5][kPH][kLTX];
  __shared__ double red[kLThreads / 32];
  const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY;
  const int tx = threadIdx.x % kLTX, ty0 = threadIdx.x / kLTX;
  const int ix = x0 + tx;
  const int H = a.H, W = a.W, C = a.C;
  double s_ssim = 0.0, s_l1 = 0.0, s_ll = 0.0, s_det = 0.0;
  for (int c = 0; c < C; ++c) {
    __syncthreads();
    load_patch(a.r, H, W, C, c, x0, y0, sx);
    load_patch(a.g, H, W, C, c, x0, y0, sy);
    __syncthreads();
    // horizontal pass over the 18 patch rows
    for (int k = threadIdx.x; k < kPH * kLTX; k += kLThreads) {
      const int py = k / kLTX, px = k % kLTX;
      float mx = 0.f, my = 0.f, mxx = 0.f, myy = 0.f, mxy = 0.f;
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const float x = sx[py][px + t], y = sy[py][px + t], w = a.win[t];
        mx = fmaf(w, x, mx);
        my = fmaf(w, y, my);
        mxx = fmaf(w, x * x, mxx);
        myy = fmaf(w, y * y, myy);
        mxy = fmaf(w, x * y, mxy);
      }
      h[0][py][px] = mx; h[1][py][px] = my; h[2][py][px] = mxx; h[3][py][px] = myy; h[4][py][px] = mxy;
    }
    __syncthreads();
    for (int rr = 0; rr < kRowsPer; ++rr) {
    const int ty = ty0 + rr * (kLThreads / kLTX), iy = y0 + ty;
    if (ix < W && iy < H) {
      float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const float w = a.win[t];
#pragma unroll
        for (int q = 0; q < 5; ++q) m[q] = fmaf(w, h[q][ty + t][tx], m[q]);
      }
      const float mu_x = m[0], mu_y = m[1];
      const float sig_x = m[2] - mu_x * mu_x, sig_y = m[3] - mu_y * mu_y, sig_xy = m[4] - mu_x * mu_y;
      const float a1 = 2.f * mu_x * mu_y + kC1, a2 = 2.f * sig_xy + kC2;
      const float b1 = mu_x * mu_x + mu_y * mu_y + kC1, b2 = sig_x + sig_y + kC2;
      s_ssim += (double)((a1 * a2) / (b1 * b2));
      // partials of the SSIM map w.r.t. the local moments (ssim.py:60-66)
      const float d_mu_x = 2.f * (mu_y * a2 * b1 - mu_x * a1 * a2) / (b1 * b1 * b2);
      const float d_sig_x = -a1 * a2 / (b1 * b2 * b2);
      const float d_sig_xy = 2.f * a1 / (b1 * b2);
      const size_t o = ((size_t)iy * W + ix) * C + c;
      a.mA[o] = d_mu_x - 2.f * mu_x * d_sig_x - mu_y * d_sig_xy;
      a.mB[o] = d_sig_x;
      a.mC[o] = d_sig_xy;
      const float xv = sx[ty + kHalo][tx + kHalo], yv = sy[ty + kHalo][tx + kHalo];
      s_l1 += (double)fabsf(xv - yv);
      // Haar band energies of (r - g) for the 2x2 block whose top-left pixel
      // this is; the padded row / column replicates the edge (dwt.py:32-38)
      if (!(ix & 1) && !(iy & 1)) {
        const int px1 = (ix + 1 < W) ? 1 : 0, py1 = (iy + 1 < H) ? 1 : 0;
        const int bx = tx + kHalo, by = ty + kHalo;
        const float d00 = xv - yv;
        const float d01 = sx[by][bx + px1] - sy[by][bx + px1];
        const float d10 = sx[by + py1][bx] - sy[by + py1][bx];
        const float d11 = sx[by + py1][bx + px1] - sy[by + py1][bx + px1];
        const float ll = 0.5f * ((d00 + d10) + (d01 + d11));
        const float hl = 0.5f * ((d00 + d10) - (d01 + d11));
        const float lh = 0.5f * ((d00 - d10) + (d01 - d11));
        const float hh = 0.5f * ((d00 - d10) - (d01 - d11));
        s_ll += (double)(ll * ll);
        s_det += (double)(lh * lh) + (double)(hl * hl) + (double)(hh * hh);
      }
    }
    }  // rows
  }
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  const double t0 = block_sum(s_ssim, red), t1 = block_sum(s_l1, red);
  const double t2 = block_sum(s_ll, red), t3 = block_sum(s_det, red);
  if (threadIdx.x == 0) {
    double *p = a.part + (size_t)blk * kNSums;
    p[0] = t0; p[1] = t1; p[2] = t2; p[3] = t3;
  }
}

__global__ void __launch_bounds__(kLThreads) k_loss_grads(LossArgs a) {
  __shared__ float pa[kPH][kPW], pb[kPH][kPW], pc[kPH][kPW];
  __shared__ float h[3][kPH][kLTX];
  const int x0 = blockIdx.x * kLTX, y0 = blockIdx.y * kLTY;
  const int tx = threadIdx.x % kLTX, ty0 = threadIdx.x / kLTX;
  const int ix = x0 + tx;
  const int H = a.H, W = a.W, C = a.C;
  const size_t plane = (size_t)H * W * C;
  const float inv_size = (float)(1.0 / ((double)H * W * C));
  const int h2 = (H + 1) / 2, w2 = (W + 1) / 2;
  const float inv_bsize = (float)(1.0 / ((double)h2 * w2 * C));
  const float lam = (float)a.lam, lam_low = (float)a.lam_low, lam_high = (float)a.lam_high;
  for (int c = 0; c < C; ++c) {
    __syncthreads();
    load_patch(a.mA, H, W, C, c, x0, y0, pa);
    load_patch(a.mB, H, W, C, c, x0, y0, pb);
    load_patch(a.mC, H, W, C, c, x0, y0, pc);
    __syncthreads();
    for (int k = threadIdx.x; k < kPH * kLTX; k += kLThreads) {
      const int py = k / kLTX, px = k % kLTX;
      float sa = 0.f, sb = 0.f, sc = 0.f;
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const float w = a.win[t];
        sa = fmaf(w, pa[py][px + t], sa);
        sb = fmaf(w, pb[py][px + t], sb);
        sc = fmaf(w, pc[py][px + t], sc);
      }
      h[0][py][px] = sa; h[1][py][px] = sb; h[2][py][px] = sc;
    }
    __syncthreads();
    for (int rr = 0; rr < kRowsPer; ++rr) {
    const int ty = ty0 + rr * (kLThreads / kLTX), iy = y0 + ty;
    if (ix >= W || iy >= H) continue;
    // 2x2 Haar block of this pixel; which padded positions fold onto it
    const int bx0 = ix & ~1, by0 = iy & ~1;
    const int ox = ix & 1, oy = iy & 1;
    const int px1 = (bx0 + 1 < W) ? 1 : 0, py1 = (by0 + 1 < H) ? 1 : 0;
    // row offsets a' (and column offsets b') whose padded pixel maps here
    const int na = (oy == 0 && !py1) ? 2 : 1, nb = (ox == 0 && !px1) ? 2 : 1;
    float ba = 0.f, bb = 0.f, bc = 0.f;
#pragma unroll
    for (int t = 0; t < 11; ++t) {
      const float w = a.win[t];
      ba = fmaf(w, h[0][ty + t][tx], ba);
      bb = fmaf(w, h[1][ty + t][tx], bb);
      bc = fmaf(w, h[2][ty + t][tx], bc);
    }
    const size_t o = ((size_t)iy * W + ix) * C + c;
    const float x = __ldg(a.r + o), y = __ldg(a.g + o);
    // d(mean SSIM)/dx (ssim.py:71-74)
    const float g_ssim = (ba + 2.f * x * bb + y * bc) * inv_size;
    const float dif = x - y;
    const float sgn = (float)((dif > 0.f) - (dif < 0.f));
    float g_col = (1.f - lam) * sgn * inv_size;  // ssim.py:92
    if (lam > 0.f) g_col -= lam * 0.5f * g_ssim;  // ssim.py:93-94
    // Haar adjoint of the band residuals of this pixel's block (dwt.py:122-137)
    auto D = [&](int yy, int xx) {
      const size_t q = ((size_t)yy * W + xx) * C + c;
      return __ldg(a.r + q) - __ldg(a.g + q);
    };
    const float d00 = D(by0, bx0), d01 = D(by0, bx0 + px1);
    const float d10 = D(by0 + py1, bx0), d11 = D(by0 + py1, bx0 + px1);
    const float ll = 0.5f * ((d00 + d10) + (d01 + d11));
    const float hl = 0.5f * ((d00 + d10) - (d01 + d11));
    const float lh = 0.5f * ((d00 - d10) + (d01 - d11));
    const float hh = 0.5f * ((d00 - d10) - (d01 - d11));
    const float dll = 2.f * ll * inv_bsize, dlh = 2.f * lh * inv_bsize;
    const float dhl = 2.f * hl * inv_bsize, dhh = 2.f * hh * inv_bsize;
    float g_low = 0.f, g_high = 0.f;
    for (int ia = 0; ia < na; ++ia) {
      const float sa_ = (oy + ia) ? -1.f : 1.f;  // row offset a' = oy (+1 for the fold)
      for (int ib = 0; ib < nb; ++ib) {
        const float sb_ = (ox + ib) ? -1.f : 1.f;
        g_low += 0.5f * dll;
        g_high += 0.5f * (sa_ * dlh + sb_ * dhl + sa_ * sb_ * dhh);
      }
    }
    if (a.out) {
      a.out[o] = g_col;
      a.out[plane + o] = lam_low * g_low;
      a.out[2 * plane + o] = lam_high * g_high;
    }
    }  // rows
  }
}

__global__ void __launch_bounds__(1024) k_loss_reduce(const double *part, int nblk, int H, int W, int C, double lam,
                                                     double *losses) {
  __shared__ double red[32][kNSums];
  double s[kNSums] = {0.0, 0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nblk; b += blockDim.x)
    for (int q = 0; q < kNSums; ++q) s[q] += part[(size_t)b * kNSums + q];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kNSums; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
    if (l == 0) red[w][q] = s[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[kNSums] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
      for (int q = 0; q < kNSums; ++q) t[q] += red[i][q];
    const double size = (double)H * W * C;
    const double bsize = (double)((H + 1) / 2) * ((W + 1) / 2) * C;
    const double l1 = t[1] / size, ssim = t[0] / size;
    losses[HGS_LOSS_L1] = l1;
    losses[HGS_LOSS_SSIM] = ssim;
    losses[HGS_LOSS_LOW] = t[2] / bsize;
    losses[HGS_LOSS_HIGH] = t[3] / bsize;
    losses[HGS_LOSS_COLOR] = lam == 0.0 ? l1 : (1.0 - lam) * l1 + lam * (1.0 - ssim) / 2.0;
  }
}

// ------------------------------------------------------------ Haar transform
__global__ void k_dwt(int H, int W, int C, const float *img, float *ll, float *lh, float *hl, float *hh) {
  const int w2 = (W + 1) / 2, h2 = (H + 1) / 2;
  const int64_t total = (int64_t)h2 * w2 * C;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(k % C);
    const int64_t bk = k / C;
    const int bx = (int)(bk % w2), by = (int)(bk / w2);
    const int x0 = 2 * bx, y0 = 2 * by;
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);  // edge replication (dwt.py:32-38)
    const float i00 = img[((size_t)y0 * W + x0) * C + c], i01 = img[((size_t)y0 * W + x1) * C + c];
    const float i10 = img[((size_t)y1 * W + x0) * C + c], i11 = img[((size_t)y1 * W + x1) * C + c];
    // rows first (lo_r / hi_r), then columns (dwt.py:66-73)
    const float s = 0.70710678118654752f;
    const float lo0 = (i00 + i10) * s, lo1 = (i01 + i11) * s;
    const float hi0 = (i00 - i10) * s, hi1 = (i01 - i11) * s;
    ll[k] = (lo0 + lo1) * s;
    hl[k] = (lo0 - lo1) * s;
    lh[k] = (hi0 + hi1) * s;
    hh[k] = (hi0 - hi1) * s;
  }
}

__global__ void k_idwt(int H, int W, int C, const float *ll, const float *lh, const float *hl, const float *hh,
                       int adjoint, float *img) {
  const int w2 = (W + 1) / 2;
  const int64_t total = (int64_t)H * W * C;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(k % C);
    const int64_t p = k / C;
    const int x = (int)(p % W), y = (int)(p / W);
    const int bx = x >> 1, by = y >> 1, ox = x & 1, oy = y & 1;
    const size_t b = ((size_t)by * w2 + bx) * C + c;
    const float s = 0.70710678118654752f;
    const float LL = ll[b], LH = lh[b], HL = hl[b], HH = hh[b];
    // dwt.py:82-90: out[2i+a, 2j+b] from (lo_r, lo_r2, hi_r, hi_r2)
    auto pix = [&](int a_, int b_) {
      const float lo = b_ ? (LL - HL) * s : (LL + HL) * s;
      const float hi = b_ ? (LH - HH) * s : (LH + HH) * s;
      return a_ ? (lo - hi) * s : (lo + hi) * s;
    };
    float v = pix(oy, ox);
    if (adjoint) {  // fold the padded row / column onto the edge (dwt.py:41-52)
      const bool fy = (H & 1) && y == H - 1, fx = (W & 1) && x == W - 1;
      if (fy) v += pix(1, ox);
      if (fx) v += pix(oy, 1);
      if (fy && fx) v += pix(1, 1);
    }
    img[k] = v;
  }
}

}  // namespace

}  // namespace hgs

using namespace hgs;

#define HGS_CUDA_OK(x)                          \
  do {                                          \
    if ((x) != cudaSuccess) return HGS_ERR_CUDA; \
  } while (0)

namespace {

size_t loss_blocks(int H, int W) { return (size_t)((W + kLTX - 1) / kLTX) * ((H + kLTY - 1) / kLTY); }

void make_window(float *wf) {
  double w[11], s = 0.0;
  for (int i = 0; i < 11; ++i) {
    const double x = i - 5;
    w[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));  // ssim.py:19-24
    s += w[i];
  }
  for (int i = 0; i < 11; ++i) wf[i] = (float)(w[i] / s);
}

}  // namespace

extern "C" {

size_t hgs_loss_scratch_bytes(int32_t height, int32_t width, int32_t channels) {
  if (height <= 0 || width <= 0 || channels <= 0) return 0;
  const size_t map = (((size_t)height * width * channels * 4) + 255) & ~(size_t)255;
  return 3 * map + loss_blocks(height, width) * kNSums * sizeof(double);
}

int hgs_image_losses(int32_t height, int32_t width, int32_t channels, const float *rendered, const float *gt,
                     const hgs_loss_weights *weights, double *losses, float *pixel_grads, void *scratch,
                     size_t scratch_bytes, void *stream) {
  NvtxScope nv("hgs_image_losses");
  if (height <= 0 || width <= 0 || channels <= 0 || !rendered || !gt || !weights || !losses) return HGS_ERR_CONFIG;
  if (weights->lam < 0.0 || weights->lam > 1.0 || weights->lambda_low < 0.0 || weights->lambda_high < 0.0)
    return HGS_ERR_CONFIG;
  if (!scratch || scratch_bytes < hgs_loss_scratch_bytes(height, width, channels)) return HGS_ERR_CONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t map = (((size_t)height * width * channels * 4) + 255) & ~(size_t)255;
  char *base = static_cast<char *>(scratch);
  LossArgs a;
  a.H = height; a.W = width; a.C = channels;
  a.r = rendered; a.g = gt;
  a.mA = reinterpret_cast<float *>(base);
  a.mB = reinterpret_cast<float *>(base + map);
  a.mC = reinterpret_cast<float *>(base + 2 * map);
  a.part = reinterpret_cast<double *>(base + 3 * map);
  a.lam = weights->lam; a.lam_low = weights->lambda_low; a.lam_high = weights->lambda_high;
  a.out = pixel_grads;
  a.losses = losses;
  make_window(a.win);
  const dim3 grid((width + kLTX - 1) / kLTX, (height + kLTY - 1) / kLTY);
  k_loss_moments<<<grid, kLThreads, 0, s>>>(a);
  HGS_CUDA_OK(cudaGetLastError());
  k_loss_reduce<<<1, 1024, 0, s>>>(a.part, (int)loss_blocks(height, width), height, width, channels, a.lam, losses);
  HGS_CUDA_OK(cudaGetLastError());
  if (pixel_grads) {
    k_loss_grads<<<grid, kLThreads, 0, s>>>(a);
    HGS_CUDA_OK(cudaGetLastError());
  }
  return HGS_OK;
}

int hgs_dwt_level1(int32_t height, int32_t width, int32_t channels, const float *image, float *ll, float *lh,
                   float *hl, float *hh, void *stream) {
  NvtxScope nv("hgs_dwt_level1");
  if (height <= 0 || width <= 0 || channels <= 0 || !image || !ll || !lh || !hl || !hh) return HGS_ERR_CONFIG;
  const int64_t total = (int64_t)((height + 1) / 2) * ((width + 1) / 2) * channels;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_dwt<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(height, width, channels, image, ll, lh, hl, hh);
  HGS_CUDA_OK(cudaGetLastError());
  return HGS_OK;
}

int hgs_dwt_inverse(int32_t height, int32_t width, int32_t channels, const float *ll, const float *lh,
                    const float *hl, const float *hh, int32_t adjoint, float *image, void *stream) {
  NvtxScope nv("hgs_dwt_inverse");
  if (height <= 0 || width <= 0 || channels <= 0 || !image || !ll || !lh || !hl || !hh) return HGS_ERR_CONFIG;
  const int64_t total = (int64_t)height * width * channels;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_idwt<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(height, width, channels, ll, lh, hl, hh, adjoint,
                                                                 image);
  HGS_CUDA_OK(cudaGetLastError());
  return HGS_OK;
}

}  // extern "C"
