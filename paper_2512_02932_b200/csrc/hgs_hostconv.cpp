// hgs_hostconv.cpp -- host-side float64 <-> float32 conversion for the
// reference-facing numpy API (raster.render / grad.backward take and return
// float64 arrays; the kernels read and write float32).
//
// The conversions are host-DRAM bound.  A plain converting copy (torch's
// copy_, numpy's astype) reads the destination's cache lines before writing
// them (write-allocate), so widening n floats costs 4n read + 8n RFO + 8n
// write bytes.  Here the destination is written with non-temporal (streaming)
// stores -- 4n + 8n -- on all requested threads (OpenMP, static split on
// 64-byte boundaries of the destination).
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <string.h>

#include "../../include/hgs.h"

namespace {

template <bool NT>
__attribute__((target("avx2"))) void widen_avx2(const float *__restrict__ s, double *__restrict__ d, int64_t n) {
  int64_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31u)) {
    d[i] = (double)s[i];
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m256 v = _mm256_loadu_ps(s + i);
    const __m256d a = _mm256_cvtps_pd(_mm256_castps256_ps128(v)), b = _mm256_cvtps_pd(_mm256_extractf128_ps(v, 1));
    if (NT) {
      _mm256_stream_pd(d + i, a);
      _mm256_stream_pd(d + i + 4, b);
    } else {
      _mm256_store_pd(d + i, a);
      _mm256_store_pd(d + i + 4, b);
    }
  }
  for (; i < n; ++i) d[i] = (double)s[i];
}

template <bool NT>
__attribute__((target("avx2"))) void narrow_avx2(const double *__restrict__ s, float *__restrict__ d, int64_t n) {
  int64_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31u)) {
    d[i] = (float)s[i];
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m128 lo = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i));
    const __m128 hi = _mm256_cvtpd_ps(_mm256_loadu_pd(s + i + 4));
    const __m256 v = _mm256_insertf128_ps(_mm256_castps128_ps256(lo), hi, 1);
    if (NT) _mm256_stream_ps(d + i, v);
    else _mm256_store_ps(d + i, v);
  }
  for (; i < n; ++i) d[i] = (float)s[i];
}

template <bool NT>
__attribute__((target("avx2"))) void copy_avx2(const uint8_t *__restrict__ s, uint8_t *__restrict__ d, int64_t n) {
  int64_t i = 0;
  const int64_t head = (int64_t)((32u - (reinterpret_cast<uintptr_t>(d) & 31u)) & 31u);
  if (head) {
    memcpy(d, s, (size_t)(head < n ? head : n));
    i = head;
  }
  for (; i + 32 <= n; i += 32) {
    const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(s + i));
    if (NT) _mm256_stream_si256(reinterpret_cast<__m256i *>(d + i), v);
    else _mm256_store_si256(reinterpret_cast<__m256i *>(d + i), v);
  }
  if (i < n) memcpy(d + i, s + i, (size_t)(n - i));
}

template <class S, class D>
void convert_scalar(const S *s, D *d, int64_t n) {
  for (int64_t i = 0; i < n; ++i) d[i] = (D)s[i];
}

bool has_avx2() {
  static const int v = __builtin_cpu_supports("avx2") ? 1 : 0;
  return v != 0;
}

// [b, e) of part t of nt, on 16-element (64-byte float64 / float32 x 16)
// boundaries so two threads never share a destination cache line
inline void part(int64_t n, int t, int nt, int64_t &b, int64_t &e) {
  const int64_t blocks = (n + 15) / 16;
  b = blocks * t / nt * 16;
  e = blocks * (t + 1) / nt * 16;
  if (b > n) b = n;
  if (e > n) e = n;
}

template <class F>
void run(int64_t n, int threads, F &&body, bool fence = true) {
  if (threads <= 0) threads = omp_get_max_threads();
  const int64_t min_per = 1 << 16;  // elements per thread below which threads do not pay
  if (n / min_per < threads) threads = (int)(n / min_per > 0 ? n / min_per : 1);
  if (threads <= 1) {
    body((int64_t)0, n);
  } else {
#pragma omp parallel num_threads(threads)
    {
      int64_t b, e;
      part(n, omp_get_thread_num(), omp_get_num_threads(), b, e);
      if (e > b) body(b, e);
      if (fence) _mm_sfence();  // this thread's streaming stores are globally visible before the join
    }
  }
  if (fence) _mm_sfence();
}

}  // namespace

extern "C" int hgs_host_widen(const float *src, double *dst, int64_t n, int threads) {
  if (n < 0 || (n > 0 && (!src || !dst))) return HGS_ERR_CONFIG;
  const bool v = has_avx2();
  run(n, threads, [&](int64_t b, int64_t e) {
    if (v) widen_avx2<true>(src + b, dst + b, e - b);
    else convert_scalar(src + b, dst + b, e - b);
  });
  return HGS_OK;
}

extern "C" int hgs_host_narrow(const double *src, float *dst, int64_t n, int threads) {
  if (n < 0 || (n > 0 && (!src || !dst))) return HGS_ERR_CONFIG;
  const bool v = has_avx2();
  run(n, threads, [&](int64_t b, int64_t e) {
    if (v) narrow_avx2<true>(src + b, dst + b, e - b);
    else convert_scalar(src + b, dst + b, e - b);
  });
  return HGS_OK;
}

extern "C" int hgs_host_copy(const void *src, void *dst, int64_t bytes, int threads) {
  if (bytes < 0 || (bytes > 0 && (!src || !dst))) return HGS_ERR_CONFIG;
  const bool v = has_avx2();
  const uint8_t *s = static_cast<const uint8_t *>(src);
  uint8_t *d = static_cast<uint8_t *>(dst);
  // parts on 64-byte multiples of the 16-"element" split: elements of 4 bytes
  run(bytes / 4, threads, [&](int64_t b, int64_t e) {
    const int64_t lo = b * 4, hi = (e == bytes / 4) ? bytes : e * 4;
    if (v) copy_avx2<true>(s + lo, d + lo, hi - lo);
    else memcpy(d + lo, s + lo, (size_t)(hi - lo));
  });
  return HGS_OK;
}

// ---------------------------------------------------------------------------
// Scene fingerprint sums (raster.scene_fingerprint: the sums of the float64
// centre / opacity / log-scale arrays, render.py:67-70).  Deterministic: the
// array is cut into fixed kSumBlock-element blocks at absolute positions,
// each block summed in one fixed order (8 lanes, then a fixed reduction);
// the caller adds the block sums in order.  The copying variant produces
// the same block sums while it copies (the upload's staging pass), so a
// render's fingerprint costs no extra read of the scene.
namespace {

constexpr int64_t kSumBlock = 32768;

template <bool COPY>
__attribute__((target("avx2"))) double block_pass(const double *__restrict__ s, double *__restrict__ d, int64_t n) {
  __m256d a0 = _mm256_setzero_pd(), a1 = _mm256_setzero_pd();
  int64_t i = 0;
  // the copy goes out with streaming stores when the destination allows
  // (the staging is read by the DMA, not by the CPU); same sums either way
  const bool nt = COPY && (reinterpret_cast<uintptr_t>(d) & 31u) == 0;
  for (; i + 8 <= n; i += 8) {
    const __m256d x0 = _mm256_loadu_pd(s + i), x1 = _mm256_loadu_pd(s + i + 4);
    a0 = _mm256_add_pd(a0, x0);
    a1 = _mm256_add_pd(a1, x1);
    if (COPY) {
      if (nt) {
        _mm256_stream_pd(d + i, x0);
        _mm256_stream_pd(d + i + 4, x1);
      } else {
        _mm256_storeu_pd(d + i, x0);
        _mm256_storeu_pd(d + i + 4, x1);
      }
    }
  }
  alignas(32) double l0[4], l1[4];
  _mm256_store_pd(l0, a0);
  _mm256_store_pd(l1, a1);
  double t = ((l0[0] + l0[1]) + (l0[2] + l0[3])) + ((l1[0] + l1[1]) + (l1[2] + l1[3]));
  for (; i < n; ++i) {
    t += s[i];
    if (COPY) d[i] = s[i];
  }
  return t;
}

template <bool COPY>
double block_pass_scalar(const double *s, double *d, int64_t n) {
  double l0[4] = {0, 0, 0, 0}, l1[4] = {0, 0, 0, 0};
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    for (int k = 0; k < 4; ++k) {
      l0[k] += s[i + k];
      l1[k] += s[i + 4 + k];
      if (COPY) {
        d[i + k] = s[i + k];
        d[i + 4 + k] = s[i + 4 + k];
      }
    }
  }
  double t = ((l0[0] + l0[1]) + (l0[2] + l0[3])) + ((l1[0] + l1[1]) + (l1[2] + l1[3]));
  for (; i < n; ++i) {
    t += s[i];
    if (COPY) d[i] = s[i];
  }
  return t;
}

template <bool COPY>
int block_sums(const double *src, double *dst, int64_t n, double *sums, int threads) {
  if (n < 0 || (n > 0 && (!src || !sums || (COPY && !dst)))) return HGS_ERR_CONFIG;
  const int64_t nb = (n + kSumBlock - 1) / kSumBlock;
  const bool v = has_avx2();
  if (threads <= 0) threads = omp_get_max_threads();
  if (nb < threads) threads = (int)(nb > 0 ? nb : 1);
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = b * kSumBlock, len = (lo + kSumBlock <= n ? kSumBlock : n - lo);
    sums[b] = v ? block_pass<COPY>(src + lo, COPY ? dst + lo : nullptr, len)
                : block_pass_scalar<COPY>(src + lo, COPY ? dst + lo : nullptr, len);
    if (COPY) _mm_sfence();
  }
  return HGS_OK;
}

}  // namespace

extern "C" int64_t hgs_host_sum_block(void) { return kSumBlock; }

extern "C" int hgs_host_block_sums(const double *src, int64_t n, double *sums, int threads) {
  return block_sums<false>(src, nullptr, n, sums, threads);
}

extern "C" int hgs_host_copy_block_sums(const double *src, double *dst, int64_t n, double *sums, int threads) {
  return block_sums<true>(src, dst, n, sums, threads);
}

// ---------------------------------------------------------------------------
// Narrowing with the finiteness check the reference applies to its float64
// upstream gradients (grad/backward.py: non-finite -> IntegrityError) in the
// same pass: the check reads the float64 values (a finite 1e300 stays
// finite, although it overflows float32), no second read, no device sync.
namespace {

__attribute__((target("avx2"))) int64_t narrow_count_avx2(const double *__restrict__ s, float *__restrict__ d, int64_t n) {
  const __m256d inf = _mm256_set1_pd(__builtin_inf());
  const __m256d absmask = _mm256_castsi256_pd(_mm256_set1_epi64x(0x7fffffffffffffffll));
  int64_t bad = 0, i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31u)) {
    bad += !(__builtin_fabs(s[i]) < __builtin_inf());
    d[i] = (float)s[i];
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m256d a = _mm256_loadu_pd(s + i), b = _mm256_loadu_pd(s + i + 4);
    // |x| < inf is false for inf and NaN
    const int ma = _mm256_movemask_pd(_mm256_cmp_pd(_mm256_and_pd(a, absmask), inf, _CMP_LT_OQ));
    const int mb = _mm256_movemask_pd(_mm256_cmp_pd(_mm256_and_pd(b, absmask), inf, _CMP_LT_OQ));
    bad += 8 - __builtin_popcount((unsigned)(ma | (mb << 4)));
    const __m256 v = _mm256_insertf128_ps(_mm256_castps128_ps256(_mm256_cvtpd_ps(a)), _mm256_cvtpd_ps(b), 1);
    _mm256_stream_ps(d + i, v);
  }
  for (; i < n; ++i) {
    bad += !(__builtin_fabs(s[i]) < __builtin_inf());
    d[i] = (float)s[i];
  }
  return bad;
}

int64_t narrow_count_scalar(const double *s, float *d, int64_t n) {
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    bad += !(__builtin_fabs(s[i]) < __builtin_inf());
    d[i] = (float)s[i];
  }
  return bad;
}

}  // namespace

extern "C" int hgs_host_narrow_count(const double *src, float *dst, int64_t n, int threads, int64_t *nonfinite) {
  if (n < 0 || !nonfinite || (n > 0 && (!src || !dst))) return HGS_ERR_CONFIG;
  const bool v = has_avx2();
  int64_t total = 0;
  if (threads <= 0) threads = omp_get_max_threads();
  const int64_t min_per = 1 << 16;
  if (n / min_per < threads) threads = (int)(n / min_per > 0 ? n / min_per : 1);
#pragma omp parallel num_threads(threads) reduction(+ : total)
  {
    int64_t b, e;
    part(n, omp_get_thread_num(), omp_get_num_threads(), b, e);
    if (e > b) total += v ? narrow_count_avx2(src + b, dst + b, e - b) : narrow_count_scalar(src + b, dst + b, e - b);
    _mm_sfence();
  }
  *nonfinite = total;
  return HGS_OK;
}

