// hgs_sort.cuh -- stable LSD radix sort (Onesweep: one read + one write per
// 8-bit digit pass, decoupled look-back for the cross-block digit prefix) and
// a decoupled look-back exclusive scan.  Written for sm_100a: 256-thread
// blocks, warp-level multi-split ranking with __match_any_sync, dynamic tile
// ids so the look-back only ever waits on blocks that are already resident.
//
// Used for the two sorts on the hot path (kernel table):
//  * depth sort  -- keys = float64 bit pattern of view z (positive, so the
//    unsigned order is the numeric order), values = Gaussian index in
//    ascending order, so stability breaks ties by index exactly like
//    lexsort((order, z)) (raster/project.py:187);
//  * tile sort   -- keys = tile id, values = depth rank; the pairs are emitted
//    in rank order, so stability keeps every tile list front-to-back
//    (raster/project.py:346-357 fills in sorted-slot order).
#pragma once

#include <cstdint>

#include "hgs_common.cuh"

namespace hgs {

constexpr int kSortThreads = 256;
#ifndef HGS_SORT_ITEMS
#define HGS_SORT_ITEMS 12
#endif
constexpr int kSortItems = HGS_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;  // 3072 keys per block
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
#ifndef HGS_LOOKBACK
#define HGS_LOOKBACK 8
#endif
constexpr int kLB = HGS_LOOKBACK;  // predecessors read per look-back round trip

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
  return (uint32_t)(key >> shift) & (kRadix - 1);
}

// Per-digit histograms of `n_digits` 8-bit digits (digit p = bits [8p, 8p+8)).
// hist: n_digits x 256 u32 (zeroed by the caller).  Grid-stride, persistent.
template <typename K>
__global__ void __launch_bounds__(256) k_radix_histogram(const K *__restrict__ keys, int64_t n, int n_digits,
                                                         uint32_t *__restrict__ hist) {
  __shared__ uint32_t sh[8 * kRadix];
  for (int i = threadIdx.x; i < n_digits * kRadix; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    K k = keys[i];
    for (int p = 0; p < n_digits; ++p) atomicAdd(&sh[p * kRadix + digit_of(k, p * kRadixBits)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_digits * kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Exclusive scan of each 256-bin histogram (one block per digit pass).
static __global__ void k_radix_offsets(const uint32_t *__restrict__ hist, uint32_t *__restrict__ offsets) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ uint32_t s[kRadix];
  const uint32_t *h = hist + blockIdx.x * kRadix;
  uint32_t *o = offsets + blockIdx.x * kRadix;
  int t = threadIdx.x;
  s[t] = h[t];
  __syncthreads();
  for (int d = 1; d < kRadix; d <<= 1) {
    uint32_t v = t >= d ? s[t - d] : 0;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  o[t] = s[t] - h[t];
}

// One Onesweep digit pass.  lookback: (#tiles x 256) u32 zeroed by the
// caller; tile_counter: u32 zeroed by the caller; digit_offsets: global
// exclusive offsets of this digit (k_radix_offsets).
#ifndef HGS_SORT_MINB32
#define HGS_SORT_MINB32 3  // CTAs per SM the passes are register-budgeted for (A/B: 1 -> 3: depth sort 0.199 -> 0.175 ms)
#endif
#ifndef HGS_SORT_MINB64
#define HGS_SORT_MINB64 3
#endif
// Device-driven passes (no host round trip, CUDA-graph capturable): with
// `plan` set, pass `pass` of the depth sort runs digit plan->sort_digit[pass]
// and exits at once if pass >= plan->sort_np (the digit is constant; the
// active passes are a prefix, so pass i always reads buffer i & 1); with
// `n_dev` set the key count is *n_dev (the tile sort's K), and the pass exits
// if the frame's status is set (pair capacity exceeded).  Blocks whose tile
// lies past the keys exit after taking their tile id.
struct SortDev {
  const unsigned *plan_np;             // &FrameState::sort_np (depth sort) or null
  const unsigned *plan_digit;          // &FrameState::sort_digit[0]
  int pass;
  const unsigned long long *n_dev;     // &FrameState::k_total (tile sort) or null
  const unsigned *status;              // &FrameState::status (with n_dev)
  // depth sort only (null otherwise): the last active pass also writes the
  // depth order (order[r] = Gaussian, rank_of[Gaussian] = r, or ~0 past M)
  // as it stores its output -- the separate rank-scatter pass is not needed
  uint32_t *rank_of = nullptr;
  uint32_t *order = nullptr;
  const uint32_t *m_count = nullptr;
};

template <typename K>
__global__ void __launch_bounds__(kSortThreads, sizeof(K) == 4 ? HGS_SORT_MINB32 : HGS_SORT_MINB64) k_onesweep(const K *__restrict__ keys_in,
                                                           const uint32_t *__restrict__ vals_in,
                                                           K *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
                                                           int64_t n, int shift,
                                                           const uint32_t *__restrict__ digit_offsets,
                                                           uint32_t *__restrict__ lookback,
                                                           uint32_t *__restrict__ tile_counter, SortDev dv) {
  // the depth sort's passes (dv.plan_np) do not trigger early: their
  // successors would wait on SM slots the preprocess beside them needs
  if (!HGS_DEPTH_SORT_TRIGGER && dv.plan_np == nullptr) pdl_launch_dependents();
  if (HGS_DEPTH_SORT_TRIGGER) pdl_launch_dependents();
  pdl_wait();
  bool emit_order = false;  // this pass writes the depth order (the last active one)
  if (dv.plan_np) {
    const unsigned np = *dv.plan_np;
    if (dv.order && np == 0u && dv.pass == 0) {
      // every digit constant: the input order is the sorted order
      const uint32_t m = *dv.m_count;
      for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = vals_in[r];
        dv.rank_of[g] = r < m ? (uint32_t)r : 0xffffffffu;
        dv.order[r] = g;
      }
      return;
    }
    if ((unsigned)dv.pass >= np) return;
    emit_order = dv.order != nullptr && (unsigned)dv.pass + 1u == np;
    const unsigned dg = dv.plan_digit[dv.pass];
    shift = (int)dg * kRadixBits;
    digit_offsets += dg * kRadix;
  }
  if (dv.n_dev) {
    if (*dv.status) return;
    n = (int64_t)*dv.n_dev;
  }
  if ((int64_t)blockIdx.x * kSortTile >= n) return;  // launched for a capacity, not for n
  constexpr int W = kSortThreads / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t warp_hist[W][kRadix];
  __shared__ uint32_t s_lstart[kRadix];
  __shared__ uint32_t s_gbase[kRadix];
  __shared__ K s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < W * kRadix; i += kSortThreads) (&warp_hist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t tile_base = (int64_t)tile * kSortTile;
  const int64_t warp_base = tile_base + (int64_t)warp * 32 * kSortItems;

  K key[kSortItems];
  uint32_t val[kSortItems];
  uint32_t rank[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    int64_t idx = warp_base + j * 32 + lane;
    bool ok = idx < n;
    key[j] = ok ? keys_in[idx] : (K)0;
    val[j] = ok ? vals_in[idx] : 0u;
  }
  // warp multi-split ranking in input order (j major, lane minor) -> stable
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    int64_t idx = warp_base + j * 32 + lane;
    bool ok = idx < n;
    uint32_t d = digit_of(key[j], shift);
    uint32_t tag = ok ? d : (uint32_t)(kRadix + lane);
    uint32_t peers = __match_any_sync(0xffffffffu, tag);
    uint32_t before = __popc(peers & lt);
    uint32_t base = ok ? warp_hist[warp][d] : 0u;
    __syncwarp();
    if (ok && before == 0) warp_hist[warp][d] = base + __popc(peers);
    __syncwarp();
    rank[j] = base + before;
  }
  __syncthreads();
  // per-digit: exclusive over warps, block count
  uint32_t count;
  {
    const int d = tid;  // kSortThreads == kRadix
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint32_t c = warp_hist[w][d];
      warp_hist[w][d] = run;
      run += c;
    }
    count = run;
    // publish aggregate / inclusive prefix, then decoupled look-back
    uint32_t *lb = lookback + (int64_t)tile * kRadix + d;
    if (tile == 0) {
      __stcg(lb, kFlagPrefix | count);
      s_gbase[d] = digit_offsets[d];
    } else {
      __stcg(lb, kFlagAgg | count);
      // look back kLB predecessors per round trip (independent loads), so a
      // tile that must sum many aggregates waits ~kLB x fewer L2 latencies
      uint32_t excl = 0;
      int64_t p = (int64_t)tile - 1;
      bool found = false;
      while (!found) {
        uint32_t v[kLB];
#pragma unroll
        for (int i = 0; i < kLB; ++i) v[i] = p - i >= 0 ? ld_volatile_u32(lookback + (p - i) * kRadix + d) : kFlagPrefix;
#pragma unroll
        for (int i = 0; i < kLB; ++i) {
          if (found) break;
          if ((v[i] & ~kValueMask) == 0) break;  // not yet published: re-poll from here
          excl += v[i] & kValueMask;
          --p;
          if (v[i] & kFlagPrefix) found = true;
        }
      }
      __stcg(lb, kFlagPrefix | (excl + count));
      s_gbase[d] = digit_offsets[d] + excl;
    }
  }
  // block-local digit starts (exclusive scan over 256 digits)
  s_lstart[tid] = count;
  __syncthreads();
  for (int off = 1; off < kRadix; off <<= 1) {
    uint32_t v = tid >= off ? s_lstart[tid - off] : 0u;
    __syncthreads();
    s_lstart[tid] += v;
    __syncthreads();
  }
  s_lstart[tid] -= count;
  __syncthreads();
  // scatter into shared memory in digit order
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    int64_t idx = warp_base + j * 32 + lane;
    if (idx < n) {
      uint32_t d = digit_of(key[j], shift);
      uint32_t pos = s_lstart[d] + warp_hist[warp][d] + rank[j];
      s_keys[pos] = key[j];
      s_vals[pos] = val[j];
    }
  }
  __syncthreads();
  const int64_t rem = n - tile_base;
  const int valid = rem < kSortTile ? (int)rem : kSortTile;
  const uint32_t m_emit = emit_order ? *dv.m_count : 0u;
  for (int p = tid; p < valid; p += kSortThreads) {
    K k = s_keys[p];
    uint32_t d = digit_of(k, shift);
    uint32_t o = s_gbase[d] + (uint32_t)p - s_lstart[d];
    keys_out[o] = k;
    const uint32_t g = s_vals[p];
    vals_out[o] = g;
    if (emit_order) {
      dv.rank_of[g] = o < m_emit ? o : 0xffffffffu;
      dv.order[o] = g;
    }
  }
}

// ---------------------------------------------------------------- scan
// Decoupled look-back exclusive scan of u32 counts into u64 offsets; the
// block handling the last tile writes the grand total to *total.
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kScanAgg = 1ull << 62;
constexpr unsigned long long kScanPrefix = 2ull << 62;
constexpr unsigned long long kScanMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long block_exclusive_scan_u64(unsigned long long v,
                                                                       unsigned long long *s_warp,
                                                                       unsigned long long &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = w;
  }
  __syncthreads();
  unsigned long long warp_prefix = warp ? s_warp[warp - 1] : 0ull;
  total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

// Look-back for tile `tile` with aggregate `agg`; returns the exclusive prefix.
// Called by one thread.
__device__ __forceinline__ unsigned long long scan_lookback(unsigned long long *lb, uint32_t tile,
                                                            unsigned long long agg) {
  if (tile == 0) {
    __stcg(lb, kScanPrefix | agg);
    return 0ull;
  }
  __stcg(lb + tile, kScanAgg | agg);
  unsigned long long excl = 0;
  int64_t p = (int64_t)tile - 1;
  bool found = false;
  while (!found) {  // kLB predecessors per round trip
    unsigned long long v[kLB];
#pragma unroll
    for (int i = 0; i < kLB; ++i) v[i] = p - i >= 0 ? ld_volatile_u64(lb + (p - i)) : kScanPrefix;
#pragma unroll
    for (int i = 0; i < kLB; ++i) {
      if (found) break;
      if ((v[i] & ~kScanMask) == 0) break;
      excl += v[i] & kScanMask;
      --p;
      if (v[i] & kScanPrefix) found = true;
    }
  }
  __stcg(lb + tile, kScanPrefix | (excl + agg));
  return excl;
}

}  // namespace hgs
