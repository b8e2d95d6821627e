// hgs_api.cu -- the C ABI declared in include/hgs.h: frame-buffer layout,
// launch orchestration, error mapping.  No device allocation happens here;
// every buffer is carved out of caller memory.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "hgs_kernels.cuh"
#include "hgs_nvtx.h"

namespace hgs {

namespace {

constexpr int kMaxGrid = 148 * 8;

#ifndef HGS_TILE_COUNTS_AUX
#define HGS_TILE_COUNTS_AUX 1  // 0: k_tile_counts on the main stream after the join (A/B: 268.4 vs 269.5 it/s)
#endif
// The depth sort's chain (plan, passes, rank scatter) is launched with
// programmatic dependence but without early triggers (HGS_DEPTH_SORT_TRIGGER
// 0): each kernel is set up while its predecessor runs and starts when it
// completes, and no waiting CTA holds an SM slot the preprocess beside the
// chain needs (A/B, stage 1: plain launches 0.354 ms, PDL with early
// triggers 0.368, PDL without them 0.345).  The binning chain, the fixups
// and the chain rule trigger early (binning 0.145 -> 0.131 ms).
#ifndef HGS_DEPTH_SORT_PDL
#define HGS_DEPTH_SORT_PDL 1
#endif
constexpr bool kDepthSortPdl = HGS_DEPTH_SORT_PDL != 0;
#ifndef HGS_FUSE_RANK_SCATTER
#define HGS_FUSE_RANK_SCATTER 0  // 1: the depth order written by the last active depth-sort pass (A/B: neutral, 278.3 vs 278.0 it/s)
#endif
#ifndef HGS_TILE_COUNTS_PDL
#define HGS_TILE_COUNTS_PDL 1
#endif
#ifndef HGS_SORT_ON_AUX
#define HGS_SORT_ON_AUX 0  // 1 (+ HGS_PRE_CTAS=64, HGS_AUX_PRIORITY=-5): stage 1 0.359 -> 0.353 ms, neutral end to end
#endif

struct Layout {
  size_t state, hist_d, off_d, hist_p, off_p, keys_a, keys_b, vals_a, vals_b, rank, order, counts, keep, kept, lb_sort, lb_tile,
      lb_scan,
      recs, recs64, cull2d, eig, pair_off,
      pk_a, pk_b, pv_a, pv_b, tile_off, pix_T, pix_last, pix_count, fwd_fix, bwd_fix, pix_mask, total;
  size_t small_end;  // [state, small_end) is zeroed at the start of a forward (with n > 0: up to the look-back end)
  size_t lb_sort_bytes, lb_tile_bytes, lb_scan_bytes;  // [lb_sort, lb_scan + lb_scan_bytes): one zeroing
};

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

Layout make_layout(int64_t n, int W, int H, int64_t cap) {
  Layout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const int64_t n_tiles = ceil_div(W, kTile) * ceil_div(H, kTile);
  const int64_t nn = std::max<int64_t>(n, 1), cc = std::max<int64_t>(cap, 1);
  L.state = take(sizeof(FrameState));
  L.hist_d = take(8 * kRadix * 4);
  L.off_d = take(8 * kRadix * 4);
  L.hist_p = take(2 * kRadix * 4);
  L.off_p = take(2 * kRadix * 4);
  L.small_end = off;
  // look-back slots of the depth sort, the tile sort and the pair-offset
  // scan, adjacent: zeroed by one memset at the start of a forward
  L.lb_sort_bytes = (size_t)(8 * ceil_div(nn, kSortTile)) * kRadix * 4;
  L.lb_sort = take(L.lb_sort_bytes);
  L.lb_tile_bytes = (size_t)(2 * ceil_div(cc, kSortTile)) * kRadix * 4;
  L.lb_tile = take(L.lb_tile_bytes);
  L.lb_scan_bytes = (size_t)ceil_div(nn, kScanThreads) * 8;
  L.lb_scan = take(L.lb_scan_bytes);
  L.keys_a = take(nn * 8);
  L.keys_b = take(nn * 8);
  L.vals_a = take(nn * 4);
  L.vals_b = take(nn * 4);
  L.rank = take(nn * 4);   // depth rank of each Gaussian (0xffffffff: culled)
  L.order = take(nn * 4);  // the depth order, rank -> Gaussian
  L.counts = take(nn * 4); // tiles per Gaussian (by index; 0: culled)
  L.keep = take(nn * 4);   // bbox tiles kept by the tile-level cull (bit mask, k_tile_counts)
  L.kept = take(nn);       // k_depth_keys' culls, read by the preprocess
  L.recs = take(nn * sizeof(SplatRec));
  L.recs64 = take(nn * sizeof(Rec64));
  L.cull2d = take(nn * 2 * sizeof(float4));
  L.eig = take(nn * sizeof(float2));  // by Gaussian index: a 3D splat's eigenbasis (c, s)
  L.pair_off = take(nn * 8);
  L.tile_off = take((n_tiles + 1) * 4);
  L.pix_T = take((size_t)W * H * 4);
  L.pix_last = take((size_t)W * H * 4);
  L.pix_count = take((size_t)W * H * 4);
  L.fwd_fix = take((size_t)W * H * sizeof(FwdFix));
  L.bwd_fix = take((size_t)W * H * sizeof(BwdFix));
  // contribution masks: one 32-bit word per (pixel, 32-entry chunk of its
  // tile list), chunk words of tile t at floor(lo_t / 32) + t + c
  L.pix_mask = take((size_t)((cc >> 5) + n_tiles + 2) * kBlock * 4);
  L.pk_a = take(cc * 4);
  L.pk_b = take(cc * 4);
  L.pv_a = take(cc * 4);
  L.pv_b = take(cc * 4);
  L.total = off;
  return L;
}

template <typename T>
T *at(void *base, size_t off) {
  return reinterpret_cast<T *>(static_cast<char *>(base) + off);
}
template <typename T>
const T *at(const void *base, size_t off) {
  return reinterpret_cast<const T *>(static_cast<const char *>(base) + off);
}

CamD make_cam(const hgs_camera &c) {
  CamD d;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) d.V[r * 3 + k] = c.world_to_camera[r * 4 + k];
    d.tv[r] = c.world_to_camera[r * 4 + 3];
  }
  const double K[16] = {c.fx, 0, c.cx, 0, 0, c.fy, c.cy, 0, 0, 0, 1, 0, 0, 0, 1, 0};
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k)
      d.T[r * 4 + k] = ((K[r * 4] * c.world_to_camera[k] + K[r * 4 + 1] * c.world_to_camera[4 + k]) +
                        K[r * 4 + 2] * c.world_to_camera[8 + k]) +
                       K[r * 4 + 3] * c.world_to_camera[12 + k];
  for (int k = 0; k < 3; ++k) d.campos[k] = -((d.V[k] * d.tv[0] + d.V[3 + k] * d.tv[1]) + d.V[6 + k] * d.tv[2]);
  d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy; d.near_plane = c.near_plane;
  d.width = c.width; d.height = c.height;
  d.tiles_x = (int)ceil_div(c.width, kTile);
  d.tiles_y = (int)ceil_div(c.height, kTile);
  return d;
}

SceneView make_scene(const hgs_scene &s) {
  SceneView v;
  v.center = s.center; v.log_scale = s.log_scale; v.rotation = s.rotation; v.opacity_logit = s.opacity_logit;
  v.sh = s.sh; v.type_spec = s.type_spec; v.n = s.n; v.sh_bases = s.sh_bases;
  const bool g64 = s.center64 && s.log_scale64 && s.rotation64 && s.opacity_logit64;
  v.center64 = g64 ? s.center64 : nullptr;
  v.log_scale64 = g64 ? s.log_scale64 : nullptr;
  v.rotation64 = g64 ? s.rotation64 : nullptr;
  v.opacity_logit64 = g64 ? s.opacity_logit64 : nullptr;
  return v;
}

int check_common(const hgs_scene *sc, const hgs_camera *cam, const hgs_settings *st) {
  if (!sc || !cam || !st) return HGS_ERR_CONFIG;
  if (st->tile_size != kTile) return HGS_ERR_CONFIG;
  if (cam->width <= 0 || cam->height <= 0 || cam->width > 65535 || cam->height > 65535) return HGS_ERR_CONFIG;
  if (!(cam->fx > 0) || !(cam->fy > 0) || !(cam->near_plane > 0) || !(cam->near_plane < cam->far_plane))
    return HGS_ERR_CONFIG;
  const int b = sc->sh_bases;
  if (b != 1 && b != 4 && b != 9 && b != 16) return HGS_ERR_CONFIG;
  if (sc->n < 0 || sc->n >= (1ll << 31)) return HGS_ERR_CONFIG;
  if (!(st->t_z > 0)) return HGS_ERR_CONFIG;
  return HGS_OK;
}

#define HGS_CUDA(x)                                         \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) return HGS_ERR_CUDA;             \
  } while (0)

#define HGS_LAUNCHED() HGS_CUDA(cudaGetLastError())

// The chain rule over Gaussians [g0, g1): one warp per CTA; shared memory:
// SH rows in + one SH-gradient set out.
cudaError_t chain_rule_range(ChainArgs c, int sh_bases, int64_t g0, int64_t g1, cudaStream_t s) {
  if (g1 <= g0) return cudaSuccess;
  c.g0 = g0;
  c.g1 = g1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(g1 - g0, 32), 148 * 48));
  const size_t smem = (size_t)2 * 32 * (3 * sh_bases + 1) * sizeof(float);
  return launch_chain_rule(c, sh_bases, grid, smem, s);
}

cudaError_t record_event(const hgs_settings *st, int i, cudaStream_t s) {
  if (!st->timing_events || i >= st->n_timing_events || !st->timing_events[i]) return cudaSuccess;
  return cudaEventRecord(static_cast<cudaEvent_t>(st->timing_events[i]), s);
}

int grid_for(int64_t work, int block) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, block), kMaxGrid));
}

// Stable LSD radix sort of (key, value) pairs over the listed 8-bit digit
// passes; returns true if the result landed in the *_b buffers.
template <typename K>
int radix_sort(K *ka, K *kb, uint32_t *va, uint32_t *vb, int64_t n, const int *passes, int npass,
               const uint32_t *offsets, uint32_t *lookback, uint32_t *counters, cudaStream_t s, bool *in_b) {
  *in_b = false;
  if (n == 0 || npass == 0) return HGS_OK;
  const int64_t tiles = ceil_div(n, kSortTile);
  HGS_CUDA(cudaMemsetAsync(lookback, 0, (size_t)tiles * kRadix * 4 * npass, s));
  HGS_CUDA(cudaMemsetAsync(counters, 0, 4 * npass, s));
  K *src = ka, *dst = kb;
  uint32_t *vs = va, *vd = vb;
  for (int i = 0; i < npass; ++i) {
    const int p = passes[i];
    HGS_CUDA(launch_pdl(k_onesweep<K>, dim3((unsigned)tiles), dim3(kSortThreads), 0, s, src, vs, dst, vd, n,
                        p * kRadixBits, offsets + p * kRadix, lookback + (size_t)i * tiles * kRadix, counters + i,
                        SortDev{nullptr, nullptr, 0, nullptr, nullptr}));
    HGS_LAUNCHED();
    std::swap(src, dst);
    std::swap(vs, vd);
    *in_b = !*in_b;
  }
  return HGS_OK;
}

}  // namespace

const float2 *frame_eig(const void *frame, const hgs_frame_info *info) {
  const Layout L = make_layout(info->n, info->width, info->height, info->pair_capacity);
  return at<float2>(frame, L.eig);
}

}  // namespace hgs

using namespace hgs;

extern "C" {

int hgs_abi_version(void) { return HGS_ABI_VERSION; }

const char *hgs_status_string(int status) {
  switch (status) {
    case HGS_OK: return "ok";
    case HGS_ERR_CONFIG: return "invalid configuration (camera, settings or shapes)";
    case HGS_ERR_INVALID_PARAMETER: return "invalid primitive parameters (quaternion norm below 1e-8)";
    case HGS_ERR_INTEGRITY: return "frame / scene / gradient mismatch";
    case HGS_ERR_DEGENERATE_SCALE: return "squared scales sum to zero or overflow";
    case HGS_ERR_PAIR_CAPACITY: return "frame buffer too small for the tile/splat pairs";
    case HGS_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

size_t hgs_frame_bytes(int64_t n, int32_t width, int32_t height, int32_t tile_size, int64_t pair_capacity) {
  if (tile_size != kTile || width <= 0 || height <= 0 || n < 0 || pair_capacity < 0) return 0;
  return make_layout(n, width, height, pair_capacity).total;
}

static int64_t capacity_of(size_t frame_bytes, int64_t n, int W, int H) {
  // largest capacity whose layout fits in frame_bytes (layout is affine in cap)
  size_t base = make_layout(n, W, H, 0).total;
  if (frame_bytes < base) return -1;
  int64_t lo = 0, hi = (int64_t)((frame_bytes - base) / 16) + 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (make_layout(n, W, H, mid).total <= frame_bytes) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// End of a forward: with HGS_FLAG_ASYNC the counts stay on the device (info
// m = k = -1 until hgs_frame_sync_info); otherwise the one host round trip
// of the frame reads M, K and the status.
static int finish_forward(void *frame, const Layout &L, hgs_frame_info *info, const hgs_settings *settings,
                          cudaStream_t s) {
  (void)L;
  if (settings->flags & HGS_FLAG_ASYNC) {
    info->m = -1;
    info->k = -1;
    return HGS_OK;
  }
  return hgs_frame_sync_info(frame, info, s);
}

int hgs_forward(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings, void *frame,
                size_t frame_bytes, const hgs_images *out, hgs_frame_info *info, void *stream) {
  NvtxScope nv("hgs_forward");
  int rc = check_common(scene, camera, settings);
  if (rc) return rc;
  if (!info || !frame) return HGS_ERR_CONFIG;
  if (!(settings->flags & HGS_FLAG_FRAME_ONLY) && (!out || !out->color || !out->depth || !out->transmittance))
    return HGS_ERR_CONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int W = camera->width, H = camera->height;
  const int64_t n = scene->n;
  const int64_t cap = capacity_of(frame_bytes, n, W, H);
  if (cap < 0) return HGS_ERR_PAIR_CAPACITY;
  const Layout L = make_layout(n, W, H, cap);
  const CamD cam = make_cam(*camera);
  const SceneView sc = make_scene(*scene);
  const ModD mod{settings->theta_z, settings->t_z, settings->lambda_z};
  const int64_t n_tiles = (int64_t)cam.tiles_x * cam.tiles_y;
  FrameState *st = at<FrameState>(frame, L.state);

  memset(info, 0, sizeof(*info));
  info->n = n; info->width = W; info->height = H; info->tiles_x = cam.tiles_x; info->tiles_y = cam.tiles_y;
  info->n_tiles = n_tiles; info->pair_capacity = cap; info->sh_bases = scene->sh_bases; info->flags = settings->flags;

  HGS_CUDA(record_event(settings, 0, s));
  nv.stage("front end: depth sort || float64 preprocess");
  // the frame state and histograms, and (n > 0) every look-back slot of the
  // frame (depth sort, tile sort, scan: adjacent), zeroed by one memset so
  // the sort and binning chains are kernels only
  HGS_CUDA(cudaMemsetAsync(frame, 0, n > 0 ? L.lb_scan + L.lb_scan_bytes : L.small_end, s));
  k_init_state<<<1, 1, 0, s>>>(sc, cam, mod, at<SplatRec>(frame, L.recs), at<Rec64>(frame, L.recs64), st);
  HGS_LAUNCHED();
  // Every launch below is sized from host-known bounds (N, the pair capacity,
  // the tile count) and reads the data-dependent counts -- M, the depth-sort
  // digit plan, K, the capacity verdict -- from the frame state on the
  // device: no host round trip inside a frame (stream-ordered, CUDA-graph
  // capturable).  Work past the device counts exits at once.
  const int64_t sort_tiles_n = ceil_div(std::max<int64_t>(n, 1), kSortTile);
  uint32_t *rank_of = at<uint32_t>(frame, L.rank);
  uint32_t *order = at<uint32_t>(frame, L.order);
  uint32_t *counts = at<uint32_t>(frame, L.counts);
  // With an auxiliary stream (hgs_settings.aux_stream + two caller events)
  // the float64 preprocess -- which needs only the scene and the culls --
  // runs on it beside the depth sort, and the main stream joins it before
  // the pair-offset scan.
  cudaStream_t aux = static_cast<cudaStream_t>(settings->aux_stream);
  const bool fork = aux && settings->aux_events[0] && settings->aux_events[1] && n > 0;
  // 1. depth keys + digit histograms + the pass plan
  if (n > 0) {
    HGS_CUDA(launch_depth_keys(sc, cam, at<unsigned long long>(frame, L.keys_a), at<uint32_t>(frame, L.vals_a),
                               at<uint8_t>(frame, L.kept), at<uint32_t>(frame, L.hist_d), st, grid_for(n, 256), s));
    HGS_CUDA(launch_ex(kDepthSortPdl, k_sort_plan, dim3(1), dim3(kRadix), 0, s, at<uint32_t>(frame, L.hist_d), n,
                        at<uint32_t>(frame, L.off_d), st));
    HGS_LAUNCHED();
    if (fork) {
      HGS_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(settings->aux_events[0]), s));
      HGS_CUDA(cudaStreamWaitEvent(aux, static_cast<cudaEvent_t>(settings->aux_events[0]), 0));
    }
    // HGS_SORT_ON_AUX: the depth sort on the side stream and the preprocess
    // on the caller's (a side stream created with a higher priority then
    // hands the sort's CTAs the SMs first as the preprocess's retire)
    cudaStream_t s_pre = (fork && !HGS_SORT_ON_AUX) ? aux : s;
    cudaStream_t s_sort = (fork && HGS_SORT_ON_AUX) ? aux : s;
    // 3a. float64 preprocess per Gaussian (record + tile count at its index)
    HGS_CUDA(launch_preprocess(sc, cam, mod, at<uint8_t>(frame, L.kept), at<SplatRec>(frame, L.recs),
                               at<Rec64>(frame, L.recs64), at<float4>(frame, L.cull2d), at<float2>(frame, L.eig),
                               counts, s_pre));
    HGS_LAUNCHED();
    if (HGS_TILE_COUNTS_AUX) {
      HGS_CUDA(launch_ex(HGS_TILE_COUNTS_PDL != 0, k_tile_counts, dim3(grid_for(n, 256)), dim3(256), 0, s_pre,
                         (const SplatRec *)at<SplatRec>(frame, L.recs), (const float4 *)at<float4>(frame, L.cull2d),
                         n, counts, at<uint32_t>(frame, L.keep)));
    }
    if (fork && !HGS_SORT_ON_AUX) HGS_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(settings->aux_events[1]), aux));
    // 2. depth sort: 8 digit passes launched, the constant ones exit at once
    uint32_t *lb = at<uint32_t>(frame, L.lb_sort);  // zeroed before the depth keys
    for (int i = 0; i < 8; ++i) {
      unsigned long long *ka = at<unsigned long long>(frame, (i & 1) ? L.keys_b : L.keys_a);
      unsigned long long *kb = at<unsigned long long>(frame, (i & 1) ? L.keys_a : L.keys_b);
      uint32_t *va = at<uint32_t>(frame, (i & 1) ? L.vals_b : L.vals_a);
      uint32_t *vb = at<uint32_t>(frame, (i & 1) ? L.vals_a : L.vals_b);
      HGS_CUDA(launch_ex(kDepthSortPdl, k_onesweep<unsigned long long>, dim3((unsigned)sort_tiles_n), dim3(kSortThreads), 0, s_sort,
                          ka, va, kb, vb, n, 0, at<uint32_t>(frame, L.off_d), lb + (size_t)i * sort_tiles_n * kRadix,
                          st->tile_counters + 1 + i,
                          HGS_FUSE_RANK_SCATTER ? SortDev{&st->sort_np, st->sort_digit, i, nullptr, nullptr, rank_of, order,
                                                          &st->m_count}
                                                : SortDev{&st->sort_np, st->sort_digit, i, nullptr, nullptr}));
      HGS_LAUNCHED();
    }
    if (!HGS_FUSE_RANK_SCATTER)
      HGS_CUDA(launch_ex(kDepthSortPdl, k_rank_scatter, dim3(grid_for(n, 256)), dim3(256), 0, s_sort,
                         at<uint32_t>(frame, L.vals_a), at<uint32_t>(frame, L.vals_b), st, n, rank_of, order));
    HGS_LAUNCHED();
    if (fork && HGS_SORT_ON_AUX) HGS_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(settings->aux_events[1]), aux));
    // join: the scan below needs both the depth order and the tile counts
    if (fork) HGS_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(settings->aux_events[1]), 0));
  }
  HGS_CUDA(record_event(settings, 1, s));  // stage 1 ends at the join
  nv.stage("pair-offset scan");
  // 3b. pair-offset scan over the depth order
  if (n > 0) {
    if (!HGS_TILE_COUNTS_AUX) {  // the tile-level cull of the counts, after the join
      k_tile_counts<<<grid_for(n, 256), 256, 0, s>>>(at<SplatRec>(frame, L.recs), at<float4>(frame, L.cull2d), n,
                                                     counts, at<uint32_t>(frame, L.keep));
      HGS_LAUNCHED();
    }
    HGS_CUDA(launch_pdl(k_scan_counts, dim3((unsigned)ceil_div(n, kScanTile)), dim3(kScanThreads), 0, s,
                        (const uint32_t *)counts, (const uint32_t *)order, (int64_t)-1,
                        at<unsigned long long>(frame, L.pair_off), at<unsigned long long>(frame, L.lb_scan), st,
                        (int64_t)std::min<int64_t>(cap, 0xffffffffll)));
  }
  HGS_CUDA(record_event(settings, 2, s));
  nv.stage("binning");
  // 4. duplicate + tile sort + ranges (K and the capacity verdict on the device)
  const int nd = n_tiles > kRadix ? 2 : 1;  // tile-sort digit passes
  const bool pairs_in_b = (nd & 1) != 0;    // where the sorted pairs land
  const uint32_t *tile_vals = at<uint32_t>(frame, pairs_in_b ? L.pv_b : L.pv_a);
  const uint32_t *tile_keys = at<uint32_t>(frame, pairs_in_b ? L.pk_b : L.pk_a);
  const int64_t sort_tiles_k = ceil_div(std::max<int64_t>(cap, 1), kSortTile);
  if (n > 0) {
    HGS_CUDA(launch_pdl(k_duplicate, dim3(grid_for(n, 256)), dim3(256), 0, s, (const SplatRec *)at<SplatRec>(frame, L.recs),
                        (const uint32_t *)order, (const unsigned long long *)at<unsigned long long>(frame, L.pair_off),
                        (int64_t)-1, (const FrameState *)st, (int)cam.tiles_x, (int)kTileShift, false, true,
                        (const uint32_t *)at<uint32_t>(frame, L.keep), at<uint32_t>(frame, L.pk_a),
                        at<uint32_t>(frame, L.pv_a), nd, at<uint32_t>(frame, L.hist_p)));
    HGS_CUDA(launch_pdl(k_radix_offsets, dim3(nd), dim3(kRadix), 0, s, (const uint32_t *)at<uint32_t>(frame, L.hist_p),
                        at<uint32_t>(frame, L.off_p)));
    uint32_t *lb = at<uint32_t>(frame, L.lb_tile);  // zeroed at the start of the frame
    for (int i = 0; i < nd; ++i) {
      HGS_CUDA(launch_pdl(k_onesweep<uint32_t>, dim3((unsigned)sort_tiles_k), dim3(kSortThreads), 0, s,
                          at<uint32_t>(frame, (i & 1) ? L.pk_b : L.pk_a), at<uint32_t>(frame, (i & 1) ? L.pv_b : L.pv_a),
                          at<uint32_t>(frame, (i & 1) ? L.pk_a : L.pk_b), at<uint32_t>(frame, (i & 1) ? L.pv_a : L.pv_b),
                          (int64_t)0, (int)(i * kRadixBits), at<uint32_t>(frame, L.off_p) + i * kRadix,
                          lb + (size_t)i * sort_tiles_k * kRadix, st->tile_counters + 12 + i,
                          SortDev{nullptr, nullptr, 0, &st->k_total, &st->status}));
      HGS_LAUNCHED();
    }
  }
  info->internal[0] = pairs_in_b ? 1u : 0u;
  info->internal[3] = (uint32_t)nd;
  HGS_CUDA(launch_pdl(k_tile_ranges, dim3(grid_for(ceil_div(std::max<int64_t>(cap, n_tiles + 1), 4), 256)), dim3(256), 0,
                      s, tile_keys, (int64_t)(n > 0 ? -1 : 0), (const FrameState *)st, (int64_t)n_tiles,
                      at<uint32_t>(frame, L.tile_off)));
  HGS_CUDA(record_event(settings, 3, s));
  nv.stage("composite + fixup");
  if (settings->flags & HGS_FLAG_FRAME_ONLY) return finish_forward(frame, L, info, settings, s);  // build_frame
  // 5. composite
  CompositeArgs a;
  a.recs = at<SplatRec>(frame, L.recs);
  a.tile_off = at<uint32_t>(frame, L.tile_off);
  a.tile_vals = (settings->flags & HGS_FLAG_NAIVE) ? order : tile_vals;
  a.rank_of = rank_of;
  a.m = -1;  // M lives in the frame state
  a.tiles_x = cam.tiles_x; a.width = W; a.height = H;
  a.flags = settings->flags;
  for (int c = 0; c < 3; ++c) a.bg[c] = settings->background[c];
  a.color = out->color; a.depth = out->depth; a.trans = out->transmittance; a.alpha = out->alpha;
  a.normal = out->normal;
  a.pix_T = at<float>(frame, L.pix_T);
  a.pix_last = at<uint32_t>(frame, L.pix_last);
  a.pix_count = at<uint32_t>(frame, L.pix_count);
  a.st = st;
  a.fwd_fix = at<FwdFix>(frame, L.fwd_fix);
  a.bwd_fix = at<BwdFix>(frame, L.bwd_fix);
  a.pix_mask = at<uint32_t>(frame, L.pix_mask);
  a.cull2d = at<float4>(frame, L.cull2d);
  const bool naive = settings->flags & HGS_FLAG_NAIVE, count = settings->flags & HGS_FLAG_COUNT;
  HGS_CUDA(launch_composite_fwd(a, n_tiles, naive, count, s));
  // deferred (float32-ambiguous) pixels, float64-exact; exits at once if none
  HGS_CUDA(launch_pdl(k_fixup_fwd, dim3(kFixupBlocks), dim3(256), 0, s, a));
  HGS_LAUNCHED();
  HGS_CUDA(record_event(settings, 4, s));
  nv.stage("finish");
  return finish_forward(frame, L, info, settings, s);
}

int hgs_frame_sync_info(void *frame, hgs_frame_info *info, void *stream) {
  if (!frame || !info) return HGS_ERR_CONFIG;
  const Layout L = make_layout(info->n, info->width, info->height, info->pair_capacity);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FrameState h;
  HGS_CUDA(cudaMemcpyAsync(&h, at<FrameState>(frame, L.state), sizeof(h), cudaMemcpyDeviceToHost, s));
  HGS_CUDA(cudaStreamSynchronize(s));
  info->m = h.m_count;
  info->k = (int64_t)h.k_total;
  info->internal[2] = h.sort_np;
  return (int)h.status;
}

static CompositeArgs composite_args_for(const hgs_scene *scene, const hgs_camera *camera,
                                        const hgs_settings *settings, const void *frame, const hgs_frame_info *info) {
  const Layout L = make_layout(info->n, info->width, info->height, info->pair_capacity);
  void *fr = const_cast<void *>(frame);
  CompositeArgs a;
  memset(&a, 0, sizeof(a));
  a.recs = at<SplatRec>(fr, L.recs);
  a.tile_off = at<uint32_t>(fr, L.tile_off);
  a.tile_vals = at<uint32_t>(fr, (info->flags & HGS_FLAG_NAIVE) ? L.order : (info->internal[0] ? L.pv_b : L.pv_a));
  a.rank_of = at<uint32_t>(fr, L.rank);
  a.m = info->m;
  a.tiles_x = info->tiles_x; a.width = info->width; a.height = info->height;
  a.flags = info->flags;
  for (int c = 0; c < 3; ++c) a.bg[c] = settings->background[c];
  a.pix_T = at<float>(fr, L.pix_T);
  a.pix_last = at<uint32_t>(fr, L.pix_last);
  a.pix_count = at<uint32_t>(fr, L.pix_count);
  a.st = at<FrameState>(fr, L.state);
  a.fwd_fix = at<FwdFix>(fr, L.fwd_fix);
  a.bwd_fix = at<BwdFix>(fr, L.bwd_fix);
  a.pix_mask = at<uint32_t>(fr, L.pix_mask);
  a.cull2d = at<float4>(fr, L.cull2d);
  (void)scene;
  (void)camera;
  return a;
}

static int check_frame(const hgs_scene *scene, const hgs_camera *camera, const hgs_frame_info *info) {
  if (!info) return HGS_ERR_INTEGRITY;
  if (info->n != scene->n || info->width != camera->width || info->height != camera->height ||
      info->sh_bases != scene->sh_bases)
    return HGS_ERR_INTEGRITY;
  return HGS_OK;
}

size_t hgs_backward_scratch_bytes(int64_t n, int32_t kg) {
  if (n < 0 || kg < 1) return 0;
  const int64_t kc = std::min<int32_t>(kg, 4);
  const int64_t nn = std::max<int64_t>(n, 1);
  constexpr int64_t A = sizeof(acc_t);
  return (size_t)(((nn * kc * 16 * A + 255) & ~255ll) + ((nn * kc * 4 * A + 255) & ~255ll) + ((nn + 255) & ~255ll));
}

}  // extern "C"

namespace {

// Deterministic-mode record buffers, after the base backward scratch.
struct DetLayout {
  size_t count, keys_a, keys_b, vals_a, vals_b, pay, hist, off, lookback, counters, total;
};

DetLayout det_layout(size_t base, int64_t kc, int64_t cap) {
  DetLayout d;
  size_t off = base;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const int64_t cc = std::max<int64_t>(cap, 1);
  d.count = take(16);
  d.keys_a = take(cc * 8);
  d.keys_b = take(cc * 8);
  d.vals_a = take(cc * 4);
  d.vals_b = take(cc * 4);
  d.pay = take((size_t)cc * kc * 20 * 4);
  d.hist = take(8 * kRadix * 4);
  d.off = take(8 * kRadix * 4);
  d.lookback = take((size_t)ceil_div(cc, kSortTile) * kRadix * 4 * 8);
  d.counters = take(64);
  d.total = off;
  return d;
}

// largest record capacity that fits in scratch_bytes (0 if none)
int64_t det_capacity(size_t base, int64_t kc, size_t scratch_bytes) {
  if (det_layout(base, kc, 1).total > scratch_bytes) return 0;
  int64_t lo = 1, hi = 2;
  while (det_layout(base, kc, hi).total <= scratch_bytes && hi < (1ll << 32)) hi *= 2;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (det_layout(base, kc, mid).total <= scratch_bytes) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace

extern "C" {

size_t hgs_backward_det_scratch_bytes(int64_t n, int32_t kg, int64_t records) {
  if (n < 0 || kg < 1 || records < 0) return 0;
  const int64_t kc = std::min<int32_t>(kg, 4);
  return det_layout(hgs_backward_scratch_bytes(n, kg), kc, records).total;
}

}  // extern "C"

extern "C" {

int hgs_backward(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings, const void *frame,
                 const hgs_frame_info *info, int32_t kg, const float *pixel_grads, const float *depth_grads,
                 const float *normal_grads, const float *alpha_grads, void *scratch, size_t scratch_bytes,
                 float *grads, uint8_t *touched, void *stream) {
  NvtxScope nv("hgs_backward");
  int rc = check_common(scene, camera, settings);
  if (rc) return rc;
  rc = check_frame(scene, camera, info);
  if (rc) return rc;
  if (info->flags & HGS_FLAG_FRAME_ONLY) return HGS_ERR_INTEGRITY;  // nothing was composited
  if (kg < 1 || !pixel_grads || (scene->n > 0 && (!grads || !touched))) return HGS_ERR_CONFIG;
  if (scratch_bytes < hgs_backward_scratch_bytes(scene->n, kg)) return HGS_ERR_CONFIG;
  const bool det = settings->flags & HGS_FLAG_DETERMINISTIC;
  const int64_t kc4 = std::min<int32_t>(kg, 4);
  const size_t base_bytes = hgs_backward_scratch_bytes(scene->n, kg);
  const int64_t rec_cap = det ? std::min<int64_t>(det_capacity(base_bytes, kc4, scratch_bytes), 0xffffffffll) : 0;
  if (det && rec_cap < 1) return HGS_ERR_CONFIG;
  const DetLayout DL = det_layout(base_bytes, kc4, std::max<int64_t>(rec_cap, 1));
  char *scr = static_cast<char *>(scratch);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = scene->n, m = info->m;
  const int64_t P = 11 + 3 * (int64_t)scene->sh_bases;
  const int64_t HW = (int64_t)info->width * info->height;
  const bool ext = depth_grads || normal_grads || alpha_grads;
  const int kc_max = std::min<int32_t>(kg, 4);
  const int64_t nn = std::max<int64_t>(n, 1);
  acc_t *acc = static_cast<acc_t *>(scratch);
  acc_t *acc_ext =
      reinterpret_cast<acc_t *>(static_cast<char *>(scratch) + ((nn * kc_max * 16 * (int64_t)sizeof(acc_t) + 255) & ~255ll));
  HGS_CUDA(record_event(settings, 0, s));
  nv.stage("back-to-front replay + fixup");
  HGS_CUDA(cudaMemsetAsync(touched, 0, (size_t)nn, s));
  BwdArgs b;
  b.c = composite_args_for(scene, camera, settings, frame, info);
  const SceneView sc = make_scene(*scene);
  const CamD cam = make_cam(*camera);
  const ModD mod{settings->theta_z, settings->t_z, settings->lambda_z};
  const Layout FLc = make_layout(info->n, info->width, info->height, info->pair_capacity);
  const bool replay_only = settings->flags & HGS_FLAG_REPLAY_ONLY;
  if (replay_only && kg > 4) return HGS_ERR_CONFIG;
  const ChainArgs c0{sc, cam, mod, acc, ext ? acc_ext : nullptr, 0, nullptr, at<float2>(frame, FLc.eig),
                     0, 0, (settings->flags & HGS_FLAG_ACCUMULATE) ? 1 : 0};
  for (int k0 = 0; k0 < kg; k0 += 4) {
    const int kc = std::min(4, kg - k0);
    HGS_CUDA(cudaMemsetAsync(acc, 0, (size_t)nn * kc * 16 * sizeof(acc_t), s));
    if (ext) HGS_CUDA(cudaMemsetAsync(acc_ext, 0, (size_t)nn * kc * 4 * sizeof(acc_t), s));
    b.pix_grad = pixel_grads + (int64_t)k0 * HW * 3;
    b.depth_grad = depth_grads ? depth_grads + (int64_t)k0 * HW : nullptr;
    b.normal_grad = normal_grads ? normal_grads + (int64_t)k0 * HW * 3 : nullptr;
    b.alpha_grad = alpha_grads ? alpha_grads + (int64_t)k0 * HW : nullptr;
    b.acc = acc;
    b.acc_ext = ext ? acc_ext : nullptr;
    b.touched = touched;
    b.rec_keys = det ? reinterpret_cast<unsigned long long *>(scr + DL.keys_a) : nullptr;
    b.rec_vals = det ? reinterpret_cast<uint32_t *>(scr + DL.vals_a) : nullptr;
    b.rec_pay = det ? reinterpret_cast<float *>(scr + DL.pay) : nullptr;
    b.rec_count = det ? reinterpret_cast<uint32_t *>(scr + DL.count) : nullptr;
    b.rec_cap = (uint32_t)rec_cap;
    // frame-state view, worklist count, diagnostics (first round) and the
    // deterministic record count: one launch, right before the compositor
    k_init_bwd<<<1, 1, 0, s>>>(sc, cam, mod, at<SplatRec>(const_cast<void *>(frame), FLc.recs),
                               at<Rec64>(const_cast<void *>(frame), FLc.recs64), b.c.st, b.rec_count, k0 == 0 ? 1 : 0);
    HGS_LAUNCHED();
    if (m != 0) {  // m < 0: an asynchronous frame (M on the device)
      HGS_CUDA(launch_composite_bwd(b, (int)kc, info->n_tiles, ext, det, s));
      if (det) {  // sort the records by (Gaussian, tile, sub) and reduce in that order
        uint32_t nrec = 0;
        HGS_CUDA(cudaMemcpyAsync(&nrec, b.rec_count, 4, cudaMemcpyDeviceToHost, s));
        HGS_CUDA(cudaStreamSynchronize(s));
        if ((int64_t)nrec > rec_cap) return HGS_ERR_PAIR_CAPACITY;  // grow the scratch, call again
        uint32_t *hist = reinterpret_cast<uint32_t *>(scr + DL.hist);
        uint32_t *offs = reinterpret_cast<uint32_t *>(scr + DL.off);
        HGS_CUDA(cudaMemsetAsync(hist, 0, 8 * kRadix * 4, s));
        if (nrec > 0) {
          k_radix_histogram<unsigned long long><<<grid_for(nrec, 256), 256, 0, s>>>(b.rec_keys, nrec, 8, hist);
          HGS_LAUNCHED();
        }
        k_radix_offsets<<<8, kRadix, 0, s>>>(hist, offs);
        HGS_LAUNCHED();
        uint32_t h[8 * kRadix];
        HGS_CUDA(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s));
        HGS_CUDA(cudaStreamSynchronize(s));
        int passes[8], np = 0;
        for (int pss = 0; pss < 8; ++pss) {
          bool trivial = false;
          for (int d = 0; d < kRadix; ++d)
            if (h[pss * kRadix + d] == nrec) trivial = true;
          if (!trivial) passes[np++] = pss;
        }
        bool in_b = false;
        rc = radix_sort<unsigned long long>(b.rec_keys, reinterpret_cast<unsigned long long *>(scr + DL.keys_b),
                                            b.rec_vals, reinterpret_cast<uint32_t *>(scr + DL.vals_b), nrec, passes,
                                            np, offs, reinterpret_cast<uint32_t *>(scr + DL.lookback),
                                            reinterpret_cast<uint32_t *>(scr + DL.counters), s, &in_b);
        if (rc) return rc;
        const unsigned long long *sk = in_b ? reinterpret_cast<unsigned long long *>(scr + DL.keys_b) : b.rec_keys;
        const uint32_t *sv = in_b ? reinterpret_cast<uint32_t *>(scr + DL.vals_b) : b.rec_vals;
        if (nrec > 0) {
          k_det_reduce<<<grid_for(nrec, 256), 256, 0, s>>>(sk, sv, b.rec_pay, nrec, kc, acc, ext ? acc_ext : nullptr);
          HGS_LAUNCHED();
        }
      }
      if (k0 == 0) {
        HGS_CUDA(record_event(settings, 1, s));
        nv.stage("chain rule");
      }
    }
    if (replay_only) break;  // kg <= 4: the accumulators stay for hgs_backward_chain
    ChainArgs c = c0;
    c.kg = kc;
    c.touched = touched;  // written by this call's replay (and its fixup)
    c.grads = grads + (int64_t)k0 * n * P;
    HGS_CUDA(chain_rule_range(c, scene->sh_bases, 0, n, s));
  }
  HGS_CUDA(record_event(settings, 2, s));
  return HGS_OK;
}

int hgs_backward_chain(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings,
                       const void *frame, const hgs_frame_info *info, int32_t kg, const float *depth_grads,
                       const float *normal_grads, const float *alpha_grads, const void *scratch,
                       size_t scratch_bytes, int64_t g0, int64_t g1, float *grads, void *stream) {
  NvtxScope nv("hgs_backward_chain");
  int rc = check_common(scene, camera, settings);
  if (rc) return rc;
  rc = check_frame(scene, camera, info);
  if (rc) return rc;
  if (kg < 1 || kg > 4 || !scratch || scratch_bytes < hgs_backward_scratch_bytes(scene->n, kg)) return HGS_ERR_CONFIG;
  if (g0 < 0 || g1 < g0 || g1 > scene->n || (g1 > g0 && !grads)) return HGS_ERR_CONFIG;
  if (g1 == g0) return HGS_OK;
  const int64_t nn = std::max<int64_t>(scene->n, 1);
  const acc_t *acc = static_cast<const acc_t *>(scratch);
  const acc_t *acc_ext = reinterpret_cast<const acc_t *>(static_cast<const char *>(scratch) +
                                                         ((nn * kg * 16 * (int64_t)sizeof(acc_t) + 255) & ~255ll));
  const bool ext = depth_grads || normal_grads || alpha_grads;
  const Layout FL = make_layout(info->n, info->width, info->height, info->pair_capacity);
  ChainArgs c{make_scene(*scene), make_cam(*camera), ModD{settings->theta_z, settings->t_z, settings->lambda_z},
              acc, ext ? acc_ext : nullptr, kg, grads, at<float2>(frame, FL.eig), 0, 0,
              (settings->flags & HGS_FLAG_ACCUMULATE) ? 1 : 0};
  HGS_CUDA(chain_rule_range(c, scene->sh_bases, g0, g1, static_cast<cudaStream_t>(stream)));
  return HGS_OK;
}

}  // extern "C"

namespace {
template <typename T>
int exchange_impl(int64_t n, T *log_scale, T *rotation, uint8_t *type_spec, double theta_e, T *eranks, void *scratch,
                  hgs_exchange_report *report, void *stream) {
  if (n < 0 || !report || !scratch || !(theta_e > 1.0 && theta_e < 3.0)) return HGS_ERR_CONFIG;
  memset(report, 0, sizeof(*report));
  if (n == 0) return HGS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ExchangeState *st = static_cast<ExchangeState *>(scratch);
  HGS_CUDA(cudaMemsetAsync(st, 0, sizeof(ExchangeState), s));
  HGS_CUDA(launch_exchange_scan<T>(n, log_scale, type_spec, theta_e, eranks, st, grid_for(n, 256), s));
  ExchangeState h;
  HGS_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  HGS_CUDA(cudaStreamSynchronize(s));
  if (h.counts[3]) return HGS_ERR_DEGENERATE_SCALE;
  HGS_CUDA(launch_exchange_apply<T>(n, log_scale, rotation, type_spec, theta_e, grid_for(n, 256), s));
  report->n_3d_to_2d = (int64_t)h.counts[0];
  report->n_2d_to_3d = (int64_t)h.counts[1];
  report->n_3d = (int64_t)h.counts[2] - (int64_t)h.counts[0] + (int64_t)h.counts[1];
  report->n_2d = n - report->n_3d;
  for (int b = 0; b < 20; ++b) report->erank_hist[b] = (int64_t)h.hist[b];
  return HGS_OK;
}
}  // namespace

extern "C" {

int hgs_exchange(int64_t n, float *log_scale, float *rotation, uint8_t *type_spec, double theta_e, float *eranks,
                 void *scratch, hgs_exchange_report *report, void *stream) {
  NvtxScope nv("hgs_exchange");
  return exchange_impl<float>(n, log_scale, rotation, type_spec, theta_e, eranks, scratch, report, stream);
}

int hgs_exchange_f64(int64_t n, double *log_scale, double *rotation, uint8_t *type_spec, double theta_e,
                     double *eranks, void *scratch, hgs_exchange_report *report, void *stream) {
  NvtxScope nv("hgs_exchange_f64");
  return exchange_impl<double>(n, log_scale, rotation, type_spec, theta_e, eranks, scratch, report, stream);
}

}  // extern "C"

// ------------------------------------------------------------- export

namespace hgs {

__global__ void k_export_frame(SceneView sc, CamD cam, ModD mod, const uint32_t *__restrict__ order, int64_t m,
                               hgs_frame_export o) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = order[r];
    ProjD p;
    if (sc.center64) project_d<true, false, true>(sc, i, cam, mod, p);
    else project_d(sc, i, cam, mod, p);
    bbox_d(p, cam.width, cam.height);
    if (o.idx) o.idx[r] = (int32_t)i;
    if (o.typ) o.typ[r] = (uint8_t)p.typ;
    if (o.depth) o.depth[r] = p.t[2];
    if (o.center2d) { o.center2d[2 * r] = p.ctr[0]; o.center2d[2 * r + 1] = p.ctr[1]; }
    for (int k = 0; k < 3; ++k) {
      if (o.cov2d) o.cov2d[3 * r + k] = p.cov[k];
      if (o.conic) o.conic[3 * r + k] = p.conic[k];
      if (o.color) o.color[3 * r + k] = p.color[k];
      if (o.normal) o.normal[3 * r + k] = p.normal[k];
    }
    if (o.mrow)
      for (int k = 0; k < 12; ++k) o.mrow[12 * r + k] = p.mrow[k];
    if (o.alpha_eff) o.alpha_eff[r] = p.alpha_eff;
    if (o.alpha) o.alpha[r] = p.alpha;
    if (o.cam_dist) o.cam_dist[r] = p.cam_dist;
    for (int k = 0; k < 3; ++k) {
      if (o.t_cam) o.t_cam[3 * r + k] = p.t[k];
      if (o.view_dir) o.view_dir[3 * r + k] = p.view_dir[k];
    }
    if (o.radius) o.radius[r] = p.radius;
    if (o.bbox)
      for (int k = 0; k < 4; ++k) o.bbox[4 * r + k] = p.bbox[k];
  }
}

// Tile lists hold Gaussian indices; SplatFrame.tile_ids holds slots.
__global__ void k_export_slots(const uint32_t *__restrict__ vals, const uint32_t *__restrict__ rank_of, int64_t k,
                               int32_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)rank_of[vals[i]];
}

__global__ void k_export_u32_to_i64(const uint32_t *__restrict__ src, int64_t *__restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Blend log (render.py:30-51): one thread per pixel re-walks its tile list
// with the forward's exact decisions and writes (position, alpha, u, v).
__global__ void k_blend_log(CompositeArgs a, const int64_t *__restrict__ offsets, int32_t *__restrict__ pos,
                            float *__restrict__ alpha, float *__restrict__ u, float *__restrict__ v) {
  const int64_t HW = (int64_t)a.width * a.height;
  const bool naive = a.flags & HGS_FLAG_NAIVE;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < HW; pix += (int64_t)gridDim.x * blockDim.x) {
    const int ix = (int)(pix % a.width), iy = (int)(pix / a.width);
    const int tile = (iy / kTile) * a.tiles_x + ix / kTile;
    const int64_t lo = naive ? 0 : a.tile_off[tile];
    const int64_t end = lo + a.pix_last[pix];
    int64_t o = offsets[pix];
    for (int64_t j = lo; j < end; ++j) {
      const uint32_t rk = a.tile_vals[j];  // NAIVE: the depth order
      const SplatRec r = a.recs[rk];
      if (!naive) {
        const int4 q = r.r5;
        const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16);
        const int x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
        if (ix < x0 || ix > x1 || iy < y0 || iy > y1) continue;
      }
      PairEval p;
      if (!eval_pair<true>(r, a.recs + rk, ix, iy, a.flags, a.st, p)) continue;
      pos[o] = (int32_t)a.rank_of[rk];  // the SplatFrame slot
      alpha[o] = p.at;
      if (rec_is3d(r)) {
        u[o] = p.u;
        v[o] = p.v;
      } else {
        // the ray/plane coordinates in float64 (_blend_py.py:38-40): near a
        // degenerate solve the float32 ones lose every digit (the pair is
        // then on the low-pass branch, so the image does not depend on them)
        const Rec64 q = a.st->recs64[rk];
        const double *m = q.g;
        const double px = ix + 0.5, py = iy + 0.5;
        const double hu0 = px * m[6] - m[0], hu1 = px * m[7] - m[1], hu3 = px * m[8] - m[2];
        const double hv0 = py * m[6] - m[3], hv1 = py * m[7] - m[4], hv3 = py * m[8] - m[5];
        const double den = hu0 * hv1 - hu1 * hv0;
        u[o] = (float)((hu1 * hv3 - hu3 * hv1) / den);
        v[o] = (float)((hu3 * hv0 - hu0 * hv3) / den);
      }
      ++o;
    }
  }
}

}  // namespace hgs

extern "C" {

int hgs_frame_export_arrays(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings,
                            const void *frame, const hgs_frame_info *info, const hgs_frame_export *out, void *stream) {
  int rc = check_common(scene, camera, settings);
  if (rc) return rc;
  rc = check_frame(scene, camera, info);
  if (rc) return rc;
  if (info->m < 0 || info->k < 0) return HGS_ERR_INTEGRITY;  // asynchronous frame: hgs_frame_sync_info first
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const CompositeArgs a = composite_args_for(scene, camera, settings, frame, info);
  if (info->m > 0) {
    const Layout FL = make_layout(info->n, info->width, info->height, info->pair_capacity);
    k_export_frame<<<grid_for(info->m, 128), 128, 0, s>>>(make_scene(*scene), make_cam(*camera),
        ModD{settings->theta_z, settings->t_z, settings->lambda_z}, at<uint32_t>(frame, FL.order), info->m, *out);
    HGS_LAUNCHED();
  }
  if (out->tile_offsets) {
    k_export_u32_to_i64<<<grid_for(info->n_tiles + 1, 256), 256, 0, s>>>(a.tile_off, out->tile_offsets,
                                                                        info->n_tiles + 1);
    HGS_LAUNCHED();
  }
  if (out->tile_ids && info->k > 0 && !(info->flags & HGS_FLAG_NAIVE)) {
    k_export_slots<<<grid_for(info->k, 256), 256, 0, s>>>(a.tile_vals, a.rank_of, info->k, out->tile_ids);
    HGS_LAUNCHED();
  }
  if (out->pixel_count) {
    if (info->flags & HGS_FLAG_NAIVE) {
      HGS_CUDA(cudaMemcpyAsync(out->pixel_count, a.pix_count, (size_t)info->width * info->height * 4,
                               cudaMemcpyDeviceToDevice, s));
    } else {
      k_pixel_counts<<<grid_for((int64_t)info->width * info->height, 256), 256, 0, s>>>(a, reinterpret_cast<uint32_t *>(out->pixel_count));
      HGS_LAUNCHED();
    }
  }
  return HGS_OK;
}

int hgs_frame_stats(const void *frame, const hgs_frame_info *info, uint64_t *out16, void *stream) {
  if (!frame || !info || !out16) return HGS_ERR_CONFIG;
  const Layout L = make_layout(info->n, info->width, info->height, info->pair_capacity);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const FrameState *st = at<FrameState>(frame, L.state);
  HGS_CUDA(cudaMemcpyAsync(out16, st->diag, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  HGS_CUDA(cudaStreamSynchronize(s));
  return HGS_OK;
}

int hgs_blend_log(const hgs_scene *scene, const hgs_camera *camera, const hgs_settings *settings, const void *frame,
                  const hgs_frame_info *info, const int64_t *offsets, int32_t *position, float *alpha, float *u,
                  float *v, void *stream) {
  int rc = check_common(scene, camera, settings);
  if (rc) return rc;
  rc = check_frame(scene, camera, info);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const CompositeArgs a = composite_args_for(scene, camera, settings, frame, info);
  const int64_t HW = (int64_t)info->width * info->height;
  k_blend_log<<<grid_for(HW, 128), 128, 0, s>>>(a, offsets, position, alpha, u, v);
  HGS_LAUNCHED();
  return HGS_OK;
}

}  // extern "C"

// ------------------------------------------------------------- re-binning

namespace {

struct RebinLayout {
  size_t state, counts, pair_off, lb_scan, hist, offs, lb_sort, ka, kb, va, vb, tile_off, total;
};

int tile_shift_of(int t) {
  switch (t) {
    case 8: return 3;
    case 16: return 4;
    case 32: return 5;
    case 64: return 6;
    default: return -1;
  }
}

RebinLayout rebin_layout(int64_t m, int W, int H, int tile, int64_t cap) {
  RebinLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const int64_t mm = std::max<int64_t>(m, 1), cc = std::max<int64_t>(cap, 1);
  const int64_t tiles = ceil_div(W, tile) * ceil_div(H, tile);
  L.state = take(sizeof(FrameState));
  L.hist = take(3 * kRadix * 4);
  L.offs = take(3 * kRadix * 4);
  L.counts = take(mm * 4);
  L.pair_off = take(mm * 8);
  L.lb_scan = take((size_t)ceil_div(mm, kScanTile) * 8);
  L.lb_sort = take((size_t)3 * ceil_div(cc, kSortTile) * kRadix * 4);
  L.ka = take(cc * 4);
  L.kb = take(cc * 4);
  L.va = take(cc * 4);
  L.vb = take(cc * 4);
  L.tile_off = take((tiles + 1) * 4);
  L.total = off;
  return L;
}

}  // namespace

extern "C" {

size_t hgs_tile_bins_scratch_bytes(int64_t m, int32_t width, int32_t height, int32_t tile_size,
                                   int64_t pair_capacity) {
  if (tile_shift_of(tile_size) < 0 || width <= 0 || height <= 0 || m < 0 || pair_capacity < 0) return 0;
  return rebin_layout(m, width, height, tile_size, pair_capacity).total;
}

int hgs_frame_tile_bins(const void *frame, const hgs_frame_info *info, int32_t tile_size, int64_t *tile_offsets,
                        int32_t *tile_ids, int64_t ids_capacity, void *scratch, size_t scratch_bytes, int64_t *k_out,
                        void *stream) {
  const int sh = tile_shift_of(tile_size);
  if (!frame || !info || sh < 0 || !tile_offsets || !k_out || ids_capacity < 0 || !scratch) return HGS_ERR_CONFIG;
  const int W = info->width, H = info->height;
  const int64_t m = info->m;
  if (m < 0) return HGS_ERR_INTEGRITY;  // asynchronous frame: hgs_frame_sync_info first
  const RebinLayout R = rebin_layout(m, W, H, tile_size, ids_capacity);
  if (scratch_bytes < R.total) return HGS_ERR_CONFIG;
  const Layout L = make_layout(info->n, W, H, info->pair_capacity);
  const SplatRec *recs = at<SplatRec>(frame, L.recs);
  const uint32_t *order = at<uint32_t>(frame, L.order);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int tiles_x = (int)ceil_div(W, tile_size);
  const int64_t n_tiles = (int64_t)tiles_x * ceil_div(H, tile_size);
  FrameState *st = at<FrameState>(scratch, R.state);
  HGS_CUDA(cudaMemsetAsync(scratch, 0, R.counts, s));  // state + histograms
  int64_t K = 0;
  if (m > 0) {
    HGS_CUDA(cudaMemsetAsync(at<char>(scratch, R.lb_scan), 0, (size_t)ceil_div(m, kScanTile) * 8, s));
    k_rebin_counts<<<grid_for(m, 256), 256, 0, s>>>(recs, order, m, sh, at<uint32_t>(scratch, R.counts));
    HGS_LAUNCHED();
    k_scan_counts<<<(unsigned)ceil_div(m, kScanTile), kScanThreads, 0, s>>>(
        at<uint32_t>(scratch, R.counts), nullptr, m, at<unsigned long long>(scratch, R.pair_off),
        at<unsigned long long>(scratch, R.lb_scan), st, -1);
    HGS_LAUNCHED();
    unsigned long long kt;
    HGS_CUDA(cudaMemcpyAsync(&kt, &st->k_total, 8, cudaMemcpyDeviceToHost, s));
    HGS_CUDA(cudaStreamSynchronize(s));
    K = (int64_t)kt;
  }
  *k_out = K;
  if (K > ids_capacity || K >= (1ll << 32)) return HGS_ERR_PAIR_CAPACITY;
  const uint32_t *keys = at<uint32_t>(scratch, R.ka), *vals = at<uint32_t>(scratch, R.va);
  if (K > 0) {
    const int nd = n_tiles > kRadix ? 2 : 1;
    if (n_tiles > (1 << 16)) return HGS_ERR_CONFIG;  // 2 digit passes cover 65536 tiles
    k_duplicate<<<grid_for(m, 256), 256, 0, s>>>(recs, order, at<unsigned long long>(scratch, R.pair_off), m, nullptr,
                                                 tiles_x, sh, true, false, nullptr,
                                                 at<uint32_t>(scratch, R.ka), at<uint32_t>(scratch, R.va),
                                                 nd, at<uint32_t>(scratch, R.hist));
    HGS_LAUNCHED();
    k_radix_offsets<<<nd, kRadix, 0, s>>>(at<uint32_t>(scratch, R.hist), at<uint32_t>(scratch, R.offs));
    HGS_LAUNCHED();
    int passes[2] = {0, 1};
    bool in_b;
    int rc = radix_sort<uint32_t>(at<uint32_t>(scratch, R.ka), at<uint32_t>(scratch, R.kb),
                                  at<uint32_t>(scratch, R.va), at<uint32_t>(scratch, R.vb), K, passes, nd,
                                  at<uint32_t>(scratch, R.offs), at<uint32_t>(scratch, R.lb_sort),
                                  st->tile_counters + 12, s, &in_b);
    if (rc) return rc;
    keys = at<uint32_t>(scratch, in_b ? R.kb : R.ka);
    vals = at<uint32_t>(scratch, in_b ? R.vb : R.va);
  }
  k_tile_ranges<<<grid_for(ceil_div(std::max<int64_t>(K, n_tiles + 1), 4), 256), 256, 0, s>>>(
      keys, K, nullptr, n_tiles, at<uint32_t>(scratch, R.tile_off));
  HGS_LAUNCHED();
  k_export_u32_to_i64<<<grid_for(n_tiles + 1, 256), 256, 0, s>>>(at<uint32_t>(scratch, R.tile_off), tile_offsets,
                                                                 n_tiles + 1);
  HGS_LAUNCHED();
  if (K > 0 && tile_ids) HGS_CUDA(cudaMemcpyAsync(tile_ids, vals, (size_t)K * 4, cudaMemcpyDeviceToDevice, s));
  return HGS_OK;
}

}  // extern "C"
