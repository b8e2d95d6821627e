// hgs_forward.cu -- forward kernels: depth keys, float64 preprocess + pair
// scan, tile duplication, tile ranges and the per-tile front-to-back
// compositor.  Semantics: raster/project.py:169-379 and
// raster/_blend_py.py:55-123 (paths relative to the reference package).
#include "hgs_kernels.cuh"

#ifndef HGS_PRE_CTAS
#define HGS_PRE_CTAS 14  // A/B 8 / 12 / 13 / 14 / 15 / 16 / 18 / 24 / 48: 14 still leaves room for the depth sort beside it
#endif
#ifndef HGS_PRE_PREFETCH
#define HGS_PRE_PREFETCH 1
#endif
#ifndef HGS_PRE_ASYNC
#define HGS_PRE_ASYNC 1
#endif
#ifndef HGS_PRE_MINB
#define HGS_PRE_MINB 1  // one-warp CTAs per SM the float64 preprocess is register-budgeted for
#endif

namespace hgs {

__global__ void k_init_state(SceneView sc, CamD cam, ModD mod, const SplatRec *recs, const Rec64 *recs64,
                             FrameState *st) {
  st->sc = sc;
  st->cam = cam;
  st->mod = mod;
  st->recs = recs;
  st->recs64 = recs64;
}

// The backward's per-round state: the scene / camera view of the frame
// state, the deferred-pixel worklist count, the backward's diagnostic
// counters (first round) and the deterministic record count -- one launch
// instead of a kernel and three small memsets.
__global__ void k_init_bwd(SceneView sc, CamD cam, ModD mod, const SplatRec *recs, const Rec64 *recs64,
                           FrameState *st, uint32_t *rec_count, int zero_diag) {
  pdl_launch_dependents();  // the backward compositor may be scheduled as this drains
  st->sc = sc;
  st->cam = cam;
  st->mod = mod;
  st->recs = recs;
  st->recs64 = recs64;
  st->n_fix_bwd = 0;
  if (zero_diag)
    for (int k = 6; k < 10; ++k) st->diag[k] = 0ull;
  if (rec_count) *rec_count = 0;
}

// The float64 projection a pair re-check needs (Rec64).
__device__ __forceinline__ void write_rec64(const ProjD &o, Rec64 *q) {
  Rec64 r;
  r.ctr[0] = o.ctr[0];
  r.ctr[1] = o.ctr[1];
  r.alpha_eff = o.alpha_eff;
  if (o.typ == 1) {
    r.g[0] = o.conic[0]; r.g[1] = o.conic[1]; r.g[2] = o.conic[2];
    for (int k = 3; k < 9; ++k) r.g[k] = 0.0;
  } else {
    const double *m = o.mrow;
    r.g[0] = m[0]; r.g[1] = m[1]; r.g[2] = m[3];
    r.g[3] = m[4]; r.g[4] = m[5]; r.g[5] = m[7];
    r.g[6] = m[8]; r.g[7] = m[9]; r.g[8] = m[11];
  }
  // six 16-byte streaming stores (the records are read only by rare re-checks)
  const double2 *src = reinterpret_cast<const double2 *>(&r);
  double2 *dst = reinterpret_cast<double2 *>(q);
#pragma unroll
  for (int k = 0; k < 6; ++k) __stcs(dst + k, src[k]);
}

// ------------------------------------------------------------ depth keys
// Per Gaussian: view depth in float64, near cull (project.py:181-185),
// singular-conic validity for 3D (project.py:225), |q| check (rotation.py:
// 19-20).  key = bits(z) for kept splats, ~0 otherwise (they sort last and
// are not counted in M).  Also accumulates the 8 digit histograms.
template <bool G64>
__global__ void __launch_bounds__(256) k_depth_keys(SceneView sc, CamD cam, unsigned long long *__restrict__ keys,
                                                    uint32_t *__restrict__ vals, uint8_t *__restrict__ kept,
                                                    uint32_t *__restrict__ hist, FrameState *__restrict__ st) {
  if (HGS_DEPTH_SORT_TRIGGER) pdl_launch_dependents();
  pdl_wait();
  using G = SceneGeom<G64>;
  __shared__ uint32_t sh[8 * kRadix];
  __shared__ uint32_t s_m;
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  uint32_t bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sc.n; i += (int64_t)gridDim.x * blockDim.x) {
    double p[3], t[3];
    load_center_d<G64>(sc, i, p);
    t_cam_d(cam, p, t);
    bool keep = t[2] > cam.near_plane;
    if (keep) {
      double R[9];
      bool qok = quat_to_matrix_d(G::rotation(sc, i, 0), G::rotation(sc, i, 1), G::rotation(sc, i, 2),
                                  G::rotation(sc, i, 3), R);
      if (!qok) {
        bad = 1;
        keep = false;
      } else if (sc.type_spec[i] == 1) {
        double s[3] = {exp(G::log_scale(sc, i, 0)), exp(G::log_scale(sc, i, 1)), exp(G::log_scale(sc, i, 2))};
        double a, b, c;
        cov2d_3d(cam, t, R, s, a, b, c);
        keep = conic_det(a, b, c) > 1e-18;
      }
    }
    unsigned long long k = keep ? (unsigned long long)__double_as_longlong(t[2]) : ~0ull;
    keys[i] = k;
    vals[i] = (uint32_t)i;
    kept[i] = keep ? 1 : 0;  // the preprocess (beside the sort) skips exactly these
    if (keep) atomicAdd(&s_m, 1u);
#pragma unroll
    for (int pss = 0; pss < 8; ++pss) atomicAdd(&sh[pss * kRadix + digit_of(k, pss * 8)], 1u);
  }
  if (bad) atomicOr(&st->status, (uint32_t)HGS_ERR_INVALID_PARAMETER);
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  if (threadIdx.x == 0 && s_m) atomicAdd(&st->m_count, s_m);
}
cudaError_t launch_depth_keys(const SceneView &sc, const CamD &cam, unsigned long long *keys, uint32_t *vals,
                              uint8_t *kept, uint32_t *hist, FrameState *st, int grid, cudaStream_t s) {
  // right behind k_init_state under PDL (set up while it runs)
  if (sc.center64) return launch_pdl(k_depth_keys<true>, dim3(grid), dim3(256), 0, s, sc, cam, keys, vals, kept, hist, st);
  return launch_pdl(k_depth_keys<false>, dim3(grid), dim3(256), 0, s, sc, cam, keys, vals, kept, hist, st);
}

// ---------------------------------------------------- preprocess + scan
__device__ __forceinline__ uint32_t tile_count_of(const int *bb) {
  if (bb[2] < bb[0]) return 0u;
  uint32_t tx = (uint32_t)(bb[2] / kTile - bb[0] / kTile + 1);
  uint32_t ty = (uint32_t)(bb[3] / kTile - bb[1] / kTile + 1);
  return tx * ty;
}

__device__ __forceinline__ void write_record(const ProjD &o, uint32_t idx, int W, int H, SplatRec *__restrict__ rec,
                                             float4 *__restrict__ cull, float2 *__restrict__ eig) {
  // anchor pixel = floor(centre), kept within +-2^30 so (ix - ax) stays exact;
  // a 3D splat's anchor is also clamped to the image (see r2 below)
  double axd = floor(o.ctr[0]), ayd = floor(o.ctr[1]);
  axd = fmin(fmax(axd, -1073741824.0), 1073741824.0);
  ayd = fmin(fmax(ayd, -1073741824.0), 1073741824.0);
  if (isnan(axd)) axd = 0.0;
  if (isnan(ayd)) ayd = 0.0;
  if (o.typ == 1) {
    axd = fmin(fmax(axd, 0.0), (double)(W - 1));
    ayd = fmin(fmax(ayd, 0.0), (double)(H - 1));
  }
  SplatRec r;
  r.r0 = make_float4((float)(o.ctr[0] - axd), (float)(o.ctr[1] - ayd), (float)o.t[2], (float)log2(o.alpha_eff));
  if (o.typ == 1) {
    // the conic in its eigenbasis, (cos t, sin t, lambda_p, lambda_q): the
    // compositors evaluate d = lambda_p p^2 + lambda_q q^2 on the rotated
    // offset (p, q), a sum of non-negative terms (the (a, b, c) form cancels
    // catastrophically for elongated splats at the cutoff)
    // eigenvector of the larger eigenvalue from the row of (Q - l1 I) without
    // cancellation; l2 = mean - h directly (its float64 cancellation, ~1e-16
    // l1, is far below the float32 the record keeps); no divisions
    const double A = o.conic[0], B = o.conic[1], C = o.conic[2];
    const double hd = 0.5 * (A - C), h = sqrt(hd * hd + B * B);
    const double l1 = 0.5 * (A + C) + h, l2 = 0.5 * (A + C) - h;
    double vx = hd >= 0.0 ? hd + h : B, vy = hd >= 0.0 ? B : h - hd;
    const double vq = vx * vx + vy * vy;
    if (vq > 0.0) {
      const double rn = rsqrt(vq);
      vx *= rn;
      vy *= rn;
    } else {
      vx = 1.0;
      vy = 0.0;
    }
    r.r1 = make_float4((float)vx, (float)vy, (float)l1, (float)fmax(l2, 0.0));
    // (P0, Q0): the anchor pixel's offset from the centre in the eigenbasis,
    // in float64, so a pixel's rotated offset is (P0, Q0) + R (pxl, pyl) with
    // (pxl, pyl) small (the anchor is on the image).  Rotating the full offset
    // in float32 instead costs eps |offset| -- 0.02 px for a near-camera splat
    // whose centre is 3e5 px off-screen, a systematic gradient error that the
    // 3D chain rule amplifies ~100x.
    const double ox = axd - o.ctr[0], oy = ayd - o.ctr[1];
    const double P0 = vx * ox + vy * oy, Q0 = vx * oy - vy * ox;
    const float P0f = (float)P0, Q0f = (float)Q0;
    r.r2 = make_float4(P0f, Q0f, fabsf(P0f) + fabsf(Q0f), 0.f);
    *eig = make_float2(r.r1.x, r.r1.y);  // the chain rule rotates the eigenbasis sums back with these
    r.r3 = make_float4(0.f, (float)o.color[0], (float)o.color[1], (float)o.color[2]);
  } else {
    const double *m = o.mrow;  // rows x(0..3), y(4..7), w(8..11)
    double m00 = m[0] - axd * m[8], m01 = m[1] - axd * m[9], m03 = m[3] - axd * m[11];
    double m10 = m[4] - ayd * m[8], m11 = m[5] - ayd * m[9], m13 = m[7] - ayd * m[11];
    r.r1 = make_float4((float)m00, (float)m01, (float)m03, (float)m10);
    r.r2 = make_float4((float)m11, (float)m13, (float)m[8], (float)m[9]);
    r.r3 = make_float4((float)m[11], (float)o.color[0], (float)o.color[1], (float)o.color[2]);
  }
  uint32_t tag = idx | ((uint32_t)(o.typ == 1) << 31);
  r.r4 = make_float4((float)o.normal[0], (float)o.normal[1], (float)o.normal[2], __uint_as_float(tag));
  int x0 = o.bbox[0], y0 = o.bbox[1], x1 = o.bbox[2], y1 = o.bbox[3];
  if (x1 < x0) {  // off screen: empty box, never binned
    x0 = 1; x1 = 0; y0 = 1; y1 = 0;
  }
  r.r5 = make_int4((int)((uint32_t)x0 | ((uint32_t)y0 << 16)), (int)((uint32_t)x1 | ((uint32_t)y1 << 16)), (int)axd,
                   (int)ayd);
  *rec = r;
  if (o.typ != 1) {  // the 2D support conic of the compositor's warp cull
    float4 k0, k1;
    cull2d_prep(r, k0, k1);
    cull[0] = k0;
    cull[1] = k1;
  }
}

// Tile counts of the compositor's lists: a splat whose bbox spans at most
// kTileCullMax tiles keeps only the tiles tile_cull_test keeps (k_duplicate
// emits exactly those bits).  A separate, fully occupied
// pass after the float64 preprocess (inside it the loop over tiles cost the
// latency-bound preprocess 0.09 ms at config 2).
__global__ void __launch_bounds__(256) k_tile_counts(const SplatRec *__restrict__ recs,
                                                     const float4 *__restrict__ cull2d, int64_t n,
                                                     uint32_t *__restrict__ counts, uint32_t *__restrict__ keep) {
  pdl_wait();  // launched right behind the preprocess (no early trigger there)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t nt = counts[i];  // bbox tiles (0: culled or off screen)
    if (nt <= 1u || nt > (uint32_t)kTileCullMax) continue;  // one tile: the compositor's warp cull suffices
    const SplatRec *gp = recs + i;
    SplatRec r;
    r.r0 = __ldg(&gp->r0); r.r1 = __ldg(&gp->r1); r.r4 = __ldg(&gp->r4); r.r5 = __ldg(&gp->r5);
    r.r2 = r.r3 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 c2[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    if (!rec_is3d(r)) {
      c2[0] = __ldg(cull2d + 2 * (size_t)i);
      c2[1] = __ldg(cull2d + 2 * (size_t)i + 1);
    }
    const int4 q = r.r5;
    const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16), x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
    // the splat's side of cull_rect, once (tile_culled per tile repeats it)
    const TileCull tc = tile_cull_prep(r, c2);
    uint32_t bits = 0, b = 1;  // bit j: the j-th bbox tile (row-major) is kept
    for (int ty = y0 / kTile; ty <= y1 / kTile; ++ty)
      for (int tx = x0 / kTile; tx <= x1 / kTile; ++tx, b <<= 1)
        if (!tile_cull_test(tc, max(tx * kTile, x0), max(ty * kTile, y0), min(tx * kTile + kTile - 1, x1),
                            min(ty * kTile + kTile - 1, y1)))
          bits |= b;
    counts[i] = (uint32_t)__popc(bits);
    keep[i] = bits;
  }
}

// Inverse depth permutation over all n sorted slots: culled Gaussians (keys
// ~0, sorted after the m kept ones) get rank 0xffffffff.
// Inverse of the depth permutation.  The sorted indices are in buffer
// (sort_np & 1) of the ping-pong pair; M = the near-culled count, both from
// the frame state (no host round trip).
__global__ void k_rank_scatter(const uint32_t *__restrict__ vals_a, const uint32_t *__restrict__ vals_b,
                               const FrameState *__restrict__ st, int64_t n, uint32_t *__restrict__ rank_of,
                               uint32_t *__restrict__ order) {
  if (HGS_DEPTH_SORT_TRIGGER) pdl_launch_dependents();
  pdl_wait();
  const uint32_t *sorted_idx = (st->sort_np & 1u) ? vals_b : vals_a;
  const int64_t m = st->m_count;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t g = sorted_idx[r];
    rank_of[g] = r < m ? (uint32_t)r : 0xffffffffu;
    order[r] = g;  // the depth order in a fixed buffer (rank -> Gaussian)
  }
}

// Depth-sort plan from the fused digit histograms (k_depth_keys): per digit
// the exclusive offsets (k_radix_offsets) and whether every key has the same
// digit (that pass is skipped); the non-constant digits, low to high, become
// the device-side pass list the onesweep passes read.
__global__ void k_sort_plan(const uint32_t *__restrict__ hist, int64_t n, uint32_t *__restrict__ offsets,
                            FrameState *__restrict__ st) {
  if (HGS_DEPTH_SORT_TRIGGER) pdl_launch_dependents();
  pdl_wait();
  __shared__ uint32_t s[kRadix];
  __shared__ int s_trivial[8];
  const int t = threadIdx.x;
  for (int p = 0; p < 8; ++p) {
    const uint32_t h = hist[p * kRadix + t];
    const int triv = __syncthreads_or(h == (uint32_t)n);
    s[t] = h;
    __syncthreads();
    for (int d = 1; d < kRadix; d <<= 1) {
      const uint32_t v = t >= d ? s[t - d] : 0u;
      __syncthreads();
      s[t] += v;
      __syncthreads();
    }
    offsets[p * kRadix + t] = s[t] - h;
    if (t == 0) s_trivial[p] = triv;
    __syncthreads();
  }
  if (t == 0) {
    uint32_t np = 0;
    for (int p = 0; p < 8; ++p)
      if (!s_trivial[p]) st->sort_digit[np++] = (uint32_t)p;
    st->sort_np = np;
  }
}

// One thread per Gaussian in index order, one warp per CTA and 32 consecutive
// Gaussians per warp step: the SH rows (3B floats each) are staged through
// shared memory as one coalesced segment (per-thread strided rows were
// LSU-throttled); float64 projection; record + tile count written at the
// Gaussian's index.  Independent of the depth sort (it runs beside it); the
// culls are k_depth_keys' (kept[]), a culled Gaussian gets count 0.
template <int B, bool G64>
__global__ void __launch_bounds__(32, HGS_PRE_MINB) k_preprocess(SceneView sc, CamD cam, ModD mod,
                                                   const uint8_t *__restrict__ kept,
                                                   SplatRec *__restrict__ recs, Rec64 *__restrict__ recs64,
                                                   float4 *__restrict__ cull2d, float2 *__restrict__ eig,
                                                   uint32_t *__restrict__ counts) {
  constexpr int SB = 3 * B, SS = 3 * B + 1;
  const int lane = threadIdx.x;
#if HGS_PRE_ASYNC
  // double-buffered SH staging: the next warp step's rows are in flight
  // (cp.async, no registers) while this step's float64 projection runs
  __shared__ float s_buf[2][32 * SS];
  const int64_t stride = (int64_t)gridDim.x * 32;
  auto stage = [&](int64_t b0, float *dst) {
    const int c = (int)(sc.n - b0 < 32 ? sc.n - b0 : 32);
    const float *src = sc.sh + b0 * SB;
    for (int e = lane; e < c * SB; e += 32) {
      const int r = e / SB;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + r * SS + (e - r * SB));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src + e) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  if ((int64_t)blockIdx.x * 32 < sc.n) stage((int64_t)blockIdx.x * 32, s_buf[0]);
  for (int64_t base = (int64_t)blockIdx.x * 32; base < sc.n; base += stride) {
    const int cnt = (int)(sc.n - base < 32 ? sc.n - base : 32);
    __syncwarp();  // every lane is done with the buffer the next copy overwrites
    if (base + stride < sc.n) {
      stage(base + stride, s_buf[buf ^ 1]);
#if HGS_PRE_PREFETCH
      {  // the next step's scalar fields into L1: 13 lines, one per lane
        const int64_t nb = base + stride;
        const char *ptr = nullptr;
        if (lane < 3) ptr = reinterpret_cast<const char *>(sc.center + 3 * nb) + 128 * lane;
        else if (lane < 6) ptr = reinterpret_cast<const char *>(sc.log_scale + 3 * nb) + 128 * (lane - 3);
        else if (lane < 10) ptr = reinterpret_cast<const char *>(sc.rotation + 4 * nb) + 128 * (lane - 6);
        else if (lane == 10) ptr = reinterpret_cast<const char *>(sc.opacity_logit + nb);
        else if (lane == 11) ptr = reinterpret_cast<const char *>(sc.type_spec + nb);
        if (ptr) asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
      }
#endif
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const float *s_sh = s_buf[buf];
    buf ^= 1;
#else
  __shared__ float s_sh[32 * SS];
  for (int64_t base = (int64_t)blockIdx.x * 32; base < sc.n; base += (int64_t)gridDim.x * 32) {
    const int cnt = (int)(sc.n - base < 32 ? sc.n - base : 32);
    __syncwarp();
    for (int e = lane; e < cnt * SB; e += 32) {
      const int r = e / SB;
      s_sh[r * SS + (e - r * SB)] = __ldg(sc.sh + base * SB + e);
    }
    __syncwarp();
#endif
    const int64_t i = base + lane;
    if (lane >= cnt) continue;
    // the culls k_depth_keys decided: z <= near (project.py:182), |q| <= 1e-8, singular 3D conic (:225)
    if (!kept[i]) {
      counts[i] = 0u;
      continue;
    }
    ProjD o;
    project_d<false, false, G64>(sc, i, cam, mod, o, s_sh + lane * SS);
    bbox_d(o, cam.width, cam.height);
    write_record(o, (uint32_t)i, cam.width, cam.height, recs + i, cull2d + 2 * (size_t)i, eig + i);
    write_rec64(o, recs64 + i);
    counts[i] = tile_count_of(o.bbox);  // bbox tiles; k_tile_counts culls them
  }
}
// Host launcher (the template is launched from this translation unit).
cudaError_t launch_preprocess(const SceneView &sc, const CamD &cam, const ModD &mod, const uint8_t *kept,
                              SplatRec *recs, Rec64 *recs64, float4 *cull2d, float2 *eig, uint32_t *counts,
                              cudaStream_t s) {
  const int64_t nb = (sc.n + 31) / 32;
  // one warp per CTA; HGS_PRE_CTAS CTAs per SM at most (grid-stride): fewer
  // than fit leaves registers for the depth sort running beside it
  const int64_t cap = 148LL * HGS_PRE_CTAS;
  const int g = (int)(nb < 1 ? 1 : (nb > cap ? cap : nb));
#define HGS_PRE(B_)                                                                                \
  (sc.center64 ? k_preprocess<B_, true><<<g, 32, 0, s>>>(sc, cam, mod, kept, recs, recs64, cull2d, eig, counts) \
               : k_preprocess<B_, false><<<g, 32, 0, s>>>(sc, cam, mod, kept, recs, recs64, cull2d, eig, counts))
  switch (sc.sh_bases) {
    case 1: HGS_PRE(1); break;
    case 4: HGS_PRE(4); break;
    case 9: HGS_PRE(9); break;
    default: HGS_PRE(16); break;
  }
#undef HGS_PRE
  return cudaGetLastError();
}

// Exclusive scan of the per-rank tile counts into pair offsets (decoupled
// look-back, kScanItems counts per thread); the last tile writes K.
// m < 0: M from the frame state.  cap >= 0: a total above it sets the
// frame's status to HGS_ERR_PAIR_CAPACITY (the pair buffer is too small).
__global__ void __launch_bounds__(kScanThreads) k_scan_counts(const uint32_t *__restrict__ counts,
                                                              const uint32_t *__restrict__ order, int64_t m,
                                                              unsigned long long *__restrict__ pair_off,
                                                              unsigned long long *__restrict__ scan_lb,
                                                              FrameState *__restrict__ st, int64_t cap) {
  pdl_launch_dependents();  // k_duplicate may be scheduled as this grid drains
  pdl_wait();
  __shared__ uint32_t s_tile;
  if (m < 0) m = st->m_count;
  if ((int64_t)blockIdx.x * kScanTile >= m) return;  // launched for N, not for M
  __shared__ unsigned long long s_warp[32];
  __shared__ unsigned long long s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(&st->tile_counters[0], 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t c[kScanItems];
  unsigned long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    c[k] = base + k < m ? counts[order ? order[base + k] : base + k] : 0u;  // order: counts by Gaussian
    sum += c[k];
  }
  unsigned long long total;
  const unsigned long long ex = block_exclusive_scan_u64(sum, s_warp, total);
  if (threadIdx.x == 0) s_excl = scan_lookback(scan_lb, tile, total);
  __syncthreads();
  unsigned long long run = s_excl + ex;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < m) pair_off[base + k] = run;
    run += c[k];
  }
  if ((int64_t)(tile + 1) * kScanTile >= m && threadIdx.x == 0) {
    st->k_total = s_excl + total;
    if (cap >= 0 && (int64_t)(s_excl + total) > cap) atomicCAS(&st->status, 0u, (uint32_t)HGS_ERR_PAIR_CAPACITY);
  }
}

// ------------------------------------------------------------ duplicate
// Emit (tile id, rank) pairs in rank order at the scanned offsets and build
// the tile-id digit histograms for the pair sort.  A lane emits the pairs of
// its own splat when it has at most kDupOwn of them; the warp emits the
// pairs of larger splats together, one splat at a time (a full-screen 2D
// surfel has 8160 pairs at 1080p: one thread looping over them was the
// kernel's whole duration).
constexpr int kDupOwn = 32;

// order: rank -> Gaussian (records are by Gaussian); the pair value is the
// Gaussian index, or the rank with emit_rank (the SplatFrame export's slots).
// tile_cull (the compositor's lists, 16 x 16 tiles): splats with 2 ..
// kTileCullMax bbox tiles emit only the tiles of their k_tile_counts keep
// mask (the counts the scan used are its popcounts).
__global__ void __launch_bounds__(256) k_duplicate(const SplatRec *__restrict__ recs,
                                                   const uint32_t *__restrict__ order,
                                                   const unsigned long long *__restrict__ pair_off, int64_t m,
                                                   const FrameState *__restrict__ st, int tiles_x, int tile_shift,
                                                   bool emit_rank, bool tile_cull, const uint32_t *__restrict__ keep,
                                                   uint32_t *__restrict__ pkeys, uint32_t *__restrict__ pvals,
                                                   int n_digits, uint32_t *__restrict__ hist) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ uint32_t sh[2 * kRadix];
  if (m < 0) {  // M and the capacity verdict from the frame state
    if (st->status) return;
    m = st->m_count;
  }
  for (int i = threadIdx.x; i < 2 * kRadix; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto emit = [&](uint32_t t, unsigned long long o, uint32_t r) {
    pkeys[o] = t;
    pvals[o] = r;
    atomicAdd(&sh[t & 0xff], 1u);
    if (n_digits > 1) atomicAdd(&sh[kRadix + ((t >> 8) & 0xff)], 1u);
  };
  // warp-aligned grid stride: the loop condition is warp-uniform
  for (int64_t r0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); r0 < m; r0 += stride) {
    const int64_t r = r0 + lane;
    int tx0 = 0, ty0 = 0, bw = 1;
    uint32_t cnt = 0;
    unsigned long long o = 0;
    uint32_t val = 0, g = 0;
    int4 q = make_int4(0, 0, 0, 0);
    if (r < m) {
      g = order[r];
      val = emit_rank ? (uint32_t)r : g;
      q = recs[g].r5;
      const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16), x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
      if (x1 >= x0) {
        tx0 = x0 >> tile_shift; ty0 = y0 >> tile_shift;
        bw = (x1 >> tile_shift) - tx0 + 1;
        cnt = (uint32_t)(bw * ((y1 >> tile_shift) - ty0 + 1));
        o = pair_off[r];
      }
    }
    static_assert(kTileCullMax <= kDupOwn, "culled splats take the per-lane path");
    if (cnt <= (uint32_t)kDupOwn) {
      const uint32_t bits = (tile_cull && cnt > 1u) ? __ldg(keep + g) : 0xffffffffu;  // the k_tile_counts rule
      uint32_t k = 0;
      for (uint32_t j = 0, dy = 0, dx = 0; j < cnt; ++j) {  // row-major over the tile rectangle
        if ((bits >> j) & 1u) emit((uint32_t)((ty0 + (int)dy) * tiles_x + tx0 + (int)dx), o + k++, val);
        if (++dx == (uint32_t)bw) { dx = 0; ++dy; }
      }
    }
    uint32_t big = __ballot_sync(0xffffffffu, cnt > (uint32_t)kDupOwn);
    while (big) {
      const int l = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t c = __shfl_sync(0xffffffffu, cnt, l);
      const unsigned long long ob = __shfl_sync(0xffffffffu, o, l);
      const int bx = __shfl_sync(0xffffffffu, tx0, l), by = __shfl_sync(0xffffffffu, ty0, l);
      const int w = __shfl_sync(0xffffffffu, bw, l);
      const uint32_t v = __shfl_sync(0xffffffffu, val, l);
      for (uint32_t j = lane; j < c; j += 32) {
        const uint32_t dy = j / (uint32_t)w, dx = j - dy * (uint32_t)w;
        emit((uint32_t)((by + (int)dy) * tiles_x + bx + (int)dx), ob + j, v);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_digits * kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Tiles per splat at another tile size (2^tile_shift px; SplatFrame export at
// settings.tile_size != 16, project.py:329-343).
__global__ void __launch_bounds__(256) k_rebin_counts(const SplatRec *__restrict__ recs,
                                                      const uint32_t *__restrict__ order, int64_t m, int tile_shift,
                                                      uint32_t *__restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int4 q = recs[order[r]].r5;
    const int x0 = q.x & 0xffff, y0 = (int)((uint32_t)q.x >> 16), x1 = q.y & 0xffff, y1 = (int)((uint32_t)q.y >> 16);
    counts[r] = x1 >= x0 ? (uint32_t)(((x1 >> tile_shift) - (x0 >> tile_shift) + 1) *
                                      ((y1 >> tile_shift) - (y0 >> tile_shift) + 1))
                         : 0u;
  }
}

// tile_offsets (n_tiles + 1) from the tile-sorted keys (project.py:344-345).
// Four keys per thread (one 16-byte load), grid-stride.
__global__ void __launch_bounds__(256) k_tile_ranges(const uint32_t *__restrict__ skeys, int64_t k,
                                                     const FrameState *__restrict__ st, int64_t n_tiles,
                                                     uint32_t *__restrict__ tile_off) {
  pdl_launch_dependents();
  pdl_wait();
  if (k < 0) {  // K from the frame state
    if (st->status) return;
    k = (int64_t)st->k_total;
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) {
    for (int64_t t = tid; t <= n_tiles; t += stride) tile_off[t] = 0;
    return;
  }
  const bool vec = ((uintptr_t)skeys & 15u) == 0;
  for (int64_t p0 = tid * 4; p0 < k; p0 += stride * 4) {
    uint32_t v[4];
    if (vec && p0 + 4 <= k) {
      const uint4 q = *reinterpret_cast<const uint4 *>(skeys + p0);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = p0 + i < k ? skeys[p0 + i] : 0u;
    }
    int64_t prev = p0 ? (int64_t)skeys[p0 - 1] : -1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t p = p0 + i;
      if (p >= k) break;
      const int64_t t = v[i];
      for (int64_t tt = prev + 1; tt <= t; ++tt) tile_off[tt] = (uint32_t)p;
      if (p == k - 1)
        for (int64_t tt = t + 1; tt <= n_tiles; ++tt) tile_off[tt] = (uint32_t)k;
      prev = t;
    }
  }
}

// -------------------------------------------------------------- composite



}  // namespace hgs
