// hgs_composite_fwd.cu -- the front-to-back compositor (raster/_blend_py.py:76-117).
//
//  k_composite_fwd : the hot kernel.  No function calls: every decision is a
//                    float32 decision with an error bound; a lane whose next
//                    decision is ambiguous saves its state to the FwdFix
//                    worklist and retires (deferred exactness).
//  k_fixup_fwd     : one warp per deferred pixel resumes the walk with the
//                    float64-exact decisions, 32 tile-list entries at a time
//                    (lane-parallel evaluation, product scan for T).
#include "hgs_kernels.cuh"

#ifndef HGS_FWD_PIN_SA
#define HGS_FWD_PIN_SA 1
#endif
#ifndef HGS_FWD_ONE_DEFER
#define HGS_FWD_ONE_DEFER 1
#endif
#ifndef HGS_FWD_MINB
#define HGS_FWD_MINB 4  // CTAs per SM the hot compositor is register-budgeted for
#endif
#ifndef HGS_FWD_PF
#define HGS_FWD_PF 0  // 1, 2: tiled forward stages the next chunk's records with cp.async while walking this one (measured slower)
#endif

namespace hgs {

// One CTA per 16 x 16 tile, one thread per pixel, warps own 8 x 4 pixel blocks
// and run independently (no block barriers): a warp walks its tile list in
// chunks of 32 entries; lane l loads entry l's rank and bbox and turns the
// bbox into a 32-bit mask of the warp's pixels it covers (the reference's
// inclusive bbox test, _blend_py.py:89-91); records of relevant entries are
// staged in the warp's slice of shared memory and walked in order.  Every
// lane sees the same splat, so the 2D / 3D branch is warp-uniform; a warp
// retires as soon as its 32 pixels are saturated or deferred.
// 16-byte asynchronous global -> shared copy (L1-allocating: the 8 warps of
// a tile read the same records) and its group fences.
__device__ __forceinline__ void cp_async16(uint32_t dst_sa, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst_sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// PF (tiled frames only): software-pipelined staging.  The records of chunk
// c + 1 are copied into the warp's second staging buffer with cp.async while
// chunk c is walked, and the tile-list ranks two chunks ahead are loaded into
// a register -- the rank -> record -> bbox gather chain (two dependent L2
// round trips per chunk) leaves the critical path.  Every entry of the chunk
// is copied (the bbox test needs the record), the culls then run on the
// shared-memory copy.
template <bool NAIVE, bool COUNT, int PF, bool EXACT>
__global__ void __launch_bounds__(kBlock, HGS_FWD_MINB) k_composite_fwd(CompositeArgs a) {
  pdl_launch_dependents();  // k_fixup_fwd may be scheduled into the tail of this grid
  pdl_wait();
  __shared__ SplatRec s_rec[PF ? 2 : 1][kBlock / 32][32];
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wx0 = tx * kTile + (warp & 1) * 8, wy0 = ty * kTile + (warp >> 1) * 4;
  const int ix = wx0 + (lane & 7), iy = wy0 + (lane >> 3);
  const bool inside = ix < a.width && iy < a.height;
  const uint32_t lane_bit = 1u << lane;
  const float lox = (float)(lane & 7), loy = (float)(lane >> 3);  // offset in the warp block
  constexpr bool exact = HGS_EXACT_ENABLED && EXACT;  // HGS_FLAG_FAST: the EXACT = false instantiation
  const bool stress = COUNT && !NAIVE && (a.flags & HGS_FLAG_DEFER_ALL);
  if (a.st->status) return;  // failed frame (bad parameters / pair capacity): nothing to composite
  uint32_t lo, hi;
  if (NAIVE) {
    lo = 0;
    hi = a.st->m_count;
  } else {
    lo = a.tile_off[tile];
    hi = a.tile_off[tile + 1];
  }
  const uint32_t pix = (uint32_t)iy * (uint32_t)a.width + (uint32_t)ix;
  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f, dep = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f;
  uint32_t cnt = 0, last = 0;
  bool done = !inside, deferred = false;
  uint32_t n_ev3 = 0, n_ev2 = 0, n_c3 = 0, n_c2 = 0;  // HGS_FLAG_COUNT
  SplatRec *wrec = s_rec[0][warp];
#if HGS_FWD_PIN_SA
  uint32_t wrec_sa = (uint32_t)__cvta_generic_to_shared(wrec);
  asm volatile("mov.u32 %0, %0;" : "+r"(wrec_sa));  // opaque: kept, not re-derived per splat
#endif
  // PF: rk_c / rk_n / rk_nn = tile-list ranks of chunks c, c + 1, c + 2 of
  // this lane's entry; q_n = the bbox word (r5) of chunk c + 1's entry
  // (PF == 2: only entries whose bbox meets the warp block are copied)
  constexpr uint32_t kNoRank = 0xffffffffu;
  constexpr uint32_t kBufBytes = (uint32_t)(kBlock / 32) * 32u * (uint32_t)sizeof(SplatRec);
  uint32_t rk_c = kNoRank, rk_n = kNoRank, rk_nn = kNoRank, slot_sa = 0u;
  int4 q_n = make_int4(0, -1, 0, 0);
  bool staged = false;  // this lane's entry of the chunk about to be walked was copied
  auto stage_async = [&](uint32_t dst_sa, uint32_t rk) {
    const char *src = reinterpret_cast<const char *>(a.recs + rk);
#pragma unroll
    for (int k = 0; k < 6; ++k) cp_async16(dst_sa + 16u * k, src + 16 * k);
  };
  auto rank_at = [&](uint32_t e) { return e < hi ? __ldg(a.tile_vals + e) : kNoRank; };
  if (PF) {
    slot_sa = (uint32_t)__cvta_generic_to_shared(&s_rec[0][warp][lane]);
    rk_c = rank_at(lo + lane);
    rk_n = rank_at(lo + 32u + lane);
    staged = rk_c != kNoRank && (PF == 1 || pixel_mask(__ldg(&a.recs[rk_c].r5), wx0, wy0));
    if (staged) stage_async(slot_sa, rk_c);
    cp_async_commit();
    if (PF == 2 && rk_n != kNoRank) q_n = __ldg(&a.recs[rk_n].r5);
    rk_nn = rank_at(lo + 64u + lane);
  }
  uint32_t buf = 0u;

  // last: one past the last contributor (tile-list position relative to lo);
  // kept per chunk from the chunk's contribution mask cm, not per pair
  auto defer = [&](uint32_t entry, uint32_t mode, uint32_t last_now) {
    FwdFix f;
    f.pix = pix; f.entry = entry; f.mode = mode; f.cnt = cnt; f.last = last_now;
    f.T = T; f.c0 = cr; f.c1 = cg; f.c2 = cb; f.dep = dep; f.n0 = n0; f.n1 = n1; f.n2 = n2;
    f.pad[0] = f.pad[1] = f.pad[2] = 0;
    a.fwd_fix[atomicAdd(&a.st->n_fix_fwd, 1u)] = f;
    deferred = true;
    done = true;
  };

  for (uint32_t base = lo; base < hi; base += 32) {
    // pixels still compositing (saturated / deferred ones drop out of the masks)
    const uint32_t alive = __ballot_sync(0xffffffffu, !done);
    if (!alive) break;
    // stage: rank + bbox of entry base + lane, pixel mask, record if relevant
    const uint32_t j = base + lane;
    uint32_t pm = 0u;
    if (PF) {
      // copies of chunk c + 1 into the other buffer (its last reader, the
      // walk of chunk c - 1, finished at that walk's closing __syncwarp)
      const uint32_t nb = buf ^ 1u;
      const bool staged_c = staged;
      staged = rk_n != kNoRank && (PF == 1 || pixel_mask(q_n, wx0, wy0));
      if (staged) stage_async(slot_sa + nb * kBufBytes, rk_n);
      cp_async_commit();
      // the pipeline's loads for chunk c + 2 (consumed next iteration)
      if (PF == 2) q_n = rk_nn != kNoRank ? __ldg(&a.recs[rk_nn].r5) : make_int4(0, -1, 0, 0);
      const uint32_t rk = rk_c;
      rk_c = rk_n;
      rk_n = rk_nn;
      rk_nn = rank_at(base + 96u + lane);
      cp_async_wait<1>();  // this lane's copies of chunk c have landed
      wrec = s_rec[buf][warp];
#if HGS_FWD_PIN_SA
      wrec_sa = (uint32_t)__cvta_generic_to_shared(wrec);
      asm volatile("mov.u32 %0, %0;" : "+r"(wrec_sa));
#endif
      if (staged_c) {
        SplatRec &sr = wrec[lane];
        const int4 q = sr.r5;
        pm = pixel_mask(q, wx0, wy0);  // PF == 2: copied iff nonzero
        if (pm) {
          SplatRec r;
          r.r0 = sr.r0; r.r1 = sr.r1; r.r2 = sr.r2; r.r3 = sr.r3; r.r4 = sr.r4; r.r5 = q;
          if (HGS_CULL_PRE ? cull_splat_pre(r, a.cull2d + 2 * (size_t)rk, pm, wx0, wy0) : cull_splat(r, pm, wx0, wy0))
            pm = 0u;
          pm &= alive;
          if (pm && HGS_STAGED_ORIGIN) {
            stage_block_origin(r, wx0, wy0);
            sr.r5 = r.r5;
          }
        }
      }
      buf ^= 1u;
    } else if (j < hi) {
      const uint32_t rk = __ldg(a.tile_vals + j);  // NAIVE: the depth order
      const SplatRec *g = a.recs + rk;
      const int4 q = __ldg(&g->r5);
      pm = NAIVE ? 0xffffffffu : pixel_mask(q, wx0, wy0);  // a rectangle: the culls rely on it
      if (pm) {
        SplatRec r;
        r.r0 = __ldg(&g->r0); r.r1 = __ldg(&g->r1); r.r2 = __ldg(&g->r2);
        r.r3 = __ldg(&g->r3); r.r4 = __ldg(&g->r4); r.r5 = q;
        if (!NAIVE && (HGS_CULL_PRE ? cull_splat_pre(r, a.cull2d + 2 * (size_t)rk, pm, wx0, wy0)
                                    : cull_splat(r, pm, wx0, wy0)))
          pm = 0u;  // bbox hit, but the 1/255 support misses every covered pixel
        pm &= alive;  // only pixels still compositing
        if (HGS_STAGED_ORIGIN && !NAIVE) stage_block_origin(r, wx0, wy0);
        if (pm) wrec[lane] = r;
      }
    }
    uint32_t rel = __ballot_sync(0xffffffffu, pm != 0u);
    __syncwarp();
    const bool walking = !done;  // this chunk's mask word is written iff the pixel walks it
    uint32_t cm = 0u;
    while (rel) {
      const int e = __ffs(rel) - 1;
      rel &= rel - 1;
      const uint32_t m = __shfl_sync(0xffffffffu, pm, e);
      if (done || !(m & lane_bit)) continue;
#if HGS_FWD_PIN_SA
      SplatRec r;
      {
        const uint32_t ra = wrec_sa + (uint32_t)e * (uint32_t)sizeof(SplatRec);
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.r0.x), "=f"(r.r0.y), "=f"(r.r0.z), "=f"(r.r0.w) : "r"(ra));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+16];" : "=f"(r.r1.x), "=f"(r.r1.y), "=f"(r.r1.z), "=f"(r.r1.w) : "r"(ra));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+32];" : "=f"(r.r2.x), "=f"(r.r2.y), "=f"(r.r2.z), "=f"(r.r2.w) : "r"(ra));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+48];" : "=f"(r.r3.x), "=f"(r.r3.y), "=f"(r.r3.z), "=f"(r.r3.w) : "r"(ra));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+64];" : "=f"(r.r4.x), "=f"(r.r4.y), "=f"(r.r4.z), "=f"(r.r4.w) : "r"(ra));
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+80];" : "=r"(r.r5.x), "=r"(r.r5.y), "=r"(r.r5.z), "=r"(r.r5.w) : "r"(ra));
      }
#else
      const SplatRec &r = wrec[e];
#endif
      const bool is3d = rec_is3d(r);
      if (COUNT) (is3d ? n_ev3 : n_ev2) += 1;
      PairEval p;
      const int c = (HGS_STAGED_ORIGIN && !NAIVE)
                        ? eval_fast<false, false, true, EXACT ? 1 : 0>(r, ix, iy, a.flags, p, lox, loy)
                        : eval_fast<false, false, false, EXACT ? 1 : 0>(r, ix, iy, a.flags, p);
      if (c == kSkip) continue;
#if HGS_FWD_ONE_DEFER
      // one deferral site (the pair's decision or the early-stop decision), so
      // the worklist address is formed only on that rare path
      uint32_t dmode = 2u;
      // HGS_FLAG_DEFER_ALL (tests, counting instantiation only): every pixel is
      // deferred at its first contribution, even pixels before it (mode 0),
      // odd pixels after it (mode 1), so the whole image goes through k_fixup_fwd
      if (c == kAmbiguous || (stress && last == 0u && cm == 0u && !(pix & 1u))) {
        if (COUNT && c == kAmbiguous) atomicAdd(&a.st->diag[is3d ? 12 : 13], 1ull);  // deferral reasons
        dmode = 0u;
      } else {
        if (stress && last == 0u && cm == 0u) dmode = 1u;
#else
      if (c == kAmbiguous) {
        if (COUNT) atomicAdd(&a.st->diag[is3d ? 12 : 13], 1ull);  // deferral reasons
        defer(base + e, 0u, cm ? base - lo + 32u - (uint32_t)__clz(cm) : last);
        continue;
      }
      {
#endif
        if (COUNT) (is3d ? n_c3 : n_c2) += 1;
        const float at = p.at;
        const float w = at * T;
        const float4 c3 = r.r3, c4 = r.r4;
        cr = fmaf(w, c3.y, cr);
        cg = fmaf(w, c3.z, cg);
        cb = fmaf(w, c3.w, cb);
        dep = fmaf(w, r.r0.z, dep);
        n0 = fmaf(w, c4.x, n0);
        n1 = fmaf(w, c4.y, n1);
        n2 = fmaf(w, c4.z, n2);
        if (NAIVE) ++cnt;  // tiled frames derive the blend-log counts from the masks
        cm |= 1u << e;
        T = T * (1.f - at);
        // early stop T < 1e-4 (_blend_py.py:111-113); near the threshold the
        // decision is deferred to the float64 transmittance replay.  One
        // compare on the common path (T well above the threshold).
        if (T <= (float)kEarlyStopT * (1.f + 2e-5f)) {
          if (exact && T >= (float)kEarlyStopT * (1.f - 2e-5f)) {
            if (COUNT) atomicAdd(&a.st->diag[14], 1ull);
#if HGS_FWD_ONE_DEFER
            dmode = 1u;
#else
            defer(base + e, 1u, cm ? base - lo + 32u - (uint32_t)__clz(cm) : last);
#endif
          }
          else if (T < (float)kEarlyStopT)
            done = true;
        }
      }
#if HGS_FWD_ONE_DEFER
      if (dmode != 2u) defer(base + e, dmode, cm ? base - lo + 32u - (uint32_t)__clz(cm) : last);
#endif
    }
    if (cm) last = base - lo + 32u - (uint32_t)__clz(cm);
    if (!NAIVE && walking)
      a.pix_mask[mask_word(lo, tile, (base - lo) >> 5, (uint32_t)((iy & (kTile - 1)) * kTile + (ix & (kTile - 1))))] = cm;
    __syncwarp();  // the next chunk overwrites this warp's staging slots
  }
  if (COUNT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n_ev3 += __shfl_xor_sync(0xffffffffu, n_ev3, o);
      n_ev2 += __shfl_xor_sync(0xffffffffu, n_ev2, o);
      n_c3 += __shfl_xor_sync(0xffffffffu, n_c3, o);
      n_c2 += __shfl_xor_sync(0xffffffffu, n_c2, o);
    }
    if (lane == 0) {
      atomicAdd(&a.st->diag[2], (unsigned long long)n_ev3);
      atomicAdd(&a.st->diag[3], (unsigned long long)n_ev2);
      atomicAdd(&a.st->diag[4], (unsigned long long)n_c3);
      atomicAdd(&a.st->diag[5], (unsigned long long)n_c2);
    }
  }
  if (PF) cp_async_wait<0>();  // no copy may still target this CTA's shared memory
  if (!inside || deferred) return;  // deferred pixels are written by k_fixup_fwd
  a.color[3 * pix + 0] = cr + a.bg[0] * T;
  a.color[3 * pix + 1] = cg + a.bg[1] * T;
  a.color[3 * pix + 2] = cb + a.bg[2] * T;
  a.depth[pix] = dep;
  a.trans[pix] = T;
  if (a.alpha) a.alpha[pix] = 1.f - T;
  if (a.normal) {
    a.normal[3 * pix + 0] = n0;
    a.normal[3 * pix + 1] = n1;
    a.normal[3 * pix + 2] = n2;
  }
  a.pix_T[pix] = T;
  a.pix_last[pix] = last;
  if (NAIVE) a.pix_count[pix] = cnt;
}

cudaError_t launch_composite_fwd(const CompositeArgs &a, int64_t n_tiles, bool naive, bool count, cudaStream_t s) {
  constexpr int PF = HGS_FWD_PF;
  const bool fast = a.flags & HGS_FLAG_FAST;
#define HGS_FWD_LAUNCH(NV, CT, P)                                                           \
  (fast ? launch_pdl(k_composite_fwd<NV, CT, P, false>, dim3((unsigned)n_tiles), dim3(kBlock), 0, s, a) \
        : launch_pdl(k_composite_fwd<NV, CT, P, true>, dim3((unsigned)n_tiles), dim3(kBlock), 0, s, a))
  if (naive && count) HGS_FWD_LAUNCH(true, true, 0);
  else if (naive) HGS_FWD_LAUNCH(true, false, 0);
  else if (count) HGS_FWD_LAUNCH(false, true, PF);
  else HGS_FWD_LAUNCH(false, false, PF);
#undef HGS_FWD_LAUNCH
  return cudaGetLastError();
}

// Blend-log entry count per pixel of a tiled frame: the popcount of its
// contribution-mask words up to its last contributor.
__global__ void k_pixel_counts(CompositeArgs a, uint32_t *counts) {
  const int64_t HW = (int64_t)a.width * a.height;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < HW; p += (int64_t)gridDim.x * blockDim.x) {
    const int ix = (int)(p % a.width), iy = (int)(p / a.width);
    const int tile = (iy / kTile) * a.tiles_x + ix / kTile;
    const uint32_t lo = a.tile_off[tile], last = a.pix_last[p];
    const uint32_t pit = (uint32_t)((iy & (kTile - 1)) * kTile + (ix & (kTile - 1)));
    uint32_t c = 0;
    for (uint32_t ch = 0; (ch << 5) < last; ++ch) {
      uint32_t w = a.pix_mask[mask_word(lo, tile, ch, pit)];
      const uint32_t rem = last - (ch << 5);
      if (rem < 32u) w &= (1u << rem) - 1u;
      c += __popc(w);
    }
    counts[p] = c;
  }
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

#ifndef HGS_FIXUP_E
#define HGS_FIXUP_E 4  // tile-list entries per lane per window of k_fixup_fwd
#endif

// Deferred pixels, one warp each (grid-stride over the worklist).  The warp
// evaluates a window of 32 x E consecutive tile-list entries in parallel with
// the exact decisions (float64 re-evaluation where the float32 bound is
// ambiguous): lane l owns entries E l .. E l + E - 1 of the window, forms
// their transmittance with a lane-local product and a warp product scan,
// resolves the early stop in entry order (float64 replay near the
// threshold) and accumulates lane-local partial sums, reduced once at the
// end.  Windows are aligned to the forward's 32-entry chunks, so each window
// writes E whole contribution-mask words.  The walk of a pixel is a serial
// chain of windows (the kernel's duration is the longest one): E entries per
// lane make it E times shorter.
__global__ void __launch_bounds__(256, HGS_FIXUP_MINB) k_fixup_fwd(CompositeArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int E = HGS_FIXUP_E;
  constexpr uint32_t WIN = 32u * E;
  constexpr int LPC = 32 / E;  // lanes per 32-entry chunk
  static_assert(E == 1 || E == 2 || E == 4, "E divides 32");
  const uint32_t nfix = a.st->n_fix_fwd;
  const int lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const bool naive = a.flags & HGS_FLAG_NAIVE;
  const float thr = (float)kEarlyStopT;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nfix; w += nw) {
    const FwdFix f = a.fwd_fix[w];
    const int ix = (int)(f.pix % (uint32_t)a.width), iy = (int)(f.pix / (uint32_t)a.width);
    const int tile = (iy / kTile) * a.tiles_x + ix / kTile;
    const uint32_t lo = naive ? 0u : a.tile_off[tile];
    const uint32_t hi = naive ? a.st->m_count : a.tile_off[tile + 1];
    float T = f.T;
    float q0 = 0.f, q1 = 0.f, q2 = 0.f, qd = 0.f, qn0 = 0.f, qn1 = 0.f, qn2 = 0.f;  // lane partial sums
    uint32_t cnt = f.cnt, last = f.last;
    bool stopped = false;
    uint32_t start = f.entry;
    if (f.mode == 1u) {  // warp-cooperative float64 replay of the transmittance
      stopped = replay_T_below(a.recs, a.tile_vals, a.flags, a.st, lo, f.entry, ix, iy);
      start = f.entry + 1u;
    }
    const uint32_t pit = (uint32_t)((iy & (kTile - 1)) * kTile + (ix & (kTile - 1)));
    const uint32_t n_chunks = (hi - lo + 31u) >> 5;  // words past the list belong to the next tile
    // the main kernel wrote the bits before the resume point of the deferral chunk
    const uint32_t c_start = (start - lo) >> 5;
    const uint32_t stored =
        (!naive && !stopped && c_start == ((f.entry - lo) >> 5)) ? a.pix_mask[mask_word(lo, tile, c_start, pit)] : 0u;
    uint32_t n_win = 0;  // HGS_FLAG_COUNT: windows walked (diag 15 = the longest walk)
    for (uint32_t base = lo + (c_start << 5); base < hi && !stopped; base += WIN) {
      ++n_win;
      float at[E], Pi[E];
      uint32_t rks[E];
      uint32_t conm = 0u;
      float P = 1.f;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const uint32_t e = base + (uint32_t)(E * lane + i);
        at[i] = 0.f;
        rks[i] = 0u;
        if (e >= start && e < hi) {
          const uint32_t rk = a.tile_vals[e];  // NAIVE: the depth order
          rks[i] = rk;
          const SplatRec r = a.recs[rk];
          if (naive || in_bbox(r.r5, ix, iy)) {
            PairEval p;
            if (eval_pair<false>(r, a.recs + rk, ix, iy, a.flags, a.st, p)) {
              conm |= 1u << i;
              at[i] = p.at;
            }
          }
        }
        P *= 1.f - at[i];  // at = 0 for non-contributing entries
        Pi[i] = P;
      }
      float S = P;  // inclusive product scan of the lane products, in entry order
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, o);
        if (lane >= o) S *= y;
      }
      float Sex = __shfl_up_sync(0xffffffffu, S, 1);
      if (lane == 0) Sex = 1.f;
      const float Tl = T * Sex;  // transmittance before this lane's first entry
      // early stop, in entry order: clear float32 decisions first, then the
      // near-threshold entries (warp-cooperative float64 replay) before them
      uint32_t nearm = 0u, clearm = 0u;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const float Ta = Tl * Pi[i];
        const bool con = (conm >> i) & 1u;
        const bool near = con && fabsf(Ta - thr) <= 2e-5f * thr;
        if (near) nearm |= 1u << i;
        if (con && !near && Ta < thr) clearm |= 1u << i;
      }
      int first = (int)WIN;  // window-relative index of the stop entry
      const uint32_t clear_lanes = __ballot_sync(0xffffffffu, clearm != 0u);
      if (clear_lanes) {
        const int l = __ffs(clear_lanes) - 1;
        first = E * l + __ffs(__shfl_sync(0xffffffffu, clearm, l)) - 1;
      }
      uint32_t near_lanes = __ballot_sync(0xffffffffu, nearm != 0u);
      bool hit = false;
      while (near_lanes && !hit) {
        const int l = __ffs(near_lanes) - 1;
        near_lanes &= near_lanes - 1;
        if (E * l > first) break;
        uint32_t nm = __shfl_sync(0xffffffffu, nearm, l);
        while (nm) {
          const int i = __ffs(nm) - 1;
          nm &= nm - 1;
          const int idx = E * l + i;
          if (idx > first) break;
          if (replay_T_below(a.recs, a.tile_vals, a.flags, a.st, lo, base + (uint32_t)idx, ix, iy)) {
            first = idx;
            hit = true;
            break;
          }
        }
      }
      // contributions up to and including the stop entry
      uint32_t vm = 0u;
      float Tb = Tl;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        if (((conm >> i) & 1u) && E * lane + i <= first) {
          vm |= 1u << i;
          const float wgt = at[i] * Tb;
          const SplatRec *g = a.recs + rks[i];  // just loaded: L1 hit
          const float4 c3 = g->r3, c4 = g->r4;
          q0 = fmaf(wgt, c3.y, q0);
          q1 = fmaf(wgt, c3.z, q1);
          q2 = fmaf(wgt, c3.w, q2);
          qd = fmaf(wgt, g->r0.z, qd);
          qn0 = fmaf(wgt, c4.x, qn0);
          qn1 = fmaf(wgt, c4.y, qn1);
          qn2 = fmaf(wgt, c4.z, qn2);
        }
        Tb = Tl * Pi[i];
      }
      cnt += __reduce_add_sync(0xffffffffu, (uint32_t)__popc(vm));
      const uint32_t hi_idx = __reduce_max_sync(0xffffffffu, vm ? (uint32_t)(E * lane + 32 - __clz(vm)) : 0u);
      if (hi_idx) last = base + hi_idx - lo;  // one past the last contributor, relative to lo
      if (!naive) {
        // contribution-mask word of each chunk of the window: OR of the
        // lanes' E-bit groups over the LPC lanes of the chunk
        uint32_t word = vm << (E * (lane % LPC));
#pragma unroll
        for (int o = 1; o < LPC; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
        const uint32_t c = ((base - lo) >> 5) + (uint32_t)(lane / LPC);
        if (lane % LPC == 0 && c < n_chunks && 32 * (lane / LPC) <= first) {
          if (c == c_start) word |= stored;
          a.pix_mask[mask_word(lo, tile, c, pit)] = word;
        }
      }
      if (first < (int)WIN) {
        const int l = first / E, i = first % E;
        float Tf = Pi[0];
#pragma unroll
        for (int k = 1; k < E; ++k)
          if (k == i) Tf = Pi[k];
        T = __shfl_sync(0xffffffffu, Tl * Tf, l);
        stopped = true;
      } else {
        T = T * __shfl_sync(0xffffffffu, S, 31);
      }
    }
    const float c0 = f.c0 + warp_sum(q0), c1 = f.c1 + warp_sum(q1), c2 = f.c2 + warp_sum(q2);
    const float dep = f.dep + warp_sum(qd);
    const float n0 = f.n0 + warp_sum(qn0), n1 = f.n1 + warp_sum(qn1), n2 = f.n2 + warp_sum(qn2);
    if (lane == 0) {
      const uint32_t pix = f.pix;
      a.color[3 * pix + 0] = c0 + a.bg[0] * T;
      a.color[3 * pix + 1] = c1 + a.bg[1] * T;
      a.color[3 * pix + 2] = c2 + a.bg[2] * T;
      a.depth[pix] = dep;
      a.trans[pix] = T;
      if (a.alpha) a.alpha[pix] = 1.f - T;
      if (a.normal) {
        a.normal[3 * pix + 0] = n0;
        a.normal[3 * pix + 1] = n1;
        a.normal[3 * pix + 2] = n2;
      }
      a.pix_T[pix] = T;
      a.pix_last[pix] = last;
      if (naive) a.pix_count[pix] = cnt;
      atomicAdd(&a.st->diag[10], 1ull);
      if (a.flags & HGS_FLAG_COUNT) atomicMax(&a.st->diag[15], (unsigned long long)n_win);
    }
  }
}

}  // namespace hgs
