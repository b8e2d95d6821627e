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

namespace hgs {

// One CTA per 16 x 16 tile, one thread per pixel, warps own 8 x 4 pixel blocks
// and run independently (no block barriers): a warp walks its tile list in
// chunks of 32 entries; lane l loads entry l's rank and bbox and turns the
// bbox into a 32-bit mask of the warp's pixels it covers (the reference's
// inclusive bbox test, _blend_py.py:89-91); records of relevant entries are
// staged in the warp's slice of shared memory and walked in order.  Every
// lane sees the same splat, so the 2D / 3D branch is warp-uniform; a warp
// retires as soon as its 32 pixels are saturated or deferred.
template <bool NAIVE, bool COUNT>
__global__ void __launch_bounds__(kBlock, HGS_FWD_MINB) k_composite_fwd(CompositeArgs a) {
  __shared__ SplatRec s_rec[kBlock / 32][32];
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wx0 = tx * kTile + (warp & 1) * 8, wy0 = ty * kTile + (warp >> 1) * 4;
  const int ix = wx0 + (lane & 7), iy = wy0 + (lane >> 3);
  const bool inside = ix < a.width && iy < a.height;
  const uint32_t lane_bit = 1u << lane;
  const float lox = (float)(lane & 7), loy = (float)(lane >> 3);  // offset in the warp block
  const bool exact = HGS_EXACT_ENABLED && !(a.flags & HGS_FLAG_FAST);
  uint32_t lo, hi;
  if (NAIVE) {
    lo = 0;
    hi = (uint32_t)a.m;
  } else {
    lo = a.tile_off[tile];
    hi = a.tile_off[tile + 1];
  }
  const uint32_t pix = (uint32_t)iy * (uint32_t)a.width + (uint32_t)ix;
  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f, dep = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f;
  uint32_t cnt = 0, last = 0;
  bool done = !inside, deferred = false;
  uint32_t n_ev3 = 0, n_ev2 = 0, n_c3 = 0, n_c2 = 0;  // HGS_FLAG_COUNT
  SplatRec *wrec = s_rec[warp];
#if HGS_FWD_PIN_SA
  uint32_t wrec_sa = (uint32_t)__cvta_generic_to_shared(wrec);
  asm volatile("mov.u32 %0, %0;" : "+r"(wrec_sa));  // opaque: kept, not re-derived per splat
#endif

  auto defer = [&](uint32_t entry, uint32_t mode) {
    FwdFix f;
    f.pix = pix; f.entry = entry; f.mode = mode; f.cnt = cnt; f.last = last;
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
    if (j < hi) {
      const uint32_t rk = NAIVE ? j : __ldg(a.tile_vals + j);
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
      const int c = (HGS_STAGED_ORIGIN && !NAIVE) ? eval_fast<false, false, true>(r, ix, iy, a.flags, p, lox, loy)
                                                  : eval_fast<false>(r, ix, iy, a.flags, p);
      if (c == kSkip) continue;
#if HGS_FWD_ONE_DEFER
      // one deferral site (the pair's decision or the early-stop decision), so
      // the worklist address is formed only on that rare path
      uint32_t dmode = 2u;
      if (c == kAmbiguous) {
        if (COUNT) atomicAdd(&a.st->diag[is3d ? 12 : 13], 1ull);  // deferral reasons
        dmode = 0u;
      } else {
#else
      if (c == kAmbiguous) {
        if (COUNT) atomicAdd(&a.st->diag[is3d ? 12 : 13], 1ull);  // deferral reasons
        defer(base + e, 0u);
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
        last = base + e - lo + 1u;
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
            defer(base + e, 1u);
#endif
          }
          else if (T < (float)kEarlyStopT)
            done = true;
        }
      }
#if HGS_FWD_ONE_DEFER
      if (dmode != 2u) defer(base + e, dmode);
#endif
    }
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
  if (naive && count) k_composite_fwd<true, true><<<(unsigned)n_tiles, kBlock, 0, s>>>(a);
  else if (naive) k_composite_fwd<true, false><<<(unsigned)n_tiles, kBlock, 0, s>>>(a);
  else if (count) k_composite_fwd<false, true><<<(unsigned)n_tiles, kBlock, 0, s>>>(a);
  else k_composite_fwd<false, false><<<(unsigned)n_tiles, kBlock, 0, s>>>(a);
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

// Deferred pixels, one warp each (grid-stride over the worklist).  The warp
// evaluates 32 consecutive tile-list entries in parallel with the exact
// decisions (float64 re-evaluation where the float32 bound is ambiguous),
// forms the transmittance with a product scan, resolves the early stop in
// lane order (float64 replay near the threshold) and accumulates.
__global__ void __launch_bounds__(256, HGS_FIXUP_MINB) k_fixup_fwd(CompositeArgs a) {
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
    const uint32_t hi = naive ? (uint32_t)a.m : a.tile_off[tile + 1];
    float T = f.T, c0 = f.c0, c1 = f.c1, c2 = f.c2, dep = f.dep, n0 = f.n0, n1 = f.n1, n2 = f.n2;
    uint32_t cnt = f.cnt, last = f.last;
    bool stopped = false;
    uint32_t start = f.entry;
    if (f.mode == 1u) {  // warp-cooperative float64 replay of the transmittance
      stopped = replay_T_below(a.recs, a.tile_vals, a.flags, a.st, lo, f.entry, ix, iy);
      start = f.entry + 1u;
    }
    // contribution-mask words from the resume point on (the main kernel wrote
    // the deferral chunk's bits before the resume point)
    const uint32_t pit = (uint32_t)((iy & (kTile - 1)) * kTile + (ix & (kTile - 1)));
    uint32_t w_cur = (start - lo) >> 5;
    uint32_t cur = (!naive && w_cur == ((f.entry - lo) >> 5)) ? a.pix_mask[mask_word(lo, tile, w_cur, pit)] : 0u;
    // software pipeline: the next window's ranks are loaded and its records
    // prefetched into L2 while this window is evaluated
    uint32_t rk_next = start + lane < hi ? (naive ? start + lane : a.tile_vals[start + lane]) : 0u;
    for (uint32_t base = start; base < hi && !stopped; base += 32) {
      const uint32_t e = base + lane;
      const uint32_t rk_cur = rk_next;
      if (base + 32 + lane < hi) {
        rk_next = naive ? base + 32 + lane : a.tile_vals[base + 32 + lane];
        prefetch_rec(a.recs + rk_next);
      }
      bool con = false;
      float at = 0.f;
      SplatRec r;
      if (e < hi) {
        const uint32_t rk = rk_cur;
        r = a.recs[rk];
        if (naive || in_bbox(r.r5, ix, iy)) {
          PairEval p;
          con = eval_pair<false>(r, a.recs + rk, ix, iy, a.flags, a.st, p);
          at = p.at;
        }
      }
      const float om = con ? 1.f - at : 1.f;
      float P = om;  // inclusive product scan in lane (= entry) order
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, P, o);
        if (lane >= o) P *= y;
      }
      float Pex = __shfl_up_sync(0xffffffffu, P, 1);
      if (lane == 0) Pex = 1.f;
      const float Tb = T * Pex, Ta = T * P;
      // early stop, in lane order: clear float32 decisions first, then the
      // near-threshold lanes (warp-cooperative float64 replay) before them
      const bool near = con && fabsf(Ta - thr) <= 2e-5f * thr;
      const uint32_t clear_stop = __ballot_sync(0xffffffffu, con && !near && Ta < thr);
      uint32_t near_mask = __ballot_sync(0xffffffffu, near);
      int first = clear_stop ? __ffs(clear_stop) - 1 : 32;
      while (near_mask) {
        const int l = __ffs(near_mask) - 1;
        if (l > first) break;
        near_mask &= near_mask - 1;
        const uint32_t el = __shfl_sync(0xffffffffu, e, l);
        if (replay_T_below(a.recs, a.tile_vals, a.flags, a.st, lo, el, ix, iy)) {
          first = l;
          break;
        }
      }
      const bool valid = con && lane <= first;
      const float wgt = valid ? at * Tb : 0.f;
      c0 += warp_sum(valid ? wgt * r.r3.y : 0.f);
      c1 += warp_sum(valid ? wgt * r.r3.z : 0.f);
      c2 += warp_sum(valid ? wgt * r.r3.w : 0.f);
      dep += warp_sum(valid ? wgt * r.r0.z : 0.f);
      n0 += warp_sum(valid ? wgt * r.r4.x : 0.f);
      n1 += warp_sum(valid ? wgt * r.r4.y : 0.f);
      n2 += warp_sum(valid ? wgt * r.r4.z : 0.f);
      const uint32_t vm = __ballot_sync(0xffffffffu, valid);
      if (!naive && lane == 0) {  // window [base, base + 32) completes word w_cur, opens w_cur + 1
        const uint32_t sh = (base - lo) & 31u;
        cur |= vm << sh;
        a.pix_mask[mask_word(lo, tile, w_cur, pit)] = cur;
        cur = sh ? vm >> (32 - sh) : 0u;
        ++w_cur;
      }
      cnt += __popc(vm);
      if (vm) last = base + (31 - __clz(vm)) - lo + 1u;
      if (first < 32) {
        T = __shfl_sync(0xffffffffu, Ta, first);
        stopped = true;
      } else {
        T = __shfl_sync(0xffffffffu, Ta, 31);
      }
    }
    if (lane == 0) {
      // the open word, if it is still a chunk of this tile list (words past
      // the list belong to the next tile)
      if (!naive && hi > lo && w_cur <= ((hi - 1 - lo) >> 5)) a.pix_mask[mask_word(lo, tile, w_cur, pit)] = cur;
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
    }
  }
}

}  // namespace hgs
