// k_pencil.cuh -- the HBM-rate pencil kernels (consumers of the bulk-copy
// stage pipeline in common.cuh).
//
//   k_range_pencil  K2a  per-tile min/max            (src/histogram.cpp:86-94)
//   k_hist_pencil   K2b  per-tile counts             (src/histogram.cpp:24-40 over
//                                                     src/nd_image.cpp:104-187)
//   k_interp_pencil K4   2^D-corner blend            (src/pipeline.cpp:94-127,
//                                                     src/interpolation.cpp:7-86)
#pragma once

#include "common.cuh"

#ifndef NB_SWITCH_KT2
#define NB_SWITCH_KT2 1
#endif

// K2a dictionary sample: one row in every 4 * K2A_SAMPLE_GROUPS (4D: 1 in 4 rows:
// range pass 0.250 ms; 1 in 8: 0.240; 1 in 16: 0.237 but the blend redoes
// more missed values, 0.713 -> 0.719 ms)
#ifndef K2A_SAMPLE_GROUPS
#define K2A_SAMPLE_GROUPS 2
#endif

namespace mg {

struct PencilSmem {
  Pipe* pipe;
  float* bufs;
  unsigned char* tail;
};

__device__ __forceinline__ PencilSmem pencil_smem(const KGeom& G, unsigned char* smem) {
  PencilSmem s;
  s.pipe = reinterpret_cast<Pipe*>(smem);
  s.bufs = reinterpret_cast<float*>(smem + pipe_bytes());
  s.tail = smem + pipe_bytes() + (size_t)G.nst * G.stage_stride * 4;
  return s;
}

// Trailing-block tile (primary; pencil kernels require merged mirror copies
// along trailing dims) and multiplicity of the element at offset e.
__device__ __forceinline__ void trailing_tile(const KGeom& G, int64_t e, int* tile, int* w) {
  int64_t t = 0;
  int wt = 1;
  for (int j = G.rank - 1; j >= G.rank - G.kt; --j) {
    const int64_t x = e % G.d[j].s;
    e /= G.d[j].s;
    const int64_t tj = (x + G.d[j].before) / G.d[j].b;
    wt *= tile_parts(G.d[j], tj).weight(x);
    t += tj * G.tstride[j];
  }
  *tile = (int)t;
  *w = wt;
}

// --------------------------------------------------------------- K2a -----
// DICT: also collects the distinct values (bit patterns) of the slab into a
// per-CTA hash set, merged into the workspace set at the end (kDict*).
template <int KO, bool DICT>
__global__ void __launch_bounds__(kPencilThreads, 3)
    k_range_pencil(const __grid_constant__ KGeom G, const __grid_constant__ CUtensorMap tmap,
                   const float* __restrict__ in, const int32_t* __restrict__ units,
                   const int32_t* __restrict__ cta_units, WS W) {
  extern __shared__ __align__(128) unsigned char smem[];
  const PencilSmem P = pencil_smem(G, smem);
  int32_t* smin = reinterpret_cast<int32_t*>(P.tail);  // [gtr] ~key32(lo)
  int32_t* smax = smin + G.gtr;                         // [gtr] key32(hi)
  uint32_t* sset =  // [kDictHS] (DICT), 16-byte buckets
      reinterpret_cast<uint32_t*>(P.tail + ((G.gtr * 8 + 15) & ~15LL));
  __shared__ int s_n, s_over;
  if (DICT) {
    for (int k = threadIdx.x; k < kDictHS; k += blockDim.x) sset[k] = kDictEmpty;
    if (threadIdx.x == 0) s_n = s_over = 0;
  }
  pipe_init(*P.pipe, G.nst);
  __syncthreads();
  const int u0 = cta_units[blockIdx.x], u1 = cta_units[blockIdx.x + 1];
  if (threadIdx.x >= kConsumers) {
    if (threadIdx.x == kConsumers)
      pipe_produce<KO, false, false>(
          G, &tmap, units, G.dyn_units ? 0 : u0, G.dyn_units ? G.dyn_units : u1, *P.pipe, P.bufs,
          nullptr, G.dyn_units ? reinterpret_cast<unsigned long long*>(&W.range[3]) : nullptr);
    return;
  }
  const int tid = threadIdx.x;
  const int slot = tid / G.tpr;
  const int64_t e0 = (int64_t)(tid % G.tpr) * 4;
  const bool lane_on = slot < G.rpi;
  // bucketised insert: a present value costs one LDS.128 and four compares
  auto dict_add = [&](float f) {
    const uint32_t b = __float_as_uint(f);
    uint32_t bk = dict_hash(b, kDictLgBS);
    const uint4 q = reinterpret_cast<const uint4*>(sset)[bk];
    if (q.x == b || q.y == b || q.z == b || q.w == b) return;
    for (int probe = 0; probe < (1 << kDictLgBS); ++probe) {
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        uint32_t* sl = sset + bk * 4 + j;
        const uint32_t k = *reinterpret_cast<volatile uint32_t*>(sl);
        if (k == b) return;
        if (k == kDictEmpty) {
          const uint32_t old = atomicCAS(sl, kDictEmpty, b);
          if (old == kDictEmpty) {
            if (atomicAdd(&s_n, 1) >= kDictHS / 2) s_over = 1;
            return;
          }
          if (old == b) return;
        }
      }
      bk = (bk + 1) & ((1u << kDictLgBS) - 1);
    }
    s_over = 1;
  };
  int trt[4], dummy;
#pragma unroll
  for (int i = 0; i < 4; ++i) trailing_tile(G, e0 + i, &trt[i], &dummy);
  float mn[4], mx[4], mn2[4], mx2[4];
  int bad = 0;
  u64 nf01 = 0, nf23 = 0;  // finiteness accumulators (see the row loop)
  const u64 zero2 = 0;
  int64_t cur = -1;
  const int64_t stage_elems = G.stage_stride;
  const int P4 = (int)G.P;
  const int rstep = G.rpi * P4;
  const int trips = slot < G.stage_rows ? (G.stage_rows - slot + G.rpi - 1) / G.rpi : 0;

  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mn[i] = fminf(mn[i], mn2[i]);
      mx[i] = fmaxf(mx[i], mx2[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane_on && mn[i] <= mx[i]) {
        atomicMax(&smin[trt[i]], ~key32(mn[i]));
        atomicMax(&smax[trt[i]], key32(mx[i]));
      }
    consumers_sync();
    for (int64_t t = tid; t < G.gtr; t += kConsumers) {
      if (smax[t] != INT32_MIN) {
        long long* r = reinterpret_cast<long long*>(W.trange + 2 * (cur + t));
        atomicMax(r, (long long)~okey((double)key32_decode(~smin[t])));
        atomicMax(r + 1, (long long)okey((double)key32_decode(smax[t])));
      }
    }
  };

  uint32_t it = 0;
  int cs_slot = 0;
  uint32_t cs_phase = 0;
  while (true) {
    const int s = cs_slot;  // it % nst, (it / nst) & 1 as counters: no division
    mbar_wait(&P.pipe->full[s], cs_phase);
    const Stage& S = P.pipe->st[s];
    if (S.unit < 0) break;
    const int64_t key = S.key;
    if (key != cur) {
      if (cur >= 0) flush();
      consumers_sync();
      for (int64_t t = tid; t < G.gtr; t += kConsumers) smin[t] = smax[t] = INT32_MIN;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mn[i] = mn2[i] = INFINITY;
        mx[i] = mx2[i] = -INFINITY;
      }
      consumers_sync();
      cur = key;
    }
    const float* buf = P.bufs + s * stage_elems;
    if (lane_on) {
      // rows in groups of four (four LDS.128 in flight, two min/max chains);
      // one row pass in 4 * K2A_SAMPLE_GROUPS (warp-uniform, rotating) feeds the
      // dictionary sample: values the sample misses are rare ones, which the
      // blend resolves from the workspace LUTs
      const float* rp = buf + slot * P4 + e0;
      const int jd = (int)((0u - it) & 3u);  // sampled row of each group
      int k = 0;
#pragma unroll 1
      for (; k + 4 <= trips; k += 4, rp += 4 * rstep) {
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = *reinterpret_cast<const float4*>(rp + j * rstep);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float a[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
          float* m0 = (j & 1) ? mn2 : mn;
          float* m1 = (j & 1) ? mx2 : mx;
          // finiteness: 0 * x is 0 for finite x and NaN for +-inf / NaN, so a
          // packed fma chain goes NaN iff some voxel is not finite
          nf01 = fma2(pk2(a[0], a[1]), zero2, nf01);
          nf23 = fma2(pk2(a[2], a[3]), zero2, nf23);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            m0[i] = fminf(m0[i], a[i]);
            m1[i] = fmaxf(m1[i], a[i]);
          }
        }
        if (DICT && (K2A_SAMPLE_GROUPS == 1 || ((k >> 2) + it) % K2A_SAMPLE_GROUPS == 0) &&
            !*reinterpret_cast<volatile int*>(&s_over)) {
          const float4 w = jd == 0 ? v[0] : jd == 1 ? v[1] : jd == 2 ? v[2] : v[3];
          const float a[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i == 0 || a[i] != a[i - 1]) dict_add(a[i]);  // runs of equal values: once
        }
      }
      for (; k < trips; ++k, rp += rstep) {
        const float4 v = *reinterpret_cast<const float4*>(rp);
        const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          bad |= !isfinite(a[i]);
          mn[i] = fminf(mn[i], a[i]);
          mx[i] = fmaxf(mx[i], a[i]);
        }
        if (DICT && ((k + it) & 3) == 0 && !*reinterpret_cast<volatile int*>(&s_over)) {
#pragma unroll
          for (int i = 0; i < 4; ++i) dict_add(a[i]);
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&P.pipe->empty[s]);
    ++it;
    if (++cs_slot == G.nst) {
      cs_slot = 0;
      cs_phase ^= 1;
    }
  }
  if (cur >= 0) flush();
  {
    float z0, z1, z2, z3;
    upk2(nf01, z0, z1);
    upk2(nf23, z2, z3);
    bad |= isnan(z0) || isnan(z1) || isnan(z2) || isnan(z3);
  }
  if (bad) atomicMax(reinterpret_cast<long long*>(&W.range[2]), 1LL);
  if (DICT) {  // merge the CTA's values into the workspace set
    consumers_sync();
    if (s_over) {
      if (tid == 0) atomicExch(&W.dmeta[1], 1);
      return;
    }
    for (int k = tid; k < kDictHS; k += kConsumers) {
      const uint32_t b = sset[k];
      if (b == kDictEmpty) continue;
      uint32_t h = dict_hash(b, 13);  // kDictHG = 2^13 slots, linear probing
      for (int probe = 0; probe < kDictHG; ++probe) {
        const uint32_t old = atomicCAS(&W.dkeys[h], kDictEmpty, b);
        if (old == b) break;
        if (old == kDictEmpty) {
          if (atomicAdd(&W.dmeta[0], 1) >= kDictHG / 2) atomicExch(&W.dmeta[1], 1);
          break;
        }
        h = (h + 1) & (kDictHG - 1);
      }
    }
  }
}

// --------------------------------------------------------------- K2b -----
// Unit switch helpers: the CTA's [gtr][n + 1] shared histogram added into the
// workspace counts (no index division; nonzero bins only), and a row copy
// with four loads in flight per thread.
// skip (optional): per-tile {lo, c}; degenerate tiles' rows (counted by the
// hot path, never used) are not flushed.
__device__ __forceinline__ void hist_flush(const uint32_t* hist, uint32_t* dst, int gtr, int n,
                                           int tid, const float2* skip = nullptr) {
  const float kDegC = degenerate_lc().y;
  for (int t = 0; t < gtr; ++t) {
    if (skip && skip[t].y == kDegC) continue;
    for (int b = tid; b < n; b += kConsumers) {
      const uint32_t c = hist[t * (n + 1) + b];
      if (c) atomicAdd(dst + (int64_t)t * n + b, c);
    }
  }
}

__device__ __forceinline__ void copy_rows(float* dst, const float* __restrict__ src, int count,
                                          int tid) {
  int k = tid;
  for (; k + 3 * kConsumers < count; k += 4 * kConsumers) {
    const float a = __ldg(src + k), b = __ldg(src + k + kConsumers),
                c = __ldg(src + k + 2 * kConsumers), d = __ldg(src + k + 3 * kConsumers);
    dst[k] = a;
    dst[k + kConsumers] = b;
    dst[k + 2 * kConsumers] = c;
    dst[k + 3 * kConsumers] = d;
  }
  for (; k < count; k += kConsumers) dst[k] = __ldg(src + k);
}

// A voxel's multiplicity in a tile is the product of its per-dimension
// multiplicities, so counting the support box with those weights equals
// kernelize + compute_histogram while reading each input byte once.  A
// thread's equal neighbouring (tile, bin) keys merge: one shared add carries
// the whole run.
// MATCH: warp-aggregated shared atomics (north_star's __match_any_sync): the
// lanes holding the same histogram word elect one lane that adds the group's
// sum (MATCH.ANY + REDUX per voxel slot) -- an A/B against the plain run-merged
// adds (MCLAHE_K2_MATCH=1).
// CARRY: the run a thread ends a row with is carried into its next row (the
// rows of a thread are rpi apart; on flat data they keep landing in the same
// bin), so a same-word add is only issued when the run breaks -- fewer
// same-address shared atomics from the 4 rows a warp holds.
// K2_PRED_RED: run tails predicated off instead of redirected to the thread's dummy word
// (lanes that skip take no part in the add's bank conflicts: 4D hist 0.309 -> 0.299 ms,
// 5D 0.379 -> 0.371 ms)
#ifndef K2_PRED_RED
#define K2_PRED_RED 1
#endif
// K2_DEDUP4: every equal pair among a thread's four keys merges, not only neighbours
// (A/B; measured slower: 4D hist 0.299 -> 0.303 ms, 5D 0.371 -> 0.383 ms -- the extra
// compares cost more than the few non-adjacent repeats save)
#ifndef K2_DEDUP4
#define K2_DEDUP4 0
#endif
// the same in the carried-run variant (global mode): Large 4D hist 1.806 -> 1.874 ms, off
#ifndef K2_PRED_RED_CARRY
#define K2_PRED_RED_CARRY 0
#endif
template <int KO, bool ADAPT, bool MATCH, bool CARRY = false>
__global__ void __launch_bounds__(kPencilThreads, 3)
    k_hist_pencil(const __grid_constant__ KGeom G, const __grid_constant__ CUtensorMap tmap,
                  const float* __restrict__ in, const int32_t* __restrict__ units,
                  const int32_t* __restrict__ cta_units, WS W) {
  extern __shared__ __align__(128) unsigned char smem[];
  const PencilSmem P = pencil_smem(G, smem);
  const int n = G.n_bins;
  // [gtr][n + 1]: the pad word puts equal bins of neighbouring tiles (one per
  // thread of a row) in different banks
  uint32_t* hist = reinterpret_cast<uint32_t*>(P.tail);
  // then one private dummy word per consumer thread (the hot path's suppressed
  // adds land there: no branches, no conflicts), then {lo, c} per tile
  const uint32_t dummy_s =
      (uint32_t)__cvta_generic_to_shared(P.tail + ((G.gtr * (n + 1) * 4 + 15) & ~15LL)) +
      4u * threadIdx.x;
  float2* lcS = reinterpret_cast<float2*>(P.tail + ((G.gtr * (n + 1) * 4 + 15) & ~15LL) +
                                          kConsumers * 4);  // [gtr]
  // bin-edge tables of the pencil's tiles (adaptive) or of the global range
  float* thrS = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(lcS) + G.gtr * 16);
  const int n1 = n + 1;  // edge-table stride: thr[0] = -inf ... thr[n] = +inf
  const TileParam<float>* tparams = reinterpret_cast<const TileParam<float>*>(W.tparams);
  const TileParam<float> g0 = tparams[0];
  if (!ADAPT && tp_degenerate(g0.lim)) return;  // constant image: every mapping is 0.5
  // quantised volume with direct dictionary cells: k_hist_cells counts it
  if (ADAPT && G.cell_hist && W.dmeta[2] != 0 && W.dmeta[4] == 2) return;
  // 4 * kMagicBits kept opaque to ptxas (one IMAD per histogram address)
  __shared__ uint32_t s_mb4;
  if (threadIdx.x == 0) s_mb4 = 4u * (uint32_t)kMagicBits;
  pipe_init(*P.pipe, G.nst);
  __syncthreads();
  uint32_t mb4;
  asm volatile("ld.volatile.shared.u32 %0, [%1];"
               : "=r"(mb4)
               : "r"((uint32_t)__cvta_generic_to_shared(&s_mb4)));
  // per-warp binning mode: bracketed floors, or the edge table for every voxel
  // once most rows needed it (quantised data on bin edges), re-probed every
  // 64 stages; G.nb_edges forces either
  int k2_edges = G.nb_edges == 1 ? 1 : 0, k2_probe = 0;
  const int u0 = cta_units[blockIdx.x], u1 = cta_units[blockIdx.x + 1];
  if (threadIdx.x >= kConsumers) {
    if (threadIdx.x == kConsumers)
      pipe_produce<KO, false>(
          G, &tmap, units, G.dyn_units ? 0 : u0, G.dyn_units ? G.dyn_units : u1, *P.pipe, P.bufs,
          nullptr, G.dyn_units ? reinterpret_cast<unsigned long long*>(&W.range[3]) : nullptr,
          ADAPT ? tparams : nullptr);
    return;
  }
  const int tid = threadIdx.x;
  const int slot = tid / G.tpr;
  const int64_t e0 = (int64_t)(tid % G.tpr) * 4;
  const bool lane_on = slot < G.rpi;
  int trt[4], trw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) trailing_tile(G, e0 + i, &trt[i], &trw[i]);
  const int64_t stage_elems = G.stage_stride;
  const float2 glc = tile_lc(g0);
  int64_t cur = -1;
  bool patho = !ADAPT && isnan(glc.y);  // a range the float guard does not cover
  __shared__ int s_bad;
  const float kDegC = degenerate_lc().y;
  float2 lc0, lc2;  // {lo, c} of voxels 0 / 2 (hot path); the others re-read
  auto lcv = [&](int i) { return i == 0 ? lc0 : i == 2 ? lc2 : (ADAPT ? lcS[trt[i]] : glc); };
  // a voxel's edge table: thrS + tile * (n + 1) (adaptive) or the global row
  auto thv = [&](int i) { return thrS + (ADAPT ? trt[i] * n1 : 0); };
  int hb[4];
  const bool same_pairs = !ADAPT || (trt[0] == trt[1] && trt[2] == trt[3]);
  const uint32_t hist_s = (uint32_t)__cvta_generic_to_shared(hist);
  const int trips = slot < G.stage_rows ? (G.stage_rows - slot + G.rpi - 1) / G.rpi : 0;

  uint32_t it = 0;
  int cs_slot = 0;
  uint32_t cs_phase = 0;
  while (true) {
    const int s = cs_slot;  // it % nst, (it / nst) & 1 as counters: no division
    mbar_wait(&P.pipe->full[s], cs_phase);
    const Stage& S = P.pipe->st[s];
    if (S.unit < 0) break;
    const int64_t key = S.key;
    if (key != cur) {
      consumers_sync();
      if (tid == 0) s_bad = 0;
      if (cur >= 0) {
        hist_flush(hist, W.counts + cur * n, (int)G.gtr, n, tid, ADAPT ? lcS : nullptr);
      }
      consumers_sync();
      for (int64_t k = tid; k < G.gtr * (n + 1); k += kConsumers) hist[k] = 0;
      if (ADAPT) {
        for (int64_t t = tid; t < G.gtr; t += kConsumers) {
          const float2 lc = tile_lc(tparams[key + t]);
          lcS[t] = lc;
          if (isnan(lc.y)) s_bad = 1;
        }
        copy_rows(thrS, W.thr + key * n1, (int)(G.gtr * n1), tid);
      } else if (cur < 0) {
        for (int k = tid; k < n1; k += kConsumers) thrS[k] = W.thr[k];
      }
      consumers_sync();
      if (ADAPT) patho = s_bad != 0;
      cur = key;
      // per-thread tile constants for this pencil
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 lc = ADAPT ? lcS[trt[i]] : glc;
        if (i == 0) lc0 = lc;
        if (i == 2) lc2 = lc;
        hb[i] = (!ADAPT || lc.y != kDegC) ? trt[i] * (n + 1) : -1;  // degenerate: none
      }
    }
    const int rows = G.stage_rows;
    const float* buf = P.bufs + s * stage_elems;
    if (lane_on && !patho && same_pairs && S.wuni != 0) {
      // hot path: uniform row weights, both voxel pairs share a tile.  Bins via
      // the edge table (edge_bin); equal neighbouring (tile, bin) runs merge
      // into one predicated shared-memory add each -- no branches.
      const uint32_t wf = (uint32_t)S.wfix;
      // degenerate tiles count into their own rows too (never flushed): no
      // per-voxel masking
      uint32_t w[4], ha[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        w[i] = wf * (uint32_t)trw[i];
        ha[i] = hist_s + (uint32_t)(trt[i] * (n + 1)) * 4u;
      }
      const uint32_t th0 = (uint32_t)__cvta_generic_to_shared(thv(0));
      const uint32_t th2 = (uint32_t)__cvta_generic_to_shared(thv(2));
      const u64 L0 = pk2(lc0.x, lc0.x), C0 = pk2(lc0.y, lc0.y);
      const u64 L2 = pk2(lc2.x, lc2.x), C2 = pk2(lc2.y, lc2.y);
      const float* rp = buf + slot * G.P + e0;
      const int64_t rstep = (int64_t)G.rpi * G.P;
      // runs of equal keys carry their sum on the first add; suppressed adds
      // (run tails) go to the thread's dummy word: every add unconditional,
      // no branches around the atomics
      auto commit = [&](const uint32_t (&a)[4]) {
#if K2_DEDUP4
        if constexpr (!MATCH) {  // every equal pair of the four keys merges, not only neighbours
          const bool q01 = a[0] == a[1], q02 = a[0] == a[2], q03 = a[0] == a[3];
          const bool q12 = a[1] == a[2], q13 = a[1] == a[3], q23 = a[2] == a[3];
          const uint32_t t0 = w[0] + (q01 ? w[1] : 0u) + (q02 ? w[2] : 0u) + (q03 ? w[3] : 0u);
          const uint32_t t1 = w[1] + (q12 ? w[2] : 0u) + (q13 ? w[3] : 0u);
          const uint32_t t2 = w[2] + (q23 ? w[3] : 0u);
          red_add(a[0], t0);
          red_add_unless(a[1], t1, q01);
          red_add_unless(a[2], t2, q02 || q12);
          red_add_unless(a[3], w[3], q03 || q13 || q23);
          return;
        }
#endif
        const bool e01 = a[0] == a[1], e12 = a[1] == a[2], e23 = a[2] == a[3];
        const uint32_t s3 = w[3];
        const uint32_t s2 = w[2] + (e23 ? s3 : 0u);
        const uint32_t s1 = w[1] + (e12 ? s2 : 0u);
        const uint32_t s0 = w[0] + (e01 ? s1 : 0u);
        if constexpr (MATCH) {
          const uint32_t ad[4] = {a[0], e01 ? dummy_s : a[1], e12 ? dummy_s : a[2],
                                  e23 ? dummy_s : a[3]};
          const uint32_t sv[4] = {s0, s1, s2, s3};
          const unsigned act = __activemask();
          const int lane = threadIdx.x & 31;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const unsigned grp = __match_any_sync(act, ad[i]);
            const uint32_t tot = __reduce_add_sync(grp, sv[i]);
            if (__ffs(grp) - 1 == lane) red_add(ad[i], tot);
          }
        } else {
          red_add(a[0], s0);
#if K2_PRED_RED
          red_add_unless(a[1], s1, e01);
          red_add_unless(a[2], s2, e12);
          red_add_unless(a[3], s3, e23);
#else
          red_add(e01 ? dummy_s : a[1], s1);
          red_add(e12 ? dummy_s : a[2], s2);
          red_add(e23 ? dummy_s : a[3], s3);
#endif
        }
      };
      // histogram words via the edge table (k = rint of the f32 estimate, th
      // decides k or k - 1)
      auto edge_addrs = [&](const float4& v, uint32_t (&a)[4]) {
        u64 t01, t23;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t01) : "l"(mul2(sub2(pk2(v.x, v.y), L0), C0)), "l"(pk2(kMagic, kMagic)));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t23) : "l"(mul2(sub2(pk2(v.z, v.w), L2), C2)), "l"(pk2(kMagic, kMagic)));
        float tf[4];
        upk2(t01, tf[0], tf[1]);
        upk2(t23, tf[2], tf[3]);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)  // histogram word of the voxel's (tile, bin)
          a[i] = edge_hist_addr(i < 2 ? th0 : th2, clamp_bits_k(tf[i], n), vv[i], ha[i]);
      };
      // adaptive mode keeps the edge table only: per-voxel tile constants leave
      // no registers for the bracketed floors (spills: 4D 0.33 -> 0.45 ms)
      // carried run (CARRY): address and sum of the last run of the previous row
      uint32_t ca = dummy_s, cs = 0;
      auto commit_carry = [&](const uint32_t (&a)[4]) {
        const bool c0 = a[0] == ca, e01 = a[1] == a[0], e12 = a[2] == a[1], e23 = a[3] == a[2];
#if K2_PRED_RED_CARRY
        red_add_unless(ca, cs, c0);  // the carried run ends unless a[0] continues it
        const uint32_t r0 = w[0] + (c0 ? cs : 0u);
        red_add_unless(a[0], r0, e01);
        const uint32_t r1 = w[1] + (e01 ? r0 : 0u);
        red_add_unless(a[1], r1, e12);
        const uint32_t r2 = w[2] + (e12 ? r1 : 0u);
        red_add_unless(a[2], r2, e23);
#else
        red_add(c0 ? dummy_s : ca, cs);  // the carried run ends unless a[0] continues it
        const uint32_t r0 = w[0] + (c0 ? cs : 0u);
        red_add(e01 ? dummy_s : a[0], r0);
        const uint32_t r1 = w[1] + (e01 ? r0 : 0u);
        red_add(e12 ? dummy_s : a[1], r1);
        const uint32_t r2 = w[2] + (e12 ? r1 : 0u);
        red_add(e23 ? dummy_s : a[2], r2);
#endif
        cs = w[3] + (e23 ? r2 : 0u);
        ca = a[3];
      };
      if (ADAPT || k2_edges) {
#pragma unroll 4
        for (int k = 0; k < trips; ++k, rp += rstep) {
          const float4 v = *reinterpret_cast<const float4*>(rp);
          uint32_t a[4];
          edge_addrs(v, a);
          if constexpr (CARRY) commit_carry(a);
          else commit(a);
        }
        if constexpr (CARRY) red_add(ca, cs);
        if (!ADAPT && G.nb_edges < 0 && ++k2_probe >= 64) k2_edges = k2_probe = 0;
      } else if constexpr (!ADAPT) {
        // bracketed floors (binning.cuh: bin_window): a voxel of the tile's
        // own support has d = v - lo >= 0, so the clamped lower floor is the
        // bin wherever both floors agree; a row where some lane's disagree is
        // redone through the edge table
        const float2 w0 = bin_window(lc0.y), w2 = bin_window(lc2.y);
        const u64 CL0 = pk2(w0.x, w0.x), CH0 = pk2(w0.y, w0.y);
        const u64 CL2 = pk2(w2.x, w2.x), CH2 = pk2(w2.y, w2.y);
        const u64 M2 = pk2(kMagic, kMagic);
        uint32_t hab[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) hab[i] = ha[i] - mb4;
        int nslow = 0;
#pragma unroll 4
        for (int k = 0; k < trips; ++k, rp += rstep) {
          const float4 v = *reinterpret_cast<const float4*>(rp);
          const u64 d01 = sub2(pk2(v.x, v.y), L0), d23 = sub2(pk2(v.z, v.w), L2);
          float fa[4], fb[4];
          upk2(fma_rm2(d01, CL0, M2), fa[0], fa[1]);
          upk2(fma_rm2(d23, CL2, M2), fa[2], fa[3]);
          upk2(fma_rm2(d01, CH0, M2), fb[0], fb[1]);
          upk2(fma_rm2(d23, CH2, M2), fb[2], fb[3]);
          uint32_t amb = 0, a[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ab = __float_as_int(fa[i]);
            amb |= (uint32_t)(ab ^ __float_as_int(fb[i]));
            a[i] = hab[i] + 4u * (uint32_t)min(max(ab, kMagicBits), kMagicBits + n - 1);
          }
          if (__any_sync(__activemask(), amb != 0)) {  // rare on continuous data
            ++nslow;
            edge_addrs(v, a);
          }
          if constexpr (CARRY) commit_carry(a);
          else commit(a);
        }
        if constexpr (CARRY) red_add(ca, cs);
        if (G.nb_edges < 0 && 4 * nslow > trips) {  // edges decide most rows: edge mode
          k2_edges = 1;
          k2_probe = 0;
        }
      }
    } else if (lane_on) {
      const bool wuni = S.wuni != 0;
      const int32_t wfix = S.wfix;
#pragma unroll 4
      for (int q = slot; q < rows; q += G.rpi) {
        uint32_t wrow;
        if (wuni) {
          wrow = (uint32_t)wfix;
        } else {
          const int r1 = q & (G.r1 - 1), r2 = q >> G.lg_r1;
          int32_t w = wfix * S.p1.weight(S.x[KO - 1] + r1);
          if (KO >= 2) w *= S.p2.weight(S.x[KO >= 2 ? KO - 2 : 0] + r2);
          wrow = (uint32_t)w;
        }
        const float4 v = *reinterpret_cast<const float4*>(buf + q * G.P + e0);
        int b[4];
        if (!patho) {
          if (same_pairs) {
            bins2_edge(pk2(v.x, v.y), v.x, v.y, lc0, thv(0), n, b[0], b[1]);
            bins2_edge(pk2(v.z, v.w), v.z, v.w, lc2, thv(2), n, b[2], b[3]);
          } else {  // pairs straddle a tile boundary: evaluate each against its own tile
            int dmy;
            bins2_edge(pk2(v.x, v.x), v.x, v.x, lc0, thv(0), n, b[0], dmy);
            bins2_edge(pk2(v.y, v.y), v.y, v.y, lcv(1), thv(1), n, b[1], dmy);
            bins2_edge(pk2(v.z, v.z), v.z, v.z, lc2, thv(2), n, b[2], dmy);
            bins2_edge(pk2(v.w, v.w), v.w, v.w, lcv(3), thv(3), n, b[3], dmy);
          }
        } else {
          const float a4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (isnan(lcv(i).y)) b[i] = bin_search(a4[i], thv(i), n);
            else bins2_edge(pk2(a4[i], a4[i]), a4[i], a4[i], lcv(i), thv(i), n, b[i], b[i]);
          }
        }
        // merge equal neighbours, one shared atomic per distinct (tile, bin);
        // degenerate tiles (hb < 0) build no histogram
        int kprev = -1;
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int key2 = hb[i] >= 0 ? hb[i] + b[i] : -2 - i;
          const uint32_t w = wrow * (uint32_t)trw[i];
          if (key2 == kprev) {
            acc += w;
          } else {
            if (kprev >= 0) atomicAdd(&hist[kprev], acc);
            kprev = key2;
            acc = w;
          }
        }
        if (kprev >= 0) atomicAdd(&hist[kprev], acc);
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&P.pipe->empty[s]);
    ++it;
    if (++cs_slot == G.nst) {
      cs_slot = 0;
      cs_phase ^= 1;
    }
  }
  consumers_sync();
  if (cur >= 0) {
    hist_flush(hist, W.counts + cur * n, (int)G.gtr, n, tid, ADAPT ? lcS : nullptr);
  }
}

// K2b for quantised volumes (adaptive mode, value dictionary with direct cells --
// kDict*, dmeta[4] == 2): voxels are counted per (tile, dictionary CELL) instead
// of per (tile, bin).  A voxel's cell is one packed FMA + clamp and one 32-bit
// check of the cell's value bits; no range, no edge table, no binning in the hot
// loop.  Every voxel of a tile with the same value falls in the same bin, so the
// unit switch turns the cell counts into bin counts exactly: one reference-rule
// binning per (tile, value) -- ~5 k per unit against ~500 k voxels.  A voxel
// whose value the (sampled) dictionary lacks is binned on the spot against the
// workspace edge table and added to the workspace counts directly.  Launched
// beside k_hist_pencil; the dictionary state in the workspace selects which of
// the two runs (the other exits at once).
template <int KO>
__global__ void __launch_bounds__(kPencilThreads, 3)
    k_hist_cells(const __grid_constant__ KGeom G, const __grid_constant__ CUtensorMap tmap,
                 const float* __restrict__ in, const int32_t* __restrict__ units,
                 const int32_t* __restrict__ cta_units, WS W) {
  if (W.dmeta[2] == 0 || W.dmeta[4] != 2) return;  // k_hist_pencil counts this volume
  constexpr int KC1 = kDictKC + 1;  // row pad: equal cells of neighbouring tiles in different banks
  extern __shared__ __align__(128) unsigned char smem[];
  const PencilSmem P = pencil_smem(G, smem);
  const int n = G.n_bins;
  uint32_t* hist = reinterpret_cast<uint32_t*>(P.tail);  // [gtr][KC1]
  uint32_t* bitsS = hist + ((G.gtr * KC1 + 3) & ~3LL);    // [kDictKC] value bits by cell
  const TileParam<float>* tparams = reinterpret_cast<const TileParam<float>*>(W.tparams);
  const int K = min(W.dmeta[3], kDictKC);
  const float dv0 = __int_as_float(W.dmeta[5]), dS = __int_as_float(W.dmeta[6]);
  const float nm05 = (float)n - 0.5f;
  for (int k = threadIdx.x; k < kDictKC; k += blockDim.x)
    bitsS[k] = k < K ? __float_as_uint(W.dvals[k]) : kDictEmpty;
  pipe_init(*P.pipe, G.nst);
  __syncthreads();
  const int u0 = cta_units[blockIdx.x], u1 = cta_units[blockIdx.x + 1];
  if (threadIdx.x >= kConsumers) {
    if (threadIdx.x == kConsumers)
      pipe_produce<KO, false>(
          G, &tmap, units, G.dyn_units ? 0 : u0, G.dyn_units ? G.dyn_units : u1, *P.pipe, P.bufs,
          nullptr, G.dyn_units ? reinterpret_cast<unsigned long long*>(&W.range[3]) : nullptr,
          tparams);
    return;
  }
  const int tid = threadIdx.x;
  const int slot = tid / G.tpr;
  const int64_t e0 = (int64_t)(tid % G.tpr) * 4;
  const bool lane_on = slot < G.rpi;
  int trt[4], trw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) trailing_tile(G, e0 + i, &trt[i], &trw[i]);
  const int64_t stage_elems = G.stage_stride;
  const uint32_t hist_s = (uint32_t)__cvta_generic_to_shared(hist);
  const uint32_t bits_s = (uint32_t)__cvta_generic_to_shared(bitsS);
  uint32_t ha[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) ha[i] = hist_s + (uint32_t)(trt[i] * KC1) * 4u;
  // cell counts of unit `key` -> bin counts (degenerate tiles build no histogram)
  // (four entries per thread at a time: their tile parameter / edge-table loads are
  // independent chains)
  auto flush = [&](int64_t key) {
    const int total = (int)G.gtr * K;
#pragma unroll 1
    for (int e0f = tid; e0f < total; e0f += 4 * kConsumers) {
      uint32_t cnt[4];
      int tt[4], cc[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0f + j * kConsumers;
        tt[j] = e < total ? e / K : 0;
        cc[j] = e < total ? e - tt[j] * K : 0;
        cnt[j] = e < total ? hist[tt[j] * KC1 + cc[j]] : 0u;
      }
      TileParam<float> tp[4];
      float dv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        tp[j] = tparams[key + tt[j]];
        dv[j] = W.dvals[cc[j]];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (cnt[j] == 0 || tp_degenerate(tp[j].lim)) continue;
        const int64_t tile = key + tt[j];
        atomicAdd(W.counts + tile * n + bin_of(dv[j], tp[j], W.thr + tile * (n + 1), n, nm05), cnt[j]);
      }
    }
  };
  int64_t cur = -1;
  uint32_t it = 0;
  int cs_slot = 0;
  uint32_t cs_phase = 0;
  while (true) {
    const int s = cs_slot;
    mbar_wait(&P.pipe->full[s], cs_phase);
    const Stage& S = P.pipe->st[s];
    if (S.unit < 0) break;
    const int64_t key = S.key;
    if (key != cur) {
      consumers_sync();
      if (cur >= 0) flush(cur);
      consumers_sync();
      for (int64_t k = tid; k < G.gtr * KC1; k += kConsumers) hist[k] = 0;
      consumers_sync();
      cur = key;
    }
    if (lane_on) {
      const int rows = G.stage_rows;
      const float* buf = P.bufs + s * stage_elems;
      const bool wuni = S.wuni != 0;
      const int32_t wfix = S.wfix;
      auto row_weight = [&](int q) {
        if (wuni) return (uint32_t)wfix;
        const int r1 = q & (G.r1 - 1), r2 = q >> G.lg_r1;
        int32_t w = wfix * S.p1.weight(S.x[KO - 1] + r1);
        if (KO >= 2) w *= S.p2.weight(S.x[KO >= 2 ? KO - 2 : 0] + r2);
        return (uint32_t)w;
      };
      // hot loop, no branches: a voxel whose bits differ from its cell's adds nothing
      // here (predicated off) and the stage is revisited for it below
      bool bad = false;
#pragma unroll 4
      for (int q = slot; q < rows; q += G.rpi) {
        const uint32_t wrow = row_weight(q);
        const float4 v = *reinterpret_cast<const float4*>(buf + q * G.P + e0);
        const float vv[4] = {v.x, v.y, v.z, v.w};
        int cl[4];
        cl[0] = dict_cell<kDictKC - 1>(v.x, v.y, dv0, dS, &cl[1]);
        cl[2] = dict_cell<kDictKC - 1>(v.z, v.w, dv0, dS, &cl[3]);
        uint32_t a[4], w[4];
        bool ok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t bw;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(bw) : "r"(bits_s + 4u * (uint32_t)cl[i]));
          ok[i] = bw == __float_as_uint(vv[i]);
          bad |= !ok[i];
          a[i] = ha[i] + 4u * (uint32_t)cl[i];
          w[i] = ok[i] ? wrow * (uint32_t)trw[i] : 0u;
        }
        // runs of equal (tile, cell) carry their sum on the first add (a miss carries
        // weight 0 and can only share an address with a voxel of another value: it
        // never merges into a real run's cell wrongly, its cell IS that address)
        const bool e01 = a[0] == a[1], e12 = a[1] == a[2], e23 = a[2] == a[3];
        const uint32_t s3 = w[3];
        const uint32_t s2 = w[2] + (e23 ? s3 : 0u);
        const uint32_t s1 = w[1] + (e12 ? s2 : 0u);
        const uint32_t s0 = w[0] + (e01 ? s1 : 0u);
        red_add_unless(a[0], s0, s0 == 0u);
        red_add_unless(a[1], s1, e01 || s1 == 0u);
        red_add_unless(a[2], s2, e12 || s2 == 0u);
        red_add_unless(a[3], s3, e23 || s3 == 0u);
      }
      if (bad) {  // values the dictionary lacks: straight into the workspace counts
#pragma unroll 1
        for (int q = slot; q < rows; q += G.rpi) {
          const uint32_t wrow = row_weight(q);
          const float4 v = *reinterpret_cast<const float4*>(buf + q * G.P + e0);
          const float vv[4] = {v.x, v.y, v.z, v.w};
          int cl[4];
          cl[0] = dict_cell<kDictKC - 1>(v.x, v.y, dv0, dS, &cl[1]);
          cl[2] = dict_cell<kDictKC - 1>(v.z, v.w, dv0, dS, &cl[3]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (bitsS[cl[i]] == __float_as_uint(vv[i])) continue;
            const int64_t tile = cur + trt[i];
            const TileParam<float> tp = tparams[tile];
            if (!tp_degenerate(tp.lim))
              atomicAdd(W.counts + tile * n + bin_of(vv[i], tp, W.thr + tile * (n + 1), n, nm05),
                        wrow * (uint32_t)trw[i]);
          }
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&P.pipe->empty[s]);
    ++it;
    if (++cs_slot == G.nst) {
      cs_slot = 0;
      cs_phase ^= 1;
    }
  }
  consumers_sync();
  if (cur >= 0) flush(cur);
}

// LUT value of one voxel against one window tile straight from the workspace
// (reference bin rule in f64): the dictionary blend's path for values its
// sampled dictionary does not hold.
static __device__ __noinline__ float lut_value_global(const WS& W, int n, int64_t tile, float v) {
  const TileParam<float> tp = reinterpret_cast<const TileParam<float>*>(W.tparams)[tile];
  const int b = tp_degenerate(tp.lim) ? 0 : bin_exact((double)v, (double)tp.lo, (double)tp.hi, n);
  return W.lut[tile * n + b];
}

// a[i] for a runtime i without local memory (N small)
// (selp in inline PTX: a plain select chain is turned back into an indexed
// local-memory load)
template <int N>
__device__ __forceinline__ float pick(const float (&a)[N], int i) {
  float r = a[0];
#pragma unroll
  for (int k = 1; k < N; ++k)
    asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, %3;\n\tselp.f32 %0, %1, %0, p;\n\t}"
        : "+f"(r)
        : "f"(a[k]), "r"(i), "r"(k));
  return r;
}

// ---------------------------------------------------------------- K4 -----
// One cell pencil (2^KO outer corners x every trailing tile) per unit; its
// LUTs, edge tables and {lo, c} pairs are staged in shared memory (rows padded
// to n+1 floats so different tiles start in different banks).  A stage holds
// R rows x one 32-float segment of the trailing block, TMA-loaded with the
// 128B swizzle.  Work item = (16-byte column, 32 rows): a warp owns one column
// -- so its 2^D corner tiles, ranges and trailing weights are warp-uniform --
// and each lane one row (outer weights per lane; neighbouring rows gather
// correlated bins).  The corner weights are products of per-dimension factors
// d/b with exact half-integer numerators; FP32 sum (the reference's sorted
// f64 sum is reproduced to <= 1e-6).
//
// NB > 0 (adaptive mode, n_bins == NB): each staged tile is one block
// [lo, c | th[0..NB] | LUT[0..NB-1] | pad] of 2*NB+4 floats, blocks ordered
// [trailing tile][outer corner], so a column's 2^D corner blocks sit at
// compile-time offsets from one or two per-item base addresses and every
// edge-table / LUT gather is a single LDS [reg + imm].
//
// NB < 0 (adaptive mode, value dictionary usable -- kDict*): blocks of
// kDictKC floats hold LUT_t[bin_t(value_i)] per dictionary value i, so a voxel
// looks its value up once (smem hash) and each corner is one LDS [reg + imm];
// no binning at all.  The dictionary and the edge-table kernels are both
// launched and whichever the device-side flag does not select exits at once.
template <int KO, int KT, bool ADAPT, int NB = 0>
__global__ void __launch_bounds__(kBlendThreads, 1)
    k_interp_pencil(const __grid_constant__ KGeom G, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ CUtensorMap omap, const float* __restrict__ in,
                    float* __restrict__ out,
                    const int32_t* __restrict__ units, const int32_t* __restrict__ cta_units, WS W) {
  constexpr int NCO = 1 << KO, NCT = 1 << KT;
  constexpr int NW = kConsumersBlend / 32;
  constexpr bool DICT = NB < 0;
  constexpr bool MORD = KT == 1 && KO == 3;
  // per-warp edge-table mode of the NB blend (see nb_edges); compiling it out
  // of the KT == 2 kernel (NB_SWITCH_KT2=0) removes a 24-byte spill (5D blend
  // 3.72 -> 3.70 ms) but leaves quantised KT == 2 data on the bracketed floors
  constexpr bool NB_SWITCH = NB > 0 && (KT == 1 || NB_SWITCH_KT2);
  if (W.range[2] != 0) return;  // non-finite input: write nothing
  if (DICT) {
    if (W.dmeta[2] == 0) return;
  } else if (ADAPT && G.dict) {
    if (W.dmeta[2] != 0) return;
  }
  extern __shared__ __align__(1024) unsigned char smem[];
  const PencilSmem P = pencil_smem(G, smem);
  const int n = G.n_bins;
  const int n1 = n + 1;
  const int64_t gtr = G.gtr;
  // Global mode with one trailing dim (PAIR): a voxel has one bin for all
  // corners, so the two trailing-corner LUTs of a column are stored side by
  // side, pairS[co][tt][b] = {L(co, tt)[b], L(co, tt+1)[b]}: one LDS.64 per
  // outer corner.  Otherwise LUT rows [NCO][gtr][n1].
  constexpr bool PAIR = !ADAPT && KT == 1;
  float* lutS = reinterpret_cast<float*>(P.tail);  // [NCO][gtr][n1] or pairs [NCO][gtr-1][n1]
  float2* pairS = reinterpret_cast<float2*>(P.tail);
  float* thrS = lutS + (PAIR ? 2 * NCO * (gtr - 1) * n1 : NCO * gtr * n1);  // edge tables
  float2* lcS = reinterpret_cast<float2*>(  // [NCO][gtr] {lo, c} (adaptive)
      P.tail + (((ADAPT ? 2 * NCO * gtr * n1
                        : (PAIR ? 2 * NCO * (gtr - 1) * n1 : NCO * gtr * n1) + n1) * 4 + 15) &
                ~15LL));
  // per trailing column: first corner tile and the 4 x NCT trailing weights
  const int ncol = (int)(G.P / 4);
  uint2* dltS =  // DICT: cuckoo lookup {bits, index} [kDictHL] after the value blocks
      reinterpret_cast<uint2*>(P.tail + NCO * gtr * kDictKC * 4);
  int* ofS = reinterpret_cast<int*>(dltS + kDictHL);  // [NCO] window tile of corner co's row
  int* colT = DICT     ? ofS + NCO
              : NB > 0 ? reinterpret_cast<int*>(P.tail + NCO * G.stiles * NbBlock::words(NB) * 4)
                       : reinterpret_cast<int*>(lcS + NCO * gtr);
  colT = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(colT) + 15) & ~uintptr_t(15));
  float* colW = reinterpret_cast<float*>(colT + ncol);  // [ncol][4][NCT], 16-byte aligned
  __shared__ int s_bad;
  __shared__ int s_wrap;   // NB: a staged tile could see t <= 0 (no RELU clamp)
  __shared__ int s_dmode;  // DICT: 1 = affine lookup
  __shared__ float s_dv0, s_dS;
  // 4 * kMagicBits through shared memory: kept opaque to ptxas so the NB fast
  // path's gather address stays one IMAD off a per-item base
  __shared__ uint32_t s_mb4;
  if (threadIdx.x == 0) s_mb4 = 4u * (uint32_t)kMagicBits;
  pipe_init(*P.pipe, G.nst, NW);
  __syncthreads();
  uint32_t mb4;
  asm volatile("ld.volatile.shared.u32 %0, [%1];"
               : "=r"(mb4)
               : "r"((uint32_t)__cvta_generic_to_shared(&s_mb4)));
  const int u0 = cta_units[blockIdx.x], u1 = cta_units[blockIdx.x + 1];
  if (threadIdx.x >= kConsumersBlend) {
    if (threadIdx.x == kConsumersBlend)
      pipe_produce<KO, true, false, true>(
          G, &tmap, units, G.dyn_units ? 0 : u0, G.dyn_units ? G.dyn_units : u1, *P.pipe, P.bufs,
          &omap, G.dyn_units ? reinterpret_cast<unsigned long long*>(&W.range[3]) : nullptr);
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TileParam<float>* tparams = reinterpret_cast<const TileParam<float>*>(W.tparams);
  const float2 glc = tile_lc(tparams[0]);
  bool patho = !ADAPT && isnan(glc.y);  // a range the float guard does not cover
  // NB: data whose values sit on bin edges (quantised counts) make the
  // bracketed floors disagree in most corner groups; each warp then switches to
  // the edge table for every voxel-corner (one extra dependent LDS, no votes)
  // and re-probes the bracketed path every 64 items.  G.nb_edges forces either.
  int nb_edges = G.nb_edges == 1 ? 1 : 0;  // warp-uniform
  int nb_probe = 0, nb_slow = 0;
  bool wrap_safe = false;
  // NB: the volume's minimum (k_params, adaptive) bounds every voxel a unit
  // blends from below; -inf when unknown (every unit takes the two-op clamp)
  float vmin = -INFINITY;
  if (NB > 0 && W.range[0] != INT64_MIN) vmin = __double2float_rd(okey_decode(~W.range[0]));

  // column table (independent of the unit): cells are shared by the column's
  // 4 voxels (the plan checks cell boundaries along the last dim are x4)
  for (int col = tid; col < ncol; col += kConsumersBlend) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t e = (int64_t)col * 4 + i;
      int64_t c[KT];
      float f1[KT];
#pragma unroll
      for (int q = KT - 1; q >= 0; --q) {
        const int j = G.rank - KT + q;
        const int64_t x = e % G.d[j].s;
        e /= G.d[j].s;
        c[q] = cell_of(G.d[j], x);
        f1[q] = (float)twice_dlo(G.d[j], x, c[q]) / (float)(2 * G.d[j].b);
      }
      if (i == 0) {
        int64_t t = 0;
#pragma unroll
        for (int q = 0; q < KT; ++q) t += c[q] * G.tstride[G.rank - KT + q];
        colT[col] = (int)t;
      }
#pragma unroll
      for (int ct = 0; ct < NCT; ++ct) {
        float w = 1.0f;
#pragma unroll
        for (int q = 0; q < KT; ++q) w *= ((ct >> (KT - 1 - q)) & 1) ? f1[q] : (1.0f - f1[q]);
        colW[(col * 4 + i) * NCT + ct] = w;
      }
    }
  }
  // trailing corner ct of a column's first tile: + bit_q * tstride[D-KT+q]
  int ctoff[NCT];
#pragma unroll
  for (int ct = 0; ct < NCT; ++ct) {
    int o = 0;
#pragma unroll
    for (int q = 0; q < KT; ++q) o += ((ct >> (KT - 1 - q)) & 1) * (int)G.tstride[G.rank - KT + q];
    ctoff[ct] = o;
  }

  const int64_t stage_elems = G.stage_stride;
  const int rows = G.stage_rows;
  const int nrb = (rows + 31) >> 5;
  int seg_lo = 0, seg_cnt = 0;  // NB: staged trailing-tile window
  float ugs[KO], ugt[KO];  // unit geometry (see the stage geometry below)
  int64_t cur = -1;
  uint32_t it = 0;
  int cs_slot = 0;
  uint32_t cs_phase = 0;
  while (true) {
    const int s = cs_slot;  // it % nst, (it / nst) & 1 as counters: no division
    mbar_wait(&P.pipe->full[s], cs_phase);
    const Stage& S = P.pipe->st[s];
    if (S.unit < 0) break;
    // NB with several segments stages one segment's trailing tiles at a time
    constexpr bool SEGW = NB > 0;
    const int64_t key = SEGW && G.nseg > 1 ? S.key * G.nseg + S.seg : S.key;
    if (key != cur) {
      consumers_sync<kConsumersBlend>();
      if (tid == 0) {
        s_bad = 0;
        s_wrap = 0;
      }
      consumers_sync<kConsumersBlend>();  // flags reset before any staging thread sets them
      if (SEGW) {  // tile window of this segment: its columns' first tiles + far corner
        seg_lo = 0;
        seg_cnt = (int)gtr;
        if (G.nseg > 1) {
          int mn = INT_MAX, mx = INT_MIN;
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            mn = min(mn, colT[S.seg * 8 + c]);
            mx = max(mx, colT[S.seg * 8 + c]);
          }
          seg_lo = mn;
          seg_cnt = min((int)gtr - mn, mx + ctoff[NCT - 1] - mn + 1);
        }
      }
      if (!ADAPT && cur < 0)
        for (int k = tid; k < n1; k += kConsumersBlend) thrS[k] = W.thr[k];
      if (DICT && cur < 0) {
        for (int k = tid; k < kDictHL; k += kConsumersBlend) dltS[k] = W.dlt[k];
        if (tid == 0) {
          s_dmode = W.dmeta[4];
          s_dv0 = __int_as_float(W.dmeta[5]);
          s_dS = __int_as_float(W.dmeta[6]);
        }
      }
      for (int co = 0; co < NCO; ++co) {
        int64_t of = (S.cell[0] + ((co >> (KO - 1)) & 1) - G.trow0) * G.tstride[0];
        for (int j = 1; j < KO; ++j) of += (S.cell[j] + ((co >> (KO - 1 - j)) & 1)) * G.tstride[j];
        const float4* src = reinterpret_cast<const float4*>(W.lut + of * n);
        if constexpr (DICT) {
          constexpr int KC4 = kDictKC / 4;
          if (tid == 0) ofS[co] = (int)of;
          float4* blk = reinterpret_cast<float4*>(P.tail) + co * KC4;  // + t * NCO * KC4
          const float4* ds = reinterpret_cast<const float4*>(W.lutd + of * kDictKC);
          for (int64_t k = tid; k < gtr * KC4; k += kConsumersBlend) {
            const int t = (int)(k / KC4), q = (int)(k - (int64_t)t * KC4);
            blk[t * NCO * KC4 + q] = __ldg(ds + k);
          }
          continue;
        }
        if constexpr (NB > 0) {
          if (co + 1 < NCO) continue;  // all corner rows at once, after the last corner
          // one pass over (tile, entry) with the NCO corners' loads independent
          // (in flight together): edge tables, LUTs, then {lo, c}
          constexpr int TBW = NbBlock::words(NB);
          constexpr int PT = NbBlock::th_words(NB), PL = NbBlock::lut_words(NB);
          int64_t ofc[NCO];
#pragma unroll
          for (int c2 = 0; c2 < NCO; ++c2) {
            int64_t o2 = (S.cell[0] + ((c2 >> (KO - 1)) & 1) - G.trow0) * G.tstride[0];
            for (int j = 1; j < KO; ++j) o2 += (S.cell[j] + ((c2 >> (KO - 1 - j)) & 1)) * G.tstride[j];
            ofc[c2] = o2 + seg_lo;  // first staged trailing tile of corner row c2
          }
          float* blk = reinterpret_cast<float*>(P.tail);
          for (int k = tid; k < seg_cnt * PL; k += kConsumersBlend) {
            const int t = k / PL, q = k - t * PL;
            float v[NCO];
#pragma unroll
            for (int c2 = 0; c2 < NCO; ++c2) v[c2] = __ldg(W.lut + (ofc[c2] + t) * NB + q);
#pragma unroll
            for (int c2 = 0; c2 < NCO; ++c2) blk[(t * NCO + c2) * TBW + NbBlock::lut_off(NB) + q] = v[c2];
          }
          for (int k = tid; k < seg_cnt * PT; k += kConsumersBlend) {
            const int t = k / PT, q = k - t * PT;
            float v[NCO];
#pragma unroll
            for (int c2 = 0; c2 < NCO; ++c2) v[c2] = __ldg(W.thr + (ofc[c2] + t) * (NB + 1) + NbBlock::src(q));
#pragma unroll
            for (int c2 = 0; c2 < NCO; ++c2) blk[(t * NCO + c2) * TBW + NbBlock::th_off(NB) + q] = v[c2];
          }
          for (int k = tid; k < seg_cnt * NCO; k += kConsumersBlend) {
            const int t = k / NCO, c2 = k - t * NCO;
            float2 lc = tile_lc(tparams[ofc[c2] + t]);
            const float2 wn = bin_window(lc.y);
            if (!(wn.y < INFINITY)) lc.y = __int_as_float(0x7fc00000);  // c_hi overflows: exact path
            *reinterpret_cast<float4*>(blk + (t * NCO + c2) * TBW) = make_float4(lc.x, wn.x, wn.y, lc.y);
            if (isnan(lc.y)) s_bad = 1;
            // t = fl(fl(v - lo) * c_hi + 1.5 * 2^23) > 0 for every v >= vmin
            // unless (lo - vmin) * c_hi reaches ~1.5 * 2^23 (margin: 2^22)
            if (!((lc.x - vmin) * wn.y < 4194304.0f)) s_wrap = 1;
          }
          continue;
        }
        if (PAIR) {
          float* dp = reinterpret_cast<float*>(pairS + co * (gtr - 1) * n1);
          for (int64_t k = tid; k < gtr * n / 4; k += kConsumersBlend) {
            const float4 q = __ldg(src + k);
            const int64_t t = (4 * k) / n, b = 4 * k - t * n;
            const float qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (t < gtr - 1) dp[2 * (t * n1 + b + j)] = qv[j];           // .x of pair t
              if (t >= 1) dp[2 * ((t - 1) * n1 + b + j) + 1] = qv[j];     // .y of pair t-1
            }
          }
        } else {
          float* dst = lutS + co * gtr * n1;
          for (int64_t k = tid; k < gtr * n / 4; k += kConsumersBlend) {
            const float4 q = __ldg(src + k);
            const int64_t t = (4 * k) / n, b = 4 * k - t * n;  // n % 4 == 0: one row
            float* d = dst + t * n1 + b;
            d[0] = q.x;
            d[1] = q.y;
            d[2] = q.z;
            d[3] = q.w;
          }
        }
        if (ADAPT) {
          const float* ts = W.thr + of * n1;
          float* td = thrS + co * gtr * n1;
          for (int64_t k = tid; k < gtr * n1; k += kConsumersBlend) td[k] = __ldg(ts + k);
          for (int64_t t = tid; t < gtr; t += kConsumersBlend) {
            const float2 lc = tile_lc(tparams[of + t]);
            lcS[co * gtr + t] = lc;
            if (isnan(lc.y)) s_bad = 1;
          }
        }
      }
      consumers_sync<kConsumersBlend>();
      if (ADAPT) patho = s_bad != 0;
      wrap_safe = s_wrap == 0;
      cur = key;
#pragma unroll
      for (int jd = 0; jd < KO; ++jd) {
        const Dim& d = G.d[jd];
        ugs[jd] = G.inv_b[jd];
        ugt[jd] = (float)(2 * d.before - 2 * (int64_t)S.cell[jd] * d.b - d.b + 1) * G.inv_2b[jd];
      }
    }
    // stage geometry: factor f_j(x) = x * s_j + t_j (exact half-integer
    // numerators); s_j, t_j depend on the unit's cell only (ugs / ugt, set at
    // the unit change), the stage contributes its coordinates
    float wfix[NCO / (KO >= 2 ? 4 : 2)];
    const float s1 = ugs[KO - 1], t1 = ugt[KO - 1];
    const float s2 = KO >= 2 ? ugs[KO >= 2 ? KO - 2 : 0] : 0.f;
    const float t2 = KO >= 2 ? ugt[KO >= 2 ? KO - 2 : 0] : 0.f;
    {
      float ff[KO > 2 ? KO - 2 : 1];
#pragma unroll
      for (int j = 0; j < KO - 2; ++j) ff[j] = fmaf((float)S.x[j], ugs[j], ugt[j]);
      constexpr int NF = NCO / (KO >= 2 ? 4 : 2);
#pragma unroll
      for (int cf = 0; cf < NF; ++cf) {
        float w = 1.0f;
#pragma unroll
        for (int j = 0; j < KO - 2; ++j) w *= ((cf >> (KO - 3 - j)) & 1) ? ff[j] : 1.0f - ff[j];
        wfix[cf] = w;
      }
    }
    const int xb1 = S.x[KO - 1], xb2 = KO >= 2 ? S.x[KO >= 2 ? KO - 2 : 0] : 0;
    const int seg = S.seg;
    unsigned char* buf = reinterpret_cast<unsigned char*>(P.bufs + s * stage_elems);
    for (int item = warp; item < 8 * nrb; item += NW) {
      const int c = item & 7, rb = item >> 3;
      // every lane runs the item (warp-uniform control flow for the votes);
      // rows past the stage's end recompute its last row and store nothing
      const bool q_on = rb * 32 + lane < rows;
      const int q = min(rb * 32 + lane, rows - 1);
      {
        const int col = seg * 8 + c;
        const int tt = colT[col];
        float tw[4][NCT];  // 4 * NCT consecutive floats (16-byte aligned): LDS.128s
#pragma unroll
        for (int h = 0; h < NCT; ++h) {
          const float4 w4 = reinterpret_cast<const float4*>(colW + col * 4 * NCT)[h];
          const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) tw[(4 * h + e) / NCT][(4 * h + e) % NCT] = wv[e];
        }
        const int r1 = q & (G.r1 - 1), r2 = q >> G.lg_r1;
        const int x1 = xb1 + r1, x2 = xb2 + r2;
        const float f1 = fmaf((float)x1, s1, t1);
        const float f2 = KO >= 2 ? fmaf((float)x2, s2, t2) : 0.f;
        float wo[NCO];
        {
          const float g1[2] = {1.0f - f1, f1};
#pragma unroll
          for (int co = 0; co < NCO; ++co) {
            float w = g1[co & 1];
            if (KO >= 2) w *= ((co >> 1) & 1) ? f2 : 1.0f - f2;
            wo[co] = w * wfix[co >> (KO >= 2 ? 2 : 1)];
          }
        }
        // 128B-swizzled stage row: 16-byte chunk c of row q sits at c ^ (q & 7)
        float4* slot4 = reinterpret_cast<float4*>(buf + q * 128 + ((c ^ (q & 7)) << 4));
        const float4 v4 = *slot4;
        const u64 V01 = pk2(v4.x, v4.y), V23 = pk2(v4.z, v4.w);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        float act[NCT][4];  // per trailing corner: sum over outer corners of wo * LUT
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
          for (int i = 0; i < 4; ++i) act[ct][i] = 0.f;
        // MORD (one trailing dim, KO == 3): the folded-pair blend
        // k_interp_mdict folds the two trailing corners first,
        // M = fma(tw1, L1, tw0 * L0), and sums act = fma(wo, M, act) over
        // co; the adaptive paths here sum in that order too (same bits)
        auto accum = [&](float w, const float (&m)[NCT][4]) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if constexpr (MORD)
              act[0][i] = fmaf(w, fmaf(tw[i][1 % NCT], m[1 % NCT][i], tw[i][0] * m[0][i]), act[0][i]);
            else
#pragma unroll
              for (int ct = 0; ct < NCT; ++ct) act[ct][i] = fmaf(w, m[ct][i], act[ct][i]);
          }
        };
        int bg[4] = {0, 0, 0, 0};
        if (!ADAPT) {
          if (!patho) {
            bins2_edge(V01, v4.x, v4.y, glc, thrS, n, bg[0], bg[1]);
            bins2_edge(V23, v4.z, v4.w, glc, thrS, n, bg[2], bg[3]);
          } else {
            bg[0] = bin_search(v4.x, thrS, n);
            bg[1] = bin_search(v4.y, thrS, n);
            bg[2] = bin_search(v4.z, thrS, n);
            bg[3] = bin_search(v4.w, thrS, n);
          }
        }
        const int n4 = 4 * n;
        if constexpr (DICT) {
          // corner (co, ct) row: base[ct >> 1] + ((ct & 1) * NCO + co) * KC floats
          constexpr int TB = kDictKC * 4;
          const char* blkc = reinterpret_cast<const char*>(P.tail);
          const char* base[KT];
          base[0] = blkc + tt * (NCO * TB);
          if (KT == 2) base[KT - 1] = base[0] + ctoff[KT == 2 ? 2 : 0] * (NCO * TB);
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
          const char* A[KT][4];
          int di[4];
          if (s_dmode) {  // affine cells: one LDS.64 per voxel
            int c[4];
            c[0] = dict_cell(vv[0], vv[1], s_dv0, s_dS, &c[1]);
            c[2] = dict_cell(vv[2], vv[3], s_dv0, s_dS, &c[3]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint2 e = dltS[c[i]];
              di[i] = e.x == __float_as_uint(vv[i]) ? (int)e.y : -1;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) di[i] = dict_lookup(dltS, __float_as_uint(vv[i]));
          }
          int miss = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            miss |= (di[i] < 0) << i;
            const int off = di[i] >= 0 ? di[i] * 4 : 0;
#pragma unroll
            for (int j = 0; j < KT; ++j) A[j][i] = base[j] + off;
          }
          static_for<0, NCO>([&](auto coc) {
            constexpr int co = decltype(coc)::value;
            float m[NCT][4];
            static_for<0, NCT>([&](auto ctc) {
              constexpr int ct = decltype(ctc)::value;
              constexpr int OFF = ((ct & 1) * NCO + co) * TB;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                m[ct][i] = *reinterpret_cast<const float*>(A[ct >> 1][i] + OFF);
            });
            accum(wo[co], m);
          });
          if (miss) {  // values the (sampled) dictionary lacks: redo them from the workspace
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if ((miss >> i) & 1) {
#pragma unroll
                for (int ct = 0; ct < NCT; ++ct) act[ct][i] = 0.0f;
#pragma unroll
                for (int co = 0; co < NCO; ++co) {
                  float L[NCT];
#pragma unroll
                  for (int ct = 0; ct < NCT; ++ct)
                    L[ct] = lut_value_global(W, n, ofS[co] + tt + ctoff[ct], vv[i]);
                  if constexpr (MORD)
                    act[0][i] = fmaf(wo[co], fmaf(tw[i][1 % NCT], L[1 % NCT], tw[i][0] * L[0]), act[0][i]);
                  else
#pragma unroll
                    for (int ct = 0; ct < NCT; ++ct) act[ct][i] = fmaf(wo[co], L[ct], act[ct][i]);
                }
              }
          }
        } else if constexpr (NB > 0) {
          // corner (co, ct) block: base[ct >> 1] + ((ct & 1) * NCO + co) * TB
          constexpr int TB = NbBlock::words(NB) * 4;
          const char* blkc = reinterpret_cast<const char*>(P.tail);
          const char* base[KT];
          base[0] = blkc + (tt - seg_lo) * (NCO * TB);
          if (KT == 2) base[KT - 1] = base[0] + ctoff[KT == 2 ? 2 : 0] * (NCO * TB);
          uint32_t sbase[KT];
#pragma unroll
          for (int j = 0; j < KT; ++j) sbase[j] = (uint32_t)__cvta_generic_to_shared(base[j]);
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
          if (NB_SWITCH && !patho && nb_edges) {  // edge-table test for every voxel-corner
            constexpr int SF = KO >= 2 ? 2 : 1;
            const float g2[2] = {1.0f - f2, f2};
            const u64 M2 = pk2(kMagic, kMagic);
#pragma unroll 1
            for (int cp = 0; cp < NCO / 2; ++cp) {
              const float wf = pick(wfix, cp >> (SF - 1));
              const float wg2 = KO >= 2 ? pick(g2, cp & 1) : 1.0f;
              const uint32_t po = (uint32_t)(2 * cp * TB);
              static_for<0, 2>([&](auto bc) {
                constexpr int b1 = decltype(bc)::value;
                float w = b1 ? f1 : 1.0f - f1;
                if (KO >= 2) w *= wg2;
                w *= wf;
                float m0[4];
                (void)m0;
                static_for<0, NCT>([&](auto ctc) {
                  constexpr int ct = decltype(ctc)::value;
                  constexpr int OFF = ((ct & 1) * NCO + b1) * TB;
                  const float4 hd = *reinterpret_cast<const float4*>(base[ct >> 1] + po + OFF);
                  u64 tq[2];
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const u64 y = mul2(sub2(h ? V23 : V01, pk2(hd.x, hd.x)), pk2(hd.w, hd.w));
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(tq[h]) : "l"(y), "l"(M2));
                  }
                  float tf[4];
                  upk2(tq[0], tf[0], tf[1]);
                  upk2(tq[1], tf[2], tf[3]);
                  float m[4];
#pragma unroll
                  for (int i = 0; i < 4; ++i)
                    m[i] = edge_gather_u<OFF + NbBlock::th_off(NB) * 4, OFF + NbBlock::lut_off(NB) * 4>(
                        sbase[ct >> 1] + po, clamp_bits_k(tf[i], NB), vv[i]);
                  if constexpr (MORD) {
                    if constexpr (ct == 0) {
#pragma unroll
                      for (int i = 0; i < 4; ++i) m0[i] = m[i];
                    } else {
#pragma unroll
                      for (int i = 0; i < 4; ++i)
                        act[0][i] = fmaf(w, fmaf(tw[i][1], m[i], tw[i][0] * m0[i]), act[0][i]);
                    }
                  } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) act[ct][i] = fmaf(w, m[i], act[ct][i]);
                  }
                });
              });
            }
          } else if (!patho) {  // hot path: bracketed floors, one LUT gather per corner
            const u64 M2 = pk2(kMagic, kMagic);
            // outer corners in pairs (runtime loop: the unrolled body is one
            // pair's 2 x NCT corners -- code size); weights as wo[] above.
            // Trailing corners in pairs share one warp vote.  Voxel pairs
            // accumulate with packed FFMA2 (per voxel the same fma order and
            // rounding as the scalar paths).
            // RELU: clamp the floor with one VIADDMNMX.RELU (min(bits - magic,
            // NB - 1), then max 0); exact unless bits - magic wraps, i.e.
            // t = fl(y + 1.5 * 2^23) <= 0, which needs y <= -1.5 * 2^23: the
            // unit's staged tiles were checked against the volume's minimum
            // (s_wrap).  Otherwise the signed-bits clamp (two ops).
            constexpr int SF = KO >= 2 ? 2 : 1;
            const float g2[2] = {1.0f - f2, f2};
            // LUT byte address straight from the clamped floor bits (signed-bits
            // clamp): lbase + 4 * bits  (lbase = base - 4 * kMagicBits, mod 2^32)
            uint32_t lbase[KT];
#pragma unroll
            for (int j = 0; j < KT; ++j) lbase[j] = sbase[j] - mb4;
            u64 a2[NCT][2];
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) a2[ct][0] = a2[ct][1] = 0;
            auto run = [&](auto relu_c) {
              constexpr bool RELU = decltype(relu_c)::value;
#pragma unroll 1
              for (int cp = 0; cp < NCO / 2; ++cp) {
                const float wf = pick(wfix, cp >> (SF - 1));
                const float wg2 = KO >= 2 ? pick(g2, cp & 1) : 1.0f;
                const uint32_t po = (uint32_t)(2 * cp * TB);
                static_for<0, 2>([&](auto bc) {
                  constexpr int b1 = decltype(bc)::value;
                  float w = b1 ? f1 : 1.0f - f1;
                  if (KO >= 2) w *= wg2;
                  w *= wf;
                  const u64 w2 = pk2(w, w);
                  static_for<0, NCT / 2>([&](auto hc) {
                    constexpr int hp = decltype(hc)::value;
                    float m[2][4];
                    uint32_t amb = 0;  // any lane-voxel whose two floors disagree
                    static_for<0, 2>([&](auto ec) {
                      constexpr int ct = 2 * hp + decltype(ec)::value;
                      constexpr int OFF = ((ct & 1) * NCO + b1) * TB;
                      const float4 hd = *reinterpret_cast<const float4*>(base[ct >> 1] + po + OFF);
                      u64 ta[2], tb[2];
#pragma unroll
                      for (int h = 0; h < 2; ++h) {
                        const u64 d = sub2(h ? V23 : V01, pk2(hd.x, hd.x));
                        ta[h] = fma_rm2(d, pk2(hd.y, hd.y), M2);
                        tb[h] = fma_rm2(d, pk2(hd.z, hd.z), M2);
                      }
                      float fa[4], fb[4];
                      upk2(ta[0], fa[0], fa[1]);
                      upk2(ta[1], fa[2], fa[3]);
                      upk2(tb[0], fb[0], fb[1]);
                      upk2(tb[1], fb[2], fb[3]);
#pragma unroll
                      for (int i = 0; i < 4; ++i) {
                        const int ab = __float_as_int(fa[i]);
                        amb |= (uint32_t)(ab ^ __float_as_int(fb[i]));
                        if constexpr (RELU)
                          m[ct & 1][i] = lut_at_relu<OFF + NbBlock::lut_off(NB) * 4>(sbase[ct >> 1] + po, ab, NB - 1);
                        else
                          m[ct & 1][i] = lut_at<OFF + NbBlock::lut_off(NB) * 4>(
                              lbase[ct >> 1] + po, min(max(ab, kMagicBits), kMagicBits + NB - 1));
                      }
                    });
                    if (__any_sync(0xffffffffu, amb != 0)) {
                      // rare (q within ~5e-7 |q| of a bin edge): the clamped floors
                      // are k - 1 and k and the edge table picks one
                      ++nb_slow;
                      static_for<0, 2>([&](auto ec) {
                        constexpr int ct = 2 * hp + decltype(ec)::value;
                        constexpr int OFF = ((ct & 1) * NCO + b1) * TB;
                        const char* B = base[ct >> 1] + po + OFF;
                        const float4 hd = *reinterpret_cast<const float4*>(B);
                        const float* th = reinterpret_cast<const float*>(B) + NbBlock::th_off(NB);
                        const float* L = reinterpret_cast<const float*>(B) + NbBlock::lut_off(NB);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {  // recomputed: fa / fb are not kept live
                          const float dd = __fsub_rn(vv[i], hd.x);
                          const int ka = clamp_bits(__fmaf_rd(dd, hd.y, kMagic), NB - 1);
                          const int kb = clamp_bits(__fmaf_rd(dd, hd.z, kMagic), NB - 1);
                          if (ka != kb && vv[i] >= th[NbBlock::pad(kb)]) m[ct & 1][i] = L[kb];
                        }
                      });
                    }
                    if constexpr (MORD) {  // fold the trailing pair, then one FMA per voxel
#pragma unroll
                      for (int h = 0; h < 2; ++h) {
                        const u64 in2 = fma2(pk2(m[1][2 * h], m[1][2 * h + 1]),
                                             pk2(tw[2 * h][1 % NCT], tw[2 * h + 1][1 % NCT]),
                                             mul2(pk2(tw[2 * h][0], tw[2 * h + 1][0]),
                                                  pk2(m[0][2 * h], m[0][2 * h + 1])));
                        a2[0][h] = fma2(in2, w2, a2[0][h]);
                      }
                    } else {
#pragma unroll
                      for (int e = 0; e < 2; ++e)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                          a2[2 * hp + e][h] = fma2(pk2(m[e][2 * h], m[e][2 * h + 1]), w2, a2[2 * hp + e][h]);
                    }
                  });
                });
              }
            };
            if (wrap_safe) run(std::integral_constant<bool, true>{});
            else run(std::integral_constant<bool, false>{});
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) {
              upk2(a2[ct][0], act[ct][0], act[ct][1]);
              upk2(a2[ct][1], act[ct][2], act[ct][3]);
            }
          } else {  // a pathological range in the pencil: exact search where needed
#pragma unroll
            for (int co = 0; co < NCO; ++co) {
              float mp[NCT][4];
#pragma unroll
              for (int ct = 0; ct < NCT; ++ct) {
                const char* B = base[ct >> 1] + ((ct & 1) * NCO + co) * TB;
                const float4 hd = *reinterpret_cast<const float4*>(B);
                const float2 lc = make_float2(hd.x, hd.w);
                const float* th = reinterpret_cast<const float*>(B) + NbBlock::th_off(NB);
                const float* L = reinterpret_cast<const float*>(B) + NbBlock::lut_off(NB);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  int b = 0;
                  if (isnan(lc.y)) {  // binary search over the padded edge table
                    int lo = 0, hi = NB - 1;
                    while (lo < hi) {
                      const int mid = (lo + hi + 1) >> 1;
                      if (vv[i] >= th[NbBlock::pad(mid)]) lo = mid;
                      else hi = mid - 1;
                    }
                    b = lo;
                  } else {
                    const u64 y = mul2(sub2(pk2(vv[i], vv[i]), pk2(lc.x, lc.x)), pk2(lc.y, lc.y));
                    u64 t2;
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t2) : "l"(y), "l"(pk2(kMagic, kMagic)));
                    float t0, t1;
                    upk2(t2, t0, t1);
                    const int k = clamp_bits(t0, NB);
                    b = vv[i] >= th[NbBlock::pad(k)] ? k : k - 1;
                  }
                  mp[ct][i] = L[b];
                }
              }
              accum(wo[co], mp);
            }
          }
          if constexpr (NB > 0) {  // per-warp mode switch (see nb_edges)
            if (NB_SWITCH && G.nb_edges < 0) {
              if (nb_edges) {
                if (++nb_probe >= 64) nb_edges = nb_probe = 0;
              } else {
                if (4 * nb_slow > NCO * NCT) nb_edges = 1;
                nb_slow = 0;
              }
            }
          }
        } else if (ADAPT && !patho) {  // hot path: branch-free edge-table gathers
#pragma unroll
          for (int co = 0; co < NCO; ++co) {
            float m[NCT][4];
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) {
              const int tile = co * (int)gtr + tt + ctoff[ct];  // warp-uniform
              const float2 lc = lcS[tile];
              const char* thb = reinterpret_cast<const char*>(thrS + tile * n1);
              const char* Lb = reinterpret_cast<const char*>(lutS + tile * n1);
              lut2_edge(V01, v4.x, v4.y, lc, thb, Lb, n4, m[ct][0], m[ct][1]);
              lut2_edge(V23, v4.z, v4.w, lc, thb, Lb, n4, m[ct][2], m[ct][3]);
            }
            accum(wo[co], m);
          }
        } else {
          int bo[4];  // global mode: byte offsets of the voxel's bin
#pragma unroll
          for (int i = 0; i < 4; ++i) bo[i] = bg[i] * (PAIR ? 8 : 4);
          if (PAIR) {
#pragma unroll
            for (int co = 0; co < NCO; ++co) {
              const char* Pb = reinterpret_cast<const char*>(pairS + (co * ((int)gtr - 1) + tt) * n1);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 p = *reinterpret_cast<const float2*>(Pb + bo[i]);
                if constexpr (MORD) {
                  act[0][i] = fmaf(wo[co], fmaf(tw[i][1 % NCT], p.y, tw[i][0] * p.x), act[0][i]);
                } else {
                  act[0][i] = fmaf(wo[co], p.x, act[0][i]);
                  act[1 % NCT][i] = fmaf(wo[co], p.y, act[1 % NCT][i]);
                }
              }
            }
          } else
#pragma unroll
          for (int co = 0; co < NCO; ++co) {
            float m[NCT][4];
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) {
              const int tile = co * (int)gtr + tt + ctoff[ct];  // warp-uniform
              const char* Lb = reinterpret_cast<const char*>(lutS + tile * n1);
              if (ADAPT) {  // a pathological range in the pencil: exact search
                const float2 lc = lcS[tile];
                const float* th = thrS + tile * n1;
                int b[4];
                if (!isnan(lc.y)) {
                  bins2_edge(V01, v4.x, v4.y, lc, th, n, b[0], b[1]);
                  bins2_edge(V23, v4.z, v4.w, lc, th, n, b[2], b[3]);
                } else {
                  b[0] = bin_search(v4.x, th, n);
                  b[1] = bin_search(v4.y, th, n);
                  b[2] = bin_search(v4.z, th, n);
                  b[3] = bin_search(v4.w, th, n);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) m[ct][i] = *reinterpret_cast<const float*>(Lb + 4 * b[i]);
              } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) m[ct][i] = *reinterpret_cast<const float*>(Lb + bo[i]);
              }
            }
            accum(wo[co], m);
          }
        }
        // trailing weights last: acc = sum_ct tw[ct] * (sum_co wo[co] * L)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if constexpr (MORD) {
            acc[i] = act[0][i];
          } else {
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) acc[i] = fmaf(tw[i][ct], act[ct][i], acc[i]);
          }
        }
        float4 r;
        r.x = fminf(fmaxf(acc[0], 0.f), 1.f);
        r.y = fminf(fmaxf(acc[1], 0.f), 1.f);
        r.z = fminf(fmaxf(acc[2], 0.f), 1.f);
        r.w = fminf(fmaxf(acc[3], 0.f), 1.f);
        if (q_on) *slot4 = r;  // in place; the producer TMA-stores the box
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&P.pipe->empty[s]);
    ++it;
    if (++cs_slot == G.nst) {
      cs_slot = 0;
      cs_phase ^= 1;
    }
  }
}

// Host-side accessors (defined in the k_*.cu translation units).
using PencilRangeFn = void (*)(const KGeom, const CUtensorMap, const float*, const int32_t*,
                               const int32_t*, WS);
using PencilHistFn = PencilRangeFn;
using PencilInterpFn = void (*)(const KGeom, const CUtensorMap, const CUtensorMap, const float*,
                                float*, const int32_t*, const int32_t*, WS);
PencilRangeFn get_range_pencil(int ko, bool dict);
PencilHistFn get_hist_pencil(int ko, bool adaptive, int variant = 0);  // 1 match, 2 carry
// fused adaptive K2 (k_fused.cu): ranges + counts in one kernel, one DRAM read
PencilRangeFn get_k2_fused(int ko, bool dict);
int k2_fused_threads();
int64_t k2_fused_tail_bytes(int64_t gtr, int64_t n_bins, bool dict);
int64_t k2_fused_tab_bytes(int64_t gtr, int64_t n_bins);
PencilInterpFn get_interp_pencil(int ko, int kt, bool adaptive, int n_bins);
PencilInterpFn get_interp_pencil_dict(int ko, int kt);
// folded-pair blend; nullptr: none for this (ko, mode, n_bins)
PencilInterpFn get_interp_mdict(int ko, bool tma_store, bool adaptive, int n_bins);
int interp_mdict_threads(bool adaptive);  // its block size (consumer warps + the producer warp)
// K2b by dictionary cell (k_hist_cells); nullptr: none for this ko
PencilHistFn get_hist_cells(int ko);

}  // namespace mg
