// k_misc.cuh -- the non-pencil kernels: workspace reset, K1 global range,
// binning parameters, K3 mappings, and the generic (any-shape, f32/f64)
// fallbacks of K2 and K4 that run one voxel per thread with global atomics.
#pragma once

#include "common.cuh"

namespace mg {

__device__ __forceinline__ int64_t window_tile(const KGeom& G, const int64_t* t) {
  int64_t f = (t[0] - G.trow0) * G.tstride[0];
  for (int j = 1; j < G.rank; ++j) f += t[j] * G.tstride[j];
  return f;
}

template <typename T>
__device__ __forceinline__ const T* thr_row(const WS& W, int64_t idx, int n);
template <>
__device__ __forceinline__ const float* thr_row<float>(const WS& W, int64_t idx, int n) {
  return W.thr + idx * (n + 1);
}
template <>
__device__ __forceinline__ const double* thr_row<double>(const WS&, int64_t, int) {
  return nullptr;  // f64 data takes the exact path near bin edges
}

__device__ __forceinline__ void decode_local(const KGeom& G, int64_t idx, int64_t* x) {
  for (int j = G.rank - 1; j >= 0; --j) {
    const int64_t ext = j == 0 ? (G.local_voxels / G.vstride[0]) : G.d[j].s;
    x[j] = idx % ext;
    idx /= ext;
  }
  x[0] += G.row0;
}

// ---------------------------------------------------------------- reset ---
__global__ void k_reset(int64_t* range, int64_t* trange, int64_t n_trange, WS W, int dict) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < 4) range[i] = i < 2 ? INT64_MIN : 0;
  for (int64_t k = i; k < n_trange; k += (int64_t)gridDim.x * blockDim.x) trange[k] = INT64_MIN;
  if (dict) {
    if (i < 8) W.dmeta[i] = 0;
    for (int64_t k = i; k < kDictHG; k += (int64_t)gridDim.x * blockDim.x) W.dkeys[k] = kDictEmpty;
  }
}

// Numbers the collected values (slot order), fills dvals and the {bits,
// index} lookup hash, and marks the dictionary usable when it fits the
// blend's capacity.  One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k_dict_finalize(WS W, int cap) {
  __shared__ int s_part[1024];
  const int tid = threadIdx.x;
  constexpr int PER = kDictHG / 1024;
  if (W.dmeta[1] != 0 || W.dmeta[0] > cap || W.dmeta[0] > 1024) {
    if (tid == 0) W.dmeta[2] = 0;
    return;
  }
  for (int k = tid; k < kDictHL; k += 1024) W.dlt[k] = make_uint2(kDictEmpty, 0);
  int c = 0;
  for (int j = 0; j < PER; ++j) c += W.dkeys[tid * PER + j] != kDictEmpty;
  s_part[tid] = c;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan
    const int v = tid >= off ? s_part[tid - off] : 0;
    __syncthreads();
    s_part[tid] += v;
    __syncthreads();
  }
  // index = rank by value: lanes gathering neighbouring values then hit
  // neighbouring shared-memory banks in the blend
  __shared__ uint32_t s_key[1024];
  const int K = s_part[1023];
  s_key[tid] = 0xFFFFFFFFu;
  __syncthreads();
  int idx = s_part[tid] - c;
  for (int j = 0; j < PER; ++j) {
    const uint32_t b = W.dkeys[tid * PER + j];
    if (b == kDictEmpty) continue;
    s_key[idx++] = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving key
  }
  __syncthreads();
  for (int k = 2; k <= 1024; k <<= 1)  // bitonic sort, ascending
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int p = tid ^ j;
      if (p > tid) {
        const uint32_t a = s_key[tid], b = s_key[p];
        if (((tid & k) == 0) == (a > b)) {
          s_key[tid] = b;
          s_key[p] = a;
        }
      }
      __syncthreads();
    }
  auto key_val = [](uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k); };
  // smallest gap between neighbouring values: block min-reduction (f64)
  __shared__ double s_gap[32];
  double gap = INFINITY;
  if (tid < K) {
    const float v = key_val(s_key[tid]);
    W.dvals[tid] = v;
    if (tid > 0) gap = (double)v - (double)key_val(s_key[tid - 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gap = fmin(gap, __shfl_xor_sync(0xffffffffu, gap, o));
  if ((tid & 31) == 0) s_gap[tid >> 5] = gap;
  __syncthreads();
  // Affine tables when the values are evenly spread (quantised data):
  // cell = rint((v - v0) * S), the same packed arithmetic as the blends
  // (dict_cell).  First try S = 1 / (smallest gap) with the cell as the value's
  // index (mode 2, "direct": the values renumbered by cell, holes empty; needs
  // every cell below cap), then S = 1.25 / gap with a {bits, index} table
  // (mode 1); both need distinct values in distinct cells.
  __shared__ int s_aff, s_maxc;
  __shared__ float s_v0, s_S;
  for (int att = 0; att < 2; ++att) {
    const bool direct = att == 0;
    if (tid == 0) {
      double g = INFINITY;
      for (int w = 0; w < 32; ++w) g = fmin(g, s_gap[w]);
      const float v0 = K > 0 ? key_val(s_key[0]) : 0.0f;
      const float S = K > 1 ? (float)((direct ? 1.0 : 1.25) / g) : 1.0f;
      const double span = K > 1 ? ((double)key_val(s_key[K - 1]) - (double)v0) * (double)S : 0.0;
      s_aff = (K > 0 && isfinite(S) && S > 0.0f && span < (direct ? cap - 2 : kDictHL - 4)) ? 1 : 0;
      s_v0 = v0;
      s_S = S;
      s_maxc = 0;
    }
    __syncthreads();
    const int tried = s_aff;
    __syncthreads();  // every thread has read s_aff before tid 0 may rewrite it
    if (!tried) continue;
    for (int i = tid; i < K; i += 1024) {
      const float v = key_val(s_key[i]);
      const int cell = dict_cell(v, v, s_v0, s_S, nullptr);
      if ((direct && cell >= cap) || atomicCAS(&W.dlt[cell].x, kDictEmpty, __float_as_uint(v)) != kDictEmpty)
        s_aff = 0;
      else {
        W.dlt[cell].y = (uint32_t)(direct ? cell : i);
        atomicMax(&s_maxc, cell);
      }
    }
    __syncthreads();
    if (s_aff) {
      if (direct) {  // renumber by cell: dvals[cell] = value, holes empty
        for (int c = tid; c < cap; c += 1024)
          W.dvals[c] = __uint_as_float(c <= s_maxc ? W.dlt[c].x : kDictEmpty);
      }
      if (tid == 0) {
        W.dmeta[4] = direct ? 2 : 1;
        W.dmeta[5] = __float_as_int(s_v0);
        W.dmeta[6] = __float_as_int(s_S);
        W.dmeta[3] = direct ? s_maxc + 1 : K;
        W.dmeta[7] = K;
        W.dmeta[2] = 1;
      }
      return;
    }
    for (int k = tid; k < kDictHL; k += 1024) W.dlt[k] = make_uint2(kDictEmpty, 0);
    __syncthreads();
  }
  if (tid == 0) {  // cuckoo placement, values in index order
    W.dmeta[4] = 0;
    bool ok = true;
    for (int i = 0; i < K && ok; ++i) {
      uint2 e = make_uint2(__float_as_uint(W.dvals[i]), (uint32_t)i);
      uint32_t h = dict_h1(e.x);
      int steps = 0;
      while (true) {
        const uint2 o = W.dlt[h];
        W.dlt[h] = e;
        if (o.x == kDictEmpty) break;
        if (++steps > 4 * kDictHL) {
          ok = false;
          break;
        }
        e = o;  // evict to its other slot
        h = dict_h1(e.x) == h ? dict_h2(e.x) : dict_h1(e.x);
      }
    }
    W.dmeta[3] = K;
    W.dmeta[7] = K;
    W.dmeta[2] = ok ? 1 : 0;
  }
}

// lutd[t][i] = LUT_t[bin_t(value_i)] with the reference bin rule in f64
// (degenerate tiles: any bin, their LUT is constant).  Grid: tiles x values.
// The reference bin of every dictionary value in every tile through the
// guarded f32 rule and the tile's edge table (bin_of: exact, one f32 estimate
// and at most one table load instead of an f64 divide per entry: 17 -> 15 us
// on the 4D volume; a CTA per tile with its rows staged measured 26 us).
template <typename T>
__global__ void k_dict_luts(WS W, int64_t win_tiles, int n) {
  if (W.dmeta[2] == 0) return;
  const int K = W.dmeta[3];
  const TileParam<T>* tp = reinterpret_cast<const TileParam<T>*>(W.tparams);
  const T nm05 = (T)n - (T)0.5;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < win_tiles * kDictKC;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / kDictKC;
    const int i = (int)(e - t * kDictKC);
    float r = 0.0f;
    if (i < K && __float_as_uint(W.dvals[i]) != kDictEmpty) {  // direct cells: holes stay 0
      const TileParam<T> p = tp[t];
      const int b = tp_degenerate(p.lim) ? 0 : bin_of((T)W.dvals[i], p, W.thr + t * (n + 1), n, nm05);
      r = W.lut[t * n + b];
    }
    W.lutd[e] = r;
  }
}

// ------------------------------------------------------ framewise ranges ----
// Batched mclahe_framewise (src/pipeline.cpp:131-153) in global mode: every
// frame is enhanced with its own global range.  The volume runs as one
// adaptive pass whose kernel is 1 along the frame axis, and each tile takes
// its frame's min/max instead of its own.  Runs r in [0, outer * frames) are
// the contiguous `inner`-element pieces of frame r % frames.
template <typename T>
__global__ void __launch_bounds__(256) k_frame_range(const T* __restrict__ in, int64_t outer,
                                                     int64_t frames, int64_t inner,
                                                     int64_t* __restrict__ frange,
                                                     int64_t* __restrict__ range) {
  for (int64_t r = blockIdx.y; r < outer * frames; r += gridDim.y) {
    const int64_t f = r % frames;
    const T* p = in + r * inner;
    T lo = INFINITY, hi = -INFINITY;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < inner;
         i += (int64_t)gridDim.x * blockDim.x) {
      const T v = p[i];
      bad |= !isfinite(v);
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
      atomicMax(reinterpret_cast<long long*>(&frange[2 * f]), (long long)~okey((double)lo));
      atomicMax(reinterpret_cast<long long*>(&frange[2 * f + 1]), (long long)okey((double)hi));
    }
    if ((threadIdx.x & 31) == 0 && bad) atomicMax(reinterpret_cast<long long*>(&range[2]), 1LL);
  }
}

// Tile range keys from the frame ranges: tile coordinate t along the frame
// axis (kernel 1) covers frame min(t, frames - 1) (the one padded tile
// mirrors the last frame).
__global__ void k_frame_tiles(const KGeom G, WS W, const int64_t* __restrict__ frange, int axis) {
  const int64_t frames = G.d[axis].s;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < G.win_tiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gt = t + G.trow0 * G.tstride[0];
    const int64_t tc = (gt / G.tstride[axis]) % G.d[axis].g;
    const int64_t f = tc < frames ? tc : frames - 1;
    W.trange[2 * t] = frange[2 * f];
    W.trange[2 * t + 1] = frange[2 * f + 1];
  }
}

// ------------------------------------------------------------------ K1 ----
// Global min/max + finiteness over the slab (NdImage::min_max / all_finite,
// src/nd_image.cpp:70-83).  Grid-stride, 16-byte loads, one atomic per CTA.
template <typename T>
__global__ void __launch_bounds__(256) k_global_range(const T* __restrict__ in, int64_t n,
                                                      int64_t* __restrict__ range) {
  constexpr int V = 16 / sizeof(T);
  T lo = INFINITY, hi = -INFINITY;
  int bad = 0;
  const int64_t nv = ((reinterpret_cast<uintptr_t>(in) & 15) == 0) ? n / V : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;  // 16-byte loads in flight per thread
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nv; i += U * stride) {
    T v[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (V == 4) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(in) + i + u * stride);
        v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
      } else {
        const double2 q = __ldcs(reinterpret_cast<const double2*>(in) + i + u * stride);
        v[u][0] = q.x; v[u][1] = q.y;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        bad |= !isfinite(v[u][k]);
        lo = fmin(lo, v[u][k]);
        hi = fmax(hi, v[u][k]);
      }
  }
  for (; i < nv; i += stride) {
    T v[V];
    if constexpr (V == 4) {
      const float4 q = __ldcs(reinterpret_cast<const float4*>(in) + i);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 q = __ldcs(reinterpret_cast<const double2*>(in) + i);
      v[0] = q.x; v[1] = q.y;
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
      bad |= !isfinite(v[k]);
      lo = fmin(lo, v[k]);
      hi = fmax(hi, v[k]);
    }
  }
  for (int64_t i = nv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const T v = in[i];
    bad |= !isfinite(v);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  // warp + block reduction
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ T slo[8], shi[8];
  __shared__ int sbad[8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    slo[w] = lo;
    shi[w] = hi;
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      lo = fmin(lo, slo[k]);
      hi = fmax(hi, shi[k]);
      bad |= sbad[k];
    }
    if (lo <= hi) {  // skip CTAs that saw no finite value
      atomicMax(reinterpret_cast<long long*>(&range[0]), (long long)~okey((double)lo));
      atomicMax(reinterpret_cast<long long*>(&range[1]), (long long)okey((double)hi));
    }
    if (bad) atomicMax(reinterpret_cast<long long*>(&range[2]), 1LL);
  }
}

// --------------------------------------------------------------- params ---
// Window tiles [t0, t0 + nt) (adaptive) or the single global range.
template <typename T>
__global__ void k_params(const KGeom G, WS W, int64_t t0, int64_t nt) {
  TileParam<T>* tp = reinterpret_cast<TileParam<T>*>(W.tparams);
  const int64_t n = G.adaptive ? t0 + nt : 1;
  // adaptive: the smallest tile minimum goes to W.range[0] (MAX of ~key, as
  // the global range pass keeps it) -- a lower bound on every voxel of the
  // window, which the n_bins-specialised blend uses to pick its clamp
  long long mkey = LLONG_MIN;
  for (int64_t t = (G.adaptive ? t0 : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* r = G.adaptive ? W.trange + 2 * t : W.range;
    const double lo = okey_decode(~r[0]);
    const double hi = okey_decode(r[1]);
    tp[t] = make_tile_param<T>(lo, hi, G.n_bins);
    if (G.adaptive && r[0] != INT64_MIN) mkey = max(mkey, (long long)r[0]);
  }
  if (G.adaptive) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mkey = max(mkey, __shfl_xor_sync(0xffffffffu, mkey, o));
    if ((threadIdx.x & 31) == 0 && mkey != LLONG_MIN)
      atomicMax(reinterpret_cast<long long*>(&W.range[0]), mkey);
  }
}

// ------------------------------------------------------ K2 generic -------
// One voxel per thread; enumerates the (<= 3^D) tiles a voxel's padded copies
// fall in.  MODE 0: per-tile min/max (adaptive ranges); MODE 1: counts.
template <typename T, int MODE, bool ADAPT>
__global__ void __launch_bounds__(256) k_tiles_generic(const KGeom G, const T* __restrict__ in,
                                                       WS W) {
  const int n = G.n_bins;
  const T nm05 = (T)n - (T)0.5;
  const TileParam<T>* tparams = reinterpret_cast<const TileParam<T>*>(W.tparams);
  int bad = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < G.local_voxels;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t x[kMaxRank];
    decode_local(G, idx, x);
    const T v = in[idx];
    if (MODE == 0) bad |= !isfinite(v);
    int64_t tl[kMaxRank][3];
    int wl[kMaxRank][3], nl[kMaxRank], ci[kMaxRank];
    for (int j = 0; j < G.rank; ++j) {
      nl[j] = voxel_tiles(G.d[j], x[j], tl[j], wl[j]);
      ci[j] = 0;
    }
    while (true) {
      int64_t t[kMaxRank];
      int w = 1;
      for (int j = 0; j < G.rank; ++j) {
        t[j] = tl[j][ci[j]];
        w *= wl[j][ci[j]];
      }
      const int64_t f = window_tile(G, t);
      if (MODE == 0) {
        atomicMax(reinterpret_cast<long long*>(W.trange + 2 * f), (long long)~okey((double)v));
        atomicMax(reinterpret_cast<long long*>(W.trange + 2 * f + 1), (long long)okey((double)v));
      } else {
        const TileParam<T> tp = tparams[ADAPT ? f : 0];
        if (!tp_degenerate(tp.lim))
          atomicAdd(W.counts + f * n + bin_of(v, tp, thr_row<T>(W, ADAPT ? f : 0, n), n, nm05),
                    (uint32_t)w);
      }
      int j = G.rank - 1;
      while (j >= 0 && ++ci[j] == nl[j]) ci[j--] = 0;
      if (j < 0) break;
    }
  }
  if (MODE == 0 && bad) atomicMax(reinterpret_cast<long long*>(&W.range[2]), 1LL);
}

// ------------------------------------------------------------------ K3 ----
// One warp per tile.  The two order-sensitive f64 sums of the reference run in
// bin order exactly as written there: the clip excess (histogram.cpp:47-48;
// only clipped bins add non-zero terms, found by ballot, summed in order) and
// the CDF prefix (histogram.cpp:59-63, one lane, sequential).  Everything else
// is bin-parallel.  Output: f32 LUT (+ optional f64 debug arrays).
template <typename T>
__global__ void __launch_bounds__(128) k_mappings(const KGeom G, WS W, Debug Dbg, int64_t t0,
                                                  int64_t nt, int dict_rows = 0) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = G.n_bins;
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* cdf = reinterpret_cast<double*>(smem) + (int64_t)wid * n;
  const TileParam<T>* tparams = reinterpret_cast<const TileParam<T>*>(W.tparams);
  // dict_rows (float32 plans with a value dictionary): the warp also writes its
  // tile's per-value row lutd[tile][i] = LUT[bin(value i)] (what k_dict_luts does in
  // a launch of its own), from the LUT it has just built
  bool drows = false;
  int dK = 0;
  if constexpr (sizeof(T) == 4) {
    drows = dict_rows != 0 && W.dmeta[2] != 0;
    dK = drows ? W.dmeta[3] : 0;
  }
  float* lutf = reinterpret_cast<float*>(cdf);  // the warp's LUT as floats, once cdf is done
  const T nm05 = (T)n - (T)0.5;
  for (int64_t tile = t0 + (int64_t)blockIdx.x * warps + wid; tile < t0 + nt;
       tile += (int64_t)gridDim.x * warps) {
    const TileParam<T> tp = tparams[G.adaptive ? tile : 0];
    const uint32_t* cnt = W.counts + tile * n;
    float* lut = W.lut + tile * n;
    if (Dbg.lo && lane == 0) {
      Dbg.lo[tile] = (double)tp.lo;
      Dbg.hi[tile] = (double)tp.hi;
    }
    if (Dbg.counts)
      for (int b = lane; b < n; b += 32) Dbg.counts[tile * n + b] = cnt[b];
    if (tp_degenerate(tp.lim)) {  // histogram.cpp:95-98
      for (int b = lane; b < n; b += 32) {
        lut[b] = 0.5f;
        if (Dbg.clipped) Dbg.clipped[tile * n + b] = 0.0;
        if (Dbg.lut) Dbg.lut[tile * n + b] = 0.5;
      }
      if (Dbg.degenerate && lane == 0) Dbg.degenerate[tile] = 1;
      if constexpr (sizeof(T) == 4) {
        if (drows)
          for (int i = lane; i < kDictKC; i += 32)
            W.lutd[tile * kDictKC + i] =
                (i < dK && __float_as_uint(W.dvals[i]) != kDictEmpty) ? 0.5f : 0.0f;
      }
      continue;
    }
    // total = sum of counts (integers: exact in any order)
    unsigned long long tot = 0;
    for (int b = lane; b < n; b += 32) tot += cnt[b];
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const double threshold = __dmul_rn(G.clip, (double)tot);
    double excess = 0.0;
    for (int base = 0; base < n; base += 32) {
      const int b = base + lane;
      const double over = b < n ? __dsub_rn((double)cnt[b], threshold) : 0.0;
      unsigned m = __ballot_sync(0xffffffffu, over > 0.0);
      while (m) {
        const int src = __ffs(m) - 1;
        excess = __dadd_rn(excess, __shfl_sync(0xffffffffu, over, src));
        m &= m - 1;
      }
    }
    const double share = __ddiv_rn(excess, (double)n);
    for (int b = lane; b < n; b += 32) {
      const double c = (double)cnt[b];
      const double cl = __dadd_rn(c < threshold ? c : threshold, share);
      cdf[b] = cl;
      if (Dbg.clipped) Dbg.clipped[tile * n + b] = cl;
    }
    __syncwarp();
    if (lane == 0) {
      double run = 0.0;
      int b = 0;
      for (; b + 8 <= n; b += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = cdf[b + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          run = __dadd_rn(run, v[k]);
          cdf[b + k] = run;
        }
      }
      for (; b < n; ++b) {
        run = __dadd_rn(run, cdf[b]);
        cdf[b] = run;
      }
    }
    __syncwarp();
    const double first = cdf[0];
    const double span = __dsub_rn(cdf[n - 1], first);
    const bool degen = !(span > 0.0);
    for (int b = lane; b < n; b += 32) {
      const double m = degen ? 0.5 : __ddiv_rn(__dsub_rn(cdf[b], first), span);
      lut[b] = (float)m;
      if (Dbg.lut) Dbg.lut[tile * n + b] = m;
    }
    if (Dbg.degenerate && lane == 0) Dbg.degenerate[tile] = degen ? 1 : 0;
    __syncwarp();
    if constexpr (sizeof(T) == 4) {
      if (drows) {
        for (int b = lane; b < n; b += 32) lutf[b] = lut[b];  // own writes, read back
        __syncwarp();
        const float* th = W.thr + tile * (n + 1);
        for (int i = lane; i < kDictKC; i += 32) {
          float r = 0.0f;
          if (i < dK && __float_as_uint(W.dvals[i]) != kDictEmpty)  // direct cells: holes stay 0
            r = lutf[bin_of((T)W.dvals[i], tp, th, n, nm05)];
          W.lutd[tile * kDictKC + i] = r;
        }
        __syncwarp();
      }
    }
  }
}

// -------------------------------------------------------- K4 generic -----
template <typename T, bool ADAPT>
__global__ void __launch_bounds__(256) k_interp_generic(const KGeom G, const T* __restrict__ in,
                                                        T* __restrict__ out, WS W) {
  if (W.range[2] != 0) return;
  const int n = G.n_bins;
  const T nm05 = (T)n - (T)0.5;
  const TileParam<T>* tparams = reinterpret_cast<const TileParam<T>*>(W.tparams);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < G.local_voxels;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t x[kMaxRank], c[kMaxRank];
    double f1[kMaxRank];
    decode_local(G, idx, x);
    const T v = in[idx];
    for (int j = 0; j < G.rank; ++j) {
      c[j] = cell_of(G.d[j], x[j]);
      f1[j] = (double)twice_dlo(G.d[j], x[j], c[j]) / (double)(2 * G.d[j].b);
    }
    const int corners = 1 << G.rank;
    const int bg = ADAPT ? 0 : bin_of(v, tparams[0], thr_row<T>(W, 0, n), n, nm05);
    double acc = 0.0;
    for (int co = 0; co < corners; ++co) {
      int64_t t[kMaxRank];
      double w = 1.0;
      for (int j = 0; j < G.rank; ++j) {
        const int bit = (co >> (G.rank - 1 - j)) & 1;
        t[j] = c[j] + bit;
        w *= bit ? f1[j] : 1.0 - f1[j];
      }
      const int64_t f = window_tile(G, t);
      const int b = ADAPT ? bin_of(v, tparams[f], thr_row<T>(W, f, n), n, nm05) : bg;
      acc += w * (double)W.lut[f * n + b];
    }
    out[idx] = (T)fmin(fmax(acc, 0.0), 1.0);
  }
}

// ------------------------------------------------------- debug binning ---
// Bin-edge tables for every binning range (f32 data): thr[t][k] = smallest
// float whose reference bin is >= k; thr[t][0] = -inf.
__global__ void k_thresholds(const KGeom G, WS W, int64_t t0, int64_t nt) {
  const TileParam<float>* tp = reinterpret_cast<const TileParam<float>*>(W.tparams);
  const int n = G.n_bins, n1 = n + 1;
  const int64_t first = (G.adaptive ? t0 : 0) * (int64_t)n1;
  const int64_t total = first + (G.adaptive ? nt : 1) * (int64_t)n1;
  for (int64_t i = first + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / n1;
    const int k = (int)(i - t * n1);
    const TileParam<float> p = tp[t];
    W.thr[i] = k == n ? INFINITY
                      : (k == 0 || tp_degenerate(p.lim))
                            ? -INFINITY
                            : bin_threshold((double)p.lo, (double)p.hi, n, k);
  }
}

__global__ void k_debug_thresholds(double lo, double hi, int n, float* thr) {
  const TileParam<float> p = make_tile_param<float>(lo, hi, n);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= n; k += gridDim.x * blockDim.x)
    thr[k] = k == n ? INFINITY
                    : (k == 0 || tp_degenerate(p.lim)) ? -INFINITY
                                                       : bin_threshold((double)p.lo, (double)p.hi, n, k);
}

template <typename T>
__global__ void k_debug_bins(const T* __restrict__ v, int64_t count, double lo, double hi, int n,
                             const T* thr, int32_t* __restrict__ out) {
  const TileParam<T> tp = make_tile_param<T>(lo, hi, n);
  const T nm05 = (T)n - (T)0.5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = tp_degenerate(tp.lim) ? -1 : bin_of(v[i], tp, thr, n, nm05);
}

// The pencil kernels' packed binning (bins2_edge: histograms; lut2_edge:
// blend gathers, here through an identity LUT; bins2_bracket: the NB blend) on arbitrary values against
// one range, pairs of consecutive values per thread.
__global__ void k_debug_bins_packed(const float* __restrict__ v, int64_t count, double lo,
                                    double hi, int n, const float* thr, const float* lut,
                                    int variant, int32_t* __restrict__ out) {
  const TileParam<float> tp = make_tile_param_f32(lo, hi, n);
  const float2 lc = tile_lc(tp);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v0 = v[2 * i], v1 = 2 * i + 1 < count ? v[2 * i + 1] : v0;
    int b0, b1;
    if (tp_degenerate(tp.lim)) {
      b0 = b1 = -1;
    } else if (isnan(lc.y)) {
      b0 = bin_search(v0, thr, n);
      b1 = bin_search(v1, thr, n);
    } else if (variant == 1) {
      bins2_edge(pk2(v0, v1), v0, v1, lc, thr, n, b0, b1);
    } else if (variant == 3) {
      const float2 w = bin_window(lc.y);
      if (w.y < INFINITY) {
        bins2_bracket(pk2(v0, v1), v0, v1, lc.x, w, thr, n, b0, b1);
      } else {
        b0 = bin_search(v0, thr, n);
        b1 = bin_search(v1, thr, n);
      }
    } else {
      float m0, m1;
      lut2_edge(pk2(v0, v1), v0, v1, lc, reinterpret_cast<const char*>(thr),
                reinterpret_cast<const char*>(lut), 4 * n, m0, m1);
      b0 = (int)m0;
      b1 = (int)m1;
    }
    out[2 * i] = b0;
    if (2 * i + 1 < count) out[2 * i + 1] = b1;
  }
}

__global__ void k_debug_identity(float* lut, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    lut[k] = (float)k;
}

}  // namespace mg
