// k_tile.cu -- tile-major K2 for the shapes and dtypes the pencil kernels do
// not take (float64 data -- the reference's own element type --, ragged
// mirror splits along trailing dims, oversized shared memory).
//
// One CTA owns one window tile at a time: it walks the tile's support box
// (the union of the mirror intervals of every dim, geometry.h tile_parts) --
// every input voxel the padded tile holds, each read once, weighted by its
// multiplicity -- and builds the tile's histogram in shared memory.  No global
// atomics (the old one-voxel-per-thread kernels hammered each tile's range
// and bin words from thousands of threads).
//
//   MODE 0  per-tile min / max + finiteness (build_mappings' adaptive range,
//           src/histogram.cpp:86-94) into the MAX-reducible range keys
//   MODE 1  counts with the tile's binning parameters (compute_histogram,
//           src/histogram.cpp:34-40, exact bin rule of bin_of)
//   MODE 2  both in one kernel (single-slab adaptive plans): min / max, the
//           tile's parameters, then the counts -- the second walk over the
//           support hits L2 (one tile's support per CTA is a few hundred KB)
//
// Counts are stored, not added: the CTA is the only writer of its tile's
// row (slab plans write their partial counts; the exchange sums them).
#include <cfloat>

#include "common.cuh"

namespace mg {
namespace {

constexpr int kTileThreads = 256;

// edge table of a binning range (float data; f64 data takes the exact rule)
template <typename T>
__device__ __forceinline__ const T* edge_row(const WS& W, int64_t idx, int n);
template <>
__device__ __forceinline__ const float* edge_row<float>(const WS& W, int64_t idx, int n) {
  return W.thr + idx * (n + 1);
}
template <>
__device__ __forceinline__ const double* edge_row<double>(const WS&, int64_t, int) {
  return nullptr;
}

// A box of original voxels (a tile's support or an interpolation cell),
// walked k = tid, tid + S, ... last dim fastest with a mixed-radix
// multi-index: one stride-digit add with carries per step, no per-voxel
// division (the 64-bit div / mod per dim per voxel dominated these kernels).
// Extents and coordinates are 32-bit (dim extents < 2^31).
struct Box {
  int32_t a[kMaxRank];    // first original coordinate per dim (dim 0: global row)
  int32_t ext[kMaxRank];  // extents
  int32_t sd[kMaxRank];   // digits of the walk stride kTileThreads in radix ext
  int32_t sdr[kMaxRank];  // the same over dims 0 .. D-2 (row walks, last dim excluded)
  int64_t base;           // input offset of the box origin (slab-local)
  int32_t n;              // voxels in the box
};

__device__ __forceinline__ void box_finish(const KGeom& G, Box& B) {
  int64_t base = 0;
  int64_t n = 1;
  int32_t s = kTileThreads;
  for (int j = G.rank - 1; j >= 0; --j) {
    base += (int64_t)(j == 0 ? B.a[j] - G.row0 : B.a[j]) * G.vstride[j];
    n *= B.ext[j];
    B.sd[j] = B.ext[j] > 0 ? s % B.ext[j] : 0;
    s = B.ext[j] > 0 ? s / B.ext[j] : 0;
  }
  B.base = base;
  B.n = (int32_t)n;
  s = kTileThreads;
  for (int j = G.rank - 2; j >= 0; --j) {
    B.sdr[j] = B.ext[j] > 0 ? s % B.ext[j] : 0;
    s = B.ext[j] > 0 ? s / B.ext[j] : 0;
  }
}

// Row walk: the multi-index over dims 0 .. D-2 (a row = the box's extent along
// the contiguous last dim), stride kTileThreads rows.
struct RowWalk {
  int32_t idx[kMaxRank];
  __device__ __forceinline__ void init(const Box& B, int D, int32_t k) {
#pragma unroll
    for (int j = kMaxRank - 1; j >= 0; --j) {
      if (j >= D - 1) { idx[j] = 0; continue; }
      const int32_t e = B.ext[j];
      idx[j] = k % e;
      k /= e;
    }
  }
  __device__ __forceinline__ void step(const Box& B, int D) {
    int32_t carry = 0;
#pragma unroll
    for (int j = kMaxRank - 1; j >= 0; --j) {
      if (j >= D - 1) continue;
      int32_t v = idx[j] + B.sdr[j] + carry;
      carry = v >= B.ext[j];
      idx[j] = carry ? v - B.ext[j] : v;
    }
  }
  __device__ __forceinline__ int64_t offset(const KGeom& G, const Box& B, int D) const {
    int64_t off = B.base;
#pragma unroll
    for (int j = 0; j < kMaxRank; ++j)
      if (j < D - 1) off += (int64_t)idx[j] * G.vstride[j];
    return off;
  }
};

struct Walk {
  int32_t idx[kMaxRank];
  __device__ __forceinline__ void init(const Box& B, int D, int32_t k) {
#pragma unroll
    for (int j = kMaxRank - 1; j >= 0; --j) {
      if (j >= D) { idx[j] = 0; continue; }
      const int32_t e = B.ext[j];
      idx[j] = k % e;
      k /= e;
    }
  }
  __device__ __forceinline__ void step(const Box& B, int D) {
    int32_t carry = 0;
#pragma unroll
    for (int j = kMaxRank - 1; j >= 0; --j) {
      if (j >= D) continue;
      int32_t v = idx[j] + B.sd[j] + carry;
      carry = v >= B.ext[j];
      idx[j] = carry ? v - B.ext[j] : v;
    }
  }
  __device__ __forceinline__ int64_t offset(const KGeom& G, const Box& B, int D) const {
    int64_t off = B.base;
#pragma unroll
    for (int j = 0; j < kMaxRank; ++j)
      if (j < D) off += (int64_t)idx[j] * G.vstride[j];
    return off;
  }
};

// Tile multiplicities as 32-bit intervals (TileParts, 0..3 per dim)
struct Parts32 {
  int32_t id_a, id_e, lo_a, lo_e, hi_a, hi_e;
  __device__ __forceinline__ uint32_t weight(int32_t x) const {
    return (uint32_t)(x >= id_a && x < id_e) + (uint32_t)(x >= lo_a && x < lo_e) +
           (uint32_t)(x >= hi_a && x < hi_e);
  }
};

struct TileBox {
  Box b;
  Parts32 tp[kMaxRank];
};

__device__ __forceinline__ void tile_box(const KGeom& G, int64_t f, TileBox& T) {
  int64_t t[kMaxRank];
  int64_t r = f;
  for (int j = G.rank - 1; j > 0; --j) {
    t[j] = r % G.d[j].g;
    r /= G.d[j].g;
  }
  t[0] = r + G.trow0;
  const int64_t row_end = G.row0 + G.local_voxels / G.vstride[0];
  for (int j = 0; j < G.rank; ++j) {
    const TileParts p = tile_parts(G.d[j], t[j]);
    T.tp[j] = Parts32{(int32_t)p.id_a, (int32_t)p.id_e, (int32_t)p.lo_a, (int32_t)p.lo_e,
                      (int32_t)p.hi_a, (int32_t)p.hi_e};
    int64_t a = p.support_begin(), e = p.support_end();
    if (j == 0) {
      a = a > G.row0 ? a : G.row0;
      e = e < row_end ? e : row_end;
    }
    T.b.a[j] = (int32_t)a;
    T.b.ext[j] = (int32_t)(e > a ? e - a : 0);
  }
  box_finish(G, T.b);
}

// accum: the workspace is shared with other plans (chunks of the streamed
// one-shot call), so keys are MAX-combined and counts added
template <typename T, int MODE>
__global__ void __launch_bounds__(kTileThreads, 2)
    k_tile_major(const KGeom G, const T* __restrict__ in, WS W, int accum) {
  extern __shared__ __align__(16) uint32_t hist[];  // [n_bins] (MODE 1 / 2)
  __shared__ TileBox TB;
  __shared__ int64_t s_klo[kTileThreads / 32], s_khi[kTileThreads / 32];
  __shared__ TileParam<T> s_tp;
  const int n = G.n_bins;
  const int D = G.rank;
  const T nm05 = (T)n - (T)0.5;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  TileParam<T>* tparams = reinterpret_cast<TileParam<T>*>(W.tparams);
  int bad = 0;
  for (int64_t f = blockIdx.x; f < G.win_tiles; f += gridDim.x) {
    if (tid == 0) tile_box(G, f, TB);
    __syncthreads();
    const Box& B = TB.b;
    const int32_t nv = B.n;
    if (MODE != 1) {  // range of the tile's support
      T lo = (T)INFINITY, hi = -(T)INFINITY;
      const int32_t L = B.ext[D - 1], nrows = L > 0 ? nv / L : 0;
      RowWalk w;
      if (tid < nrows) w.init(B, D, tid);
      for (int32_t r = tid; r < nrows; r += kTileThreads, w.step(B, D)) {
        const T* row = in + w.offset(G, B, D);
        int32_t i = 0;
        for (; i + 4 <= L; i += 4) {  // four loads in flight
          T v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = row[i + q];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            bad |= !isfinite(v[q]);
            lo = fmin(lo, v[q]);
            hi = fmax(hi, v[q]);
          }
        }
        for (; i < L; ++i) {
          const T v = row[i];
          bad |= !isfinite(v);
          lo = fmin(lo, v);
          hi = fmax(hi, v);
        }
      }
      int64_t klo = lo <= hi ? okey((double)lo) : INT64_MAX;
      int64_t khi = lo <= hi ? okey((double)hi) : INT64_MIN;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t a = __shfl_xor_sync(0xffffffffu, klo, o);
        const int64_t b = __shfl_xor_sync(0xffffffffu, khi, o);
        klo = a < klo ? a : klo;
        khi = b > khi ? b : khi;
      }
      if (lane == 0) {
        s_klo[wid] = klo;
        s_khi[wid] = khi;
      }
      __syncthreads();
      if (tid == 0) {
        for (int i = 1; i < kTileThreads / 32; ++i) {
          klo = s_klo[i] < klo ? s_klo[i] : klo;
          khi = s_khi[i] > khi ? s_khi[i] : khi;
        }
        if (nv > 0 && accum) {
          atomicMax(reinterpret_cast<long long*>(W.trange + 2 * f), (long long)~klo);
          atomicMax(reinterpret_cast<long long*>(W.trange + 2 * f + 1), (long long)khi);
        } else if (nv > 0) {  // an empty box (window row outside the slab) keeps the reset keys
          W.trange[2 * f] = ~klo;
          W.trange[2 * f + 1] = khi;
        }
        if (MODE == 2) s_tp = make_tile_param<T>(okey_decode(klo), okey_decode(khi), n);
      }
    }
    if (MODE != 0) {  // counts of the tile's support
      if (MODE == 1 && tid == 0) s_tp = tparams[G.adaptive ? f : 0];
      for (int b = tid; b < n; b += kTileThreads) hist[b] = 0;
      __syncthreads();
      const TileParam<T> tp = s_tp;
      if (!tp_degenerate(tp.lim)) {  // degenerate tiles are never binned (histogram.cpp:95-98)
        const T* thr = edge_row<T>(W, G.adaptive ? f : 0, n);
        const int32_t L = B.ext[D - 1], nrows = L > 0 ? nv / L : 0;
        const int32_t aL = B.a[D - 1];
        RowWalk w;
        if (tid < nrows) w.init(B, D, tid);
        for (int32_t r = tid; r < nrows; r += kTileThreads, w.step(B, D)) {
          const T* row = in + w.offset(G, B, D);
          uint32_t mrow = 1;  // multiplicity over dims 0 .. D-2
#pragma unroll
          for (int j = 0; j < kMaxRank; ++j)
            if (j < D - 1) mrow *= TB.tp[j].weight(B.a[j] + w.idx[j]);
          // runs of equal bins along the row merge into one shared add
          int prev = -1;
          uint32_t acc = 0;
          int32_t i = 0;
          for (; i < L; i += 4) {
            T v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = i + q < L ? row[i + q] : (T)0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (i + q >= L) break;
              const int b = bin_of(v[q], tp, thr, n, nm05);
              const uint32_t m = mrow * TB.tp[D - 1].weight(aL + i + q);
              if (b == prev) {
                acc += m;
              } else {
                if (prev >= 0 && acc) atomicAdd(&hist[prev], acc);
                prev = b;
                acc = m;
              }
            }
          }
          if (prev >= 0 && acc) atomicAdd(&hist[prev], acc);
        }
      }
      __syncthreads();
      if (accum) {
        for (int b = tid; b < n; b += kTileThreads)
          if (hist[b]) atomicAdd(W.counts + f * n + b, hist[b]);
      } else {
        for (int b = tid; b < n; b += kTileThreads) W.counts[f * n + b] = hist[b];
      }
    }
    __syncthreads();
  }
  if (MODE != 1 && bad) atomicMax(reinterpret_cast<long long*>(&W.range[2]), 1LL);
}

// ------------------------------------------------------------- K4 -----
// Cell-major blend for the same shapes / dtypes: one CTA per interpolation
// cell (the box of original voxels sharing one set of 2^D neighbour tiles,
// src/interpolation.cpp:24-35).  The 2^D corner LUTs and binning parameters
// and every position's per-dim factor d_lo / b (exact half-integer
// numerators) are staged in shared memory once per cell; voxels are walked
// last dim fastest (coalesced) without divisions.  Per voxel: 2^D exact bins
// (bin_of: the reference rule in the data's own precision) and the f64 sum
// of w * LUT, clamped.
struct CellBox {
  Box b;
  int64_t cc[kMaxRank];
  int32_t foff[kMaxRank];  // per-dim offset into the factor table
};

// Per corner binning constants: the f64 reference rule evaluated through an
// f32 estimate with a guard band (as binning.cuh does for float data): y =
// fl32(fl32(v - lo) * fl32(c)) is within 1.8e-7 * n of the reference value q,
// so when frac(y) is further than that from an integer floor(y) is the
// reference bin; otherwise (rare for continuous data) the exact rule.
struct CornerBin {
  double lo;
  float c, lim;  // lim < 0: always exact; degenerate tiles: c = 0, lim = 2 (bin 0)
};

template <typename T>
__device__ __forceinline__ CornerBin corner_bin(const TileParam<T>& tp, int n) {
  CornerBin cb;
  cb.lo = (double)tp.lo;
  const float c32 = (float)tp.c;
  if (tp_degenerate(tp.lim)) {
    cb.c = 0.0f;
    cb.lim = 2.0f;
  } else {
    const bool ok = tp.lim > 0 && isfinite(c32) && c32 >= FLT_MIN && n <= (1 << 20);
    cb.c = ok ? c32 : 0.0f;
    cb.lim = ok ? 0.5f - (float)n * 2.5e-7f : -1.0f;
  }
  return cb;
}

// the exact rule, out of line: the unrolled corner loops keep one call site
// each instead of a copy of the f64 divide sequence
template <typename T>
__device__ __noinline__ int exact_bin(T v, const TileParam<T>* tpp, const T* thr, int n, T nm05) {
  return bin_of(v, *tpp, thr, n, nm05);
}

// The corner's constants are read from shared memory at every use (volatile):
// hoisted out of the voxel loop, 2^D corners' worth would spill.
template <typename T>
__device__ __forceinline__ int corner_bin_of(T v, const CornerBin* cbp, const TileParam<T>* tpp,
                                             const T* thr, int n, T nm05, float nm05f) {
  const volatile CornerBin* vc = cbp;
  const double lo = vc->lo;
  const float c = vc->c, lim = vc->lim;
  float y = __fmul_rn(__double2float_rn((double)v - lo), c);
  y = fminf(fmaxf(y, 0.5f), nm05f);
  const float t = __fadd_rd(y, 12582912.0f);  // floor(y) + 1.5 * 2^23
  const float fr = __fsub_rn(y, __fsub_rn(t, 12582912.0f));
  if (fabsf(__fsub_rn(fr, 0.5f)) < lim) return __float_as_int(t) - 0x4B400000;
  return exact_bin(v, tpp, thr, n, nm05);  // the reference rule in the data's precision
}

// DC: the rank when it is small enough to unroll (the corner weights are then
// built by doubling, one multiply per corner); 0 = any rank, per-corner products.
template <typename T, bool ADAPT, int DC>
__global__ void __launch_bounds__(kTileThreads, 2)
    k_interp_cell(const KGeom G, const T* __restrict__ in, T* __restrict__ out, WS W,
                  int64_t cell0, int64_t ncells0) {
  extern __shared__ __align__(16) float lutS[];  // [2^D][n], then the factor table
  __shared__ TileParam<T> tpS[1 << kMaxRank];
  __shared__ CornerBin cbS[1 << kMaxRank];
  __shared__ int32_t tileS[1 << kMaxRank];
  __shared__ CellBox C;
  if (W.range[2] != 0) return;  // non-finite input: write nothing
  const int D = DC ? DC : G.rank, NC = 1 << D, n = G.n_bins;
  double* facS = reinterpret_cast<double*>(lutS + ((NC * n + 1) & ~1));  // [sum of cell extents]
  const T nm05 = (T)n - (T)0.5;
  const float nm05f = (float)n - 0.5f;
  const TileParam<T>* tparams = reinterpret_cast<const TileParam<T>*>(W.tparams);
  const int64_t row_end = G.row0 + G.local_voxels / G.vstride[0];
  int64_t ncells = ncells0;  // the slab's dim-0 cells x every cell of the other dims
  for (int j = 1; j < D; ++j) ncells *= G.d[j].g - 1;
  for (int64_t c = blockIdx.x; c < ncells; c += gridDim.x) {
    if (threadIdx.x == 0) {
      int64_t r = c;
      for (int j = D - 1; j > 0; --j) {
        C.cc[j] = r % (G.d[j].g - 1);
        r /= G.d[j].g - 1;
      }
      C.cc[0] = cell0 + r;
      int32_t fo = 0;
      for (int j = 0; j < D; ++j) {
        int64_t a, e;
        cell_range(G.d[j], C.cc[j], &a, &e);
        if (j == 0) {
          a = a > G.row0 ? a : G.row0;
          e = e < row_end ? e : row_end;
        }
        C.b.a[j] = (int32_t)a;
        C.b.ext[j] = (int32_t)(e > a ? e - a : 0);
        C.foff[j] = fo;
        fo += C.b.ext[j];
      }
      box_finish(G, C.b);
    }
    __syncthreads();
    if (threadIdx.x < NC) {  // corner co: tile cc + bits (dimension 0 the MSB)
      int64_t f = (C.cc[0] + ((threadIdx.x >> (D - 1)) & 1) - G.trow0) * G.tstride[0];
      for (int j = 1; j < D; ++j) f += (C.cc[j] + ((threadIdx.x >> (D - 1 - j)) & 1)) * G.tstride[j];
      tileS[threadIdx.x] = (int32_t)f;
      const TileParam<T> tp = tparams[ADAPT ? f : 0];
      tpS[threadIdx.x] = tp;
      cbS[threadIdx.x] = corner_bin(tp, n);
    }
    for (int j = 0; j < D; ++j)  // factors d_lo / b of the cell's positions
      for (int i = threadIdx.x; i < C.b.ext[j]; i += kTileThreads)
        facS[C.foff[j] + i] =
            (double)twice_dlo(G.d[j], (int64_t)C.b.a[j] + i, C.cc[j]) / (double)(2 * G.d[j].b);
    __syncthreads();
    for (int k = threadIdx.x; k < NC * n; k += kTileThreads) {
      const int co = k / n;
      lutS[k] = W.lut[(int64_t)tileS[co] * n + (k - co * n)];
    }
    __syncthreads();
    const Box& B = C.b;
    const int32_t nv = B.n;
    if constexpr (DC > 0) {
      // rows along the contiguous last dim: the weights of dims 0 .. D-2 once
      // per row (doubling, dim 0 the MSB), four voxel loads in flight
      constexpr int NH = 1 << (DC - 1);
      const int32_t L = B.ext[DC - 1], nrows = L > 0 ? nv / L : 0;
      const double* facL = facS + C.foff[DC - 1];
      RowWalk rw;
      if ((int32_t)threadIdx.x < nrows) rw.init(B, DC, threadIdx.x);
      for (int32_t r = threadIdx.x; r < nrows; r += kTileThreads, rw.step(B, DC)) {
        const int64_t off = rw.offset(G, B, DC);
        double wh[NH];
        wh[0] = 1.0;
#pragma unroll
        for (int j = 0; j < DC - 1; ++j) {
          const double g = facS[C.foff[j] + rw.idx[j]];
#pragma unroll
          for (int q = (1 << j) - 1; q >= 0; --q) {
            wh[2 * q + 1] = wh[q] * g;
            wh[2 * q] = wh[q] * (1.0 - g);
          }
        }
        for (int32_t i = 0; i < L; i += 4) {
          T v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = i + q < L ? in[off + i + q] : (T)0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (i + q >= L) break;
            const double g = facL[i + q];
            const int bg = ADAPT ? 0 : corner_bin_of(v[q], &cbS[0], &tpS[0], edge_row<T>(W, 0, n), n, nm05, nm05f);
            double acc = 0.0;  // f64 weights and sum: a constant LUT blends to exactly itself
#pragma unroll
            for (int co = 0; co < (1 << DC); ++co) {
              const int b = ADAPT ? corner_bin_of(v[q], &cbS[co], &tpS[co], edge_row<T>(W, tileS[co], n), n,
                                                  nm05, nm05f)
                                  : bg;
              acc = fma(wh[co >> 1] * ((co & 1) ? g : 1.0 - g), (double)lutS[co * n + b], acc);
            }
            out[off + i + q] = (T)fmin(fmax(acc, 0.0), 1.0);
          }
        }
      }
    } else {
      Walk w;
      if ((int32_t)threadIdx.x < nv) w.init(B, D, threadIdx.x);
      for (int32_t k = threadIdx.x; k < nv; k += kTileThreads, w.step(B, D)) {
        const int64_t off = w.offset(G, B, D);
        const T v = in[off];
        const int bg = ADAPT ? 0 : corner_bin_of(v, &cbS[0], &tpS[0], edge_row<T>(W, 0, n), n, nm05, nm05f);
        double g1[kMaxRank];
#pragma unroll
        for (int j = 0; j < kMaxRank; ++j) g1[j] = j < D ? facS[C.foff[j] + w.idx[j]] : 0.0;
        double acc = 0.0;
        for (int co = 0; co < NC; ++co) {
          double wt = 1.0;
#pragma unroll
          for (int j = 0; j < kMaxRank; ++j)
            if (j < D) wt *= ((co >> (D - 1 - j)) & 1) ? g1[j] : 1.0 - g1[j];
          const int b = ADAPT ? corner_bin_of(v, &cbS[co], &tpS[co], edge_row<T>(W, tileS[co], n), n, nm05, nm05f)
                              : bg;
          acc = fma(wt, (double)lutS[co * n + b], acc);
        }
        out[off] = (T)fmin(fmax(acc, 0.0), 1.0);
      }
    }
    __syncthreads();
  }
}

template <typename T, bool ADAPT>
void launch_cell_t(int rank, int grid, size_t smem, cudaStream_t st, const KGeom& G, const T* x, T* y, WS W,
                   int64_t c0, int64_t nc) {
  switch (rank) {
    case 1: k_interp_cell<T, ADAPT, 1><<<grid, kTileThreads, smem, st>>>(G, x, y, W, c0, nc); break;
    case 2: k_interp_cell<T, ADAPT, 2><<<grid, kTileThreads, smem, st>>>(G, x, y, W, c0, nc); break;
    case 3: k_interp_cell<T, ADAPT, 3><<<grid, kTileThreads, smem, st>>>(G, x, y, W, c0, nc); break;
    case 4: k_interp_cell<T, ADAPT, 4><<<grid, kTileThreads, smem, st>>>(G, x, y, W, c0, nc); break;
    case 5: k_interp_cell<T, ADAPT, 5><<<grid, kTileThreads, smem, st>>>(G, x, y, W, c0, nc); break;
    default: k_interp_cell<T, ADAPT, 0><<<grid, kTileThreads, smem, st>>>(G, x, y, W, c0, nc); break;
  }
}

}  // namespace

// Cell-major blend launch (k_interp_cell); shared memory 2^D * n_bins floats.
void launch_interp_cell(int dtype_f64, int adaptive, int grid, cudaStream_t st, const KGeom& G,
                        const void* in, void* out, WS W, int64_t cell0, int64_t ncells0) {
  size_t fac = 0;  // factor table: one float per position of each dim's largest cell
  for (int j = 0; j < G.rank; ++j) fac += (size_t)G.d[j].b + 1;
  const size_t smem = ((((size_t)1 << G.rank) * (size_t)G.n_bins + 1) & ~(size_t)1) * 4 + fac * 8;
  if (dtype_f64) {
    const double* x = static_cast<const double*>(in);
    double* y = static_cast<double*>(out);
    if (adaptive) launch_cell_t<double, true>(G.rank, grid, smem, st, G, x, y, W, cell0, ncells0);
    else launch_cell_t<double, false>(G.rank, grid, smem, st, G, x, y, W, cell0, ncells0);
  } else {
    const float* x = static_cast<const float*>(in);
    float* y = static_cast<float*>(out);
    if (adaptive) launch_cell_t<float, true>(G.rank, grid, smem, st, G, x, y, W, cell0, ncells0);
    else launch_cell_t<float, false>(G.rank, grid, smem, st, G, x, y, W, cell0, ncells0);
  }
}

// Host accessors (mclahe_gpu.cu): MODE 0 / 1 / 2 for float or double.
void launch_tile_major(int dtype_f64, int mode, int grid, cudaStream_t st, const KGeom& G,
                       const void* in, WS W, int accum) {
  const size_t smem = mode == 0 ? 0 : (size_t)G.n_bins * 4;
  if (dtype_f64) {
    const double* x = static_cast<const double*>(in);
    if (mode == 0) k_tile_major<double, 0><<<grid, kTileThreads, smem, st>>>(G, x, W, accum);
    else if (mode == 1) k_tile_major<double, 1><<<grid, kTileThreads, smem, st>>>(G, x, W, accum);
    else k_tile_major<double, 2><<<grid, kTileThreads, smem, st>>>(G, x, W, accum);
  } else {
    const float* x = static_cast<const float*>(in);
    if (mode == 0) k_tile_major<float, 0><<<grid, kTileThreads, smem, st>>>(G, x, W, accum);
    else k_tile_major<float, 1><<<grid, kTileThreads, smem, st>>>(G, x, W, accum);
  }
}

cudaError_t tile_major_smem_cap(int max_smem) {
#define MG_CELL_FNS(T, A)                                                          \
  reinterpret_cast<const void*>(k_interp_cell<T, A, 0>),                           \
      reinterpret_cast<const void*>(k_interp_cell<T, A, 1>),                       \
      reinterpret_cast<const void*>(k_interp_cell<T, A, 2>),                       \
      reinterpret_cast<const void*>(k_interp_cell<T, A, 3>),                       \
      reinterpret_cast<const void*>(k_interp_cell<T, A, 4>),                       \
      reinterpret_cast<const void*>(k_interp_cell<T, A, 5>)
  const void* fns[] = {reinterpret_cast<const void*>(k_tile_major<double, 1>),
                       reinterpret_cast<const void*>(k_tile_major<double, 2>),
                       reinterpret_cast<const void*>(k_tile_major<float, 1>),
                       MG_CELL_FNS(double, true), MG_CELL_FNS(double, false),
                       MG_CELL_FNS(float, true), MG_CELL_FNS(float, false)};
#undef MG_CELL_FNS
  for (const void* f : fns) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_smem - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mg
