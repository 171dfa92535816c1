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

struct SupportBox {
  int64_t a[kMaxRank];    // first original coordinate per dim (dim 0: global row)
  int64_t ext[kMaxRank];  // extents
  TileParts tp[kMaxRank];
  int64_t n;              // voxels in the box
};

__device__ __forceinline__ void tile_box(const KGeom& G, int64_t f, SupportBox& B) {
  int64_t t[kMaxRank];
  int64_t r = f;
  for (int j = G.rank - 1; j > 0; --j) {
    t[j] = r % G.d[j].g;
    r /= G.d[j].g;
  }
  t[0] = r + G.trow0;
  const int64_t row_end = G.row0 + G.local_voxels / G.vstride[0];
  B.n = 1;
  for (int j = 0; j < G.rank; ++j) {
    B.tp[j] = tile_parts(G.d[j], t[j]);
    int64_t a = B.tp[j].support_begin(), e = B.tp[j].support_end();
    if (j == 0) {
      a = a > G.row0 ? a : G.row0;
      e = e < row_end ? e : row_end;
    }
    B.a[j] = a;
    B.ext[j] = e > a ? e - a : 0;
    B.n *= B.ext[j];
  }
}

// k-th voxel of the box (last dim fastest): input offset and multiplicity
__device__ __forceinline__ int64_t box_voxel(const KGeom& G, const SupportBox& B, int64_t k,
                                             uint32_t* w) {
  int64_t off = 0;
  uint32_t m = 1;
  for (int j = G.rank - 1; j >= 0; --j) {
    const int64_t x = B.a[j] + k % B.ext[j];
    k /= B.ext[j];
    m *= (uint32_t)B.tp[j].weight(x);
    off += (j == 0 ? x - G.row0 : x) * G.vstride[j];
  }
  *w = m;
  return off;
}

// accum: the workspace is shared with other plans (chunks of the streamed
// one-shot call), so keys are MAX-combined and counts added
template <typename T, int MODE>
__global__ void __launch_bounds__(kTileThreads)
    k_tile_major(const KGeom G, const T* __restrict__ in, WS W, int accum) {
  extern __shared__ __align__(16) uint32_t hist[];  // [n_bins] (MODE 1 / 2)
  __shared__ SupportBox B;
  __shared__ int64_t s_klo[kTileThreads / 32], s_khi[kTileThreads / 32];
  __shared__ TileParam<T> s_tp;
  const int n = G.n_bins;
  const T nm05 = (T)n - (T)0.5;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  TileParam<T>* tparams = reinterpret_cast<TileParam<T>*>(W.tparams);
  int bad = 0;
  for (int64_t f = blockIdx.x; f < G.win_tiles; f += gridDim.x) {
    if (tid == 0) tile_box(G, f, B);
    __syncthreads();
    const int64_t nv = B.n;
    if (MODE != 1) {  // range of the tile's support
      int64_t klo = INT64_MAX, khi = INT64_MIN;
      for (int64_t k = tid; k < nv; k += kTileThreads) {
        uint32_t w;
        const T v = in[box_voxel(G, B, k, &w)];
        bad |= !isfinite(v);
        const int64_t key = okey((double)v);
        klo = key < klo ? key : klo;
        khi = key > khi ? key : khi;
      }
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
        for (int64_t k = tid; k < nv; k += kTileThreads) {
          uint32_t w;
          const T v = in[box_voxel(G, B, k, &w)];
          atomicAdd(&hist[bin_of(v, tp, thr, n, nm05)], w);
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
// are staged in shared memory once per cell; voxels are walked last dim
// fastest (coalesced), with 32-bit index arithmetic inside the box.  Per
// voxel: the per-dim factors d_lo / b (exact half-integer numerators), 2^D
// bins (bin_of: the reference rule) and the f64 sum of w * LUT, clamped.
struct CellBox {
  int64_t a[kMaxRank];
  int32_t ext[kMaxRank];
  int64_t cc[kMaxRank];
  int64_t n;
};

template <typename T, bool ADAPT>
__global__ void __launch_bounds__(kTileThreads)
    k_interp_cell(const KGeom G, const T* __restrict__ in, T* __restrict__ out, WS W,
                  int64_t cell0, int64_t ncells0) {
  extern __shared__ __align__(16) float lutS[];  // [2^D][n]
  __shared__ TileParam<T> tpS[1 << kMaxRank];
  __shared__ int32_t tileS[1 << kMaxRank];
  __shared__ CellBox B;
  if (W.range[2] != 0) return;  // non-finite input: write nothing
  const int D = G.rank, NC = 1 << D, n = G.n_bins;
  const T nm05 = (T)n - (T)0.5;
  const TileParam<T>* tparams = reinterpret_cast<const TileParam<T>*>(W.tparams);
  const int64_t row_end = G.row0 + G.local_voxels / G.vstride[0];
  int64_t ncells = ncells0;  // the slab's dim-0 cells x every cell of the other dims
  for (int j = 1; j < D; ++j) ncells *= G.d[j].g - 1;
  for (int64_t c = blockIdx.x; c < ncells; c += gridDim.x) {
    if (threadIdx.x == 0) {
      int64_t r = c;
      for (int j = D - 1; j > 0; --j) {
        B.cc[j] = r % (G.d[j].g - 1);
        r /= G.d[j].g - 1;
      }
      B.cc[0] = cell0 + r;
      B.n = 1;
      for (int j = 0; j < D; ++j) {
        int64_t a, e;
        cell_range(G.d[j], B.cc[j], &a, &e);
        if (j == 0) {
          a = a > G.row0 ? a : G.row0;
          e = e < row_end ? e : row_end;
        }
        B.a[j] = a;
        B.ext[j] = (int32_t)(e > a ? e - a : 0);
        B.n *= B.ext[j];
      }
    }
    __syncthreads();
    if (threadIdx.x < NC) {  // corner co: tile cc + bits (dimension 0 the MSB)
      int64_t f = (B.cc[0] + ((threadIdx.x >> (D - 1)) & 1) - G.trow0) * G.tstride[0];
      for (int j = 1; j < D; ++j) f += (B.cc[j] + ((threadIdx.x >> (D - 1 - j)) & 1)) * G.tstride[j];
      tileS[threadIdx.x] = (int32_t)f;
      tpS[threadIdx.x] = tparams[ADAPT ? f : 0];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < NC * n; k += kTileThreads) {
      const int co = k / n;
      lutS[k] = W.lut[(int64_t)tileS[co] * n + (k - co * n)];
    }
    __syncthreads();
    const int64_t nv = B.n;
    for (int64_t k = threadIdx.x; k < nv; k += kTileThreads) {
      int64_t off = 0;
      double fl[kMaxRank];
      int64_t q = k;
      for (int j = D - 1; j >= 0; --j) {
        const int32_t e = B.ext[j];
        const int32_t i = (int32_t)(q % e);
        q /= e;
        const int64_t x = B.a[j] + i;
        off += (j == 0 ? x - G.row0 : x) * G.vstride[j];
        fl[j] = (double)twice_dlo(G.d[j], x, B.cc[j]) / (double)(2 * G.d[j].b);
      }
      const T v = in[off];
      const int bg = ADAPT ? 0 : bin_of(v, tpS[0], edge_row<T>(W, 0, n), n, nm05);
      double acc = 0.0;
      for (int co = 0; co < NC; ++co) {
        double w = 1.0;
        for (int j = 0; j < D; ++j) w *= ((co >> (D - 1 - j)) & 1) ? fl[j] : 1.0 - fl[j];
        const int b = ADAPT ? bin_of(v, tpS[co], edge_row<T>(W, tileS[co], n), n, nm05) : bg;
        acc += w * (double)lutS[co * n + b];
      }
      out[off] = (T)fmin(fmax(acc, 0.0), 1.0);
    }
    __syncthreads();
  }
}

}  // namespace

// Cell-major blend launch (k_interp_cell); shared memory 2^D * n_bins floats.
void launch_interp_cell(int dtype_f64, int adaptive, int grid, cudaStream_t st, const KGeom& G,
                        const void* in, void* out, WS W, int64_t cell0, int64_t ncells0) {
  const size_t smem = ((size_t)1 << G.rank) * (size_t)G.n_bins * 4;
  if (dtype_f64) {
    const double* x = static_cast<const double*>(in);
    double* y = static_cast<double*>(out);
    if (adaptive) k_interp_cell<double, true><<<grid, kTileThreads, smem, st>>>(G, x, y, W, cell0, ncells0);
    else k_interp_cell<double, false><<<grid, kTileThreads, smem, st>>>(G, x, y, W, cell0, ncells0);
  } else {
    const float* x = static_cast<const float*>(in);
    float* y = static_cast<float*>(out);
    if (adaptive) k_interp_cell<float, true><<<grid, kTileThreads, smem, st>>>(G, x, y, W, cell0, ncells0);
    else k_interp_cell<float, false><<<grid, kTileThreads, smem, st>>>(G, x, y, W, cell0, ncells0);
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
  const void* fns[] = {reinterpret_cast<const void*>(k_tile_major<double, 1>),
                       reinterpret_cast<const void*>(k_tile_major<double, 2>),
                       reinterpret_cast<const void*>(k_tile_major<float, 1>),
                       reinterpret_cast<const void*>(k_interp_cell<double, true>),
                       reinterpret_cast<const void*>(k_interp_cell<double, false>),
                       reinterpret_cast<const void*>(k_interp_cell<float, true>),
                       reinterpret_cast<const void*>(k_interp_cell<float, false>)};
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
