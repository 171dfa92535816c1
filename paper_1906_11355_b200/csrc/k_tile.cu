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

}  // namespace

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
                       reinterpret_cast<const void*>(k_tile_major<float, 1>)};
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
