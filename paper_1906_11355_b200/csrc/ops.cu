// ops.cu -- the reference's per-operation public API on the device, for
// callers of the reference headers that use the building blocks directly
// instead of mclahe::mclahe (include/mclahe/{nd_image,histogram}.hpp):
//
//   mclahe_block_mappings  build_mappings / compute_histogram over the blocks
//                          of a KernelGrid (src/histogram.cpp:34-106): one CTA
//                          per block -- range (adaptive: the block's own
//                          min/max), shared-memory histogram with the exact
//                          f64 bin rule, then clip_histogram + normalized_cdf
//                          by one warp in the reference's summation order.
//   mclahe_nd_gather       symmetric_pad / kernelize / crop
//                          (src/nd_image.cpp:104-218): one gather kernel,
//                          every output element from its source index.
//
// The hot path (mclahe_gpu_run & co.) never materialises padded or
// block-major copies; these exist so a reference caller that does keeps
// compiling and gets identical results.  Host buffers in and out.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/mclahe_gpu.h"
#include "binning.cuh"
#include "host_err.h"

namespace mg {
namespace {

// First-of-the-minimal-class selection (NdImage::min_max /
// build_mappings' scan keeps the EARLIEST element among equal extremes and
// never lets a NaN replace a number): (value, index) pairs, NaN = empty.
struct Ext {
  double v;
  int64_t i;
};

__device__ __forceinline__ Ext pick_lo(Ext a, Ext b) {
  if (isnan(a.v)) return b;
  if (isnan(b.v)) return a;
  if (b.v < a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ Ext pick_hi(Ext a, Ext b) {
  if (isnan(a.v)) return b;
  if (isnan(b.v)) return a;
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ Ext shfl_ext(Ext e, int o) {
  Ext r;
  r.v = __shfl_xor_sync(0xffffffffu, e.v, o);
  r.i = __shfl_xor_sync(0xffffffffu, e.i, o);
  return r;
}

constexpr int kOpsThreads = 256;

// One CTA per block (grid-stride over blocks).  Shared memory: n u32 counts +
// n f64 CDF scratch.  want: 1 = counts only (compute_histogram), 2 = the full
// mapping (build_mappings).
__global__ void __launch_bounds__(kOpsThreads)
    k_block_mappings(const double* __restrict__ blocks, int64_t n_blocks, int64_t len, int n,
                     double clip, int adaptive, double glo, double ghi, int want,
                     double* __restrict__ lo_o, double* __restrict__ hi_o,
                     double* __restrict__ counts_o, double* __restrict__ clipped_o,
                     double* __restrict__ lut_o, uint8_t* __restrict__ deg_o) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
  double* cdf = reinterpret_cast<double*>(smem + ((n * 4 + 15) & ~15));
  __shared__ Ext s_lo[kOpsThreads / 32], s_hi[kOpsThreads / 32];
  __shared__ double s_range[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const double* b = blocks + blk * len;
    if (adaptive) {  // build_mappings (histogram.cpp:86-94): the block's own min/max
      Ext lo{NAN, 0}, hi{NAN, 0};
      for (int64_t k = tid; k < len; k += blockDim.x) {
        const Ext e{b[k], k};
        lo = pick_lo(lo, e);
        hi = pick_hi(hi, e);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = pick_lo(lo, shfl_ext(lo, o));
        hi = pick_hi(hi, shfl_ext(hi, o));
      }
      if (lane == 0) {
        s_lo[wid] = lo;
        s_hi[wid] = hi;
      }
      __syncthreads();
      if (tid == 0) {
        Ext L = s_lo[0], H = s_hi[0];
        for (int w = 1; w < kOpsThreads / 32; ++w) {
          L = pick_lo(L, s_lo[w]);
          H = pick_hi(H, s_hi[w]);
        }
        // the scan starts from the front element: a NaN there never leaves
        const bool front_nan = isnan(b[0]);
        s_range[0] = front_nan ? b[0] : L.v;
        s_range[1] = front_nan ? b[0] : H.v;
      }
    } else if (tid == 0) {
      s_range[0] = glo;
      s_range[1] = ghi;
    }
    for (int k = tid; k < n; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    const double lo = s_range[0], hi = s_range[1];
    const bool degen_range = !(lo < hi);  // IntensityRange::degenerate (histogram.hpp:27)
    if (tid == 0) {
      if (lo_o) lo_o[blk] = lo;
      if (hi_o) hi_o[blk] = hi;
    }
    if (!degen_range) {  // compute_histogram (histogram.cpp:34-40), exact f64 bins
      for (int64_t k = tid; k < len; k += blockDim.x) atomicAdd(&cnt[bin_exact(b[k], lo, hi, n)], 1u);
    }
    __syncthreads();
    if (counts_o)
      for (int k = tid; k < n; k += blockDim.x) counts_o[blk * n + k] = (double)cnt[k];
    if (want == 2 && wid == 0) {
      if (degen_range) {  // degenerate_mapping (histogram.cpp:17-19)
        for (int k = lane; k < n; k += 32) {
          lut_o[blk * n + k] = 0.5;
          if (clipped_o) clipped_o[blk * n + k] = 0.0;
        }
        if (lane == 0) deg_o[blk] = 1;
      } else {
        // clip_histogram (histogram.cpp:42-55): integer total (exact in any
        // order), excess summed in bin order over the positive terms (zero
        // terms are exact no-ops), share, min(c, T) + share
        unsigned long long tot = 0;
        for (int k = lane; k < n; k += 32) tot += cnt[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        const double thr = __dmul_rn(clip, (double)tot);
        double excess = 0.0;
        for (int base = 0; base < n; base += 32) {
          const int k = base + lane;
          const double over = k < n ? __dsub_rn((double)cnt[k], thr) : 0.0;
          unsigned m = __ballot_sync(0xffffffffu, over > 0.0);
          while (m) {
            const int src = __ffs(m) - 1;
            excess = __dadd_rn(excess, __shfl_sync(0xffffffffu, over, src));
            m &= m - 1;
          }
        }
        const double share = __ddiv_rn(excess, (double)n);
        for (int k = lane; k < n; k += 32) {
          const double c = (double)cnt[k];
          const double cl = __dadd_rn(thr < c ? thr : c, share);
          cdf[k] = cl;
          if (clipped_o) clipped_o[blk * n + k] = cl;
        }
        __syncwarp();
        if (lane == 0) {  // normalized_cdf (histogram.cpp:57-70): sequential prefix
          double run = 0.0;
          for (int k = 0; k < n; ++k) {
            run = __dadd_rn(run, cdf[k]);
            cdf[k] = run;
          }
        }
        __syncwarp();
        const double first = cdf[0];
        const double span = __dsub_rn(cdf[n - 1], first);
        const bool degen = !(span > 0.0);
        for (int k = lane; k < n; k += 32)
          lut_o[blk * n + k] = degen ? 0.5 : __ddiv_rn(__dsub_rn(cdf[k], first), span);
        if (lane == 0) deg_o[blk] = degen ? 1 : 0;
      }
    }
    __syncthreads();
  }
}

struct GatherGeom {
  int rank;
  int op;                    // 0 symmetric_pad, 1 kernelize, 2 crop
  int64_t in_shape[MCLAHE_MAX_RANK];
  int64_t out_shape[MCLAHE_MAX_RANK];  // pad / crop: output shape; kernelize: grid shape
  int64_t a[MCLAHE_MAX_RANK];          // pad: before; kernelize: kernel; crop: offset
  int64_t in_stride[MCLAHE_MAX_RANK];
  int64_t block_len;                   // kernelize
};

// mirror_index (nd_image.cpp:27-34): edge-including reflection, any period
__device__ __forceinline__ int64_t reflect(int64_t i, int64_t n) {
  const int64_t period = 2 * n;
  int64_t m = i % period;
  if (m < 0) m += period;
  return m >= n ? period - 1 - m : m;
}

__global__ void __launch_bounds__(256) k_nd_gather(GatherGeom G, const double* __restrict__ in,
                                                  double* __restrict__ out, int64_t n_out) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_out;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t src = 0;
    if (G.op == 1) {  // kernelize: block-major, pixels row-major inside a block
      int64_t k = f / G.block_len, r = f % G.block_len;
      for (int j = G.rank - 1; j >= 0; --j) {
        const int64_t w = r % G.a[j];
        r /= G.a[j];
        const int64_t g = k % G.out_shape[j];
        k /= G.out_shape[j];
        src += (g * G.a[j] + w) * G.in_stride[j];
      }
    } else {
      int64_t r = f;
      for (int j = G.rank - 1; j >= 0; --j) {
        const int64_t c = r % G.out_shape[j];
        r /= G.out_shape[j];
        const int64_t s = G.op == 0 ? reflect(c - G.a[j], G.in_shape[j]) : c + G.a[j];
        src += s * G.in_stride[j];
      }
    }
    out[f] = in[src];
  }
}

int grid_for(int64_t n, int cap) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, cap));
}

// Device buffers of one host-facing call, released on every exit path.
struct DevBufs {
  void* p[8] = {};
  ~DevBufs() {
    for (void* q : p)
      if (q) cudaFree(q);
  }
};

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" {

int mclahe_block_mappings(const double* host_blocks, int64_t n_blocks, int64_t block_len,
                          int64_t n_bins, double clip_limit, int32_t adaptive, double global_lo,
                          double global_hi, double* lo, double* hi, double* counts,
                          double* clipped, double* lut, uint8_t* degenerate) {
  if (!host_blocks || n_blocks < 1 || block_len < 1)
    return host_fail(MCLAHE_ERR_VALIDATION, "blocks must be non-empty");
  if (n_bins < 2) return host_fail(MCLAHE_ERR_VALIDATION, "n_bins must be at least 2");
  if (n_bins > 16384)
    return host_fail(MCLAHE_ERR_UNSUPPORTED, "n_bins above 16384 is not supported on the GPU path");
  if (block_len >= (int64_t{1} << 32))
    return host_fail(MCLAHE_ERR_UNSUPPORTED, "block too large for 32-bit counts");
  const bool full = lut != nullptr;
  if (full && !degenerate)
    return host_fail(MCLAHE_ERR_VALIDATION, "lut and degenerate must be given together");
  if (full && (!(clip_limit > 0.0) || !(clip_limit <= 1.0)))
    return host_fail(MCLAHE_ERR_VALIDATION, "clip_limit must be in (0, 1]");
  const int64_t n = n_bins, nb = n_blocks;
  DevBufs B;
  const size_t in_bytes = (size_t)(nb * block_len) * sizeof(double);
  MGH_CUDA(cudaMalloc(&B.p[0], in_bytes));
  MGH_CUDA(cudaMemcpy(B.p[0], host_blocks, in_bytes, cudaMemcpyHostToDevice));
  double* d_lo = nullptr;
  double* d_hi = nullptr;
  double* d_cnt = nullptr;
  double* d_clip = nullptr;
  double* d_lut = nullptr;
  uint8_t* d_deg = nullptr;
  MGH_CUDA(cudaMalloc(&B.p[1], (size_t)nb * 2 * sizeof(double)));
  d_lo = static_cast<double*>(B.p[1]);
  d_hi = d_lo + nb;
  if (counts) {
    MGH_CUDA(cudaMalloc(&B.p[2], (size_t)(nb * n) * sizeof(double)));
    d_cnt = static_cast<double*>(B.p[2]);
  }
  if (full) {
    MGH_CUDA(cudaMalloc(&B.p[3], (size_t)(nb * n) * sizeof(double)));
    d_lut = static_cast<double*>(B.p[3]);
    MGH_CUDA(cudaMalloc(&B.p[4], (size_t)nb));
    d_deg = static_cast<uint8_t*>(B.p[4]);
    if (clipped) {
      MGH_CUDA(cudaMalloc(&B.p[5], (size_t)(nb * n) * sizeof(double)));
      d_clip = static_cast<double*>(B.p[5]);
    }
  }
  const size_t smem = (size_t)((n * 4 + 15) & ~int64_t(15)) + (size_t)n * 8;
  MGH_CUDA(cudaFuncSetAttribute(k_block_mappings, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int dev = 0, sms = 148;
  MGH_CUDA(cudaGetDevice(&dev));
  MGH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = (int)std::min<int64_t>(nb, (int64_t)sms * 8);
  k_block_mappings<<<grid, kOpsThreads, smem>>>(static_cast<const double*>(B.p[0]), nb, block_len,
                                                (int)n, clip_limit, adaptive ? 1 : 0, global_lo,
                                                global_hi, full ? 2 : 1, d_lo, d_hi, d_cnt, d_clip,
                                                d_lut, d_deg);
  MGH_LAUNCHED();
  if (lo) MGH_CUDA(cudaMemcpy(lo, d_lo, (size_t)nb * sizeof(double), cudaMemcpyDeviceToHost));
  if (hi) MGH_CUDA(cudaMemcpy(hi, d_hi, (size_t)nb * sizeof(double), cudaMemcpyDeviceToHost));
  if (counts)
    MGH_CUDA(cudaMemcpy(counts, d_cnt, (size_t)(nb * n) * sizeof(double), cudaMemcpyDeviceToHost));
  if (full) {
    MGH_CUDA(cudaMemcpy(lut, d_lut, (size_t)(nb * n) * sizeof(double), cudaMemcpyDeviceToHost));
    MGH_CUDA(cudaMemcpy(degenerate, d_deg, (size_t)nb, cudaMemcpyDeviceToHost));
    if (clipped)
      MGH_CUDA(cudaMemcpy(clipped, d_clip, (size_t)(nb * n) * sizeof(double),
                          cudaMemcpyDeviceToHost));
  }
  return MCLAHE_OK;
}

int mclahe_nd_gather(int32_t op, int32_t rank, const int64_t* in_shape, const int64_t* a,
                     const int64_t* b, const double* host_in, double* host_out) {
  if (op < 0 || op > 2) return host_fail(MCLAHE_ERR_VALIDATION, "gather op must be 0, 1 or 2");
  if (rank < 1 || rank > MCLAHE_MAX_RANK)
    return host_fail(MCLAHE_ERR_VALIDATION, "rank must be in [1, 8]");
  if (!in_shape || !a || (op != 1 && !b) || !host_in || !host_out)
    return host_fail(MCLAHE_ERR_VALIDATION, "null argument");
  GatherGeom G{};
  G.rank = rank;
  G.op = op;
  int64_t n_in = 1, n_out = 1;
  for (int j = 0; j < rank; ++j) {
    if (in_shape[j] < 1) return host_fail(MCLAHE_ERR_VALIDATION, "shape extents must be positive");
    G.in_shape[j] = in_shape[j];
    G.a[j] = a[j];
    n_in *= in_shape[j];
    if (op == 0) {  // symmetric_pad: before a, after b (one fold)
      if (a[j] < 0 || b[j] < 0 || a[j] > in_shape[j] || b[j] > in_shape[j])
        return host_fail(MCLAHE_ERR_VALIDATION,
                         "pad length exceeds extent along dimension " + std::to_string(j));
      G.out_shape[j] = in_shape[j] + a[j] + b[j];
    } else if (op == 1) {  // kernelize: kernel a, extent divisible
      if (a[j] < 1 || in_shape[j] % a[j] != 0)
        return host_fail(MCLAHE_ERR_VALIDATION,
                         "padded extent not divisible by kernel size along dimension " +
                             std::to_string(j));
      G.out_shape[j] = in_shape[j] / a[j];
    } else {  // crop: offset a, extents b
      if (a[j] < 0 || b[j] < 1 || a[j] + b[j] > in_shape[j])
        return host_fail(MCLAHE_ERR_VALIDATION,
                         "crop region out of bounds along dimension " + std::to_string(j));
      G.out_shape[j] = b[j];
    }
  }
  G.in_stride[rank - 1] = 1;
  for (int j = rank - 1; j > 0; --j) G.in_stride[j - 1] = G.in_stride[j] * in_shape[j];
  if (op == 1) {
    G.block_len = 1;
    for (int j = 0; j < rank; ++j) G.block_len *= a[j];
    n_out = n_in;
  } else {
    for (int j = 0; j < rank; ++j) n_out *= G.out_shape[j];
  }
  DevBufs B;
  MGH_CUDA(cudaMalloc(&B.p[0], (size_t)n_in * sizeof(double)));
  MGH_CUDA(cudaMalloc(&B.p[1], (size_t)n_out * sizeof(double)));
  MGH_CUDA(cudaMemcpy(B.p[0], host_in, (size_t)n_in * sizeof(double), cudaMemcpyHostToDevice));
  int dev = 0, sms = 148;
  MGH_CUDA(cudaGetDevice(&dev));
  MGH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  k_nd_gather<<<grid_for(n_out, sms * 16), 256>>>(G, static_cast<const double*>(B.p[0]),
                                                  static_cast<double*>(B.p[1]), n_out);
  MGH_LAUNCHED();
  MGH_CUDA(cudaMemcpy(host_out, B.p[1], (size_t)n_out * sizeof(double), cudaMemcpyDeviceToHost));
  return MCLAHE_OK;
}

}  // extern "C"
