// filters.cu -- the steps either side of the MCLAHE path
// on the device, in float64 like the reference:
//   gaussian_filter  separable, sampled Gaussian, mirror boundary (src/filters.cpp:12-96)
//   median_filter    window median, mirror boundary                (src/filters.cpp:98-142)
//   metrics          mse / psnr / rms contrast / Shannon entropy   (src/metrics.cpp:11-72)
// Gaussian taps are computed on the host with the same libm as the reference
// and each output is the same sequential sum with separately rounded
// products and adds (the reference's SSE2 build has no FMA), so the filter
// is bit-identical.  The median is a selection (exact).  Entropy counts use
// the reference bin rule in f64 (exact) and the entropy sum runs on the host
// in bin order; mse and the variance are parallel sums (within 1e-12).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/mclahe_gpu.h"
#include "binning.cuh"
#include "host_err.h"

namespace mg {
namespace {

constexpr int kMedianMax = 343;  // window values per output on the GPU path (7 x 7 x 7)

__device__ __forceinline__ int64_t mirror_d(int64_t i, int64_t n) {  // nd_image.cpp:27-34
  if ((uint64_t)i < (uint64_t)n) return i;
  // one reflection covers |overhang| <= n; the periodic form only when the
  // window is wider than the line
  int64_t m = i < 0 ? -i - 1 : i;
  m = m >= n ? 2 * n - 1 - m : m;
  if (m >= 0 && m < n) return m;
  const int64_t period = 2 * n;
  m = i % period;
  if (m < 0) m += period;
  return m >= n ? period - 1 - m : m;
}

// convolve_axis (filters.cpp:28-80): out = sum_k tap_k * line[mirror(x + k)],
// k ascending, products and sums rounded separately.
// Same arithmetic, laid out for reuse: a work item is a run of kRun
// consecutive positions along the axis for one (outer, inner) pair, so the
// (run + 2r) values it reads stay in L1.  Items are numbered inner-fastest,
// so a warp reads consecutive inner indices (S > 1) or, on the contiguous
// axis (S == 1), neighbouring runs of the same rows.  I is the index type
// (32-bit when the volume allows).
constexpr int kRun = 16;

template <typename I>
__global__ void k_gauss_axis_runs(const double* __restrict__ in, double* __restrict__ out,
                                  I items, I runs, I extent, I stride,
                                  const double* __restrict__ taps, int radius) {
  for (I it = blockIdx.x * (I)blockDim.x + threadIdx.x; it < items; it += (I)gridDim.x * blockDim.x) {
    const I inner = it % stride, rest = it / stride;
    const I run = rest % runs, o = rest / runs;
    const I x0 = run * kRun;
    const I x1 = x0 + kRun < extent ? x0 + kRun : extent;
    const double* line = in + (int64_t)o * extent * stride + inner;
    double* dst = out + (int64_t)o * extent * stride + inner;
    for (I x = x0; x < x1; ++x) {
      double acc = 0.0;
      for (int k = -radius; k <= radius; ++k)
        acc = __dadd_rn(acc, __dmul_rn(__ldg(taps + k + radius),
                                       __ldg(line + mirror_d((int64_t)x + k, extent) * (int64_t)stride)));
      dst[(int64_t)x * stride] = acc;
    }
  }
}

// The contiguous axis (S == 1): one output per thread, consecutive threads on
// consecutive positions (coalesced; the 2r + 1 reads per output hit L1).
template <typename I>
__global__ void k_gauss_last(const double* __restrict__ in, double* __restrict__ out, I n,
                             I extent, const double* __restrict__ taps, int radius) {
  for (I idx = blockIdx.x * (I)blockDim.x + threadIdx.x; idx < n; idx += (I)gridDim.x * blockDim.x) {
    const I x = idx % extent;
    const double* line = in + (idx - x);
    double acc = 0.0;
    for (int k = -radius; k <= radius; ++k)
      acc = __dadd_rn(acc, __dmul_rn(__ldg(taps + k + radius),
                                     __ldg(line + mirror_d((int64_t)x + k, extent))));
    out[idx] = acc;
  }
}

struct MedGeom {
  int rank;
  int64_t shape[MCLAHE_MAX_RANK];
  int64_t stride[MCLAHE_MAX_RANK];
  int64_t win[MCLAHE_MAX_RANK];
  int64_t lo[MCLAHE_MAX_RANK];  // first offset: -floor((w-1)/2)
  int wl;
};

// median_filter (filters.cpp:98-142): gather the mirrored window, order it,
// the middle value (odd) or the mean of the two middle values (even).
__global__ void k_median(const double* __restrict__ in, double* __restrict__ out, int64_t total,
                         const MedGeom g) {
  double w[kMedianMax];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[MCLAHE_MAX_RANK];
    int64_t rem = idx;
    for (int j = g.rank - 1; j >= 0; --j) {
      c[j] = rem % g.shape[j];
      rem /= g.shape[j];
    }
    for (int n = 0; n < g.wl; ++n) {
      int64_t r = n, flat = 0;
      for (int j = g.rank - 1; j >= 0; --j) {
        const int64_t o = r % g.win[j];
        r /= g.win[j];
        flat += mirror_d(c[j] + g.lo[j] + o, g.shape[j]) * g.stride[j];
      }
      // insertion into the sorted prefix
      const double v = __ldg(in + flat);
      int p = n;
      while (p > 0 && w[p - 1] > v) {
        w[p] = w[p - 1];
        --p;
      }
      w[p] = v;
    }
    const int mid = g.wl / 2;
    out[idx] = (g.wl & 1) ? w[mid] : 0.5 * (w[mid - 1] + w[mid]);
  }
}

__global__ void k_nonfinite(const double* __restrict__ a, int64_t n, int* flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(a[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Per-block partial sums (fixed order inside a block, partials summed on the
// host in block order): deterministic.  mode 0: sum (a - b)^2, 1: sum a,
// 2: sum (a - m)^2.
__global__ void k_partial_sum(const double* __restrict__ a, const double* __restrict__ b,
                              int64_t n, double m, int mode, double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d;
    if (mode == 0) {
      d = __dsub_rn(a[i], b[i]);
      d = __dmul_rn(d, d);
    } else if (mode == 1) {
      d = a[i];
    } else {
      d = __dsub_rn(a[i], m);
      d = __dmul_rn(d, d);
    }
    acc = __dadd_rn(acc, d);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_minmax(const double* __restrict__ a, int64_t n, int64_t* keys) {
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    lo = fmin(lo, a[i]);
    hi = fmax(hi, a[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<long long*>(&keys[0]), (long long)~okey(lo));
    atomicMax(reinterpret_cast<long long*>(&keys[1]), (long long)okey(hi));
  }
}

// shannon_entropy counts (metrics.cpp:44-58): bin_index over [min, max].
__global__ void k_entropy_counts(const double* __restrict__ a, int64_t n, const int64_t* keys,
                                 int nb, unsigned long long* counts) {
  extern __shared__ unsigned int hist[];
  for (int k = threadIdx.x; k < nb; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  const double lo = okey_decode(~keys[0]), hi = okey_decode(keys[1]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[bin_exact(a[i], lo, hi, nb)], 1u);
  __syncthreads();
  for (int k = threadIdx.x; k < nb; k += blockDim.x)
    if (hist[k]) atomicAdd(&counts[k], (unsigned long long)hist[k]);
}

int64_t product(int rank, const int64_t* shape) {
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) n *= shape[i];
  return n;
}

int check_shape(int rank, const int64_t* shape) {
  if (rank < 1 || rank > MCLAHE_MAX_RANK)
    return host_fail(MCLAHE_ERR_VALIDATION, "rank must be in [1, " +
                                                std::to_string(MCLAHE_MAX_RANK) + "]");
  for (int i = 0; i < rank; ++i)
    if (shape[i] <= 0) return host_fail(MCLAHE_ERR_VALIDATION, "shape extents must be positive");
  return MCLAHE_OK;
}

int grid_for(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

// Device buffers for a host call; freed on scope exit.
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// The device's default memory pool keeps freed blocks (no release at every
// synchronisation), so repeated filter calls do not re-map their scratch.
void keep_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = true;
}

int nonfinite(const double* d, int64_t n, cudaStream_t st, int* flag_dev, bool* bad) {
  MGH_CUDA(cudaMemsetAsync(flag_dev, 0, sizeof(int), st));
  k_nonfinite<<<grid_for(n), 256, 0, st>>>(d, n, flag_dev);
  MGH_LAUNCHED();
  int h = 0;
  MGH_CUDA(cudaMemcpyAsync(&h, flag_dev, sizeof h, cudaMemcpyDeviceToHost, st));
  MGH_CUDA(cudaStreamSynchronize(st));
  *bad = h != 0;
  return MCLAHE_OK;
}

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" {

int mclahe_gaussian_filter_device(int32_t rank, const int64_t* shape, const double* sigmas,
                                  double truncate, const double* in, double* out, void* stream) {
  int rc = check_shape(rank, shape);
  if (rc) return rc;
  if (!(truncate > 0.0)) return host_fail(MCLAHE_ERR_VALIDATION, "truncate must be positive");
  for (int i = 0; i < rank; ++i)
    if (!(sigmas[i] >= 0.0)) return host_fail(MCLAHE_ERR_VALIDATION, "sigma must be non-negative");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = product(rank, shape);
  // scratch: flag | taps | ping-pong volume
  std::vector<std::vector<double>> taps(rank);
  size_t ntaps = 0;
  for (int ax = 0; ax < rank; ++ax) {
    if (sigmas[ax] == 0.0) continue;
    // gaussian_taps (filters.cpp:12-23), host libm like the reference
    const long long radius = static_cast<long long>(std::ceil(truncate * sigmas[ax]));
    std::vector<double>& t = taps[ax];
    t.resize(2 * radius + 1);
    double total = 0.0;
    for (long long k = -radius; k <= radius; ++k) {
      const double x = static_cast<double>(k) / sigmas[ax];
      t[k + radius] = std::exp(-0.5 * x * x);
      total += t[k + radius];
    }
    for (double& w : t) w /= total;
    ntaps += t.size();
  }
  keep_pool();
  DevBuf scratch;
  MGH_CUDA(cudaMallocAsync(&scratch.p, 256 + ntaps * 8 + (size_t)n * 8, st));
  int* flag = static_cast<int*>(scratch.p);
  double* dtaps = reinterpret_cast<double*>(static_cast<char*>(scratch.p) + 256);
  double* tmp = dtaps + ntaps;
  // the finiteness scan runs ahead of the passes; its verdict is read once
  // at the end (the filtered values are discarded on failure)
  MGH_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  k_nonfinite<<<grid_for(n), 256, 0, st>>>(in, n, flag);
  MGH_LAUNCHED();
  // passes ping-pong so the last one lands in `out`
  int passes = 0;
  for (int ax = 0; ax < rank; ++ax) passes += !taps[ax].empty();
  const double* src = in;
  double* bufs[2] = {(passes % 2) ? out : tmp, (passes % 2) ? tmp : out};
  int p = 0;
  size_t off = 0;
  for (int ax = 0; ax < rank; ++ax) {
    if (taps[ax].empty()) continue;
    MGH_CUDA(cudaMemcpyAsync(dtaps + off, taps[ax].data(), taps[ax].size() * 8,
                             cudaMemcpyHostToDevice, st));
    int64_t stride = 1;
    for (int j = ax + 1; j < rank; ++j) stride *= shape[j];
    double* dst = bufs[p & 1];
    const int64_t outer = n / (shape[ax] * stride);
    const int64_t runs = (shape[ax] + kRun - 1) / kRun;
    const int64_t items = outer * runs * stride;
    const int r = (int)((taps[ax].size() - 1) / 2);
    if (stride == 1 && n < (int64_t{1} << 31))
      k_gauss_last<uint32_t><<<grid_for(n), 256, 0, st>>>(src, dst, (uint32_t)n,
                                                           (uint32_t)shape[ax], dtaps + off, r);
    else if (stride == 1)
      k_gauss_last<uint64_t><<<grid_for(n), 256, 0, st>>>(src, dst, (uint64_t)n,
                                                           (uint64_t)shape[ax], dtaps + off, r);
    else if (n < (int64_t{1} << 31))
      k_gauss_axis_runs<uint32_t><<<grid_for(items), 256, 0, st>>>(
          src, dst, (uint32_t)items, (uint32_t)runs, (uint32_t)shape[ax], (uint32_t)stride,
          dtaps + off, r);
    else
      k_gauss_axis_runs<uint64_t><<<grid_for(items), 256, 0, st>>>(
          src, dst, (uint64_t)items, (uint64_t)runs, (uint64_t)shape[ax], (uint64_t)stride,
          dtaps + off, r);
    MGH_LAUNCHED();
    src = dst;
    off += taps[ax].size();
    ++p;
  }
  if (passes == 0) MGH_CUDA(cudaMemcpyAsync(out, in, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
  int bad = 0;
  MGH_CUDA(cudaMemcpyAsync(&bad, flag, sizeof bad, cudaMemcpyDeviceToHost, st));
  MGH_CUDA(cudaFreeAsync(scratch.p, st));
  scratch.p = nullptr;
  MGH_CUDA(cudaStreamSynchronize(st));
  if (bad) return host_fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
  return MCLAHE_OK;
}

int mclahe_median_filter_device(int32_t rank, const int64_t* shape, const int64_t* window,
                                const double* in, double* out, void* stream) {
  int rc = check_shape(rank, shape);
  if (rc) return rc;
  MedGeom g{};
  g.rank = rank;
  int64_t wl = 1;
  for (int i = 0; i < rank; ++i) {
    if (window[i] <= 0) return host_fail(MCLAHE_ERR_VALIDATION, "window extents must be positive");
    g.shape[i] = shape[i];
    g.win[i] = window[i];
    g.lo[i] = -((window[i] - 1) / 2);
    wl *= window[i];
    if (wl > kMedianMax)
      return host_fail(MCLAHE_ERR_UNSUPPORTED, "median window holds more than " +
                                                   std::to_string(kMedianMax) +
                                                   " values (GPU path limit)");
  }
  g.wl = (int)wl;
  g.stride[rank - 1] = 1;
  for (int j = rank - 1; j > 0; --j) g.stride[j - 1] = g.stride[j] * shape[j];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = product(rank, shape);
  DevBuf flag;
  MGH_CUDA(cudaMallocAsync(&flag.p, 256, st));
  bool bad = false;
  if ((rc = nonfinite(in, n, st, static_cast<int*>(flag.p), &bad))) return rc;
  if (bad) return host_fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
  k_median<<<grid_for(n), 128, 0, st>>>(in, out, n, g);
  MGH_LAUNCHED();
  MGH_CUDA(cudaStreamSynchronize(st));
  return MCLAHE_OK;
}

int mclahe_metrics_device(int32_t rank, const int64_t* shape, const double* a, const double* b,
                          int64_t n_bins, double peak, mclahe_metrics_t* report, void* stream) {
  int rc = check_shape(rank, shape);
  if (rc) return rc;
  if (!report) return host_fail(MCLAHE_ERR_VALIDATION, "report must be non-NULL");
  // the reference's order of checks: psnr (after mse), then the entropy
  if (!(peak > 0.0)) return host_fail(MCLAHE_ERR_VALIDATION, "psnr peak must be positive");
  if (n_bins < 2) return host_fail(MCLAHE_ERR_VALIDATION, "entropy needs at least 2 bins");
  if (n_bins > 16384) return host_fail(MCLAHE_ERR_UNSUPPORTED, "n_bins above 16384 on the GPU path");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = product(rank, shape);
  const int grid = grid_for(n);
  DevBuf scratch;  // partials[grid] | keys[2] | counts[n_bins]
  MGH_CUDA(cudaMallocAsync(&scratch.p, (size_t)grid * 8 + 16 + (size_t)n_bins * 8, st));
  double* part = static_cast<double*>(scratch.p);
  int64_t* keys = reinterpret_cast<int64_t*>(part + grid);
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(keys + 2);
  std::vector<double> hp(grid);
  auto reduce = [&](int mode, double m, double* result) -> int {
    k_partial_sum<<<grid, 256, 0, st>>>(a, b, n, m, mode, part);
    MGH_LAUNCHED();
    MGH_CUDA(cudaMemcpyAsync(hp.data(), part, (size_t)grid * 8, cudaMemcpyDeviceToHost, st));
    MGH_CUDA(cudaStreamSynchronize(st));
    double acc = 0.0;
    for (double v : hp) acc += v;
    *result = acc;
    return MCLAHE_OK;
  };
  double s = 0.0;
  report->mse = 0.0;
  report->psnr_db = 0.0;
  if (b) {  // mse (metrics.cpp:11-21), psnr (:23-28)
    if ((rc = reduce(0, 0.0, &s))) return rc;
    report->mse = s / static_cast<double>(n);
    report->psnr_db = report->mse == 0.0 ? std::numeric_limits<double>::infinity()
                                         : 10.0 * std::log10(peak * peak / report->mse);
  }
  if ((rc = reduce(1, 0.0, &s))) return rc;  // rms_contrast (metrics.cpp:30-41)
  const double mean = s / static_cast<double>(n);
  if ((rc = reduce(2, mean, &s))) return rc;
  report->std = std::sqrt(s / static_cast<double>(n));
  // shannon_entropy (metrics.cpp:43-60)
  const int64_t init[2] = {INT64_MIN, INT64_MIN};
  MGH_CUDA(cudaMemcpyAsync(keys, init, sizeof init, cudaMemcpyHostToDevice, st));
  k_minmax<<<grid, 256, 0, st>>>(a, n, keys);
  MGH_LAUNCHED();
  int64_t hk[2];
  MGH_CUDA(cudaMemcpyAsync(hk, keys, sizeof hk, cudaMemcpyDeviceToHost, st));
  MGH_CUDA(cudaStreamSynchronize(st));
  const double lo = okey_decode(~hk[0]), hi = okey_decode(hk[1]);
  report->entropy_bits = 0.0;
  report->n_bins_used = n_bins;
  if (hi > lo) {
    MGH_CUDA(cudaMemsetAsync(counts, 0, (size_t)n_bins * 8, st));
    k_entropy_counts<<<grid, 256, (size_t)n_bins * 4, st>>>(a, n, keys, (int)n_bins, counts);
    MGH_LAUNCHED();
    std::vector<unsigned long long> hc(n_bins);
    MGH_CUDA(cudaMemcpyAsync(hc.data(), counts, (size_t)n_bins * 8, cudaMemcpyDeviceToHost, st));
    MGH_CUDA(cudaStreamSynchronize(st));
    const double total = static_cast<double>(n);
    double e = 0.0;
    for (unsigned long long c : hc) {  // bin order, host libm: as the reference
      if (c == 0) continue;
      const double p = static_cast<double>(c) / total;
      e -= p * std::log2(p);
    }
    report->entropy_bits = e;
  }
  MGH_CUDA(cudaFreeAsync(scratch.p, st));
  scratch.p = nullptr;
  MGH_CUDA(cudaStreamSynchronize(st));
  return MCLAHE_OK;
}

// Host-buffer forms (float64), like mclahe_gpu_run.
namespace {
int to_device(const double* h, int64_t n, double** d, cudaStream_t st) {
  MGH_CUDA(cudaMallocAsync(reinterpret_cast<void**>(d), (size_t)n * 8, st));
  MGH_CUDA(cudaMemcpyAsync(*d, h, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  return MCLAHE_OK;
}
}  // namespace

int mclahe_gaussian_filter(int32_t rank, const int64_t* shape, const double* sigmas,
                           double truncate, const double* host_in, double* host_out) {
  int rc = check_shape(rank, shape);
  if (rc) return rc;
  const int64_t n = product(rank, shape);
  double *din = nullptr, *dout = nullptr;
  if ((rc = to_device(host_in, n, &din, 0))) return rc;
  MGH_CUDA(cudaMalloc(&dout, (size_t)n * 8));
  rc = mclahe_gaussian_filter_device(rank, shape, sigmas, truncate, din, dout, nullptr);
  if (!rc) rc = cudaMemcpy(host_out, dout, (size_t)n * 8, cudaMemcpyDeviceToHost) == cudaSuccess
                    ? MCLAHE_OK : host_cuda_fail(cudaGetLastError(), "cudaMemcpy");
  cudaFree(din);
  cudaFree(dout);
  return rc;
}

int mclahe_median_filter(int32_t rank, const int64_t* shape, const int64_t* window,
                         const double* host_in, double* host_out) {
  int rc = check_shape(rank, shape);
  if (rc) return rc;
  const int64_t n = product(rank, shape);
  double *din = nullptr, *dout = nullptr;
  if ((rc = to_device(host_in, n, &din, 0))) return rc;
  MGH_CUDA(cudaMalloc(&dout, (size_t)n * 8));
  rc = mclahe_median_filter_device(rank, shape, window, din, dout, nullptr);
  if (!rc) rc = cudaMemcpy(host_out, dout, (size_t)n * 8, cudaMemcpyDeviceToHost) == cudaSuccess
                    ? MCLAHE_OK : host_cuda_fail(cudaGetLastError(), "cudaMemcpy");
  cudaFree(din);
  cudaFree(dout);
  return rc;
}

int mclahe_metrics(int32_t rank, const int64_t* shape, const double* host_a, const double* host_b,
                   int64_t n_bins, double peak, mclahe_metrics_t* report) {
  int rc = check_shape(rank, shape);
  if (rc) return rc;
  const int64_t n = product(rank, shape);
  double *da = nullptr, *db = nullptr;
  if ((rc = to_device(host_a, n, &da, 0))) return rc;
  if (host_b && (rc = to_device(host_b, n, &db, 0))) {
    cudaFree(da);
    return rc;
  }
  rc = mclahe_metrics_device(rank, shape, da, db, n_bins, peak, report, nullptr);
  cudaFree(da);
  if (db) cudaFree(db);
  return rc;
}

}  // extern "C"
