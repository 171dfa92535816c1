// dropin.cpp -- the C++ drop-in (include/mclahe/pipeline.hpp, filters.hpp,
// metrics.hpp) over the C ABI.
// Host-side only: validation messages, dtype selection, frame loop; all
// compute goes through mclahe_gpu_run (include/mclahe_gpu.h).
#include "mclahe/filters.hpp"
#include "mclahe/metrics.hpp"
#include "mclahe/pipeline.hpp"

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/mclahe_gpu.h"

namespace mclahe {

namespace {

void raise(int rc) {
  const std::string msg = mclahe_last_error();
  if (rc == MCLAHE_ERR_VALIDATION) throw ValidationError(msg);
  throw std::runtime_error("mclahe GPU error " + std::to_string(rc) + ": " + msg);
}

// ---- host staging -------------------------------------------------------
// The reference API hands over float64 vectors.  The GPU path wants the
// values in page-locked memory (full-rate, asynchronous PCIe copies that the
// streamed call overlaps with the kernels), as float32 when every value is
// float32-representable (then the bins are bit-identical: f32 -> f64 is
// exact).  One pinned in / out pair per process, grown on demand, guarded by
// a mutex (the GPU call itself is serialised by the library anyway); the
// narrowing (with the exactness check) and widening loops run on all host
// threads.
struct Staging {
  std::mutex mu;
  void* in = nullptr;
  void* out = nullptr;
  size_t cap = 0;
};

Staging& staging() {
  static Staging* s = new Staging();  // process lifetime
  return *s;
}

void ensure_staging(Staging& S, size_t bytes) {
  if (S.cap >= bytes) return;
  mclahe_host_free(S.in);
  mclahe_host_free(S.out);
  S.in = mclahe_host_alloc(bytes);
  S.out = mclahe_host_alloc(bytes);
  S.cap = (S.in && S.out) ? bytes : 0;
  if (!S.cap) raise(MCLAHE_ERR_OOM);
}

// fn(begin, end) over [0, n) on up to hardware_concurrency threads (chunks of
// whole 64 KiB pages of doubles)
template <typename Fn>
void host_parallel(std::size_t n, Fn&& fn) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const std::size_t grain = std::size_t{1} << 16;
  const std::size_t workers = std::min<std::size_t>(hw, (n + grain - 1) / grain);
  if (workers <= 1) {
    fn(std::size_t{0}, n);
    return;
  }
  const std::size_t chunk = ((n + workers - 1) / workers + grain - 1) / grain * grain;
  std::vector<std::thread> pool;
  for (std::size_t w = 1; w < workers && w * chunk < n; ++w)
    pool.emplace_back([&, w] { fn(w * chunk, std::min(n, (w + 1) * chunk)); });
  fn(0, std::min(n, chunk));
  for (auto& t : pool) t.join();
}

// Runs one request on the GPU from float64 host values: narrows into the
// pinned float32 stage when exact (else copies the doubles), calls `gpu`
// (mclahe_gpu_run or the framewise form) on the pinned buffers, and widens
// the result into a fresh vector, whose allocation (page faults of a zeroed
// multi-GB vector) overlaps the GPU call.
using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}
bool trace() {
  static const bool on = std::getenv("MCLAHE_DROPIN_TRACE") != nullptr;
  return on;
}

template <typename Gpu>
std::vector<double> run_staged(mclahe_params_t& p, std::span<const double> src, Gpu&& gpu) {
  const auto t0 = Clock::now();
  const std::size_t n = src.size();
  // The result vector, allocated while the input is staged and the GPU runs:
  // zeroing a fresh multi-GB vector is page-fault bound, so its (untouched)
  // buffer first gets transparent huge pages and is faulted in by all host
  // threads (one byte per page of the raw storage); the vector's own zero
  // fill then runs on mapped memory.
  std::vector<double> out;
  std::thread alloc([&] {
    out.reserve(n);
    char* raw = reinterpret_cast<char*>(out.data());
    const std::size_t bytes = n * sizeof(double);
    const uintptr_t huge = uintptr_t{2} << 20;
    const uintptr_t a = (reinterpret_cast<uintptr_t>(raw) + huge - 1) & ~(huge - 1);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(raw) + bytes) & ~(huge - 1);
    if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    host_parallel(bytes / 4096, [&](std::size_t b, std::size_t en) {
      for (std::size_t pg = b; pg < en; ++pg) reinterpret_cast<volatile char*>(raw)[pg * 4096] = 0;
    });
    out.resize(n);
  });
  Staging& S = staging();
  std::lock_guard<std::mutex> lock(S.mu);
  try {
    ensure_staging(S, n * sizeof(double));
  } catch (...) {
    alloc.join();
    throw;
  }
  std::atomic<bool> exact{true};
  float* in32 = static_cast<float*>(S.in);
  host_parallel(n, [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; i += 4096) {
      if (!exact.load(std::memory_order_relaxed)) return;
      const std::size_t ie = std::min(e, i + 4096);
      bool ok = true;
      for (std::size_t k = i; k < ie; ++k) {
        const float f = static_cast<float>(src[k]);
        ok &= static_cast<double>(f) == src[k];
        in32[k] = f;
      }
      if (!ok) exact.store(false, std::memory_order_relaxed);
    }
  });
  const bool f32 = exact.load();
  if (!f32)
    host_parallel(n, [&](std::size_t b, std::size_t e) {
      std::memcpy(static_cast<double*>(S.in) + b, src.data() + b, (e - b) * sizeof(double));
    });
  p.dtype = f32 ? MCLAHE_F32 : MCLAHE_F64;
  const auto t1 = Clock::now();
  const int rc = gpu(S.in, S.out);
  const auto t2 = Clock::now();
  alloc.join();
  const auto t3 = Clock::now();
  if (rc != MCLAHE_OK) raise(rc);
  if (f32) {
    const float* o = static_cast<const float*>(S.out);
    host_parallel(n, [&](std::size_t b, std::size_t e) {
      for (std::size_t k = b; k < e; ++k) out[k] = static_cast<double>(o[k]);
    });
  } else {
    host_parallel(n, [&](std::size_t b, std::size_t e) {
      std::memcpy(out.data() + b, static_cast<const double*>(S.out) + b, (e - b) * sizeof(double));
    });
  }
  if (trace())
    std::fprintf(stderr, "[mclahe drop-in] %zu values (%s): stage-in %.3f s, gpu %.3f s, "
                 "out-alloc wait %.3f s, stage-out %.3f s\n", n, f32 ? "f32" : "f64",
                 secs(t0, t1), secs(t1, t2), secs(t2, t3), secs(t3, Clock::now()));
  return out;
}

}  // namespace

NdImage mclahe(const McLaheRequest& request, PhaseTimings* timings) {
  const NdImage& img = request.image;
  // validate_request (src/pipeline.cpp:19-23): the kernel-rank message
  if (request.kernel.sizes.size() != img.rank())
    throw ValidationError("kernel rank " + std::to_string(request.kernel.sizes.size()) +
                          " does not match image rank " + std::to_string(img.rank()));
  mclahe_params_t p;
  std::memset(&p, 0, sizeof p);
  p.rank = static_cast<int32_t>(img.rank());
  p.adaptive = request.params.range_mode == RangeMode::Adaptive ? 1 : 0;
  for (std::size_t i = 0; i < img.rank(); ++i) {
    p.shape[i] = static_cast<int64_t>(img.shape()[i]);
    p.kernel[i] = static_cast<int64_t>(request.kernel.sizes[i]);
  }
  p.n_bins = static_cast<int64_t>(request.params.n_bins);
  p.clip_limit = request.params.clip_limit;
  if (const int rc = mclahe_validate(&p)) raise(rc);  // before any staging, as the reference
  mclahe_timings_t t{0.0, 0.0, 0.0};
  std::vector<double> out = run_staged(p, img.values(), [&](const void* in, void* o) {
    return mclahe_gpu_run(&p, in, o, &t);
  });
  if (timings) {
    timings->pad_s += t.pad_s;
    timings->histograms_s += t.histograms_s;
    timings->interpolation_s += t.interpolation_s;
  }
  return NdImage(img.shape(), std::move(out));
}

NdImage mclahe_framewise(const NdImage& image, std::size_t frame_axis, const KernelSpec& kernel,
                         const EnhanceParams& params, unsigned threads, bool renormalize_slices,
                         PhaseTimings* timings) {
  // src/pipeline.cpp:131-153, batched: one GPU run over all slices
  // (mclahe_gpu_run_framewise) instead of a host loop of crops and pastes
  (void)threads;
  if (image.rank() < 2) throw ValidationError("framewise mode needs rank >= 2");
  if (frame_axis >= image.rank())
    throw ValidationError("frame axis " + std::to_string(frame_axis) + " out of range for rank " +
                          std::to_string(image.rank()));
  if (kernel.sizes.size() != image.rank() - 1)
    throw ValidationError("framewise kernel rank must be image rank - 1");
  const Shape& sh = image.shape();
  std::size_t outer = 1, inner = 1;
  for (std::size_t i = 0; i < frame_axis; ++i) outer *= sh[i];
  for (std::size_t i = frame_axis + 1; i < sh.size(); ++i) inner *= sh[i];
  const std::size_t frames = sh[frame_axis];
  std::vector<double> src(image.values().begin(), image.values().end());
  if (renormalize_slices) {  // normalize_to_unit per slice, in place
    Shape slice_shape;
    for (std::size_t i = 0; i < sh.size(); ++i)
      if (i != frame_axis) slice_shape.push_back(sh[i]);
    for (std::size_t f = 0; f < frames; ++f) {
      std::vector<double> buf(outer * inner);
      for (std::size_t o = 0; o < outer; ++o)
        std::memcpy(&buf[o * inner], &src[(o * frames + f) * inner], inner * sizeof(double));
      const NdImage norm = normalize_to_unit(NdImage(slice_shape, std::move(buf)));
      for (std::size_t o = 0; o < outer; ++o)
        std::memcpy(&src[(o * frames + f) * inner], &norm.values()[o * inner], inner * sizeof(double));
    }
  }
  mclahe_params_t p;
  std::memset(&p, 0, sizeof p);
  p.rank = static_cast<int32_t>(image.rank());
  p.adaptive = params.range_mode == RangeMode::Adaptive ? 1 : 0;
  for (std::size_t i = 0; i < image.rank(); ++i) p.shape[i] = static_cast<int64_t>(sh[i]);
  for (std::size_t i = 0; i + 1 < image.rank(); ++i)
    p.kernel[i] = static_cast<int64_t>(kernel.sizes[i]);
  p.n_bins = static_cast<int64_t>(params.n_bins);
  p.clip_limit = params.clip_limit;
  {  // the slice request, checked before any staging (messages as per slice)
    mclahe_params_t sl = p;
    sl.rank = p.rank - 1;
    for (int j = 0, k = 0; j < p.rank; ++j)
      if (j != static_cast<int>(frame_axis)) sl.shape[k++] = p.shape[j];
    for (int j = sl.rank; j < MCLAHE_MAX_RANK; ++j) sl.shape[j] = sl.kernel[j] = 0;
    if (const int rc = mclahe_validate(&sl)) raise(rc);
  }
  mclahe_timings_t t{0.0, 0.0, 0.0};
  std::vector<double> out = run_staged(p, src, [&](const void* in, void* o) {
    return mclahe_gpu_run_framewise(&p, static_cast<int32_t>(frame_axis), in, o, &t);
  });
  if (timings) {
    timings->pad_s += t.pad_s;
    timings->histograms_s += t.histograms_s;
    timings->interpolation_s += t.interpolation_s;
  }
  return NdImage(sh, std::move(out));
}

NdImage normalize_to_unit(const NdImage& image) {
  // src/pipeline.cpp:155-165
  if (!image.all_finite()) throw ValidationError("image contains non-finite values");
  double lo, hi;
  image.min_max(lo, hi);
  if (!(hi > lo)) return NdImage::constant(image.shape(), 0.5);
  const double span = hi - lo;
  std::vector<double> d(image.size());
  for (std::size_t i = 0; i < d.size(); ++i) d[i] = (image[i] - lo) / span;
  return NdImage(image.shape(), std::move(d));
}

namespace {

std::vector<int64_t> shape64(const NdImage& a) {
  return std::vector<int64_t>(a.shape().begin(), a.shape().end());
}

MetricsReport metrics_call(const NdImage& a, const NdImage* b, std::size_t n_bins, double peak) {
  if (b && a.shape() != b->shape()) throw ValidationError("mse operands differ in shape");
  const std::vector<int64_t> sh = shape64(a);
  mclahe_metrics_t r{};
  const int rc = mclahe_metrics(static_cast<int32_t>(a.rank()), sh.data(), a.values().data(),
                                b ? b->values().data() : nullptr, static_cast<int64_t>(n_bins),
                                peak, &r);
  if (rc != MCLAHE_OK) raise(rc);
  MetricsReport m;
  m.mse = r.mse;
  m.psnr_db = r.psnr_db;
  m.std = r.std;
  m.entropy_bits = r.entropy_bits;
  m.n_bins_used = static_cast<std::size_t>(r.n_bins_used);
  return m;
}

}  // namespace

NdImage gaussian_filter(const NdImage& image, const GaussianSpec& spec, unsigned threads) {
  (void)threads;
  if (spec.sigmas.size() != image.rank())
    throw ValidationError("sigma count does not match image rank");
  const std::vector<int64_t> sh = shape64(image);
  std::vector<double> out(image.size());
  const int rc = mclahe_gaussian_filter(static_cast<int32_t>(image.rank()), sh.data(),
                                        spec.sigmas.data(), spec.truncate, image.values().data(),
                                        out.data());
  if (rc != MCLAHE_OK) raise(rc);
  return NdImage(image.shape(), std::move(out));
}

NdImage median_filter(const NdImage& image, const MedianSpec& spec, unsigned threads) {
  (void)threads;
  if (spec.window.size() != image.rank())
    throw ValidationError("window rank does not match image rank");
  const std::vector<int64_t> sh = shape64(image);
  const std::vector<int64_t> win(spec.window.begin(), spec.window.end());
  std::vector<double> out(image.size());
  const int rc = mclahe_median_filter(static_cast<int32_t>(image.rank()), sh.data(), win.data(),
                                      image.values().data(), out.data());
  if (rc != MCLAHE_OK) raise(rc);
  return NdImage(image.shape(), std::move(out));
}

double mse(const NdImage& a, const NdImage& b) { return metrics_call(a, &b, 256, 1.0).mse; }

double psnr(const NdImage& a, const NdImage& b, double peak) {
  return metrics_call(a, &b, 256, peak).psnr_db;
}

double rms_contrast(const NdImage& a) { return metrics_call(a, nullptr, 256, 1.0).std; }

double shannon_entropy(const NdImage& a, std::size_t n_bins) {
  return metrics_call(a, nullptr, n_bins, 1.0).entropy_bits;
}

MetricsReport compute_metrics(const NdImage& a, const NdImage& b, std::size_t n_bins,
                              double peak) {
  return metrics_call(a, &b, n_bins, peak);
}

}  // namespace mclahe
