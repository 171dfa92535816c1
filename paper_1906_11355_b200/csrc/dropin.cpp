// dropin.cpp -- the C++ drop-in (include/mclahe/pipeline.hpp, filters.hpp,
// metrics.hpp) over the C ABI.
// Host-side only: validation messages, dtype selection, frame loop; all
// compute goes through mclahe_gpu_run (include/mclahe_gpu.h).
#include "mclahe/filters.hpp"
#include "mclahe/metrics.hpp"
#include "mclahe/pipeline.hpp"

#include <cmath>
#include <cstring>
#include <limits>

#include "../../include/mclahe_gpu.h"

namespace mclahe {

namespace {

void raise(int rc) {
  const std::string msg = mclahe_last_error();
  if (rc == MCLAHE_ERR_VALIDATION) throw ValidationError(msg);
  throw std::runtime_error("mclahe GPU error " + std::to_string(rc) + ": " + msg);
}

bool all_f32_exact(std::span<const double> v) {
  for (double x : v)
    if (static_cast<double>(static_cast<float>(x)) != x) return false;
  return true;
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
  mclahe_timings_t t{0.0, 0.0, 0.0};
  std::vector<double> out(img.size());
  const std::span<const double> src = img.values();
  int rc;
  if (all_f32_exact(src)) {  // float32 pencil kernels, bit-identical bins
    p.dtype = MCLAHE_F32;
    std::vector<float> in32(src.begin(), src.end()), out32(src.size());
    rc = mclahe_gpu_run(&p, in32.data(), out32.data(), &t);
    if (rc == MCLAHE_OK) out.assign(out32.begin(), out32.end());
  } else {
    p.dtype = MCLAHE_F64;
    rc = mclahe_gpu_run(&p, src.data(), out.data(), &t);
  }
  if (rc != MCLAHE_OK) raise(rc);
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
  mclahe_timings_t t{0.0, 0.0, 0.0};
  std::vector<double> out(src.size());
  int rc;
  if (all_f32_exact(src)) {
    p.dtype = MCLAHE_F32;
    std::vector<float> in32(src.begin(), src.end()), out32(src.size());
    rc = mclahe_gpu_run_framewise(&p, static_cast<int32_t>(frame_axis), in32.data(), out32.data(),
                                  &t);
    if (rc == MCLAHE_OK) out.assign(out32.begin(), out32.end());
  } else {
    p.dtype = MCLAHE_F64;
    rc = mclahe_gpu_run_framewise(&p, static_cast<int32_t>(frame_axis), src.data(), out.data(), &t);
  }
  if (rc != MCLAHE_OK) raise(rc);
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
