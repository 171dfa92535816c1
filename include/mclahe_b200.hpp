// include/mclahe_b200.hpp -- C++ drop-in for the reference's public MCLAHE API.
//
// Source-compatible with the reference's mclahe:: pipeline interface
// (/root/reference/proj/core/include/mclahe/pipeline.hpp:12-43 and the types
// it uses from nd_image.hpp / histogram.hpp): the same namespace, type names,
// fields and call
//
//     mclahe::NdImage out = mclahe::mclahe(request, &timings);
//
// so a caller swaps the include and links libmclahe_cpp.so (+ libmclahe_gpu.so)
// instead of libmclahe.a.  Compute runs on the GPU through the C ABI in
// mclahe_gpu.h; float64 images whose values are all float32-representable
// take the float32 pencil kernels (bit-identical bins, since f32 -> f64 is
// exact), others the exact float64 path.  Errors: ValidationError with the
// reference's messages; CUDA failures as std::runtime_error.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mclahe {

inline constexpr std::size_t kMaxRank = 8;

class ValidationError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

using Shape = std::vector<std::size_t>;

// Dense row-major N-D array of doubles (nd_image.hpp:54-77).
class NdImage {
 public:
  NdImage(Shape shape, std::vector<double> data);
  static NdImage zeros(Shape shape);
  static NdImage constant(Shape shape, double value);

  const Shape& shape() const noexcept { return shape_; }
  std::size_t rank() const noexcept { return shape_.size(); }
  std::size_t size() const noexcept { return data_.size(); }
  const std::vector<double>& data() const noexcept { return data_; }
  std::vector<double>& data() noexcept { return data_; }
  double operator[](std::size_t i) const noexcept { return data_[i]; }
  double& operator[](std::size_t i) noexcept { return data_[i]; }

 private:
  Shape shape_;
  std::vector<double> data_;
};

struct KernelSpec {
  std::vector<std::size_t> sizes;
};

enum class RangeMode { Global, Adaptive };

struct EnhanceParams {
  double clip_limit = 1.0;
  std::size_t n_bins = 256;
  RangeMode range_mode = RangeMode::Global;
};

struct McLaheRequest {
  NdImage image;
  KernelSpec kernel;
  EnhanceParams params;
  unsigned threads = 0;  // accepted for compatibility; the GPU path ignores it
};

struct PhaseTimings {
  double pad_s = 0.0;
  double histograms_s = 0.0;
  double interpolation_s = 0.0;
};

// pipeline.hpp:30 -- full MCLAHE on the current CUDA device.
NdImage mclahe(const McLaheRequest& request, PhaseTimings* timings = nullptr);

// pipeline.hpp:37-40 -- mclahe on every slice along frame_axis, batched into
// one GPU run (mclahe_gpu_run_framewise); `threads` is ignored.
NdImage mclahe_framewise(const NdImage& image, std::size_t frame_axis, const KernelSpec& kernel,
                         const EnhanceParams& params, unsigned threads = 0,
                         bool renormalize_slices = false, PhaseTimings* timings = nullptr);

// pipeline.hpp:43 -- affine map of [min, max] onto [0, 1]; constant -> 0.5.
NdImage normalize_to_unit(const NdImage& image);

// ---- filters.hpp / metrics.hpp: the steps either side of the path, on the GPU ----

struct GaussianSpec {  // filters.hpp:11-15
  std::vector<double> sigmas;
  double truncate = 4.0;
};

struct MedianSpec {  // filters.hpp:17-21
  std::vector<std::size_t> window;
};

// filters.hpp:24-25 -- bit-identical to the reference.
NdImage gaussian_filter(const NdImage& image, const GaussianSpec& spec, unsigned threads = 1);

// filters.hpp:30-32 -- windows of at most 343 values on the GPU path.
NdImage median_filter(const NdImage& image, const MedianSpec& spec, unsigned threads = 1);

struct MetricsReport {  // metrics.hpp:9-17
  double mse = 0.0;
  double psnr_db = 0.0;
  double std = 0.0;
  double entropy_bits = 0.0;
  std::size_t n_bins_used = 0;
};

double mse(const NdImage& a, const NdImage& b);                        // metrics.hpp:19-20
double psnr(const NdImage& a, const NdImage& b, double peak = 1.0);     // metrics.hpp:22-23
double rms_contrast(const NdImage& a);                                  // metrics.hpp:25-26
double shannon_entropy(const NdImage& a, std::size_t n_bins = 256);     // metrics.hpp:28-30
MetricsReport compute_metrics(const NdImage& a, const NdImage& b, std::size_t n_bins = 256,
                              double peak = 1.0);                       // metrics.hpp:35-36

// ---- npy.hpp:12-60: array files (host code; NPY v1.0 written, v1.0/v2.0 read) ----

enum class Dtype { f4, f8, u1, u2, i2, i4 };  // all little-endian

std::size_t dtype_item_size(Dtype dtype);
std::string dtype_descr(Dtype dtype);            // NPY descr string, e.g. "<f4"
Dtype dtype_from_name(const std::string& name);  // "f4", "f8", "u1", ...

enum class NpyErrc {
  io_failure,
  bad_magic,
  unsupported_version,
  bad_header,
  unsupported_dtype,
  fortran_order,
  truncated_payload,
  size_mismatch,
  value_out_of_range,
};

class NpyError : public std::runtime_error {
 public:
  NpyError(NpyErrc code, const std::string& message) : std::runtime_error(message), code_(code) {}
  NpyErrc code() const noexcept { return code_; }

 private:
  NpyErrc code_;
};

struct ArrayFileMeta {
  Dtype dtype = Dtype::f8;
  bool fortran_order = false;
  Shape shape;
};

// Fortran-ordered files are rejected (NpyErrc::fortran_order), not transposed.
std::pair<NdImage, ArrayFileMeta> read_npy(const std::string& path);
// Integer dtypes round to nearest and reject out-of-range values.
void write_npy(const std::string& path, const NdImage& image, Dtype dtype);
// Headerless file whose size must equal item_size * product(meta.shape).
NdImage read_raw(const std::string& path, const ArrayFileMeta& meta);

}  // namespace mclahe
