// histogram_api.cpp -- include/mclahe/histogram.hpp for the C++ drop-in.
// build_mappings and compute_histogram bin every block on the GPU
// (mclahe_block_mappings, csrc/ops.cu: one CTA per block, exact f64 bins,
// clip / CDF in the reference's order); the per-histogram scalar steps are
// host code with the reference's arithmetic (src/histogram.cpp:24-70,
// 108-111), compiled without FP contraction.
#include "mclahe/histogram.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/mclahe_gpu.h"

namespace mclahe {

namespace {

[[noreturn]] void raise_gpu(int rc) {
  const std::string msg = mclahe_last_error();
  if (rc == MCLAHE_ERR_VALIDATION) throw ValidationError(msg);
  throw std::runtime_error("mclahe GPU error " + std::to_string(rc) + ": " + msg);
}

void check_params(const EnhanceParams& p) {  // histogram.cpp:11-15
  if (!(p.clip_limit > 0.0) || !(p.clip_limit <= 1.0))
    throw ValidationError("clip_limit must be in (0, 1]");
  if (p.n_bins < 2) throw ValidationError("n_bins must be at least 2");
}

}  // namespace

std::size_t bin_index(double value, const IntensityRange& range, std::size_t n_bins) {
  // histogram.cpp:24-32
  if (range.degenerate()) throw ValidationError("bin_index requires a non-degenerate range");
  const double n = static_cast<double>(n_bins);
  const double s = std::floor((value - range.lo) / (range.hi - range.lo) * n);
  if (!(s > 0.0)) return 0;
  return s >= n ? n_bins - 1 : static_cast<std::size_t>(s);
}

std::vector<double> compute_histogram(std::span<const double> block,
                                      const IntensityRange& range, std::size_t n_bins) {
  // histogram.cpp:34-40, binned on the GPU
  if (block.empty()) throw ValidationError("histogram of an empty block");
  if (range.degenerate()) throw ValidationError("bin_index requires a non-degenerate range");
  std::vector<double> counts(n_bins, 0.0);
  const int rc = mclahe_block_mappings(block.data(), 1, static_cast<int64_t>(block.size()),
                                       static_cast<int64_t>(n_bins), 1.0, 0, range.lo, range.hi,
                                       nullptr, nullptr, counts.data(), nullptr, nullptr, nullptr);
  if (rc != MCLAHE_OK) raise_gpu(rc);
  return counts;
}

std::vector<double> clip_histogram(std::span<const double> counts, double clip_limit) {
  // histogram.cpp:42-55: every sum sequential in bin order
  double total = 0.0;
  for (const double c : counts) total += c;
  const double cap = clip_limit * total;
  double excess = 0.0;
  for (const double c : counts) excess += std::max(c - cap, 0.0);
  const double share = excess / static_cast<double>(counts.size());
  std::vector<double> out;
  out.reserve(counts.size());
  for (const double c : counts) out.push_back((cap < c ? cap : c) + share);
  return out;
}

NormalizedCdf normalized_cdf(std::span<const double> clipped_counts) {  // histogram.cpp:57-70
  NormalizedCdf r;
  r.values.resize(clipped_counts.size());
  double acc = 0.0;
  for (std::size_t b = 0; b < clipped_counts.size(); ++b) r.values[b] = acc += clipped_counts[b];
  const double first = r.values.front();
  const double span = r.values.back() - first;
  if (!(span > 0.0)) {
    r.values.assign(clipped_counts.size(), 0.5);
    r.degenerate = true;
    return r;
  }
  for (double& v : r.values) v = (v - first) / span;
  return r;
}

MappingGrid build_mappings(const KernelGrid& grid, const EnhanceParams& params,
                           const IntensityRange& global_range, unsigned threads) {
  // histogram.cpp:72-106, every block on the GPU
  (void)threads;
  check_params(params);
  const bool adaptive = params.range_mode == RangeMode::Adaptive;
  if (!adaptive && global_range.hi < global_range.lo)
    throw ValidationError("global range must satisfy lo <= hi");
  MappingGrid out;
  out.grid_shape = grid.grid_shape;
  out.n_bins = params.n_bins;
  const std::size_t nb = grid.block_count(), n = params.n_bins;
  out.mappings.resize(nb);
  if (nb == 0) return out;
  std::vector<double> lo(nb), hi(nb), lut(nb * n);
  std::vector<uint8_t> degen(nb);
  const int rc = mclahe_block_mappings(grid.blocks.data(), static_cast<int64_t>(nb),
                                       static_cast<int64_t>(grid.block_len),
                                       static_cast<int64_t>(n), params.clip_limit,
                                       adaptive ? 1 : 0, global_range.lo, global_range.hi,
                                       lo.data(), hi.data(), nullptr, nullptr, lut.data(),
                                       degen.data());
  if (rc != MCLAHE_OK) raise_gpu(rc);
  for (std::size_t k = 0; k < nb; ++k) {
    KernelMapping& m = out.mappings[k];
    m.range = IntensityRange{lo[k], hi[k]};
    m.values.assign(lut.begin() + static_cast<std::ptrdiff_t>(k * n),
                    lut.begin() + static_cast<std::ptrdiff_t>((k + 1) * n));
    m.degenerate = degen[k] != 0;
  }
  return out;
}

double apply_mapping(double value, const KernelMapping& mapping) {  // histogram.cpp:108-111
  return mapping.degenerate ? 0.5
                            : mapping.values[bin_index(value, mapping.range, mapping.values.size())];
}

}  // namespace mclahe
