// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the reference library compiled from its own sources under
// /root/reference/proj/core (oracle/Makefile builds both into
// oracle/_ref/libmclahe_ref.so).  It lets the Python tests and bench.py's
// reference arm drive the UNMODIFIED reference code through its public API:
// mclahe::mclahe (pipeline.hpp:30), build_mappings / compute_histogram /
// clip_histogram / normalized_cdf / bin_index / apply_mapping
// (histogram.hpp:51-80), neighbor_kernels / interp_coefficients /
// transform_pixel (interpolation.hpp:28-45), gaussian_filter / median_filter
// (filters.hpp:24-32) and the contrast metrics (metrics.hpp:19-36).
#include <array>
#include <cstdint>
#include <stdexcept>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mclahe/filters.hpp"
#include "mclahe/histogram.hpp"
#include "mclahe/interpolation.hpp"
#include "mclahe/metrics.hpp"
#include "mclahe/npy.hpp"
#include "mclahe/parallel.hpp"
#include "mclahe/nd_image.hpp"
#include "mclahe/pipeline.hpp"

namespace {

void put_err(char* err, int len, const char* what) {
  if (err && len > 0) {
    std::strncpy(err, what, static_cast<size_t>(len) - 1);
    err[len - 1] = '\0';
  }
}

mclahe::NdImage make_image(const double* data, int rank, const int64_t* shape) {
  mclahe::Shape s(shape, shape + rank);
  size_t n = 1;
  for (int i = 0; i < rank; ++i) n *= static_cast<size_t>(shape[i]);
  return mclahe::NdImage(std::move(s), std::vector<double>(data, data + n));
}

}  // namespace

extern "C" {

// Runs mclahe::mclahe end to end.  timings (nullable) receives
// {pad_s, histograms_s, interpolation_s}.  Returns 0, 1 (ValidationError) or
// 2 (other exception) with the message in err.
int ref_mclahe(const double* data, int rank, const int64_t* shape, const int64_t* kernel,
               int64_t n_bins, double clip_limit, int adaptive, unsigned threads,
               double* out, double* timings, char* err, int err_len) {
  try {
    mclahe::McLaheRequest req{make_image(data, rank, shape),
                              mclahe::KernelSpec{std::vector<size_t>(kernel, kernel + rank)},
                              mclahe::EnhanceParams{}, threads};
    req.params.clip_limit = clip_limit;
    req.params.n_bins = static_cast<size_t>(n_bins);
    req.params.range_mode = adaptive ? mclahe::RangeMode::Adaptive : mclahe::RangeMode::Global;
    mclahe::PhaseTimings pt;
    const mclahe::NdImage res = mclahe::mclahe(req, &pt);
    std::memcpy(out, res.values().data(), res.size() * sizeof(double));
    if (timings) {
      timings[0] = pt.pad_s;
      timings[1] = pt.histograms_s;
      timings[2] = pt.interpolation_s;
    }
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 2;
  }
}

// Per-tile intermediates through the reference's public API: pad plan,
// symmetric_pad, kernelize, then build_mappings for ranges / LUTs and
// compute_histogram + clip_histogram per block for counts and clipped counts
// (zero for degenerate-range tiles, which build_mappings never bins).
int ref_tile_stats(const double* data, int rank, const int64_t* shape, const int64_t* kernel,
                   int64_t n_bins, double clip_limit, int adaptive, double* lo, double* hi,
                   double* counts, double* clipped, double* lut, uint8_t* degenerate,
                   char* err, int err_len) {
  try {
    const mclahe::NdImage image = make_image(data, rank, shape);
    const mclahe::KernelSpec ks{std::vector<size_t>(kernel, kernel + rank)};
    const mclahe::PadPlan plan = mclahe::compute_pad_plan(image.shape(), ks);
    const mclahe::NdImage padded = mclahe::symmetric_pad(image, plan);
    const mclahe::KernelGrid grid = mclahe::kernelize(padded, ks);
    mclahe::EnhanceParams params;
    params.clip_limit = clip_limit;
    params.n_bins = static_cast<size_t>(n_bins);
    params.range_mode = adaptive ? mclahe::RangeMode::Adaptive : mclahe::RangeMode::Global;
    mclahe::IntensityRange global;
    image.min_max(global.lo, global.hi);
    const mclahe::MappingGrid maps = mclahe::build_mappings(grid, params, global, 1);
    const size_t nb = static_cast<size_t>(n_bins);
    for (size_t k = 0; k < grid.block_count(); ++k) {
      const mclahe::KernelMapping& m = maps.at(k);
      if (lo) lo[k] = m.range.lo;
      if (hi) hi[k] = m.range.hi;
      if (degenerate) degenerate[k] = m.degenerate ? 1 : 0;
      if (lut) std::memcpy(lut + k * nb, m.values.data(), nb * sizeof(double));
      std::vector<double> c(nb, 0.0), cl(nb, 0.0);
      if (!m.range.degenerate()) {
        c = mclahe::compute_histogram(grid.block(k), m.range, nb);
        cl = mclahe::clip_histogram(c, clip_limit);
      }
      if (counts) std::memcpy(counts + k * nb, c.data(), nb * sizeof(double));
      if (clipped) std::memcpy(clipped + k * nb, cl.data(), nb * sizeof(double));
    }
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 2;
  }
}

// ref_tile_stats for a window of tile rows [tile_row0, tile_row0 + tile_rows)
// along dim 0, multi-threaded through the reference's own parallel_for
// (parallel.hpp:23-61; results do not depend on the worker count).  With
// has_global the Global-mode range is (glo, hi) instead of the image's own
// min/max: the full-size gate runs the reference on dim-0 crops of a volume
// too large for its padded + kernelized copies, and a crop's interior tile
// rows equal the full volume's once the full volume's range is used.
int ref_tile_stats_window(const double* data, int rank, const int64_t* shape,
                          const int64_t* kernel, int64_t n_bins, double clip_limit, int adaptive,
                          int has_global, double glo, double ghi, int64_t tile_row0,
                          int64_t tile_rows, unsigned threads, double* lo, double* hi,
                          double* counts, double* clipped, double* lut, uint8_t* degenerate,
                          char* err, int err_len) {
  try {
    const mclahe::NdImage image = make_image(data, rank, shape);
    const mclahe::KernelSpec ks{std::vector<size_t>(kernel, kernel + rank)};
    const mclahe::PadPlan plan = mclahe::compute_pad_plan(image.shape(), ks);
    const mclahe::NdImage padded = mclahe::symmetric_pad(image, plan);
    const mclahe::KernelGrid grid = mclahe::kernelize(padded, ks);
    mclahe::EnhanceParams params;
    params.clip_limit = clip_limit;
    params.n_bins = static_cast<size_t>(n_bins);
    params.range_mode = adaptive ? mclahe::RangeMode::Adaptive : mclahe::RangeMode::Global;
    mclahe::IntensityRange global;
    if (has_global) {
      global.lo = glo;
      global.hi = ghi;
    } else {
      image.min_max(global.lo, global.hi);
    }
    const mclahe::MappingGrid maps = mclahe::build_mappings(grid, params, global, threads);
    const size_t per_row = grid.block_count() / grid.grid_shape[0];
    const size_t k0 = static_cast<size_t>(tile_row0) * per_row;
    const size_t nk = static_cast<size_t>(tile_rows) * per_row;
    if (k0 + nk > grid.block_count()) throw std::runtime_error("tile-row window out of range");
    const size_t nb = static_cast<size_t>(n_bins);
    mclahe::parallel_for(nk, threads, [&](size_t begin, size_t end) {
      for (size_t i = begin; i < end; ++i) {
        const size_t k = k0 + i;
        const mclahe::KernelMapping& m = maps.at(k);
        lo[i] = m.range.lo;
        hi[i] = m.range.hi;
        degenerate[i] = m.degenerate ? 1 : 0;
        std::memcpy(lut + i * nb, m.values.data(), nb * sizeof(double));
        std::vector<double> c(nb, 0.0), cl(nb, 0.0);
        if (!m.range.degenerate()) {
          c = mclahe::compute_histogram(grid.block(k), m.range, nb);
          cl = mclahe::clip_histogram(c, clip_limit);
        }
        std::memcpy(counts + i * nb, c.data(), nb * sizeof(double));
        std::memcpy(clipped + i * nb, cl.data(), nb * sizeof(double));
      }
    });
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 2;
  }
}

// The per-voxel loop of mclahe::mclahe (src/pipeline.cpp:94-127) for the
// original rows [row0, row1) of a volume of shape `shape`, over mappings given
// for the tile rows [tile_row0, tile_row0 + tile_rows) (lo / hi / lut /
// degenerate as ref_tile_stats_window returns them).  `rows` holds only those
// voxel rows.  Each voxel goes through the reference's neighbor_kernels,
// interp_coefficients and transform_pixel; mappings outside the window throw.
int ref_blend_rows(const double* rows, int rank, const int64_t* shape, const int64_t* kernel,
                   int64_t row0, int64_t row1, int64_t n_bins, int64_t tile_row0,
                   int64_t tile_rows, const double* lo, const double* hi, const double* lut,
                   const uint8_t* degenerate, unsigned threads, double* out, char* err,
                   int err_len) {
  try {
    const mclahe::Shape full(shape, shape + rank);
    const mclahe::KernelSpec ks{std::vector<size_t>(kernel, kernel + rank)};
    const mclahe::PadPlan plan = mclahe::compute_pad_plan(full, ks);
    mclahe::Shape gshape(rank);
    for (int j = 0; j < rank; ++j)
      gshape[j] = (full[j] + plan.before[j] + plan.after[j]) / ks.sizes[j];
    const auto gstrides = mclahe::row_major_strides(gshape);
    const size_t per_row = gstrides[0];
    const size_t nb = static_cast<size_t>(n_bins);
    std::vector<mclahe::KernelMapping> maps(static_cast<size_t>(tile_rows) * per_row);
    for (size_t i = 0; i < maps.size(); ++i) {
      maps[i].range = {lo[i], hi[i]};
      maps[i].values.assign(lut + i * nb, lut + (i + 1) * nb);
      maps[i].degenerate = degenerate[i] != 0;
    }
    mclahe::Shape local = full;
    local[0] = static_cast<size_t>(row1 - row0);
    const size_t n = mclahe::shape_product(local);
    const size_t corners = mclahe::corner_count(static_cast<size_t>(rank));
    const size_t first = static_cast<size_t>(tile_row0) * per_row;
    mclahe::parallel_for(n, threads, [&](size_t begin, size_t end) {
      std::array<size_t, mclahe::kMaxRank> pixel{};
      std::array<double, mclahe::kMaxCorners> coeffs;
      std::array<const mclahe::KernelMapping*, mclahe::kMaxCorners> nmaps;
      std::vector<size_t> coord(rank, 0);
      mclahe::unflatten(begin, local, coord);
      for (size_t flat = begin; flat < end; ++flat) {
        for (int j = 0; j < rank; ++j) pixel[j] = coord[j] + plan.before[j];
        pixel[0] += static_cast<size_t>(row0);
        const mclahe::NeighborSet ns = mclahe::neighbor_kernels({pixel.data(), size_t(rank)}, ks, gshape);
        mclahe::interp_coefficients(ns, ks, {coeffs.data(), corners});
        for (size_t c = 0; c < corners; ++c) {
          size_t g = 0;
          for (int j = 0; j < rank; ++j) g += (ns.lower[j] + ((c >> (rank - 1 - j)) & 1u)) * gstrides[j];
          if (g < first || g - first >= maps.size()) throw std::runtime_error("mapping outside the window");
          nmaps[c] = &maps[g - first];
        }
        out[flat] = mclahe::transform_pixel(rows[flat], {nmaps.data(), corners}, {coeffs.data(), corners});
        mclahe::next_coord(coord, local);
      }
    });
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 2;
  }
}

int64_t ref_bin_index(double value, double lo, double hi, int64_t n_bins) {
  try {
    return static_cast<int64_t>(
        mclahe::bin_index(value, mclahe::IntensityRange{lo, hi}, static_cast<size_t>(n_bins)));
  } catch (...) {
    return -1;
  }
}

void ref_clip_histogram(const double* counts, int64_t n, double clip_limit, double* out) {
  const std::vector<double> r =
      mclahe::clip_histogram(std::span<const double>(counts, static_cast<size_t>(n)), clip_limit);
  std::memcpy(out, r.data(), r.size() * sizeof(double));
}

int ref_normalized_cdf(const double* clipped, int64_t n, double* out) {
  const mclahe::NormalizedCdf r =
      mclahe::normalized_cdf(std::span<const double>(clipped, static_cast<size_t>(n)));
  std::memcpy(out, r.values.data(), r.values.size() * sizeof(double));
  return r.degenerate ? 1 : 0;
}

// neighbor_kernels + interp_coefficients for one padded pixel.  Returns 0 or
// 1 (ValidationError).
int ref_neighbors(int rank, const int64_t* pixel, const int64_t* kernel, const int64_t* grid,
                  int64_t* lower, double* dist_lo, double* dist_hi, double* coeff) {
  try {
    std::vector<size_t> px(pixel, pixel + rank), gs(grid, grid + rank);
    const mclahe::KernelSpec ks{std::vector<size_t>(kernel, kernel + rank)};
    const mclahe::NeighborSet ns = mclahe::neighbor_kernels(px, ks, gs);
    for (int j = 0; j < rank; ++j) {
      lower[j] = static_cast<int64_t>(ns.lower[j]);
      dist_lo[j] = ns.dist_lo[j];
      dist_hi[j] = ns.dist_hi[j];
    }
    mclahe::interp_coefficients(ns, ks, std::span<double>(coeff, size_t{1} << rank));
    return 0;
  } catch (const mclahe::ValidationError&) {
    return 1;
  }
}

// transform_pixel over explicit per-corner LUTs (n_bins each, ranges lo/hi,
// degenerate flags).
double ref_transform_pixel(double value, int corners, const double* luts, int64_t n_bins,
                           const double* lo, const double* hi, const uint8_t* degenerate,
                           const double* coeff) {
  std::vector<mclahe::KernelMapping> maps(static_cast<size_t>(corners));
  std::vector<const mclahe::KernelMapping*> ptrs;
  for (int c = 0; c < corners; ++c) {
    maps[c].range = {lo[c], hi[c]};
    maps[c].values.assign(luts + c * n_bins, luts + (c + 1) * n_bins);
    maps[c].degenerate = degenerate[c] != 0;
    ptrs.push_back(&maps[c]);
  }
  return mclahe::transform_pixel(value, ptrs,
                                 std::span<const double>(coeff, static_cast<size_t>(corners)));
}

// gaussian_filter (filters.hpp:24-25): 0 ok, 1 ValidationError (message in err).
int ref_gaussian(const double* data, int rank, const int64_t* shape, const double* sigmas,
                 double truncate, double* out, char* err, int err_len) {
  try {
    mclahe::GaussianSpec spec;
    spec.sigmas.assign(sigmas, sigmas + rank);
    spec.truncate = truncate;
    const mclahe::NdImage r = mclahe::gaussian_filter(make_image(data, rank, shape), spec, 1);
    std::memcpy(out, r.values().data(), r.size() * sizeof(double));
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// median_filter (filters.hpp:30-32).
int ref_median(const double* data, int rank, const int64_t* shape, const int64_t* window,
               double* out, char* err, int err_len) {
  try {
    mclahe::MedianSpec spec;
    for (int i = 0; i < rank; ++i) spec.window.push_back(static_cast<size_t>(window[i]));
    const mclahe::NdImage r = mclahe::median_filter(make_image(data, rank, shape), spec, 1);
    std::memcpy(out, r.values().data(), r.size() * sizeof(double));
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// compute_metrics (metrics.hpp:35-36): out = {mse, psnr_db, std, entropy_bits}.
int ref_metrics(const double* a, const double* b, int rank, const int64_t* shape,
                int64_t n_bins, double peak, double* out, char* err, int err_len) {
  try {
    const mclahe::MetricsReport m = mclahe::compute_metrics(
        make_image(a, rank, shape), make_image(b, rank, shape), static_cast<size_t>(n_bins), peak);
    out[0] = m.mse;
    out[1] = m.psnr_db;
    out[2] = m.std;
    out[3] = m.entropy_bits;
    return 0;
  } catch (const mclahe::ValidationError& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// write_npy (npy.hpp:50-53): dtype by name ("f4", ...); 0 ok, else the NpyErrc + 1.
int ref_write_npy(const char* path, const double* data, int rank, const int64_t* shape,
                  const char* dtype, char* err, int err_len) {
  try {
    mclahe::write_npy(path, make_image(data, rank, shape), mclahe::dtype_from_name(dtype));
    return 0;
  } catch (const mclahe::NpyError& e) {
    put_err(err, err_len, e.what());
    return static_cast<int>(e.code()) + 1;
  }
}

// read_npy (npy.hpp:46-48) into caller buffers (at most max_count values).
int ref_read_npy(const char* path, double* data, int64_t max_count, int* rank, int64_t* shape,
                 char* descr, char* err, int err_len) {
  try {
    auto [img, meta] = mclahe::read_npy(path);
    if (static_cast<int64_t>(img.size()) > max_count) return 100;
    std::memcpy(data, img.values().data(), img.size() * sizeof(double));
    *rank = static_cast<int>(meta.shape.size());
    for (size_t i = 0; i < meta.shape.size(); ++i) shape[i] = static_cast<int64_t>(meta.shape[i]);
    std::strcpy(descr, mclahe::dtype_descr(meta.dtype).c_str());
    return 0;
  } catch (const mclahe::NpyError& e) {
    put_err(err, err_len, e.what());
    return static_cast<int>(e.code()) + 1;
  }
}

}  // extern "C"
