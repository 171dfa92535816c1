// A caller of the reference API (the reference headers mclahe/*.hpp, rebuilt
// under include/mclahe): builds an
// image, runs mclahe::mclahe, prints a checksum (or exercises validation).
#include <cstdio>
#include <cstring>
#include <vector>

#include "mclahe/pipeline.hpp"
#include "mclahe/filters.hpp"
#include "mclahe/metrics.hpp"

int main(int argc, char** argv) {
  const bool validate_only = argc > 1 && std::strcmp(argv[1], "validate") == 0;
  mclahe::Shape shape{24, 20, 16};
  std::vector<double> data(24 * 20 * 16);
  for (std::size_t i = 0; i < data.size(); ++i) data[i] = static_cast<double>((i * 37) % 101) / 100.0;
  mclahe::McLaheRequest req{mclahe::NdImage(shape, data), mclahe::KernelSpec{{8, 4, 4}},
                            mclahe::EnhanceParams{}, 0};
  req.params.clip_limit = 0.05;
  req.params.n_bins = 32;
  req.params.range_mode = mclahe::RangeMode::Adaptive;
  if (validate_only) {
    int caught = 0;
    try {
      mclahe::McLaheRequest bad = req;
      bad.params.clip_limit = 0.0;
      mclahe::mclahe(bad);
    } catch (const mclahe::ValidationError& e) {
      std::printf("ValidationError: %s\n", e.what());
      caught += std::strcmp(e.what(), "clip_limit must be in (0, 1]") == 0;
    }
    try {
      mclahe::McLaheRequest bad = req;
      bad.kernel.sizes = {8, 4};
      mclahe::mclahe(bad);
    } catch (const mclahe::ValidationError& e) {
      std::printf("ValidationError: %s\n", e.what());
      caught += std::strcmp(e.what(), "kernel rank 2 does not match image rank 3") == 0;
    }
    return caught == 2 ? 0 : 1;
  }
  mclahe::PhaseTimings t;
  if (argc > 1 && std::strcmp(argv[1], "framewise") == 0) {  // slices along axis 1, global range
    mclahe::EnhanceParams prm = req.params;
    prm.range_mode = mclahe::RangeMode::Global;
    const mclahe::NdImage out =
        mclahe::mclahe_framewise(req.image, 1, mclahe::KernelSpec{{8, 4}}, prm, 0, false, &t);
    for (std::size_t i = 0; i < out.size(); ++i) std::printf("%.17g\n", out[i]);
    return 0;
  }
  if (argc > 1 && std::strcmp(argv[1], "filters") == 0) {  // smooth, enhance, measure
    const mclahe::NdImage g = mclahe::gaussian_filter(req.image, mclahe::GaussianSpec{{1.0, 0.5, 0.0}, 4.0});
    const mclahe::NdImage m = mclahe::median_filter(g, mclahe::MedianSpec{{3, 1, 2}});
    const mclahe::MetricsReport r = mclahe::compute_metrics(m, req.image, 64, 1.0);
    for (std::size_t i = 0; i < m.size(); ++i) std::printf("%.17g\n", m[i]);
    std::printf("%.17g\n%.17g\n%.17g\n%.17g\n", r.mse, r.psnr_db, r.std, r.entropy_bits);
    return 0;
  }
  const mclahe::NdImage out = mclahe::mclahe(req, &t);
  for (std::size_t i = 0; i < out.size(); ++i) std::printf("%.17g\n", out[i]);
  std::fprintf(stderr, "hist %.3g s interp %.3g s\n", t.histograms_s, t.interpolation_s);
  return 0;
}
