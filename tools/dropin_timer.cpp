// tools/dropin_timer.cpp -- times mclahe::mclahe as a reference user calls it:
// an NdImage (float64) read from an NPY file, one request, the call alone
// between two steady_clock reads.  The same source links either the compiled
// reference (oracle/_ref/libmclahe_ref.so) or the B200 drop-in
// (libmclahe_cpp.so + libmclahe_gpu.so): only the library differs.
//   dropin_timer FILE.npy k0,k1,... n_bins clip adaptive reps threads
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "mclahe/npy.hpp"
#include "mclahe/pipeline.hpp"

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s FILE.npy k0,k1,.. n_bins clip adaptive reps threads\n", argv[0]);
    return 2;
  }
  auto loaded = mclahe::read_npy(argv[1]);
  mclahe::NdImage image = std::move(loaded.first);
  std::vector<std::size_t> k;
  std::stringstream ks(argv[2]);
  for (std::string t; std::getline(ks, t, ',');) k.push_back(std::stoul(t));
  mclahe::McLaheRequest req{std::move(image), mclahe::KernelSpec{k}, mclahe::EnhanceParams{},
                            static_cast<unsigned>(std::atoi(argv[7]))};
  req.params.n_bins = std::stoul(argv[3]);
  req.params.clip_limit = std::atof(argv[4]);
  req.params.range_mode = std::atoi(argv[5]) ? mclahe::RangeMode::Adaptive : mclahe::RangeMode::Global;
  const int reps = std::atoi(argv[6]);
  double best = 1e30, total = 0.0, checksum = 0.0;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    const mclahe::NdImage out = mclahe::mclahe(req);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    best = s < best ? s : best;
    total += s;
    checksum = 0.0;
    for (std::size_t i = 0; i < out.size(); i += 4099) checksum += out[i];
  }
  std::printf("{\"voxels\": %zu, \"reps\": %d, \"best_s\": %.6f, \"mean_s\": %.6f, \"checksum\": %.12g}\n",
              req.image.size(), reps, best, total / reps, checksum);
  return 0;
}
