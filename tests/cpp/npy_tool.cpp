// Drives the drop-in's array-file API (mclahe_b200.hpp, the reference's
// npy.hpp): `write <path> <dtype> <rank> <extents...>` writes the pattern
// v_i = (i * 7 % 23) - 9.25 (integers: rounded, in range); `read <path>`
// prints descr, shape and values; `raw <path> <dtype> <extents...>`.
// Errors print "NpyError <code> <message>" and exit 3.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mclahe/npy.hpp"

int main(int argc, char** argv) {
  try {
    if (argc >= 5 && std::strcmp(argv[1], "write") == 0) {
      const mclahe::Dtype dt = mclahe::dtype_from_name(argv[3]);
      const int rank = std::atoi(argv[4]);
      mclahe::Shape shape;
      std::size_t n = 1;
      for (int i = 0; i < rank; ++i) {
        shape.push_back(std::strtoull(argv[5 + i], nullptr, 10));
        n *= shape.back();
      }
      std::vector<double> v(n);
      const bool integer = dt != mclahe::Dtype::f4 && dt != mclahe::Dtype::f8;
      const bool unsigned_ = dt == mclahe::Dtype::u1 || dt == mclahe::Dtype::u2;
      for (std::size_t i = 0; i < n; ++i) {
        v[i] = static_cast<double>(i * 7 % 23) - 9.25;
        if (integer && unsigned_) v[i] += 9.75;  // 0.5 .. 22.5: halves round away from zero
      }
      mclahe::write_npy(argv[2], mclahe::NdImage(shape, v), dt);
      return 0;
    }
    if (argc == 5 && std::strcmp(argv[1], "writev") == 0) {  // one value
      mclahe::write_npy(argv[2], mclahe::NdImage({1}, {std::strtod(argv[4], nullptr)}),
                        mclahe::dtype_from_name(argv[3]));
      return 0;
    }
    if (argc >= 3 && (std::strcmp(argv[1], "read") == 0 || std::strcmp(argv[1], "raw") == 0)) {
      mclahe::NdImage img = mclahe::NdImage::zeros({1});
      mclahe::ArrayFileMeta meta;
      if (argv[1][1] == 'e') {
        auto r = mclahe::read_npy(argv[2]);
        img = std::move(r.first);
        meta = r.second;
      } else {
        meta.dtype = mclahe::dtype_from_name(argv[3]);
        for (int i = 4; i < argc; ++i) meta.shape.push_back(std::strtoull(argv[i], nullptr, 10));
        img = mclahe::read_raw(argv[2], meta);
      }
      std::printf("%s", mclahe::dtype_descr(meta.dtype).c_str());
      for (std::size_t e : img.shape()) std::printf(" %zu", e);
      std::printf("\n");
      for (std::size_t i = 0; i < img.size(); ++i) std::printf("%.17g\n", img[i]);
      return 0;
    }
  } catch (const mclahe::NpyError& e) {
    std::printf("NpyError %d %s\n", static_cast<int>(e.code()), e.what());
    return 3;
  }
  return 2;
}
