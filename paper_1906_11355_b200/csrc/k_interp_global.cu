// k_interp_global.cu -- instantiations of the K4 pencil kernel, global range mode.
#include "k_pencil.cuh"

namespace mg {

template <int KT>
static PencilInterpFn interp_global(int ko) {
  switch (ko) {
    case 1: return k_interp_pencil<1, KT, false>;
    case 2: return k_interp_pencil<2, KT, false>;
    case 3: return k_interp_pencil<3, KT, false>;
    default: return k_interp_pencil<4, KT, false>;
  }
}

PencilInterpFn get_interp_pencil_global(int ko, int kt) {
  return kt == 1 ? interp_global<1>(ko) : interp_global<2>(ko);
}

}  // namespace mg

namespace mg {
PencilInterpFn get_interp_pencil_adaptive(int ko, int kt);
PencilInterpFn get_interp_pencil_adaptive_nb(int ko, int kt, int n_bins);
PencilInterpFn get_interp_pencil(int ko, int kt, bool adaptive, int n_bins) {
  if (!adaptive) return get_interp_pencil_global(ko, kt);
  if (PencilInterpFn f = get_interp_pencil_adaptive_nb(ko, kt, n_bins)) return f;
  return get_interp_pencil_adaptive(ko, kt);
}
}  // namespace mg
