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
PencilInterpFn get_interp_pencil(int ko, int kt, bool adaptive) {
  return adaptive ? get_interp_pencil_adaptive(ko, kt) : get_interp_pencil_global(ko, kt);
}
}  // namespace mg
