// k_interp_adaptive.cu -- instantiations of the K4 pencil kernel, adaptive range mode.
#include "k_pencil.cuh"

namespace mg {

template <int KT>
static PencilInterpFn interp_adaptive(int ko) {
  switch (ko) {
    case 1: return k_interp_pencil<1, KT, true>;
    case 2: return k_interp_pencil<2, KT, true>;
    case 3: return k_interp_pencil<3, KT, true>;
    default: return k_interp_pencil<4, KT, true>;
  }
}

PencilInterpFn get_interp_pencil_adaptive(int ko, int kt) {
  return kt == 1 ? interp_adaptive<1>(ko) : interp_adaptive<2>(ko);
}

}  // namespace mg
