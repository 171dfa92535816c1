// k_interp_adaptive_nb.cu -- K4 pencil kernels, adaptive range mode, with the
// bin count fixed at compile time (per-tile blocks, immediate-offset gathers).
#include "k_pencil.cuh"

namespace mg {

template <int KT, int NB>
static PencilInterpFn interp_nb(int ko) {
  switch (ko) {
    case 1: return k_interp_pencil<1, KT, true, NB>;
    case 2: return k_interp_pencil<2, KT, true, NB>;
    case 3: return k_interp_pencil<3, KT, true, NB>;
    default: return k_interp_pencil<4, KT, true, NB>;
  }
}

// nullptr when n_bins has no specialisation (the runtime-n kernel runs).
PencilInterpFn get_interp_pencil_adaptive_nb(int ko, int kt, int n_bins) {
  switch (n_bins) {
    case 128: return kt == 1 ? interp_nb<1, 128>(ko) : interp_nb<2, 128>(ko);
    case 256: return kt == 1 ? interp_nb<1, 256>(ko) : interp_nb<2, 256>(ko);
    default: return nullptr;
  }
}

template <int KT>
static PencilInterpFn interp_dict(int ko) {
  switch (ko) {
    case 1: return k_interp_pencil<1, KT, true, -1>;
    case 2: return k_interp_pencil<2, KT, true, -1>;
    case 3: return k_interp_pencil<3, KT, true, -1>;
    default: return k_interp_pencil<4, KT, true, -1>;
  }
}

PencilInterpFn get_interp_pencil_dict(int ko, int kt) {
  return kt == 1 ? interp_dict<1>(ko) : interp_dict<2>(ko);
}

}  // namespace mg
