// k_hist.cu -- instantiations of the K2a/K2b pencil kernels (own translation
// unit so the build compiles kernel families in parallel).
#include "k_pencil.cuh"

namespace mg {

template <bool DICT>
static PencilRangeFn range_t(int ko) {
  switch (ko) {
    case 1: return k_range_pencil<1, DICT>;
    case 2: return k_range_pencil<2, DICT>;
    case 3: return k_range_pencil<3, DICT>;
    case 4: return k_range_pencil<4, DICT>;
    default: return k_range_pencil<5, DICT>;
  }
}

PencilRangeFn get_range_pencil(int ko, bool dict) {
  return dict ? range_t<true>(ko) : range_t<false>(ko);
}

template <bool A, bool MATCH, bool CARRY>
static PencilHistFn hist_t(int ko) {
  switch (ko) {
    case 1: return k_hist_pencil<1, A, MATCH, CARRY>;
    case 2: return k_hist_pencil<2, A, MATCH, CARRY>;
    case 3: return k_hist_pencil<3, A, MATCH, CARRY>;
    case 4: return k_hist_pencil<4, A, MATCH, CARRY>;
    default: return k_hist_pencil<5, A, MATCH, CARRY>;
  }
}

PencilHistFn get_hist_pencil(int ko, bool adaptive, int variant) {
  if (variant == 1) return adaptive ? hist_t<true, true, false>(ko) : hist_t<false, true, false>(ko);
  if (variant == 2) return adaptive ? hist_t<true, false, true>(ko) : hist_t<false, false, true>(ko);
  return adaptive ? hist_t<true, false, false>(ko) : hist_t<false, false, false>(ko);
}

PencilHistFn get_hist_cells(int ko) {
  switch (ko) {
    case 1: return k_hist_cells<1>;
    case 2: return k_hist_cells<2>;
    case 3: return k_hist_cells<3>;
    case 4: return k_hist_cells<4>;
    default: return k_hist_cells<5>;
  }
}

}  // namespace mg
