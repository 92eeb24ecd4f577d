// sets_p4.cu -- kernel instantiations for one group of level shapes
// <N_p, N_cub, N_g, ...> (see cdg_sets.cuh); compiled as its own translation unit.
#define CDG_SET_TU
#include "cdg_sets.cuh"

namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p4() {
  return {
      with_row<35, 70, 16, 8, 32, 4, 0>(make_set<35, 70, 16, 16, 24, 2, 64>()),
      with_row<35, 70, 56, 8, 32, 4, 0>(make_set<35, 70, 56, 16, 24, 2>()),
      // P=4 straight tuning variants, selected with CDG_KCFG=<n> (bench sweeps)
      make_set<35, 70, 16, 16, 24, 2, 64>(),
      with_rowp<35, 70, 16, 4, false>(make_set<35, 70, 16, 16, 24, 2, 64>()),
      with_rowp<35, 70, 16, 4, true>(make_set<35, 70, 16, 16, 24, 2, 64>()),
      with_rowp<35, 70, 16, 3, true>(make_set<35, 70, 16, 16, 24, 2, 64>())};
}

}  // namespace cdg_gpu
