// sets_p7_8.cu -- kernel instantiations for one group of level shapes
// <N_p, N_cub, N_g, ...> (see cdg_sets.cuh); compiled as its own translation unit.
#define CDG_SET_TU
#include "cdg_sets.cuh"

namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p7_8() {
  return {
      // (the warp-autonomous kernel measured equal at p=7)
      make_set<120, 330, 120, 16>(), make_set<165, 495, 165, 16>(),
      make_set<120, 715, 220, 16>(), make_set<165, 1001, 364, 16>()};
}

}  // namespace cdg_gpu
