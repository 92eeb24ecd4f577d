// sets_p5_6.cu -- kernel instantiations for one group of level shapes
// <N_p, N_cub, N_g, ...> (see cdg_sets.cuh); compiled as its own translation unit.
#define CDG_SET_TU
#include "cdg_sets.cuh"


namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p5_6() {
  return {
      // p=5: the warp-autonomous kernel with fused traces, 16 warps x 1 CTA/SM
      // (56.2 ms per step at 511k tets vs 64.7 for the row kernel + trace kernel)
      with_wa<56, 126, 56, 8, 32, 16, 1, false, true>(make_set<56, 126, 56, 16, 16, 2>()),
      // p=6: CTA kernel with 8-node chunks (27.8 vs 34.8 ms; the warp-autonomous
      // kernel 3% slower here)
      make_set<84, 210, 84, 16, 8, 2, 16>(),
      with_rowc<56, 210, 84, 8, 32, 3>(with_row<56, 210, 84, 8, 32, 3, 192>(make_set<56, 210, 84, 16, 16, 2>())), make_set<84, 330, 165, 16>()};
}

}  // namespace cdg_gpu
