// sets_p4.cu -- kernel instantiations for one group of level shapes
// <N_p, N_cub, N_g, ...> (see cdg_sets.cuh); compiled as its own translation unit.
#define CDG_SET_TU
#include "cdg_sets.cuh"

namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p4() {
  return {
      // default: row kernel with fused traces (the next stage's traces from its
      // epilogue), unrolled GEMM k-steps and fused-trace n-tile groups
      with_row<35, 70, 16, 8, 32, 4, 1248>(make_set<35, 70, 16, 16, 24, 2, 64>()),
      with_rowc<35, 70, 56, 8, 32, 4>(with_row<35, 70, 56, 8, 32, 4, 192>(make_set<35, 70, 56, 16, 24, 2>()))};
}

}  // namespace cdg_gpu
