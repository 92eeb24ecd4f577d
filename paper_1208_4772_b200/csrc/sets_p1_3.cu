// sets_p1_3.cu -- kernel instantiations for one group of level shapes
// <N_p, N_cub, N_g, ...> (see cdg_sets.cuh); compiled as its own translation unit.
#define CDG_SET_TU
#include "cdg_sets.cuh"

#ifndef CDG_P1NS_MINB
#define CDG_P1NS_MINB 4
#endif
#ifndef CDG_P1NS_WARPS
#define CDG_P1NS_WARPS 4
#endif

namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p1_3() {
  return {
      // straight-sided strengths (2p+1 / 2p): refelem.cpp:311-317
      // p=1: warp-tile kernel, 4 CTAs (16 warps) per SM at 128 registers (0.40 ms
      // vs 0.52 at 2 CTAs/SM and 0.50 for the row kernel, make_cube_mesh(44))
      with_ns<4, 5, 3, CDG_P1NS_WARPS, CDG_P1NS_MINB>(with_rowc<4, 5, 3, 8, 32, 4>(with_warp<4, 5, 3, 4, 4>(make_set<4, 5, 3, 16, 8, 2>()))),
      // p=2: row-per-warp kernel with fused traces and unrolled k-steps (3.14e10
      // DOF-updates/s vs 2.41e10 for the warp-tile kernel + trace kernel; the
      // warp-autonomous kernel 8% slower here); the set serves curved-mesh p=2
      // levels too (16-element affine tiles)
      with_rowc<10, 15, 6, 8, 32, 4>(with_row<10, 15, 6, 8, 32, 4, 224>(make_set<10, 15, 6, 16, 16, 2>())),
      // p=3 (straight): the warp-autonomous kernel, 16 warps x 1 CTA per SM
      // (0.454 of the FP64 peak vs 0.441 for the row kernel)
      with_wa<20, 35, 12, 8, 32, 16, 1>(make_set<20, 35, 12, 16, 16, 2>()),
      // curved-mesh strengths (3p-3 / 3p-2): refelem.hpp:118-119
      with_rowc<20, 35, 16, 8, 32, 4>(with_row<20, 35, 16, 8, 32, 4, 192>(make_set<20, 35, 16, 16, 16, 2>()))};
}

}  // namespace cdg_gpu
