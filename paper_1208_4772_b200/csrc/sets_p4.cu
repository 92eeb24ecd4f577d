// sets_p4.cu -- kernel instantiations for one group of level shapes
// <N_p, N_cub, N_g, ...> (see cdg_sets.cuh); compiled as its own translation unit.
#define CDG_SET_TU
#include "cdg_sets.cuh"

// <CH, FCH, CTAs/SM, MODE, E> of the P=4 straight row kernel (RCfg); tuning
// builds (build.build_variant) override it, the product build uses this
#ifndef CDG_P4_CH
#define CDG_P4_CH 8
#endif
#ifndef CDG_P4_FCH
#define CDG_P4_FCH 32
#endif
#ifndef CDG_P4_MINB
#define CDG_P4_MINB 4
#endif
#ifndef CDG_P4_MODE
#define CDG_P4_MODE 1248
#endif
#ifndef CDG_P4_E
#define CDG_P4_E 16
#endif

// <CH, FCH, CTAs/SM> of the P=4 curved-mesh row kernel (k_rhs_rowc)
#ifndef CDG_P4C_CH
#define CDG_P4C_CH 8
#endif
#ifndef CDG_P4C_FCH
#define CDG_P4C_FCH 32
#endif
#ifndef CDG_P4C_MINB
#define CDG_P4C_MINB 4
#endif

namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p4() {
  return {
      // default: row kernel with fused traces (the next stage's traces from its
      // epilogue), unrolled GEMM k-steps and fused-trace n-tile groups
      with_row<35, 70, 16, CDG_P4_CH, CDG_P4_FCH, CDG_P4_MINB, CDG_P4_MODE, CDG_P4_E>(make_set<35, 70, 16, 16, 24, 2, 64>()),
      with_rowc<35, 70, 56, CDG_P4C_CH, CDG_P4C_FCH, CDG_P4C_MINB>(with_row<35, 70, 56, 8, 32, 4, 192>(make_set<35, 70, 56, 16, 24, 2>()))};
}

}  // namespace cdg_gpu
