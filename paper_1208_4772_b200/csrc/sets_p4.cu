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
// 1 (default): the warp-autonomous kernel (cdg_wa.cuh) for the straight P=4
// set -- 16 warps x 1 CTA per SM, 128 registers (0.62 of the FP64 peak vs
// 0.58 for the row kernel, scripts/tune_p4.py)
#ifndef CDG_P4_WA
#define CDG_P4_WA 1
#endif
#ifndef CDG_P4_WA_WARPS
#define CDG_P4_WA_WARPS 16
#endif
#ifndef CDG_P4_WA_MINB
#define CDG_P4_WA_MINB 1
#endif
#ifndef CDG_P4_WA_UREG
#define CDG_P4_WA_UREG 0
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

// 1 (default): the warp-autonomous curved kernel (cdg_wac.cuh) for the curved
// P=4 set, 16 warps x 1 CTA per SM (0.434 / 0.367 of the FP64 peak LLF / HLLC
// vs 0.422 / 0.355 for k_rhs_rowc; 12 / 10 / 8 warps with 168+ registers:
// 0.403 / 0.342 / 0.324); the aux gradient: CDG_P4C_AUXW below
#ifndef CDG_P4C_WAC
#define CDG_P4C_WAC 1
#endif
// MODE of the row kernel that serves the affine elements of curved P=4 levels
// (192: no fused traces -- mixed levels keep the trace kernel; 224: fused,
// measured 2-3% slower per step at 40% / 10% curved)
#ifndef CDG_P4C_ROWMODE
#define CDG_P4C_ROWMODE 192
#endif
#ifndef CDG_P4C_WAC_WARPS
#define CDG_P4C_WAC_WARPS 16
#endif
#ifndef CDG_P4C_WAC_MINB
#define CDG_P4C_WAC_MINB 1
#endif
// warps of the warp-autonomous aux-gradient kernel (0: k_rhs_rowc KIND 2);
// 8 warps x 1 CTA/SM at 255 registers: AV step 33.1 -> 29.8 ms at 82,944 curved tets
#ifndef CDG_P4C_AUXW
#define CDG_P4C_AUXW 8
#endif

namespace cdg_gpu {

std::vector<KernelSet> kernel_sets_p4() {
  return {
      // default: row kernel with fused traces (the next stage's traces from its
      // epilogue), unrolled GEMM k-steps and fused-trace n-tile groups
#if CDG_P4_WA
      with_wa<35, 70, 16, 8, CDG_P4_FCH, CDG_P4_WA_WARPS, CDG_P4_WA_MINB, CDG_P4_WA_UREG>(make_set<35, 70, 16, 16, 24, 2, 64>()),
#else
      with_row<35, 70, 16, CDG_P4_CH, CDG_P4_FCH, CDG_P4_MINB, CDG_P4_MODE, CDG_P4_E>(make_set<35, 70, 16, 16, 24, 2, 64>()),
#endif
#if CDG_P4C_WAC && CDG_P4C_AUXW
      with_wac_aux<35, 70, 56, 8, 32, CDG_P4C_AUXW>(with_wac<35, 70, 56, 8, CDG_P4C_FCH, CDG_P4C_WAC_WARPS, CDG_P4C_WAC_MINB>(
          with_rowc<35, 70, 56, CDG_P4C_CH, CDG_P4C_FCH, CDG_P4C_MINB>(with_row<35, 70, 56, 8, 32, 4, CDG_P4C_ROWMODE>(make_set<35, 70, 56, 16, 24, 2>()))))};
#elif CDG_P4C_WAC
      with_wac<35, 70, 56, 8, CDG_P4C_FCH, CDG_P4C_WAC_WARPS, CDG_P4C_WAC_MINB>(
          with_rowc<35, 70, 56, CDG_P4C_CH, CDG_P4C_FCH, CDG_P4C_MINB>(with_row<35, 70, 56, 8, 32, 4, CDG_P4C_ROWMODE>(make_set<35, 70, 56, 16, 24, 2>())))};
#else
      with_rowc<35, 70, 56, CDG_P4C_CH, CDG_P4C_FCH, CDG_P4C_MINB>(with_row<35, 70, 56, 8, 32, 4, CDG_P4C_ROWMODE>(make_set<35, 70, 56, 16, 24, 2>()))};
#endif
}

}  // namespace cdg_gpu
