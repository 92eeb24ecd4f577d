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
      with_rowc<35, 70, 56, 8, 32, 4>(with_row<35, 70, 56, 8, 32, 4, 192>(make_set<35, 70, 56, 16, 24, 2>())),
      // P=4 straight tuning variants, selected with CDG_KCFG=<n> (bench sweeps;
      // DESIGN.md §6 lists what each measured)
      make_set<35, 70, 16, 16, 24, 2, 64>(),                                 // 1 CTA kernel, 8 warps
      with_row<35, 70, 16, 16, 32, 4, 0>(make_set<35, 70, 16, 16, 24, 2, 64>()),  // 2 16-node chunks
      with_row<35, 70, 16, 8, 32, 4, 1>(make_set<35, 70, 16, 16, 24, 2, 64>()),   // 3 operator ring
      with_row<35, 70, 16, 8, 32, 4, 8>(make_set<35, 70, 16, 16, 24, 2, 64>()),   // 4 U staged in smem
      with_row<35, 70, 16, 8, 32, 4, 4>(make_set<35, 70, 16, 16, 24, 2, 64>()),   // 5 res staged in smem
      with_row<35, 70, 16, 8, 32, 3, 2>(make_set<35, 70, 16, 16, 24, 2, 64>()),   // 6 U in registers, 3 CTAs
      with_rowp<35, 70, 16, 4, false>(make_set<35, 70, 16, 16, 24, 2, 64>()),     // 7 pipelined chunks
      with_row<35, 70, 16, 8, 32, 2, 0, 32>(make_set<35, 70, 16, 16, 24, 2, 64>()),  // 8 32-element tiles
      with_row<35, 70, 16, 8, 32, 4, 0>(make_set<35, 70, 16, 16, 24, 2, 64>()),       // 9 separate trace kernel
      with_row<35, 70, 16, 8, 32, 4, 32>(make_set<35, 70, 16, 16, 24, 2, 64>()),      // 10 k-steps not unrolled
      with_row<35, 70, 16, 8, 32, 4, 96>(make_set<35, 70, 16, 16, 24, 2, 64>()),      // 11 volume k-steps unrolled
      with_row<35, 70, 16, 8, 32, 4, 160>(make_set<35, 70, 16, 16, 24, 2, 64>()),     // 12 face k-steps unrolled
      with_row<35, 70, 16, 8, 32, 3, 224>(make_set<35, 70, 16, 16, 24, 2, 64>()),     // 13 unrolled, 3 CTAs/SM
      with_row<35, 70, 16, 8, 64, 4, 224>(make_set<35, 70, 16, 16, 24, 2, 64>()),     // 14 unrolled, 64-node face chunks
      with_row<35, 70, 16, 8, 32, 4, 480>(make_set<35, 70, 16, 16, 24, 2, 64>()),     // 15 both rows' res loaded up front
      with_row<35, 70, 16, 8, 32, 4, 228>(make_set<35, 70, 16, 16, 24, 2, 64>()),     // 16 res staged in smem (cp.async)
      with_row<35, 70, 16, 8, 32, 4, 224>(make_set<35, 70, 16, 16, 24, 2, 64>())};    // 17 fused-trace groups not unrolled
}

}  // namespace cdg_gpu
