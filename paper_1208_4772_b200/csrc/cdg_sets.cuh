// cdg_sets.cuh -- kernel-set table types: one KernelSet per (N_p, N_cub, N_g)
// level shape, holding the instantiated sm_100a kernels. The instantiations
// are spread over several translation units (sets_*.cu) so that nvcc builds
// them in parallel.
#pragma once

#include <vector>

#include "cdg_aux.cuh"
#include "cdg_curved.cuh"
#include "cdg_kernels.cuh"
#include "cdg_ns.cuh"
#include "cdg_row.cuh"
#include "cdg_rowc.cuh"
#include "cdg_wa.cuh"
#include "cdg_wac.cuh"
#include "cdg_warp.cuh"

namespace cdg_gpu {

struct KernelSet {
  int np, ncub, ng, E, minb, ch, nth;
  size_t smem_traces, smem_rhs, smem_aux;
  void (*traces)(const double*, double*, const double*, int, int, const unsigned long long*, int);
  void (*cubinterp)(const double*, double*, const double*, int, int, const unsigned long long*, int);
  void (*qn_traces)(const double*, size_t, double*, const double*, const double4*, const double4*, const int*, int, int,
                    const unsigned long long*, int);
  size_t smem_qn = 0;
  int qn_rows = 16;  // rows per CTA pass of qn_traces
  void (*rhs_update)(RhsParams);
  void (*rhs_only)(RhsParams);
  void (*aux_q)(AuxParams);
  void (*visc_rhs_update)(RhsParams);
  void (*visc_rhs_only)(RhsParams);
  void (*curved_update)(CurvedParams);
  void (*curved_only)(CurvedParams);
  void (*curved_visc_update)(CurvedParams);
  void (*curved_visc_only)(CurvedParams);
  void (*aux_curved)(CurvedParams);
  size_t smem_curved;
  // warp-tile inviscid kernel (cdg_warp.cuh), p <= 3
  void (*warp_update[2])(WarpParams) = {nullptr, nullptr};  // [riemann]
  void (*warp_only[2])(WarpParams) = {nullptr, nullptr};
  size_t smem_warp = 0;
  int warp_warps = 0, warp_minb = 0;
  // neighbour-state kernel (cdg_ns.cuh): affine levels, no stored traces, p <= 2
  void (*ns_update[2])(WarpParams) = {nullptr, nullptr};  // [riemann]
  size_t smem_ns = 0;
  int ns_warps = 0, ns_minb = 0;
  // row-per-warp inviscid kernel (cdg_row.cuh), p = 4
  void (*row_update[2])(RhsParams) = {nullptr, nullptr};  // [riemann]
  void (*row_only[2])(RhsParams) = {nullptr, nullptr};
  size_t smem_row = 0;
  int row_minb = 0, row_ch = 0, row_e = 16, row_nth = 160;
  bool row_ft = false;  // row kernel writes the next stage's traces (MODE 32)
  const char* row_name = "k_rhs_row";  // the kernel in the row slots
  // row-per-warp inviscid kernel for curved elements (cdg_rowc.cuh)
  void (*rowc_update[2])(CurvedParams) = {nullptr, nullptr};  // [riemann]
  void (*rowc_only[2])(CurvedParams) = {nullptr, nullptr};
  void (*rowc_visc_update[2])(CurvedParams) = {nullptr, nullptr};
  void (*rowc_visc_only[2])(CurvedParams) = {nullptr, nullptr};
  void (*rowc_aux)(CurvedParams) = nullptr;
  size_t smem_rowc = 0, smem_rowc_aux = 0;
  int rowc_aux_minb = 0, rowc_aux_e = 16, rowc_aux_nth = 160;
  const char* rowc_name = "k_rhs_rowc";
  bool rowc_ft = false;  // the curved update kernel writes the next stage's traces (k_rhs_wac)
  int rowc_minb = 0, rowc_ch = 0, rowc_e = 16, rowc_nth = 160;
};

template <int NP, int NCUB, int NG, int CH = 8, int FCH = 32, int MINB = 3, int MODE = 0, int E = 16>
KernelSet with_rowc(KernelSet k) {
  using RC = RCfg<NP, NCUB, NG, CH, FCH, MINB, MODE, E>;
  k.rowc_update[0] = &k_rhs_rowc<RC, true, 0>;
  k.rowc_update[1] = &k_rhs_rowc<RC, true, 1>;
  k.rowc_only[0] = &k_rhs_rowc<RC, false, 0>;
  k.rowc_only[1] = &k_rhs_rowc<RC, false, 1>;
  k.rowc_visc_update[0] = &k_rhs_rowc<RC, true, 0, 1>;
  k.rowc_visc_update[1] = &k_rhs_rowc<RC, true, 1, 1>;
  k.rowc_visc_only[0] = &k_rhs_rowc<RC, false, 0, 1>;
  k.rowc_visc_only[1] = &k_rhs_rowc<RC, false, 1, 1>;
  // aux gradient: the three directions in one pass (3 accumulator sets, 3x the
  // panels) at 2 CTAs/SM
  using RCA = RCfg<NP, NCUB, NG, CH, FCH, 2, MODE, E>;
  k.rowc_aux = &k_rhs_rowc<RCA, false, 0, 2>;
  k.smem_rowc_aux = RowCurvedLayout<RCA, 3>::SMEM_BYTES;
  k.rowc_aux_minb = 2;
  k.rowc_aux_e = RCA::E;
  k.rowc_aux_nth = RCA::NTH;
  k.smem_rowc = RowCurvedLayout<RC>::SMEM_BYTES;
  k.rowc_minb = MINB;
  k.rowc_ch = CH;
  k.rowc_e = RC::E;
  k.rowc_nth = RC::NTH;
  return k;
}

template <int NP, int NCUB, int NG, int CH = 8, int FCH = 32, int MINB = 3, int MODE = 7, int E = 16>
KernelSet with_row(KernelSet k) {
  using RC = RCfg<NP, NCUB, NG, CH, FCH, MINB, MODE, E>;
  k.row_update[0] = &k_rhs_row<RC, true, 0>;
  k.row_update[1] = &k_rhs_row<RC, true, 1>;
  k.row_only[0] = &k_rhs_row<RC, false, 0>;
  k.row_only[1] = &k_rhs_row<RC, false, 1>;
  k.smem_row = RC::SMEM_BYTES;
  k.row_minb = MINB;
  k.row_ch = CH;
  k.row_e = RC::E;
  k.row_nth = RC::NTH;
  k.row_ft = RC::FT;
  return k;
}

// warp-autonomous curved kernel (cdg_wac.cuh) in the curved RHS slots (apply
// after with_rowc: the aux gradient stays on k_rhs_rowc)
template <int NP, int NCUB, int NG, int CH = 8, int FCH = 32, int WARPS = 16, int MINB = 1>
KernelSet with_wac(KernelSet k) {
  using WC = WacCfg<NP, NCUB, NG, CH, FCH, WARPS, MINB>;
  k.rowc_update[0] = &k_rhs_wac<WC, true, 0>;
  k.rowc_update[1] = &k_rhs_wac<WC, true, 1>;
  k.rowc_only[0] = &k_rhs_wac<WC, false, 0>;
  k.rowc_only[1] = &k_rhs_wac<WC, false, 1>;
  k.rowc_visc_update[0] = &k_rhs_wac<WC, true, 0, 1>;
  k.rowc_visc_update[1] = &k_rhs_wac<WC, true, 1, 1>;
  k.rowc_visc_only[0] = &k_rhs_wac<WC, false, 0, 1>;
  k.rowc_visc_only[1] = &k_rhs_wac<WC, false, 1, 1>;
  k.smem_rowc = WC::SMEM_BYTES;
  k.rowc_minb = MINB;
  k.rowc_e = WC::E;
  k.rowc_nth = WC::NTH;
  k.rowc_name = "k_rhs_wac";
  k.rowc_ft = WC::FT;
  return k;
}

// the aux gradient (three directions, one pass) on the warp-autonomous curved
// mapping: AWARPS warps x 1 CTA per SM
template <int NP, int NCUB, int NG, int CH = 8, int FCH = 32, int AWARPS = 8>
KernelSet with_wac_aux(KernelSet k) {
  using WA = WacCfg<NP, NCUB, NG, CH, FCH, AWARPS, 1, 3>;
  k.rowc_aux = &k_rhs_wac<WA, false, 0, 2>;
  k.smem_rowc_aux = WA::SMEM_BYTES;
  k.rowc_aux_minb = 1;
  k.rowc_aux_e = WA::E;
  k.rowc_aux_nth = WA::NTH;
  return k;
}

// warp-autonomous affine kernel (cdg_wa.cuh) in the row kernel's slots: same
// operator fragments (natural pairing, CH-node chunks), fused traces; a CTA
// "tile" is 3 elements per warp
template <int NP, int NCUB, int NG, int CH = 8, int FCH = 32, int WARPS = 5, int MINB = 4, bool UREG = false,
          bool FT = true>
KernelSet with_wa(KernelSet k) {
  using WC = WaCfg<NP, NCUB, NG, CH, FCH, WARPS, MINB, UREG, FT>;
  k.row_update[0] = &k_rhs_wa<WC, true, 0>;
  k.row_update[1] = &k_rhs_wa<WC, true, 1>;
  k.row_only[0] = &k_rhs_wa<WC, false, 0>;
  k.row_only[1] = &k_rhs_wa<WC, false, 1>;
  k.smem_row = WC::SMEM_BYTES;
  k.row_minb = MINB;
  k.row_ch = CH;
  k.row_e = WC::E;
  k.row_nth = WC::NTH;
  k.row_ft = FT;
  k.row_name = "k_rhs_wa";
  return k;
}

template <int NP, int NCUB, int NG, int WARPS = 4, int MINB = 2>
KernelSet with_warp(KernelSet k) {
  using W = WCfg<NP, NCUB, NG, WARPS, MINB>;
  k.warp_update[0] = &k_rhs_warp<W, true, 0>;
  k.warp_update[1] = &k_rhs_warp<W, true, 1>;
  k.warp_only[0] = &k_rhs_warp<W, false, 0>;
  k.warp_only[1] = &k_rhs_warp<W, false, 1>;
  k.smem_warp = W::SMEM_BYTES;
  k.warp_warps = WARPS;
  k.warp_minb = MINB;
  return k;
}

template <int NP, int NCUB, int NG, int WARPS = 4, int MINB = 4>
KernelSet with_ns(KernelSet k) {
  using N = NsCfg<NP, NCUB, NG, WARPS, MINB>;
  k.ns_update[0] = &k_rhs_ns<N, 0>;
  k.ns_update[1] = &k_rhs_ns<N, 1>;
  k.smem_ns = N::SMEM_BYTES;
  k.ns_warps = WARPS;
  k.ns_minb = MINB;
  return k;
}

// <N_p, N_cub, N_g, E elements/tile, CH cubature chunk, CTAs/SM, FCH face
// chunk, NW warps/CTA of k_rhs>. The aux-gradient and curved kernels always
// run with 8 warps on the same tile shape (same host operator layout).
template <int NP, int NCUB, int NG, int E, int CH = 16, int MINB = 1, int FCH = 32, int NW = 8>
KernelSet make_set() {
  using C = Cfg<NP, NCUB, NG, E, CH, MINB, FCH, NW>;
  using C8 = Cfg<NP, NCUB, NG, E, CH, (NW == 8 ? MINB : 1), FCH, 8>;
  KernelSet k;
  k.np = NP;
  k.ncub = NCUB;
  k.ng = NG;
  k.E = E;
  k.minb = MINB;
  k.ch = CH;
  k.nth = C::NTH;
  k.smem_traces = sizeof(double) * C8::R * C8::LDU;
  k.smem_rhs = C::SMEM_BYTES;
  k.smem_aux = C8::SMEM_BYTES;
  k.traces = &k_interp<C8, C8::NF, C8::TB, true>;
  k.cubinterp = &k_interp<C8, C8::NCUB, round_up(NCUB, 8)>;
  k.qn_traces = &k_qn_traces<C8>;
  k.smem_qn = sizeof(double) * 3 * qn_block_rows<C8>() * C8::LDU;
  k.qn_rows = qn_block_rows<C8>();
  k.rhs_update = &k_rhs<C, true, false>;
  k.rhs_only = &k_rhs<C, false, false>;
  k.aux_q = &k_aux_q<C8>;
  k.visc_rhs_update = &k_rhs<C, true, true>;
  k.visc_rhs_only = &k_rhs<C, false, true>;
  k.curved_update = &k_rhs_curved<C8, true>;
  k.curved_only = &k_rhs_curved<C8, false>;
  k.curved_visc_update = &k_rhs_curved<C8, true, true>;
  k.curved_visc_only = &k_rhs_curved<C8, false, true>;
  k.aux_curved = &k_aux_curved<C8>;
  k.smem_curved = CurvedLayout<C8>::SMEM_BYTES;
  return k;
}

// one function per translation unit (sets_*.cu)
std::vector<KernelSet> kernel_sets_p1_3();
std::vector<KernelSet> kernel_sets_p4();
std::vector<KernelSet> kernel_sets_p5_6();
std::vector<KernelSet> kernel_sets_p7_8();

}  // namespace cdg_gpu
