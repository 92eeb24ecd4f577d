// cdg_warp.cuh -- warp-tile RHS + LSRK kernel for affine tets (p <= 4).
//
// Same math as k_rhs (cdg_kernels.cuh; reference solver.cpp:325-492), mapped
// so that ONE warp owns a tile of 16 elements from the first load to the last
// store, with no CTA-wide barriers:
//
//   rows of every contraction are (field c, element e) -> m-tile c is field c
//   of the 16 elements, so an m16n8k8 accumulator fragment of the cubature
//   GEMM holds, per lane (g = lane/4, t = lane%4), ALL FIVE conserved
//   variables of elements g and g+8 at cubature nodes 2t and 2t+1 -- four
//   complete states. The pointwise Euler flux is evaluated on those registers
//   and written straight into the A fragments of the next GEMM (the
//   accumulator layout (row, 2t | 2t+1) equals the A layout (row, k=t | t+4)
//   once logical k=t is bound to node 2t and k=t+4 to node 2t+1, which the
//   host-built B fragments follow). U_cub and the flux never touch shared
//   memory; only the nodal state U (the A operand of the first GEMM and the
//   old u of the update) is staged, per warp, with cp.async.
//
//   per 8-node cubature chunk:  U_cub = U I_cub^T          (25 DMMA, p=4)
//                               G_m = sum_d r_md F_d(U_cub) (registers)
//                               acc += G_m A_m^T            (75 DMMA)
//   per 8-node face chunk:      F* = LLF/HLLC(own trace, neighbour trace)
//                               acc -= (sjac/J) F* LIFT^T   (25 DMMA)
//   epilogue:                   res = a res + dt acc ; u += b res
//
// The FP64 DMMA and the FP64 SIMT instructions share one pipe on B200
// (microbench/fp64_mix.cu), so the kernel's job is to keep that pipe fed from
// 8 independent warps per SM: every warp has 5 x NT independent accumulator
// chains and no barrier couples it to another warp.
#pragma once

#include "cdg_kernels.cuh"

namespace cdg_gpu {

template <int NP_, int NCUB_, int NG_, int WARPS_ = 4, int MINB_ = 2>
struct WCfg {
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int EW = 16;                    // elements per warp tile
  static constexpr int WARPS = WARPS_, MINB = MINB_;
  static constexpr int BP = dev_block(NP);         // device SolutionStore block
  static constexpr int TB = dev_tblock(NF);        // device trace block
  static constexpr int KP = round_up(NP, 8);       // K of the nodal->cubature GEMM
  static constexpr int KS1 = KP / 8;
  static constexpr int NT = round_up(NP, 8) / 8;   // n-tiles of the RHS
  static constexpr int NCH = ceil_div(NCUB, 8);    // cubature chunks
  static constexpr int NFCH = ceil_div(NF, 8);     // face chunks
  static constexpr int LDU = frag_ld8(KP);         // conflict-free 128-bit A loads
  static constexpr int PANEL = 5 * EW * LDU;       // doubles per warp panel
  static constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)WARPS * (PANEL + EW * 9);
};

// Host-side fragment order shared with the kernel: for an operator Op[n][k]
// (row-major, zero outside rows x cols) the B fragment of (n-tile nt, k-step
// ks) for lane (g, t) is the pair (Op[8nt+g][8ks+2t], Op[8nt+g][8ks+2t+1]).

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // zero-fill past the last element
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

struct WarpParams {
  double* u;                  // [K*5][BP]   (updated in place when UPDATE)
  double* res;                // [K*5][BP]
  double* rhs_out;            // [K*5][BP]   (RHS-only mode)
  const double* traces;       // [(K+halo)*5][TB]
  const double* metric;       // [K][9]
  const double4* face;        // [K][4] (nx, ny, nz, sjac/J)
  const int2* conn;           // [K][4] (neighbour, packed word)
  const int* code_map;        // [n_codes][NG]
  const double2* frag1;       // [NCH][KS1][32]      I_cub
  const double2* frag2v;      // [NCH][3][NT][32]    A_m = M^-1 D_m^T W
  const double2* frag2f;      // [NFCH][NT][32]      -LIFT
  const StageCoef* coef;
  int stage;
  int K;
  int elem_offset;
  GasParams gas;
  DevError* err;
  const int* tiles;  // optional 16-element tile list (multi-GPU interior / halo split)
  int n_list;
  const unsigned long long* gate;  // optional launch gate (see gated_off)
  int gate_when;
  double* traces_out;         // fused traces of u_new (next stage), or null
  const double2* frag_ig_nat; // I_g B fragments, natural pairing [NF8/8][KS1][32]
  double* u_out;              // k_rhs_ns: the new state (u is the stage-start state)
  const double* ig;           // k_rhs_ns: I_g row-major [NF][NP]
};

template <class C, bool UPDATE, int RIEMANN>
__global__ void __launch_bounds__(32 * C::WARPS, C::MINB) k_rhs_warp(WarpParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* sU = smem + (size_t)warp * (C::PANEL + C::EW * 9);  // [5][16][LDU] rows (c, e)
  double* sMet = sU + C::PANEL;                                // [16][9]
  const double gamma = p.gas.gamma;
  const int n_tiles = (p.K + C::EW - 1) / C::EW;
  const int warps_total = gridDim.x * C::WARPS;

  const int n_iter = p.tiles ? p.n_list : n_tiles;
  for (int it_t = blockIdx.x * C::WARPS + warp; it_t < n_iter; it_t += warps_total) {
    const int tile = p.tiles ? __ldg(p.tiles + it_t) : it_t;
    if (*(volatile int*)&p.err->flag) return;  // warp-uniform: no barrier to desynchronise
    const int e0 = tile * C::EW;
    // ---- stage U (rows (c, e), natural node order) + metrics ----------------
    {
      constexpr int V = C::KP / 2;  // 16-byte pieces per row
      for (int idx = lane; idx < 5 * C::EW * V; idx += 32) {
        const int r = idx / V, j = idx - r * V;
        const int c = r / C::EW, e = r - c * C::EW;
        const bool ok = e0 + e < p.K;
        const double* src = p.u + ((size_t)(ok ? e0 + e : 0) * 5 + c) * C::BP + 2 * j;
        cp_async16(sU + r * C::LDU + 2 * j, src, ok);
      }
      for (int idx = lane; idx < C::EW * 9; idx += 32)
        sMet[idx] = (e0 + idx / 9 < p.K) ? __ldg(p.metric + (size_t)e0 * 9 + idx) : 0.0;
      // next tile of this warp -> L2 while this one computes
      const int nt_e0 = (tile + warps_total) * C::EW;
      if (!p.tiles && nt_e0 < p.K) {
        const char* base = reinterpret_cast<const char*>(p.u + (size_t)nt_e0 * 5 * C::BP);
        const int bytes = min(C::EW, p.K - nt_e0) * 5 * C::BP * 8;
        for (int off = lane * 128; off < bytes; off += 32 * 128) prefetch_l2(base + off);
      }
      cp_async_wait_all();
      __syncwarp();
    }
    const bool ev0 = e0 + g < p.K, ev1 = e0 + g + 8 < p.K;

    double acc[5][C::NT][4];
#pragma unroll
    for (int c = 0; c < 5; ++c)
#pragma unroll
      for (int n = 0; n < C::NT; ++n) acc[c][n][0] = acc[c][n][1] = acc[c][n][2] = acc[c][n][3] = 0.0;

    // ---- volume ------------------------------------------------------------
#pragma unroll 1
    for (int ch = 0; ch < C::NCH; ++ch) {
      double uc[5][4];
#pragma unroll
      for (int c = 0; c < 5; ++c) uc[c][0] = uc[c][1] = uc[c][2] = uc[c][3] = 0.0;
#pragma unroll 1
      for (int ks = 0; ks < C::KS1; ++ks) {
        const double2 b = __ldg(p.frag1 + ((size_t)ch * C::KS1 + ks) * 32 + lane);
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const double* s = sU + (c * C::EW + g) * C::LDU + ks * 8 + 2 * t;
          const double2 x = *reinterpret_cast<const double2*>(s);
          const double2 y = *reinterpret_cast<const double2*>(s + 8 * C::LDU);
          dmma_k8(uc[c], x.x, y.x, x.y, y.y, b.x, b.y);
        }
      }
      // points j: 0 (g, 2t) 1 (g, 2t+1) 2 (g+8, 2t) 3 (g+8, 2t+1)
      const int q = ch * 8 + 2 * t;
      const bool vq0 = q < C::NCUB, vq1 = q + 1 < C::NCUB;
      const bool valid[4] = {ev0 && vq0, ev0 && vq1, ev1 && vq0, ev1 && vq1};
      double ir[4], pr[4], vx[4], vy[4], vz[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const State5 s{uc[0][j], uc[1][j], uc[2][j], uc[3][j], uc[4][j]};
        if (valid[j] && !admissible(s, gamma))
          record_error(p.err, 1, p.elem_offset + e0 + g + 8 * (j >> 1), q + (j & 1), 0, s.r);
        const double rr = valid[j] ? s.r : 1.0;
        ir[j] = 1.0 / rr;
        pr[j] = valid[j] ? (gamma - 1.0) * (s.E - 0.5 * ir[j] * (s.mx * s.mx + s.my * s.my + s.mz * s.mz)) : 0.0;
        vx[j] = s.mx * ir[j];
        vy[j] = s.my * ir[j];
        vz[j] = s.mz * ir[j];
        uc[4][j] += pr[j];  // E + p (the energy flux factor)
      }
#pragma unroll 1
      for (int m = 0; m < 3; ++m) {
        double2 b[C::NT];
#pragma unroll
        for (int n = 0; n < C::NT; ++n) b[n] = __ldg(p.frag2v + (((size_t)ch * 3 + m) * C::NT + n) * 32 + lane);
        const double* m0 = sMet + g * 9 + m * 3;
        const double* m1 = sMet + (g + 8) * 9 + m * 3;
        const double r00 = m0[0], r01 = m0[1], r02 = m0[2], r10 = m1[0], r11 = m1[1], r12 = m1[2];
        // contravariant velocity U_m = sum_d r_md v_d  and  G_m = sum_d r_md F_d
        //   = (rho U_m, m U_m + p r_m, (E + p) U_m)     (solver.cpp:382-394 x S_m)
        double um[4], rm[4][3];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double a0 = j < 2 ? r00 : r10, a1 = j < 2 ? r01 : r11, a2 = j < 2 ? r02 : r12;
          rm[j][0] = a0;
          rm[j][1] = a1;
          rm[j][2] = a2;
          um[j] = valid[j] ? a0 * vx[j] + a1 * vy[j] + a2 * vz[j] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double gv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (c == 0) gv[j] = uc[0][j] * um[j];
            else if (c == 4) gv[j] = uc[4][j] * um[j];
            else gv[j] = uc[c][j] * um[j] + pr[j] * rm[j][c - 1];
          }
          // A fragment: a0 (g, k=t)=j0, a1 (g+8, t)=j2, a2 (g, t+4)=j1, a3 (g+8, t+4)=j3
#pragma unroll
          for (int n = 0; n < C::NT; ++n) dmma_k8(acc[c][n], gv[0], gv[2], gv[1], gv[3], b[n].x, b[n].y);
        }
      }
    }

    // ---- surface: chunks of 8 face nodes -------------------------------------
#pragma unroll 1
    for (int fc = 0; fc < C::NFCH; ++fc) {
      double2 b[C::NT];
#pragma unroll
      for (int n = 0; n < C::NT; ++n) b[n] = __ldg(p.frag2f + ((size_t)fc * C::NT + n) * 32 + lane);
      double fl[4][5];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = g + 8 * (j >> 1), fq = fc * 8 + 2 * t + (j & 1);
        const int eg = e0 + e;
        if (eg >= p.K || fq >= C::NF) {
#pragma unroll
          for (int c = 0; c < 5; ++c) fl[j][c] = 0.0;
          continue;
        }
        const int f = fq / C::NG, gq = fq - f * C::NG;
        const double* tm = p.traces + (size_t)eg * 5 * C::TB + fq;
        const State5 um{tm[0], tm[C::TB], tm[2 * C::TB], tm[3 * C::TB], tm[4 * C::TB]};
        const double4 fn = p.face[(size_t)eg * 4 + f];
        const int2 cw = __ldg(p.conn + (size_t)eg * 4 + f);
        State5 up;
        if (cw.x >= 0) {
          const int h = __ldg(p.code_map + (cw.y >> 8) * C::NG + gq);
          const double* tp = p.traces + (size_t)cw.x * 5 * C::TB + (cw.y & 3) * C::NG + h;
          up = State5{tp[0], tp[C::TB], tp[2 * C::TB], tp[3 * C::TB], tp[4 * C::TB]};
        } else {
          up = boundary_state(um, fn.x, fn.y, fn.z, (cw.y >> 2) & 3, p.gas);
        }
        if (!admissible(um, gamma) || !admissible(up, gamma)) {
          record_error(p.err, 2, p.elem_offset + eg, f, gq, um.r);
#pragma unroll
          for (int c = 0; c < 5; ++c) fl[j][c] = 0.0;
          continue;
        }
        double fs[5];
        if (RIEMANN == 1)
          hllc_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs, p.gas.hllc_fallbacks);
        else
          llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
#pragma unroll
        for (int c = 0; c < 5; ++c) fl[j][c] = fn.w * fs[c];
      }
#pragma unroll
      for (int c = 0; c < 5; ++c)
#pragma unroll
        for (int n = 0; n < C::NT; ++n) dmma_k8(acc[c][n], fl[0][c], fl[2][c], fl[1][c], fl[3][c], b[n].x, b[n].y);
    }

    // ---- epilogue: rhs -> (res, u) update or rhs store -----------------------
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int e = g + 8 * hh, eg = e0 + e;
      if (eg >= p.K) continue;
      if (__ldg(reinterpret_cast<const int*>(p.conn + (size_t)eg * 4) + 1) & kCurvedBit) continue;  // k_rhs_curved
      // the element's old res values are loaded before any of its stores (loads
      // of p.res cannot be moved above stores to p.u / p.res by the compiler)
      double2 rsv[5][C::NT];
      if (UPDATE)
#pragma unroll
        for (int c = 0; c < 5; ++c)
#pragma unroll
          for (int n = 0; n < C::NT; ++n)
            rsv[c][n] = *reinterpret_cast<const double2*>(p.res + ((size_t)eg * 5 + c) * C::BP + n * 8 + 2 * t);
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const size_t rowoff = ((size_t)eg * 5 + c) * C::BP;
#pragma unroll
        for (int n = 0; n < C::NT; ++n) {
          const int col = n * 8 + 2 * t;  // < NT*8 <= BP; padded columns carry exact zeros
          const double r0 = acc[c][n][2 * hh], r1 = acc[c][n][2 * hh + 1];
          if (UPDATE) {
            const double2 rs = rsv[c][n];
            const double n0 = a_c * rs.x + dt * r0, n1 = a_c * rs.y + dt * r1;
            *reinterpret_cast<double2*>(p.res + rowoff + col) = make_double2(n0, n1);
            const double2 uo = *reinterpret_cast<const double2*>(sU + (c * C::EW + e) * C::LDU + col);
            const double w0 = uo.x + b_c * n0, w1 = uo.y + b_c * n1;
            *reinterpret_cast<double2*>(p.u + rowoff + col) = make_double2(w0, w1);
            acc[c][n][2 * hh] = w0;  // u_new in the accumulator (= natural-pairing A fragment) layout
            acc[c][n][2 * hh + 1] = w1;
          } else {
            *reinterpret_cast<double2*>(p.rhs_out + rowoff + col) = make_double2(r0, r1);
          }
        }
      }
    }
    if (UPDATE && p.traces_out) {
      // next stage's traces T = u_new I_g^T (solver.cpp:200-208) from the
      // registers, field by field; the trace kernel's pairing and fragments
      // (k_interp<NAT>), so fused and separate traces agree bit for bit
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int eg = e0 + g + 8 * hh;
        const bool skip = eg >= p.K || (__ldg(reinterpret_cast<const int*>(p.conn + (size_t)min(eg, p.K - 1) * 4) + 1) &
                                        kCurvedBit);
        if (skip)
#pragma unroll
          for (int c = 0; c < 5; ++c)
#pragma unroll
            for (int n = 0; n < C::NT; ++n) acc[c][n][2 * hh] = acc[c][n][2 * hh + 1] = 0.0;
      }
      constexpr int NFT = round_up(C::NF, 8) / 8;
#pragma unroll
      for (int c = 0; c < 5; ++c) {
#pragma unroll
        for (int nt = 0; nt < NFT; ++nt) {
          double tacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int ks = 0; ks < C::NT; ++ks)
            mma_frag(tacc, AFrag{acc[c][ks][0], acc[c][ks][2], acc[c][ks][1], acc[c][ks][3]},
                     __ldg(p.frag_ig_nat + ((size_t)nt * C::NT + ks) * 32 + lane));
          const int col = nt * 8 + 2 * t;
          if (col < C::NF) {
            const int e_lo = e0 + g, e_hi = e_lo + 8;
            if (e_lo < p.K)
              *reinterpret_cast<double2*>(p.traces_out + ((size_t)e_lo * 5 + c) * C::TB + col) = make_double2(tacc[0], tacc[1]);
            if (e_hi < p.K)
              *reinterpret_cast<double2*>(p.traces_out + ((size_t)e_hi * 5 + c) * C::TB + col) = make_double2(tacc[2], tacc[3]);
          }
        }
      }
    }
    __syncwarp();  // the panel is restaged next iteration
  }
}

}  // namespace cdg_gpu
