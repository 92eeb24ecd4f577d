// cdg_wa.cuh -- warp-autonomous RHS + LSRK kernel for affine tets: the math,
// operators (natural-pairing B fragments of the row kernel) and per-element
// evaluation order of k_rhs_row (cdg_row.cuh; reference solver.cpp:325-492),
// with NO CTA barrier.
//
// In k_rhs_row a 16-element tile is 80 (element, field) rows over 5 warps, so
// an element's 5 rows straddle warps and every cubature / face chunk needs
// two CTA barriers (U_cub ready, flux ready): the warps wait for the slowest
// one, 30-44% of the GEMM phases' stall samples (profiles/r2/ncu_k_rhs_row.txt).
// Here each warp owns THREE whole elements: its m16 tile is their 15 rows
// (element-major, field-minor, contiguous in the SolutionStore) plus one
// padding row, so GEMM1 -> pointwise flux -> GEMM2 and face flux -> face
// GEMM -> epilogue (+ fused next-stage traces) only exchange data within the
// warp (warp-private shared panels, __syncwarp). Warps never wait for each
// other; 1/16 of the MMA work is the padding row. A CTA of W warps covers
// 3W consecutive elements (the "tile" of the host's tile lists).
#pragma once

#include "cdg_row.cuh"

#ifndef CDG_WA_FUNROLL
#define CDG_WA_FUNROLL 1
#endif
#ifndef CDG_WA_ASTAGE
#define CDG_WA_ASTAGE 1  // HLLC: the tile's metrics / face geometry / connectivity by cp.async, waited after the first GEMM1
#endif
#ifndef CDG_WA_RES2
#define CDG_WA_RES2 1  // LLF, p <= 4: both rows' old res values loaded before the first store (+0.5% at P=4)
#endif

namespace cdg_gpu {

template <int NP_, int NCUB_, int NG_, int CH_ = 8, int FCH_ = 32, int WARPS_ = 5, int MINB_ = 4, bool UREG_ = false,
          bool FT_ = true>
struct WaCfg {
  static constexpr bool FT = FT_;  // the epilogue writes the next stage's traces (else the trace kernel does)
  static constexpr bool UREG = UREG_;  // U fragments kept in registers for the whole tile (else reloaded per chunk)
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int EPW = 3, WARPS = WARPS_, E = EPW * WARPS_, NTH = 32 * WARPS_, MINB = MINB_;
  static constexpr int BP = dev_block(NP), TB = dev_tblock(NF);
  static constexpr int KP = round_up(NP, 8), KS1 = KP / 8, NT2 = KS1;
  static constexpr int NCUB8 = round_up(NCUB, 8), NF8 = round_up(NF, 8);
  static constexpr int CH = CH_, NCH = ceil_div(NCUB8, CH);
  static constexpr int FCH = FCH_, NFCH = ceil_div(NF, FCH);
  static constexpr int K2CUB = 3 * NCUB8, K2 = K2CUB + NF8;
  static constexpr int LDC = frag_ld8(CH), LDG = frag_ld8(3 * CH), LDF = frag_ld8(FCH);
  static constexpr int VOLW = 16 * LDC + 16 * LDG, FACEW = 16 * LDF;
  static constexpr int WORKW = VOLW > FACEW ? VOLW : FACEW;  // doubles per warp (phases alias)
  // per warp: [face table (double4, 32-byte aligned) | work panels | metric | conn],
  // a multiple of 4 doubles so every warp's base stays 32-byte aligned
  static constexpr int PERW = round_up(EPW * 4 * 4 + WORKW + EPW * 9 + EPW * 4, 4);
  static constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)PERW * WARPS_;
  static constexpr int IT_P = ceil_div(EPW * CH, 32), IT_F = ceil_div(EPW * FCH, 32);
  static constexpr int FUNROLL = CDG_WA_FUNROLL;  // face-item loop unroll (tuning)
};

template <class C, bool UPDATE, int RM>
__global__ void __launch_bounds__(C::NTH, C::MINB) k_rhs_wa(RhsParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  double* base = smem + (size_t)warp * C::PERW;
  double4* sFace = reinterpret_cast<double4*>(base);               // [3][4]
  double* sWork = base + C::EPW * 4 * 4;                           // [16][LDC] + [16][LDG] | [16][LDF]
  double* sC = sWork;
  double* sG = sWork + 16 * C::LDC;
  double* sF = sWork;
  double* sMet = sWork + C::WORKW;                                 // [3][9]
  int2* sConn = reinterpret_cast<int2*>(sMet + C::EPW * 9);        // [3][4]
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const int n_tiles = (p.K + C::E - 1) / C::E;
  const int n_iter = p.tiles ? p.n_list : n_tiles;
  const double2* fb1all = reinterpret_cast<const double2*>(p.frag_icub);  // [NCUB8/8][KS1][32]
  const double2* fb2all = reinterpret_cast<const double2*>(p.frag_op2);   // [K2/8][NT2][32]

  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = tile_at(p, it_t);
    const int e0 = tile * C::E + warp * C::EPW;  // this warp's three elements
    if (e0 >= p.K) continue;                      // warp-uniform
    // warp-uniform early exit after a recorded error
    if (__shfl_sync(0xffffffffu, lane == 0 ? *(volatile int*)&p.err->flag : 0, 0)) return;
    const int row0 = e0 * 5;
    // row r of the m-tile: element e0 + r/5, field r%5 (r = 15: padding)
    const int r_lo = row0 + g, r_hi = r_lo + 8;
    const bool ok_lo = r_lo < n_rows, ok_hi = (g + 8 < 15) && r_hi < n_rows;
    constexpr bool AST = CDG_WA_ASTAGE && RM == 1;  // measured: HLLC +1.4%, LLF -0.5%
    if (AST) {  // in flight during the first chunk's GEMM1
      for (int idx = lane; idx < C::EPW * 9; idx += 32) {
        if (e0 + idx / 9 < p.K)
          cp_async8_sh(sMet + idx, p.metric + (size_t)e0 * 9 + idx);
        else
          sMet[idx] = 0.0;
      }
      for (int idx = lane; idx < C::EPW * 8; idx += 32) {  // 16-byte halves of the double4s
        if (e0 + idx / 8 < p.K)
          cp_async16_sh(reinterpret_cast<double*>(sFace) + 2 * idx, reinterpret_cast<const double*>(p.face + (size_t)e0 * 4) + 2 * idx);
        else
          reinterpret_cast<double2*>(sFace)[idx] = (idx & 1) ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0);
      }
      for (int idx = lane; idx < C::EPW * 4; idx += 32) {
        if (e0 + idx / 4 < p.K)
          cp_async8_sh(sConn + idx, p.conn + (size_t)e0 * 4 + idx);
        else
          sConn[idx] = make_int2(-1, pack_face(0, 0, 1, 0));
      }
    } else {
      for (int idx = lane; idx < C::EPW * 9; idx += 32)
        sMet[idx] = e0 + idx / 9 < p.K ? __ldg(p.metric + (size_t)e0 * 9 + idx) : 0.0;
      for (int idx = lane; idx < C::EPW * 4; idx += 32) {
        const bool ok = e0 + idx / 4 < p.K;
        sFace[idx] = ok ? p.face[(size_t)e0 * 4 + idx] : make_double4(0, 0, 1, 0);
        sConn[idx] = ok ? p.conn[(size_t)e0 * 4 + idx] : make_int2(-1, pack_face(0, 0, 1, 0));
      }
      __syncwarp();
    }

    const double* u_lo = p.u + (size_t)min(r_lo, n_rows - 1) * C::BP + 2 * tq;
    const double* u_hi = p.u + (size_t)min(r_hi, n_rows - 1) * C::BP + 2 * tq;
    double uA[C::KS1][4];
    auto load_u = [&]() {
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) {
        double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
        if (ok_lo) x = *reinterpret_cast<const double2*>(u_lo + ks * 8);
        if (ok_hi) y = *reinterpret_cast<const double2*>(u_hi + ks * 8);
        uA[ks][0] = x.x, uA[ks][1] = y.x, uA[ks][2] = x.y, uA[ks][3] = y.y;
      }
    };
    double acc[C::NT2][4];
#pragma unroll
    for (int i = 0; i < C::NT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
    auto contract = [&](const double* panel, int ld, int nks, int nks_full, const double2* fb2) {
      auto kstep = [&](int ks) {
        const AFrag a = load_afrag(panel, ld, 0, ks * 8, g, tq);
#pragma unroll
        for (int nt = 0; nt < C::NT2; ++nt) mma_frag(acc[nt], a, __ldg(fb2 + (ks * C::NT2 + nt) * 32 + lane));
      };
      if (nks == nks_full) {
#pragma unroll
        for (int ks = 0; ks < nks_full; ++ks) kstep(ks);
      } else {
#pragma unroll 1
        for (int ks = 0; ks < nks; ++ks) kstep(ks);
      }
    };

    // ---- volume: chunks of CH cubature nodes --------------------------------
    if (C::UREG) load_u();
#pragma unroll 1
    for (int ch = 0; ch < C::NCH; ++ch) {
      const int q0 = ch * C::CH;
      const int w = min(C::CH, C::NCUB8 - q0);
      const double2* fb1 = fb1all + (size_t)(q0 / 8) * C::KS1 * 32;
      if (!C::UREG) load_u();
      {  // GEMM1: U_cub of the warp's rows at the chunk's nodes
        double c1[C::CH / 8][4];
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j) c1[j][0] = c1[j][1] = c1[j][2] = c1[j][3] = 0.0;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks)
#pragma unroll
          for (int j = 0; j < C::CH / 8; ++j)
            if (j * 8 < w) {
              const double2 b = __ldg(fb1 + (j * C::KS1 + ks) * 32 + lane);
              dmma_k8(c1[j], uA[ks][0], uA[ks][1], uA[ks][2], uA[ks][3], b.x, b.y);
            }
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j)
          if (j * 8 < w) {
            double* o = sC + g * C::LDC + j * 8 + 2 * tq;
            *reinterpret_cast<double2*>(o) = make_double2(c1[j][0], c1[j][1]);
            *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c1[j][2], c1[j][3]);
          }
      }
      if (AST && ch == 0) cp_async_wait0();  // the tile's staged metrics / faces / connectivity
      __syncwarp();
      // pointwise Euler flux -> contravariant flux G_m = sum_d (dr_m/dx_d) F_d
#pragma unroll
      for (int it = 0; it < C::IT_P; ++it) {
        const int idx = lane + it * 32;
        if (idx < C::EPW * w) {
          const int e = idx / w, ql = idx - e * w, q = q0 + ql;
          const double* uc = sC + (e * 5) * C::LDC + ql;
          double* gout = sG + (e * 5) * C::LDG + ql;
          if (q < C::NCUB && e0 + e < p.K) {
            const State5 s{uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
            if (!admissible(s, gamma)) record_error(p.err, 1, p.elem_offset + e0 + e, q, 0, s.r);
            const double ir = 1.0 / s.r;
            const double pr = (gamma - 1.0) * (s.E - 0.5 * ir * (s.mx * s.mx + s.my * s.my + s.mz * s.mz));
            const double vx = s.mx * ir, vy = s.my * ir, vz = s.mz * ir;
            const double ep = s.E + pr;
            const double* met = sMet + e * 9;
            // G_m = (rho U_m, m U_m + p r_m, (E+p) U_m), U_m = sum_d r_md v_d
            // (solver.cpp:382-394 contracted with S_m, operators.cpp:139-147)
#pragma unroll
            for (int m = 0; m < 3; ++m) {
              const double r0 = met[m * 3 + 0], r1 = met[m * 3 + 1], r2 = met[m * 3 + 2];
              const double um = r0 * vx + r1 * vy + r2 * vz;
              double* o = gout + m * w;
              o[0] = s.r * um;
              o[C::LDG] = s.mx * um + pr * r0;
              o[2 * C::LDG] = s.my * um + pr * r1;
              o[3 * C::LDG] = s.mz * um + pr * r2;
              o[4 * C::LDG] = ep * um;
            }
          } else {
#pragma unroll
            for (int m = 0; m < 3; ++m)
#pragma unroll
              for (int c = 0; c < 5; ++c) gout[m * w + c * C::LDG] = 0.0;
          }
        }
      }
      if (lane < 3 * w) sG[15 * C::LDG + lane] = 0.0;  // the padding row
      __syncwarp();
      contract(sG, C::LDG, (3 * w) / 8, 3 * C::CH / 8, fb2all + (size_t)(3 * q0 / 8) * C::NT2 * 32);
      __syncwarp();  // sC / sG are rewritten by the next chunk
    }

    // ---- surface: chunks of FCH face nodes ------------------------------------
#pragma unroll 1
    for (int fc = 0; fc < C::NFCH; ++fc) {
      const int f0 = fc * C::FCH;
      const int wr = min(C::FCH, C::NF - f0), wp = round_up(wr, 8);
#pragma unroll C::FUNROLL
      for (int it = 0; it < C::IT_F; ++it) {
        const int idx = lane + it * 32;
        if (idx >= C::EPW * wp) break;
        const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
        double* gout = sF + (e * 5) * C::LDF + fl;
        const int eg = e0 + e;
        if (eg >= p.K || fl >= wr) {
#pragma unroll
          for (int c = 0; c < 5; ++c) gout[c * C::LDF] = 0.0;
          continue;
        }
        const int f = fq / C::NG, gq = fq - f * C::NG;
        const double* tm = p.traces + (size_t)eg * 5 * C::TB + fq;
        const State5 um{tm[0], tm[C::TB], tm[2 * C::TB], tm[3 * C::TB], tm[4 * C::TB]};
        const double4 fn = sFace[e * 4 + f];
        const int2 cw = sConn[e * 4 + f];
        State5 up;
        if (cw.x >= 0) {
          const int h = __ldg(p.code_map + (cw.y >> 8) * C::NG + gq);
          const double* tp = p.traces + (size_t)cw.x * 5 * C::TB + (cw.y & 3) * C::NG + h;
          up = State5{tp[0], tp[C::TB], tp[2 * C::TB], tp[3 * C::TB], tp[4 * C::TB]};
        } else {
          up = boundary_state(um, fn.x, fn.y, fn.z, (cw.y >> 2) & 3, p.gas);
        }
        if (!admissible(um, gamma) || !admissible(up, gamma)) record_error(p.err, 2, p.elem_offset + eg, f, gq, um.r);
        double fs[5];
        if (RM == 1)
          hllc_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs, p.gas.hllc_fallbacks);
        else
          llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
#pragma unroll
        for (int c = 0; c < 5; ++c) gout[c * C::LDF] = fn.w * fs[c];
      }
      if (lane < wp) sF[15 * C::LDF + lane] = 0.0;  // the padding row
      __syncwarp();
      contract(sF, C::LDF, wp / 8, C::FCH / 8, fb2all + (size_t)((C::K2CUB + f0) / 8) * C::NT2 * 32);
      __syncwarp();
    }

    // ---- epilogue: rhs -> (res, u) update or rhs store (+ next-stage traces) --
    if (!C::UREG) load_u();  // old u (the A fragment of k-step j holds (row, 8j+2t), (row, 8j+2t+1))
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
    const bool cur_lo = (sConn[(g / 5) * 4].y & kCurvedBit) != 0;
    const bool cur_hi = g + 8 < 15 && (sConn[((g + 8) / 5) * 4].y & kCurvedBit) != 0;
    constexpr bool R2 = CDG_WA_RES2 && RM == 0 && C::NT2 <= 5;  // HLLC and p=5 spill with both rows live
    double2 rsv2[R2 ? 2 : 1][C::NT2];
    if (R2 && UPDATE)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const bool ok = (hh ? ok_hi : ok_lo) && !(hh ? cur_hi : cur_lo);
        const size_t rowoff = (size_t)(hh ? r_hi : r_lo) * C::BP;
#pragma unroll
        for (int j = 0; j < C::NT2; ++j)
          rsv2[R2 ? hh : 0][j] =
              ok ? *reinterpret_cast<const double2*>(p.res + rowoff + j * 8 + 2 * tq) : make_double2(0.0, 0.0);
      }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const bool ok = hh ? ok_hi : ok_lo;
      if (!ok || (hh ? cur_hi : cur_lo)) continue;  // curved rows: the curved kernel
      const size_t rowoff = (size_t)(hh ? r_hi : r_lo) * C::BP;
      double2* rsv = rsv2[R2 ? hh : 0];
      if (UPDATE && !R2)  // every old res value of the row before any store
#pragma unroll
        for (int j = 0; j < C::NT2; ++j) rsv[j] = *reinterpret_cast<const double2*>(p.res + rowoff + j * 8 + 2 * tq);
#pragma unroll
      for (int j = 0; j < C::NT2; ++j) {
        const int col = j * 8 + 2 * tq;  // < KP == BP; padded columns carry exact zeros
        const double r0 = acc[j][2 * hh], r1 = acc[j][2 * hh + 1];
        if (UPDATE) {
          const double n0 = a_c * rsv[j].x + dt * r0, n1 = a_c * rsv[j].y + dt * r1;
          *reinterpret_cast<double2*>(p.res + rowoff + col) = make_double2(n0, n1);
          const double u0 = hh ? uA[j][1] : uA[j][0], u1 = hh ? uA[j][3] : uA[j][2];
          const double w0 = u0 + b_c * n0, w1 = u1 + b_c * n1;
          *reinterpret_cast<double2*>(p.u + rowoff + col) = make_double2(w0, w1);
          acc[j][2 * hh] = w0;  // u_new in the accumulator (= A fragment) layout
          acc[j][2 * hh + 1] = w1;
        } else {
          *reinterpret_cast<double2*>(p.rhs_out + rowoff + col) = make_double2(r0, r1);
        }
      }
    }
    if (C::FT && UPDATE && p.traces_out) {
      // next stage's traces T = u_new I_g^T (solver.cpp:200-208) from the
      // registers; the trace kernel's pairing and fragments (bit-identical)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const bool ok = hh ? ok_hi : ok_lo;
        if (!ok || (hh ? cur_hi : cur_lo))
#pragma unroll
          for (int j = 0; j < C::NT2; ++j) acc[j][2 * hh] = acc[j][2 * hh + 1] = 0.0;
      }
      constexpr int NFT = C::NF8 / 8;
      const double2* fbi = reinterpret_cast<const double2*>(p.frag_ig_nat);  // [NFT][KS1][32]
      AFrag fa[C::KS1];
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) fa[ks] = AFrag{acc[ks][0], acc[ks][2], acc[ks][1], acc[ks][3]};
#pragma unroll
      for (int nt0 = 0; nt0 < NFT; nt0 += 4) {
        double tacc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) tacc[i][0] = tacc[i][1] = tacc[i][2] = tacc[i][3] = 0.0;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (nt0 + i < NFT) mma_frag(tacc[i], fa[ks], __ldg(fbi + ((size_t)(nt0 + i) * C::KS1 + ks) * 32 + lane));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int col = (nt0 + i) * 8 + 2 * tq;
          if (nt0 + i < NFT && col < C::NF) {
            if (ok_lo)
              *reinterpret_cast<double2*>(p.traces_out + (size_t)r_lo * C::TB + col) = make_double2(tacc[i][0], tacc[i][1]);
            if (ok_hi)
              *reinterpret_cast<double2*>(p.traces_out + (size_t)r_hi * C::TB + col) = make_double2(tacc[i][2], tacc[i][3]);
          }
        }
      }
    }
    __syncwarp();  // the warp's panels / tables are restaged next tile
  }
}

}  // namespace cdg_gpu
