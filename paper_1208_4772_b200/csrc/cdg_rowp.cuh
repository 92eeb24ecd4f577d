// cdg_rowp.cuh -- software-pipelined row-per-warp RHS + LSRK kernel (p = 4).
//
// Same math, row mapping and operators as k_rhs_row (cdg_row.cuh; reference
// solver.cpp:325-492). The K dimension of the RHS contraction is walked in
// chunks of 24 columns -- a cubature chunk (3 directions x 8 nodes) or a face
// chunk (24 face nodes) -- and the chunks are software-pipelined so that a
// CTA needs ONE barrier per chunk instead of two:
//
//   phase A(c):  GEMM1 of chunk c+1 (U_cub for 8 cubature nodes -> sC[c+1 & 1])
//   barrier
//   phase B(c):  pointwise flux of chunk c+1 (cubature) or Riemann flux of
//                face chunk c+1  -> sG[c+1 & 1]
//                then the RHS GEMM of chunk c from sG[c & 1]
//
// Double buffers make both hazards disappear without a second barrier: sC[c&1]
// is rewritten in A(c+1) only after every warp has passed B(c-1) (its last
// reader), and sG[c&1] in B(c+1) only after every warp has finished B(c).
// The SIMT flux work of chunk c+1 and the DMMA work of chunk c now sit in the
// same phase, so the warp that has no flux points (128 points over 160
// threads) starts its GEMM early instead of idling at a barrier.
#pragma once

#include "cdg_row.cuh"

namespace cdg_gpu {

template <int NP_, int NCUB_, int NG_, int MINB_ = 4, bool USMEM_ = false>
struct RPCfg {
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int E = 16, R = 80, NW = 5, NTH = 160, MINB = MINB_;
  static constexpr bool USMEM = USMEM_;
  static constexpr int BP = round_up(NP, 16), TB = round_up(NF, 16);
  static constexpr int KP = round_up(NP, 8), KS1 = KP / 8, NT2 = KS1;
  static constexpr int NCUB8 = round_up(NCUB, 8), NF8 = round_up(NF, 8);
  static constexpr int CH = 8, FCH = 24;           // 3 k-steps per chunk either way
  static constexpr int NCH = NCUB8 / CH, NFCH = ceil_div(NF, FCH), NCHT = NCH + NFCH;
  static constexpr int K2CUB = 3 * NCUB8;
  static constexpr int LDC = CH + 4;               // U_cub chunk (pointwise reads columns)
  static constexpr int LDG = frag_ld8(3 * CH);     // flux chunk (24 columns, conflict-free A loads)
  static constexpr int LDU = frag_ld8(KP);
  static constexpr int UPANEL = USMEM ? R * LDU : 0;
  static constexpr int IT_P = ceil_div(E * CH, NTH);
  static constexpr int IT_F = ceil_div(E * FCH, NTH);
  static constexpr size_t SMEM_BYTES =
      sizeof(double) * ((size_t)2 * R * LDC + 2 * R * LDG + UPANEL + E * 9 + E * 4 * 4) + sizeof(int) * (E * 4 * 2);
};

template <class C, bool UPDATE, int RM>
__global__ void __launch_bounds__(C::NTH, C::MINB) k_rhs_rowp(RhsParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sCb = smem;                                  // [2][R][LDC]
  double* sGb = sCb + 2 * C::R * C::LDC;               // [2][R][LDG]
  double* sUp = sGb + 2 * C::R * C::LDG;               // [R][LDU] (USMEM)
  double* sMet = sUp + C::UPANEL;                      // [E][9]
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);
  int2* sConn = reinterpret_cast<int2*>(sFace + C::E * 4);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const int n_tiles = (p.K + C::E - 1) / C::E;
  const double2* fb1g = reinterpret_cast<const double2*>(p.frag_icub);  // [NCUB8/8][KS1][32]
  const double2* fb2g = reinterpret_cast<const double2*>(p.frag_op2);   // [KS2][NT2][32]
  __shared__ int s_stop;

  const int n_iter = p.tiles ? p.n_list : n_tiles;
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = tile_at(p, it_t);
    if (tid == 0) s_stop = *(volatile int*)&p.err->flag;
    __syncthreads();
    if (s_stop) return;
    const int e0 = tile * C::E, row0 = e0 * 5;
    const int r_lo = row0 + warp * 16 + g, r_hi = r_lo + 8;
    const bool ok_lo = r_lo < n_rows, ok_hi = r_hi < n_rows;
    const double* u_lo = p.u + (size_t)min(r_lo, n_rows - 1) * C::BP + 2 * tq;
    const double* u_hi = p.u + (size_t)min(r_hi, n_rows - 1) * C::BP + 2 * tq;
    if (p.prefetch) {
      const int rows = min(C::R, n_rows - row0);
      if (UPDATE && (p.prefetch & 1)) l2_prefetch_range(p.res + (size_t)row0 * C::BP, (size_t)rows * C::BP * 8, tid, C::NTH);
      if (p.prefetch & 4) l2_prefetch_range(p.traces + (size_t)row0 * C::TB, (size_t)rows * C::TB * 8, tid, C::NTH);
      const int nrow0 = (tile + gridDim.x) * C::R;
      if ((p.prefetch & 2) && nrow0 < n_rows)
        l2_prefetch_range(p.u + (size_t)nrow0 * C::BP, (size_t)min(C::R, n_rows - nrow0) * C::BP * 8, tid, C::NTH);
    }
    if (C::USMEM) {
      constexpr int V = C::KP / 2;
      for (int idx = tid; idx < C::R * V; idx += C::NTH) {
        const int r = idx / V, j = idx - r * V;
        double* dst = sUp + r * C::LDU + 2 * j;
        if (row0 + r < n_rows)
          cp_async16_sh(dst, p.u + (size_t)(row0 + r) * C::BP + 2 * j);
        else
          *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
      }
      cp_async_wait0();
    }
    for (int idx = tid; idx < C::E * 9; idx += C::NTH)
      sMet[idx] = e0 + idx / 9 < p.K ? __ldg(p.metric + (size_t)e0 * 9 + idx) : 0.0;
    for (int idx = tid; idx < C::E * 4; idx += C::NTH) {
      const bool ok = e0 + idx / 4 < p.K;
      sFace[idx] = ok ? p.face[(size_t)e0 * 4 + idx] : make_double4(0, 0, 1, 0);
      sConn[idx] = ok ? p.conn[(size_t)e0 * 4 + idx] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    __syncthreads();
    if (p.prefetch & 8) {
      for (int idx = tid; idx < C::E * 4 * 5; idx += C::NTH) {
        const int ef = idx / 5, c = idx - ef * 5;
        const int2 cw = sConn[ef];
        if (cw.x >= 0) {
          const double* seg = p.traces + ((size_t)cw.x * 5 + c) * C::TB + (cw.y & 3) * C::NG;
          l2_prefetch(seg);
          if (C::NG * 8 > 128) l2_prefetch(seg + C::NG - 1);
        }
      }
    }

    // ---- stage functions -------------------------------------------------------
    // GEMM1 of cubature chunk ch: U_cub[warp rows, 8 nodes] -> sC[ch & 1]
    auto gemm1 = [&](int ch) {
      double c1[4] = {0.0, 0.0, 0.0, 0.0};
      const double2* fb1 = fb1g + (size_t)ch * C::KS1 * 32;
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) {
        double a0, a1, a2, a3;
        if (C::USMEM) {
          const AFrag a = load_afrag(sUp, C::LDU, warp * 16, ks * 8, g, tq);
          a0 = a.a0, a1 = a.a1, a2 = a.a2, a3 = a.a3;
        } else {
          double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
          if (ok_lo) x = *reinterpret_cast<const double2*>(u_lo + ks * 8);
          if (ok_hi) y = *reinterpret_cast<const double2*>(u_hi + ks * 8);
          a0 = x.x, a1 = y.x, a2 = x.y, a3 = y.y;
        }
        const double2 b = __ldg(fb1 + ks * 32 + lane);
        dmma_k8(c1, a0, a1, a2, a3, b.x, b.y);
      }
      double* o = sCb + (ch & 1) * (C::R * C::LDC) + (warp * 16 + g) * C::LDC + 2 * tq;
      *reinterpret_cast<double2*>(o) = make_double2(c1[0], c1[1]);
      *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c1[2], c1[3]);
    };
    // flux of chunk c (cubature pointwise flux, or Riemann flux of a face chunk) -> sG[c & 1]
    auto flux = [&](int c) {
      double* sG = sGb + (c & 1) * (C::R * C::LDG);
      if (c < C::NCH) {
        const double* sC = sCb + (c & 1) * (C::R * C::LDC);
        const int q0 = c * C::CH;
#pragma unroll 1
        for (int it = 0; it < C::IT_P; ++it) {
          const int idx = tid + it * C::NTH;
          if (idx >= C::E * C::CH) continue;
          const int e = idx / C::CH, ql = idx - e * C::CH, q = q0 + ql;
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
              double* o = gout + m * C::CH;
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
              for (int k = 0; k < 5; ++k) gout[m * C::CH + k * C::LDG] = 0.0;
          }
        }
      } else {
        const int f0 = (c - C::NCH) * C::FCH;
        const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
        const int wp = round_up(wr, 8);
#pragma unroll 1
        for (int it = 0; it < C::IT_F; ++it) {
          const int idx = tid + it * C::NTH;
          if (idx >= C::E * wp) continue;
          const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
          double* gout = sG + (e * 5) * C::LDG + fl;
          const int eg = e0 + e;
          if (eg >= p.K || fl >= wr) {
#pragma unroll
            for (int k = 0; k < 5; ++k) gout[k * C::LDG] = 0.0;
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
          if (!admissible(um, gamma) || !admissible(up, gamma))
            record_error(p.err, 2, p.elem_offset + eg, f, gq, um.r);
          double fs[5];
          if (RM == 1)
            hllc_flux(um, up, fn.x, fn.y, fn.z, gamma, fs);
          else
            llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
#pragma unroll
          for (int k = 0; k < 5; ++k) gout[k * C::LDG] = fn.w * fs[k];
        }
      }
    };
    double acc[C::NT2][4];
#pragma unroll
    for (int i = 0; i < C::NT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
    // RHS GEMM of chunk c from sG[c & 1] (k-steps of the chunked op2 layout)
    auto gemm2 = [&](int c) {
      const double* sG = sGb + (c & 1) * (C::R * C::LDG);
      int ks0, nks;
      if (c < C::NCH) {
        ks0 = 3 * c;
        nks = 3;
      } else {
        const int f0 = (c - C::NCH) * C::FCH;
        ks0 = (C::K2CUB + f0) / 8;
        nks = round_up(min(C::FCH, C::NF - f0), 8) / 8;
      }
#pragma unroll 1
      for (int ks = 0; ks < nks; ++ks) {
        const AFrag a = load_afrag(sG, C::LDG, warp * 16, ks * 8, g, tq);
#pragma unroll
        for (int nt = 0; nt < C::NT2; ++nt)
          mma_frag(acc[nt], a, __ldg(fb2g + ((size_t)(ks0 + ks) * C::NT2 + nt) * 32 + lane));
      }
    };

    // ---- pipelined chunk loop ---------------------------------------------------
    gemm1(0);
    __syncthreads();
    flux(0);
#pragma unroll 1
    for (int c = 0; c < C::NCHT; ++c) {
      if (c + 1 < C::NCH) gemm1(c + 1);
      __syncthreads();
      if (c + 1 < C::NCHT) flux(c + 1);
      gemm2(c);
    }

    // ---- epilogue: rhs -> (res, u) update or rhs store ---------------------------
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
    const bool cur_lo = (sConn[((warp * 16 + g) / 5) * 4].y & kCurvedBit) != 0;
    const bool cur_hi = (sConn[((warp * 16 + g + 8) / 5) * 4].y & kCurvedBit) != 0;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int grow = hh ? r_hi : r_lo;
      if (grow >= n_rows || (hh ? cur_hi : cur_lo)) continue;  // curved rows: k_rhs_curved
      const size_t rowoff = (size_t)grow * C::BP;
#pragma unroll
      for (int j = 0; j < C::NT2; ++j) {
        const int col = j * 8 + 2 * tq;  // < KP <= BP; padded columns carry exact zeros
        const double r0 = acc[j][2 * hh], r1 = acc[j][2 * hh + 1];
        if (UPDATE) {
          const double2 rs = *reinterpret_cast<const double2*>(p.res + rowoff + col);
          const double n0 = a_c * rs.x + dt * r0, n1 = a_c * rs.y + dt * r1;
          *reinterpret_cast<double2*>(p.res + rowoff + col) = make_double2(n0, n1);
          const double2 uo = C::USMEM ? *reinterpret_cast<const double2*>(sUp + (warp * 16 + g + 8 * hh) * C::LDU + col)
                                      : *reinterpret_cast<const double2*>(p.u + rowoff + col);
          *reinterpret_cast<double2*>(p.u + rowoff + col) = make_double2(uo.x + b_c * n0, uo.y + b_c * n1);
        } else {
          *reinterpret_cast<double2*>(p.rhs_out + rowoff + col) = make_double2(r0, r1);
        }
      }
    }
    __syncthreads();  // sConn / buffers are restaged next tile
  }
}

}  // namespace cdg_gpu
