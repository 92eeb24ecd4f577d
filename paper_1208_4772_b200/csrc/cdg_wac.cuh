// cdg_wac.cuh -- warp-autonomous RHS + LSRK kernel for CURVED elements: the
// math of k_rhs_rowc (cdg_rowc.cuh; reference operators.cpp:32-167,
// solver.cpp:325-464) -- per-node metrics, per-face-node (n, sjac w), the
// M_e^-1 epilogue -- mapped like k_rhs_wa (cdg_wa.cuh): each warp owns THREE
// curved elements (15 gathered (element, field) rows + 1 padding row), so the
// GEMMs, the pointwise and face fluxes and the M_e^-1 GEMV only exchange data
// through warp-private shared panels (__syncwarp); no CTA barrier.
// KIND 0: inviscid RHS (+ update); 1: viscous RHS (+ update); 2: the aux
// gradient q_0..q_2 in one pass (NA = 3 accumulator sets and panels).
#pragma once

#include "cdg_rowc.cuh"

#ifndef CDG_WAC_FUNROLL
#define CDG_WAC_FUNROLL 1
#endif
#ifndef CDG_WAC_FT
#define CDG_WAC_FT 1  // fused next-stage traces from the update kernel (fused-trace path)
#endif
#ifndef CDG_WAC_METPRE
#define CDG_WAC_METPRE 1  // a lane's per-node metrics loaded before the chunk's GEMM1 (latency hidden)
#endif

namespace cdg_gpu {

template <int NP_, int NCUB_, int NG_, int CH_ = 8, int FCH_ = 32, int WARPS_ = 16, int MINB_ = 1, int NA_ = 1>
struct WacCfg {
  static constexpr int NA = NA_;  // accumulator sets: 1 (RHS) or 3 (aux gradient)
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int EPW = 3, WARPS = WARPS_, E = EPW * WARPS_, NTH = 32 * WARPS_, MINB = MINB_;
  static constexpr int BP = dev_block(NP), TB = dev_tblock(NF);
  static constexpr int KP = round_up(NP, 8), KS1 = KP / 8, NT2 = KS1;
  static constexpr int NCUB8 = round_up(NCUB, 8), NF8 = round_up(NF, 8);
  static constexpr int CH = CH_, NCH = ceil_div(NCUB8, CH);
  static constexpr int FCH = FCH_, NFCH = ceil_div(NF, FCH);
  static constexpr int K2CUB = 3 * NCUB8, K2 = K2CUB + NF8;
  static constexpr int LDC = frag_ld8(CH), LDG = frag_ld8(3 * CH), LDF = frag_ld8(FCH);
  static constexpr int LDV = KP + 1;  // vol panel of the epilogue
  static constexpr int VOLW = 16 * LDC + NA_ * 16 * LDG, FACEW = NA_ * 16 * LDF, EPIW = NA_ * 16 * LDV;
  static constexpr int W1 = VOLW > FACEW ? VOLW : FACEW;
  static constexpr int WORKW = W1 > EPIW ? W1 : EPIW;  // doubles per warp (phases alias)
  // per warp: [work panels | conn (int2) | ids (int)], a multiple of 2 doubles
  static constexpr int PERW = round_up(WORKW + EPW * 4 + ceil_div(EPW, 2), 2);
  static constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)PERW * WARPS_;
  static constexpr int IT_P = ceil_div(EPW * CH, 32), IT_F = ceil_div(EPW * FCH, 32);
  static constexpr int FUNROLL = CDG_WAC_FUNROLL;  // face-item loop unroll (tuning)
  static constexpr bool METPRE = CDG_WAC_METPRE && IT_P == 1;
  static constexpr bool FT = CDG_WAC_FT;
  static constexpr int NFT = NF8 / 8;  // n-tiles of the fused traces
};

template <class C, bool UPDATE, int RM, int KIND = 0>
__global__ void __launch_bounds__(C::NTH, C::MINB) k_rhs_wac(CurvedParams cp) {
  constexpr bool VISC = KIND == 1, AUX = KIND == 2;
  constexpr int NA = C::NA;
  static_assert(NA == (AUX ? 3 : 1), "the aux gradient needs the 3-panel layout");
  constexpr bool UPD = UPDATE && !AUX;
  const RhsParams& p = cp.base;
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  double* sWork = smem + (size_t)warp * C::PERW;
  double* sC = sWork;                      // [16][LDC]
  double* sG = sWork + 16 * C::LDC;        // [16][LDG]
  double* sF = sWork;                      // [16][LDF]
  double* sV = sWork;                      // [16][LDV] (epilogue)
  int2* sConn = reinterpret_cast<int2*>(sWork + C::WORKW);  // [3][4]
  int* sId = reinterpret_cast<int*>(sConn + C::EPW * 4);    // [3]
  const double gamma = p.gas.gamma;
  const int n_tiles = (cp.Kc + C::E - 1) / C::E;
  const double2* fb1all = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fb2all = reinterpret_cast<const double2*>(cp.frag_opc);
  constexpr int LDQ = round_up(C::NCUB, 8);       // qcub row stride
  const size_t qcs = (size_t)p.K * 5 * LDQ;       // qcub direction stride
  const size_t qstride = (size_t)p.K * 5 * C::BP;  // q_out direction stride

  const int n_iter = cp.ctiles ? cp.n_clist : n_tiles;  // optional curved-tile list (multi-GPU split)
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = cp.ctiles ? __ldg(cp.ctiles + it_t) : it_t;
    const int c0 = tile * C::E + warp * C::EPW;  // this warp's three curved-list entries
    if (c0 >= cp.Kc) continue;                    // warp-uniform
    if (!AUX && __shfl_sync(0xffffffffu, lane == 0 ? *(volatile int*)&p.err->flag : 0, 0)) return;
    if (lane < C::EPW) sId[lane] = c0 + lane < cp.Kc ? __ldg(cp.ids + c0 + lane) : -1;
    __syncwarp();
    if (lane < C::EPW * 4) {
      const int e = sId[lane / 4];
      sConn[lane] = e >= 0 ? p.conn[(size_t)e * 4 + lane % 4] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    // rows r = g and g + 8 of the m-tile: element r / 5 of the warp, field r % 5
    const int el_lo = sId[g / 5], el_hi = g + 8 < 15 ? sId[(g + 8) / 5] : -1;
    const bool ok_lo = el_lo >= 0, ok_hi = el_hi >= 0;
    const double* u_lo = p.u + (ok_lo ? (size_t)el_lo * 5 + g % 5 : 0) * C::BP + 2 * tq;
    const double* u_hi = p.u + (ok_hi ? (size_t)el_hi * 5 + (g + 8) % 5 : 0) * C::BP + 2 * tq;
    __syncwarp();

    double acc[NA][C::NT2][4];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int i = 0; i < C::NT2; ++i) acc[a][i][0] = acc[a][i][1] = acc[a][i][2] = acc[a][i][3] = 0.0;
    // acc[a] += P_a Op^T over the NA panels P_a = panel + a * pstride (one B load feeds NA MMAs)
    auto contract = [&](const double* panel, int ld, int nks, int nks_full, const double2* fb2) {
      const int pstride = 16 * ld;
      auto kstep = [&](int ks) {
        AFrag a[NA];
#pragma unroll
        for (int k = 0; k < NA; ++k) a[k] = load_afrag(panel + k * pstride, ld, 0, ks * 8, g, tq);
#pragma unroll
        for (int nt = 0; nt < C::NT2; ++nt) {
          const double2 b = __ldg(fb2 + (ks * C::NT2 + nt) * 32 + lane);
#pragma unroll
          for (int k = 0; k < NA; ++k) mma_frag(acc[k][nt], a[k], b);
        }
      };
      if (nks == nks_full) {
#pragma unroll
        for (int ks = 0; ks < nks_full; ++ks) kstep(ks);
      } else {
#pragma unroll 1
        for (int ks = 0; ks < nks; ++ks) kstep(ks);
      }
    };

    // ---- volume: chunks of CH cubature nodes ----------------------------------
#pragma unroll 1
    for (int ch = 0; ch < C::NCH; ++ch) {
      const int q0 = ch * C::CH;
      const int w = min(C::CH, C::NCUB8 - q0);
      const double2* fb1 = fb1all + (size_t)(q0 / 8) * C::KS1 * 32;
      double mpre[9];  // METPRE: this lane's pointwise item's metrics, in flight during GEMM1
      if (C::METPRE) {
        const int e = lane / w, q = q0 + lane - e * w;
        const bool ok = lane < C::EPW * w && q < C::NCUB && c0 + e < cp.Kc;
        const double* met = cp.jwr + (ok ? ((size_t)(c0 + e) * C::NCUB + q) * 9 : 0);
#pragma unroll
        for (int k = 0; k < 9; ++k) mpre[k] = ok ? __ldg(met + k) : 0.0;
      }
      {  // GEMM1: U_cub[rows, q0:q0+w], the gathered U rows as A fragments
        double c1[C::CH / 8][4];
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j) c1[j][0] = c1[j][1] = c1[j][2] = c1[j][3] = 0.0;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks) {
          double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
          if (ok_lo) x = *reinterpret_cast<const double2*>(u_lo + ks * 8);
          if (ok_hi) y = *reinterpret_cast<const double2*>(u_hi + ks * 8);
#pragma unroll
          for (int j = 0; j < C::CH / 8; ++j)
            if (j * 8 < w) {
              const double2 b = __ldg(fb1 + (j * C::KS1 + ks) * 32 + lane);
              dmma_k8(c1[j], x.x, y.x, x.y, y.y, b.x, b.y);
            }
        }
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j)
          if (j * 8 < w) {
            double* o = sC + g * C::LDC + j * 8 + 2 * tq;
            *reinterpret_cast<double2*>(o) = make_double2(c1[j][0], c1[j][1]);
            *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c1[j][2], c1[j][3]);
          }
      }
      __syncwarp();
      // pointwise: G_m = sum_d (J W dr_m/dx_d) F_d per cubature node
#pragma unroll
      for (int it = 0; it < C::IT_P; ++it) {
        const int idx = lane + it * 32;
        if (idx < C::EPW * w) {
          const int e = idx / w, ql = idx - e * w, q = q0 + ql;
          const double* uc = sC + (e * 5) * C::LDC + ql;
          double* gout = sG + (e * 5) * C::LDG + ql;
          const int ce = c0 + e;
          if (q < C::NCUB && ce < cp.Kc && AUX) {
            // G_k = -se (J W dr_k/dx_m) U_cub for the three directions m
            const double* met = cp.jwr + ((size_t)ce * C::NCUB + q) * 9;
            const double se = p.sqrt_eps[sId[e]];
            const double uv[5] = {uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
#pragma unroll
            for (int ma = 0; ma < 3; ++ma)
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                const double jk = C::METPRE ? mpre[k * 3 + ma] : __ldg(met + k * 3 + ma);
#pragma unroll
                for (int c = 0; c < 5; ++c) gout[ma * 16 * C::LDG + k * w + c * C::LDG] = -se * (jk * uv[c]);
              }
          } else if (q < C::NCUB && ce < cp.Kc) {
            const double* met = cp.jwr + ((size_t)ce * C::NCUB + q) * 9;
            const State5 s{uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
            if (!admissible(s, gamma)) record_error(p.err, 1, p.elem_offset + sId[e], q, 0, s.r);
            const double ir = 1.0 / s.r;
            const double pr = (gamma - 1.0) * (s.E - 0.5 * ir * (s.mx * s.mx + s.my * s.my + s.mz * s.mz));
            const double vx = s.mx * ir, vy = s.my * ir, vz = s.mz * ir;
            const double ep = s.E + pr;
            double se = 0.0;
            if (VISC) se = p.sqrt_eps[sId[e]];
#pragma unroll
            for (int m = 0; m < 3; ++m) {
              const double r0 = C::METPRE ? mpre[m * 3] : __ldg(met + m * 3),
                           r1 = C::METPRE ? mpre[m * 3 + 1] : __ldg(met + m * 3 + 1),
                           r2 = C::METPRE ? mpre[m * 3 + 2] : __ldg(met + m * 3 + 2);
              const double um = r0 * vx + r1 * vy + r2 * vz;
              double gm[5] = {s.r * um, s.mx * um + pr * r0, s.my * um + pr * r1, s.mz * um + pr * r2, ep * um};
              if (VISC && se > 0.0) {
                // F_d -= se I_cub q_d  (solver.cpp:398-406), contracted with r_m
                const size_t qo = ((size_t)sId[e] * 5) * LDQ + q;
#pragma unroll
                for (int c = 0; c < 5; ++c)
                  gm[c] -= se * (r0 * __ldg(p.qcub + qo + c * LDQ) + r1 * __ldg(p.qcub + qcs + qo + c * LDQ) +
                                 r2 * __ldg(p.qcub + 2 * qcs + qo + c * LDQ));
              }
#pragma unroll
              for (int c = 0; c < 5; ++c) gout[m * w + c * C::LDG] = gm[c];
            }
          } else {
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
              for (int m = 0; m < 3; ++m)
#pragma unroll
                for (int c = 0; c < 5; ++c) gout[a * 16 * C::LDG + m * w + c * C::LDG] = 0.0;
          }
        }
      }
      if (lane < 3 * w)
#pragma unroll
        for (int a = 0; a < NA; ++a) sG[a * 16 * C::LDG + 15 * C::LDG + lane] = 0.0;  // the padding row
      __syncwarp();
      contract(sG, C::LDG, (3 * w) / 8, 3 * C::CH / 8, fb2all + (size_t)(3 * q0 / 8) * C::NT2 * 32);
      __syncwarp();
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
        const int ce = c0 + e, eg = sId[e];
        if (ce >= cp.Kc || fl >= wr) {
#pragma unroll
          for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int c = 0; c < 5; ++c) gout[a * 16 * C::LDF + c * C::LDF] = 0.0;
          continue;
        }
        const int f = fq / C::NG, gq = fq - f * C::NG;
        const double* tm = p.traces + (size_t)eg * 5 * C::TB + fq;
        const State5 um{tm[0], tm[C::TB], tm[2 * C::TB], tm[3 * C::TB], tm[4 * C::TB]};
        const double4 fn = cp.face[(size_t)ce * C::NF + fq];
        const int2 cw = sConn[e * 4 + f];
        State5 up;
        int h = 0;
        if (cw.x >= 0) {
          h = __ldg(p.code_map + (cw.y >> 8) * C::NG + gq);
          const double* tp = p.traces + (size_t)cw.x * 5 * C::TB + (cw.y & 3) * C::NG + h;
          up = State5{tp[0], tp[C::TB], tp[2 * C::TB], tp[3 * C::TB], tp[4 * C::TB]};
        } else {
          up = boundary_state(um, fn.x, fn.y, fn.z, (cw.y >> 2) & 3, p.gas);
        }
        if (AUX) {
          // central trace average with per-side sqrt(eps) (solver.cpp:291-309),
          // fed negated to the [D^T | -I_g^T] operator, for the three directions
          const double se = p.sqrt_eps[eg];
          const double snb = cw.x >= 0 ? p.sqrt_eps[cw.x] : se;
          const double umv[5] = {um.r, um.mx, um.my, um.mz, um.E};
          const double upv[5] = {up.r, up.mx, up.my, up.mz, up.E};
          const double nrm[3] = {fn.x, fn.y, fn.z};
#pragma unroll
          for (int ma = 0; ma < 3; ++ma)
#pragma unroll
            for (int c = 0; c < 5; ++c)
              gout[ma * 16 * C::LDF + c * C::LDF] = -fn.w * (0.5 * (se * umv[c] + snb * upv[c]) * nrm[ma]);
          continue;
        }
        if (!admissible(um, gamma) || !admissible(up, gamma)) record_error(p.err, 2, p.elem_offset + eg, f, gq, um.r);
        double fs[5];
        if (RM == 1)
          hllc_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs, p.gas.hllc_fallbacks);
        else
          llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
        if (VISC) {
          // BR1 central viscous flux with per-side sqrt(eps) (solver.cpp:438-453)
          const double se = p.sqrt_eps[eg];
          const bool has_nb = cw.x >= 0;
          const double snb = has_nb ? p.sqrt_eps[cw.x] : se;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            // q.n on both sides from the normal-projected traces (k_qn_traces); the
            // neighbour's value is on its own outward normal, -n here
            const double qs = p.qtr[((size_t)eg * 5 + c) * C::TB + fq];
            const double qn = has_nb ? -p.qtr[((size_t)cw.x * 5 + c) * C::TB + (cw.y & 3) * C::NG + h] : qs;
            fs[c] -= 0.5 * (se * qs + snb * qn);
          }
        }
#pragma unroll
        for (int c = 0; c < 5; ++c) gout[c * C::LDF] = fn.w * fs[c];
      }
      if (lane < wp)
#pragma unroll
        for (int a = 0; a < NA; ++a) sF[a * 16 * C::LDF + 15 * C::LDF + lane] = 0.0;  // the padding row
      __syncwarp();
      contract(sF, C::LDF, wp / 8, C::FCH / 8, fb2all + (size_t)((C::K2CUB + f0) / 8) * C::NT2 * 32);
      __syncwarp();
    }

    // ---- epilogue: vol -> warp panel, M_e^-1 vol -> update / rhs ----------------
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int nt = 0; nt < C::NT2; ++nt) {
        const int col = nt * 8 + 2 * tq;
        double* va = sV + a * 16 * C::LDV;
        va[g * C::LDV + col] = acc[a][nt][0];
        va[g * C::LDV + col + 1] = acc[a][nt][1];
        va[(g + 8) * C::LDV + col] = acc[a][nt][2];
        va[(g + 8) * C::LDV + col + 1] = acc[a][nt][3];
      }
    __syncwarp();
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPD) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
    // one lane per (element, node i): out_f(i) = sum_j (M_e^-1)[i][j] vol_f(j),
    // the column stream of M_e^-1 software-pipelined in groups of MG
    constexpr int MG = 7, NGR = ceil_div(C::NP, MG);
    for (int idx = lane; idx < C::EPW * C::NP; idx += 32) {
      const int e = idx / C::NP, i = idx - e * C::NP;
      const int ce = c0 + e;
      if (ce >= cp.Kc) continue;
      const double* mcol = cp.minv + (size_t)ce * C::NP * C::NP + i;  // (M_e^-1)[i][j] at j*NP + i
      const double* v = sV + (e * 5) * C::LDV;
      const size_t g0 = ((size_t)sId[e] * 5) * C::BP + i;
      double m[MG];
#pragma unroll
      for (int k = 0; k < MG; ++k) m[k] = k < C::NP ? __ldg(mcol + (size_t)k * C::NP) : 0.0;
      double ro[5], uo[5];
      if (UPD) {
#pragma unroll
        for (int f = 0; f < 5; ++f) {
          ro[f] = p.res[g0 + (size_t)f * C::BP];
          uo[f] = p.u[g0 + (size_t)f * C::BP];
        }
      }
      double out[NA][5];
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int f = 0; f < 5; ++f) out[a][f] = 0.0;
#pragma unroll 1
      for (int gr = 0; gr < NGR; ++gr) {
        const int j0 = gr * MG;
        double mn[MG];
#pragma unroll
        for (int k = 0; k < MG; ++k) {
          const int j = j0 + MG + k;
          mn[k] = j < C::NP ? __ldg(mcol + (size_t)j * C::NP) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < MG; ++k)
          if (j0 + k < C::NP)
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
              for (int f = 0; f < 5; ++f) out[a][f] += m[k] * v[a * 16 * C::LDV + f * C::LDV + j0 + k];
#pragma unroll
        for (int k = 0; k < MG; ++k) m[k] = mn[k];
      }
#pragma unroll
      for (int f = 0; f < 5; ++f) {
        const size_t gi = g0 + (size_t)f * C::BP;
        if (AUX) {
#pragma unroll
          for (int a = 0; a < NA; ++a) cp.q_out[a * qstride + gi] = out[a][f];
        } else if (UPD) {
          const double rn = a_c * ro[f] + dt * out[0][f];
          p.res[gi] = rn;
          p.u[gi] = uo[f] + b_c * rn;
        } else {
          p.rhs_out[gi] = out[0][f];
        }
      }
    }
    if (C::FT && UPD && !VISC && p.traces_out) {
      // next stage's traces T = u_new I_g^T (solver.cpp:200-208): the warp's
      // rows of u_new (just stored; visible to the warp after __syncwarp) as
      // natural-pairing A fragments times the trace kernel's B fragments --
      // k_interp<NAT>'s arithmetic, so fused and separate traces agree bit for bit
      __syncwarp();
      AFrag ua[C::KS1];
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) {
        double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
        if (ok_lo) x = *reinterpret_cast<const double2*>(u_lo + ks * 8);
        if (ok_hi) y = *reinterpret_cast<const double2*>(u_hi + ks * 8);
        ua[ks] = AFrag{x.x, y.x, x.y, y.y};
      }
      const double2* fig = reinterpret_cast<const double2*>(p.frag_ig_nat);
      double* t_lo = p.traces_out + ((size_t)(ok_lo ? el_lo : 0) * 5 + g % 5) * C::TB;
      double* t_hi = p.traces_out + ((size_t)(ok_hi ? el_hi : 0) * 5 + (g + 8) % 5) * C::TB;
#pragma unroll 2
      for (int nt = 0; nt < C::NFT; ++nt) {
        double tacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks) mma_frag(tacc, ua[ks], __ldg(fig + ((size_t)nt * C::KS1 + ks) * 32 + lane));
        const int col = nt * 8 + 2 * tq;
        if (col < C::NF) {
          if (ok_lo) *reinterpret_cast<double2*>(t_lo + col) = make_double2(tacc[0], tacc[1]);
          if (ok_hi) *reinterpret_cast<double2*>(t_hi + col) = make_double2(tacc[2], tacc[3]);
        }
      }
    }
    __syncwarp();  // the warp's panels are rewritten by its next tile
  }
}

}  // namespace cdg_gpu
