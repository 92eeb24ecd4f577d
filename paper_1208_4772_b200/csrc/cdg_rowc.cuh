// cdg_rowc.cuh -- CURVED (isoparametric) elements on the row-per-warp layout
// of k_rhs_row (cdg_row.cuh): the inviscid RHS + LSRK update, the viscous RHS
// and the auxiliary gradient q.
//
// Math as k_rhs_curved / k_aux_curved (cdg_curved.cuh; reference
// operators.cpp:32-167, solver.cpp:264-464):
//   vol = sum_m D_m^T (JW r_m . F) - I_g^T ((sjac w) F*),   rhs = M_e^-1 vol
//   q_m = M_e^-1 [ -se sum_k D_k^T (JW dr_k/dx_m U_cub)
//                  + I_g^T ((sjac w) 1/2 (se U- + snb U+) n_m) ]
// Mapping as k_rhs_row: a CTA is 5E/16 warps on a tile of E curved elements
// (consecutive entries of the curved list), warp w owns rows [16w, 16w+16)
// of the (element, field) rows in both contractions, so each A fragment is
// reused across all N_p/8 n-tiles and the B fragments of the shared
// [D^T | -I_g^T] operator come from L1/L2 in the natural pairing. What is
// per element here and shared there:
//   * pointwise flux: the contravariant metric J W dr_m/dx_d is read per
//     cubature node (9 doubles) instead of once per element;
//   * face flux: (n, sjac w) per face node instead of per face;
//   * epilogue: vol goes through shared memory and M_e^-1 (dense, per
//     element, stored transposed so that the threads of a warp -- consecutive
//     output nodes i -- read consecutive addresses) is applied as a SIMT GEMV,
//     one thread per (element, node) for all five fields, its column stream
//     software-pipelined (on B200 the DFMA pipe matches the DMMA pipe per
//     flop; the GEMV is ~5% of the work).
// KIND 0: inviscid RHS (+ update); 1: viscous RHS (+ update; volume
// F_d -= se I_cub q_d, face F* -= 1/2 sum_m (se q-_m + snb q+_m) n_m,
// solver.cpp:398-406, 438-453); 2: aux gradient q_m, three passes m = 0..2.
#pragma once

#include "cdg_curved.cuh"
#include "cdg_row.cuh"

namespace cdg_gpu {

// NA = 1: one accumulator set (RHS); NA = 3: the aux gradient's three
// directions q_0..q_2 in ONE pass -- three G panels (volume) and three face
// panels share the U_cub chunk, the face gathers and every B fragment.
template <class C, int NA = 1>
struct RowCurvedLayout {
  static constexpr int LDV = C::KP + 1;  // vol panel [R][LDV] (aliases the work area)
  static constexpr int VOLA = C::R * C::LDC + NA * C::R * C::LDG;
  static constexpr int FACEA = NA * C::R * C::LDF;
  static constexpr int W1 = VOLA > FACEA ? VOLA : FACEA;
  static constexpr int W2 = C::WORK > W1 ? C::WORK : W1;
  static constexpr int WORK = W2 > NA * C::R * LDV ? W2 : NA * C::R * LDV;  // NA vol panels in the epilogue
  static constexpr size_t SMEM_BYTES = sizeof(double) * WORK + sizeof(int) * (C::E + C::E * 4 * 2);
};

template <class C, bool UPDATE, int RM, int KIND = 0>
__global__ void __launch_bounds__(C::NTH, C::MINB) k_rhs_rowc(CurvedParams cp) {
  constexpr bool VISC = KIND == 1, AUX = KIND == 2;
  constexpr int NA = AUX ? 3 : 1;  // accumulator sets (AUX: q_0, q_1, q_2 in one pass)
  using L = RowCurvedLayout<C, NA>;
  constexpr bool UPD = UPDATE && !AUX;
  const RhsParams& p = cp.base;
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sWork = smem;
  int2* sConn = reinterpret_cast<int2*>(sWork + L::WORK);  // [E][4]
  int* sId = reinterpret_cast<int*>(sConn + C::E * 4);     // [E] element ids of the tile
  __shared__ int s_stop;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const double gamma = p.gas.gamma;
  const int n_tiles = (cp.Kc + C::E - 1) / C::E;
  const double2* fb1all = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fb2all = reinterpret_cast<const double2*>(cp.frag_opc);
  const int lr_lo = warp * 16 + g, lr_hi = lr_lo + 8;  // this thread's two tile rows
  constexpr int LDQ = round_up(C::NCUB, 8);                // qcub row stride
  const size_t qcs = (size_t)p.K * 5 * LDQ;                // qcub direction stride
  const size_t qstride = (size_t)p.K * 5 * C::BP;          // q_out direction stride

  const int n_iter = cp.ctiles ? cp.n_clist : n_tiles;  // optional curved-tile list (multi-GPU split)
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = cp.ctiles ? __ldg(cp.ctiles + it_t) : it_t;
    const int c0 = tile * C::E;  // index into the curved list
    if (tid == 0) s_stop = *(volatile int*)&p.err->flag;
    for (int idx = tid; idx < C::E; idx += C::NTH) sId[idx] = c0 + idx < cp.Kc ? __ldg(cp.ids + c0 + idx) : -1;
    __syncthreads();
    if (!AUX && s_stop) return;  // block-uniform
    for (int idx = tid; idx < C::E * 4; idx += C::NTH) {
      const int e = sId[idx / 4];
      sConn[idx] = e >= 0 ? p.conn[(size_t)e * 4 + idx % 4] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    const int el_lo = sId[lr_lo / 5], el_hi = sId[lr_hi / 5];
    const bool ok_lo = el_lo >= 0, ok_hi = el_hi >= 0;
    const double* u_lo = p.u + (ok_lo ? (size_t)el_lo * 5 + lr_lo % 5 : 0) * C::BP + 2 * tq;
    const double* u_hi = p.u + (ok_hi ? (size_t)el_hi * 5 + lr_hi % 5 : 0) * C::BP + 2 * tq;

    {
      double acc[NA][C::NT2][4];
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int i = 0; i < C::NT2; ++i) acc[a][i][0] = acc[a][i][1] = acc[a][i][2] = acc[a][i][3] = 0.0;
      // acc[a] += P_a[rows, 8 nks] Op^T over the NA panels P_a = panel + a * pstride:
      // one B fragment load feeds NA MMAs
      auto contract = [&](const double* panel, int ld, size_t pstride, int nks, int nks_full, const double2* fb2) {
        auto kstep = [&](int ks) {
          AFrag a[NA];
#pragma unroll
          for (int k = 0; k < NA; ++k) a[k] = load_afrag(panel + k * pstride, ld, warp * 16, ks * 8, g, tq);
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

      // ---- volume: chunks of CH cubature nodes ------------------------------
#pragma unroll 1
      for (int ch = 0; ch < C::NCH; ++ch) {
        const int q0 = ch * C::CH;
        const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;
        double* sC = sWork;
        double* sG = sWork + C::R * C::LDC;
        const double2* fb1 = fb1all + (size_t)(q0 / 8) * C::KS1 * 32;
        const double2* fb2 = fb2all + (size_t)(3 * q0 / 8) * C::NT2 * 32;
        {  // GEMM1: U_cub[rows, q0:q0+w], U rows as A fragments straight from HBM/L2
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
              double* o = sC + lr_lo * C::LDC + j * 8 + 2 * tq;
              *reinterpret_cast<double2*>(o) = make_double2(c1[j][0], c1[j][1]);
              *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c1[j][2], c1[j][3]);
            }
        }
        __syncthreads();
        // pointwise: G_m = sum_d (J W dr_m/dx_d) F_d per cubature node (AUX:
        // G_k = -se (J W dr_k/dx_m) U_cub)
#pragma unroll 1
        for (int it = 0; it < C::IT_P; ++it) {
          const int idx = tid + it * C::NTH;
          if (idx < C::E * w) {
            const int e = idx / w, ql = idx - e * w, q = q0 + ql;
            const double* uc = sC + (e * 5) * C::LDC + ql;
            double* gout = sG + (e * 5) * C::LDG + ql;
            const int ce = c0 + e;
            if (q < C::NCUB && ce < cp.Kc) {
              const double* met = cp.jwr + ((size_t)ce * C::NCUB + q) * 9;
              if (AUX) {
                const double se = p.sqrt_eps[sId[e]];
                const double uv[5] = {uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
#pragma unroll
                for (int ma = 0; ma < 3; ++ma)
#pragma unroll
                  for (int k = 0; k < 3; ++k) {
                    const double jk = __ldg(met + k * 3 + ma);
#pragma unroll
                    for (int c = 0; c < 5; ++c) gout[ma * C::R * C::LDG + k * w + c * C::LDG] = -se * (jk * uv[c]);
                  }
              } else {
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
                  const double r0 = __ldg(met + m * 3), r1 = __ldg(met + m * 3 + 1), r2 = __ldg(met + m * 3 + 2);
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
              }
            } else {
#pragma unroll
              for (int a = 0; a < NA; ++a)
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                  for (int c = 0; c < 5; ++c) gout[a * C::R * C::LDG + m * w + c * C::LDG] = 0.0;
            }
          }
        }
        __syncthreads();
        // GEMM2 (volume part): acc += G[rows, 3w] [D^T chunk]; full chunks unrolled
        contract(sG, C::LDG, (size_t)C::R * C::LDG, (3 * w) / 8, 3 * C::CH / 8, fb2);
      }
      __syncthreads();  // the face phase reuses the volume buffers

      // ---- surface: chunks of FCH face nodes ---------------------------------
      double* sF = sWork;
#pragma unroll 1
      for (int fc = 0; fc < C::NFCH; ++fc) {
        const int f0 = fc * C::FCH;
        const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
        const int wp = round_up(wr, 8);
#pragma unroll 1
        for (int it = 0; it < C::IT_F; ++it) {
          const int idx = tid + it * C::NTH;
          if (idx >= C::E * wp) continue;
          const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
          double* gout = sF + (e * 5) * C::LDF + fl;
          const int ce = c0 + e, eg = sId[e];
          if (ce >= cp.Kc || fl >= wr) {
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
              for (int c = 0; c < 5; ++c) gout[a * C::R * C::LDF + c * C::LDF] = 0.0;
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
                gout[ma * C::R * C::LDF + c * C::LDF] = -fn.w * (0.5 * (se * umv[c] + snb * upv[c]) * nrm[ma]);
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
        __syncthreads();
        contract(sF, C::LDF, (size_t)C::R * C::LDF, wp / 8, C::FCH / 8,
                 fb2all + (size_t)((C::K2CUB + f0) / 8) * C::NT2 * 32);
        __syncthreads();  // sF is rewritten by the next chunk / the vol panel
      }

      // ---- epilogue: vol -> smem, M_e^-1 vol -> update / rhs / q_m ------------
      double* sV = sWork;  // [NA][R][LDV]
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int nt = 0; nt < C::NT2; ++nt) {
          const int col = nt * 8 + 2 * tq;
          double* va = sV + (size_t)a * C::R * L::LDV;
          va[lr_lo * L::LDV + col] = acc[a][nt][0];
          va[lr_lo * L::LDV + col + 1] = acc[a][nt][1];
          va[lr_hi * L::LDV + col] = acc[a][nt][2];
          va[lr_hi * L::LDV + col + 1] = acc[a][nt][3];
        }
      __syncthreads();
      double a_c = 0.0, b_c = 0.0, dt = 0.0;
      if (UPD) {
        a_c = p.coef->a[p.stage];
        b_c = p.coef->b[p.stage];
        dt = p.coef->dt;
      }
      // one thread per (element, node i): out_f(i) = sum_j (M_e^-1)[i][j] vol_f(j)
      // for the five fields (AUX: of the three directions, one column stream of
      // M_e^-1). The column stream is software-pipelined in groups of MG (the
      // next group's loads are in flight while the current one is consumed);
      // res and u are loaded up front, before the sums.
      constexpr int MG = 7, NGR = ceil_div(C::NP, MG);
      for (int idx = tid; idx < C::E * C::NP; idx += C::NTH) {
        const int e = idx / C::NP, i = idx - e * C::NP;
        const int ce = c0 + e;
        if (ce >= cp.Kc) continue;
        const double* mcol = cp.minv + (size_t)ce * C::NP * C::NP + i;  // (M_e^-1)[i][j] at j*NP + i
        const double* v = sV + (e * 5) * L::LDV;
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
                for (int f = 0; f < 5; ++f) out[a][f] += m[k] * v[(size_t)a * C::R * L::LDV + f * L::LDV + j0 + k];
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
      __syncthreads();  // sWork is reused by the next tile
    }
  }
}

}  // namespace cdg_gpu
