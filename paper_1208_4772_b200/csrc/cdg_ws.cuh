// cdg_ws.cuh -- warp-specialised fused RHS + LSRK kernel (inviscid path).
//
// Same math and data layout as k_rhs (cdg_kernels.cuh), but the CTA is split
// into 4 "MMA" warps (GEMM1 U_cub = U I_cub^T and GEMM2 acc += G Op2^T on the
// FP64 tensor pipe, plus the epilogue) and 4 "SIMT" warps (pointwise Euler
// flux at cubature nodes and the Riemann fluxes at face nodes). Chunks flow
// through double-buffered shared panels (sC: U at cubature nodes, sG: the A
// operand of GEMM2) guarded by named barriers, so the tensor pipe works on
// chunk k while the SIMT warps produce chunk k+1 -- the serial
// GEMM -> __syncthreads -> SIMT -> __syncthreads schedule of k_rhs left the
// DMMA pipe idle ~50% of the time (profiles/r1).
#pragma once

#include "cdg_kernels.cuh"

namespace cdg_gpu {

__device__ __forceinline__ void nb_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <class C>
struct WsLayout {
  static constexpr int MW = 4;  // MMA warps (0..3); SIMT warps 4..7
  static constexpr int NITEMS = C::NCH + C::NFCH;
  static constexpr int T2W = ceil_div(C::T2, MW);          // GEMM2 tiles per MMA warp
  static constexpr int T1 = C::MT * (C::CH / 8);
  static constexpr int T1W = ceil_div(T1, MW);
  static constexpr size_t SMEM_BYTES =
      sizeof(double) * (C::SMEM_U + 2 * C::SMEM_C + 2 * C::SMEM_G + C::E * 9 + C::E * 4 * 4) +
      sizeof(int) * (C::E * 4 * 2);
  // named barrier ids (0 is __syncthreads)
  static constexpr int CF = 1, CE = 3, GF = 5, GE = 7;
  static constexpr int NB = kThreads;  // all 8 warps take part in every handoff
};

template <class C>
__global__ void __launch_bounds__(kThreads, C::MINB) k_rhs_ws(RhsParams p) {
  using L = WsLayout<C>;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  double* sC = sU + C::SMEM_U;                 // [2][R][LDC]
  double* sG = sC + 2 * C::SMEM_C;             // [2][R][LDG]
  double* sMet = sG + 2 * C::SMEM_G;
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);
  int2* sConn = reinterpret_cast<int2*>(sFace + C::E * 4);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const bool is_mma = warp < L::MW;
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const double2* fb1 = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fb2 = reinterpret_cast<const double2*>(p.frag_op2);
  const int mw = warp;                              // MMA warp index
  const int t_begin = (mw * C::T2) / L::MW, t_end = ((mw + 1) * C::T2) / L::MW;
  const int st = tid - L::MW * 32;                  // SIMT thread index 0..127

  __shared__ int s_stop;
  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    // block-uniform early exit after a recorded error (no divergent barriers)
    if (tid == 0) s_stop = *(volatile int*)&p.err->flag;
    __syncthreads();
    if (s_stop) return;
    const int e0 = tile * C::E, row0 = e0 * 5;
    stage_rows<C>(p.u, row0, n_rows, sU, tid);
    for (int idx = tid; idx < C::E * 9; idx += kThreads)
      sMet[idx] = e0 + idx / 9 < p.K ? __ldg(p.metric + (size_t)e0 * 9 + idx) : 0.0;
    for (int idx = tid; idx < C::E * 4; idx += kThreads) {
      const bool ok = e0 + idx / 4 < p.K;
      sFace[idx] = ok ? p.face[(size_t)e0 * 4 + idx] : make_double4(0, 0, 1, 0);
      sConn[idx] = ok ? p.conn[(size_t)e0 * 4 + idx] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    __syncthreads();

    if (is_mma) {
      // ===================== MMA warps =====================================
      double acc[L::T2W][4];
#pragma unroll
      for (int i = 0; i < L::T2W; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
      auto gemm1 = [&](int item) {
        const int q0 = item * C::CH;
        const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;
        const int nt1 = w / 8, T1 = C::MT * nt1;
        double* dst = sC + (item & 1) * C::SMEM_C;
        double c[L::T1W][4];
#pragma unroll
        for (int i = 0; i < L::T1W; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks)
#pragma unroll
          for (int i = 0; i < L::T1W; ++i) {
            const int t = mw + i * L::MW;
            if (t < T1) {
              const int mt = t / nt1, nt = t % nt1;
              mma_frag(c[i], load_afrag(sU, C::LDU, mt * 16, ks * 8, g, tq),
                       __ldg(fb1 + ((size_t)(q0 / 8 + nt) * C::KS1 + ks) * 32 + lane));
            }
          }
#pragma unroll
        for (int i = 0; i < L::T1W; ++i) {
          const int t = mw + i * L::MW;
          if (t < T1) {
            const int mt = t / nt1, nt = t % nt1;
            double* o = dst + (mt * 16 + g) * C::LDC + nt * 8 + 2 * tq;
            *reinterpret_cast<double2*>(o) = make_double2(c[i][0], c[i][1]);
            *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c[i][2], c[i][3]);
          }
        }
      };
      gemm1(0);
      nb_arrive(L::CF + 0, L::NB);
      for (int k = 0; k < L::NITEMS; ++k) {
        if (k + 1 < C::NCH) {
          if (k + 1 >= 2) nb_sync(L::CE + ((k + 1) & 1), L::NB);
          gemm1(k + 1);
          nb_arrive(L::CF + ((k + 1) & 1), L::NB);
        }
        nb_sync(L::GF + (k & 1), L::NB);
        const double* a_src = sG + (k & 1) * C::SMEM_G;
        int ks0, nks;
        if (k < C::NCH) {
          const int q0 = k * C::CH;
          const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;
          ks0 = (3 * q0) / 8;
          nks = (3 * w) / 8;
        } else {
          const int f0 = (k - C::NCH) * C::FCH;
          const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
          ks0 = (C::K2CUB + f0) / 8;
          nks = round_up(wr, 8) / 8;
        }
        for (int ks = 0; ks < nks; ++ks) {
#pragma unroll
          for (int i = 0; i < L::T2W; ++i) {
            const int t = t_begin + i;
            if (t < t_end) {
              const int nt = t / C::MT, mt = t % C::MT;
              mma_frag(acc[i], load_afrag(a_src, C::LDG, mt * 16, ks * 8, g, tq),
                       __ldg(fb2 + ((size_t)nt * C::KS2 + ks0 + ks) * 32 + lane));
            }
          }
        }
        if (k + 2 < L::NITEMS) nb_arrive(L::GE + (k & 1), L::NB);
      }
      // ---- epilogue: res = a res + dt rhs; u += b res ----------------------
      const double a_c = p.coef->a[p.stage], b_c = p.coef->b[p.stage], dt = p.coef->dt;
#pragma unroll
      for (int i = 0; i < L::T2W; ++i) {
        const int t = t_begin + i;
        if (t < t_end) {
          const int nt = t / C::MT, mt = t % C::MT;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int r = mt * 16 + g + 8 * hh;
            const int grow = row0 + r;
            const int col = nt * 8 + 2 * tq;
            if (grow >= n_rows || col >= C::NP) continue;
            if (sConn[(r / 5) * 4].y & kCurvedBit) continue;
            const size_t gi = (size_t)grow * C::BP + col;
            const double r0 = acc[i][2 * hh], r1 = acc[i][2 * hh + 1];
            if (col + 1 < C::NP) {
              const double2 rs = *reinterpret_cast<const double2*>(p.res + gi);
              const double n0 = a_c * rs.x + dt * r0, n1 = a_c * rs.y + dt * r1;
              *reinterpret_cast<double2*>(p.res + gi) = make_double2(n0, n1);
              *reinterpret_cast<double2*>(p.u + gi) = make_double2(sU[r * C::LDU + pcol(col)] + b_c * n0,
                                                                     sU[r * C::LDU + pcol(col + 1)] + b_c * n1);
            } else {
              const double n0 = a_c * p.res[gi] + dt * r0;
              p.res[gi] = n0;
              p.u[gi] = sU[r * C::LDU + pcol(col)] + b_c * n0;
            }
          }
        }
      }
    } else {
      // ===================== SIMT warps ====================================
      for (int k = 0; k < L::NITEMS; ++k) {
        if (k >= 2) nb_sync(L::GE + (k & 1), L::NB);
        double* gdst = sG + (k & 1) * C::SMEM_G;
        if (k < C::NCH) {
          nb_sync(L::CF + (k & 1), L::NB);
          const double* csrc = sC + (k & 1) * C::SMEM_C;
          const int q0 = k * C::CH;
          const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;
          for (int idx = st; idx < C::E * w; idx += 128) {
            const int e = idx / w, ql = idx - e * w, q = q0 + ql;
            const double* uc = csrc + (e * 5) * C::LDC + ql;
            double G[3][5];
            if (q < C::NCUB && e0 + e < p.K) {
              const State5 s{uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
              if (!admissible(s, gamma)) record_error(p.err, 1, p.elem_offset + e0 + e, q, 0, s.r);
              const double ir = 1.0 / s.r;
              const double pr = (gamma - 1.0) * (s.E - 0.5 * ir * (s.mx * s.mx + s.my * s.my + s.mz * s.mz));
              const double vx = s.mx * ir, vy = s.my * ir, vz = s.mz * ir;
              const double ep = s.E + pr;
              const double* met = sMet + e * 9;
#pragma unroll
              for (int m = 0; m < 3; ++m) {
                const double r0 = met[m * 3 + 0], r1 = met[m * 3 + 1], r2 = met[m * 3 + 2];
                const double um = r0 * vx + r1 * vy + r2 * vz;  // contravariant velocity
                G[m][0] = s.r * um;
                G[m][1] = s.mx * um + pr * r0;
                G[m][2] = s.my * um + pr * r1;
                G[m][3] = s.mz * um + pr * r2;
                G[m][4] = ep * um;
              }
            } else {
#pragma unroll
              for (int m = 0; m < 3; ++m)
#pragma unroll
                for (int c = 0; c < 5; ++c) G[m][c] = 0.0;
            }
            double* gout = gdst + (e * 5) * C::LDG;
#pragma unroll
            for (int m = 0; m < 3; ++m) {
              const int col = pcol(m * w + ql);
#pragma unroll
              for (int c = 0; c < 5; ++c) gout[c * C::LDG + col] = G[m][c];
            }
          }
          if (k + 2 < C::NCH) nb_arrive(L::CE + (k & 1), L::NB);
        } else {
          const int f0 = (k - C::NCH) * C::FCH;
          const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
          const int wp = round_up(wr, 8);
          for (int idx = st; idx < C::E * wp; idx += 128) {
            const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
            double* gout = gdst + (e * 5) * C::LDG + pcol(fl);
            const int eg = e0 + e;
            if (eg >= p.K || fl >= wr) {
#pragma unroll
              for (int c = 0; c < 5; ++c) gout[c * C::LDG] = 0.0;
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
            if (p.gas.riemann == 1)
              hllc_flux(um, up, fn.x, fn.y, fn.z, gamma, fs);
            else
              llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
#pragma unroll
            for (int c = 0; c < 5; ++c) gout[c * C::LDG] = fn.w * fs[c];
          }
        }
        nb_arrive(L::GF + (k & 1), L::NB);
      }
    }
    __syncthreads();
  }
}

}  // namespace cdg_gpu
