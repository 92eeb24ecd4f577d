// cdg_sp.cuh -- software-pipelined fused RHS + LSRK kernel (inviscid path).
//
// Same math, layout and operators as k_rhs (cdg_kernels.cuh). The chunk loop
// is pipelined over double-buffered panels so that ONE iteration issues
//   A: GEMM2(k)    acc += sG[k%2] * Op2^T          (tensor pipe)
//   B: SIMT(k+1)   pointwise flux / Riemann flux -> sG[(k+1)%2]
//   C: GEMM1(k+2)  sC[k%2] = U * I_cub^T           (tensor pipe)
// with a single __syncthreads per chunk. A, B and C touch disjoint buffers,
// and with compile-time chunk widths the iteration is one basic block, so
// the scheduler interleaves the DMMA stream with the FP64/LSU work of the
// flux evaluation instead of serialising GEMM -> barrier -> SIMT -> barrier.
#pragma once

#include "cdg_kernels.cuh"

namespace cdg_gpu {

template <class C>
struct SpLayout {
  static constexpr int NITEMS = C::NCH + C::NFCH;
  static constexpr size_t SMEM_BYTES =
      sizeof(double) * (C::SMEM_U + 2 * C::SMEM_C + 2 * C::SMEM_G + C::E * 9 + C::E * 4 * 4) +
      sizeof(int) * (C::E * 4 * 2);
  __host__ __device__ static constexpr int cub_w(int k) {
    return (C::NCUB8 - k * C::CH) < C::CH ? (C::NCUB8 - k * C::CH) : C::CH;
  }
  __host__ __device__ static constexpr int face_wr(int j) {
    return (C::NF - j * C::FCH) < C::FCH ? (C::NF - j * C::FCH) : C::FCH;
  }
};

template <class C, int K, bool LAST>
struct SpItem;  // (helpers are written inline below)

template <class C, bool UPDATE>
__global__ void __launch_bounds__(kThreads, C::MINB) k_rhs_sp(RhsParams p) {
  using L = SpLayout<C>;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  double* sC = sU + C::SMEM_U;      // [2][R][LDC]
  double* sG = sC + 2 * C::SMEM_C;  // [2][R][LDG]
  double* sMet = sG + 2 * C::SMEM_G;
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);
  int2* sConn = reinterpret_cast<int2*>(sFace + C::E * 4);
  __shared__ int s_stop;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const double2* fb1 = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fb2 = reinterpret_cast<const double2*>(p.frag_op2);
  const int t_begin = (warp * C::T2) / kWarps, t_end = ((warp + 1) * C::T2) / kWarps;

  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
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

    // ---- stage helpers ----------------------------------------------------
    auto gemm1 = [&](int k) {  // sC[k%2] = U * I_cub[q0:q0+w]^T
      const int q0 = k * C::CH, w = L::cub_w(k), nt1 = w / 8, T1 = C::MT * nt1;
      double* dst = sC + (k & 1) * C::SMEM_C;
      double c[C::MAXT1][4];
#pragma unroll
      for (int i = 0; i < C::MAXT1; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks)
#pragma unroll
        for (int i = 0; i < C::MAXT1; ++i) {
          const int t = warp + i * kWarps;
          if (t < T1)
            mma_frag(c[i], load_afrag(sU, C::LDU, (t / nt1) * 16, ks * 8, g, tq),
                     __ldg(fb1 + ((size_t)(q0 / 8 + t % nt1) * C::KS1 + ks) * 32 + lane));
        }
#pragma unroll
      for (int i = 0; i < C::MAXT1; ++i) {
        const int t = warp + i * kWarps;
        if (t < T1) {
          double* o = dst + ((t / nt1) * 16 + g) * C::LDC + (t % nt1) * 8 + 2 * tq;
          *reinterpret_cast<double2*>(o) = make_double2(c[i][0], c[i][1]);
          *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c[i][2], c[i][3]);
        }
      }
    };
    auto pointwise = [&](int k) {  // sC[k%2] -> sG[k%2]
      const int q0 = k * C::CH, w = L::cub_w(k);
      const double* csrc = sC + (k & 1) * C::SMEM_C;
      double* gdst = sG + (k & 1) * C::SMEM_G;
#pragma unroll
      for (int it = 0; it < C::IT_P; ++it) {
        const int idx = tid + it * kThreads;
        if (idx < C::E * w) {
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
              const double um = r0 * vx + r1 * vy + r2 * vz;
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
      }
    };
    auto faceflux = [&](int k) {  // face chunk j = k - NCH -> sG[k%2]
      const int j = k - C::NCH, f0 = j * C::FCH, wr = L::face_wr(j), wp = round_up(wr, 8);
      double* gdst = sG + (k & 1) * C::SMEM_G;
#pragma unroll
      for (int it = 0; it < C::IT_F; ++it) {
        const int idx = tid + it * kThreads;
        if (idx >= C::E * wp) continue;
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
    };

    double acc[C::MAXT2][4];
#pragma unroll
    for (int i = 0; i < C::MAXT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
    auto gemm2 = [&](int k) {  // acc += sG[k%2] * Op2[:, item k]^T
      const double* a_src = sG + (k & 1) * C::SMEM_G;
      const int ks0 = k < C::NCH ? (3 * k * C::CH) / 8 : (C::K2CUB + (k - C::NCH) * C::FCH) / 8;
      const int nks = k < C::NCH ? (3 * L::cub_w(k)) / 8 : round_up(L::face_wr(k - C::NCH), 8) / 8;
#pragma unroll
      for (int ks = 0; ks < nks; ++ks)
#pragma unroll
        for (int i = 0; i < C::MAXT2; ++i) {
          const int t = t_begin + i;
          if (t < t_end) {
            const int nt = t / C::MT, mt = t % C::MT;
            mma_frag(acc[i], load_afrag(a_src, C::LDG, mt * 16, ks * 8, g, tq),
                     __ldg(fb2 + ((size_t)nt * C::KS2 + ks0 + ks) * 32 + lane));
          }
        }
    };

    // ---- prologue -------------------------------------------------------------
    gemm1(0);
    if (C::NCH > 1) gemm1(1);
    __syncthreads();
    pointwise(0);
    __syncthreads();
    // ---- pipelined items --------------------------------------------------------
#pragma unroll
    for (int k = 0; k < L::NITEMS; ++k) {
      gemm2(k);
      if (k + 1 < C::NCH)
        pointwise(k + 1);
      else if (k + 1 < L::NITEMS)
        faceflux(k + 1);
      if (k + 2 < C::NCH) gemm1(k + 2);
      __syncthreads();
    }

    // ---- epilogue --------------------------------------------------------------
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
#pragma unroll
    for (int i = 0; i < C::MAXT2; ++i) {
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
            if (UPDATE) {
              const double2 rs = *reinterpret_cast<const double2*>(p.res + gi);
              const double n0 = a_c * rs.x + dt * r0, n1 = a_c * rs.y + dt * r1;
              *reinterpret_cast<double2*>(p.res + gi) = make_double2(n0, n1);
              *reinterpret_cast<double2*>(p.u + gi) = make_double2(sU[r * C::LDU + pcol(col)] + b_c * n0,
                                                                     sU[r * C::LDU + pcol(col + 1)] + b_c * n1);
            } else {
              *reinterpret_cast<double2*>(p.rhs_out + gi) = make_double2(r0, r1);
            }
          } else {
            if (UPDATE) {
              const double n0 = a_c * p.res[gi] + dt * r0;
              p.res[gi] = n0;
              p.u[gi] = sU[r * C::LDU + pcol(col)] + b_c * n0;
            } else {
              p.rhs_out[gi] = r0;
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace cdg_gpu
