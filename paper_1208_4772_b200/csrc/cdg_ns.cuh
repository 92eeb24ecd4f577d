// cdg_ns.cuh -- neighbour-state RHS + LSRK kernel for low-order affine levels.
//
// Same math as k_rhs_warp (cdg_warp.cuh; reference solver.cpp:200-208,
// 325-492) on the same warp tile of 16 elements, with the face data read a
// different way. The reference interpolates every element's state to its face
// nodes (interpolate_to_faces) and the surface loop reads the neighbour's
// TRACE through the node map. At p <= 2 the whole nodal state (K x 5 x N_p
// doubles: 82 MB for the 511k-tet order sweep at p=1) fits the B200's 126 MB
// L2, while the traces are 3x (p=1) / 2.4x (p=2) larger than the state and
// make a write + two reads through HBM per stage. Here no trace is stored:
//
//   own trace      u_e(x_fq)  = sum_j I_g[fq][j] U_e[j]        (staged U, smem)
//   neighbour      u_n(x_h)   = sum_j I_g[f' N_g + h][j] U_n[j] (U_n: L2)
//
// with h = code_map[...][gq] the same node pairing the stored traces use.
// The stage reads the stage-start state u_in (neighbours included) and writes
// the new state to u_out (ping-pong buffers, swapped by the driver), so no
// element's update can race a neighbour's read. Each warp stages its tile
// (compact U rows, metrics, face connectivity and geometry: 6.3 KB at p=1)
// with cp.async; shared memory stays at 100 KB per SM so the L1 keeps ~150 KB
// for the neighbour-row gathers (staging the NEXT tile too -- 200 KB per SM --
// measured 26% slower, profiles/r2/ns_experiment.md).
//
// Measured at p=1 only (make_cube_mesh(44)): 0.333 vs 0.372 ms per stage
// (LLF), 0.452 vs 0.492 (HLLC); at p=2 the per-node interpolation (2 x 5 x 10
// FMAs + 25 neighbour-row loads per face node) makes it 40% slower than the
// stored-trace row kernel, so p=2 keeps the traces.
//
// The traces are sums in a different order than the DMMA trace kernel's, so
// this path agrees with the stored-trace paths to rounding, not bit for bit;
// CDG_GPU_PATH_TRACED selects the stored-trace kernels (bitwise-comparison
// tests).
#pragma once

#include "cdg_warp.cuh"

namespace cdg_gpu {

template <int NP_, int NCUB_, int NG_, int WARPS_ = 4, int MINB_ = 4>
struct NsCfg {
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int EW = 16, WARPS = WARPS_, MINB = MINB_;
  static constexpr int BP = dev_block(NP);
  static constexpr int KP = round_up(NP, 8), KS1 = KP / 8, NT = KP / 8;
  static constexpr int NCH = ceil_div(NCUB, 8), NFCH = ceil_div(NF, 8);
  static constexpr int VP = (NP + 1) / 2;  // live 16-byte pieces of a U row
  static constexpr int LDU = 2 * VP;       // compact rows: the k-step padding is masked in registers
  // one staging buffer (doubles): U rows [5][16][LDU] | metrics [16][9] |
  // conn int2 [16][4] | face double4 [16][4]
  static constexpr int U_D = 5 * EW * LDU, MET_D = EW * 9, CONN_D = EW * 4, FACE_D = EW * 4 * 4;
  static constexpr int BUF_D = round_up(U_D + MET_D + CONN_D + FACE_D, 4);
  static constexpr int IG_D = round_up(NF * NP, 4);  // I_g, row-major [NF][NP]
  static constexpr size_t SMEM_BYTES = sizeof(double) * ((size_t)IG_D + (size_t)WARPS * BUF_D);
  static_assert((U_D + MET_D + CONN_D) % 4 == 0, "32-byte alignment of the double4 face block");
};

__device__ __forceinline__ void cp_async16_n(void* smem, const void* gmem, int nbytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(nbytes));
}

// stage one 16-element tile into a buffer (the warp's lanes, cp.async)
template <class C>
__device__ __forceinline__ void ns_stage(const WarpParams& p, double* buf, int e0, int lane) {
  double* sU = buf;
  double* sMet = buf + C::U_D;
  double* sConn = sMet + C::MET_D;
  double* sFace = sConn + C::CONN_D;
  const int ne = min(C::EW, p.K - e0);
  for (int idx = lane; idx < 5 * C::EW * C::VP; idx += 32) {
    const int r = idx / C::VP, j = idx - r * C::VP;
    const int c = r / C::EW, e = r - c * C::EW;
    const bool ok = e < ne;
    cp_async16(sU + r * C::LDU + 2 * j, p.u + ((size_t)(ok ? e0 + e : 0) * 5 + c) * C::BP + 2 * j, ok);
  }
  {  // metrics: 9 doubles per element, contiguous (the tail piece may be half valid)
    const double* src = p.metric + (size_t)e0 * 9;
    const int nd = ne * 9;
    for (int i = lane; i < C::MET_D / 2; i += 32) {
      const int left = nd - 2 * i;
      cp_async16_n(sMet + 2 * i, left > 0 ? src + 2 * i : p.metric, left >= 2 ? 16 : left == 1 ? 8 : 0);
    }
  }
  for (int i = lane; i < C::CONN_D / 2; i += 32) {  // conn: 2 faces (2 int2) per piece
    const bool ok = i / 2 < ne;
    cp_async16(sConn + 2 * i, reinterpret_cast<const double*>(p.conn + (size_t)e0 * 4) + (ok ? 2 * i : 0), ok);
  }
  for (int i = lane; i < C::FACE_D / 2; i += 32) {  // face: one (n, sjac/J) per 2 pieces
    const bool ok = i / 8 < ne;
    cp_async16(sFace + 2 * i, reinterpret_cast<const double*>(p.face + (size_t)e0 * 4) + (ok ? 2 * i : 0), ok);
  }
}

template <class C, int RIEMANN>
__global__ void __launch_bounds__(32 * C::WARPS, C::MINB) k_rhs_ns(WarpParams p) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* sIg = smem;
  double* const sbuf = smem + C::IG_D + (size_t)warp * C::BUF_D;
  for (int i = threadIdx.x; i < C::NF * C::NP; i += blockDim.x) sIg[i] = __ldg(p.ig + i);
  __syncthreads();
  const double gamma = p.gas.gamma;
  const int n_tiles = (p.K + C::EW - 1) / C::EW;
  const int warps_total = gridDim.x * C::WARPS;
  const double* u_in = p.u;  // stage-start state: own and neighbour rows (never written here)
  const double a_c = p.coef->a[p.stage], b_c = p.coef->b[p.stage], dt = p.coef->dt;

  for (int tile = blockIdx.x * C::WARPS + warp; tile < n_tiles; tile += warps_total) {
    if (*(volatile int*)&p.err->flag) return;  // warp-uniform: no barrier to desynchronise
    ns_stage<C>(p, sbuf, tile * C::EW, lane);
    cp_async_wait_all();
    __syncwarp();
    const double* sU = sbuf;
    const double* sMet = sU + C::U_D;
    const int2* sConn = reinterpret_cast<const int2*>(sMet + C::MET_D);
    const double4* sFace = reinterpret_cast<const double4*>(sMet + C::MET_D + C::CONN_D);
    const int e0 = tile * C::EW;
    const bool ev0 = e0 + g < p.K, ev1 = e0 + g + 8 < p.K;

    double acc[5][C::NT][4];
#pragma unroll
    for (int c = 0; c < 5; ++c)
#pragma unroll
      for (int n = 0; n < C::NT; ++n) acc[c][n][0] = acc[c][n][1] = acc[c][n][2] = acc[c][n][3] = 0.0;

    // ---- volume (k_rhs_warp's mapping) --------------------------------------
#pragma unroll 1
    for (int ch = 0; ch < C::NCH; ++ch) {
      double uc[5][4];
#pragma unroll
      for (int c = 0; c < 5; ++c) uc[c][0] = uc[c][1] = uc[c][2] = uc[c][3] = 0.0;
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) {
        const double2 b = __ldg(p.frag1 + ((size_t)ch * C::KS1 + ks) * 32 + lane);
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double2 x = make_double2(0.0, 0.0), y = x;
          if (ks * 8 + 2 * t < C::NP) {  // columns past N_p: zeros of the k-step
            const double* s = sU + (c * C::EW + g) * C::LDU + ks * 8 + 2 * t;
            x = *reinterpret_cast<const double2*>(s);
            y = *reinterpret_cast<const double2*>(s + 8 * C::LDU);
          }
          dmma_k8(uc[c], x.x, y.x, x.y, y.y, b.x, b.y);
        }
      }
      const int q = ch * 8 + 2 * t;
      const bool vq0 = q < C::NCUB, vq1 = q + 1 < C::NCUB;
      const bool valid[4] = {ev0 && vq0, ev0 && vq1, ev1 && vq0, ev1 && vq1};
      double pr[4], vx[4], vy[4], vz[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const State5 s{uc[0][j], uc[1][j], uc[2][j], uc[3][j], uc[4][j]};
        if (valid[j] && !admissible(s, gamma))
          record_error(p.err, 1, p.elem_offset + e0 + g + 8 * (j >> 1), q + (j & 1), 0, s.r);
        const double ir = 1.0 / (valid[j] ? s.r : 1.0);
        pr[j] = valid[j] ? (gamma - 1.0) * (s.E - 0.5 * ir * (s.mx * s.mx + s.my * s.my + s.mz * s.mz)) : 0.0;
        vx[j] = s.mx * ir;
        vy[j] = s.my * ir;
        vz[j] = s.mz * ir;
        uc[4][j] += pr[j];  // E + p
      }
#pragma unroll 1
      for (int m = 0; m < 3; ++m) {
        double2 b[C::NT];
#pragma unroll
        for (int n = 0; n < C::NT; ++n) b[n] = __ldg(p.frag2v + (((size_t)ch * 3 + m) * C::NT + n) * 32 + lane);
        const double* m0 = sMet + g * 9 + m * 3;
        const double* m1 = sMet + (g + 8) * 9 + m * 3;
        const double r00 = m0[0], r01 = m0[1], r02 = m0[2], r10 = m1[0], r11 = m1[1], r12 = m1[2];
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
#pragma unroll
          for (int n = 0; n < C::NT; ++n) dmma_k8(acc[c][n], gv[0], gv[2], gv[1], gv[3], b[n].x, b[n].y);
        }
      }
    }

    // ---- surface: traces from the nodal states, chunks of 8 face nodes --------
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
        const int2 cw = sConn[e * 4 + f];
        const double4 fn = sFace[e * 4 + f];
        double mv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        {  // own trace: I_g row fq . U_e
          const double* ir = sIg + fq * C::NP;
#pragma unroll
          for (int k = 0; k < C::NP; ++k) {
            const double w = ir[k];
#pragma unroll
            for (int c = 0; c < 5; ++c) mv[c] = fma(w, sU[(c * C::EW + e) * C::LDU + k], mv[c]);
          }
        }
        const State5 um{mv[0], mv[1], mv[2], mv[3], mv[4]};
        State5 up;
        if (cw.x >= 0) {  // neighbour trace: I_g row (f', h) . U_n (L2-resident state)
          const int h = __ldg(p.code_map + (cw.y >> 8) * C::NG + gq);
          const double* nr = sIg + ((cw.y & 3) * C::NG + h) * C::NP;
          const double* un = u_in + (size_t)cw.x * 5 * C::BP;
          double pv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int k2 = 0; k2 < C::VP; ++k2) {
            const double w0 = nr[2 * k2], w1 = 2 * k2 + 1 < C::NP ? nr[2 * k2 + 1] : 0.0;
#pragma unroll
            for (int c = 0; c < 5; ++c) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(un + c * C::BP + 2 * k2));
              pv[c] = fma(w0, v.x, pv[c]);
              if (2 * k2 + 1 < C::NP) pv[c] = fma(w1, v.y, pv[c]);
            }
          }
          up = State5{pv[0], pv[1], pv[2], pv[3], pv[4]};
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

    // ---- epilogue: res = a res + dt rhs (in place); u_out = u_in + b res -------
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int e = g + 8 * hh, eg = e0 + e;
      if (eg >= p.K) continue;
      double2 rsv[5][C::NT];
#pragma unroll
      for (int c = 0; c < 5; ++c)
#pragma unroll
        for (int n = 0; n < C::NT; ++n)
          rsv[c][n] = n * 8 + 2 * t < C::NP
                          ? *reinterpret_cast<const double2*>(p.res + ((size_t)eg * 5 + c) * C::BP + n * 8 + 2 * t)
                          : make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const size_t rowoff = ((size_t)eg * 5 + c) * C::BP;
#pragma unroll
        for (int n = 0; n < C::NT; ++n) {
          const int col = n * 8 + 2 * t;
          if (col >= C::NP) continue;  // padding: never loaded, never stored
          const double2 rs = rsv[c][n];
          const double n0 = a_c * rs.x + dt * acc[c][n][2 * hh], n1 = a_c * rs.y + dt * acc[c][n][2 * hh + 1];
          *reinterpret_cast<double2*>(p.res + rowoff + col) = make_double2(n0, n1);
          const double2 uo = *reinterpret_cast<const double2*>(sU + (c * C::EW + e) * C::LDU + col);
          *reinterpret_cast<double2*>(p.u_out + rowoff + col) = make_double2(uo.x + b_c * n0, uo.y + b_c * n1);
        }
      }
    }
    __syncwarp();  // the buffer is restaged by the warp's next tile
  }
}

}  // namespace cdg_gpu
