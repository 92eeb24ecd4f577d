// cdg_ws.cuh -- warp-specialized RHS + LSRK kernel for affine tets (the P=4
// headline path): the same math, operators and per-element evaluation order
// per contraction as k_rhs_row (cdg_row.cuh; reference solver.cpp:325-492),
// mapped onto the SM as a producer / consumer pipeline instead of a
// CTA-barrier lock-step.
//
// Why: in k_rhs_row every warp alternates between DMMA contractions and SIMT
// pointwise / face-flux work, separated by two CTA barriers per 8-node
// cubature chunk; the DMMA pipe idles while the CTA's warps compute fluxes or
// wait for the slowest warp (ncu: 58% DMMA-busy, barrier stalls 30-44% of the
// GEMM phases, profiles/r1/ncu_k_rhs_row.txt).
//
// Here a CTA (one 16-element tile = 80 (element, field) rows at a time) has
//  * NMW = 5 MMA warps: warp w owns rows [16w, 16w+16) of every contraction
//    (A fragments reused across all N_p/8 n-tiles), keeps its rows of U in
//    registers for the whole tile, and only issues DMMA work + the epilogue
//    (LSRK update, next-stage traces u_new I_g^T from the registers);
//  * NFW flux warps: the pointwise Euler flux G_m = sum_d (dr_m/dx_d) F_d at
//    the cubature nodes and the face fluxes (gather, BC ghost, LLF / HLLC),
//    written to shared memory.
// Hand-offs use named barriers (bar.arrive by the producer role, bar.sync by
// the consumer role, every barrier counting all NTH threads) over
// double-buffered chunk panels: U_cub (MMA -> flux), G (flux -> MMA), face
// flux F* (flux -> MMA). Per tile the flux warps compute the tile's face
// fluxes FIRST -- they depend only on the traces, so they overlap the MMA
// warps' epilogue of the previous tile -- then the cubature chunks; the MMA
// warps contract the face chunks first, then stream GEMM1 of chunk c+2
// interleaved with GEMM2 of chunk c (two independent MMA streams per warp).
// Summation order per element: face block, then the cubature chunks in order
// (k_rhs_row sums the cubature chunks first), so results agree with k_rhs_row
// and the reference to rounding; the fused traces use the trace kernel's
// pairing, so they stay bit-identical to k_interp<NAT>.
#pragma once

#include "cdg_row.cuh"

namespace cdg_gpu {

__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <int NP_, int NCUB_, int NG_, int CH_ = 8, int FCH_ = 32, int NFW_ = 4, int MINB_ = 2>
struct WsCfg {
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int E = 16, R = 5 * E, NMW = R / 16, NFW = NFW_;
  static constexpr int NTH = 32 * (NMW + NFW_), NFT = 32 * NFW_, MINB = MINB_;
  // registers per thread for MINB resident CTAs (8-register allocation units)
  static constexpr int MAXREG = (65536 / (MINB_ * NTH)) / 8 * 8 > 255 ? 255 : (65536 / (MINB_ * NTH)) / 8 * 8;
  static constexpr int BP = dev_block(NP), TB = dev_block(NF);
  static constexpr int KP = round_up(NP, 8), KS1 = KP / 8, NT2 = KS1;
  static constexpr int NCUB8 = round_up(NCUB, 8), NF8 = round_up(NF, 8);
  static constexpr int CH = CH_, NCH = ceil_div(NCUB8, CH);
  static constexpr int FCH = FCH_, NFCH = ceil_div(NF, FCH);
  static constexpr int K2CUB = 3 * NCUB8, K2 = K2CUB + NF8;
  static constexpr int LDC = frag_ld8(CH), LDG = frag_ld8(3 * CH), LDF = frag_ld8(FCH);
  static constexpr int IT_P = ceil_div(E * CH, NFT), IT_F = ceil_div(E * FCH, NFT);
  static constexpr size_t SMEM_BYTES =
      sizeof(double) * ((size_t)2 * R * (LDC + LDG + LDF) + E * 9 + E * 4 * 4) + sizeof(int) * (E * 4 * 2);
  static_assert(NCH >= 2, "the MMA warps prefetch two cubature chunks");
  static_assert(NTH <= 1024, "CTA size");
};

// named barrier ids (0 is __syncthreads); [b] = buffer parity
enum : int { kBarCFull = 1, kBarCEmpty = 3, kBarGFull = 5, kBarGEmpty = 7, kBarFFull = 9, kBarFEmpty = 11, kBarFlux = 13 };

template <class C, bool UPDATE, int RM>
__global__ void __launch_bounds__(C::NTH) __maxnreg__(C::MAXREG) k_rhs_ws(RhsParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sC = smem;                                            // [2][R][LDC] U at the chunk's cubature nodes
  double* sG = sC + 2 * C::R * C::LDC;                          // [2][R][LDG] contravariant flux of the chunk
  double* sF = sG + 2 * C::R * C::LDG;                          // [2][R][LDF] (sjac/J) F* of the face chunk
  double* sMet = sF + 2 * C::R * C::LDF;                        // [E][9]  (flux warps)
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);  // [E][4]
  int2* sConn = reinterpret_cast<int2*>(sFace + C::E * 4);       // [E][4]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const int n_tiles = (p.K + C::E - 1) / C::E;
  const int n_iter = p.tiles ? p.n_list : n_tiles;
  constexpr int NTH = C::NTH;

  if (warp < C::NMW) {
    // =========================== MMA warps ====================================
    const int g = lane >> 2, tq = lane & 3;
    // the G and F* buffers start empty (their producers sync on these)
    nbar_arrive(kBarGEmpty + 0, NTH);
    nbar_arrive(kBarGEmpty + 1, NTH);
    nbar_arrive(kBarFEmpty + 0, NTH);
    nbar_arrive(kBarFEmpty + 1, NTH);
    const double2* fb1all = reinterpret_cast<const double2*>(p.frag_icub);  // [NCUB8/8][KS1][32]
    const double2* fb2all = reinterpret_cast<const double2*>(p.frag_op2);   // [K2/8][NT2][32]
    int nc = 0, nf = 0;  // global cubature / face chunk counters (buffer parity)
    for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
      const int tile = tile_at(p, it_t);
      const int e0 = tile * C::E, row0 = e0 * 5;
      const int r_lo = row0 + warp * 16 + g, r_hi = r_lo + 8;  // this thread's two rows
      const bool ok_lo = r_lo < n_rows, ok_hi = r_hi < n_rows;
      // U rows -> registers: A fragments of GEMM1 for the whole tile (natural
      // pairing: k = t <-> node 8ks+2t, k = t+4 <-> 8ks+2t+1), and the old u of
      // the update
      double uA[C::KS1][4];
      {
        const double* u_lo = p.u + (size_t)min(r_lo, n_rows - 1) * C::BP + 2 * tq;
        const double* u_hi = p.u + (size_t)min(r_hi, n_rows - 1) * C::BP + 2 * tq;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks) {
          double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
          if (ok_lo) x = *reinterpret_cast<const double2*>(u_lo + ks * 8);
          if (ok_hi) y = *reinterpret_cast<const double2*>(u_hi + ks * 8);
          uA[ks][0] = x.x, uA[ks][1] = y.x, uA[ks][2] = x.y, uA[ks][3] = y.y;
        }
      }
      double acc[C::NT2][4];
#pragma unroll
      for (int i = 0; i < C::NT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;

      // GEMM1 of cubature chunk ch: c1 = U_rows I_cub[chunk]^T
      auto gemm1 = [&](int ch, double (&c1)[C::CH / 8][4]) {
        const int q0 = ch * C::CH, w = min(C::CH, C::NCUB8 - q0);
        const double2* fb1 = fb1all + (size_t)(q0 / 8) * C::KS1 * 32;
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j) c1[j][0] = c1[j][1] = c1[j][2] = c1[j][3] = 0.0;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks)
#pragma unroll
          for (int j = 0; j < C::CH / 8; ++j)
            if (j * 8 < w) {
              const double2 bf = __ldg(fb1 + (j * C::KS1 + ks) * 32 + lane);
              dmma_k8(c1[j], uA[ks][0], uA[ks][1], uA[ks][2], uA[ks][3], bf.x, bf.y);
            }
      };
      auto store_c = [&](int b, int ch, const double (&c1)[C::CH / 8][4]) {
        const int w = min(C::CH, C::NCUB8 - ch * C::CH);
        double* base = sC + (size_t)b * C::R * C::LDC;
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j)
          if (j * 8 < w) {
            double* o = base + (warp * 16 + g) * C::LDC + j * 8 + 2 * tq;
            *reinterpret_cast<double2*>(o) = make_double2(c1[j][0], c1[j][1]);
            *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c1[j][2], c1[j][3]);
          }
      };
      // acc += P[rows, 8 nks] Op[k0 : k0 + 8 nks]^T from the panel P (ld), k-steps unrolled when full
      auto contract = [&](const double* panel, int ld, int nks, int nks_full, const double2* fb2) {
        auto kstep = [&](int ks) {
          const AFrag a = load_afrag(panel, ld, warp * 16, ks * 8, g, tq);
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

      // prologue: U_cub of chunks 0 and 1 (both panels)
#pragma unroll 1
      for (int ch = 0; ch < 2; ++ch) {
        double c1[C::CH / 8][4];
        gemm1(ch, c1);
        const int b = (nc + ch) & 1;
        nbar_sync(kBarCEmpty + b, NTH);
        store_c(b, ch, c1);
        nbar_arrive(kBarCFull + b, NTH);
      }
      // surface: acc += F* (-LIFT)^T, face chunks in order (the flux warps compute them first)
#pragma unroll 1
      for (int fc = 0; fc < C::NFCH; ++fc) {
        const int b = (nf + fc) & 1, f0 = fc * C::FCH;
        const int wp = round_up(min(C::FCH, C::NF - f0), 8);
        nbar_sync(kBarFFull + b, NTH);
        contract(sF + (size_t)b * C::R * C::LDF, C::LDF, wp / 8, C::FCH / 8,
                 fb2all + (size_t)((C::K2CUB + f0) / 8) * C::NT2 * 32);
        nbar_arrive(kBarFEmpty + b, NTH);
      }
      nf += C::NFCH;
      // volume: GEMM2 of chunk ch interleaved with GEMM1 of chunk ch + 2
#pragma unroll 1
      for (int ch = 0; ch < C::NCH; ++ch) {
        const int b = (nc + ch) & 1, q0 = ch * C::CH;
        const int w = min(C::CH, C::NCUB8 - q0);
        const bool next = ch + 2 < C::NCH;
        nbar_sync(kBarGFull + b, NTH);
        double c1[C::CH / 8][4];
        if (next) gemm1(ch + 2, c1);
        contract(sG + (size_t)b * C::R * C::LDG, C::LDG, 3 * w / 8, 3 * C::CH / 8,
                 fb2all + (size_t)(3 * q0 / 8) * C::NT2 * 32);
        nbar_arrive(kBarGEmpty + b, NTH);
        if (next) {
          nbar_sync(kBarCEmpty + b, NTH);  // the flux warps are done with chunk ch's panel
          store_c(b, ch + 2, c1);
          nbar_arrive(kBarCFull + b, NTH);
        }
      }
      nc += C::NCH;

      // ---- epilogue: rhs -> (res, u) update or rhs store (+ next-stage traces)
      double a_c = 0.0, b_c = 0.0, dt = 0.0;
      if (UPDATE) {
        a_c = p.coef->a[p.stage];
        b_c = p.coef->b[p.stage];
        dt = p.coef->dt;
      }
      const int el_lo = min(r_lo, n_rows - 1) / 5, el_hi = min(r_hi, n_rows - 1) / 5;
      const bool cur_lo = (__ldg(&p.conn[(size_t)el_lo * 4].y) & kCurvedBit) != 0;
      const bool cur_hi = (__ldg(&p.conn[(size_t)el_hi * 4].y) & kCurvedBit) != 0;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int grow = hh ? r_hi : r_lo;
        if (grow >= n_rows || (hh ? cur_hi : cur_lo)) continue;  // curved rows: the curved kernel
        const size_t rowoff = (size_t)grow * C::BP;
        double2 rsv[C::NT2];
        if (UPDATE)  // every old res value of the row before any store (no serialised round trips)
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
      if (UPDATE && p.traces_out) {
        // next stage's traces T = u_new I_g^T (solver.cpp:200-208) from the registers
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int grow = hh ? r_hi : r_lo;
          if (grow >= n_rows || (hh ? cur_hi : cur_lo))
#pragma unroll
            for (int j = 0; j < C::NT2; ++j) acc[j][2 * hh] = acc[j][2 * hh + 1] = 0.0;
        }
        constexpr int NFT8 = C::NF8 / 8;
        const double2* fbi = reinterpret_cast<const double2*>(p.frag_ig_nat);  // [NFT8][KS1][32]
        AFrag fa[C::KS1];
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks) fa[ks] = AFrag{acc[ks][0], acc[ks][2], acc[ks][1], acc[ks][3]};
#pragma unroll
        for (int nt0 = 0; nt0 < NFT8; nt0 += 4) {
          double tacc[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i) tacc[i][0] = tacc[i][1] = tacc[i][2] = tacc[i][3] = 0.0;
#pragma unroll
          for (int ks = 0; ks < C::KS1; ++ks)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (nt0 + i < NFT8) mma_frag(tacc[i], fa[ks], __ldg(fbi + ((size_t)(nt0 + i) * C::KS1 + ks) * 32 + lane));
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int col = (nt0 + i) * 8 + 2 * tq;
            if (nt0 + i < NFT8 && col < C::NF) {
              if (r_lo < n_rows)
                *reinterpret_cast<double2*>(p.traces_out + (size_t)r_lo * C::TB + col) = make_double2(tacc[i][0], tacc[i][1]);
              if (r_hi < n_rows)
                *reinterpret_cast<double2*>(p.traces_out + (size_t)r_hi * C::TB + col) = make_double2(tacc[i][2], tacc[i][3]);
            }
          }
        }
      }
    }
  } else {
    // =========================== flux warps ===================================
    const int ft = tid - 32 * C::NMW;  // 0 .. NFT-1
    nbar_arrive(kBarCEmpty + 0, NTH);  // both U_cub panels start empty
    nbar_arrive(kBarCEmpty + 1, NTH);
    int nc = 0, nf = 0;
    for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
      const int tile = tile_at(p, it_t);
      const int e0 = tile * C::E;
      nbar_sync(kBarFlux, C::NFT);  // the previous tile's readers of sMet / sFace / sConn are done
      for (int idx = ft; idx < C::E * 9; idx += C::NFT)
        sMet[idx] = e0 + idx / 9 < p.K ? __ldg(p.metric + (size_t)e0 * 9 + idx) : 0.0;
      for (int idx = ft; idx < C::E * 4; idx += C::NFT) {
        const bool ok = e0 + idx / 4 < p.K;
        sFace[idx] = ok ? p.face[(size_t)e0 * 4 + idx] : make_double4(0, 0, 1, 0);
        sConn[idx] = ok ? p.conn[(size_t)e0 * 4 + idx] : make_int2(-1, pack_face(0, 0, 1, 0));
      }
      nbar_sync(kBarFlux, C::NFT);

      // ---- face fluxes: (sjac/J) F* per face node (solver.cpp:415-457)
#pragma unroll 1
      for (int fc = 0; fc < C::NFCH; ++fc) {
        const int b = (nf + fc) & 1, f0 = fc * C::FCH;
        const int wr = min(C::FCH, C::NF - f0), wp = round_up(wr, 8);
        double* sFb = sF + (size_t)b * C::R * C::LDF;
        nbar_sync(kBarFEmpty + b, NTH);
#pragma unroll 1
        for (int it = 0; it < C::IT_F; ++it) {
          const int idx = ft + it * C::NFT;
          if (idx >= C::E * wp) break;
          const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
          double* gout = sFb + (e * 5) * C::LDF + fl;
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
            hllc_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
          else
            llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
#pragma unroll
          for (int c = 0; c < 5; ++c) gout[c * C::LDF] = fn.w * fs[c];
        }
        nbar_arrive(kBarFFull + b, NTH);
      }
      nf += C::NFCH;

      // ---- pointwise Euler flux -> contravariant flux G_m per cubature chunk
#pragma unroll 1
      for (int ch = 0; ch < C::NCH; ++ch) {
        const int b = (nc + ch) & 1, q0 = ch * C::CH;
        const int w = min(C::CH, C::NCUB8 - q0);
        const double* sCb = sC + (size_t)b * C::R * C::LDC;
        double* sGb = sG + (size_t)b * C::R * C::LDG;
        nbar_sync(kBarCFull + b, NTH);
        nbar_sync(kBarGEmpty + b, NTH);
#pragma unroll 1
        for (int it = 0; it < C::IT_P; ++it) {
          const int idx = ft + it * C::NFT;
          if (idx >= C::E * w) break;
          const int e = idx / w, ql = idx - e * w, q = q0 + ql;
          const double* uc = sCb + (e * 5) * C::LDC + ql;
          double* gout = sGb + (e * 5) * C::LDG + ql;
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
        nbar_arrive(kBarCEmpty + b, NTH);
        nbar_arrive(kBarGFull + b, NTH);
      }
      nc += C::NCH;
    }
  }
}

}  // namespace cdg_gpu
