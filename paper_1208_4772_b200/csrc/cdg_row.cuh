// cdg_row.cuh -- RHS + LSRK kernel with one m-tile ROW per warp (affine tets,
// inviscid; p = 4 and the curved-mesh p = 3/4 levels' affine elements).
//
// Same math and evaluation order as k_rhs (cdg_kernels.cuh; reference
// solver.cpp:325-492). What changes is the mapping onto the SM:
//
//  * A CTA is 5 warps on a tile of 16 elements = 80 (element, field) rows =
//    5 m16 tiles; warp w owns rows [16w, 16w+16) in EVERY contraction. Its
//    GEMM output is one full row of n-tiles, so each A fragment (2 x LDS.128)
//    is reused across all N_p/8 n-tiles.
//  * The nodal state U never goes to shared memory: the warp keeps its rows
//    of U as the A fragments of the nodal->cubature GEMM in registers (with
//    logical k = t <-> node 8ks+2t and k = t+4 <-> node 8ks+2t+1, the
//    fragment of k-step ks holds exactly the (row, 8ks+2t..+1) values the
//    accumulator of output n-tile ks holds), so the same registers are the
//    old u of the LSRK update in the epilogue.
//  * The B fragments of the shared operators (115 KB at p = 4) are streamed
//    chunk by chunk into a double-buffered shared-memory ring by the bulk-copy
//    (TMA) engine, one elected thread per CTA issuing cp.async.bulk with an
//    mbarrier transaction count; the copy of chunk n+1 overlaps chunk n.
//  * Without the U panel a CTA needs ~69 KB of shared memory (double-buffered
//    U_cub / flux chunks, reused for the face fluxes and the staged res of the
//    epilogue, plus the operator ring), so 3 CTAs share an SM.
//  * Two CTA barriers per cubature chunk (U_cub ready, flux ready); the
//    double buffers remove the third.
#pragma once

#include "cdg_kernels.cuh"

namespace cdg_gpu {

// MODE bits: 1 operator ring (bulk-copy staged B fragments; else __ldg from
// L1/L2), 2 U fragments register-resident for the whole tile (else reloaded
// per chunk, which frees ~40 registers), 4 res staged to smem for the epilogue,
// 8 U rows staged once per tile in smem by cp.async (GEMM1 A fragments and the
// epilogue's old u come from there; excludes 2), 32 fused traces, 64 / 128
// volume / face GEMM k-steps unrolled (the next k-step's A fragment and B
// fragments in flight during the current one's MMAs), 256 both rows' old res
// loaded up front, 1024 the fused-trace n-tile groups unrolled.
template <int NP_, int NCUB_, int NG_, int CH_ = 8, int FCH_ = 32, int MINB_ = 3, int MODE_ = 7, int E_ = 16>
struct RCfg {
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_;
  static constexpr int MODE = MODE_;
  // E elements per tile (multiple of 16): 5E rows = 5E/16 m-tiles, one warp each
  static constexpr int E = E_, R = 5 * E_, NW = R / 16, NTH = 32 * NW, MINB = MINB_;
  static constexpr bool OPRING = MODE_ & 1, RESS = MODE_ & 4, USMEM = MODE_ & 8;
  static constexpr bool UREG = (MODE_ & 2) && !USMEM;
  // 32: fused traces -- the epilogue also writes I_g u_new (the next stage's
  // face traces) to p.traces_out, which replaces the separate trace kernel
  static constexpr bool FT = MODE_ & 32;
  static constexpr int BP = dev_block(NP), TB = dev_tblock(NF);
  static constexpr int KP = round_up(NP, 8), KS1 = KP / 8, NT2 = KS1;
  static constexpr int NCUB8 = round_up(NCUB, 8), NF8 = round_up(NF, 8);
  static constexpr int CH = CH_, NCH = ceil_div(NCUB8, CH);
  static constexpr int FCH = FCH_, NFCH = ceil_div(NF, FCH);
  static constexpr int K2CUB = 3 * NCUB8, K2 = K2CUB + NF8, KS2 = K2 / 8;
  // U_cub chunk: LDC = 8 (mod 16) doubles makes both the GEMM1 stores (rows g,
  // g+1 of a quarter-warp 64 B apart) and the pointwise column reads (elements
  // e, e+1 of a half-warp 5*LDC doubles = 64 B (mod 128) apart) bank-conflict free
  static constexpr int LDC = frag_ld8(CH);
  static constexpr int LDG = frag_ld8(3 * CH);        // flux chunk, conflict-free 128-bit A loads
  static constexpr int LDF = frag_ld8(FCH);           // face-flux chunk
  // volume phase: one U_cub chunk (rewritten only after the barrier that
  // follows the pointwise pass) + two flux chunks (double buffer)
  // (single buffers suffice: PW(i+1) writes the flux chunk only after the
  // barrier that follows GEMM1(i+1), which every warp reaches after GEMM2(i))
  static constexpr int VOL = R * LDC + R * LDG;
  static constexpr int LDU = frag_ld8(KP);
  static constexpr int UPANEL = USMEM ? R * LDU : 0;  // doubles
  static constexpr int RES = RESS ? NTH * 2 * NT2 * 2 : 0;  // doubles: each thread's epilogue res values
  static constexpr int FACE = R * LDF + RES;              // doubles, face phase (aliases VOL)
  static constexpr int WORK = VOL > FACE ? VOL : FACE;
  static constexpr int IT_P = ceil_div(E * CH, NTH);
  static constexpr int IT_F = ceil_div(E * FCH, NTH);
  // operator chunks staged by the bulk-copy engine: a cubature chunk needs the
  // I_cub fragments of its CH/8 n-tiles and the [A_r A_s A_t] fragments of
  // its 3CH/8 k-steps; a face chunk the -LIFT fragments of its FCH/8 k-steps
  static constexpr int OPV = (CH / 8) * KS1 * 64 + (3 * CH / 8) * NT2 * 64;  // doubles
  static constexpr int OPF = (FCH / 8) * NT2 * 64;
  static constexpr int OPB = !OPRING ? 0 : (OPV > OPF ? OPV : OPF);
  static constexpr int NCHT = NCH + NFCH;  // operator chunks per tile
  static constexpr size_t SMEM_BYTES = sizeof(double) * ((size_t)WORK + UPANEL + 2 * OPB + E * 9 + E * 4 * 4) +
                                       sizeof(int) * (E * 4 * 2) + 2 * sizeof(unsigned long long);
};

// ---- bulk-copy (TMA engine) + mbarrier helpers -----------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async16_sh(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_sh(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Issue the operator chunk with global index n (per CTA, counting over its
// tiles) into buffer n & 1. Chunk k = n % NCHT of a tile: k < NCH cubature
// chunk k, else face chunk k - NCH.
template <class C>
__device__ __forceinline__ void issue_op_chunk(int n, double* sOp, unsigned long long* bars, const double* f1,
                                               const double* f2) {
  const int k = n % C::NCHT, b = n & 1;
  double* dst = sOp + b * C::OPB;
  if (k < C::NCH) {
    const int q0 = k * C::CH, w = min(C::CH, C::NCUB8 - q0);
    const unsigned b1 = (unsigned)((w / 8) * C::KS1 * 64 * sizeof(double));
    const unsigned b2 = (unsigned)((3 * w / 8) * C::NT2 * 64 * sizeof(double));
    mbar_expect_tx(&bars[b], b1 + b2);
    bulk_g2s(dst, f1 + (size_t)(q0 / 8) * C::KS1 * 64, b1, &bars[b]);
    bulk_g2s(dst + (C::CH / 8) * C::KS1 * 64, f2 + (size_t)(3 * q0 / 8) * C::NT2 * 64, b2, &bars[b]);
  } else {
    const int f0 = (k - C::NCH) * C::FCH;
    const int wp = round_up(min(C::FCH, C::NF - f0), 8);
    const unsigned b2 = (unsigned)((wp / 8) * C::NT2 * 64 * sizeof(double));
    mbar_expect_tx(&bars[b], b2);
    bulk_g2s(dst, f2 + (size_t)((C::K2CUB + f0) / 8) * C::NT2 * 64, b2, &bars[b]);
  }
}

// B fragments (natural pairing, see cdg_warp.cuh): frag1[(qt*KS1 + ks)*32 + lane]
// for I_cub n-tile qt; frag2[(ks*NT2 + nt)*32 + lane] for the chunked
// [A_r A_s A_t | -LIFT] operator (k-step-major: one k-step's n-tiles adjacent).
template <class C, bool UPDATE, int RM>
__global__ void __launch_bounds__(C::NTH, C::MINB) k_rhs_row(RhsParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sWork = smem;
  double* sUp = sWork + C::WORK;                                  // [R][LDU] U rows (USMEM)
  double* sOp = sUp + C::UPANEL;                                  // [2][OPB] operator chunks
  double* sMet = sOp + 2 * C::OPB;                                // [E][9]
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);    // [E][4]
  int2* sConn = reinterpret_cast<int2*>(sFace + C::E * 4);         // [E][4]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sConn + C::E * 4);  // [2]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const int n_tiles = (p.K + C::E - 1) / C::E;
  __shared__ int s_stop;
  // operator chunk pipeline: chunk n of this CTA lives in buffer n & 1
  const int n_iter = p.tiles ? p.n_list : n_tiles;
  const int my_tiles = blockIdx.x < n_iter ? (n_iter - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int n_chunks = my_tiles * C::NCHT;
  int n = 0;  // current chunk
  if (C::OPRING) {
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0 && n_chunks > 0) issue_op_chunk<C>(0, sOp, bars, p.frag_icub, p.frag_op2);
  }

  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = tile_at(p, it_t);
    // block-uniform early exit after a recorded error (no divergent barriers)
    if (tid == 0) s_stop = *(volatile int*)&p.err->flag;
    __syncthreads();
    if (s_stop) return;
    const int e0 = tile * C::E, row0 = e0 * 5;
    const int r_lo = row0 + warp * 16 + g, r_hi = r_lo + 8;  // this thread's two rows
    if (p.prefetch) {
      const int rows = min(C::R, n_rows - row0);
      if (UPDATE && (p.prefetch & 1)) l2_prefetch_range(p.res + (size_t)row0 * C::BP, (size_t)rows * C::BP * 8, tid, C::NTH);
      (void)rows;
      if (p.prefetch & 4) l2_prefetch_range(p.traces + (size_t)row0 * C::TB, (size_t)rows * C::TB * 8, tid, C::NTH);
      const int nrow0 = (tile + gridDim.x) * C::R;
      if ((p.prefetch & 2) && nrow0 < n_rows)
        l2_prefetch_range(p.u + (size_t)nrow0 * C::BP, (size_t)min(C::R, n_rows - nrow0) * C::BP * 8, tid, C::NTH);
    }
    // ---- U rows -> registers (A fragments of the nodal->cubature GEMM) ------
    const double* u_lo = p.u + (size_t)min(r_lo, n_rows - 1) * C::BP + 2 * tq;
    const double* u_hi = p.u + (size_t)min(r_hi, n_rows - 1) * C::BP + 2 * tq;
    const bool ok_lo = r_lo < n_rows, ok_hi = r_hi < n_rows;
    double uA[C::KS1][4];
    auto load_u = [&]() {
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) {
        double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
        if (ok_lo) x = *reinterpret_cast<const double2*>(u_lo + ks * 8);
        if (ok_hi) y = *reinterpret_cast<const double2*>(u_hi + ks * 8);
        uA[ks][0] = x.x;
        uA[ks][1] = y.x;
        uA[ks][2] = x.y;
        uA[ks][3] = y.y;
      }
    };
    if (C::UREG) load_u();
    if (C::USMEM) {
      constexpr int V = C::KP / 2;  // 16-byte pieces per row
      for (int idx = tid; idx < C::R * V; idx += C::NTH) {
        const int r = idx / V, j = idx - r * V;
        const bool ok = row0 + r < n_rows;
        double* dst = sUp + r * C::LDU + 2 * j;
        if (ok)
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

    double acc[C::NT2][4];
#pragma unroll
    for (int i = 0; i < C::NT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;

    // ---- volume: chunks of CH cubature nodes ----------------------------------
#pragma unroll 1
    for (int ch = 0; ch < C::NCH; ++ch) {
      const int q0 = ch * C::CH;
      const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;  // multiple of 8
      double* sC = sWork;
      double* sG = sWork + C::R * C::LDC;
      const double2 *fb1, *fb2;  // [CH/8][KS1][32], [3CH/8][NT2][32]
      if (C::OPRING) {
        fb1 = reinterpret_cast<const double2*>(sOp + (n & 1) * C::OPB);
        fb2 = fb1 + (C::CH / 8) * C::KS1 * 32;
        mbar_wait(&bars[n & 1], (n >> 1) & 1);
      } else {
        fb1 = reinterpret_cast<const double2*>(p.frag_icub) + (size_t)(q0 / 8) * C::KS1 * 32;
        fb2 = reinterpret_cast<const double2*>(p.frag_op2) + (size_t)(3 * q0 / 8) * C::NT2 * 32;
      }
      if (!C::UREG && !C::USMEM) load_u();
      // GEMM1: U_cub[rows, q0:q0+w] for this warp's 16 rows
      {
        double c1[C::CH / 8][4];
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j) c1[j][0] = c1[j][1] = c1[j][2] = c1[j][3] = 0.0;
#pragma unroll
        for (int ks = 0; ks < C::KS1; ++ks) {
          double a0, a1, a2, a3;
          if (C::USMEM) {
            const AFrag a = load_afrag(sUp, C::LDU, warp * 16, ks * 8, g, tq);
            a0 = a.a0, a1 = a.a1, a2 = a.a2, a3 = a.a3;
          } else {
            a0 = uA[ks][0], a1 = uA[ks][1], a2 = uA[ks][2], a3 = uA[ks][3];
          }
#pragma unroll
          for (int j = 0; j < C::CH / 8; ++j)
            if (j * 8 < w) {
              const double2 b = C::OPRING ? fb1[(j * C::KS1 + ks) * 32 + lane] : __ldg(fb1 + (j * C::KS1 + ks) * 32 + lane);
              dmma_k8(c1[j], a0, a1, a2, a3, b.x, b.y);
            }
        }
#pragma unroll
        for (int j = 0; j < C::CH / 8; ++j)
          if (j * 8 < w) {
            double* o = sC + (warp * 16 + g) * C::LDC + j * 8 + 2 * tq;
            *reinterpret_cast<double2*>(o) = make_double2(c1[j][0], c1[j][1]);
            *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c1[j][2], c1[j][3]);
          }
      }
      __syncthreads();
      // every warp is past GEMM2 of chunk n-1: its buffer takes chunk n+1
      if (C::OPRING && tid == 0 && n + 1 < n_chunks) {
        fence_proxy_async();
        issue_op_chunk<C>(n + 1, sOp, bars, p.frag_icub, p.frag_op2);
      }
      // pointwise Euler flux -> contravariant flux G_m = sum_d (dr_m/dx_d) F_d
#pragma unroll 1
      for (int it = 0; it < C::IT_P; ++it) {
        const int idx = tid + it * C::NTH;
        if (idx < C::E * w) {
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
      __syncthreads();
      // GEMM2 (volume part of K): acc += G[rows, 3w] * Op2[:, 3 q0 : 3 q0 + 3w]^T
      {
        const int nks = (3 * w) / 8;
        auto kstep = [&](int ks) {
          const AFrag a = load_afrag(sG, C::LDG, warp * 16, ks * 8, g, tq);
#pragma unroll
          for (int nt = 0; nt < C::NT2; ++nt)
            mma_frag(acc[nt], a, C::OPRING ? fb2[(ks * C::NT2 + nt) * 32 + lane] : __ldg(fb2 + (ks * C::NT2 + nt) * 32 + lane));
        };
        if constexpr (C::MODE & 64) {  // unrolled k-steps (A fragments of the next k-step in flight)
          if (w == C::CH) {
#pragma unroll
            for (int ks = 0; ks < 3 * C::CH / 8; ++ks) kstep(ks);
          } else {
#pragma unroll 1
            for (int ks = 0; ks < nks; ++ks) kstep(ks);
          }
        } else {
#pragma unroll 1
          for (int ks = 0; ks < nks; ++ks) kstep(ks);
        }
      }
      ++n;
    }
    __syncthreads();  // the face phase reuses the volume buffers

    // ---- surface: chunks of FCH face nodes -------------------------------------
    double* sF = sWork;
    // this thread's epilogue res values -> smem while the face phase runs
    double* sRes = sWork + C::R * C::LDF + tid * (2 * C::NT2 * 2);
    if (UPDATE && C::RESS) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int grow = hh ? r_hi : r_lo;
        if (grow < n_rows)
#pragma unroll
          for (int nt = 0; nt < C::NT2; ++nt)
            cp_async16_sh(sRes + (hh * C::NT2 + nt) * 2, p.res + (size_t)grow * C::BP + nt * 8 + 2 * tq);
      }
    }
#pragma unroll 1
    for (int fc = 0; fc < C::NFCH; ++fc) {
      const int f0 = fc * C::FCH;
      const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
      const int wp = round_up(wr, 8);
      auto face_item = [&](int it) {
        const int idx = tid + it * C::NTH;
        if (idx >= C::E * wp) return;
        const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
        double* gout = sF + (e * 5) * C::LDF + fl;
        const int eg = e0 + e;
        if (eg >= p.K || fl >= wr) {
#pragma unroll
          for (int c = 0; c < 5; ++c) gout[c * C::LDF] = 0.0;
          return;
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
      };
#pragma unroll 1
      for (int it = 0; it < C::IT_F; ++it) face_item(it);
      __syncthreads();
      if (C::OPRING && tid == 0 && n + 1 < n_chunks) {  // every warp is past the GEMM of chunk n-1
        fence_proxy_async();
        issue_op_chunk<C>(n + 1, sOp, bars, p.frag_icub, p.frag_op2);
      }
      {
        const double2* fb2;
        if (C::OPRING) {
          fb2 = reinterpret_cast<const double2*>(sOp + (n & 1) * C::OPB);
          mbar_wait(&bars[n & 1], (n >> 1) & 1);
        } else {
          fb2 = reinterpret_cast<const double2*>(p.frag_op2) + (size_t)((C::K2CUB + f0) / 8) * C::NT2 * 32;
        }
        const int nks = wp / 8;
        auto kstep = [&](int ks) {
          const AFrag a = load_afrag(sF, C::LDF, warp * 16, ks * 8, g, tq);
#pragma unroll
          for (int nt = 0; nt < C::NT2; ++nt)
            mma_frag(acc[nt], a, C::OPRING ? fb2[(ks * C::NT2 + nt) * 32 + lane] : __ldg(fb2 + (ks * C::NT2 + nt) * 32 + lane));
        };
        if constexpr (C::MODE & 128) {
          if (wp == C::FCH) {
#pragma unroll
            for (int ks = 0; ks < C::FCH / 8; ++ks) kstep(ks);
          } else {
#pragma unroll 1
            for (int ks = 0; ks < nks; ++ks) kstep(ks);
          }
        } else {
#pragma unroll 1
          for (int ks = 0; ks < nks; ++ks) kstep(ks);
        }
      }
      ++n;
      if (fc + 1 < C::NFCH) __syncthreads();
    }
    if (UPDATE && C::RESS) cp_async_wait0();
    if (UPDATE && !C::UREG && !C::USMEM) load_u();  // old u for the update

    // ---- epilogue: rhs -> (res, u) update or rhs store ---------------------------
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
    const bool cur_lo = (sConn[((warp * 16 + g) / 5) * 4].y & kCurvedBit) != 0;
    const bool cur_hi = (sConn[((warp * 16 + g + 8) / 5) * 4].y & kCurvedBit) != 0;
    // old res values are loaded before any store of the row (the compiler
    // cannot move loads of p.res above stores to p.u / p.res, so loads
    // interleaved with the stores would serialise NT2 memory round trips);
    // MODE 256: both rows' values up front
    constexpr bool RES2 = C::MODE & 256;
    double2 rsv[RES2 ? 2 : 1][C::NT2];
    auto load_res = [&](int hh, double2* dst) {
      const int grow = hh ? r_hi : r_lo;
      if (grow >= n_rows || (hh ? cur_hi : cur_lo)) return;
#pragma unroll
      for (int j = 0; j < C::NT2; ++j)
        dst[j] = *reinterpret_cast<const double2*>(p.res + (size_t)grow * C::BP + j * 8 + 2 * tq);
    };
    if (UPDATE && !C::RESS && RES2) {
      load_res(0, rsv[0]);
      load_res(1, rsv[RES2 ? 1 : 0]);
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int grow = hh ? r_hi : r_lo;
      if (grow >= n_rows || (hh ? cur_hi : cur_lo)) continue;  // curved rows: k_rhs_curved
      const size_t rowoff = (size_t)grow * C::BP;
      if (UPDATE && !C::RESS && !RES2) load_res(hh, rsv[0]);
#pragma unroll
      for (int j = 0; j < C::NT2; ++j) {
        const int col = j * 8 + 2 * tq;  // < KP <= BP; padded columns carry exact zeros
        const double r0 = acc[j][2 * hh], r1 = acc[j][2 * hh + 1];
        if (UPDATE) {
          const double2 rs = C::RESS ? *reinterpret_cast<const double2*>(sRes + (hh * C::NT2 + j) * 2)
                                     : rsv[RES2 ? hh : 0][j];
          const double n0 = a_c * rs.x + dt * r0, n1 = a_c * rs.y + dt * r1;
          *reinterpret_cast<double2*>(p.res + rowoff + col) = make_double2(n0, n1);
          // old u: the A fragment of k-step j holds (row, 8j+2t) / (row, 8j+2t+1)
          double u0, u1;
          if (C::USMEM) {
            const double2 uo = *reinterpret_cast<const double2*>(sUp + (warp * 16 + g + 8 * hh) * C::LDU + col);
            u0 = uo.x, u1 = uo.y;
          } else {
            u0 = hh ? uA[j][1] : uA[j][0], u1 = hh ? uA[j][3] : uA[j][2];
          }
          const double w0 = u0 + b_c * n0, w1 = u1 + b_c * n1;
          *reinterpret_cast<double2*>(p.u + rowoff + col) = make_double2(w0, w1);
          if (C::FT) {  // keep u_new in the accumulator (= A fragment) layout
            acc[j][2 * hh] = w0;
            acc[j][2 * hh + 1] = w1;
          }
        } else {
          *reinterpret_cast<double2*>(p.rhs_out + rowoff + col) = make_double2(r0, r1);
        }
      }
    }
    if (UPDATE && C::FT && p.traces_out) {
      // next stage's traces  T = u_new I_g^T  (solver.cpp:200-208) from the
      // registers: accumulator fragment of n-tile j == A fragment of k-step j
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int grow = hh ? r_hi : r_lo;
        if (grow >= n_rows || (hh ? cur_hi : cur_lo))
#pragma unroll
          for (int j = 0; j < C::NT2; ++j) acc[j][2 * hh] = acc[j][2 * hh + 1] = 0.0;
      }
      constexpr int NFT = C::NF8 / 8;
      // natural pairing (accumulator fragment of n-tile j == A fragment of
      // k-step j), the pairing of the trace kernel too (k_interp<NAT>): fused
      // and separate traces agree bit for bit
      const double2* fbi = reinterpret_cast<const double2*>(p.frag_ig_nat);  // [NFT][KS1][32]
      AFrag fa[C::KS1];
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks) fa[ks] = AFrag{acc[ks][0], acc[ks][2], acc[ks][1], acc[ks][3]};
      auto ft_group = [&](int nt0) {
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
            if (r_lo < n_rows)
              *reinterpret_cast<double2*>(p.traces_out + (size_t)r_lo * C::TB + col) = make_double2(tacc[i][0], tacc[i][1]);
            if (r_hi < n_rows)
              *reinterpret_cast<double2*>(p.traces_out + (size_t)r_hi * C::TB + col) = make_double2(tacc[i][2], tacc[i][3]);
          }
        }
      };
      if constexpr (C::MODE & 1024) {  // both 4-n-tile groups unrolled
#pragma unroll
        for (int nt0 = 0; nt0 < NFT; nt0 += 4) ft_group(nt0);
      } else {
#pragma unroll 1
        for (int nt0 = 0; nt0 < NFT; nt0 += 4) ft_group(nt0);
      }
    }
    __syncthreads();  // sConn / sWork are restaged next tile
  }
}

}  // namespace cdg_gpu
