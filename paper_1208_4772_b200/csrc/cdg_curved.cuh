// cdg_curved.cuh -- RHS + LSRK kernel for CURVED (isoparametric) elements.
//
// Reference math (operators.cpp:32-167, solver.cpp:362-464) for an element
// whose map is not affine: per cubature node the metric terms vary, so
//   vol  = sum_m D_m^T ( JW r_m . F )  -  I_g^T ( (sjac w) F* )
//   rhs  = M_e^-1 vol,     M_e = I_cub^T diag(J W) I_cub
// G_m(q) = sum_d (J W dr_m/dx_d)(q) F_d(q) is formed pointwise from per-node
// metrics; the shared operator [D_r^T D_s^T D_t^T | -I_g^T] runs on the DMMA
// pipe exactly like k_rhs; M_e^-1 (dense, per element, precomputed on the
// host -- a GEMV instead of the reference's two triangular solves,
// operators.cpp:8-22) is applied in the epilogue. Curved elements are a
// list (ids); the affine kernels skip them (curved flag in the coupling word).
#pragma once

#include "cdg_kernels.cuh"

namespace cdg_gpu {

struct CurvedParams {
  RhsParams base;
  const int* ids;          // [Kc] element ids
  const double* jwr;       // [Kc][NCUB][9]  J W dr_m/dx_d  (m*3+d)
  const double4* face;     // [Kc][NF]       (nx, ny, nz, sjac*w)
  const double* minv;      // [Kc][NP][NP], transposed: (M_e^-1)[i][j] at [c][j][i]
  const double* frag_opc;  // B fragments of [D^T | -I_g^T]
  double* vol;             // [Kc*5][NP8] epilogue scratch when the tile's vol does not fit smem
  double* q_out;           // [3][K*5][BP] aux gradient (k_aux_curved)
  int Kc;
  const int* ctiles;       // optional list of curved tiles (E consecutive list entries each); null = all
  int n_clist;
};

template <class C>
struct CurvedLayout {
  static constexpr int LDV = C::NP8 + 1;
  static constexpr size_t SMEM_NO_V =
      sizeof(double) * (C::SMEM_U + C::SMEM_C + C::SMEM_G) + sizeof(int) * (C::E * 4 * 2 + C::E);
  // p=8: the [R][NP8] vol panel does not fit next to the GEMM panels (227 KB
  // opt-in limit); it then goes through a global scratch (GV).
  static constexpr bool GV = SMEM_NO_V + sizeof(double) * (size_t)C::R * LDV > 232448;
  static constexpr size_t SMEM_BYTES = SMEM_NO_V + (GV ? 0 : sizeof(double) * (size_t)C::R * LDV);
};

template <class C, bool UPDATE, bool VISC = false>
__global__ void __launch_bounds__(kThreads, 1) k_rhs_curved(CurvedParams cp) {
  using L = CurvedLayout<C>;
  const RhsParams& p = cp.base;
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  double* sC = sU + C::SMEM_U;
  double* sG = sC + C::SMEM_C;
  double* sV = sG + C::SMEM_G;  // [R][LDV] vol (epilogue), unless GV
  int2* sConn = reinterpret_cast<int2*>(sV + (L::GV ? 0 : (size_t)C::R * L::LDV));
  int* sId = reinterpret_cast<int*>(sConn + C::E * 4);
  __shared__ int s_stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const double gamma = p.gas.gamma;
  const double2* fb1 = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fbc = reinterpret_cast<const double2*>(cp.frag_opc);
  const int t_begin = (warp * C::T2) / kWarps, t_end = ((warp + 1) * C::T2) / kWarps;
  const int n_tiles = (cp.Kc + C::E - 1) / C::E;

  const int n_iter = cp.ctiles ? cp.n_clist : n_tiles;  // optional curved-tile list (multi-GPU split)
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = cp.ctiles ? __ldg(cp.ctiles + it_t) : it_t;
    if (tid == 0) s_stop = *(volatile int*)&p.err->flag;
    __syncthreads();
    if (s_stop) return;
    const int c0 = tile * C::E;  // index into the curved list
    for (int idx = tid; idx < C::E; idx += kThreads) sId[idx] = c0 + idx < cp.Kc ? cp.ids[c0 + idx] : -1;
    __syncthreads();
    // stage U rows of the listed elements (pcol-permuted panel)
    constexpr int V8 = C::KP / 8;
    for (int idx = tid; idx < C::R * V8 * 2; idx += kThreads) {
      const int h = idx & 1, j = (idx >> 1) % V8, r = (idx >> 1) / V8;
      const int e = sId[r / 5];
      double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
      if (e >= 0) {
        const double* src = p.u + ((size_t)e * 5 + r % 5) * C::BP + 8 * j + 2 * h;
        x = *reinterpret_cast<const double2*>(src);
        y = *reinterpret_cast<const double2*>(src + 4);
      }
      double* o = sU + r * C::LDU + 8 * j + 4 * h;
      *reinterpret_cast<double2*>(o) = make_double2(x.x, y.x);
      *reinterpret_cast<double2*>(o + 2) = make_double2(x.y, y.y);
    }
    for (int idx = tid; idx < C::E * 4; idx += kThreads) {
      const int e = sId[idx / 4];
      sConn[idx] = e >= 0 ? p.conn[(size_t)e * 4 + idx % 4] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    __syncthreads();

    double acc[C::MAXT2][4];
#pragma unroll
    for (int i = 0; i < C::MAXT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;

    for (int ch = 0; ch < C::NCH; ++ch) {
      const int q0 = ch * C::CH;
      const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;
      gemm1_chunk<C>(sU, sC, fb1, q0, w, warp, lane);
      __syncthreads();
      for (int idx = tid; idx < C::E * w; idx += kThreads) {
        const int e = idx / w, ql = idx - e * w, q = q0 + ql;
        const double* uc = sC + (e * 5) * C::LDC + ql;
        double G[3][5];
        const int ce = c0 + e;
        if (q < C::NCUB && ce < cp.Kc) {
          const State5 s{uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
          if (!admissible(s, gamma)) record_error(p.err, 1, p.elem_offset + sId[e], q, 0, s.r);
          const double pr = pressure(s, gamma);
          const double vx = s.mx / s.r, vy = s.my / s.r, vz = s.mz / s.r;
          const double ep = s.E + pr;
          double F[3][5] = {{s.mx, s.mx * vx + pr, s.my * vx, s.mz * vx, vx * ep},
                            {s.my, s.mx * vy, s.my * vy + pr, s.mz * vy, vy * ep},
                            {s.mz, s.mx * vz, s.my * vz, s.mz * vz + pr, vz * ep}};
          if (VISC) {
            // F_m <- F_m - sqrt(eps) I_cub q_m  (solver.cpp:398-406)
            const double se = p.sqrt_eps[sId[e]];
            if (se > 0.0) {
              constexpr int LDQ = round_up(C::NCUB, 8);
              const size_t qcs = (size_t)p.K * 5 * LDQ;
#pragma unroll
              for (int m = 0; m < 3; ++m)
#pragma unroll
                for (int c = 0; c < 5; ++c)
                  F[m][c] -= se * __ldg(p.qcub + m * qcs + ((size_t)sId[e] * 5 + c) * LDQ + q);
            }
          }
          const double* met = cp.jwr + ((size_t)ce * C::NCUB + q) * 9;
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const double r0 = __ldg(met + m * 3), r1 = __ldg(met + m * 3 + 1), r2 = __ldg(met + m * 3 + 2);
#pragma unroll
            for (int c = 0; c < 5; ++c) G[m][c] = r0 * F[0][c] + r1 * F[1][c] + r2 * F[2][c];
          }
        } else {
#pragma unroll
          for (int m = 0; m < 3; ++m)
#pragma unroll
            for (int c = 0; c < 5; ++c) G[m][c] = 0.0;
        }
        double* gout = sG + (e * 5) * C::LDG;
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
          for (int c = 0; c < 5; ++c) gout[c * C::LDG + pcol(m * w + ql)] = G[m][c];
      }
      __syncthreads();
      gemm2_partial<C>(acc, sG, fbc, (3 * q0) / 8, (3 * w) / 8, t_begin, t_end, lane);
      __syncthreads();
    }
    for (int fc = 0; fc < C::NFCH; ++fc) {
      const int f0 = fc * C::FCH;
      const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
      const int wp = round_up(wr, 8);
      for (int idx = tid; idx < C::E * wp; idx += kThreads) {
        const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
        double* gout = sG + (e * 5) * C::LDG + pcol(fl);
        const int ce = c0 + e, eg = sId[e];
        if (ce >= cp.Kc || fl >= wr) {
#pragma unroll
          for (int c = 0; c < 5; ++c) gout[c * C::LDG] = 0.0;
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
        if (!admissible(um, gamma) || !admissible(up, gamma))
          record_error(p.err, 2, p.elem_offset + eg, f, gq, um.r);
        double fs[5];
        if (p.gas.riemann == 1)
          hllc_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs, p.gas.hllc_fallbacks);
        else
          llf_flux(um, up, fn.x, fn.y, fn.z, gamma, fs);
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
        for (int c = 0; c < 5; ++c) gout[c * C::LDG] = fn.w * fs[c];
      }
      __syncthreads();
      gemm2_partial<C>(acc, sG, fbc, (C::K2CUB + f0) / 8, wp / 8, t_begin, t_end, lane);
      __syncthreads();
    }
    // vol -> smem (or the global scratch), then rhs = M_e^-1 vol (per element
    // dense GEMV), update
    double* vbase = L::GV ? cp.vol + (size_t)c0 * 5 * L::LDV : sV;
#pragma unroll
    for (int i = 0; i < C::MAXT2; ++i) {
      const int t = t_begin + i;
      if (t < t_end) {
        const int nt = t / C::MT, mt = t % C::MT;
        for (int hh = 0; hh < 2; ++hh) {
          const int r = mt * 16 + g + 8 * hh;
          if (L::GV && c0 + r / 5 >= cp.Kc) continue;
          vbase[r * L::LDV + nt * 8 + 2 * tq] = acc[i][2 * hh];
          vbase[r * L::LDV + nt * 8 + 2 * tq + 1] = acc[i][2 * hh + 1];
        }
      }
    }
    __syncthreads();
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
    // thread <-> (element, output node i): one pass over row i of M_e^-1 serves
    // all five fields
    for (int idx = tid; idx < C::E * C::NP; idx += kThreads) {
      const int e = idx / C::NP, i = idx - e * C::NP;
      const int ce = c0 + e;
      if (ce >= cp.Kc) continue;
      const double* mcol = cp.minv + (size_t)ce * C::NP * C::NP + i;  // (M_e^-1)[i][j] at j*NP + i
      const double* v = vbase + (e * 5) * L::LDV;
      double rhs[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (int j = 0; j < C::NP; ++j) {
        const double mij = __ldg(mcol + (size_t)j * C::NP);
#pragma unroll
        for (int f = 0; f < 5; ++f) rhs[f] += mij * v[f * L::LDV + j];
      }
#pragma unroll
      for (int f = 0; f < 5; ++f) {
        const int r = e * 5 + f;
        const size_t gi = ((size_t)sId[e] * 5 + f) * C::BP + i;
        if (UPDATE) {
          const double rn = a_c * p.res[gi] + dt * rhs[f];
          p.res[gi] = rn;
          p.u[gi] = sU[r * C::LDU + pcol(i)] + b_c * rn;
        } else {
          p.rhs_out[gi] = rhs[f];
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Auxiliary gradient on curved elements (compute_aux_gradient, solver.cpp:
// 264-312) with per-node metrics:
//   q_m = M_e^-1 [ -se sum_k D_k^T (JW dr_k/dx_m U_cub)
//                  + I_g^T ((sjac w) 1/2 (se U- + snb U+) n_m) ]
// The shared operator is frag_opc = [D^T | -I_g^T]; the face term is fed
// negated. Overwrites the affine kernel's q rows of the listed elements.
// ---------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(kThreads, 1) k_aux_curved(CurvedParams cp) {
  using L = CurvedLayout<C>;
  const RhsParams& p = cp.base;
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  double* sC = sU + C::SMEM_U;
  double* sG = sC + C::SMEM_C;
  double* sV = sG + C::SMEM_G;
  int2* sConn = reinterpret_cast<int2*>(sV + (L::GV ? 0 : (size_t)C::R * L::LDV));
  int* sId = reinterpret_cast<int*>(sConn + C::E * 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const double2* fb1 = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fbc = reinterpret_cast<const double2*>(cp.frag_opc);
  const int t_begin = (warp * C::T2) / kWarps, t_end = ((warp + 1) * C::T2) / kWarps;
  const int n_tiles = (cp.Kc + C::E - 1) / C::E;
  const size_t qstride = (size_t)p.K * 5 * C::BP;

  const int n_iter = cp.ctiles ? cp.n_clist : n_tiles;  // optional curved-tile list (multi-GPU split)
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = cp.ctiles ? __ldg(cp.ctiles + it_t) : it_t;
    const int c0 = tile * C::E;
    for (int idx = tid; idx < C::E; idx += kThreads) sId[idx] = c0 + idx < cp.Kc ? cp.ids[c0 + idx] : -1;
    __syncthreads();
    constexpr int V8 = C::KP / 8;
    for (int idx = tid; idx < C::R * V8 * 2; idx += kThreads) {
      const int hh = idx & 1, j = (idx >> 1) % V8, r = (idx >> 1) / V8;
      const int e = sId[r / 5];
      double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
      if (e >= 0) {
        const double* src = p.u + ((size_t)e * 5 + r % 5) * C::BP + 8 * j + 2 * hh;
        x = *reinterpret_cast<const double2*>(src);
        y = *reinterpret_cast<const double2*>(src + 4);
      }
      double* o = sU + r * C::LDU + 8 * j + 4 * hh;
      *reinterpret_cast<double2*>(o) = make_double2(x.x, y.x);
      *reinterpret_cast<double2*>(o + 2) = make_double2(x.y, y.y);
    }
    for (int idx = tid; idx < C::E * 4; idx += kThreads) {
      const int e = sId[idx / 4];
      sConn[idx] = e >= 0 ? p.conn[(size_t)e * 4 + idx % 4] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    __syncthreads();
    for (int m = 0; m < 3; ++m) {
      double acc[C::MAXT2][4];
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
      for (int ch = 0; ch < C::NCH; ++ch) {
        const int q0 = ch * C::CH;
        const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;
        gemm1_chunk<C>(sU, sC, fb1, q0, w, warp, lane);
        __syncthreads();
        // G_k = -se (JW dr_k/dx_m) U_cub   (solver.cpp:283-289, operators.cpp:135-149)
        for (int idx = tid; idx < C::R * w; idx += kThreads) {
          const int r = idx / w, ql = idx % w, e = r / 5, q = q0 + ql;
          const int ce = c0 + e;
          double* o = sG + r * C::LDG;
          if (q < C::NCUB && ce < cp.Kc) {
            const double uc = sC[r * C::LDC + ql];
            const double se = p.sqrt_eps[sId[e]];
            const double* jw = cp.jwr + ((size_t)ce * C::NCUB + q) * 9;
#pragma unroll
            for (int k = 0; k < 3; ++k) o[pcol(k * w + ql)] = -se * (__ldg(jw + k * 3 + m) * uc);
          } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) o[pcol(k * w + ql)] = 0.0;
          }
        }
        __syncthreads();
        gemm2_partial<C>(acc, sG, fbc, (3 * q0) / 8, (3 * w) / 8, t_begin, t_end, lane);
        __syncthreads();
      }
      for (int fc = 0; fc < C::NFCH; ++fc) {
        const int f0 = fc * C::FCH;
        const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
        const int wp = round_up(wr, 8);
        for (int idx = tid; idx < C::E * wp; idx += kThreads) {
          const int e = idx / wp, fl = idx % wp, fq = f0 + fl;
          const int ce = c0 + e, eg = sId[e];
          double* gout = sG + (e * 5) * C::LDG + pcol(fl);
          if (ce >= cp.Kc || fl >= wr) {
            for (int c = 0; c < 5; ++c) gout[c * C::LDG] = 0.0;
            continue;
          }
          const int f = fq / C::NG, gq = fq - f * C::NG;
          const double* tm = p.traces + (size_t)eg * 5 * C::TB + fq;
          const State5 um{tm[0], tm[C::TB], tm[2 * C::TB], tm[3 * C::TB], tm[4 * C::TB]};
          const double4 fn = cp.face[(size_t)ce * C::NF + fq];
          const int2 cw = sConn[e * 4 + f];
          const double se = p.sqrt_eps[eg];
          State5 up;
          double snb;
          if (cw.x >= 0) {
            const int hn = __ldg(p.code_map + (cw.y >> 8) * C::NG + gq);
            const double* tp = p.traces + (size_t)cw.x * 5 * C::TB + (cw.y & 3) * C::NG + hn;
            up = State5{tp[0], tp[C::TB], tp[2 * C::TB], tp[3 * C::TB], tp[4 * C::TB]};
            snb = p.sqrt_eps[cw.x];
          } else {
            up = boundary_state(um, fn.x, fn.y, fn.z, (cw.y >> 2) & 3, p.gas);
            snb = se;
          }
          const double nm = m == 0 ? fn.x : (m == 1 ? fn.y : fn.z);
          const double umv[5] = {um.r, um.mx, um.my, um.mz, um.E};
          const double upv[5] = {up.r, up.mx, up.my, up.mz, up.E};
          for (int c = 0; c < 5; ++c) gout[c * C::LDG] = -fn.w * (0.5 * (se * umv[c] + snb * upv[c]) * nm);
        }
        __syncthreads();
        gemm2_partial<C>(acc, sG, fbc, (C::K2CUB + f0) / 8, wp / 8, t_begin, t_end, lane);
        __syncthreads();
      }
      // q_m = M_e^-1 vol
      double* vbase = L::GV ? cp.vol + (size_t)c0 * 5 * L::LDV : sV;
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) {
        const int t = t_begin + i;
        if (t < t_end) {
          const int nt = t / C::MT, mt = t % C::MT;
          for (int hh = 0; hh < 2; ++hh) {
            const int r = mt * 16 + g + 8 * hh;
            if (L::GV && c0 + r / 5 >= cp.Kc) continue;
            vbase[r * L::LDV + nt * 8 + 2 * tq] = acc[i][2 * hh];
            vbase[r * L::LDV + nt * 8 + 2 * tq + 1] = acc[i][2 * hh + 1];
          }
        }
      }
      __syncthreads();
      for (int idx = tid; idx < C::E * C::NP; idx += kThreads) {
        const int e = idx / C::NP, i = idx - e * C::NP;
        const int ce = c0 + e;
        if (ce >= cp.Kc) continue;
        const double* mcol = cp.minv + (size_t)ce * C::NP * C::NP + i;
        const double* v = vbase + (e * 5) * L::LDV;
        double qv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int j = 0; j < C::NP; ++j) {
          const double mij = __ldg(mcol + (size_t)j * C::NP);
#pragma unroll
          for (int f = 0; f < 5; ++f) qv[f] += mij * v[f * L::LDV + j];
        }
#pragma unroll
        for (int f = 0; f < 5; ++f) cp.q_out[m * qstride + ((size_t)sId[e] * 5 + f) * C::BP + i] = qv[f];
      }
      __syncthreads();
    }
  }
}

}  // namespace cdg_gpu
