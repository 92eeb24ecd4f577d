// cdg_aux.cuh -- artificial-viscosity sensor, auxiliary gradient, time step,
// residual and halo kernels (sm_100a).
#pragma once

#include "cdg_kernels.cuh"

namespace cdg_gpu {

// ---------------------------------------------------------------------------
// Persson-Peraire modal-decay sensor + viscosity ramp, one warp per element
// (compute_element_viscosities, solver.cpp:239-260; smoothness_indicator,
// viscosity.cpp:11-34; viscosity_amount, viscosity.cpp:48-56).
// ---------------------------------------------------------------------------
struct SensorParams {
  const double* u;
  const double* vinv;  // [np][np]
  double* eps;
  double* sqrt_eps;
  unsigned long long* maxeps;  // bit pattern of max eps (non-negative doubles)
  int K, np, np_prev, bp, comp;
  double eps0, kappa, s0;
  // J-weighted variant (viscosity.cpp:28-45)
  const double* vcub;       // [ncub][np] modal basis at the cubature nodes
  const double* wcub;       // [ncub]
  const double* jac;        // [K] affine cub_jac
  const int* curved_slot;   // [K] index into curved_jac or -1 (may be null)
  const double* curved_jac; // [Kc][ncub]
  int ncub;
};

// viscosity_amount (viscosity.cpp:48-56) of the indicator value sk_val
__device__ __forceinline__ double viscosity_ramp(double sk_val, const SensorParams& p) {
  if (!(sk_val > 0.0)) return 0.0;
  const double sk = log10(sk_val);
  if (sk < p.s0 - p.kappa) return 0.0;
  if (sk > p.s0 + p.kappa) return p.eps0;
  return 0.5 * p.eps0 * (1.0 + sin(M_PI * (sk - p.s0) / (2.0 * p.kappa)));
}

#ifndef CDG_SET_TU  // non-template kernels: defined once, in cdg_gpu.cu
__global__ void __launch_bounds__(256) k_sensor(SensorParams p) {
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (e >= p.K) return;
  const double* f = p.u + ((size_t)e * 5 + p.comp) * p.bp;
  double total = 0.0, top = 0.0;
  for (int j = lane; j < p.np; j += 32) {
    double m = 0.0;
    const double* row = p.vinv + (size_t)j * p.np;
    for (int i = 0; i < p.np; ++i) m += __ldg(row + i) * f[i];
    const double en = m * m;
    total += en;
    if (j >= p.np_prev) top += en;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    total += __shfl_xor_sync(0xffffffffu, total, off);
    top += __shfl_xor_sync(0xffffffffu, top, off);
  }
  if (lane == 0) {
    const double eps = viscosity_ramp(total <= 0.0 ? 0.0 : top / total, p);
    p.eps[e] = eps;
    p.sqrt_eps[e] = sqrt(eps);
    atomicMax(p.maxeps, (unsigned long long)__double_as_longlong(eps));
  }
}

// Physical-space indicator (viscosity.cpp:28-45): modal = V^-1 u,
// u_q = Vc modal, ut_q = Vc modal_trunc, S = sum JW (u-ut)^2 / sum JW u^2.
// One warp per element; the modal vector goes through shared memory.
__global__ void __launch_bounds__(256) k_sensor_jw(SensorParams p) {
  __shared__ double s_modal[8][176];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int e = blockIdx.x * 8 + wib;
  if (e >= p.K) return;
  const double* f = p.u + ((size_t)e * 5 + p.comp) * p.bp;
  for (int j = lane; j < p.np; j += 32) {
    double m = 0.0;
    const double* row = p.vinv + (size_t)j * p.np;
    for (int i = 0; i < p.np; ++i) m += __ldg(row + i) * f[i];
    s_modal[wib][j] = m;
  }
  __syncwarp();
  const int slot = p.curved_slot ? p.curved_slot[e] : -1;
  double num = 0.0, den = 0.0;
  for (int q = lane; q < p.ncub; q += 32) {
    const double* vr = p.vcub + (size_t)q * p.np;
    double uq = 0.0, ut = 0.0;
    for (int j = 0; j < p.np; ++j) {
      const double v = __ldg(vr + j) * s_modal[wib][j];
      uq += v;
      if (j < p.np_prev) ut += v;
    }
    const double jq = slot >= 0 ? p.curved_jac[(size_t)slot * p.ncub + q] : p.jac[e];
    const double jw = p.wcub[q] * jq;
    num += jw * (uq - ut) * (uq - ut);
    den += jw * uq * uq;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, off);
    den += __shfl_xor_sync(0xffffffffu, den, off);
  }
  if (lane == 0) {
    const double eps = viscosity_ramp(den <= 0.0 ? 0.0 : num / den, p);
    p.eps[e] = eps;
    p.sqrt_eps[e] = sqrt(eps);
    atomicMax(p.maxeps, (unsigned long long)__double_as_longlong(eps));
  }
}
#endif  // CDG_SET_TU

// ---------------------------------------------------------------------------
// Auxiliary gradient (compute_aux_gradient, solver.cpp:264-312), affine form:
//   q_m = -se sum_k A_k (r_{k,m} U_cub) + LIFT (scale * 1/2 (se U- + snb U+) n_m)
// Same chunked DMMA structure as k_rhs, one pass per direction m.
// ---------------------------------------------------------------------------
struct AuxParams {
  const double* u;
  double* q;  // [3][K*5][BP]
  const double* traces;
  const double* metric;
  const double4* face;
  const int2* conn;
  const int* code_map;
  const double* frag_icub;
  const double* frag_aux;
  const double* frag_dtil;  // [3][NT2][KS1][32] B fragments of A_k I_cub (N_p x N_p)
  const double* sqrt_eps;
  int K, n_tiles;
  GasParams gas;
  const unsigned long long* gate;  // optional launch gate (see gated_off)
  int gate_when;
  const int* tiles;  // optional tile list (curved levels: tiles holding an affine element)
  int n_list;
};

template <class C>
__global__ void __launch_bounds__(kThreads, C::MINB) k_aux_q(AuxParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  double* sC = sU + C::SMEM_U;
  double* sG = sC + C::SMEM_C;
  double* sMet = sG + C::SMEM_G;
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);
  double* sSe = reinterpret_cast<double*>(sFace + C::E * 4);
  int2* sConn = reinterpret_cast<int2*>(sSe + C::E);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int n_rows = p.K * 5;
  const size_t qstride = (size_t)p.K * 5 * C::BP;
  const int t_begin = (warp * C::T2) / kWarps, t_end = ((warp + 1) * C::T2) / kWarps;
  const double2* fba = reinterpret_cast<const double2*>(p.frag_aux);

  const int n_iter = p.tiles ? p.n_list : p.n_tiles;
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = p.tiles ? __ldg(p.tiles + it_t) : it_t;
    const int e0 = tile * C::E, row0 = e0 * 5;
    stage_rows<C>(p.u, row0, n_rows, sU, tid);
    for (int idx = tid; idx < C::E * 9; idx += kThreads)
      sMet[idx] = e0 + idx / 9 < p.K ? p.metric[(size_t)e0 * 9 + idx] : 0.0;
    for (int idx = tid; idx < C::E * 4; idx += kThreads) {
      const bool ok = e0 + idx / 4 < p.K;
      sFace[idx] = ok ? p.face[(size_t)e0 * 4 + idx] : make_double4(0, 0, 1, 0);
      sConn[idx] = ok ? p.conn[(size_t)e0 * 4 + idx] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    for (int idx = tid; idx < C::E; idx += kThreads) sSe[idx] = e0 + idx < p.K ? p.sqrt_eps[e0 + idx] : 0.0;
    __syncthreads();

    for (int m = 0; m < 3; ++m) {
      double acc[C::MAXT2][4];
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
      // volume part: for an affine element the metric r_km is constant, so
      //   -se sum_k A_k (r_km U_cub) = sum_k (A_k I_cub) (-se r_km U)
      // (matrix associativity; A_k I_cub = M_ref^-1 D_k^T W I_cub precomputed,
      // N_p x N_p): three N_p-deep contractions of row-scaled U instead of the
      // cubature round trip (solver.cpp:283-289 with operators.cpp:135-149).
      for (int k = 0; k < 3; ++k) {
        for (int idx = tid; idx < C::R * C::KP; idx += kThreads) {
          const int r = idx / C::KP, j = idx - r * C::KP, e = r / 5;
          sG[r * C::LDG + j] = -sSe[e] * sMet[e * 9 + k * 3 + m] * sU[r * C::LDU + j];  // same pcol layout
        }
        __syncthreads();
        const double2* fbd = reinterpret_cast<const double2*>(p.frag_dtil) + (size_t)k * C::NT2 * C::KS1 * 32;
#pragma unroll
        for (int i = 0; i < C::MAXT2; ++i) {
          const int t = t_begin + i;
          if (t < t_end) {
            const int nt = t / C::MT, mt = t % C::MT;
#pragma unroll
            for (int ks = 0; ks < C::KS1; ++ks)
              mma_frag(acc[i], load_afrag(sG, C::LDG, mt * 16, ks * 8, g, tq),
                       __ldg(fbd + ((size_t)nt * C::KS1 + ks) * 32 + lane));
          }
        }
        __syncthreads();
      }
      for (int fc = 0; fc < C::NFCH; ++fc) {
        const int f0 = fc * C::FCH;
        const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;
        const int wp = round_up(wr, 8);
        for (int idx = tid; idx < C::E * wp; idx += kThreads) {
          const int e = idx / wp, fl = idx % wp, fq = f0 + fl;
          const int eg = e0 + e;
          double* gout = sG + (e * 5) * C::LDG + pcol(fl);
          if (eg >= p.K || fl >= wr) {
            for (int c = 0; c < 5; ++c) gout[c * C::LDG] = 0.0;
            continue;
          }
          const int f = fq / C::NG, gq = fq - f * C::NG;
          const double* tm = p.traces + (size_t)eg * 5 * C::TB + fq;
          const State5 um{tm[0], tm[C::TB], tm[2 * C::TB], tm[3 * C::TB], tm[4 * C::TB]};
          const double4 fn = sFace[e * 4 + f];
          const int2 cw = sConn[e * 4 + f];
          const double se = sSe[e];
          State5 up;
          double snb;
          if (cw.x >= 0) {
            const int h = __ldg(p.code_map + (cw.y >> 8) * C::NG + gq);
            const double* tp = p.traces + (size_t)cw.x * 5 * C::TB + (cw.y & 3) * C::NG + h;
            up = State5{tp[0], tp[C::TB], tp[2 * C::TB], tp[3 * C::TB], tp[4 * C::TB]};
            snb = p.sqrt_eps[cw.x];
          } else {
            up = boundary_state(um, fn.x, fn.y, fn.z, (cw.y >> 2) & 3, p.gas);
            snb = se;
          }
          const double nm = m == 0 ? fn.x : (m == 1 ? fn.y : fn.z);
          const double umv[5] = {um.r, um.mx, um.my, um.mz, um.E};
          const double upv[5] = {up.r, up.mx, up.my, up.mz, up.E};
          for (int c = 0; c < 5; ++c) gout[c * C::LDG] = fn.w * (0.5 * (se * umv[c] + snb * upv[c]) * nm);
        }
        __syncthreads();
        gemm2_partial<C>(acc, sG, fba, (C::K2CUB + f0) / 8, wp / 8, t_begin, t_end, lane);
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) {
        const int t = t_begin + i;
        if (t < t_end) {
          const int nt = t / C::MT, mt = t % C::MT;
          for (int hh = 0; hh < 2; ++hh) {
            const int grow = row0 + mt * 16 + g + 8 * hh;
            if (grow >= n_rows) continue;
            for (int v = 0; v < 2; ++v) {
              const int col = nt * 8 + 2 * tq + v;
              if (col < C::NP) p.q[m * qstride + (size_t)grow * C::BP + col] = acc[i][2 * hh + v];
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// CFL time step (compute_timestep, solver.cpp:494-526): min over elements.
// ---------------------------------------------------------------------------
struct TimestepParams {
  const double* u;
  const double* h;
  const double* eps;
  int K, np, bp;
  double gamma, pfac;
  unsigned long long* out;
  DevError* err;
};

#ifndef CDG_SET_TU
// one warp per element, lanes over nodes (coalesced rows), shuffle max
__global__ void __launch_bounds__(256) k_timestep(TimestepParams p) {
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (e >= p.K) return;
  const double* f = p.u + (size_t)e * 5 * p.bp;
  double lambda = 0.0;
  int bad = -1;
  double bad_rho = 0.0;
  for (int i = lane; i < p.np; i += 32) {
    const State5 s{f[i], f[p.bp + i], f[2 * p.bp + i], f[3 * p.bp + i], f[4 * p.bp + i]};
    if (!admissible(s, p.gamma)) {
      bad = i;
      bad_rho = s.r;
      continue;
    }
    const double pres = pressure(s, p.gamma);
    const double c = sqrt(p.gamma * pres / s.r);
    lambda = fmax(lambda, sqrt(s.mx * s.mx + s.my * s.my + s.mz * s.mz) / s.r + c);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) lambda = fmax(lambda, __shfl_xor_sync(0xffffffffu, lambda, off));
  const unsigned badmask = __ballot_sync(0xffffffffu, bad >= 0);
  if (badmask) {
    if (lane == __ffs(badmask) - 1) record_error(p.err, 3, e, bad, 0, bad_rho);
    return;
  }
  if (lane != 0) return;
  const double h = p.h[e];
  if (h <= 0.0 || lambda <= 0.0) {
    record_error(p.err, 4, e, 0, 0, 0.0);
    return;
  }
  double dte = h / (lambda * p.pfac);
  if (p.eps && p.eps[e] > 0.0) dte = fmin(dte, h * h / (p.eps[e] * p.pfac * p.pfac));
  atomicMin(p.out, (unsigned long long)__double_as_longlong(dte));
}

// ---------------------------------------------------------------------------
// Residual partials (residual_norm, solver.cpp:572-590): per-block max|d| or
// sum d^2 in a fixed order (deterministic run to run).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_residual(const double* __restrict__ a, const double* __restrict__ b,
                                                  size_t n, int kind, double* partial) {
  __shared__ double red[256];
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double d = a[i] - b[i];
    acc = kind == 1 ? acc + d * d : fmax(acc, fabs(d));
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (threadIdx.x < s)
      red[threadIdx.x] = kind == 1 ? red[threadIdx.x] + red[threadIdx.x + s]
                                   : fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// ---------------------------------------------------------------------------
// Halo face traces: dir 0 packs traces[(elem, face)] -> buf, dir 1 unpacks.
// idx[i] = elem*4 + face; buf[i][5][ng].
// ---------------------------------------------------------------------------
__global__ void k_halo_copy(double* traces, double* buf, const int* idx, int n, int ng, int tb, int dir) {
  const int item = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (item >= n) return;
  const int ef = idx[item], elem = ef >> 2, face = ef & 3;
  for (int k = threadIdx.x & 31; k < 5 * ng; k += 32) {
    const int c = k / ng, gq = k % ng;
    double* t = traces + ((size_t)elem * 5 + c) * tb + face * ng + gq;
    double* s = buf + ((size_t)item * 5 + c) * ng + gq;
    if (dir == 0)
      *s = *t;
    else
      *t = *s;
  }
}

// Halo payload rows of the multi-rank driver: row i of buf (width W doubles)
// holds, for the face (elem, face) = idx[i] >> 2, idx[i] & 3, the 5 N_g face
// values of each of `nplanes` trace-layout arrays (plane p at buf[i W + p 5 N_g])
// and, when eps is given, eps[elem] after them. dir 0 packs (arrays -> buf),
// 1 unpacks (buf -> the ghost rows). One warp per row.
struct HaloXfer {
  double* plane[3];
  int nplanes;
  double* eps;
  double* buf;
  const int* idx;
  int n, ng, tb, W, dir;
};

__global__ void __launch_bounds__(256) k_halo_xfer(HaloXfer x) {
  const int item = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (item >= x.n) return;
  const int ef = __ldg(x.idx + item), elem = ef >> 2, face = ef & 3;
  double* row = x.buf + (size_t)item * x.W;
  for (int pl = 0; pl < x.nplanes; ++pl)
    for (int k = lane; k < 5 * x.ng; k += 32) {
      const int c = k / x.ng, gq = k - c * x.ng;
      double* t = x.plane[pl] + ((size_t)elem * 5 + c) * x.tb + face * x.ng + gq;
      double* s = row + pl * 5 * x.ng + k;
      if (x.dir == 0)
        *s = *t;
      else
        *t = *s;
    }
  if (x.eps && lane == 0) {
    double* s = row + x.nplanes * 5 * x.ng;
    if (x.dir == 0)
      *s = x.eps[elem];
    else
      x.eps[elem] = *s;
  }
}

// max over the ranks' local max-eps words (u64 bit patterns of non-negative
// doubles order like the values): the viscous gate of an in-process
// multi-rank group (peer pointers; NVLink loads across devices)
__global__ void k_gate_max(const unsigned long long* const* src, int n, unsigned long long* dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long m = 0;
    for (int i = 0; i < n; ++i) m = max(m, *(volatile const unsigned long long*)src[i]);
    *dst = m;
  }
}

// ---------------------------------------------------------------------------
// p_refine_embed (solver.cpp:528-549): out(e, c) = E in(e, c), one warp per
// (element, field) row, lanes over the target nodes.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_embed(const double* __restrict__ in, double* __restrict__ out,
                                               const double* __restrict__ E, int rows, int np_in, int bp_in,
                                               int np_out, int bp_out) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* src = in + (size_t)row * bp_in;
  for (int i = lane; i < bp_out; i += 32) {
    double s = 0.0;
    if (i < np_out)
      for (int j = 0; j < np_in; ++j) s += __ldg(E + (size_t)i * np_in + j) * __ldg(src + j);
    out[(size_t)row * bp_out + i] = s;
  }
}

// freestream_store (solver.cpp:559-568): u(e, c)[i] = u_inf[c], padding 0
__global__ void __launch_bounds__(256) k_fill_freestream(double* u, GasParams gp, size_t rows, int np, int bp) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * bp) return;
  const int i = (int)(idx % bp);
  const int c = (int)((idx / bp) % 5);
  u[idx] = i < np ? gp.fs[c] : 0.0;
}
#endif  // CDG_SET_TU

}  // namespace cdg_gpu
