// cdg_kernels.cuh -- sm_100a kernels of the RKDG hot path (affine tets).
//
// Math (per element e, field c; reference: solver.cpp:325-492):
//   U_cub   = I_cub U                                         (solver.cpp:362-363)
//   F_d     = Euler flux at cubature nodes                    (solver.cpp:374-395)
//   G_m     = sum_d (dr_m/dx_d) F_d        (contravariant flux; J cancels)
//   F*      = LLF/HLLC(U-, U+, n) at face nodes               (solver.cpp:415-456)
//   rhs     = sum_m A_m G_m - LIFT ((sjac_f / J) F*)
// with the shared (per-level) operators
//   A_m  = M_ref^-1 D_m^T diag(W),  LIFT = M_ref^-1 I_g^T diag(w_face),
//   M_ref = I_cub^T diag(W) I_cub,
// which is the reference's  M_e^-1 (sum S_m F_m - M_dOmega F*)  for affine
// elements (M_e = J M_ref, S_m = J sum_k D_k^T diag(W r_{k,m}); operators.cpp:
// 135-165) with the Cholesky solve folded into the operators.
//
// Layout: a "row" is one (element, field) pair; the tile's 5E rows are
// contiguous rows of the SolutionStore matrix [K*5][block] (offset(e,c) =
// (e*5+c)*block, solution_store.hpp:29-31). All three contractions are
//   Out[rows x N] = In[rows x K] * Op^T
// on the FP64 tensor pipe (DMMA, mma.sync.m16n8k4.f64): In (A operand) is
// staged in shared memory, Op (B operand) is pre-swizzled on the host into
// fragment order so each warp's B fragment is one coalesced 256-byte L1/L2 load.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cdg_gpu {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
// Device row length of the state (u, res, rhs: N_p values) and of the face
// traces (4 N_g values): the values rounded up to the 8-wide k-step of the
// DMMA contractions (the padding columns hold exact zeros, so every A-fragment
// load and every epilogue store of a k-step stays inside its own row). The
// reference's SolutionStore pads to 16 (padded.hpp:12); that is the CALLER's
// layout -- set/get_state convert (cudaMemcpy2D) -- while HBM holds the
// tighter rows: P=4 40 instead of 48 doubles (-17% state traffic), P=3 24
// instead of 32, P=1 8 instead of 16.
__host__ __device__ constexpr int dev_block(int values) { return round_up(values, 8); }
// Face-trace rows (4 N_g values, always a multiple of 4): only pairs of
// values are ever loaded or stored together, so the rows stay unpadded (P=1:
// 12 instead of 16 doubles).
__host__ __device__ constexpr int dev_tblock(int nf) { return round_up(nf, 4); }
__host__ __device__ constexpr int ceil_div(int x, int m) { return (x + m - 1) / m; }
// leading dimension >= n with ld % 16 in {4, 12}: conflict-free A-fragment
// loads (8 rows x 4 consecutive doubles per warp)
__host__ __device__ constexpr int frag_ld(int n) {
  return (n % 16 == 4 || n % 16 == 12) ? n : frag_ld(n + 4);
}
__host__ __device__ constexpr int imax(int a, int b) { return a > b ? a : b; }

// leading dimension >= n with ld % 16 == 8: conflict-free 128-bit A-fragment
// loads from the k8-permuted layout (see pcol)
__host__ __device__ constexpr int frag_ld8(int n) { return (n % 16 == 8) ? n : frag_ld8(n + 8); }

template <int NP_, int NCUB_, int NG_, int E_, int CH_ = 16, int MINB_ = 1, int FCH_ = 32, int NW_ = 8>
struct Cfg {
  static constexpr int NP = NP_, NCUB = NCUB_, NG = NG_, NF = 4 * NG_, E = E_;
  static constexpr int NW = NW_, NTH = 32 * NW_;  // warps / threads per CTA (k_rhs)
  static constexpr int MINB = MINB_;              // resident CTAs per SM (launch bounds)
  static constexpr int R = 5 * E;                 // rows per tile
  static constexpr int MT = R / 16;               // m16 tiles per tile
  static constexpr int BP = dev_block(NP);        // device SolutionStore block (see dev_block)
  static constexpr int TB = dev_tblock(NF);       // device trace block
  static constexpr int KP = round_up(NP, 8);      // K of the node->point GEMMs (k8 steps)
  static constexpr int KS1 = KP / 8;
  static constexpr int NCUB8 = round_up(NCUB, 8);
  static constexpr int NP8 = round_up(NP, 8);
  static constexpr int NF8 = round_up(NF, 8);
  static constexpr int NT2 = NP8 / 8;             // n-tiles of the RHS GEMM
  static constexpr int CH = CH_;                  // cubature nodes per chunk (multiple of 8)
  static constexpr int NCH = ceil_div(NCUB8, CH);
  static constexpr int FCH = FCH_;                // face nodes per chunk (multiple of 8)
  static constexpr int NFCH = ceil_div(NF, FCH);
  static constexpr int K2CUB = 3 * NCUB8;         // volume part of the RHS K
  static constexpr int K2 = K2CUB + NF8;          // + face part (padded to 8)
  static constexpr int KS2 = K2 / 8;
  static constexpr int LDU = frag_ld8(KP);
  static constexpr int LDC = CH + 4;
  static constexpr int LDG = frag_ld8(imax(3 * CH, FCH));
  static constexpr int T2 = MT * NT2;             // RHS output tiles
  static constexpr int MAXT2 = ceil_div(T2, NW);
  // one m-tile row per warp (NW == MT): the warp's A fragment is loaded once
  // per k-step and reused across all NT2 n-tiles
  static constexpr bool WROW = (NW == MT);
  static constexpr int T1MAX = MT * (CH / 8);     // GEMM1 tiles per chunk
  static constexpr int MAXT1 = (NW == MT) ? CH / 8 : ceil_div(T1MAX, NW);
  static constexpr int IT_P = ceil_div(E * CH, NTH);   // pointwise pairs per thread
  static constexpr int IT_F = ceil_div(E * FCH, NTH);  // face pairs per thread
  static constexpr int SMEM_U = R * LDU;
  static constexpr int SMEM_C = R * LDC;
  static constexpr int SMEM_G = R * LDG;
  static constexpr size_t SMEM_BYTES =
      sizeof(double) * (SMEM_U + SMEM_C + SMEM_G + E * 9 + E * 4 * 4 + E) +
      sizeof(int) * (E * 4 * 2);
};

// Column permutation inside each 8-column group so that a thread's two k8
// A-fragment values (k = t and t+4) are adjacent: one 128-bit shared load.
__host__ __device__ __forceinline__ int pcol(int k) { return (k & ~7) | ((k & 3) << 1) | ((k >> 2) & 1); }

// Launch gate for graph-captured viscous stages: the decision viscous_active
// (max eps > 0, solver.cpp:257-259) is made on the device by the sensor; a
// gated kernel returns at once (grid-uniform) unless (max eps bits != 0) ==
// run_if_active. gate == nullptr: always run.
__device__ __forceinline__ bool gated_off(const unsigned long long* gate, int run_if_active) {
  return gate && ((*(volatile const unsigned long long*)gate != 0ull) != (run_if_active != 0));
}

// First-error record (the reference's RhsWorkspace::record_error,
// solver.cpp:54-69, made device-side: first writer wins).
struct DevError {
  int flag;   // 0 none, 1 set
  int kind;   // 1 cub-node state, 2 trace state, 3 timestep state
  int elem;
  int a;      // cub node / face
  int b;      // face node
  int pad;
  double value;
};

__device__ __forceinline__ void record_error(DevError* err, int kind, int elem, int a, int b,
                                             double value) {
  if (atomicCAS(&err->flag, 0, 1) == 0) {
    err->kind = kind;
    err->elem = elem;
    err->a = a;
    err->b = b;
    err->value = value;
    __threadfence();
  }
}

// Per-stage coefficients, read from global so that captured graphs stay valid
// when dt / a / b change (solver.cpp:476-488).
struct StageCoef {
  double dt;
  double a[5];
  double b[5];
};

struct GasParams {
  double gamma;
  double fs[5];  // freestream
  int riemann;   // 0 llf, 1 hllc
  unsigned long long* hllc_fallbacks;  // RhsWorkspace::hllc_fallbacks (solver.cpp:52,436), may be null
};

// ---------------------------------------------------------------------------
// DMMA helper: D(16x8) += A(16x4, row) * B(4x8, col), fp64.
// A frag: a0=(g, t) a1=(g+8, t); B frag: b0=(k=t, n=g); C: c0,c1=(g, 2t..2t+1),
// c2,c3=(g+8, 2t..2t+1)   with g = lane/4, t = lane%4.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_k4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// D(16x8) += A(16x8, row) * B(8x8, col), fp64: the native DMMA shape on
// sm_100 (m16n8k4 lowers to two DMMA.8x8x4 and reaches only ~80% of the
// measured FP64 peak; profiles/r1). A: a0=(g,t) a1=(g+8,t) a2=(g,t+4)
// a3=(g+8,t+4); B: b0=(k=t,n=g) b1=(k=t+4,n=g).
__device__ __forceinline__ void dmma_k8(double (&d)[4], double a0, double a1, double a2, double a3,
                                        double b0, double b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

struct AFrag {
  double a0, a1, a2, a3;
};
// A fragment of m-tile rows [r0, r0+16) at k8 step k0 from a pcol-permuted panel
__device__ __forceinline__ AFrag load_afrag(const double* s, int ld, int r0, int k0, int g, int tq) {
  const double2 x = *reinterpret_cast<const double2*>(s + (r0 + g) * ld + k0 + 2 * tq);
  const double2 y = *reinterpret_cast<const double2*>(s + (r0 + g + 8) * ld + k0 + 2 * tq);
  return AFrag{x.x, y.x, x.y, y.y};
}
__device__ __forceinline__ void mma_frag(double (&d)[4], const AFrag& a, const double2 b) {
  dmma_k8(d, a.a0, a.a1, a.a2, a.a3, b.x, b.y);
}

// Stage rows [row0, row0+R) of a [*][BP] store into a pcol-permuted panel.
template <class C, int NTH = kThreads>
__device__ __forceinline__ void stage_rows(const double* __restrict__ src, int row0, int n_rows, double* s,
                                           int tid) {
  constexpr int V8 = C::KP / 8;
  for (int idx = tid; idx < C::R * V8 * 2; idx += NTH) {
    const int h = idx & 1, j = (idx >> 1) % V8, r = (idx >> 1) / V8;
    double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
    if (row0 + r < n_rows) {
      const double* p = src + (size_t)(row0 + r) * C::BP + 8 * j + 2 * h;
      x = *reinterpret_cast<const double2*>(p);
      y = *reinterpret_cast<const double2*>(p + 4);
    }
    double* o = s + r * C::LDU + 8 * j + 4 * h;
    *reinterpret_cast<double2*>(o) = make_double2(x.x, y.x);
    *reinterpret_cast<double2*>(o + 2) = make_double2(x.y, y.y);
  }
}

// ---------------------------------------------------------------------------
// Euler state algebra (euler.cpp:7-161), device versions.
// ---------------------------------------------------------------------------
struct State5 {
  double r, mx, my, mz, E;
};

__device__ __forceinline__ bool admissible(const State5& u, double gamma) {
  if (u.r <= 0.0) return false;
  return (u.E - (u.mx * u.mx + u.my * u.my + u.mz * u.mz) / (2.0 * u.r)) > 0.0 && gamma > 1.0;
}

__device__ __forceinline__ double pressure(const State5& u, double gamma) {
  return (gamma - 1.0) * (u.E - (u.mx * u.mx + u.my * u.my + u.mz * u.mz) / (2.0 * u.r));
}

// flux_dot_n (euler.cpp:42-50)
__device__ __forceinline__ void flux_dot_n(const State5& u, double p, double nx, double ny,
                                           double nz, double (&f)[5]) {
  const double vn = (u.mx * nx + u.my * ny + u.mz * nz) / u.r;
  f[0] = u.r * vn;
  f[1] = u.mx * vn + p * nx;
  f[2] = u.my * vn + p * ny;
  f[3] = u.mz * vn + p * nz;
  f[4] = vn * (u.E + p);
}

// llf_flux (euler.cpp:59-68)
__device__ __forceinline__ void llf_flux(const State5& um, const State5& up, double nx, double ny,
                                         double nz, double gamma, double (&out)[5]) {
  const double pm = pressure(um, gamma), pp = pressure(up, gamma);
  const double lm = fabs((um.mx * nx + um.my * ny + um.mz * nz) / um.r) + sqrt(gamma * pm / um.r);
  const double lp = fabs((up.mx * nx + up.my * ny + up.mz * nz) / up.r) + sqrt(gamma * pp / up.r);
  const double lambda = fmax(lm, lp);
  double fm[5], fp[5];
  flux_dot_n(um, pm, nx, ny, nz, fm);
  flux_dot_n(up, pp, nx, ny, nz, fp);
  const double dm[5] = {up.r - um.r, up.mx - um.mx, up.my - um.my, up.mz - um.mz, up.E - um.E};
#pragma unroll
  for (int c = 0; c < 5; ++c) out[c] = 0.5 * (fm[c] + fp[c]) - 0.5 * lambda * dm[c];
}

// llf_flux with one reciprocal per side (rounding differs from the reference's
// divisions at the 1-ulp level; parity budget 1e-12)
__device__ __forceinline__ void llf_flux_fast(const State5& um, const State5& up, double nx, double ny,
                                              double nz, double gamma, double (&out)[5]) {
  const double im = 1.0 / um.r, ip = 1.0 / up.r;
  const double pm = (gamma - 1.0) * (um.E - 0.5 * im * (um.mx * um.mx + um.my * um.my + um.mz * um.mz));
  const double pp = (gamma - 1.0) * (up.E - 0.5 * ip * (up.mx * up.mx + up.my * up.my + up.mz * up.mz));
  const double vm = (um.mx * nx + um.my * ny + um.mz * nz) * im;
  const double vp = (up.mx * nx + up.my * ny + up.mz * nz) * ip;
  const double lambda = fmax(fabs(vm) + sqrt(gamma * pm * im), fabs(vp) + sqrt(gamma * pp * ip));
  const double fm[5] = {um.r * vm, um.mx * vm + pm * nx, um.my * vm + pm * ny, um.mz * vm + pm * nz,
                        vm * (um.E + pm)};
  const double fp[5] = {up.r * vp, up.mx * vp + pp * nx, up.my * vp + pp * ny, up.mz * vp + pp * nz,
                        vp * (up.E + pp)};
  const double dm[5] = {up.r - um.r, up.mx - um.mx, up.my - um.my, up.mz - um.mz, up.E - um.E};
#pragma unroll
  for (int c = 0; c < 5; ++c) out[c] = 0.5 * (fm[c] + fp[c]) - 0.5 * lambda * dm[c];
}

// hllc_flux with Einfeldt/Roe bounds and LLF fallback (euler.cpp:70-138)
__device__ __forceinline__ void hllc_flux(const State5& um, const State5& up, double nx, double ny,
                                          double nz, double g, double (&out)[5]) {
  const double pl = pressure(um, g), pr = pressure(up, g);
  const double vlx = um.mx / um.r, vly = um.my / um.r, vlz = um.mz / um.r;
  const double vrx = up.mx / up.r, vry = up.my / up.r, vrz = up.mz / up.r;
  const double unl = vlx * nx + vly * ny + vlz * nz;
  const double unr = vrx * nx + vry * ny + vrz * nz;
  const double cl = sqrt(g * pl / um.r), cr = sqrt(g * pr / up.r);
  const double sl_ = sqrt(um.r), sr_ = sqrt(up.r);
  const double den = sl_ + sr_;
  const double vx = (sl_ * vlx + sr_ * vrx) / den, vy = (sl_ * vly + sr_ * vry) / den,
               vz = (sl_ * vlz + sr_ * vrz) / den;
  const double hl = (um.E + pl) / um.r, hr = (up.E + pr) / up.r;
  const double h_roe = (sl_ * hl + sr_ * hr) / den;
  const double c2_roe = (g - 1.0) * (h_roe - 0.5 * (vx * vx + vy * vy + vz * vz));
  const double un_roe = vx * nx + vy * ny + vz * nz;
  double s_left, s_right;
  if (c2_roe <= 0.0) {
    s_left = fmin(unl - cl, unr - cr);
    s_right = fmax(unl + cl, unr + cr);
  } else {
    const double c_roe = sqrt(c2_roe);
    s_left = fmin(unl - cl, un_roe - c_roe);
    s_right = fmax(unr + cr, un_roe + c_roe);
  }
  if (!(s_left < s_right)) {
    llf_flux(um, up, nx, ny, nz, g, out);
    return;
  }
  const double s_star = (pr - pl + um.r * unl * (s_left - unl) - up.r * unr * (s_right - unr)) /
                        (um.r * (s_left - unl) - up.r * (s_right - unr));
  if (!isfinite(s_star)) {
    llf_flux(um, up, nx, ny, nz, g, out);
    return;
  }
  if (0.0 <= s_left) {
    flux_dot_n(um, pl, nx, ny, nz, out);
    return;
  }
  if (0.0 >= s_right) {
    flux_dot_n(up, pr, nx, ny, nz, out);
    return;
  }
  const bool left = 0.0 <= s_star;
  const State5& u = left ? um : up;
  const double un_k = left ? unl : unr, p_k = left ? pl : pr, s_k = left ? s_left : s_right;
  const double factor = u.r * (s_k - un_k) / (s_k - s_star);
  const double vx_ = u.mx / u.r, vy_ = u.my / u.r, vz_ = u.mz / u.r;
  const double ds = s_star - un_k;
  const double star[5] = {factor, factor * (vx_ + ds * nx), factor * (vy_ + ds * ny),
                          factor * (vz_ + ds * nz),
                          factor * (u.E / u.r + ds * (s_star + p_k / (u.r * (s_k - un_k))))};
  double f[5];
  flux_dot_n(u, p_k, nx, ny, nz, f);
  const double uu[5] = {u.r, u.mx, u.my, u.mz, u.E};
#pragma unroll
  for (int c = 0; c < 5; ++c) out[c] = f[c] + s_k * (star[c] - uu[c]);
}

// hllc_flux with one reciprocal per side and one for the Roe average (the
// reference divides at every use, euler.cpp:70-138; rounding differs at the
// 1e-16 level, the branch structure and the LLF fallback are the same)
__device__ __forceinline__ void hllc_flux_fast(const State5& um, const State5& up, double nx, double ny,
                                               double nz, double g, double (&out)[5],
                                               unsigned long long* fallbacks = nullptr) {
  const double il = 1.0 / um.r, ir = 1.0 / up.r;
  const double pl = (g - 1.0) * (um.E - 0.5 * il * (um.mx * um.mx + um.my * um.my + um.mz * um.mz));
  const double pr = (g - 1.0) * (up.E - 0.5 * ir * (up.mx * up.mx + up.my * up.my + up.mz * up.mz));
  const double vlx = um.mx * il, vly = um.my * il, vlz = um.mz * il;
  const double vrx = up.mx * ir, vry = up.my * ir, vrz = up.mz * ir;
  const double unl = vlx * nx + vly * ny + vlz * nz;
  const double unr = vrx * nx + vry * ny + vrz * nz;
  const double cl = sqrt(g * pl * il), cr = sqrt(g * pr * ir);
  const double sl_ = sqrt(um.r), sr_ = sqrt(up.r);
  const double iden = 1.0 / (sl_ + sr_);
  const double vx = (sl_ * vlx + sr_ * vrx) * iden, vy = (sl_ * vly + sr_ * vry) * iden,
               vz = (sl_ * vlz + sr_ * vrz) * iden;
  const double hl = (um.E + pl) * il, hr = (up.E + pr) * ir;
  const double h_roe = (sl_ * hl + sr_ * hr) * iden;
  const double c2_roe = (g - 1.0) * (h_roe - 0.5 * (vx * vx + vy * vy + vz * vz));
  const double un_roe = vx * nx + vy * ny + vz * nz;
  double s_left, s_right;
  if (c2_roe <= 0.0) {
    s_left = fmin(unl - cl, unr - cr);
    s_right = fmax(unl + cl, unr + cr);
  } else {
    const double c_roe = sqrt(c2_roe);
    s_left = fmin(unl - cl, un_roe - c_roe);
    s_right = fmax(unr + cr, un_roe + c_roe);
  }
  if (!(s_left < s_right)) {  // LLF fallback, counted (euler.cpp:99-102)
    if (fallbacks) atomicAdd(fallbacks, 1ULL);
    llf_flux_fast(um, up, nx, ny, nz, g, out);
    return;
  }
  const double s_star = (pr - pl + um.r * unl * (s_left - unl) - up.r * unr * (s_right - unr)) /
                        (um.r * (s_left - unl) - up.r * (s_right - unr));
  if (!isfinite(s_star)) {  // (euler.cpp:106-109)
    if (fallbacks) atomicAdd(fallbacks, 1ULL);
    llf_flux_fast(um, up, nx, ny, nz, g, out);
    return;
  }
  const bool left = 0.0 <= s_star;
  const bool sup_l = 0.0 <= s_left, sup_r = 0.0 >= s_right;  // supersonic: plain one-sided flux
  const bool use_l = sup_l || (!sup_r && left);
  const State5& u = use_l ? um : up;
  const double iu = use_l ? il : ir;
  const double un_k = use_l ? unl : unr, p_k = use_l ? pl : pr;
  double f[5] = {u.r * un_k, u.mx * un_k + p_k * nx, u.my * un_k + p_k * ny, u.mz * un_k + p_k * nz,
                 un_k * (u.E + p_k)};
  if (!(sup_l || sup_r)) {
    const double s_k = left ? s_left : s_right;
    const double dk = s_k - un_k;
    const double factor = u.r * dk / (s_k - s_star);
    const double ds = s_star - un_k;
    const double star[5] = {factor, factor * (u.mx * iu + ds * nx), factor * (u.my * iu + ds * ny),
                            factor * (u.mz * iu + ds * nz), factor * (u.E * iu + ds * (s_star + p_k * iu / dk))};
    const double uu[5] = {u.r, u.mx, u.my, u.mz, u.E};
#pragma unroll
    for (int c = 0; c < 5; ++c) f[c] += s_k * (star[c] - uu[c]);
  }
#pragma unroll
  for (int c = 0; c < 5; ++c) out[c] = f[c];
}

// boundary_state (euler.cpp:147-161)
__device__ __forceinline__ State5 boundary_state(const State5& in, double nx, double ny, double nz,
                                                 int kind, const GasParams& gp) {
  if (kind == 1) return State5{gp.fs[0], gp.fs[1], gp.fs[2], gp.fs[3], gp.fs[4]};
  State5 gh = in;
  const double mn = in.mx * nx + in.my * ny + in.mz * nz;
  gh.mx = in.mx - 2.0 * mn * nx;
  gh.my = in.my - 2.0 * mn * ny;
  gh.mz = in.mz - 2.0 * mn * nz;
  return gh;
}

// Face coupling word: bits 0-1 neighbour face, 2-3 bc kind, 4 boundary flag,
// 5 (face 0 only) element is curved -> handled by k_rhs_curved, 8-31 node-map code.
constexpr int kCurvedBit = 1 << 5;
__host__ __device__ constexpr int pack_face(int nface, int bc, int boundary, int code) {
  return (nface & 3) | ((bc & 3) << 2) | ((boundary & 1) << 4) | (code << 8);
}

// ---------------------------------------------------------------------------
// Kernel 1: nodal -> point interpolation  Out[rows x NO] = U[rows x KP] * Op^T
// with Op = I_g (traces, solver.cpp:200-208; NO = N_f, LDO = pad16(N_f)) or
// Op = I_cub (the aux gradient at the cubature nodes for the viscous volume
// term, solver.cpp:364-369; NO = N_cub). Non-persistent (one tile per CTA,
// several CTAs per SM): memory-bound.
// ---------------------------------------------------------------------------
// NAT: the U panel is staged in natural node order and frag_op uses the natural
// pairing (k = t <-> node 8ks+2t, k = t+4 <-> 8ks+2t+1; cdg_warp.cuh), which is
// the pairing the row kernel's fused traces use -- both then agree bit for bit.
template <class C, int NO, int LDO, bool NAT = false>
__global__ void __launch_bounds__(kThreads)
k_interp(const double* __restrict__ u, double* __restrict__ out, const double* __restrict__ frag_op, int n_rows,
         int n_tiles, const unsigned long long* gate, int gate_when) {
  if (gated_off(gate, gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  constexpr int NT = round_up(NO, 8) / 8;
  constexpr int T = C::MT * NT;
  const double2* fb = reinterpret_cast<const double2*>(frag_op);
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int row0 = tile * C::R;
    if (NAT) {
      constexpr int V = C::KP / 2;
      for (int idx = tid; idx < C::R * V; idx += kThreads) {
        const int r = idx / V, j = idx - r * V;
        double2 x = make_double2(0.0, 0.0);
        if (row0 + r < n_rows) x = *reinterpret_cast<const double2*>(u + (size_t)(row0 + r) * C::BP + 2 * j);
        *reinterpret_cast<double2*>(sU + r * C::LDU + 2 * j) = x;
      }
    } else {
      stage_rows<C>(u, row0, n_rows, sU, tid);
    }
    __syncthreads();
    for (int t = warp; t < T; t += kWarps) {
      const int mt = t / NT, nt = t % NT;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < C::KS1; ++ks)
        mma_frag(acc, load_afrag(sU, C::LDU, mt * 16, ks * 8, g, tq), __ldg(fb + ((size_t)nt * C::KS1 + ks) * 32 + lane));
      const int col = nt * 8 + 2 * tq;
      if (col < NO) {
        const int r0 = row0 + mt * 16 + g;
        if (r0 < n_rows)
          *reinterpret_cast<double2*>(out + (size_t)r0 * LDO + col) = make_double2(acc[0], acc[1]);
        if (r0 + 8 < n_rows)
          *reinterpret_cast<double2*>(out + (size_t)(r0 + 8) * LDO + col) = make_double2(acc[2], acc[3]);
      }
    }
    __syncthreads();
  }
}

// Normal component of the aux-gradient traces, the only combination the BR1
// viscous face term uses (solver.cpp:438-453: sum_m 0.5 (se q_m + snb q_m^+) n_m):
//   qn[e][c][fq] = sum_m n_m(e, fq) (I_g q_m)[e][c][fq]
// the three q_m tiles staged like k_interp<NAT> (same fragments and pairing,
// so each I_g q_m equals the trace kernel's bit for bit), projected on the
// element's own outward normal at the face node (per face on straight
// elements, per face node on curved ones). The consumer flips the sign of a
// neighbour's value (its outward normal is -n at the paired node). One row
// of 5 N_g values per face instead of 15.
// rows per CTA pass of k_qn_traces: two m16 blocks (AV step at 82,944 curved
// P=4 tets: 16 / 32 / 48 / 80 rows -> 27.9 / 27.4 / 27.5 / 27.5 ms); the
// three panels fit shared memory at every order (p=8: 129 KB)
template <class C>
__host__ __device__ constexpr int qn_block_rows() { return 32; }

template <class C>
__global__ void __launch_bounds__(kThreads)
k_qn_traces(const double* __restrict__ q, size_t qstride, double* __restrict__ out, const double* __restrict__ frag_op,
            const double4* __restrict__ face, const double4* __restrict__ curved_face,
            const int* __restrict__ curved_slot, int n_rows, int n_blocks, const unsigned long long* gate,
            int gate_when) {
  if (gated_off(gate, gate_when)) return;
  constexpr int BR = qn_block_rows<C>();
  extern __shared__ __align__(16) double smem[];  // [3][BR][LDU]: a row block of the three q_m
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  constexpr int NT = round_up(C::NF, 8) / 8;
  constexpr int T = (BR / 16) * NT;
  constexpr int V = C::KP / 2;
  const double2* fb = reinterpret_cast<const double2*>(frag_op);
  for (int blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const int row0 = blk * BR;
    for (int idx = tid; idx < 3 * BR * V; idx += kThreads) {
      const int m = idx / (BR * V), rj = idx - m * (BR * V), r = rj / V, j = rj - r * V;
      double2 x = make_double2(0.0, 0.0);
      if (row0 + r < n_rows) x = *reinterpret_cast<const double2*>(q + m * qstride + (size_t)(row0 + r) * C::BP + 2 * j);
      *reinterpret_cast<double2*>(smem + (m * BR + r) * C::LDU + 2 * j) = x;
    }
    __syncthreads();
    for (int t = warp; t < T; t += kWarps) {
      const int mt = t / NT, nt = t % NT;
      double acc[3][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
#pragma unroll 4
      for (int ks = 0; ks < C::KS1; ++ks) {
        const double2 b = __ldg(fb + ((size_t)nt * C::KS1 + ks) * 32 + lane);
#pragma unroll
        for (int m = 0; m < 3; ++m) mma_frag(acc[m], load_afrag(smem + m * BR * C::LDU, C::LDU, mt * 16, ks * 8, g, tq), b);
      }
      const int col = nt * 8 + 2 * tq;
      if (col < C::NF) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int r = row0 + mt * 16 + g + 8 * hh;
          if (r >= n_rows) continue;
          const int e = r / 5;
          const int slot = curved_slot ? __ldg(curved_slot + e) : -1;
          double v[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int fq = col + i;
            const double4 n = slot >= 0 ? curved_face[(size_t)slot * C::NF + fq] : face[(size_t)e * 4 + fq / C::NG];
            v[i] = n.x * acc[0][2 * hh + i] + n.y * acc[1][2 * hh + i] + n.z * acc[2][2 * hh + i];
          }
          *reinterpret_cast<double2*>(out + (size_t)r * C::TB + col) = make_double2(v[0], v[1]);
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Kernel 2: fused volume + surface + lift (+ low-storage RK update)
// ---------------------------------------------------------------------------
struct RhsParams {
  double* u;                  // [K*5][BP]    (updated in place when UPDATE)
  double* res;                // [K*5][BP]
  double* rhs_out;            // [K*5][BP]    (RHS-only mode)
  const double* traces;       // [(K+halo)*5][TB]
  const double* metric;       // [K][9]
  const double4* face;        // [K][4] (nx, ny, nz, sjac/J)
  const int2* conn;           // [K][4] (neighbour, packed word)
  const int* code_map;        // [n_codes][NG]
  const double* frag_icub;    // GEMM1 B fragments
  const double* frag_op2;     // GEMM2 B fragments
  const StageCoef* coef;
  int stage;
  int K;
  int n_tiles;
  int elem_offset;            // global element id of local element 0 (messages)
  GasParams gas;
  DevError* err;
  // viscous extension (solver.cpp:364-369, 398-406, 438-453)
  const double* q;            // [3][K*5][BP]   aux gradient q_m
  const double* qtr;          // [3][(K+halo)*5][TB] its traces
  const double* sqrt_eps;     // [K+halo]
  const double* qcub;         // [3][K*5][round_up(NCUB, 8)] I_cub q_m (viscous volume term)
  size_t qtr_stride;          // elements per direction of qtr
  int prefetch;               // L2 prefetch mask: 1 res, 2 next-tile u, 4 own traces, 8 neighbour traces
  const int* tiles;           // optional tile list (multi-GPU interior / halo split); null = all tiles
  int n_list;                 // entries of `tiles`
  const unsigned long long* gate;  // optional launch gate (see gated_off)
  int gate_when;
  double* traces_out;         // fused traces of u_new (k_rhs_row MODE 32)
  const double* frag_ig_nat;  // I_g B fragments, natural pairing
};

// i-th tile of a launch: the tile list when given, else tile i
__device__ __forceinline__ int tile_at(const RhsParams& p, int i) { return p.tiles ? __ldg(p.tiles + i) : i; }

__device__ __forceinline__ void l2_prefetch(const void* ptr) { asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr)); }

// Touch `bytes` bytes from `base` (128-byte lines) into L2, lines spread over the CTA.
__device__ __forceinline__ void l2_prefetch_range(const void* base, size_t bytes, int tid, int nthreads) {
  const char* b = reinterpret_cast<const char*>(base);
  for (size_t off = (size_t)tid * 128; off < bytes; off += (size_t)nthreads * 128) l2_prefetch(b + off);
}

// GEMM1 for one cubature chunk: sC[:, 0:w] = U * I_cub[q0:q0+w, :]^T
template <class C>
__device__ __forceinline__ void gemm1_chunk(const double* sU, double* sC, const double2* fb, int q0, int w,
                                            int warp, int lane) {
  const int g = lane >> 2, tq = lane & 3;
  const int nt1 = w / 8, T1 = C::MT * nt1;
  double c[C::MAXT1][4];
#pragma unroll
  for (int i = 0; i < C::MAXT1; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  // tile i of this warp: WROW -> (m-tile warp, n-tile i), else round robin
#pragma unroll
  for (int ks = 0; ks < C::KS1; ++ks) {
    if constexpr (C::WROW) {
      const AFrag a = load_afrag(sU, C::LDU, warp * 16, ks * 8, g, tq);
#pragma unroll
      for (int i = 0; i < C::MAXT1; ++i)
        if (i < nt1) mma_frag(c[i], a, __ldg(fb + ((size_t)(q0 / 8 + i) * C::KS1 + ks) * 32 + lane));
    } else {
#pragma unroll
      for (int i = 0; i < C::MAXT1; ++i) {
        const int t = warp + i * C::NW;
        if (t < T1) {
          const int mt = t / nt1, nt = t % nt1;
          mma_frag(c[i], load_afrag(sU, C::LDU, mt * 16, ks * 8, g, tq),
                   __ldg(fb + ((size_t)(q0 / 8 + nt) * C::KS1 + ks) * 32 + lane));
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < C::MAXT1; ++i) {
    int mt, nt;
    bool ok;
    if constexpr (C::WROW) {
      mt = warp;
      nt = i;
      ok = i < nt1;
    } else {
      const int t = warp + i * C::NW;
      ok = t < T1;
      mt = ok ? t / nt1 : 0;
      nt = ok ? t % nt1 : 0;
    }
    if (ok) {
      double* o = sC + (mt * 16 + g) * C::LDC + nt * 8 + 2 * tq;
      *reinterpret_cast<double2*>(o) = make_double2(c[i][0], c[i][1]);
      *reinterpret_cast<double2*>(o + 8 * C::LDC) = make_double2(c[i][2], c[i][3]);
    }
  }
}

// GEMM2 partial: acc[warp tiles] += sG[:, 0:8*nks] * Op2[:, k0:...]^T
// (k-steps outer, the warp's independent output tiles inner for ILP)
template <class C, int NKS>
__device__ __forceinline__ void gemm2_fixed(double (&acc)[C::MAXT2][4], const double* sG, const double2* fb,
                                            int ks0, int t_begin, int t_end, int lane) {
  const int g = lane >> 2, tq = lane & 3;
  if constexpr (C::WROW) {
    const int mt = t_begin / C::NT2;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      const AFrag a = load_afrag(sG, C::LDG, mt * 16, ks * 8, g, tq);
#pragma unroll
      for (int i = 0; i < C::NT2; ++i) mma_frag(acc[i], a, __ldg(fb + ((size_t)i * C::KS2 + ks0 + ks) * 32 + lane));
    }
  } else {
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) {
        const int t = t_begin + i;
        if (t < t_end) {
          const int nt = t / C::MT, mt = t % C::MT;
          mma_frag(acc[i], load_afrag(sG, C::LDG, mt * 16, ks * 8, g, tq),
                   __ldg(fb + ((size_t)nt * C::KS2 + ks0 + ks) * 32 + lane));
        }
      }
    }
  }
}

template <class C>
__device__ __forceinline__ void gemm2_partial(double (&acc)[C::MAXT2][4], const double* sG, const double2* fb,
                                              int ks0, int nks, int t_begin, int t_end, int lane) {
  const int g = lane >> 2, tq = lane & 3;
  if constexpr (C::WROW) {
    const int mt = t_begin / C::NT2;
    for (int ks = 0; ks < nks; ++ks) {
      const AFrag a = load_afrag(sG, C::LDG, mt * 16, ks * 8, g, tq);
#pragma unroll
      for (int i = 0; i < C::NT2; ++i) mma_frag(acc[i], a, __ldg(fb + ((size_t)i * C::KS2 + ks0 + ks) * 32 + lane));
    }
  } else {
    for (int ks = 0; ks < nks; ++ks) {
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) {
        const int t = t_begin + i;
        if (t < t_end) {
          const int nt = t / C::MT, mt = t % C::MT;  // n-major: a warp's run reuses B fragments
          mma_frag(acc[i], load_afrag(sG, C::LDG, mt * 16, ks * 8, g, tq),
                   __ldg(fb + ((size_t)nt * C::KS2 + ks0 + ks) * 32 + lane));
        }
      }
    }
  }
}

// output tile i of this warp -> (m-tile, n-tile)
template <class C>
__device__ __forceinline__ void tile_coords(int t_begin, int i, int& mt, int& nt) {
  if constexpr (C::WROW) {
    mt = t_begin / C::NT2;
    nt = i;
  } else {
    const int t = t_begin + i;
    nt = t / C::MT;
    mt = t % C::MT;
  }
}

// RM: Riemann solver baked in at compile time (0 LLF, 1 HLLC, -1 runtime
// p.gas.riemann): the LLF-only instantiation needs far fewer registers.
template <class C, bool UPDATE, bool VISC, int RM = -1>
__global__ void __launch_bounds__(C::NTH, C::MINB) k_rhs(RhsParams p) {
  if (gated_off(p.gate, p.gate_when)) return;
  extern __shared__ __align__(16) double smem[];
  double* sU = smem;                       // [R][LDU] nodal state (pcol-permuted)
  double* sC = sU + C::SMEM_U;             // [R][LDC] U at a cubature chunk
  double* sG = sC + C::SMEM_C;             // [R][LDG] flux chunk (A operand, pcol-permuted)
  double* sMet = sG + C::SMEM_G;           // [E][9]
  double4* sFace = reinterpret_cast<double4*>(sMet + C::E * 9);  // [E][4]
  double* sSe = reinterpret_cast<double*>(sFace + C::E * 4);      // [E] sqrt(eps)
  int2* sConn = reinterpret_cast<int2*>(sSe + C::E);              // [E][4]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int n_rows = p.K * 5;
  const double gamma = p.gas.gamma;
  const size_t qstride = (size_t)p.K * 5 * C::BP;
  const double2* fb1 = reinterpret_cast<const double2*>(p.frag_icub);
  const double2* fb2 = reinterpret_cast<const double2*>(p.frag_op2);
  // contiguous run of RHS output tiles for this warp (m-major order)
  const int t_begin = (warp * C::T2) / C::NW, t_end = ((warp + 1) * C::T2) / C::NW;

  __shared__ int s_stop;
  const int n_iter = p.tiles ? p.n_list : p.n_tiles;
  for (int it_t = blockIdx.x; it_t < n_iter; it_t += gridDim.x) {
    const int tile = tile_at(p, it_t);
    // block-uniform early exit after a recorded error (no divergent barriers)
    if (tid == 0) s_stop = *(volatile int*)&p.err->flag;
    __syncthreads();
    if (s_stop) return;
    const int e0 = tile * C::E;
    const int row0 = e0 * 5;
    // ---- L2 prefetch of what this tile reads late (res in the epilogue, traces
    // in the face phase) and of the next tile's state: their HBM latency then
    // overlaps the volume phase instead of stalling the whole CTA.
    if (p.prefetch) {
      const int rows = min(C::R, n_rows - row0);
      if (UPDATE && (p.prefetch & 1)) l2_prefetch_range(p.res + (size_t)row0 * C::BP, (size_t)rows * C::BP * 8, tid, C::NTH);
      if (p.prefetch & 4) l2_prefetch_range(p.traces + (size_t)row0 * C::TB, (size_t)rows * C::TB * 8, tid, C::NTH);
      const int nrow0 = (tile + gridDim.x) * C::R;
      if ((p.prefetch & 2) && nrow0 < n_rows)
        l2_prefetch_range(p.u + (size_t)nrow0 * C::BP, (size_t)min(C::R, n_rows - nrow0) * C::BP * 8, tid, C::NTH);
    }
    // ---- stage nodal state + per-element geometry --------------------------
    stage_rows<C, C::NTH>(p.u, row0, n_rows, sU, tid);
    for (int idx = tid; idx < C::E * 9; idx += C::NTH) {
      const int e = e0 + idx / 9;
      sMet[idx] = e < p.K ? __ldg(p.metric + (size_t)e0 * 9 + idx) : 0.0;
    }
    for (int idx = tid; idx < C::E * 4; idx += C::NTH) {
      const int e = e0 + idx / 4;
      sFace[idx] = e < p.K ? p.face[(size_t)e0 * 4 + idx] : make_double4(0, 0, 1, 0);
      sConn[idx] = e < p.K ? p.conn[(size_t)e0 * 4 + idx] : make_int2(-1, pack_face(0, 0, 1, 0));
    }
    if (VISC)
      for (int idx = tid; idx < C::E; idx += C::NTH)
        sSe[idx] = e0 + idx < p.K ? p.sqrt_eps[e0 + idx] : 0.0;
    __syncthreads();
    if (p.prefetch & 8) {
      // neighbour trace segments (5 fields x one face of N_g nodes each)
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

    double acc[C::MAXT2][4];
#pragma unroll
    for (int i = 0; i < C::MAXT2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;

    // ---- volume: chunks of CH cubature nodes --------------------------------
    for (int ch = 0; ch < C::NCH; ++ch) {
      const int q0 = ch * C::CH;
      const int w = (C::NCUB8 - q0) < C::CH ? (C::NCUB8 - q0) : C::CH;  // 16 or 8
      gemm1_chunk<C>(sU, sC, fb1, q0, w, warp, lane);
      __syncthreads();
      // pointwise Euler flux -> contravariant flux G_m = sum_d (dr_m/dx_d) F_d
#pragma unroll
      for (int it = 0; it < C::IT_P; ++it) {
        const int idx = tid + it * C::NTH;
        if (idx < C::E * w) {
          const int e = idx / w, ql = idx - e * w, q = q0 + ql;
          const double* uc = sC + (e * 5) * C::LDC + ql;
          double* gout = sG + (e * 5) * C::LDG;
          double G[3][5];
          if (q < C::NCUB && e0 + e < p.K) {
            const State5 s{uc[0], uc[C::LDC], uc[2 * C::LDC], uc[3 * C::LDC], uc[4 * C::LDC]};
            if (!admissible(s, gamma)) record_error(p.err, 1, p.elem_offset + e0 + e, q, 0, s.r);
            const double ir = 1.0 / s.r;
            const double pr = (gamma - 1.0) * (s.E - 0.5 * ir * (s.mx * s.mx + s.my * s.my + s.mz * s.mz));
            const double vx = s.mx * ir, vy = s.my * ir, vz = s.mz * ir;
            const double ep = s.E + pr;
            const double* met = sMet + e * 9;
            if (!VISC) {
              // contravariant flux directly: with U_m = sum_d r_md v_d,
              // G_m = (rho U_m, m U_m + p r_m, (E+p) U_m)  ==  sum_d r_md F_d
              // (solver.cpp:382-394 contracted with S_m, operators.cpp:139-147)
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
              // F_d (d = x, y, z) for the 5 fields (solver.cpp:382-394)
              double F[3][5] = {{s.mx, s.mx * vx + pr, s.my * vx, s.mz * vx, vx * ep},
                                {s.my, s.mx * vy, s.my * vy + pr, s.mz * vy, vy * ep},
                                {s.mz, s.mx * vz, s.my * vz, s.mz * vz + pr, vz * ep}};
              // F_m <- F_m - sqrt(eps) I_cub q_m   (solver.cpp:398-406)
              const double se = sSe[e];
              if (se > 0.0) {
                constexpr int LDQ = round_up(C::NCUB, 8);
                const size_t qcs = (size_t)p.K * 5 * LDQ;
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                  for (int c = 0; c < 5; ++c)
                    F[m][c] -= se * __ldg(p.qcub + m * qcs + (size_t)(row0 + e * 5 + c) * LDQ + q);
              }
#pragma unroll
              for (int m = 0; m < 3; ++m) {
                const double r0 = met[m * 3 + 0], r1 = met[m * 3 + 1], r2 = met[m * 3 + 2];
#pragma unroll
                for (int c = 0; c < 5; ++c) G[m][c] = r0 * F[0][c] + r1 * F[1][c] + r2 * F[2][c];
              }
            }
          } else {
#pragma unroll
            for (int m = 0; m < 3; ++m)
#pragma unroll
              for (int c = 0; c < 5; ++c) G[m][c] = 0.0;
          }
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const int col = pcol(m * w + ql);
#pragma unroll
            for (int c = 0; c < 5; ++c) gout[c * C::LDG + col] = G[m][c];
          }
        }
      }
      __syncthreads();
      if (w == C::CH)
        gemm2_fixed<C, 3 * C::CH / 8>(acc, sG, fb2, (3 * q0) / 8, t_begin, t_end, lane);
      else
        gemm2_partial<C>(acc, sG, fb2, (3 * q0) / 8, (3 * w) / 8, t_begin, t_end, lane);
      __syncthreads();
    }

    // ---- surface: chunks of FCH face nodes ---------------------------------
    for (int fc = 0; fc < C::NFCH; ++fc) {
      const int f0 = fc * C::FCH;
      const int wr = (C::NF - f0) < C::FCH ? (C::NF - f0) : C::FCH;  // real nodes (multiple of 4)
      const int wp = round_up(wr, 8);                                 // padded to the k8 step
#pragma unroll 1
      for (int it = 0; it < C::IT_F; ++it) {
        const int idx = tid + it * C::NTH;
        if (idx >= C::E * wp) continue;
        const int e = idx / wp, fl = idx - e * wp, fq = f0 + fl;
        double* gout = sG + (e * 5) * C::LDG + pcol(fl);
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
        int h = 0;
        if (cw.x >= 0) {
          const int nface = cw.y & 3, code = cw.y >> 8;
          h = __ldg(p.code_map + code * C::NG + gq);
          const double* tp = p.traces + (size_t)cw.x * 5 * C::TB + nface * C::NG + h;
          up = State5{tp[0], tp[C::TB], tp[2 * C::TB], tp[3 * C::TB], tp[4 * C::TB]};
        } else {
          up = boundary_state(um, fn.x, fn.y, fn.z, (cw.y >> 2) & 3, p.gas);
        }
        if (!admissible(um, gamma) || !admissible(up, gamma))
          record_error(p.err, 2, p.elem_offset + eg, f, gq, um.r);
        double fs[5];
        if (RM == 1 || (RM == -1 && p.gas.riemann == 1))
          hllc_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs, p.gas.hllc_fallbacks);
        else
          llf_flux_fast(um, up, fn.x, fn.y, fn.z, gamma, fs);
        if (VISC) {
          // BR1 central viscous flux with per-side sqrt(eps) (solver.cpp:438-453)
          const double se = sSe[e];
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
      if (wp == C::FCH)
        gemm2_fixed<C, C::FCH / 8>(acc, sG, fb2, (C::K2CUB + f0) / 8, t_begin, t_end, lane);
      else
        gemm2_partial<C>(acc, sG, fb2, (C::K2CUB + f0) / 8, wp / 8, t_begin, t_end, lane);
      __syncthreads();
    }

    // ---- epilogue: rhs -> (res, u) update or rhs store ---------------------
    double a_c = 0.0, b_c = 0.0, dt = 0.0;
    if (UPDATE) {
      a_c = p.coef->a[p.stage];
      b_c = p.coef->b[p.stage];
      dt = p.coef->dt;
    }
    // all old res pairs of this thread are loaded before its first store (the
    // compiler cannot move loads of p.res above stores to p.u / p.res; loads
    // interleaved with the stores would serialise the memory round trips)
    double2 rsv[C::MAXT2][2];
    if (UPDATE) {
#pragma unroll
      for (int i = 0; i < C::MAXT2; ++i) {
        rsv[i][0] = rsv[i][1] = make_double2(0.0, 0.0);
        if (C::WROW || t_begin + i < t_end) {
          int mt, nt;
          tile_coords<C>(t_begin, i, mt, nt);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int r = mt * 16 + g + 8 * hh;
            const int grow = row0 + r;
            const int col = nt * 8 + 2 * tq;
            if (grow >= n_rows || col + 1 >= C::NP) continue;
            rsv[i][hh] = *reinterpret_cast<const double2*>(p.res + (size_t)grow * C::BP + col);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < C::MAXT2; ++i) {
      if (C::WROW || t_begin + i < t_end) {
        int mt, nt;
        tile_coords<C>(t_begin, i, mt, nt);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int r = mt * 16 + g + 8 * hh;
          const int grow = row0 + r;
          const int col = nt * 8 + 2 * tq;
          if (grow >= n_rows || col >= C::NP) continue;
          if (sConn[(r / 5) * 4].y & kCurvedBit) continue;  // written by k_rhs_curved
          const size_t gi = (size_t)grow * C::BP + col;
          const double r0 = acc[i][2 * hh], r1 = acc[i][2 * hh + 1];
          if (col + 1 < C::NP) {
            if (UPDATE) {
              const double2 rs = rsv[i][hh];
              const double n0 = a_c * rs.x + dt * r0, n1 = a_c * rs.y + dt * r1;
              *reinterpret_cast<double2*>(p.res + gi) = make_double2(n0, n1);
              *reinterpret_cast<double2*>(p.u + gi) =
                  make_double2(sU[r * C::LDU + pcol(col)] + b_c * n0, sU[r * C::LDU + pcol(col + 1)] + b_c * n1);
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
