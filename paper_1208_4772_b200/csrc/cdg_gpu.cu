// cdg_gpu.cu -- host side of the C ABI (include/cdg_gpu.h) and the level's
// device resources. Kernels live in cdg_kernels.cuh / cdg_aux.cuh.
//
// Reference interfaces replaced: see include/cdg_gpu.h. Host-side operator
// preparation restates operators.cpp:123-167 (mass matrix, stiffness and face
// mass) in the factored, element-independent form the GPU kernels consume.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cdg_gpu.h"
#include "cdg_peak.cuh"
#include "cdg_sets.cuh"

using namespace cdg_gpu;

namespace {

// NVTX ranges around the host entry points (a profiler attached via
// NVTX_INJECTION64_PATH sees them; otherwise the calls are no-ops)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw Status(CDG_GPU_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                         " at " #x);                                     \
  } while (0)

void set_err(char* err, size_t n, const std::string& msg) {
  if (err && n) {
    std::strncpy(err, msg.c_str(), n - 1);
    err[n - 1] = 0;
  }
}

int pad16(int n) { return 16 * ((n + 15) / 16); }

const std::vector<KernelSet>& kernel_sets() {
  static const std::vector<KernelSet> sets = [] {
    std::vector<KernelSet> all;
    for (auto part : {kernel_sets_p1_3(), kernel_sets_p4(), kernel_sets_p5_6(), kernel_sets_p7_8()})
      all.insert(all.end(), part.begin(), part.end());
    return all;
  }();
  return sets;
}

// The kernel set of a level shape is fixed at compile time: one KernelSet per
// (N_p, N_cub, N_g) in the sets_*.cu tables (the measured-best choice, see
// DESIGN.md §6); nothing is selected at run time.
const KernelSet* find_set(int np, int ncub, int ng) {
  for (const auto& k : kernel_sets())
    if (k.np == np && k.ncub == ncub && k.ng == ng) return &k;
  return nullptr;
}

// ---- small dense host linear algebra (setup only) --------------------------
// Inverse of an SPD matrix via Cholesky (the reference factors M per element,
// operators.cpp:151-158; here the reference mass matrix is inverted once).
std::vector<double> spd_inverse(const std::vector<double>& m, int n) {
  std::vector<double> l(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = m[j * n + j];
    for (int k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
    if (!(d > 0.0)) throw Status(CDG_GPU_ERR_NUMERICS, "build_operators: mass matrix factorization failed");
    const double ljj = std::sqrt(d);
    l[j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = m[i * n + j];
      for (int k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      l[i * n + j] = s / ljj;
    }
  }
  std::vector<double> inv(n * n, 0.0), y(n), x(n);
  for (int col = 0; col < n; ++col) {
    for (int i = 0; i < n; ++i) {
      double s = (i == col) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= l[i * n + k] * y[k];
      y[i] = s / l[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= l[k * n + i] * x[k];
      x[i] = s / l[i * n + i];
    }
    for (int i = 0; i < n; ++i) inv[i * n + col] = x[i];
  }
  return inv;
}

// General dense inverse (Gauss-Jordan with partial pivoting), setup only.
std::vector<double> dense_inverse(std::vector<double> a, int n) {
  std::vector<double> inv((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[(size_t)i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[(size_t)r * n + c]) > std::fabs(a[(size_t)piv * n + c])) piv = r;
    if (a[(size_t)piv * n + c] == 0.0) throw Status(CDG_GPU_ERR_NUMERICS, "singular Vandermonde inverse");
    if (piv != c)
      for (int k = 0; k < n; ++k) {
        std::swap(a[(size_t)c * n + k], a[(size_t)piv * n + k]);
        std::swap(inv[(size_t)c * n + k], inv[(size_t)piv * n + k]);
      }
    const double d = 1.0 / a[(size_t)c * n + c];
    for (int k = 0; k < n; ++k) {
      a[(size_t)c * n + k] *= d;
      inv[(size_t)c * n + k] *= d;
    }
    for (int r = 0; r < n; ++r)
      if (r != c) {
        const double m = a[(size_t)r * n + c];
        if (m == 0.0) continue;
        for (int k = 0; k < n; ++k) {
          a[(size_t)r * n + k] -= m * a[(size_t)c * n + k];
          inv[(size_t)r * n + k] -= m * inv[(size_t)c * n + k];
        }
      }
  }
  return inv;
}

// B-operand fragments for mma.m16n8k8 (.col): frag[nt][ks][lane] = the pair
// (op[nt*8 + lane/4][ks*8 + lane%4], op[nt*8 + lane/4][ks*8 + lane%4 + 4]),
// zero outside [rows x cols]: one coalesced 16-byte load per thread per step.
std::vector<double> make_frag(const std::vector<double>& op, int rows, int cols, int rows8,
                              int cols8) {
  std::vector<double> f((size_t)rows8 / 8 * (cols8 / 8) * 64, 0.0);
  for (int nt = 0; nt < rows8 / 8; ++nt)
    for (int ks = 0; ks < cols8 / 8; ++ks)
      for (int lane = 0; lane < 32; ++lane)
        for (int v = 0; v < 2; ++v) {
          const int r = nt * 8 + lane / 4, c = ks * 8 + lane % 4 + 4 * v;
          if (r < rows && c < cols)
            f[(((size_t)nt * (cols8 / 8) + ks) * 32 + lane) * 2 + v] = op[(size_t)r * cols + c];
        }
  return f;
}

// B fragments for the warp-tile kernel (cdg_warp.cuh): lane (g, t) of
// (n-tile nt, k-step ks) holds (op[8nt+g][8ks+2t], op[8nt+g][8ks+2t+1]).
void frag_nat(std::vector<double>& out, const std::vector<double>& op, int rows, int cols, int nt, int ks) {
  for (int lane = 0; lane < 32; ++lane)
    for (int v = 0; v < 2; ++v) {
      const int r = nt * 8 + lane / 4, c = ks * 8 + 2 * (lane % 4) + v;
      out.push_back(r < rows && c < cols ? op[(size_t)r * cols + c] : 0.0);
    }
}

template <typename T>
T* dev_upload(const std::vector<T>& h) {
  T* d = nullptr;
  if (h.empty()) return nullptr;
  CUDA_OK(cudaMalloc(&d, h.size() * sizeof(T)));
  CUDA_OK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

}  // namespace

struct cdg_gpu_level {
  int device = 0;
  int K = 0, n_halo = 0, np = 0, ncub = 0, ng = 0, nf = 0, degree = 0;
  int caller_block = 0, caller_tblock = 0, bp = 0, tb = 0;
  bool caller_padded = true;
  const KernelSet* ks = nullptr;
  cudaStream_t stream = nullptr;
  int n_sms = 148;
  int max_ctas = 0;  // cap on persistent-kernel grids (0: n_sms x CTAs/SM); cdg_gpu_set_max_ctas
  long long launches = 0;
  // state
  double *u = nullptr, *res = nullptr, *rhs = nullptr, *traces = nullptr, *before = nullptr;
  // pinned two-slot ring of the host <-> device state copies (copy_rows)
  double* ring[2] = {nullptr, nullptr};
  size_t ring_doubles = 0;
  cudaEvent_t ring_ev[2] = {nullptr, nullptr};
  // viscous workspace
  double *q = nullptr, *qtr = nullptr, *qcub = nullptr, *eps = nullptr, *sqrt_eps = nullptr;
  double* d_vinv = nullptr;
  // J-weighted indicator (viscosity.cpp:28-45)
  double *d_vcub = nullptr, *d_wcub = nullptr, *d_jac = nullptr, *d_curved_jac = nullptr;
  int* d_curved_slot = nullptr;
  unsigned long long* d_maxeps = nullptr;
  unsigned long long* d_fallbacks = nullptr;  // HLLC -> LLF fallbacks (RhsWorkspace::hllc_fallbacks)
  bool last_viscous = false;
  // geometry / coupling
  double* metric = nullptr;
  double4* face = nullptr;
  int2* conn = nullptr;
  int* code_map = nullptr;
  double* h = nullptr;
  // operators
  double *frag_icub = nullptr, *frag_op2 = nullptr, *frag_ig = nullptr, *frag_aux = nullptr, *frag_dtil = nullptr;
  double *wfrag1 = nullptr, *wfrag2v = nullptr, *wfrag2f = nullptr;  // warp-tile kernel
  bool use_warp = false;
  double* rfrag2 = nullptr;  // row kernel (its I_cub fragments are wfrag1)
  double* tbuf[2] = {nullptr, nullptr};  // trace double buffer of the fused-trace path
  int tcur = 0;                          // tbuf[tcur] == traces (current)
  bool traces_valid = false;             // traces == I_g u for the current u (owned rows)
  double* cur_traces_out = nullptr;
  cudaGraphExec_t gft[2] = {nullptr, nullptr};
  int gft_riemann[2] = {-1, -1};
  double gft_gamma[2] = {0.0, 0.0};
  int gft_launches = 0;
  bool use_row = false;
  // neighbour-state path (cdg_ns.cuh): state ping-pong u = ubuf[ucur], no stored traces
  bool use_ns = false;
  double* ubuf[2] = {nullptr, nullptr};
  int ucur = 0;
  double* d_ig = nullptr;  // I_g row-major [NF][NP]
  cudaGraphExec_t gns[2] = {nullptr, nullptr};
  int gns_riemann[2] = {-1, -1};
  double gns_gamma[2] = {0.0, 0.0};
  int gns_launches = 0;
  const int* cur_tiles = nullptr;  // tile list of the next RHS launch (null: all)
  const unsigned long long* cur_gate = nullptr;  // launch gate of the next launches (null: none)
  int cur_gate_when = 0;
  // graph of one viscous RK step (gated stages) and the config it was captured with
  cudaGraphExec_t graph_visc = nullptr;
  cdg_gpu_run_config graph_visc_cfg{};
  int graph_launches = 0, graph_visc_launches = 0;
  std::vector<char> ghost_adjacent;  // [K] element has a ghost (halo) neighbour
  int cur_n_list = 0;
  // curved elements
  int n_curved = 0;
  int* curved_ids = nullptr;
  double *curved_jwr = nullptr, *curved_minv = nullptr, *frag_opc = nullptr, *curved_vol = nullptr;
  double* rfrag_opc = nullptr;  // [D^T | -I_g^T] for k_rhs_rowc (natural pairing)
  bool use_rowc = false;
  int* d_affine_tiles = nullptr;  // 16-element tiles holding an affine element (curved levels)
  int n_affine_tiles = 0;
  double4* curved_face = nullptr;
  // control
  StageCoef* d_coef = nullptr;
  StageCoef* h_coef = nullptr;  // pinned
  DevError* d_err = nullptr;
  DevError* h_err = nullptr;  // pinned
  GasParams gas{};
  double* d_scratch = nullptr;  // reductions
  std::vector<double> h_scratch;
  int scratch_n = 0;
  // graph cache for rk_steps
  cudaGraphExec_t graph = nullptr;
  int graph_riemann = -1;
  double graph_gamma = 0.0;
  // profiling
  bool profiling = false;
  double prof[3] = {0, 0, 0};
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  // halo
  int n_send = 0, n_recv = 0;
  // interior / halo tile lists (E = 16 element tiles) for comm-compute overlap
  int *d_tiles_int = nullptr, *d_tiles_halo = nullptr;
  int n_tiles_int = 0, n_tiles_halo = 0;
  int *d_send_idx = nullptr, *d_recv_idx = nullptr;
  double *send_buf = nullptr, *recv_buf = nullptr;
  // library-owned halo rows of the multi-rank driver (cdg_gpu_halo_define):
  // per peer, rows [off, off + n) of the send / receive lists; send rows
  // double-buffered by exchange parity (cdg_comm.cuh)
  struct Peer {
    int rank, send_off, send_n, recv_off, recv_n;
  };
  std::vector<Peer> peers;
  double* hsend[2] = {nullptr, nullptr};
  double* hrecv = nullptr;
  bool halo_defined = false;
  // curved-list tiles split the same way (curved levels; k_rhs_rowc / k_rhs_curved)
  int *d_ctiles_int = nullptr, *d_ctiles_halo = nullptr;
  int n_ctiles_int = 0, n_ctiles_halo = 0;
  const int* cur_ctiles = nullptr;  // curved-tile list of the next curved launch (null: all)
  int cur_n_clist = 0;
  std::vector<int> curved_ids_h;    // host copy of the curved list
  // halo payload: row width (doubles) of send/recv rows; 5 N_g (traces only)
  // unless a multi-rank driver (cdg_gpu_comm) owns the buffers
  int halo_w = 0;
  // launch gate of the viscous kernels: null = the local max eps (d_maxeps);
  // a multi-rank driver points it at the all-rank max
  unsigned long long* gate_buf = nullptr;
  double freestream[5] = {0, 0, 0, 0, 0};

  int n_rows() const { return K * 5; }
  int n_tiles() const { return (K + ks->E - 1) / ks->E; }
  // persistent grid: min(work items, resident CTAs), optionally capped
  int cap(int items, int per_sm) const {
    int g = std::min(items, n_sms * per_sm);
    if (max_ctas > 0) g = std::min(g, max_ctas);
    return std::max(1, g);
  }
  int grid(int tiles) const { return cap(tiles, ks->minb); }
};

namespace {

void check_device_error(cdg_gpu_level* lv) {
  CUDA_OK(cudaMemcpyAsync(lv->h_err, lv->d_err, sizeof(DevError), cudaMemcpyDeviceToHost,
                          lv->stream));
  CUDA_OK(cudaStreamSynchronize(lv->stream));
  if (lv->h_err->flag) {
    lv->traces_valid = false;  // an aborted fused stage leaves partial traces
    const DevError e = *lv->h_err;
    CUDA_OK(cudaMemsetAsync(lv->d_err, 0, sizeof(DevError), lv->stream));
    CUDA_OK(cudaStreamSynchronize(lv->stream));
    char buf[256];
    if (e.kind == 1)
      std::snprintf(buf, sizeof buf, "inadmissible state in element %d at cubature node %d (rho=%f)",
                    e.elem, e.a, e.value);
    else if (e.kind == 2)
      std::snprintf(buf, sizeof buf, "inadmissible trace state in element %d face %d node %d",
                    e.elem, e.a, e.b);
    else if (e.kind == 3)
      std::snprintf(buf, sizeof buf, "inadmissible state in compute_timestep: rho=%f", e.value);
    else
      std::snprintf(buf, sizeof buf, "compute_timestep: degenerate h or wavespeed in element %d",
                    e.elem);
    throw Status(CDG_GPU_ERR_NUMERICS, buf);
  }
}

void launch_traces(cdg_gpu_level* lv, const double* u, double* traces) {
  const int tiles = lv->n_tiles();
  lv->ks->traces<<<tiles, kThreads, lv->ks->smem_traces, lv->stream>>>(
      u, traces, lv->frag_ig, lv->n_rows(), tiles, lv->cur_gate, lv->cur_gate_when);
  ++lv->launches;
}

// the RHS kernels of the level write the next stage's traces: the affine
// kernel (row kernel with MODE 32, warp-autonomous with FT, or the warp-tile
// kernel) for the affine elements and, on curved levels, k_rhs_wac for the
// curved ones (all-curved levels need only the latter)
bool fused_traces(const cdg_gpu_level* lv) {
  const bool affine_ft = (lv->use_row && lv->ks->row_ft) || (!lv->use_row && lv->use_warp);
  if (lv->n_curved == 0) return affine_ft;
  const bool curved_ft = lv->use_rowc && lv->ks->rowc_ft;
  return curved_ft && (affine_ft || lv->n_curved == lv->K);
}

// Grid sizing of the warp-autonomous kernel on a single-shard level: one warp
// per 3-element group, 16 warps per SM. A level whose groups fill the resident
// warps once and then less than 60% of them a second time (e.g. 7,986 tets:
// 2,662 groups on 2,368 warps) takes the CTA kernel (16-element tiles), 12-17%
// faster there; from ~16k tets up the warp-autonomous kernel wins.
bool wa_poorly_quantized(const cdg_gpu_level* lv) {
  if (std::strcmp(lv->ks->row_name, "k_rhs_wa") != 0 || lv->n_halo > 0 || lv->n_curved > 0) return false;
  const long groups = (lv->K + 2) / 3;
  const long slots = (long)lv->n_sms * (lv->ks->row_nth / 32) * lv->ks->row_minb;
  const long waves = (groups + slots - 1) / slots;
  return waves == 2 && (double)groups / (double)(slots * waves) < 0.6;
}

// the captured graphs that bake the state pointer u and the trace buffers
void drop_graphs_except_ns(cdg_gpu_level* lv) {
  if (lv->graph) cudaGraphExecDestroy(lv->graph), lv->graph = nullptr;
  if (lv->graph_visc) cudaGraphExecDestroy(lv->graph_visc), lv->graph_visc = nullptr;
  for (auto& ge : lv->gft)
    if (ge) cudaGraphExecDestroy(ge), ge = nullptr;
}

// the neighbour-state kernel runs inviscid stages of an all-affine level
// without halo rows or phase lists (single-shard runs)
bool ns_path(const cdg_gpu_level* lv) {
  return lv->use_ns && lv->n_curved == 0 && lv->n_halo == 0 && !lv->cur_tiles && !lv->cur_gate;
}

void ensure_ubuf(cdg_gpu_level* lv) {
  if (lv->ubuf[1]) return;
  const size_t n = (size_t)lv->K * 5 * lv->bp;
  CUDA_OK(cudaMalloc(&lv->ubuf[1], n * sizeof(double)));
  CUDA_OK(cudaMemset(lv->ubuf[1], 0, n * sizeof(double)));  // padding columns: zero, never written
}

void ensure_tbuf(cdg_gpu_level* lv) {
  if (lv->tbuf[1]) return;
  const size_t ntr = (size_t)(lv->K + lv->n_halo) * 5 * lv->tb;
  CUDA_OK(cudaMalloc(&lv->tbuf[1], ntr * sizeof(double)));
  CUDA_OK(cudaMemset(lv->tbuf[1], 0, ntr * sizeof(double)));
  lv->tbuf[0] = lv->traces;
  lv->tcur = 0;
}

// the traces of the current u, unless they are already there
void seed_traces(cdg_gpu_level* lv) {
  if (lv->traces_valid) return;
  launch_traces(lv, lv->u, lv->traces);
  lv->traces_valid = true;
}

// tile list of the next affine-kernel launch: the phase list (multi-GPU), else
// on a curved level the tiles that hold an affine element, else all (null)
const int* affine_tiles(const cdg_gpu_level* lv, int* n_list) {
  if (lv->cur_tiles) {
    *n_list = lv->cur_n_list;
    return lv->cur_tiles;
  }
  *n_list = lv->n_affine_tiles;
  return lv->d_affine_tiles;
}

RhsParams rhs_params(cdg_gpu_level* lv, int stage) {
  RhsParams p{};
  p.tiles = affine_tiles(lv, &p.n_list);
  p.gate = lv->cur_gate;
  p.gate_when = lv->cur_gate_when;
  p.traces_out = lv->cur_traces_out;
  p.frag_ig_nat = lv->frag_ig;  // the trace kernel's fragments (bitwise-identical fused traces)
  p.u = lv->u;
  p.res = lv->res;
  p.rhs_out = lv->rhs;
  p.traces = lv->traces;
  p.metric = lv->metric;
  p.face = lv->face;
  p.conn = lv->conn;
  p.code_map = lv->code_map;
  p.frag_icub = lv->frag_icub;
  p.frag_op2 = lv->frag_op2;
  p.coef = lv->d_coef;
  p.stage = stage;
  p.K = lv->K;
  p.n_tiles = lv->n_tiles();
  p.elem_offset = 0;
  p.gas = lv->gas;
  p.err = lv->d_err;
  p.q = lv->q;
  p.qtr = lv->qtr;
  p.sqrt_eps = lv->sqrt_eps;
  p.qcub = lv->qcub;
  p.qtr_stride = (size_t)(lv->K + lv->n_halo) * 5 * lv->tb;
  p.prefetch = 15;  // L2 prefetch of res / traces / next tile (CTA kernel, measured: DESIGN.md §6)
  return p;
}

// mode 0: inviscid RHS(+update), 1: viscous RHS(+update), 2: aux gradient q
void launch_curved(cdg_gpu_level* lv, bool update, int stage, int mode = 0) {
  if (!lv->n_curved) return;
  CurvedParams cp{};
  cp.base = rhs_params(lv, stage);
  cp.ctiles = lv->cur_ctiles;
  cp.n_clist = lv->cur_n_clist;
  if (cp.ctiles && cp.n_clist == 0) return;  // empty phase list
  cp.ids = lv->curved_ids;
  cp.jwr = lv->curved_jwr;
  cp.face = lv->curved_face;
  cp.minv = lv->curved_minv;
  cp.frag_opc = lv->frag_opc;
  cp.vol = lv->curved_vol;
  cp.q_out = lv->q;
  cp.Kc = lv->n_curved;
  if (lv->use_rowc) {  // row-per-warp curved kernels (cdg_rowc.cuh)
    cp.base.frag_icub = lv->wfrag1;
    cp.frag_opc = lv->rfrag_opc;
    const int rm = lv->gas.riemann == 1 ? 1 : 0;
    auto fr = mode == 2   ? lv->ks->rowc_aux
              : mode == 1 ? (update ? lv->ks->rowc_visc_update[rm] : lv->ks->rowc_visc_only[rm])
                          : (update ? lv->ks->rowc_update[rm] : lv->ks->rowc_only[rm]);
    const int Ec = mode == 2 ? lv->ks->rowc_aux_e : lv->ks->rowc_e;  // curved entries per CTA tile
    const int tiles = cp.ctiles ? cp.n_clist : (lv->n_curved + Ec - 1) / Ec;
    fr<<<lv->cap(tiles, mode == 2 ? lv->ks->rowc_aux_minb : lv->ks->rowc_minb),
         mode == 2 ? lv->ks->rowc_aux_nth : lv->ks->rowc_nth, mode == 2 ? lv->ks->smem_rowc_aux : lv->ks->smem_rowc,
         lv->stream>>>(cp);
    ++lv->launches;
    return;
  }
  const int tiles = cp.ctiles ? cp.n_clist : (lv->n_curved + lv->ks->E - 1) / lv->ks->E;
  auto fn = mode == 2 ? lv->ks->aux_curved
                      : mode == 1 ? (update ? lv->ks->curved_visc_update : lv->ks->curved_visc_only)
                                  : (update ? lv->ks->curved_update : lv->ks->curved_only);
  fn<<<lv->cap(tiles, 1), kThreads, lv->ks->smem_curved, lv->stream>>>(cp);
  ++lv->launches;
}

void launch_rhs_warp(cdg_gpu_level* lv, bool update, int stage) {
  WarpParams w{};
  w.u = lv->u;
  w.res = lv->res;
  w.rhs_out = lv->rhs;
  w.traces = lv->traces;
  w.metric = lv->metric;
  w.face = lv->face;
  w.conn = lv->conn;
  w.code_map = lv->code_map;
  w.frag1 = reinterpret_cast<const double2*>(lv->wfrag1);
  w.frag2v = reinterpret_cast<const double2*>(lv->wfrag2v);
  w.frag2f = reinterpret_cast<const double2*>(lv->wfrag2f);
  w.coef = lv->d_coef;
  w.stage = stage;
  w.K = lv->K;
  w.elem_offset = 0;
  w.gas = lv->gas;
  w.err = lv->d_err;
  w.tiles = affine_tiles(lv, &w.n_list);
  w.gate = lv->cur_gate;
  w.gate_when = lv->cur_gate_when;
  w.traces_out = lv->cur_traces_out;
  w.frag_ig_nat = reinterpret_cast<const double2*>(lv->frag_ig);
  const int tiles = w.tiles ? w.n_list : (lv->K + 15) / 16;
  if (tiles == 0) {
    launch_curved(lv, update, stage);
    return;
  }
  const int ctas = lv->cap((tiles + lv->ks->warp_warps - 1) / lv->ks->warp_warps, lv->ks->warp_minb);
  const int rm = lv->gas.riemann == 1 ? 1 : 0;
  auto fn = update ? lv->ks->warp_update[rm] : lv->ks->warp_only[rm];
  fn<<<ctas, 32 * lv->ks->warp_warps, lv->ks->smem_warp, lv->stream>>>(w);
  ++lv->launches;
  launch_curved(lv, update, stage);
}

// one stage of the neighbour-state kernel: reads u_in (own + neighbour rows)
// and res, writes res and u_out (cdg_ns.cuh)
void launch_rhs_ns(cdg_gpu_level* lv, int stage, const double* u_in, double* u_out) {
  WarpParams w{};
  w.u = const_cast<double*>(u_in);
  w.u_out = u_out;
  w.res = lv->res;
  w.metric = lv->metric;
  w.face = lv->face;
  w.conn = lv->conn;
  w.code_map = lv->code_map;
  w.frag1 = reinterpret_cast<const double2*>(lv->wfrag1);
  w.frag2v = reinterpret_cast<const double2*>(lv->wfrag2v);
  w.frag2f = reinterpret_cast<const double2*>(lv->wfrag2f);
  w.ig = lv->d_ig;
  w.coef = lv->d_coef;
  w.stage = stage;
  w.K = lv->K;
  w.elem_offset = 0;
  w.gas = lv->gas;
  w.err = lv->d_err;
  const int tiles = (lv->K + 15) / 16;
  const int ctas = lv->cap((tiles + lv->ks->ns_warps - 1) / lv->ks->ns_warps, lv->ks->ns_minb);
  const int rm = lv->gas.riemann == 1 ? 1 : 0;
  lv->ks->ns_update[rm]<<<ctas, 32 * lv->ks->ns_warps, lv->ks->smem_ns, lv->stream>>>(w);
  ++lv->launches;
}

void launch_rhs_row(cdg_gpu_level* lv, bool update, int stage) {
  RhsParams p = rhs_params(lv, stage);
  p.frag_icub = lv->wfrag1;
  p.frag_op2 = lv->rfrag2;
  // L2 prefetching measured neutral-to-negative for the row kernel (4 CTAs/SM
  // already cover the latency; profiles/r1); it stays on for the CTA kernel
  p.prefetch = 0;
  const int rm = lv->gas.riemann == 1 ? 1 : 0;
  auto fn = update ? lv->ks->row_update[rm] : lv->ks->row_only[rm];
  const int E = lv->ks->row_e;
  const int tiles = p.tiles ? p.n_list : (lv->K + E - 1) / E;
  if (tiles == 0) {
    launch_curved(lv, update, stage);
    return;
  }
  fn<<<lv->cap(tiles, lv->ks->row_minb), lv->ks->row_nth, lv->ks->smem_row, lv->stream>>>(p);
  ++lv->launches;
  launch_curved(lv, update, stage);
}

void launch_rhs(cdg_gpu_level* lv, bool update, bool viscous, int stage) {
  if (!viscous && lv->use_row) {
    launch_rhs_row(lv, update, stage);
    return;
  }
  if (!viscous && lv->use_warp) {
    launch_rhs_warp(lv, update, stage);
    return;
  }
  RhsParams p = rhs_params(lv, stage);
  const int tiles = p.tiles ? p.n_list : lv->n_tiles();
  if (tiles == 0) {
    launch_curved(lv, update, stage, viscous ? 1 : 0);
    return;
  }
  auto fn = viscous ? (update ? lv->ks->visc_rhs_update : lv->ks->visc_rhs_only)
                    : (update ? lv->ks->rhs_update : lv->ks->rhs_only);
  fn<<<lv->grid(tiles), lv->ks->nth, lv->ks->smem_rhs, lv->stream>>>(p);
  ++lv->launches;
  launch_curved(lv, update, stage, viscous ? 1 : 0);
}

// Viscosity phase: sensor -> eps, then (if any eps > 0) aux gradient q and its
// traces (solver.cpp:239-321). Returns whether the viscous path is active.
void ensure_viscous_buffers(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg) {
  if (cfg->eps0 < 0.0) throw Status(CDG_GPU_ERR_CONFIG, "viscosity_amount: eps0 must be >= 0");
  if (cfg->jacobian_weighted && lv->n_curved && !lv->d_curved_jac)
    throw Status(CDG_GPU_ERR_CONFIG, "jacobian_weighted indicator on curved elements needs curved_jac");
  if (cfg->jacobian_weighted && !lv->d_vcub)
    throw Status(CDG_GPU_ERR_CONFIG, "jacobian_weighted indicator needs vandermonde_inv");
  if (!lv->q) {
    const size_t n = (size_t)lv->K * 5 * lv->bp;
    const size_t nt = (size_t)(lv->K + lv->n_halo) * 5 * lv->tb;
    CUDA_OK(cudaMalloc(&lv->q, 3 * n * sizeof(double)));
    CUDA_OK(cudaMemset(lv->q, 0, 3 * n * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->qtr, 3 * nt * sizeof(double)));
    CUDA_OK(cudaMemset(lv->qtr, 0, 3 * nt * sizeof(double)));
    const size_t nc = (size_t)lv->K * 5 * ((lv->ncub + 7) / 8 * 8);
    CUDA_OK(cudaMalloc(&lv->qcub, 3 * nc * sizeof(double)));
    CUDA_OK(cudaMemset(lv->qcub, 0, 3 * nc * sizeof(double)));
  }
}

// sensor -> eps, sqrt(eps), max eps bits (compute_element_viscosities, solver.cpp:239-260)
void launch_sensor(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg) {
  CUDA_OK(cudaMemsetAsync(lv->d_maxeps, 0, sizeof(unsigned long long), lv->stream));
  SensorParams sp{};
  sp.u = lv->u;
  sp.vinv = lv->d_vinv;
  sp.eps = lv->eps;
  sp.sqrt_eps = lv->sqrt_eps;
  sp.maxeps = lv->d_maxeps;
  sp.K = lv->K;
  sp.np = lv->np;
  sp.np_prev = lv->degree >= 1 ? (lv->degree) * (lv->degree + 1) * (lv->degree + 2) / 6 : 0;
  sp.bp = lv->bp;
  sp.comp = cfg->indicator_component;
  sp.eps0 = cfg->eps0;
  sp.kappa = cfg->kappa;
  sp.s0 = std::log10(1.0 / std::pow((double)lv->degree, 4)) + cfg->s0_offset;
  if (cfg->jacobian_weighted) {
    sp.vcub = lv->d_vcub;
    sp.wcub = lv->d_wcub;
    sp.jac = lv->d_jac;
    sp.curved_slot = lv->d_curved_slot;
    sp.curved_jac = lv->d_curved_jac;
    sp.ncub = lv->ncub;
    k_sensor_jw<<<(lv->K + 7) / 8, 256, 0, lv->stream>>>(sp);
  } else {
    k_sensor<<<(lv->K + 7) / 8, 256, 0, lv->stream>>>(sp);
  }
  ++lv->launches;
}

// aux gradient q_m of every element + its traces (solver.cpp:264-321); needs
// the U traces first
void launch_aux(cdg_gpu_level* lv) {
  AuxParams ap{};
  ap.u = lv->u;
  ap.q = lv->q;
  ap.traces = lv->traces;
  ap.metric = lv->metric;
  ap.face = lv->face;
  ap.conn = lv->conn;
  ap.code_map = lv->code_map;
  ap.frag_icub = lv->frag_icub;
  ap.frag_aux = lv->frag_aux;
  ap.frag_dtil = lv->frag_dtil;
  ap.sqrt_eps = lv->sqrt_eps;
  ap.K = lv->K;
  ap.n_tiles = lv->n_tiles();
  ap.gas = lv->gas;
  ap.gate = lv->cur_gate;
  ap.gate_when = lv->cur_gate_when;
  ap.tiles = lv->d_affine_tiles;  // curved levels: skip the all-curved tiles
  ap.n_list = lv->n_affine_tiles;
  const int aux_tiles = ap.tiles ? ap.n_list : lv->n_tiles();
  if (aux_tiles > 0) {
    lv->ks->aux_q<<<lv->grid(aux_tiles), kThreads, lv->ks->smem_aux, lv->stream>>>(ap);
    ++lv->launches;
  }
  launch_curved(lv, false, 0, 2);  // per-node-metric q of the curved elements
  const size_t n = (size_t)lv->K * 5 * lv->bp;
  const size_t nt = (size_t)(lv->K + lv->n_halo) * 5 * lv->tb;
  const size_t nc = (size_t)lv->K * 5 * ((lv->ncub + 7) / 8 * 8);
  {  // the normal component of q's traces (the BR1 face term's only use of them)
    const int blocks = (lv->n_rows() + lv->ks->qn_rows - 1) / lv->ks->qn_rows;  // row blocks, one per CTA
    lv->ks->qn_traces<<<blocks, kThreads, lv->ks->smem_qn, lv->stream>>>(
        lv->q, n, lv->qtr, lv->frag_ig, lv->face, lv->curved_face, lv->n_curved ? lv->d_curved_slot : nullptr,
        lv->n_rows(), blocks, lv->cur_gate, lv->cur_gate_when);
    ++lv->launches;
  }
  (void)nt;
  for (int m = 0; m < 3; ++m) {
    // I_cub q_m once per element (the RHS kernels' viscous volume term)
    const int tiles = lv->n_tiles();
    lv->ks->cubinterp<<<tiles, kThreads, lv->ks->smem_traces, lv->stream>>>(
        lv->q + m * n, lv->qcub + m * nc, lv->frag_icub, lv->n_rows(), tiles, lv->cur_gate, lv->cur_gate_when);
    ++lv->launches;
  }
}

// Viscosity phase with the host decision (compute_rhs path): sensor -> eps,
// then (if any eps > 0) aux gradient q and its traces (solver.cpp:239-321).
// Returns whether the viscous path is active.
bool viscosity_phase(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg) {
  if (!cfg->visc_enabled) return false;
  ensure_viscous_buffers(lv, cfg);
  launch_sensor(lv, cfg);
  unsigned long long bits = 0;
  CUDA_OK(cudaMemcpyAsync(&bits, lv->d_maxeps, sizeof bits, cudaMemcpyDeviceToHost, lv->stream));
  CUDA_OK(cudaStreamSynchronize(lv->stream));
  double maxeps;
  std::memcpy(&maxeps, &bits, sizeof maxeps);
  if (!(maxeps > 0.0)) return false;
  launch_traces(lv, lv->u, lv->traces);
  launch_aux(lv);
  return true;
}

// One viscous RK stage with the decision on the device (graph-capturable):
// the same kernels as viscosity_phase + launch_rhs, each gated on max eps.
void viscous_stage_gated(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, int stage) {
  launch_sensor(lv, cfg);
  launch_traces(lv, lv->u, lv->traces);  // both paths need the U traces
  lv->cur_gate = lv->gate_buf ? lv->gate_buf : lv->d_maxeps;
  lv->cur_gate_when = 1;
  launch_aux(lv);
  launch_rhs(lv, true, true, stage);
  lv->cur_gate_when = 0;
  launch_rhs(lv, true, false, stage);
  lv->cur_gate = nullptr;
}

}  // namespace

namespace {
// Interior / halo tile lists of the overlapped multi-GPU stage: a tile is a
// halo tile when one of the elements it updates has a ghost (halo) neighbour.
// Affine tiles (the affine kernel's E) that hold only curved elements are in
// neither list; curved tiles (E consecutive curved-list entries) are split
// the same way.
void build_phase_lists(cdg_gpu_level* lv) {
  const int K = lv->K;
  std::vector<char> curved(K, 0);
  for (int e : lv->curved_ids_h) curved[e] = 1;
  auto ghost = [&](int e) { return !lv->ghost_adjacent.empty() && lv->ghost_adjacent[e]; };
  const int E = lv->use_row ? lv->ks->row_e : lv->ks->E;
  std::vector<int> ti, th;
  for (int t = 0; t * E < K; ++t) {
    bool any = false, halo = false;
    for (int e = t * E; e < std::min(K, (t + 1) * E); ++e)
      if (!curved[e]) any = true, halo = halo || ghost(e);
    if (any) (halo ? th : ti).push_back(t);
  }
  for (int* p : {lv->d_tiles_int, lv->d_tiles_halo, lv->d_ctiles_int, lv->d_ctiles_halo})
    if (p) cudaFree(p);
  lv->d_tiles_int = dev_upload(ti.empty() ? std::vector<int>{0} : ti);
  lv->d_tiles_halo = dev_upload(th.empty() ? std::vector<int>{0} : th);
  lv->n_tiles_int = (int)ti.size();
  lv->n_tiles_halo = (int)th.size();
  std::vector<int> ci, chh;
  const int Ec = lv->use_rowc ? lv->ks->rowc_e : lv->ks->E;
  const int nc = (int)lv->curved_ids_h.size();
  for (int t = 0; t * Ec < nc; ++t) {
    bool halo = false;
    for (int i = t * Ec; i < std::min(nc, (t + 1) * Ec); ++i) halo = halo || ghost(lv->curved_ids_h[i]);
    (halo ? chh : ci).push_back(t);
  }
  lv->d_ctiles_int = dev_upload(ci.empty() ? std::vector<int>{0} : ci);
  lv->d_ctiles_halo = dev_upload(chh.empty() ? std::vector<int>{0} : chh);
  lv->n_ctiles_int = (int)ci.size();
  lv->n_ctiles_halo = (int)chh.size();
}
}  // namespace

namespace {
int guarded(char* err, size_t errlen, const std::function<void()>& fn) {
  try {
    fn();
    return CDG_GPU_OK;
  } catch (const Status& s) {
    set_err(err, errlen, s.what());
    return s.code;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return CDG_GPU_ERR_OTHER;
  }
}
}  // namespace

namespace {
// run_steady's per-level loop (solver.cpp:622-668) over a set of operations:
// one level (cdg_gpu_run_level_live) or every shard of a multi-rank driver
// (cdg_gpu_comm_run_level, global dt MIN / residual reductions).
struct SteadyOps {
  std::function<void(int, double, const double*, const double*)> rk_steps;
  std::function<void()> snapshot;
  std::function<double(int, double)> residual;
  std::function<double(int)> timestep;
};

int run_level_loop(const SteadyOps& ops, const cdg_gpu_run_config* cfg, const cdg_gpu_steady_params* sp,
                   cdg_gpu_row_fn on_row, void* user, double* rows, int max_rows, int* n_rows, int* converged,
                   char* err, size_t errlen) {
  NvtxRange nvtx_("run_steady level");
  // Carpenter-Kennedy LSRK4(5) coefficients (rk.hpp:15-24)
  static const double A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                              -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
  static const double B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                              1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                              2277821191437.0 / 14882151754819.0};
  *n_rows = 0;
  *converged = 0;
  return guarded(err, errlen, [&] {
    if (sp->check_interval <= 0) throw Status(CDG_GPU_ERR_CONFIG, "run_steady: check_interval must be positive");
    double dt = sp->dt_override > 0.0 ? sp->dt_override : ops.timestep(0);
    double initial = -1.0;
    long iter = 0;
    bool done = false;
    while (!done && iter < sp->max_iterations) {
      // next check iteration: iter % interval == 0, the last iteration, or the fixed count
      long next = (iter / sp->check_interval + 1) * sp->check_interval;
      next = std::min(next, sp->max_iterations);
      if (sp->fixed_iterations > iter) next = std::min(next, sp->fixed_iterations);
      if (next - iter - 1 > 0) ops.rk_steps((int)(next - iter - 1), dt, A, B);
      ops.snapshot();
      ops.rk_steps(1, dt, A, B);
      iter = next;
      const double r = ops.residual(sp->residual_kind, dt);
      if (*n_rows < max_rows) {
        rows[3 * *n_rows + 0] = (double)iter;
        rows[3 * *n_rows + 1] = dt;
        rows[3 * *n_rows + 2] = r;
      }
      ++*n_rows;
      if (on_row) on_row(user, iter, dt, r);  // live, as the reference's loop emits it (solver.cpp:643-647)
      if (initial < 0.0) initial = std::max(r, 1e-300);
      if (r > 1e6 * initial && r > 1e-12) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "run_steady: divergence detected at p=%d iteration %ld (residual %f)",
                      sp->degree, iter, r);
        throw Status(CDG_GPU_ERR_NUMERICS, buf);
      }
      if (sp->fixed_iterations > 0) {
        if (iter >= sp->fixed_iterations) done = true;
      } else if (r < sp->tolerance) {
        done = true;
        *converged = 1;
      }
      if (!done && sp->dt_override <= 0.0) dt = ops.timestep(cfg->visc_enabled ? 1 : 0);
    }
  });
}
}  // namespace

extern "C" {

int cdg_gpu_fused_traces(const cdg_gpu_level* lv) {
  return fused_traces(lv) ? 1 : 0;
}

const char* cdg_gpu_rhs_kernel(const cdg_gpu_level* lv) {
  if (ns_path(lv)) return "k_rhs_ns";  // inviscid rk_steps
  if (lv->use_row) return lv->ks->row_name;
  if (lv->use_warp) return "k_rhs_warp";
  return "k_rhs";
}

const char* cdg_gpu_curved_kernel(const cdg_gpu_level* lv) {
  if (!lv->n_curved) return "";
  return lv->use_rowc ? lv->ks->rowc_name : "k_rhs_curved";
}

const char* cdg_gpu_version(void) { return "cdg_gpu 0.1 (sm_100a, fp64 DMMA)"; }

// out[0] = DMMA m16n8k4, out[1] = DFMA, out[2] = DMMA m16n8k8, out[3] = DMMA m16n8k16 TFLOP/s
// (best of 5, 4 CTAs x 8 warps per SM)
int cdg_gpu_measure_fp64_peak(int device, double* out) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    double* d = nullptr;
    CUDA_OK(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    const int blocks = prop.multiProcessorCount * 4, iters = 20000;
    for (int kind = 0; kind < 4; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        CUDA_OK(cudaEventRecord(e0));
        if (kind == 0)
          k_peak_dmma<<<blocks, 256>>>(d, iters);
        else if (kind == 1)
          k_peak_dfma<<<blocks, 256>>>(d, iters);
        else if (kind == 2)
          k_peak_dmma8<<<blocks, 256>>>(d, iters / 2);
        else
          k_peak_dmma16<<<blocks, 256>>>(d, iters / 4);
        CUDA_OK(cudaEventRecord(e1));
        CUDA_OK(cudaEventSynchronize(e1));
        float ms;
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0) best = std::min(best, ms);
      }
      const double warps = blocks * 8.0;
      double flops = warps * iters * 8.0 * 16 * 8 * 4 * 2;  // 8 mma/iter, 16x8x4 FMA (k8: iters/2, k16: iters/4)
      if (kind == 1) flops = blocks * 256.0 * iters * 8.0 * 2;  // 8 fma/iter/thread
      out[kind] = flops / (best * 1e-3) / 1e12;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
  });
}

int cdg_gpu_level_create(const cdg_gpu_level_desc* d, int device, cdg_gpu_level** out, char* err,
                         size_t errlen) {
  *out = nullptr;
  auto* lv = new cdg_gpu_level;
  const int st = guarded(err, errlen, [&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Status(CDG_GPU_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
    if (device < 0 || device >= ndev) throw Status(CDG_GPU_ERR_CONFIG, "bad device index");
    CUDA_OK(cudaSetDevice(device));
    lv->device = device;
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    lv->n_sms = prop.multiProcessorCount;
    if (d->degree < 1 || d->degree > 8) throw Status(CDG_GPU_ERR_CONFIG, "degree must be 1..8");
    lv->degree = d->degree;
    lv->np = d->n_basis;
    lv->ncub = d->n_cub;
    lv->ng = d->n_face_quad;
    lv->nf = 4 * d->n_face_quad;
    lv->K = d->n_elements;
    lv->n_halo = d->n_halo;
    if (lv->K < 1) throw Status(CDG_GPU_ERR_CONFIG, "level has no elements");
    lv->ks = find_set(lv->np, lv->ncub, lv->ng);
    if (!lv->ks)
      throw Status(CDG_GPU_ERR_CONFIG, "no kernel instantiation for (N_p, N_cub, N_g) = (" +
                                           std::to_string(lv->np) + ", " + std::to_string(lv->ncub) +
                                           ", " + std::to_string(lv->ng) + ")");
    lv->caller_padded = d->padded != 0;
    lv->caller_block = lv->caller_padded ? pad16(lv->np) : lv->np;
    lv->caller_tblock = lv->caller_padded ? pad16(lv->nf) : lv->nf;
    lv->bp = dev_block(lv->np);  // device layout (cdg_kernels.cuh); the caller's is pad16 or unpadded
    lv->tb = dev_tblock(lv->nf);
    const int np = lv->np, ncub = lv->ncub, nf = lv->nf, ng = lv->ng, K = lv->K;

    // ---- shared operators (operators.cpp:135-165, factored) ---------------
    std::vector<double> icub(d->interp_cub, d->interp_cub + (size_t)ncub * np);
    std::vector<double> ig(d->interp_face, d->interp_face + (size_t)nf * np);
    const double* dm[3] = {d->deriv_r, d->deriv_s, d->deriv_t};
    std::vector<double> mref((size_t)np * np, 0.0);
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) {
        double s = 0.0;
        for (int q = 0; q < ncub; ++q) s += icub[(size_t)q * np + i] * d->cub_weights[q] * icub[(size_t)q * np + j];
        mref[(size_t)i * np + j] = s;
      }
    const std::vector<double> minv = spd_inverse(mref, np);
    // A_m = M^-1 D_m^T diag(W)  [np][ncub];   LIFT = M^-1 I_g^T diag(w)  [np][nf]
    std::vector<double> amat[3];
    for (int m = 0; m < 3; ++m) {
      amat[m].assign((size_t)np * ncub, 0.0);
      for (int i = 0; i < np; ++i)
        for (int q = 0; q < ncub; ++q) {
          double s = 0.0;
          for (int j = 0; j < np; ++j) s += minv[(size_t)i * np + j] * dm[m][(size_t)q * np + j];
          amat[m][(size_t)i * ncub + q] = s * d->cub_weights[q];
        }
    }
    std::vector<double> lift((size_t)np * nf, 0.0);
    for (int i = 0; i < np; ++i)
      for (int fq = 0; fq < nf; ++fq) {
        double s = 0.0;
        for (int j = 0; j < np; ++j) s += minv[(size_t)i * np + j] * ig[(size_t)fq * np + j];
        lift[(size_t)i * nf + fq] = s * d->face_weights[fq % ng];
      }
    const int kp = (np + 7) / 8 * 8, ncub8 = (ncub + 7) / 8 * 8, np8 = (np + 7) / 8 * 8,
              nf8 = (nf + 7) / 8 * 8;
    const int k2cub = 3 * ncub8, k2 = k2cub + nf8;
    // RHS operator rows i: [chunked (m, q) volume block | -LIFT]; the aux
    // operator (viscous gradient) has the same volume block and +LIFT
    // (solver.cpp:283-309). The K order follows the kernel's cubature chunk.
    auto build_op2 = [&](int CH, double lift_sign) {
      std::vector<double> op((size_t)np * k2, 0.0);
      for (int q0 = 0; q0 < ncub8; q0 += CH) {
        const int w = std::min(CH, ncub8 - q0);
        for (int m = 0; m < 3; ++m)
          for (int ql = 0; ql < w; ++ql) {
            const int q = q0 + ql;
            if (q >= ncub) continue;
            for (int i = 0; i < np; ++i) op[(size_t)i * k2 + 3 * q0 + m * w + ql] = amat[m][(size_t)i * ncub + q];
          }
      }
      for (int i = 0; i < np; ++i)
        for (int fq = 0; fq < nf; ++fq) op[(size_t)i * k2 + k2cub + fq] = lift_sign * lift[(size_t)i * nf + fq];
      return op;
    };
    const std::vector<double> op2 = build_op2(lv->ks->ch, -1.0), opaux = build_op2(lv->ks->ch, 1.0);
    lv->frag_icub = dev_upload(make_frag(icub, ncub, np, ncub8, kp));
    {  // I_g B fragments in the natural pairing (k_interp<NAT> + fused traces)
      std::vector<double> fi;
      for (int n = 0; n < nf8 / 8; ++n)
        for (int k = 0; k < kp / 8; ++k) frag_nat(fi, ig, nf, np, n, k);
      lv->frag_ig = dev_upload(fi);
    }
    lv->frag_op2 = dev_upload(make_frag(op2, np, k2, np8, k2));
    lv->frag_aux = dev_upload(make_frag(opaux, np, k2, np8, k2));
    {  // A_k I_cub (N_p x N_p) for the affine aux-gradient volume term
      std::vector<double> fd;
      for (int m = 0; m < 3; ++m) {
        std::vector<double> dt((size_t)np * np, 0.0);
        for (int i = 0; i < np; ++i)
          for (int j = 0; j < np; ++j) {
            double s = 0.0;
            for (int q = 0; q < ncub; ++q) s += amat[m][(size_t)i * ncub + q] * icub[(size_t)q * np + j];
            dt[(size_t)i * np + j] = s;
          }
        const std::vector<double> f = make_frag(dt, np, np, np8, kp);
        fd.insert(fd.end(), f.begin(), f.end());
      }
      lv->frag_dtil = dev_upload(fd);
    }
    if (lv->ks->row_update[0]) {
      const std::vector<double> op2r = build_op2(lv->ks->row_ch, -1.0);
      std::vector<double> f2;
      for (int k = 0; k < k2 / 8; ++k)
        for (int n = 0; n < np8 / 8; ++n) frag_nat(f2, op2r, np, k2, n, k);
      lv->rfrag2 = dev_upload(f2);

      lv->use_row = true;
    }
    if (lv->ks->warp_update[0] || lv->ks->row_update[0]) {
      const int nch = (ncub + 7) / 8, nfch = (nf + 7) / 8, ks1 = kp / 8, nt = np8 / 8;
      std::vector<double> f1, f2v, f2f;
      std::vector<double> neg_lift(lift.size());
      for (size_t i = 0; i < lift.size(); ++i) neg_lift[i] = -lift[i];
      for (int ch = 0; ch < nch; ++ch)
        for (int k = 0; k < ks1; ++k) frag_nat(f1, icub, ncub, np, ch, k);
      for (int ch = 0; ch < nch; ++ch)
        for (int m = 0; m < 3; ++m)
          for (int n = 0; n < nt; ++n) frag_nat(f2v, amat[m], np, ncub, n, ch);
      for (int fc = 0; fc < nfch; ++fc)
        for (int n = 0; n < nt; ++n) frag_nat(f2f, neg_lift, np, nf, n, fc);
      lv->wfrag1 = dev_upload(f1);
      if (!lv->ks->warp_update[0] && !lv->ks->ns_update[0]) f2v.clear(), f2f.clear();
      lv->wfrag2v = dev_upload(f2v);
      lv->wfrag2f = dev_upload(f2f);
      lv->use_warp = lv->ks->warp_update[0] != nullptr;
    }
    if (lv->ks->ns_update[0] && lv->wfrag2v) {
      lv->d_ig = dev_upload(ig);
      lv->use_ns = true;
    }
    if (d->vandermonde_inv) {
      lv->d_vinv = dev_upload(std::vector<double>(d->vandermonde_inv, d->vandermonde_inv + (size_t)np * np));
      // modal basis at the cubature nodes for the J-weighted indicator:
      // the caller's modal_basis_eval table, else I_cub (V^-1)^-1
      std::vector<double> vcub;
      if (d->modal_cub) {
        vcub.assign(d->modal_cub, d->modal_cub + (size_t)ncub * np);
      } else {
        const std::vector<double> v = dense_inverse(std::vector<double>(d->vandermonde_inv,
                                                                        d->vandermonde_inv + (size_t)np * np), np);
        vcub.assign((size_t)ncub * np, 0.0);
        for (int q = 0; q < ncub; ++q)
          for (int j = 0; j < np; ++j) {
            double s = 0.0;
            for (int i = 0; i < np; ++i) s += icub[(size_t)q * np + i] * v[(size_t)i * np + j];
            vcub[(size_t)q * np + j] = s;
          }
      }
      lv->d_vcub = dev_upload(vcub);
      lv->d_wcub = dev_upload(std::vector<double>(d->cub_weights, d->cub_weights + ncub));
    }

    // ---- per-element geometry + coupling -----------------------------------
    std::vector<double> met(d->metric, d->metric + (size_t)K * 9);
    std::vector<double4> face((size_t)K * 4);
    std::vector<int2> conn((size_t)K * 4);
    std::vector<int> codes;  // [n_codes][ng]
    std::map<std::vector<int>, int> code_of;
    if (d->face_code) {
      if (!d->code_node_map || d->n_codes < 1) throw Status(CDG_GPU_ERR_CONFIG, "face_code needs code_node_map");
      codes.assign(d->code_node_map, d->code_node_map + (size_t)d->n_codes * ng);
    } else if (!d->node_map) {
      throw Status(CDG_GPU_ERR_CONFIG, "level descriptor needs node_map or face_code");
    }
    std::vector<char> is_curved(K, 0);
    for (int i = 0; i < d->n_curved; ++i)
      if (d->curved_ids && d->curved_ids[i] >= 0 && d->curved_ids[i] < K) is_curved[d->curved_ids[i]] = 1;
    for (int e = 0; e < K; ++e) {
      const double jac = is_curved[e] ? 1.0 : d->jac[e];
      if (!(jac > 1e-14))
        throw Status(CDG_GPU_ERR_NUMERICS, "inverted element " + std::to_string(e) + ": mapping Jacobian " +
                                               std::to_string(jac) + " at quadrature node 0");
      for (int f = 0; f < 4; ++f) {
        const size_t i4 = (size_t)e * 4 + f;
        face[i4] = make_double4(d->face_normal[i4 * 3 + 0], d->face_normal[i4 * 3 + 1],
                                d->face_normal[i4 * 3 + 2], d->face_sjac[i4] / jac);
        const int nb = d->neighbor[i4];
        if (nb >= 0) {
          if (nb >= K + lv->n_halo) throw Status(CDG_GPU_ERR_CONFIG, "neighbor index out of range");
          int code = 0;
          if (d->face_code) {
            code = d->face_code[i4];
          } else {
            std::vector<int> row(d->node_map + i4 * ng, d->node_map + (i4 + 1) * ng);
            auto it = code_of.find(row);
            if (it == code_of.end()) {
              code = (int)code_of.size();
              code_of.emplace(row, code);
              codes.insert(codes.end(), row.begin(), row.end());
            } else {
              code = it->second;
            }
          }
          conn[i4] = make_int2(nb, pack_face(d->neighbor_face[i4], 0, 0, code));
        } else {
          const int bc = d->bc[i4];
          if (bc < 0 || bc > 2) throw Status(CDG_GPU_ERR_CONFIG, "boundary_state: unknown kind");
          conn[i4] = make_int2(-1, pack_face(0, bc, 1, 0));
        }
      }
    }
    if (codes.empty()) codes.assign(ng, 0);
    if (lv->n_halo > 0) {
      lv->ghost_adjacent.assign(K, 0);
      for (int e = 0; e < K; ++e)
        for (int f = 0; f < 4; ++f)
          if (d->neighbor[(size_t)e * 4 + f] >= K) lv->ghost_adjacent[e] = 1;
    }
    if (d->n_curved > 0) {
      if (!d->curved_ids || !d->curved_jwr || !d->curved_face || !d->curved_minv)
        throw Status(CDG_GPU_ERR_CONFIG, "curved elements need curved_ids/jwr/face/minv");
      for (int i = 0; i < d->n_curved; ++i) {
        const int e = d->curved_ids[i];
        if (e < 0 || e >= K) throw Status(CDG_GPU_ERR_CONFIG, "curved element id out of range");
        conn[(size_t)e * 4].y |= kCurvedBit;
      }
      lv->n_curved = d->n_curved;
      lv->curved_ids = dev_upload(std::vector<int>(d->curved_ids, d->curved_ids + d->n_curved));
      lv->curved_ids_h.assign(d->curved_ids, d->curved_ids + d->n_curved);
      lv->curved_jwr = dev_upload(std::vector<double>(d->curved_jwr, d->curved_jwr + (size_t)d->n_curved * ncub * 9));
      std::vector<double4> cf((size_t)d->n_curved * nf);
      for (size_t i = 0; i < cf.size(); ++i)
        cf[i] = make_double4(d->curved_face[4 * i], d->curved_face[4 * i + 1], d->curved_face[4 * i + 2],
                             d->curved_face[4 * i + 3]);
      lv->curved_face = dev_upload(cf);
      {  // M_e^-1 transposed per element: the epilogue threads (consecutive
         // output nodes i) then read consecutive addresses
        std::vector<double> mt((size_t)d->n_curved * np * np);
        for (int c = 0; c < d->n_curved; ++c)
          for (int i = 0; i < np; ++i)
            for (int j = 0; j < np; ++j)
              mt[((size_t)c * np + j) * np + i] = d->curved_minv[((size_t)c * np + i) * np + j];
        lv->curved_minv = dev_upload(mt);
      }
      // [D_r^T D_s^T D_t^T | -I_g^T] in the chunked K layout of op2
      std::vector<double> opc((size_t)np * k2, 0.0);
      const int CHc = lv->ks->ch;
      for (int q0 = 0; q0 < ncub8; q0 += CHc) {
        const int w = std::min(CHc, ncub8 - q0);
        for (int m = 0; m < 3; ++m)
          for (int ql = 0; ql < w; ++ql) {
            const int q = q0 + ql;
            if (q >= ncub) continue;
            for (int i = 0; i < np; ++i) opc[(size_t)i * k2 + 3 * q0 + m * w + ql] = dm[m][(size_t)q * np + i];
          }
      }
      for (int i = 0; i < np; ++i)
        for (int fq = 0; fq < nf; ++fq) opc[(size_t)i * k2 + k2cub + fq] = -ig[(size_t)fq * np + i];
      lv->frag_opc = dev_upload(make_frag(opc, np, k2, np8, k2));
      if (lv->ks->rowc_update[0]) {  // the same operator for k_rhs_rowc: its chunking, natural pairing
        std::vector<double> opr((size_t)np * k2, 0.0);
        const int CHr = lv->ks->rowc_ch;
        for (int q0 = 0; q0 < ncub8; q0 += CHr) {
          const int w = std::min(CHr, ncub8 - q0);
          for (int m = 0; m < 3; ++m)
            for (int ql = 0; ql < w; ++ql) {
              const int q = q0 + ql;
              if (q >= ncub) continue;
              for (int i = 0; i < np; ++i) opr[(size_t)i * k2 + 3 * q0 + m * w + ql] = dm[m][(size_t)q * np + i];
            }
        }
        for (int i = 0; i < np; ++i)
          for (int fq = 0; fq < nf; ++fq) opr[(size_t)i * k2 + k2cub + fq] = -ig[(size_t)fq * np + i];
        std::vector<double> f2;
        for (int k = 0; k < k2 / 8; ++k)
          for (int n = 0; n < np8 / 8; ++n) frag_nat(f2, opr, np, k2, n, k);
        lv->rfrag_opc = dev_upload(f2);
        lv->use_rowc = lv->ks->warp_update[0] || lv->ks->row_update[0];
      }
      // tiles (of the affine kernel's E elements) with at least one affine
      // element: the affine kernels skip the all-curved tiles. The warp-tile
      // kernel and the aux kernel walk 16-element tiles as well.
      {
        const int E = lv->use_row ? lv->ks->row_e : lv->ks->E;
        if (E != 16 || lv->ks->E != 16)
          throw Status(CDG_GPU_ERR_CONFIG, "curved levels need 16-element affine tiles");
        std::vector<int> at;
        for (int t = 0; t * E < K; ++t) {
          bool any = false;
          for (int e = t * E; e < std::min(K, t * E + E); ++e) any = any || !is_curved[e];
          if (any) at.push_back(t);
        }
        lv->n_affine_tiles = (int)at.size();
        if (at.empty()) at.push_back(0);
        lv->d_affine_tiles = dev_upload(at);
      }
      // epilogue scratch for configurations whose vol panel does not fit smem (p=8)
      CUDA_OK(cudaMalloc(&lv->curved_vol, sizeof(double) * (size_t)d->n_curved * 5 * (np8 + 1)));
    }
    {
      std::vector<double> jv(K);
      for (int e = 0; e < K; ++e) jv[e] = is_curved[e] ? 1.0 : d->jac[e];
      lv->d_jac = dev_upload(jv);
      if (d->n_curved > 0) {
        std::vector<int> slot(K, -1);
        for (int i = 0; i < d->n_curved; ++i) slot[d->curved_ids[i]] = i;
        lv->d_curved_slot = dev_upload(slot);
        if (d->curved_jac)
          lv->d_curved_jac = dev_upload(std::vector<double>(d->curved_jac, d->curved_jac + (size_t)d->n_curved * ncub));
      }
    }
    lv->metric = dev_upload(met);
    lv->face = dev_upload(face);
    lv->conn = dev_upload(conn);
    lv->code_map = dev_upload(codes);
    if (d->h) lv->h = dev_upload(std::vector<double>(d->h, d->h + K));

    if (lv->use_row && wa_poorly_quantized(lv)) lv->use_row = false;  // (n_curved known here)

    // ---- state + workspace -------------------------------------------------
    const size_t n = (size_t)K * 5 * lv->bp;
    const size_t ntr = (size_t)(K + lv->n_halo) * 5 * lv->tb;
    CUDA_OK(cudaMalloc(&lv->u, n * sizeof(double)));
    lv->ubuf[0] = lv->u;
    CUDA_OK(cudaMalloc(&lv->res, n * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->rhs, n * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->traces, ntr * sizeof(double)));
    CUDA_OK(cudaMemset(lv->u, 0, n * sizeof(double)));
    CUDA_OK(cudaMemset(lv->res, 0, n * sizeof(double)));
    CUDA_OK(cudaMemset(lv->rhs, 0, n * sizeof(double)));
    CUDA_OK(cudaMemset(lv->traces, 0, ntr * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->eps, K * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->sqrt_eps, (K + lv->n_halo) * sizeof(double)));
    CUDA_OK(cudaMemset(lv->eps, 0, K * sizeof(double)));
    CUDA_OK(cudaMemset(lv->sqrt_eps, 0, (K + lv->n_halo) * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->d_maxeps, sizeof(unsigned long long)));
    CUDA_OK(cudaMalloc(&lv->d_fallbacks, sizeof(unsigned long long)));
    CUDA_OK(cudaMemset(lv->d_fallbacks, 0, sizeof(unsigned long long)));
    lv->gas.hllc_fallbacks = lv->d_fallbacks;
    CUDA_OK(cudaMalloc(&lv->d_coef, sizeof(StageCoef)));
    CUDA_OK(cudaMallocHost(&lv->h_coef, sizeof(StageCoef)));
    CUDA_OK(cudaMalloc(&lv->d_err, sizeof(DevError)));
    CUDA_OK(cudaMemset(lv->d_err, 0, sizeof(DevError)));
    CUDA_OK(cudaMallocHost(&lv->h_err, sizeof(DevError)));
    lv->scratch_n = 1024;
    CUDA_OK(cudaMalloc(&lv->d_scratch, lv->scratch_n * sizeof(double)));
    lv->h_scratch.resize(lv->scratch_n);
    CUDA_OK(cudaStreamCreateWithFlags(&lv->stream, cudaStreamNonBlocking));
    for (auto& e : lv->ev) CUDA_OK(cudaEventCreate(&e));
    std::memcpy(lv->freestream, d->freestream, sizeof(lv->freestream));
    for (int c = 0; c < 5; ++c) lv->gas.fs[c] = d->freestream[c];
    // opt in to > 48 KB dynamic shared memory
    for (auto fn : {lv->ks->rhs_update, lv->ks->rhs_only, lv->ks->visc_rhs_update, lv->ks->visc_rhs_only})
      CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_rhs));
    CUDA_OK(cudaFuncSetAttribute(lv->ks->aux_q, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)lv->ks->smem_aux));
    if (lv->ks->row_update[0])
      for (auto fn : {lv->ks->row_update[0], lv->ks->row_update[1], lv->ks->row_only[0], lv->ks->row_only[1]})
        CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_row));
    if (lv->ks->warp_update[0])
      for (auto fn : {lv->ks->warp_update[0], lv->ks->warp_update[1], lv->ks->warp_only[0], lv->ks->warp_only[1]})
        CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_warp));
    if (lv->ks->ns_update[0])
      for (auto fn : {lv->ks->ns_update[0], lv->ks->ns_update[1]})
        CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_ns));
    if (lv->n_curved && lv->ks->rowc_aux) {
      CUDA_OK(cudaFuncSetAttribute(lv->ks->rowc_aux, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)lv->ks->smem_rowc_aux));
      for (auto fn : {lv->ks->rowc_update[0], lv->ks->rowc_update[1], lv->ks->rowc_only[0], lv->ks->rowc_only[1],
                      lv->ks->rowc_visc_update[0], lv->ks->rowc_visc_update[1], lv->ks->rowc_visc_only[0],
                      lv->ks->rowc_visc_only[1]})
        CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_rowc));
    }
    if (lv->n_curved)
      for (auto fn : {lv->ks->curved_update, lv->ks->curved_only, lv->ks->curved_visc_update,
                      lv->ks->curved_visc_only, lv->ks->aux_curved})
        CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_curved));
    for (auto fn : {lv->ks->traces, lv->ks->cubinterp})
      CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_traces));
    CUDA_OK(cudaFuncSetAttribute(lv->ks->qn_traces, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv->ks->smem_qn));
    CUDA_OK(cudaDeviceSynchronize());
  });
  if (st != CDG_GPU_OK) {
    cdg_gpu_level_destroy(lv);
    return st;
  }
  *out = lv;
  return CDG_GPU_OK;
}

// Scalable level setup from the mesh itself (the C++ caller's Mesh /
// FaceLink, mesh.hpp:23-57): the compact affine geometry (compute_mapping,
// operators.cpp:32-121, for a straight tet: one metric, Jacobian and normal
// per element / face) and the face-node pairing from FaceLink.perm (one table
// per vertex permutation; on conforming faces with the symmetric face rules it
// equals the reference's nearest-point node_map, solver.cpp:144-172) -- O(K),
// ~100 bytes per element, instead of DgLevel's ~140 KB per element and
// O(K N_g^2) pairing.
int cdg_gpu_level_create_from_mesh(const cdg_gpu_level_desc* tables, const cdg_gpu_mesh_desc* m, int device,
                                   cdg_gpu_level** out, char* err, size_t errlen) {
  *out = nullptr;
  cdg_gpu_level_desc d = *tables;
  std::vector<double> metric, jac, normal, sjac, h;
  std::vector<int> nb, nbf, bc, code, cmap;
  const int st = guarded(err, errlen, [&] {
    static const double TV[4][3] = {{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}};  // refelem.hpp
    static const int FV[4][3] = {{0, 2, 1}, {0, 1, 3}, {1, 2, 3}, {0, 3, 2}};             // reference face order
    static const int PERMS[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int K = m->n_elements, ng = tables->n_face_quad;
    if (K < 1 || !m->vertices || !m->tets || !m->neighbor || !m->neighbor_face || !m->face_perm || !m->bc ||
        !m->face_nodes)
      throw Status(CDG_GPU_ERR_CONFIG, "level_create_from_mesh: incomplete mesh descriptor");
    double wc = 0.0, wf = 0.0;
    for (int q = 0; q < tables->n_cub; ++q) wc += tables->cub_weights[q];
    for (int g = 0; g < ng; ++g) wf += tables->face_weights[g];
    metric.resize((size_t)K * 9), jac.resize(K), normal.resize((size_t)K * 12), sjac.resize((size_t)K * 4),
        h.resize(K), nb.resize((size_t)K * 4), nbf.resize((size_t)K * 4), bc.resize((size_t)K * 4),
        code.resize((size_t)K * 4);
    for (int e = 0; e < K; ++e) {
      const int* t = m->tets + (size_t)e * 4;
      double f[3][3];  // f[i][m] = dx_i/dr_m
      for (int v = 0; v < 4; ++v)
        if (t[v] < 0 || t[v] >= m->n_vertices) throw Status(CDG_GPU_ERR_CONFIG, "tet vertex index out of range");
      const double* x0 = m->vertices + (size_t)t[0] * 3;
      for (int mm = 0; mm < 3; ++mm) {
        const double* x1 = m->vertices + (size_t)t[mm + 1] * 3;
        for (int i = 0; i < 3; ++i) f[i][mm] = 0.5 * (x1[i] - x0[i]);
      }
      const double c00 = f[1][1] * f[2][2] - f[1][2] * f[2][1], c01 = f[1][2] * f[2][0] - f[1][0] * f[2][2],
                   c02 = f[1][0] * f[2][1] - f[1][1] * f[2][0];
      const double J = f[0][0] * c00 + f[0][1] * c01 + f[0][2] * c02;
      if (!(J > 1e-14))
        throw Status(CDG_GPU_ERR_NUMERICS, "inverted element " + std::to_string(e) + ": mapping Jacobian " +
                                               std::to_string(J) + " at quadrature node 0");
      const double inv[3][3] = {{c00 / J, (f[0][2] * f[2][1] - f[0][1] * f[2][2]) / J, (f[0][1] * f[1][2] - f[0][2] * f[1][1]) / J},
                                {c01 / J, (f[0][0] * f[2][2] - f[0][2] * f[2][0]) / J, (f[0][2] * f[1][0] - f[0][0] * f[1][2]) / J},
                                {c02 / J, (f[0][1] * f[2][0] - f[0][0] * f[2][1]) / J, (f[0][0] * f[1][1] - f[0][1] * f[1][0]) / J}};
      for (int mm = 0; mm < 3; ++mm)
        for (int i = 0; i < 3; ++i) metric[(size_t)e * 9 + mm * 3 + i] = inv[mm][i];
      jac[e] = J;
      double area = 0.0;
      for (int fc = 0; fc < 4; ++fc) {
        double xa[3], xb[3];
        for (int i = 0; i < 3; ++i) {
          xa[i] = xb[i] = 0.0;
          for (int mm = 0; mm < 3; ++mm) {
            xa[i] += f[i][mm] * 0.5 * (TV[FV[fc][1]][mm] - TV[FV[fc][0]][mm]);
            xb[i] += f[i][mm] * 0.5 * (TV[FV[fc][2]][mm] - TV[FV[fc][0]][mm]);
          }
        }
        const double n[3] = {xa[1] * xb[2] - xa[2] * xb[1], xa[2] * xb[0] - xa[0] * xb[2], xa[0] * xb[1] - xa[1] * xb[0]};
        const double s = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        for (int i = 0; i < 3; ++i) normal[(size_t)e * 12 + fc * 3 + i] = n[i] / s;
        sjac[(size_t)e * 4 + fc] = s;
        area += s * wf;
        const size_t i4 = (size_t)e * 4 + fc;
        nb[i4] = m->neighbor[i4];
        nbf[i4] = nb[i4] >= 0 ? m->neighbor_face[i4] : 0;
        bc[i4] = nb[i4] >= 0 ? 0 : m->bc[i4];
        code[i4] = 0;
        if (nb[i4] >= 0) {
          const int* pm = m->face_perm + i4 * 3;
          int c = -1;
          for (int k = 0; k < 6; ++k)
            if (PERMS[k][0] == pm[0] && PERMS[k][1] == pm[1] && PERMS[k][2] == pm[2]) c = k;
          if (c < 0) throw Status(CDG_GPU_ERR_CONFIG, "face_perm is not a permutation of (0, 1, 2)");
          code[i4] = c;
        }
      }
      h[e] = 6.0 * J * wc / area;  // ElementGeometry::h() = 6V/A (operators.hpp:37)
    }
    // node maps per permutation: barycentric coordinates of face 0's rule on its
    // vertices (A, B, C) = TV[0], TV[2], TV[1]; x = A + u (B - A) + v (C - A)
    std::vector<double> lam((size_t)ng * 3);
    {
      const double* A = TV[FV[0][0]];
      const double* B = TV[FV[0][1]];
      const double* Cc = TV[FV[0][2]];
      double e1[3], e2[3];
      for (int i = 0; i < 3; ++i) e1[i] = B[i] - A[i], e2[i] = Cc[i] - A[i];
      const double a11 = e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2], a12 = e1[0] * e2[0] + e1[1] * e2[1] + e1[2] * e2[2],
                   a22 = e2[0] * e2[0] + e2[1] * e2[1] + e2[2] * e2[2], det = a11 * a22 - a12 * a12;
      for (int g = 0; g < ng; ++g) {
        double r[3];
        for (int i = 0; i < 3; ++i) r[i] = m->face_nodes[g * 3 + i] - A[i];
        const double b1 = r[0] * e1[0] + r[1] * e1[1] + r[2] * e1[2], b2 = r[0] * e2[0] + r[1] * e2[1] + r[2] * e2[2];
        const double u = (a22 * b1 - a12 * b2) / det, v = (a11 * b2 - a12 * b1) / det;
        lam[g * 3 + 0] = 1.0 - u - v, lam[g * 3 + 1] = u, lam[g * 3 + 2] = v;
      }
    }
    cmap.resize((size_t)6 * ng);
    for (int k = 0; k < 6; ++k)
      for (int g = 0; g < ng; ++g) {
        double theirs[3];
        for (int i = 0; i < 3; ++i) theirs[PERMS[k][i]] = lam[g * 3 + i];
        int best_h = -1;
        double best = 1e300;
        for (int hh = 0; hh < ng; ++hh) {
          double dd = 0.0;
          for (int i = 0; i < 3; ++i) dd += (theirs[i] - lam[hh * 3 + i]) * (theirs[i] - lam[hh * 3 + i]);
          if (dd < best) best = dd, best_h = hh;
        }
        if (std::sqrt(best) > 1e-10)
          throw Status(CDG_GPU_ERR_CONFIG, "face rule is not invariant under the vertex permutation");
        cmap[(size_t)k * ng + g] = best_h;
      }
    d.n_elements = K;
    d.n_halo = m->n_halo;
    d.metric = metric.data();
    d.jac = jac.data();
    d.face_normal = normal.data();
    d.face_sjac = sjac.data();
    d.h = h.data();
    d.neighbor = nb.data();
    d.neighbor_face = nbf.data();
    d.bc = bc.data();
    d.node_map = nullptr;
    d.face_code = code.data();
    d.code_node_map = cmap.data();
    d.n_codes = 6;
    d.n_curved = 0;
  });
  if (st != CDG_GPU_OK) return st;
  return cdg_gpu_level_create(&d, device, out, err, errlen);
}

void cdg_gpu_level_destroy(cdg_gpu_level* lv) {
  if (!lv) return;
  cudaSetDevice(lv->device);
  if (lv->graph) cudaGraphExecDestroy(lv->graph);
  if (lv->graph_visc) cudaGraphExecDestroy(lv->graph_visc);
  for (auto ge : lv->gft)
    if (ge) cudaGraphExecDestroy(ge);
  for (auto ge : lv->gns)
    if (ge) cudaGraphExecDestroy(ge);
  for (void* p : {(void*)lv->ubuf[0], (void*)lv->ubuf[1], (void*)lv->d_ig, (void*)lv->res, (void*)lv->rhs, (void*)(lv->tbuf[1] ? lv->tbuf[0] : lv->traces), (void*)lv->before,
                  (void*)lv->q, (void*)lv->qtr, (void*)lv->qcub, (void*)lv->eps, (void*)lv->sqrt_eps, (void*)lv->d_vinv, (void*)lv->d_vcub, (void*)lv->d_wcub, (void*)lv->d_jac,
                  (void*)lv->d_curved_jac, (void*)lv->d_curved_slot,
                  (void*)lv->d_maxeps, (void*)lv->d_fallbacks, (void*)lv->metric, (void*)lv->face, (void*)lv->conn,
                  (void*)lv->code_map, (void*)lv->h, (void*)lv->frag_icub, (void*)lv->frag_op2,
                  (void*)lv->frag_ig, (void*)lv->frag_aux, (void*)lv->frag_dtil, (void*)lv->wfrag1, (void*)lv->wfrag2v, (void*)lv->wfrag2f, (void*)lv->rfrag2, (void*)lv->tbuf[1],
                  (void*)lv->curved_ids, (void*)lv->curved_jwr, (void*)lv->curved_minv, (void*)lv->frag_opc,
                  (void*)lv->rfrag_opc, (void*)lv->d_affine_tiles, (void*)lv->curved_vol, (void*)lv->curved_face, (void*)lv->d_coef, (void*)lv->d_err,
                  (void*)lv->d_scratch, (void*)lv->d_send_idx, (void*)lv->d_recv_idx,
                  (void*)lv->d_tiles_int, (void*)lv->d_tiles_halo,
                  (void*)lv->d_ctiles_int, (void*)lv->d_ctiles_halo})
    if (p) cudaFree(p);
  for (double* p : {lv->hsend[0], lv->hsend[1], lv->hrecv})
    if (p) cudaFree(p);
  for (int s = 0; s < 2; ++s) {
    if (lv->ring[s]) cudaFreeHost(lv->ring[s]);
    if (lv->ring_ev[s]) cudaEventDestroy(lv->ring_ev[s]);
  }
  if (lv->h_coef) cudaFreeHost(lv->h_coef);
  if (lv->h_err) cudaFreeHost(lv->h_err);
  for (auto& e : lv->ev)
    if (e) cudaEventDestroy(e);
  if (lv->stream) cudaStreamDestroy(lv->stream);
  delete lv;
}

void cdg_gpu_level_sizes(const cdg_gpu_level* lv, int* s) {
  s[0] = lv->K;
  s[1] = lv->np;
  s[2] = lv->ncub;
  s[3] = lv->ng;
  s[4] = lv->caller_block;
  s[5] = lv->caller_tblock;
  s[6] = lv->bp;
  s[7] = lv->n_halo;
}

void* cdg_gpu_stream(cdg_gpu_level* lv) { return lv->stream; }
long long cdg_gpu_launch_count(const cdg_gpu_level* lv) { return lv->launches; }

// Row copy between the caller's layout and the device rows. Host <-> device
// with different row lengths goes through a device staging buffer in the
// CALLER's layout (one contiguous PCIe transfer + a pitched device-to-device
// copy) -- a pitched copy straight from pageable host memory moves row by row.
// The staging buffer is zeroed once and only its value columns are ever
// written, so the caller's padding stays exactly zero.
// rows [0, rows) split over up to 16 host threads (the pinned-ring packing)
static void parallel_rows(int rows, const std::function<void(int, int)>& f) {
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int nt = std::min({hw, 16, std::max(1, rows / 4096)});
  if (nt <= 1) {
    f(0, rows);
    return;
  }
  std::vector<std::thread> th;
  const int per = (rows + nt - 1) / nt;
  for (int i = 0; i < nt; ++i) {
    const int r0 = i * per, r1 = std::min(rows, r0 + per);
    if (r0 < r1) th.emplace_back([&f, r0, r1] { f(r0, r1); });
  }
  for (auto& t : th) t.join();
}

// Rows of `values` doubles between a row length of src_block and dst_block.
// Host <-> device: the caller's (pageable) rows are packed by host threads into
// a pinned two-slot ring in the device layout and moved by DMA, one slot
// packing while the other transfers (the reference's SolutionStore round trip
// of rk_step through the adapter); device <-> device: one 2D copy.
static void copy_rows(cdg_gpu_level* lv, double* dst, int dst_block, const double* src, int src_block,
                      int values, int rows, cudaMemcpyKind kind) {
  if (kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost) {
    const bool h2d = kind == cudaMemcpyHostToDevice;
    const int db = h2d ? dst_block : src_block, hb = h2d ? src_block : dst_block;  // device / host rows
    // slots of up to 64 MB, no larger than the copy (small levels pin little)
    const size_t want = std::min<size_t>((size_t)8 << 20, std::max<size_t>((size_t)rows * db, 1));
    if (lv->ring_doubles < want) {
      for (int s = 0; s < 2; ++s) {
        if (lv->ring_ev[s]) CUDA_OK(cudaEventSynchronize(lv->ring_ev[s]));
        if (lv->ring[s]) cudaFreeHost(lv->ring[s]);
        lv->ring[s] = nullptr;
      }
      lv->ring_doubles = 0;
      for (int s = 0; s < 2; ++s) {
        CUDA_OK(cudaHostAlloc(&lv->ring[s], want * sizeof(double), cudaHostAllocDefault));
        if (!lv->ring_ev[s]) CUDA_OK(cudaEventCreateWithFlags(&lv->ring_ev[s], cudaEventDisableTiming));
      }
      lv->ring_doubles = want;
    }
    const int rc = (int)std::max<size_t>(1, lv->ring_doubles / db);  // rows per slot
    const int nchunks = (rows + rc - 1) / rc;
    auto chunk = [&](int c, int* r0, int* n) {
      *r0 = c * rc;
      *n = std::min(rc, rows - *r0);
    };
    if (h2d) {
      for (int c = 0; c < nchunks; ++c) {
        int r0, n;
        chunk(c, &r0, &n);
        const int s = c & 1;
        CUDA_OK(cudaEventSynchronize(lv->ring_ev[s]));  // the slot's previous transfer is done
        double* pin = lv->ring[s];
        parallel_rows(n, [&](int a, int b) {
          for (int r = a; r < b; ++r) {
            double* pr = pin + (size_t)r * db;
            std::memcpy(pr, src + (size_t)(r0 + r) * hb, (size_t)values * sizeof(double));
            if (db > values) std::memset(pr + values, 0, (size_t)(db - values) * sizeof(double));
          }
        });
        CUDA_OK(cudaMemcpyAsync(dst + (size_t)r0 * db, pin, (size_t)n * db * sizeof(double), kind, lv->stream));
        CUDA_OK(cudaEventRecord(lv->ring_ev[s], lv->stream));
      }
    } else {
      auto unpack = [&](int c) {
        int r0, n;
        chunk(c, &r0, &n);
        const int s = c & 1;
        CUDA_OK(cudaEventSynchronize(lv->ring_ev[s]));
        const double* pin = lv->ring[s];
        parallel_rows(n, [&](int a, int b) {
          for (int r = a; r < b; ++r) {
            double* hr = dst + (size_t)(r0 + r) * hb;
            std::memcpy(hr, pin + (size_t)r * db, (size_t)values * sizeof(double));
            if (hb > values) std::memset(hr + values, 0, (size_t)(hb - values) * sizeof(double));  // caller padding
          }
        });
      };
      for (int c = 0; c < nchunks; ++c) {
        int r0, n;
        chunk(c, &r0, &n);
        const int s = c & 1;  // its previous chunk (c - 2) was unpacked in iteration c - 1
        CUDA_OK(cudaMemcpyAsync(lv->ring[s], src + (size_t)r0 * db, (size_t)n * db * sizeof(double), kind, lv->stream));
        CUDA_OK(cudaEventRecord(lv->ring_ev[s], lv->stream));
        if (c > 0) unpack(c - 1);
      }
      if (nchunks > 0) unpack(nchunks - 1);
    }
    return;
  }
  if (dst_block == src_block) {
    CUDA_OK(cudaMemcpyAsync(dst, src, (size_t)rows * src_block * sizeof(double), kind, lv->stream));
    return;
  }
  CUDA_OK(cudaMemcpy2DAsync(dst, dst_block * sizeof(double), src, src_block * sizeof(double),
                            values * sizeof(double), rows, kind, lv->stream));
}

int cdg_gpu_set_state(cdg_gpu_level* lv, const double* u, const double* res) {
  lv->traces_valid = false;
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    copy_rows(lv, lv->u, lv->bp, u, lv->caller_block, lv->np, lv->n_rows(), cudaMemcpyHostToDevice);
    if (res)
      copy_rows(lv, lv->res, lv->bp, res, lv->caller_block, lv->np, lv->n_rows(), cudaMemcpyHostToDevice);
    else
      CUDA_OK(cudaMemsetAsync(lv->res, 0, (size_t)lv->n_rows() * lv->bp * sizeof(double), lv->stream));
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_set_state_device(cdg_gpu_level* lv, const double* u, const double* res) {
  lv->traces_valid = false;
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    copy_rows(lv, lv->u, lv->bp, u, lv->caller_block, lv->np, lv->n_rows(), cudaMemcpyDeviceToDevice);
    if (res)
      copy_rows(lv, lv->res, lv->bp, res, lv->caller_block, lv->np, lv->n_rows(), cudaMemcpyDeviceToDevice);
    else
      CUDA_OK(cudaMemsetAsync(lv->res, 0, (size_t)lv->n_rows() * lv->bp * sizeof(double), lv->stream));
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_get_state(cdg_gpu_level* lv, double* u, double* res) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    if (u) copy_rows(lv, u, lv->caller_block, lv->u, lv->bp, lv->np, lv->n_rows(), cudaMemcpyDeviceToHost);
    if (res)
      copy_rows(lv, res, lv->caller_block, lv->res, lv->bp, lv->np, lv->n_rows(), cudaMemcpyDeviceToHost);
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_device_buffers(cdg_gpu_level* lv, double** u, double** res, double** traces) {
  if (u) *u = lv->u;
  if (res) *res = lv->res;
  if (traces) *traces = lv->traces;
  return CDG_GPU_OK;
}

int cdg_gpu_interpolate_to_faces(cdg_gpu_level* lv, double* traces_out) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    launch_traces(lv, lv->u, lv->traces);
    CUDA_OK(cudaGetLastError());
    if (traces_out)
      copy_rows(lv, traces_out, lv->caller_tblock, lv->traces, lv->tb, lv->nf, lv->n_rows(),
                cudaMemcpyDeviceToHost);
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_compute_rhs(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, double* rhs_out, char* err,
                        size_t errlen) {
  NvtxRange nvtx_("cdg_gpu_compute_rhs");
  return guarded(err, errlen, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    if (cfg->riemann != 0 && cfg->riemann != 1)
      throw Status(CDG_GPU_ERR_CONFIG, "unknown Riemann solver (llf|hllc)");
    lv->gas.gamma = cfg->gamma;
    lv->gas.riemann = cfg->riemann;
    const bool viscous = viscosity_phase(lv, cfg);
    lv->last_viscous = viscous;
    if (!viscous) launch_traces(lv, lv->u, lv->traces);
    launch_rhs(lv, false, viscous, 0);
    CUDA_OK(cudaGetLastError());
    check_device_error(lv);
    if (rhs_out)
      copy_rows(lv, rhs_out, lv->caller_block, lv->rhs, lv->bp, lv->np, lv->n_rows(), cudaMemcpyDeviceToHost);
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_rk_steps(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, int nsteps, double dt,
                     const double a[5], const double b[5], char* err, size_t errlen) {
  NvtxRange nvtx_("cdg_gpu_rk_steps");
  return guarded(err, errlen, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    if (cfg->riemann != 0 && cfg->riemann != 1)
      throw Status(CDG_GPU_ERR_CONFIG, "unknown Riemann solver (llf|hllc)");
    lv->gas.gamma = cfg->gamma;
    lv->gas.riemann = cfg->riemann;
    lv->h_coef->dt = dt;
    for (int i = 0; i < 5; ++i) {
      lv->h_coef->a[i] = a[i];
      lv->h_coef->b[i] = b[i];
    }
    CUDA_OK(cudaMemcpyAsync(lv->d_coef, lv->h_coef, sizeof(StageCoef), cudaMemcpyHostToDevice, lv->stream));
    if (cfg->visc_enabled) {
      // viscous_active (solver.cpp:257-259) is decided per stage on the device
      // (gated kernels), so one viscous RK step is a CUDA graph as well
      ensure_viscous_buffers(lv, cfg);
      lv->traces_valid = false;
      if (!lv->graph_visc || std::memcmp(&lv->graph_visc_cfg, cfg, sizeof *cfg) != 0) {
        if (lv->graph_visc) {
          cudaGraphExecDestroy(lv->graph_visc);
          lv->graph_visc = nullptr;
        }
        cudaGraph_t g;
        const long long l0 = lv->launches;
        CUDA_OK(cudaStreamBeginCapture(lv->stream, cudaStreamCaptureModeThreadLocal));
        try {
          for (int stage = 0; stage < 5; ++stage) viscous_stage_gated(lv, cfg, stage);
        } catch (...) {
          lv->cur_gate = nullptr;
          cudaStreamEndCapture(lv->stream, &g);
          throw;
        }
        lv->graph_visc_launches = (int)(lv->launches - l0);
        lv->launches = l0;  // counted at replay
        CUDA_OK(cudaStreamEndCapture(lv->stream, &g));
        CUDA_OK(cudaGraphInstantiate(&lv->graph_visc, g, 0));
        CUDA_OK(cudaGraphDestroy(g));
        lv->graph_visc_cfg = *cfg;
      }
      for (int s = 0; s < nsteps; ++s) {
        CUDA_OK(cudaGraphLaunch(lv->graph_visc, lv->stream));
        lv->launches += lv->graph_visc_launches;
      }
      CUDA_OK(cudaGetLastError());
      check_device_error(lv);
      unsigned long long bits = 0;  // viscous_active of the last stage (aux_gradient validity)
      CUDA_OK(cudaMemcpy(&bits, lv->d_maxeps, sizeof bits, cudaMemcpyDeviceToHost));
      lv->last_viscous = bits != 0;
      return;
    }
    if (ns_path(lv)) {
      // neighbour-state kernel: stage s reads ubuf[(b+s)%2] and writes the
      // other; five stages per step, so the state changes buffer every step
      ensure_ubuf(lv);
      double* const u_entry = lv->u;
      auto stage_launch = [&](int b, int stage) {
        launch_rhs_ns(lv, stage, lv->ubuf[(b + stage) & 1], lv->ubuf[(b + stage + 1) & 1]);
      };
      if (lv->profiling) {
        float t_rhs = 0.f;
        for (int s = 0; s < nsteps; ++s) {
          for (int stage = 0; stage < 5; ++stage) {
            CUDA_OK(cudaEventRecord(lv->ev[1], lv->stream));
            stage_launch(lv->ucur, stage);
            CUDA_OK(cudaEventRecord(lv->ev[2], lv->stream));
            CUDA_OK(cudaEventSynchronize(lv->ev[2]));
            float y;
            CUDA_OK(cudaEventElapsedTime(&y, lv->ev[1], lv->ev[2]));
            t_rhs += y;
          }
          lv->ucur ^= 1;
          lv->u = lv->ubuf[lv->ucur];
        }
        lv->prof[0] = 0.0;
        lv->prof[1] = t_rhs;
        lv->prof[2] = 5.0 * nsteps;
      } else {
        for (int s = 0; s < nsteps; ++s) {
          const int b = lv->ucur;
          if (!lv->gns[b] || lv->gns_riemann[b] != cfg->riemann || lv->gns_gamma[b] != cfg->gamma) {
            if (lv->gns[b]) cudaGraphExecDestroy(lv->gns[b]);
            lv->gns[b] = nullptr;
            cudaGraph_t g;
            const long long l0 = lv->launches;
            CUDA_OK(cudaStreamBeginCapture(lv->stream, cudaStreamCaptureModeThreadLocal));
            for (int stage = 0; stage < 5; ++stage) stage_launch(b, stage);
            lv->gns_launches = (int)(lv->launches - l0);
            lv->launches = l0;
            CUDA_OK(cudaStreamEndCapture(lv->stream, &g));
            CUDA_OK(cudaGraphInstantiate(&lv->gns[b], g, 0));
            CUDA_OK(cudaGraphDestroy(g));
            lv->gns_riemann[b] = cfg->riemann;
            lv->gns_gamma[b] = cfg->gamma;
          }
          CUDA_OK(cudaGraphLaunch(lv->gns[b], lv->stream));
          lv->launches += lv->gns_launches;
          lv->ucur ^= 1;
          lv->u = lv->ubuf[lv->ucur];
        }
      }
      lv->traces_valid = false;                       // no traces on this path
      if (lv->u != u_entry) drop_graphs_except_ns(lv);  // they baked the other state buffer
      CUDA_OK(cudaGetLastError());
      check_device_error(lv);
      return;
    }
    if (fused_traces(lv)) {
      // fused traces: each RHS launch writes the next stage's traces into the
      // other half of a double buffer; a trace kernel seeds it only when the
      // state changed since the last fused stage
      ensure_tbuf(lv);
      auto stage_launch = [&](int b, int stage) {  // reads tbuf[(b+s)%2], writes the other
        lv->traces = lv->tbuf[(b + stage) & 1];
        lv->cur_traces_out = lv->tbuf[(b + stage + 1) & 1];
        launch_rhs(lv, true, false, stage);
        lv->cur_traces_out = nullptr;
        lv->traces = lv->tbuf[lv->tcur];
      };
      float t_tr = 0.f, t_rhs = 0.f;
      if (lv->profiling) CUDA_OK(cudaEventRecord(lv->ev[0], lv->stream));
      seed_traces(lv);
      if (lv->profiling) {
        CUDA_OK(cudaEventRecord(lv->ev[1], lv->stream));
        CUDA_OK(cudaEventSynchronize(lv->ev[1]));
        CUDA_OK(cudaEventElapsedTime(&t_tr, lv->ev[0], lv->ev[1]));
        for (int s = 0; s < nsteps; ++s) {
          for (int stage = 0; stage < 5; ++stage) {
            CUDA_OK(cudaEventRecord(lv->ev[1], lv->stream));
            stage_launch(lv->tcur, stage);
            CUDA_OK(cudaEventRecord(lv->ev[2], lv->stream));
            CUDA_OK(cudaEventSynchronize(lv->ev[2]));
            float y;
            CUDA_OK(cudaEventElapsedTime(&y, lv->ev[1], lv->ev[2]));
            t_rhs += y;
          }
          lv->tcur ^= 1;
          lv->traces = lv->tbuf[lv->tcur];
        }
        lv->prof[0] = t_tr;
        lv->prof[1] = t_rhs;
        lv->prof[2] = 5.0 * nsteps + 1;
      } else {
        for (int s = 0; s < nsteps; ++s) {
          const int b = lv->tcur;
          if (!lv->gft[b] || lv->gft_riemann[b] != cfg->riemann || lv->gft_gamma[b] != cfg->gamma) {
            if (lv->gft[b]) cudaGraphExecDestroy(lv->gft[b]);
            lv->gft[b] = nullptr;
            cudaGraph_t g;
            const long long l0 = lv->launches;
            CUDA_OK(cudaStreamBeginCapture(lv->stream, cudaStreamCaptureModeThreadLocal));
            for (int stage = 0; stage < 5; ++stage) stage_launch(b, stage);
            lv->gft_launches = (int)(lv->launches - l0);
            lv->launches = l0;
            CUDA_OK(cudaStreamEndCapture(lv->stream, &g));
            CUDA_OK(cudaGraphInstantiate(&lv->gft[b], g, 0));
            CUDA_OK(cudaGraphDestroy(g));
            lv->gft_riemann[b] = cfg->riemann;
            lv->gft_gamma[b] = cfg->gamma;
          }
          CUDA_OK(cudaGraphLaunch(lv->gft[b], lv->stream));
          lv->launches += lv->gft_launches;
          lv->tcur ^= 1;
          lv->traces = lv->tbuf[lv->tcur];
        }
      }
      lv->traces_valid = true;
      CUDA_OK(cudaGetLastError());
      check_device_error(lv);
      return;
    }
    lv->traces_valid = false;  // the unfused paths leave the previous stage's traces
    if (lv->profiling) {
      float t_tr = 0.f, t_rhs = 0.f;
      for (int s = 0; s < nsteps; ++s)
        for (int stage = 0; stage < 5; ++stage) {
          CUDA_OK(cudaEventRecord(lv->ev[0], lv->stream));
          launch_traces(lv, lv->u, lv->traces);
          CUDA_OK(cudaEventRecord(lv->ev[1], lv->stream));
          launch_rhs(lv, true, false, stage);
          CUDA_OK(cudaEventRecord(lv->ev[2], lv->stream));
          CUDA_OK(cudaEventSynchronize(lv->ev[2]));
          float x, y;
          CUDA_OK(cudaEventElapsedTime(&x, lv->ev[0], lv->ev[1]));
          CUDA_OK(cudaEventElapsedTime(&y, lv->ev[1], lv->ev[2]));
          t_tr += x;
          t_rhs += y;
        }
      lv->prof[0] = t_tr;
      lv->prof[1] = t_rhs;
      lv->prof[2] = 10.0 * nsteps;
      CUDA_OK(cudaGetLastError());
      check_device_error(lv);
      return;
    }
    // one RK step (5 x [traces, rhs+update]) captured once as a CUDA graph
    if (!lv->graph || lv->graph_riemann != cfg->riemann || lv->graph_gamma != cfg->gamma) {
      if (lv->graph) {
        cudaGraphExecDestroy(lv->graph);
        lv->graph = nullptr;
      }
      cudaGraph_t g;
      const long long l0 = lv->launches;
      CUDA_OK(cudaStreamBeginCapture(lv->stream, cudaStreamCaptureModeThreadLocal));
      for (int stage = 0; stage < 5; ++stage) {
        launch_traces(lv, lv->u, lv->traces);
        launch_rhs(lv, true, false, stage);
      }
      lv->graph_launches = (int)(lv->launches - l0);
      lv->launches = l0;  // counted at replay
      CUDA_OK(cudaStreamEndCapture(lv->stream, &g));
      CUDA_OK(cudaGraphInstantiate(&lv->graph, g, 0));
      CUDA_OK(cudaGraphDestroy(g));
      lv->graph_riemann = cfg->riemann;
      lv->graph_gamma = cfg->gamma;
    }
    for (int s = 0; s < nsteps; ++s) {
      CUDA_OK(cudaGraphLaunch(lv->graph, lv->stream));
      lv->launches += lv->graph_launches;
    }
    CUDA_OK(cudaGetLastError());
    check_device_error(lv);
  });
}

int cdg_gpu_set_freestream(cdg_gpu_level* lv, const double* fs) {
  bool same = true;
  for (int c = 0; c < 5; ++c) same = same && lv->gas.fs[c] == fs[c];
  if (!same && lv->graph) {  // kernel params are baked into the captured graph
    cudaGraphExecDestroy(lv->graph);
    lv->graph = nullptr;
  }
  if (!same && lv->graph_visc) {
    cudaGraphExecDestroy(lv->graph_visc);
    lv->graph_visc = nullptr;
  }
  for (auto* gs : {lv->gft, lv->gns})
    for (int i = 0; i < 2; ++i)
      if (!same && gs[i]) {
        cudaGraphExecDestroy(gs[i]);
        gs[i] = nullptr;
      }
  for (int c = 0; c < 5; ++c) {
    lv->freestream[c] = fs[c];
    lv->gas.fs[c] = fs[c];
  }
  return CDG_GPU_OK;
}

int cdg_gpu_set_max_ctas(cdg_gpu_level* lv, int max_ctas) {
  if (max_ctas < 0) return CDG_GPU_ERR_CONFIG;
  lv->max_ctas = max_ctas;
  // grids are baked into the captured graphs
  drop_graphs_except_ns(lv);
  for (auto& ge : lv->gns)
    if (ge) cudaGraphExecDestroy(ge), ge = nullptr;
  return CDG_GPU_OK;
}

int cdg_gpu_set_kernel_path(cdg_gpu_level* lv, int path) {
  if (path != CDG_GPU_PATH_DEFAULT && path != CDG_GPU_PATH_GENERIC && path != CDG_GPU_PATH_TRACED)
    return CDG_GPU_ERR_CONFIG;
  const bool generic = path == CDG_GPU_PATH_GENERIC;
  lv->use_ns = path == CDG_GPU_PATH_DEFAULT && lv->d_ig != nullptr;
  lv->use_row = !generic && lv->ks->row_update[0] != nullptr && !wa_poorly_quantized(lv);
  lv->use_warp = !generic && lv->ks->warp_update[0] != nullptr;
  lv->use_rowc = !generic && lv->rfrag_opc != nullptr;
  lv->traces_valid = false;
  if (lv->d_tiles_int || lv->d_tiles_halo) build_phase_lists(lv);  // tile sizes may differ per family
  cdg_gpu_set_max_ctas(lv, lv->max_ctas);  // drops the captured graphs
  return CDG_GPU_OK;
}

int cdg_gpu_hllc_fallbacks(cdg_gpu_level* lv, long long* count) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    unsigned long long v = 0;
    CUDA_OK(cudaMemcpyAsync(&v, lv->d_fallbacks, sizeof v, cudaMemcpyDeviceToHost, lv->stream));
    CUDA_OK(cudaStreamSynchronize(lv->stream));
    *count = (long long)v;
  });
}

int cdg_gpu_set_profiling(cdg_gpu_level* lv, int enabled) {
  lv->profiling = enabled != 0;
  return CDG_GPU_OK;
}

int cdg_gpu_last_profile(cdg_gpu_level* lv, double* out3) {
  for (int i = 0; i < 3; ++i) out3[i] = lv->prof[i];
  return CDG_GPU_OK;
}

int cdg_gpu_viscosity(cdg_gpu_level* lv, double* eps_out) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    CUDA_OK(cudaMemcpyAsync(eps_out, lv->eps, lv->K * sizeof(double), cudaMemcpyDeviceToHost, lv->stream));
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_aux_gradient(cdg_gpu_level* lv, int m, double* q_out) {
  return guarded(nullptr, 0, [&] {
    if (!lv->q || !lv->last_viscous) throw Status(CDG_GPU_ERR_CONFIG, "no viscous RHS evaluated yet");
    if (m < 0 || m > 2) throw Status(CDG_GPU_ERR_CONFIG, "aux_gradient: direction must be 0..2");
    CUDA_OK(cudaSetDevice(lv->device));
    const size_t n = (size_t)lv->K * 5 * lv->bp;
    copy_rows(lv, q_out, lv->caller_block, lv->q + m * n, lv->bp, lv->np, lv->n_rows(),
              cudaMemcpyDeviceToHost);
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_timestep(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, int use_viscosity, double* dt_out,
                     char* err, size_t errlen) {
  NvtxRange nvtx_("cdg_gpu_timestep");
  return guarded(err, errlen, [&] {
    if (cfg->cfl <= 0.0) throw Status(CDG_GPU_ERR_CONFIG, "compute_timestep: CFL must be positive");
    if (!lv->h) throw Status(CDG_GPU_ERR_CONFIG, "compute_timestep: level created without h");
    CUDA_OK(cudaSetDevice(lv->device));
    CUDA_OK(cudaMemsetAsync(lv->d_scratch, 0xff, sizeof(double), lv->stream));
    TimestepParams tp{};
    tp.u = lv->u;
    tp.h = lv->h;
    tp.eps = use_viscosity ? lv->eps : nullptr;
    tp.K = lv->K;
    tp.np = lv->np;
    tp.bp = lv->bp;
    tp.gamma = cfg->gamma;
    tp.pfac = (lv->degree + 1.0) * (lv->degree + 1.0);
    tp.out = reinterpret_cast<unsigned long long*>(lv->d_scratch);
    tp.err = lv->d_err;
    k_timestep<<<(lv->K + 7) / 8, 256, 0, lv->stream>>>(tp);
    ++lv->launches;
    CUDA_OK(cudaGetLastError());
    check_device_error(lv);
    unsigned long long bits;
    CUDA_OK(cudaMemcpy(&bits, lv->d_scratch, sizeof bits, cudaMemcpyDeviceToHost));
    double m;
    std::memcpy(&m, &bits, sizeof m);
    *dt_out = cfg->cfl * m;
  });
}

int cdg_gpu_snapshot(cdg_gpu_level* lv) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    const size_t n = (size_t)lv->K * 5 * lv->bp;
    if (!lv->before) CUDA_OK(cudaMalloc(&lv->before, n * sizeof(double)));
    CUDA_OK(cudaMemcpyAsync(lv->before, lv->u, n * sizeof(double), cudaMemcpyDeviceToDevice, lv->stream));
  });
}

int cdg_gpu_residual(cdg_gpu_level* lv, int kind, double dt, double* out) {
  NvtxRange nvtx_("cdg_gpu_residual");
  return guarded(nullptr, 0, [&] {
    if (!lv->before) throw Status(CDG_GPU_ERR_CONFIG, "residual: no snapshot taken");
    CUDA_OK(cudaSetDevice(lv->device));
    const size_t n = (size_t)lv->K * 5 * lv->bp;
    const int blocks = 592;
    k_residual<<<blocks, 256, 0, lv->stream>>>(lv->u, lv->before, n, kind, lv->d_scratch);
    ++lv->launches;
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(lv->h_scratch.data(), lv->d_scratch, blocks * sizeof(double),
                            cudaMemcpyDeviceToHost, lv->stream));
    CUDA_OK(cudaStreamSynchronize(lv->stream));
    double acc = 0.0;
    for (int i = 0; i < blocks; ++i)
      acc = kind == 1 ? acc + lv->h_scratch[i] : std::max(acc, lv->h_scratch[i]);
    *out = (kind == 1 ? std::sqrt(acc) : acc) / dt;
  });
}

// ---- device-resident run_steady -----------------------------------------------
int cdg_gpu_fill_freestream(cdg_gpu_level* lv) {
  lv->traces_valid = false;
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    const size_t rows = (size_t)lv->K * 5, n = rows * lv->bp;
    k_fill_freestream<<<(unsigned)((n + 255) / 256), 256, 0, lv->stream>>>(lv->u, lv->gas, rows, lv->np, lv->bp);
    ++lv->launches;
    CUDA_OK(cudaMemsetAsync(lv->res, 0, n * sizeof(double), lv->stream));
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaStreamSynchronize(lv->stream));
  });
}

int cdg_gpu_p_refine_embed(cdg_gpu_level* to, const cdg_gpu_level* from, const double* embed) {
  to->traces_valid = false;
  return guarded(nullptr, 0, [&] {
    if (to->K != from->K || to->device != from->device)
      throw Status(CDG_GPU_ERR_CONFIG, "p_refine_embed: levels differ in element count or device");
    if (to->degree < from->degree) throw Status(CDG_GPU_ERR_CONFIG, "p_refine_embed: target degree must not decrease");
    CUDA_OK(cudaSetDevice(to->device));
    // the source state must be complete before the target stream reads it
    CUDA_OK(cudaStreamSynchronize(from->stream));
    double* dE = dev_upload(std::vector<double>(embed, embed + (size_t)to->np * from->np));
    const int rows = to->K * 5;
    k_embed<<<(rows + 7) / 8, 256, 0, to->stream>>>(from->u, to->u, dE, rows, from->np, from->bp, to->np, to->bp);
    ++to->launches;
    CUDA_OK(cudaMemsetAsync(to->res, 0, (size_t)rows * to->bp * sizeof(double), to->stream));
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaStreamSynchronize(to->stream));
    cudaFree(dE);
  });
}

int cdg_gpu_run_level(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, const cdg_gpu_steady_params* sp,
                      double* rows, int max_rows, int* n_rows, int* converged, char* err, size_t errlen) {
  return cdg_gpu_run_level_live(lv, cfg, sp, nullptr, nullptr, rows, max_rows, n_rows, converged, err, errlen);
}

int cdg_gpu_run_level_live(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, const cdg_gpu_steady_params* sp,
                           cdg_gpu_row_fn on_row, void* user, double* rows, int max_rows, int* n_rows,
                           int* converged, char* err, size_t errlen) {
  auto ok = [&](int st) {
    if (st != CDG_GPU_OK) throw Status(st, err && errlen ? std::string(err) : std::string("run_level failed"));
  };
  SteadyOps ops;
  ops.rk_steps = [&](int n, double dt, const double* A, const double* B) {
    ok(cdg_gpu_rk_steps(lv, cfg, n, dt, A, B, err, errlen));
  };
  ops.snapshot = [&] { ok(cdg_gpu_snapshot(lv)); };
  ops.residual = [&](int kind, double dt) {
    double r = 0.0;
    ok(cdg_gpu_residual(lv, kind, dt, &r));
    return r;
  };
  ops.timestep = [&](int use_visc) {
    double dt = 0.0;
    ok(cdg_gpu_timestep(lv, cfg, use_visc, &dt, err, errlen));
    return dt;
  };
  return run_level_loop(ops, cfg, sp, on_row, user, rows, max_rows, n_rows, converged, err, errlen);
}

// ---- multi-GPU halo plumbing -------------------------------------------------
}  // extern "C"

namespace {

void drop_halo(cdg_gpu_level* lv) {
  for (double*& p : {std::ref(lv->hsend[0]), std::ref(lv->hsend[1]), std::ref(lv->hrecv)})
    if (p) cudaFree(p), p = nullptr;
  lv->peers.clear();
  lv->halo_defined = false;
}

// upload a (possibly empty) index list; never null, so an empty list stays a list
int* upload_list(const std::vector<int>& v) {
  return dev_upload(v.empty() ? std::vector<int>{0} : v);
}

void set_halo_lists(cdg_gpu_level* lv, int n_send, const int* send_ef, int n_recv, const int* recv_ef) {
  for (int i = 0; i < n_send; ++i)
    if ((send_ef[i] >> 2) < 0 || (send_ef[i] >> 2) >= lv->K)
      throw Status(CDG_GPU_ERR_CONFIG, "halo: send rows must be owned elements");
  for (int i = 0; i < n_recv; ++i)
    if ((recv_ef[i] >> 2) < lv->K || (recv_ef[i] >> 2) >= lv->K + lv->n_halo)
      throw Status(CDG_GPU_ERR_CONFIG, "halo_setup: receive rows must be ghost elements");
  lv->n_send = n_send;
  lv->n_recv = n_recv;
  if (lv->d_send_idx) cudaFree(lv->d_send_idx);
  if (lv->d_recv_idx) cudaFree(lv->d_recv_idx);
  lv->d_send_idx = upload_list(std::vector<int>(send_ef, send_ef + n_send));
  lv->d_recv_idx = upload_list(std::vector<int>(recv_ef, recv_ef + n_recv));
}

// what: 0 U traces, 1 U traces + sqrt(eps) of the element, 2 the three q_m traces
int halo_width(const cdg_gpu_level* lv, int what) { return what == 2 ? 5 * lv->ng : 5 * lv->ng + (what == 1); }

// pack (dir 0: owned faces -> buf) / unpack (dir 1: buf -> ghost faces)
void halo_move(cdg_gpu_level* lv, int dir, int what, double* buf) {
  const int n = dir == 0 ? lv->n_send : lv->n_recv;
  if (!n) return;
  HaloXfer x{};
  if (what == 2) {  // the normal component of q's traces (one plane)
    x.nplanes = 1;
    x.plane[0] = lv->qtr;
  } else {
    x.nplanes = 1;
    x.plane[0] = lv->traces;
    x.eps = what == 1 ? lv->sqrt_eps : nullptr;
  }
  x.buf = buf;
  x.idx = dir == 0 ? lv->d_send_idx : lv->d_recv_idx;
  x.n = n;
  x.ng = lv->ng;
  x.tb = lv->tb;
  x.W = halo_width(lv, what);
  x.dir = dir;
  k_halo_xfer<<<(n + 7) / 8, 256, 0, lv->stream>>>(x);
  ++lv->launches;
}

void upload_coef(cdg_gpu_level* lv, double dt, const double* a, const double* b) {
  lv->h_coef->dt = dt;
  for (int i = 0; i < 5; ++i) {
    lv->h_coef->a[i] = a[i];
    lv->h_coef->b[i] = b[i];
  }
  CUDA_OK(cudaMemcpyAsync(lv->d_coef, lv->h_coef, sizeof(StageCoef), cudaMemcpyHostToDevice, lv->stream));
}

// One inviscid RK stage in split form (no host synchronisation):
//  0: (stage 0: RK coefficients) traces of u (seeded, or already written by
//     the previous fused stage) + pack the halo rows;
//  1: unpack + RHS/update of every tile;
//  2: RHS/update of the interior tiles (overlaps the exchange);
//  3: unpack + RHS/update of the halo tiles.
void stage_phase(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, int stage, int phase, double dt,
                 const double* a, const double* b) {
  if (cfg->riemann != 0 && cfg->riemann != 1) throw Status(CDG_GPU_ERR_CONFIG, "unknown Riemann solver (llf|hllc)");
  lv->gas.gamma = cfg->gamma;
  lv->gas.riemann = cfg->riemann;
  const bool ft = fused_traces(lv);
  if (ft) ensure_tbuf(lv);
  // fused traces: the RHS of stage s writes the traces of stage s+1 into the
  // other buffer (owned rows); the ghost rows arrive by the halo exchange
  auto rhs = [&](const int* tiles, int n_list, const int* ctiles, int n_clist) {
    lv->cur_tiles = tiles;
    lv->cur_n_list = n_list;
    lv->cur_ctiles = ctiles;
    lv->cur_n_clist = n_clist;
    if (ft) lv->cur_traces_out = lv->tbuf[lv->tcur ^ 1];
    auto reset = [&] {
      lv->cur_tiles = nullptr;
      lv->cur_n_list = 0;
      lv->cur_ctiles = nullptr;
      lv->cur_n_clist = 0;
      lv->cur_traces_out = nullptr;
    };
    try {
      launch_rhs(lv, true, false, stage);
    } catch (...) {
      reset();
      throw;
    }
    reset();
  };
  auto swap = [&] {
    if (ft) {
      lv->tcur ^= 1;
      lv->traces = lv->tbuf[lv->tcur];
      lv->traces_valid = true;
    } else {
      lv->traces_valid = false;
    }
  };
  if (phase == 0) {
    if (stage == 0) upload_coef(lv, dt, a, b);
    if (ft)
      seed_traces(lv);
    else
      launch_traces(lv, lv->u, lv->traces);
    halo_move(lv, 0, 0, lv->send_buf);
  } else if (phase == 1) {
    halo_move(lv, 1, 0, lv->recv_buf);
    rhs(nullptr, 0, nullptr, 0);
    swap();
  } else if (phase == 2 || phase == 3) {
    if (!lv->d_tiles_int) throw Status(CDG_GPU_ERR_CONFIG, "phases 2/3 need halo_setup");
    if (phase == 3) halo_move(lv, 1, 0, lv->recv_buf);
    if (phase == 2)
      rhs(lv->d_tiles_int, lv->n_tiles_int, lv->d_ctiles_int, lv->n_ctiles_int);
    else
      rhs(lv->d_tiles_halo, lv->n_tiles_halo, lv->d_ctiles_halo, lv->n_ctiles_halo);
    if (phase == 3) swap();
  } else {
    throw Status(CDG_GPU_ERR_CONFIG, "rk_stage_phase: phase must be 0..3");
  }
}

}  // namespace

extern "C" {

int cdg_gpu_halo_setup(cdg_gpu_level* lv, int n_send, const int* send_ef, int n_recv, const int* recv_ef,
                       double* send_buf, double* recv_buf) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    if ((n_send && !send_buf) || (n_recv && !recv_buf))
      throw Status(CDG_GPU_ERR_CONFIG, "halo_setup: device buffers required");
    set_halo_lists(lv, n_send, send_ef, n_recv, recv_ef);
    lv->send_buf = send_buf;  // caller-owned (e.g. NCCL-registered torch tensors)
    lv->recv_buf = recv_buf;
    // interior tiles (no element with a ghost neighbour) run while the halo
    // traces are in flight; halo tiles after they land (rk_stage_phase 2 / 3)
    build_phase_lists(lv);
  });
}

int cdg_gpu_halo_pack(cdg_gpu_level* lv) {
  return guarded(nullptr, 0, [&] {
    halo_move(lv, 0, 0, lv->send_buf);
    CUDA_OK(cudaGetLastError());
  });
}

int cdg_gpu_halo_unpack(cdg_gpu_level* lv) {
  return guarded(nullptr, 0, [&] {
    halo_move(lv, 1, 0, lv->recv_buf);
    CUDA_OK(cudaGetLastError());
  });
}

int cdg_gpu_rk_stage_phase(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, int stage, int phase, double dt,
                           const double a[5], const double b[5], char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    if (cfg->visc_enabled)
      throw Status(CDG_GPU_ERR_CONFIG,
                   "split-phase stages support the inviscid path only (viscous multi-rank steps: cdg_gpu_comm_rk_steps)");
    stage_phase(lv, cfg, stage, phase, dt, a, b);
    if (stage == 4 && (phase == 1 || phase == 3)) check_device_error(lv);
    CUDA_OK(cudaGetLastError());
  });
}

}  // extern "C"

#include "cdg_comm.cuh"
