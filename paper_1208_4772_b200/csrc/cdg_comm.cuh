// cdg_comm.cuh -- the multi-rank driver of the C ABI (include/cdg_gpu.h,
// "multi-rank driver"): one shard (cdg_gpu_level with ghost elements) per
// rank, a halo exchange of face traces at every RK stage, and the two global
// reductions of run_steady (time step MIN, residual MAX / SUM).
//
// Reference: the single-process loop it distributes -- rk_step
// (solver.cpp:469-492), compute_rhs with its barrier-separated viscous phases
// (sensor -> aux gradient -> RHS, solver.cpp:239-321,349-354,438-453),
// compute_timestep (:494-526), residual_norm (:572-590), run_steady (:594-676).
//
// Two transports, one stage sequence:
//  * NCCL (one process per GPU): ncclSend/ncclRecv of the packed halo rows on
//    a comm stream, ncclAllReduce for the viscous gate / dt / residual.
//    libnccl.so.2 is resolved at run time (dlopen), so the library loads on a
//    machine without NCCL and binds to the NCCL a host framework already
//    loaded (torch's) when there is one.
//  * in-process (one host thread drives every shard; shards on one GPU or on
//    several, peer copies over NVLink): each shard PULLS its ghost rows from
//    its peers' send buffers with cudaMemcpyPeerAsync on its comm stream once
//    every shard's pack is done (all-to-all event waits). Send buffers are
//    double-buffered by exchange parity, so a shard never overwrites rows a
//    slower peer has not pulled yet (its next-but-one pack is ordered after
//    that peer's next exchange point, which follows the pull on the peer's
//    stream).
// Inviscid stage: pack the U traces -> exchange || RHS+update of the interior
// tiles -> (wait) unpack + RHS+update of the halo tiles. Viscous stage (the
// reference's three phases): sensor + U traces -> pack U traces and sqrt(eps)
// -> exchange + all-rank max eps (the gate of every viscous kernel, so every
// rank takes the same branch of viscous_active, solver.cpp:257-259) -> unpack,
// aux gradient q_m of the owned elements and their traces -> exchange of the
// q traces -> unpack, gated viscous / inviscid RHS+update. Per-element
// arithmetic never depends on the partition: R-rank states are bitwise equal
// to the single-level run (tests/test_gpu_comm.py).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.h, name)); };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.init_rank, "ncclCommInitRank");
    sym(a.destroy, "ncclCommDestroy");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.error_string, "ncclGetErrorString");
    if (!a.get_unique_id || !a.init_rank || !a.send || !a.recv || !a.all_reduce) a.h = nullptr;
    return a;
  }();
  if (!api.h) throw Status(CDG_GPU_ERR_CONFIG, "multi-rank driver: NCCL (libnccl.so.2) not found");
  return api;
}

#define NCCL_OK(x)                                                                                  \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess)                                                                          \
      throw Status(CDG_GPU_ERR_CUDA, std::string("NCCL error: ") + nccl().error_string(r_) + " at " #x); \
  } while (0)

using PeerSeg = cdg_gpu_level::Peer;

// an in-process pull: rows [dst_off, +n) of shard r's receive buffer come from
// rows [src_off, +n) of shard `src`'s send buffer
struct Pull {
  int src, dst_off, src_off, n;
};

}  // namespace

struct cdg_gpu_comm {
  bool use_nccl = false;
  int rank = 0, nranks = 1;
  std::vector<cdg_gpu_level*> lv;        // in-process: shard r = lv[r]; NCCL: lv[0] is this rank
  ncclComm_t nc = nullptr;
  std::vector<cudaStream_t> cs;          // per shard: transfer stream
  std::vector<cudaEvent_t> ev_pre, ev_post;
  std::vector<unsigned long long*> gate;             // per shard: all-rank max eps (viscous gate)
  std::vector<const unsigned long long**> gate_src;  // in-process: per shard, device array of every shard's d_maxeps
  std::vector<std::vector<Pull>> pulls;  // in-process: per shard
  double* d_red = nullptr;               // NCCL: reduction scratch (2 doubles) on this rank's device
  int parity = 0;                        // send-buffer half of the next exchange
  long long exchanges = 0;
};

namespace {

const cdg_gpu_level& halo_of(const cdg_gpu_level* lv) {
  if (!lv->halo_defined) throw Status(CDG_GPU_ERR_CONFIG, "multi-rank driver: shard has no cdg_gpu_halo_define");
  return *lv;
}

// Exchange the rows every shard just packed into send[parity] (width W =
// halo_width(what)); what == 1 also reduces the shards' max eps into their gate.
void comm_exchange(cdg_gpu_comm* c, int what) {
  NvtxRange nvtx_(what == 2 ? "halo exchange (q traces)" : what == 1 ? "halo exchange (traces + sqrt eps)" : "halo exchange (traces)");
  const int n = (int)c->lv.size();
  for (int r = 0; r < n; ++r) {
    CUDA_OK(cudaSetDevice(c->lv[r]->device));
    CUDA_OK(cudaEventRecord(c->ev_pre[r], c->lv[r]->stream));
  }
  if (c->use_nccl) {
    cdg_gpu_level* lv = c->lv[0];
    const cdg_gpu_level& H = halo_of(lv);
    const int W = halo_width(lv, what);
    CUDA_OK(cudaStreamWaitEvent(c->cs[0], c->ev_pre[0], 0));
    const NcclApi& N = nccl();
    if (what == 1)
      NCCL_OK(N.all_reduce(lv->d_maxeps, c->gate[0], 1, ncclUint64, ncclMax, c->nc, c->cs[0]));
    NCCL_OK(N.group_start());
    for (const PeerSeg& s : H.peers) {
      if (s.send_n) NCCL_OK(N.send(H.hsend[c->parity] + (size_t)s.send_off * W, (size_t)s.send_n * W, ncclFloat64, s.rank, c->nc, c->cs[0]));
      if (s.recv_n) NCCL_OK(N.recv(H.hrecv + (size_t)s.recv_off * W, (size_t)s.recv_n * W, ncclFloat64, s.rank, c->nc, c->cs[0]));
    }
    NCCL_OK(N.group_end());
    CUDA_OK(cudaEventRecord(c->ev_post[0], c->cs[0]));
  } else {
    for (int r = 0; r < n; ++r) {
      cdg_gpu_level* lv = c->lv[r];
      CUDA_OK(cudaSetDevice(lv->device));
      for (int j = 0; j < n; ++j) CUDA_OK(cudaStreamWaitEvent(c->cs[r], c->ev_pre[j], 0));
      const int W = halo_width(lv, what);
      const cdg_gpu_level& H = halo_of(lv);
      for (const Pull& p : c->pulls[r]) {
        const cdg_gpu_level* src = c->lv[p.src];
        CUDA_OK(cudaMemcpyPeerAsync(H.hrecv + (size_t)p.dst_off * W, lv->device,
                                    halo_of(src).hsend[c->parity] + (size_t)p.src_off * W, src->device,
                                    (size_t)p.n * W * sizeof(double), c->cs[r]));
      }
      if (what == 1) k_gate_max<<<1, 32, 0, c->cs[r]>>>(c->gate_src[r], n, c->gate[r]);
      CUDA_OK(cudaEventRecord(c->ev_post[r], c->cs[r]));
    }
  }
  c->parity ^= 1;
  ++c->exchanges;
}

void comm_wait(cdg_gpu_comm* c, int r) {
  CUDA_OK(cudaSetDevice(c->lv[r]->device));
  CUDA_OK(cudaStreamWaitEvent(c->lv[r]->stream, c->ev_post[r], 0));
}

void comm_point_send(cdg_gpu_comm* c, cdg_gpu_level* lv) {
  halo_of(lv);
  lv->send_buf = lv->hsend[c->parity];
  lv->recv_buf = lv->hrecv;
}

// all-rank agreement on a recorded device error (NCCL: a rank that stops
// alone would leave its peers waiting in the next exchange)
void comm_check_errors(cdg_gpu_comm* c) {
  if (c->use_nccl) {
    cdg_gpu_level* lv = c->lv[0];
    CUDA_OK(cudaSetDevice(lv->device));
    CUDA_OK(cudaStreamWaitEvent(c->cs[0], c->ev_post[0], 0));
    CUDA_OK(cudaEventRecord(c->ev_pre[0], lv->stream));
    CUDA_OK(cudaStreamWaitEvent(c->cs[0], c->ev_pre[0], 0));
    int* flag = reinterpret_cast<int*>(c->d_red);
    NCCL_OK(nccl().all_reduce(&lv->d_err->flag, flag, 1, ncclInt32, ncclMax, c->nc, c->cs[0]));
    int h = 0;
    CUDA_OK(cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, c->cs[0]));
    CUDA_OK(cudaStreamSynchronize(c->cs[0]));
    check_device_error(lv);  // this rank's own record (reference message) first
    if (h) throw Status(CDG_GPU_ERR_NUMERICS, "inadmissible state on another rank");
    return;
  }
  for (cdg_gpu_level* lv : c->lv) {
    CUDA_OK(cudaSetDevice(lv->device));
    check_device_error(lv);
  }
}

void comm_rk_steps(cdg_gpu_comm* c, const cdg_gpu_run_config* cfg, int nsteps, double dt, const double* a,
                   const double* b) {
  if (cfg->riemann != 0 && cfg->riemann != 1) throw Status(CDG_GPU_ERR_CONFIG, "unknown Riemann solver (llf|hllc)");
  NvtxRange nvtx_("cdg_gpu_comm_rk_steps");
  const int n = (int)c->lv.size();
  auto each = [&](auto&& fn) {
    for (int r = 0; r < n; ++r) {
      CUDA_OK(cudaSetDevice(c->lv[r]->device));
      fn(r, c->lv[r]);
    }
  };
  for (int s = 0; s < nsteps; ++s)
    for (int stage = 0; stage < 5; ++stage) {
      if (!cfg->visc_enabled) {
        each([&](int, cdg_gpu_level* lv) {
          comm_point_send(c, lv);
          stage_phase(lv, cfg, stage, 0, dt, a, b);
        });
        comm_exchange(c, 0);
        each([&](int, cdg_gpu_level* lv) { stage_phase(lv, cfg, stage, 2, dt, a, b); });
        each([&](int r, cdg_gpu_level* lv) {
          comm_wait(c, r);
          stage_phase(lv, cfg, stage, 3, dt, a, b);
        });
        continue;
      }
      // viscous stage: the reference's barrier-separated phases, one exchange each
      each([&](int r, cdg_gpu_level* lv) {
        ensure_viscous_buffers(lv, cfg);
        lv->gas.gamma = cfg->gamma;
        lv->gas.riemann = cfg->riemann;
        lv->gate_buf = c->gate[r];
        lv->traces_valid = false;
        if (stage == 0) upload_coef(lv, dt, a, b);
        comm_point_send(c, lv);
        launch_sensor(lv, cfg);
        launch_traces(lv, lv->u, lv->traces);
        halo_move(lv, 0, 1, lv->send_buf);
      });
      comm_exchange(c, 1);
      each([&](int r, cdg_gpu_level* lv) {
        comm_wait(c, r);
        halo_move(lv, 1, 1, lv->recv_buf);
        lv->cur_gate = c->gate[r];
        lv->cur_gate_when = 1;
        launch_aux(lv);
        lv->cur_gate = nullptr;
        comm_point_send(c, lv);
        halo_move(lv, 0, 2, lv->send_buf);
      });
      comm_exchange(c, 2);
      each([&](int r, cdg_gpu_level* lv) {
        comm_wait(c, r);
        halo_move(lv, 1, 2, lv->recv_buf);
        lv->cur_gate = c->gate[r];
        lv->cur_gate_when = 1;
        launch_rhs(lv, true, true, stage);
        lv->cur_gate_when = 0;
        launch_rhs(lv, true, false, stage);
        lv->cur_gate = nullptr;
      });
    }
  each([&](int, cdg_gpu_level*) { CUDA_OK(cudaGetLastError()); });
  comm_check_errors(c);
  if (cfg->visc_enabled)
    for (int r = 0; r < n; ++r) {  // viscous_active of the last stage (aux_gradient validity)
      unsigned long long bits = 0;
      CUDA_OK(cudaSetDevice(c->lv[r]->device));
      CUDA_OK(cudaMemcpy(&bits, c->gate[r], sizeof bits, cudaMemcpyDeviceToHost));
      c->lv[r]->last_viscous = bits != 0;
    }
}

// global reduction of one double per shard: op 0 MIN, 1 MAX, 2 SUM
double comm_reduce(cdg_gpu_comm* c, const std::vector<double>& local, int op) {
  double v = local[0];
  for (size_t i = 1; i < local.size(); ++i)
    v = op == 0 ? std::min(v, local[i]) : op == 1 ? std::max(v, local[i]) : v + local[i];
  if (!c->use_nccl) return v;
  cdg_gpu_level* lv = c->lv[0];
  CUDA_OK(cudaSetDevice(lv->device));
  CUDA_OK(cudaMemcpyAsync(c->d_red, &v, sizeof v, cudaMemcpyHostToDevice, c->cs[0]));
  NCCL_OK(nccl().all_reduce(c->d_red, c->d_red + 1, 1, ncclFloat64, op == 0 ? ncclMin : op == 1 ? ncclMax : ncclSum,
                            c->nc, c->cs[0]));
  CUDA_OK(cudaMemcpyAsync(&v, c->d_red + 1, sizeof v, cudaMemcpyDeviceToHost, c->cs[0]));
  CUDA_OK(cudaStreamSynchronize(c->cs[0]));
  return v;
}

double level_timestep(cdg_gpu_level* lv, const cdg_gpu_run_config* cfg, int use_visc) {
  double dt = 0.0;
  char err[256] = {0};
  const int st = cdg_gpu_timestep(lv, cfg, use_visc, &dt, err, sizeof err);
  if (st != CDG_GPU_OK) throw Status(st, err);
  return dt;
}

// residual_norm partials of one shard: inf -> max |du|, l2 -> sum du^2 (no sqrt, no /dt)
double level_residual_raw(cdg_gpu_level* lv, int kind) {
  if (!lv->before) throw Status(CDG_GPU_ERR_CONFIG, "residual: no snapshot taken");
  CUDA_OK(cudaSetDevice(lv->device));
  const size_t n = (size_t)lv->K * 5 * lv->bp;
  const int blocks = 592;
  k_residual<<<blocks, 256, 0, lv->stream>>>(lv->u, lv->before, n, kind, lv->d_scratch);
  ++lv->launches;
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpyAsync(lv->h_scratch.data(), lv->d_scratch, blocks * sizeof(double), cudaMemcpyDeviceToHost,
                          lv->stream));
  CUDA_OK(cudaStreamSynchronize(lv->stream));
  double acc = 0.0;
  for (int i = 0; i < blocks; ++i) acc = kind == 1 ? acc + lv->h_scratch[i] : std::max(acc, lv->h_scratch[i]);
  return acc;
}

void comm_destroy(cdg_gpu_comm* c) {
  if (!c) return;
  for (size_t r = 0; r < c->lv.size(); ++r) {
    cudaSetDevice(c->lv[r]->device);
    if (r < c->cs.size() && c->cs[r]) cudaStreamSynchronize(c->cs[r]), cudaStreamDestroy(c->cs[r]);
    if (r < c->ev_pre.size() && c->ev_pre[r]) cudaEventDestroy(c->ev_pre[r]);
    if (r < c->ev_post.size() && c->ev_post[r]) cudaEventDestroy(c->ev_post[r]);
    if (r < c->gate.size() && c->gate[r]) cudaFree(c->gate[r]);
    if (r < c->gate_src.size() && c->gate_src[r]) cudaFree(c->gate_src[r]);
    c->lv[r]->gate_buf = nullptr;
  }
  if (c->d_red) cudaFree(c->d_red);
  if (c->nc && nccl().destroy) nccl().destroy(c->nc);
  delete c;
}

void comm_alloc_streams(cdg_gpu_comm* c) {
  const size_t n = c->lv.size();
  c->cs.assign(n, nullptr);
  c->ev_pre.assign(n, nullptr);
  c->ev_post.assign(n, nullptr);
  c->gate.assign(n, nullptr);
  for (size_t r = 0; r < n; ++r) {
    CUDA_OK(cudaSetDevice(c->lv[r]->device));
    CUDA_OK(cudaStreamCreateWithFlags(&c->cs[r], cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_pre[r], cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_post[r], cudaEventDisableTiming));
    CUDA_OK(cudaMalloc(&c->gate[r], sizeof(unsigned long long)));
    CUDA_OK(cudaMemset(c->gate[r], 0, sizeof(unsigned long long)));
  }
}

}  // namespace

extern "C" {

int cdg_gpu_halo_define(cdg_gpu_level* lv, int n_peers, const int* peer_rank, const int* send_count,
                        const int* recv_count, const int* send_elem_face, const int* recv_elem_face) {
  return guarded(nullptr, 0, [&] {
    CUDA_OK(cudaSetDevice(lv->device));
    drop_halo(lv);
    int ns = 0, nr = 0;
    for (int i = 0; i < n_peers; ++i) {
      if (send_count[i] < 0 || recv_count[i] < 0) throw Status(CDG_GPU_ERR_CONFIG, "halo_define: negative count");
      lv->peers.push_back(PeerSeg{peer_rank[i], ns, send_count[i], nr, recv_count[i]});
      ns += send_count[i];
      nr += recv_count[i];
    }
    set_halo_lists(lv, ns, send_elem_face, nr, recv_elem_face);
    const int W = halo_width(lv, 2) > halo_width(lv, 1) ? halo_width(lv, 2) : halo_width(lv, 1);
    for (double*& p : lv->hsend) CUDA_OK(cudaMalloc(&p, ((size_t)ns * W + 1) * sizeof(double)));
    CUDA_OK(cudaMalloc(&lv->hrecv, ((size_t)nr * W + 1) * sizeof(double)));
    lv->send_buf = lv->hsend[0];
    lv->recv_buf = lv->hrecv;
    lv->halo_defined = true;
    build_phase_lists(lv);
  });
}

int cdg_gpu_comm_unique_id(unsigned char id[128], char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    NCCL_OK(nccl().get_unique_id(&u));
    std::memcpy(id, &u, 128);
  });
}

int cdg_gpu_comm_create_nccl(cdg_gpu_level* lv, const unsigned char id[128], int rank, int nranks,
                             cdg_gpu_comm** out, char* err, size_t errlen) {
  *out = nullptr;
  auto* c = new cdg_gpu_comm;
  const int st = guarded(err, errlen, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Status(CDG_GPU_ERR_CONFIG, "comm: bad rank / nranks");
    halo_of(lv);
    c->use_nccl = true;
    c->rank = rank;
    c->nranks = nranks;
    c->lv = {lv};
    comm_alloc_streams(c);
    CUDA_OK(cudaSetDevice(lv->device));
    CUDA_OK(cudaMalloc(&c->d_red, 2 * sizeof(double)));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    NCCL_OK(nccl().init_rank(&c->nc, nranks, u, rank));
    lv->gate_buf = c->gate[0];
  });
  if (st != CDG_GPU_OK) {
    comm_destroy(c);
    return st;
  }
  *out = c;
  return CDG_GPU_OK;
}

int cdg_gpu_comm_create_local(int nranks, cdg_gpu_level* const* levels, cdg_gpu_comm** out, char* err,
                              size_t errlen) {
  *out = nullptr;
  auto* c = new cdg_gpu_comm;
  const int st = guarded(err, errlen, [&] {
    if (nranks < 1) throw Status(CDG_GPU_ERR_CONFIG, "comm: nranks must be >= 1");
    c->nranks = nranks;
    c->lv.assign(levels, levels + nranks);
    for (cdg_gpu_level* lv : c->lv) halo_of(lv);
    comm_alloc_streams(c);
    // peer access for shards on different GPUs (NVLink loads/copies)
    for (int i = 0; i < nranks; ++i)
      for (int j = 0; j < nranks; ++j) {
        const int di = c->lv[i]->device, dj = c->lv[j]->device;
        if (di == dj) continue;
        int ok = 0;
        CUDA_OK(cudaDeviceCanAccessPeer(&ok, di, dj));
        if (!ok) throw Status(CDG_GPU_ERR_CONFIG, "comm: no peer access between devices");
        CUDA_OK(cudaSetDevice(di));
        const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_OK(e);
        cudaGetLastError();
      }
    // pull lists: shard r's receive segment from peer j is j's send segment towards r
    c->pulls.assign(nranks, {});
    for (int r = 0; r < nranks; ++r)
      for (const PeerSeg& s : halo_of(c->lv[r]).peers) {
        if (s.rank < 0 || s.rank >= nranks || s.rank == r) throw Status(CDG_GPU_ERR_CONFIG, "comm: bad peer rank");
        const PeerSeg* back = nullptr;
        for (const PeerSeg& t : halo_of(c->lv[s.rank]).peers)
          if (t.rank == r) back = &t;
        if (!back || back->send_n != s.recv_n)
          throw Status(CDG_GPU_ERR_CONFIG, "comm: halo lists of ranks " + std::to_string(r) + " and " +
                                               std::to_string(s.rank) + " do not match");
        if (s.recv_n) c->pulls[r].push_back(Pull{s.rank, s.recv_off, back->send_off, s.recv_n});
      }
    c->gate_src.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
      std::vector<const unsigned long long*> src;
      for (cdg_gpu_level* lv : c->lv) src.push_back(lv->d_maxeps);
      CUDA_OK(cudaSetDevice(c->lv[r]->device));
      c->gate_src[r] = dev_upload(src);
      c->lv[r]->gate_buf = c->gate[r];
    }
  });
  if (st != CDG_GPU_OK) {
    comm_destroy(c);
    return st;
  }
  *out = c;
  return CDG_GPU_OK;
}

void cdg_gpu_comm_destroy(cdg_gpu_comm* c) { comm_destroy(c); }

int cdg_gpu_comm_rk_steps(cdg_gpu_comm* c, const cdg_gpu_run_config* cfg, int nsteps, double dt, const double a[5],
                          const double b[5], char* err, size_t errlen) {
  return guarded(err, errlen, [&] { comm_rk_steps(c, cfg, nsteps, dt, a, b); });
}

int cdg_gpu_comm_timestep(cdg_gpu_comm* c, const cdg_gpu_run_config* cfg, int use_viscosity, double* dt_out,
                          char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    std::vector<double> v;
    for (cdg_gpu_level* lv : c->lv) v.push_back(level_timestep(lv, cfg, use_viscosity));
    *dt_out = comm_reduce(c, v, 0);
  });
}

int cdg_gpu_comm_snapshot(cdg_gpu_comm* c) {
  return guarded(nullptr, 0, [&] {
    for (cdg_gpu_level* lv : c->lv) {
      const int st = cdg_gpu_snapshot(lv);
      if (st != CDG_GPU_OK) throw Status(st, "snapshot failed");
    }
  });
}

int cdg_gpu_comm_residual(cdg_gpu_comm* c, int kind, double dt, double* out) {
  return guarded(nullptr, 0, [&] {
    std::vector<double> v;
    for (cdg_gpu_level* lv : c->lv) v.push_back(level_residual_raw(lv, kind));
    const double g = comm_reduce(c, v, kind == 1 ? 2 : 1);
    *out = (kind == 1 ? std::sqrt(g) : g) / dt;
  });
}

int cdg_gpu_comm_fill_freestream(cdg_gpu_comm* c) {
  return guarded(nullptr, 0, [&] {
    for (cdg_gpu_level* lv : c->lv) {
      const int st = cdg_gpu_fill_freestream(lv);
      if (st != CDG_GPU_OK) throw Status(st, "fill_freestream failed");
    }
  });
}

int cdg_gpu_comm_run_level(cdg_gpu_comm* c, const cdg_gpu_run_config* cfg, const cdg_gpu_steady_params* sp,
                           cdg_gpu_row_fn on_row, void* user, double* rows, int max_rows, int* n_rows, int* converged,
                           char* err, size_t errlen) {
  SteadyOps ops;
  ops.rk_steps = [&](int n, double dt, const double* A, const double* B) { comm_rk_steps(c, cfg, n, dt, A, B); };
  ops.snapshot = [&] {
    const int st = cdg_gpu_comm_snapshot(c);
    if (st != CDG_GPU_OK) throw Status(st, "snapshot failed");
  };
  ops.residual = [&](int kind, double dt) {
    double r = 0.0;
    const int st = cdg_gpu_comm_residual(c, kind, dt, &r);
    if (st != CDG_GPU_OK) throw Status(st, "residual failed");
    return r;
  };
  ops.timestep = [&](int use_visc) {
    std::vector<double> v;
    for (cdg_gpu_level* lv : c->lv) v.push_back(level_timestep(lv, cfg, use_visc));
    return comm_reduce(c, v, 0);
  };
  return run_level_loop(ops, cfg, sp, on_row, user, rows, max_rows, n_rows, converged, err, errlen);
}

int cdg_gpu_comm_exchange_count(const cdg_gpu_comm* c) { return (int)c->exchanges; }

}  // extern "C"
