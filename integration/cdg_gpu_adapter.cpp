// cdg_gpu_adapter.cpp -- the reference-side binding: implements the reference
// solver kernel API (proj/core/include/cdg/solver.hpp:83-109) on top of the
// C ABI in include/cdg_gpu.h, so reference code (run_steady, the CLI, the
// reference's own unit tests) calls the B200 path unchanged.
//
//   cdg::make_workspace        solver.hpp:84   -> cdg_gpu_level_create
//   cdg::interpolate_to_faces  solver.hpp:87   -> cdg_gpu_interpolate_to_faces
//   cdg::compute_rhs           solver.hpp:94   -> cdg_gpu_compute_rhs
//   cdg::current_viscosity     solver.hpp:100  -> cdg_gpu_viscosity
//   cdg::aux_gradient          solver.hpp:103  -> cdg_gpu_aux_gradient
//   cdg::rk_step               solver.hpp:107  -> cdg_gpu_rk_steps (1 step)
//   cdg::run_steady            solver.hpp:128  -> cdg_gpu_fill_freestream / cdg_gpu_p_refine_embed /
//                                                 cdg_gpu_run_level (device-resident levels; the host
//                                                 syncs only at check iterations)
//
// Build (reference side): compile this file against proj/core/include, link
// libcdg_gpu.so, and compile solver.cpp with the six names above renamed
// (e.g. -Dcompute_rhs=compute_rhs_cpu ...; oracle/Makefile target
// test_solver_gpu does exactly this to run the reference's test_solver.cpp on
// the GPU). Exceptions and messages are the reference's: status 3 ->
// NumericsError, 2 -> ConfigError.
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "cdg/solver.hpp"
#include "cdg_gpu.h"
#include "cdg_gpu_adapter.hpp"

namespace cdg {

struct RhsWorkspace {
  const DgLevel* level = nullptr;
  cdg_gpu_level* lv = nullptr;
  std::vector<double> eps;
  std::array<SolutionStore, 3> q;
  ~RhsWorkspace() {
    if (lv) cdg_gpu_level_destroy(lv);
  }
};

namespace {

void throw_status(int st, const char* msg) {
  if (st == 0) return;
  if (st == CDG_GPU_ERR_NUMERICS) throw NumericsError(msg);
  if (st == CDG_GPU_ERR_CONFIG) throw ConfigError(msg);
  throw std::runtime_error(std::string("cdg_gpu: ") + msg);
}

std::vector<double> row_major(const Eigen::MatrixXd& m) {
  std::vector<double> out(static_cast<size_t>(m.rows() * m.cols()));
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) out[static_cast<size_t>(i * m.cols() + j)] = m(i, j);
  return out;
}

// Device of the levels the adapter creates: cdg::gpu_select_device(), else
// $CDG_GPU_DEVICE, else 0 (one process per GPU).
int g_device = -1;
int adapter_device() {
  if (g_device < 0) {
    const char* v = std::getenv("CDG_GPU_DEVICE");
    g_device = v ? std::atoi(v) : 0;
  }
  return g_device;
}

// CurvedMesh::is_curved(e) as DgLevel recorded it: DgLevel's constructor maps
// every element from CurvedMesh::element_nodes_for_degree, which returns
// straight_nodes(mesh, e, re) exactly when the element is not curved
// (solver.cpp:116-118, curved_mesh.cpp:24-27), and keeps those nodes in
// ElementGeometry::phys_nodes (operators.hpp:15). So an element is curved iff
// its stored nodes are not bit-identical to its straight nodes -- no tolerance.
std::vector<char> curved_mask(const DgLevel& level) {
  const int K = level.n_elements();
  std::vector<char> mask(K, 0);
  for (int e = 0; e < K; ++e) {
    const auto straight = CurvedMesh::straight_nodes(level.mesh(), e, level.refelem());
    const auto& nodes = level.geom(e).phys_nodes;
    bool same = nodes.size() == straight.size();
    for (size_t i = 0; same && i < nodes.size(); ++i)
      same = nodes[i].x == straight[i].x && nodes[i].y == straight[i].y && nodes[i].z == straight[i].z;
    mask[e] = same ? 0 : 1;
  }
  return mask;
}

cdg_gpu_level* create_level(const DgLevel& level, const ConservedState& fs, const std::vector<char>& is_curved) {
  const auto& re = level.refelem();
  const int K = level.n_elements(), np = re.n_basis(), ncub = re.n_cub(), ng = re.n_face_quad();
  std::vector<double> icub = row_major(re.interp_cub()), ig = row_major(re.interp_face()),
                      dr = row_major(re.deriv_r()), ds = row_major(re.deriv_s()),
                      dt = row_major(re.deriv_t()), vinv = row_major(re.vandermonde_inv());
  std::vector<double> metric(9 * (size_t)K), jac(K), normal(12 * (size_t)K), sjac(4 * (size_t)K), h(K);
  std::vector<int> nb(4 * (size_t)K), nbf(4 * (size_t)K), bc(4 * (size_t)K), nmap(4 * (size_t)K * ng);
  // curved (isoparametric) elements: per-node geometry + M_e^-1
  std::vector<int> cids;
  std::vector<double> cjwr, cface, cminv, cjac;
  for (int e = 0; e < K; ++e) {
    const auto& g = level.geom(e);
    if (is_curved[e]) {
      cids.push_back(e);
      for (int q = 0; q < ncub; ++q) cjac.push_back(g.cub_jac[q]);
      for (int q = 0; q < ncub; ++q)
        for (int k = 0; k < 9; ++k) cjwr.push_back(g.cub_jac[q] * re.cub_weights()[q] * g.cub_dr[q][k]);
      for (int q = 0; q < 4 * ng; ++q) {
        for (int d = 0; d < 3; ++d) cface.push_back(g.face_normal[q][d]);
        cface.push_back(g.face_sjac[q] * re.face_weights()[q % ng]);
      }
      // M^-1 = L^-T L^-1 from the reference's Cholesky factor (operators.cpp:151-158)
      const auto& l = level.ops(e).mass_chol;
      std::vector<double> inv((size_t)np * np), y(np), x(np);
      for (int col = 0; col < np; ++col) {
        for (int i = 0; i < np; ++i) {
          double s2 = (i == col) ? 1.0 : 0.0;
          for (int j = 0; j < i; ++j) s2 -= l[j * np + i] * y[j];
          y[i] = s2 / l[i * np + i];
        }
        for (int i = np - 1; i >= 0; --i) {
          double s2 = y[i];
          for (int j = i + 1; j < np; ++j) s2 -= l[i * np + j] * x[j];
          x[i] = s2 / l[i * np + i];
        }
        for (int i = 0; i < np; ++i) inv[(size_t)i * np + col] = x[i];
      }
      cminv.insert(cminv.end(), inv.begin(), inv.end());
    }
    for (int k = 0; k < 9; ++k) metric[9 * (size_t)e + k] = g.cub_dr[0][k];
    jac[e] = g.cub_jac[0];
    h[e] = g.h();
    for (int f = 0; f < 4; ++f) {
      for (int d = 0; d < 3; ++d) normal[12 * (size_t)e + 3 * f + d] = g.face_normal[f * ng][d];
      sjac[4 * (size_t)e + f] = g.face_sjac[f * ng];
      const auto& fc = level.coupling(e, f);
      nb[4 * (size_t)e + f] = fc.neighbor;
      nbf[4 * (size_t)e + f] = fc.neighbor >= 0 ? fc.neighbor_face : 0;
      bc[4 * (size_t)e + f] = static_cast<int>(fc.bc);
      for (int gg = 0; gg < ng; ++gg)
        nmap[(4 * (size_t)e + f) * ng + gg] = fc.neighbor >= 0 ? fc.node_map[gg] : 0;
    }
  }
  cdg_gpu_level_desc d{};
  d.degree = re.degree();
  d.n_basis = np;
  d.n_cub = ncub;
  d.n_face_quad = ng;
  d.n_elements = K;
  d.n_halo = 0;
  d.padded = level.padded() ? 1 : 0;
  d.interp_cub = icub.data();
  d.interp_face = ig.data();
  d.deriv_r = dr.data();
  d.deriv_s = ds.data();
  d.deriv_t = dt.data();
  d.cub_weights = re.cub_weights().data();
  d.face_weights = re.face_weights().data();
  d.vandermonde_inv = vinv.data();
  d.metric = metric.data();
  d.jac = jac.data();
  d.face_normal = normal.data();
  d.face_sjac = sjac.data();
  d.h = h.data();
  d.neighbor = nb.data();
  d.neighbor_face = nbf.data();
  d.bc = bc.data();
  d.node_map = nmap.data();
  for (int c = 0; c < 5; ++c) d.freestream[c] = fs[c];
  d.n_curved = static_cast<int>(cids.size());
  d.curved_ids = cids.data();
  d.curved_jwr = cjwr.data();
  d.curved_face = cface.data();
  d.curved_minv = cminv.data();
  d.curved_jac = cjac.data();
  // modal basis at the cubature nodes: the J-weighted indicator's V_cub (viscosity.cpp:35)
  const std::vector<double> vcub = row_major(modal_basis_eval(re.degree(), re.cub_nodes()));
  d.modal_cub = vcub.data();
  cdg_gpu_level* lv = nullptr;
  char err[512] = {0};
  throw_status(cdg_gpu_level_create(&d, adapter_device(), &lv, err, sizeof err), err);
  return lv;
}

// Straight-sided meshes: the level straight from the Mesh (no DgLevel) --
// cdg_gpu_level_create_from_mesh computes the affine geometry and the
// FaceLink.perm pairing in the library, O(K) and ~100 bytes per element, so
// run_steady reaches the 4M-element configuration (DgLevel needs ~140 KB per
// element at P=4, solver.cpp:97-179).
cdg_gpu_level* create_level_from_mesh(const Mesh& mesh, const ReferenceElement& re, const BcMap& bc_map,
                                      const ConservedState& fs, bool padded) {
  const int K = mesh.n_elements(), ng = re.n_face_quad();
  std::vector<double> icub = row_major(re.interp_cub()), ig = row_major(re.interp_face()),
                      dr = row_major(re.deriv_r()), ds = row_major(re.deriv_s()),
                      dt = row_major(re.deriv_t()), vinv = row_major(re.vandermonde_inv());
  const std::vector<double> vcub = row_major(modal_basis_eval(re.degree(), re.cub_nodes()));
  std::vector<double> verts(3 * mesh.vertices.size()), fnodes(3 * (size_t)ng);
  for (size_t v = 0; v < mesh.vertices.size(); ++v)
    verts[3 * v] = mesh.vertices[v].x, verts[3 * v + 1] = mesh.vertices[v].y, verts[3 * v + 2] = mesh.vertices[v].z;
  for (int g = 0; g < ng; ++g)
    fnodes[3 * g] = re.face_nodes()[g].x, fnodes[3 * g + 1] = re.face_nodes()[g].y, fnodes[3 * g + 2] = re.face_nodes()[g].z;
  std::vector<int> tets(4 * (size_t)K), nb(4 * (size_t)K), nbf(4 * (size_t)K), perm(12 * (size_t)K), bc(4 * (size_t)K);
  for (int e = 0; e < K; ++e)
    for (int f = 0; f < 4; ++f) {
      const size_t i4 = 4 * (size_t)e + f;
      tets[i4] = mesh.tets[e][f];
      if (mesh.links[e][f]) {
        const FaceLink& l = *mesh.links[e][f];
        nb[i4] = l.other.element;
        nbf[i4] = l.other.local_face;
        for (int k = 0; k < 3; ++k) perm[3 * i4 + k] = l.perm[k];
        bc[i4] = 0;
      } else {
        nb[i4] = -1;
        nbf[i4] = 0;
        perm[3 * i4] = 0, perm[3 * i4 + 1] = 1, perm[3 * i4 + 2] = 2;
        const std::string& tag = mesh.boundary_faces[mesh.boundary_index[e][f]].tag;
        int kind = -1;  // kind_for_tag (solver.cpp:136-140)
        for (const auto& [name, k] : bc_map)
          if (name == tag) {
            kind = static_cast<int>(k);
            break;
          }
        if (kind < 0) throw ConfigError("no boundary condition configured for mesh tag '" + tag + "'");
        bc[i4] = kind;
      }
    }
  cdg_gpu_level_desc d{};
  d.degree = re.degree();
  d.n_basis = re.n_basis();
  d.n_cub = re.n_cub();
  d.n_face_quad = ng;
  d.padded = padded ? 1 : 0;
  d.interp_cub = icub.data();
  d.interp_face = ig.data();
  d.deriv_r = dr.data();
  d.deriv_s = ds.data();
  d.deriv_t = dt.data();
  d.cub_weights = re.cub_weights().data();
  d.face_weights = re.face_weights().data();
  d.vandermonde_inv = vinv.data();
  d.modal_cub = vcub.data();
  for (int c = 0; c < 5; ++c) d.freestream[c] = fs[c];
  cdg_gpu_mesh_desc md{};
  md.n_vertices = static_cast<int>(mesh.vertices.size());
  md.vertices = verts.data();
  md.n_elements = K;
  md.tets = tets.data();
  md.neighbor = nb.data();
  md.neighbor_face = nbf.data();
  md.face_perm = perm.data();
  md.bc = bc.data();
  md.face_nodes = fnodes.data();
  cdg_gpu_level* lv = nullptr;
  char err[512] = {0};
  throw_status(cdg_gpu_level_create_from_mesh(&d, &md, adapter_device(), &lv, err, sizeof err), err);
  return lv;
}

cdg_gpu_run_config to_cfg(const RunConfig& cfg) {
  cdg_gpu_run_config c{};
  if (cfg.riemann == "llf")
    c.riemann = CDG_GPU_RIEMANN_LLF;
  else if (cfg.riemann == "hllc")
    c.riemann = CDG_GPU_RIEMANN_HLLC;
  else
    throw ConfigError("unknown Riemann solver '" + cfg.riemann + "' (llf|hllc)");
  c.gamma = cfg.gas.gamma;
  c.visc_enabled = cfg.viscosity.enabled;
  c.eps0 = cfg.viscosity.eps0;
  c.kappa = cfg.viscosity.kappa;
  c.s0_offset = cfg.viscosity.s0_offset;
  c.indicator_component = cfg.viscosity.indicator_component;
  c.jacobian_weighted = cfg.viscosity.jacobian_weighted;
  c.cfl = cfg.cfl;
  return c;
}

void ensure_level(RhsWorkspace& ws, const ConservedState& fs) {
  if (!ws.lv) ws.lv = create_level(*ws.level, fs, curved_mask(*ws.level));
  double f[5] = {fs[0], fs[1], fs[2], fs[3], fs[4]};
  throw_status(cdg_gpu_set_freestream(ws.lv, f), "set_freestream failed");
}

}  // namespace

void gpu_select_device(int device) { g_device = device; }

std::shared_ptr<RhsWorkspace> make_workspace(const DgLevel& level) {
  auto ws = std::make_shared<RhsWorkspace>();
  ws->level = &level;
  ws->eps.assign(level.n_elements(), 0.0);
  return ws;
}

void interpolate_to_faces(const DgLevel& level, const SolutionStore& u, SolutionStore& traces) {
  RhsWorkspace ws;
  ws.level = &level;
  ensure_level(ws, ConservedState{});
  throw_status(cdg_gpu_set_state(ws.lv, u.raw().data(), nullptr), "set_state failed");
  throw_status(cdg_gpu_interpolate_to_faces(ws.lv, traces.raw().data()), "interpolate_to_faces failed");
}

void compute_rhs(const DgLevel& level, const SolutionStore& u, const RunConfig& cfg,
                 const ConservedState& freestream, SolutionStore& rhs, RhsWorkspace& ws) {
  (void)level;
  ensure_level(ws, freestream);
  const cdg_gpu_run_config c = to_cfg(cfg);
  char err[512] = {0};
  throw_status(cdg_gpu_set_state(ws.lv, u.raw().data(), nullptr), "set_state failed");
  throw_status(cdg_gpu_compute_rhs(ws.lv, &c, rhs.raw().data(), err, sizeof err), err);
  if (cfg.viscosity.enabled) {
    throw_status(cdg_gpu_viscosity(ws.lv, ws.eps.data()), "viscosity failed");
    for (int m = 0; m < 3; ++m) {
      if (ws.q[m].n_elements() == 0) ws.q[m] = ws.level->make_store();
      if (cdg_gpu_aux_gradient(ws.lv, m, ws.q[m].raw().data()) != 0) break;  // inviscid evaluation
    }
  }
}

const std::vector<double>& current_viscosity(const RhsWorkspace& ws) { return ws.eps; }

const SolutionStore& aux_gradient(const RhsWorkspace& ws, int direction) { return ws.q[direction]; }

void rk_step(const DgLevel& level, SolutionStore& u, SolutionStore& res, const RunConfig& cfg,
             const ConservedState& freestream, double dt, const RKScheme& scheme, RhsWorkspace& ws) {
  (void)level;
  ensure_level(ws, freestream);
  const cdg_gpu_run_config c = to_cfg(cfg);
  char err[512] = {0};
  throw_status(cdg_gpu_set_state(ws.lv, u.raw().data(), res.raw().data()), "set_state failed");
  throw_status(cdg_gpu_rk_steps(ws.lv, &c, 1, dt, scheme.a.data(), scheme.b.data(), err, sizeof err), err);
  throw_status(cdg_gpu_get_state(ws.lv, u.raw().data(), res.raw().data()), "get_state failed");
  if (cfg.viscosity.enabled) throw_status(cdg_gpu_viscosity(ws.lv, ws.eps.data()), "viscosity failed");
}

// run_steady (solver.cpp:594-676) with every level device-resident. Host work
// per level: the level setup (straight meshes: in the library from the Mesh,
// O(K); curved meshes: the reference's DgLevel for the curved geometry), then
// one cdg_gpu_run_level_live call; rows reach on_row live, at each check
// iteration.
SteadyResult run_steady(const CurvedMesh& cmesh, const BcMap& bc_map, const RunConfig& cfg,
                        const ConservedState& freestream, const std::function<void(const ConvergenceRow&)>& on_row) {
  if (cfg.p_schedule.empty()) throw ConfigError("run_steady: empty p-schedule");
  for (size_t i = 1; i < cfg.p_schedule.size(); ++i)
    if (cfg.p_schedule[i] <= cfg.p_schedule[i - 1])
      throw ConfigError("run_steady: p-schedule must be strictly increasing");
  SteadyResult result;
  const auto wall_start = std::chrono::steady_clock::now();
  const cdg_gpu_run_config c = to_cfg(cfg);
  std::unique_ptr<cdg_gpu_level, void (*)(cdg_gpu_level*)> prev(nullptr, cdg_gpu_level_destroy);
  std::shared_ptr<const ReferenceElement> re_prev;
  for (size_t li = 0; li < cfg.p_schedule.size(); ++li) {
    const int p = cfg.p_schedule[li];
    auto re = level_reference_element(cmesh, p, cfg);
    // straight-sided meshes: the level straight from the Mesh (scalable
    // setup); curved meshes: the reference's DgLevel supplies the per-node
    // geometry of the curved elements (compute_mapping, operators.cpp:32-121)
    std::unique_ptr<DgLevel> level;
    std::unique_ptr<cdg_gpu_level, void (*)(cdg_gpu_level*)> lv(nullptr, cdg_gpu_level_destroy);
    if (cmesh.n_curved() == 0) {
      lv.reset(create_level_from_mesh(cmesh.mesh(), *re, bc_map, freestream, cfg.padded));
    } else {
      level = std::make_unique<DgLevel>(cmesh, re, bc_map, cfg.padded);
      std::vector<char> mask(level->n_elements());
      for (int e = 0; e < level->n_elements(); ++e) mask[e] = cmesh.is_curved(e) ? 1 : 0;
      lv.reset(create_level(*level, freestream, mask));
    }
    if (li == 0) {
      throw_status(cdg_gpu_fill_freestream(lv.get()), "fill_freestream failed");
    } else {
      const Eigen::MatrixXd embed = re->vandermonde().leftCols(re_prev->n_basis()) * re_prev->vandermonde_inv();
      const std::vector<double> e = row_major(embed);
      throw_status(cdg_gpu_p_refine_embed(lv.get(), prev.get(), e.data()), "p_refine_embed failed");
    }
    prev.reset();
    re_prev = re;
    const bool last = li + 1 == cfg.p_schedule.size();
    cdg_gpu_steady_params sp{};
    sp.max_iterations = cfg.max_iterations_per_level;
    sp.fixed_iterations = li < cfg.fixed_iterations.size() ? cfg.fixed_iterations[li] : -1;
    sp.check_interval = cfg.check_interval;
    sp.residual_kind = cfg.residual_norm == "l2" ? 1 : 0;  // anything else: inf (solver.cpp:572-590)
    sp.tolerance = last ? cfg.final_tolerance : cfg.intermediate_tolerance;
    sp.dt_override = cfg.dt_override;
    sp.degree = p;
    const int max_rows = static_cast<int>(cfg.max_iterations_per_level / std::max(1, cfg.check_interval)) + 2;
    std::vector<double> rows(3 * (size_t)max_rows);
    int n_rows = 0, converged = 0;
    char err[512] = {0};
    // rows go to the log and on_row as each check iteration completes, with
    // the wall time since run_steady started (solver.cpp:643-647)
    struct Sink {
      int p;
      SteadyResult* result;
      const std::function<void(const ConvergenceRow&)>* on_row;
      std::chrono::steady_clock::time_point t0;
    } sink{p, &result, &on_row, wall_start};
    auto emit = [](void* user, long iteration, double dt, double residual) {
      auto* k = static_cast<Sink*>(user);
      const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - k->t0).count();
      ConvergenceRow row{k->p, iteration, dt, residual, wall};
      k->result->log.push_back(row);
      if (*k->on_row) (*k->on_row)(row);
    };
    throw_status(cdg_gpu_run_level_live(lv.get(), &c, &sp, emit, &sink, rows.data(), max_rows, &n_rows, &converged,
                                        err, sizeof err),
                 err);
    if (last) {
      result.converged = converged != 0;
      if (sp.fixed_iterations > 0 && !result.log.empty())
        result.converged = result.log.back().residual < cfg.final_tolerance;
      result.solution = SolutionStore(cmesh.mesh().n_elements(), re->n_basis(), cfg.padded);
      throw_status(cdg_gpu_get_state(lv.get(), result.solution.raw().data(), nullptr), "get_state failed");
    }
    result.final_degree = p;
    prev = std::move(lv);
  }
  return result;
}

}  // namespace cdg
