// ORACLE TEST INFRASTRUCTURE ONLY.
//
// extern "C" façade over the UNMODIFIED reference library (compiled in place
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libcdg_ref.so). It lets pytest (ctypes) drive the reference's
// own mesh generators, DgLevel construction, compute_rhs, rk_step and the
// viscosity model on the same inputs the GPU path sees. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load this library, and only as the checker / CPU baseline.
//
// Reference entry points wrapped (all under /root/reference/proj/core):
//   make_cube_mesh / make_single_tet / make_two_tets / make_sphere_shell_mesh
//                                           src/meshgen.cpp:41-225
//   DgLevel::DgLevel                         src/solver.cpp:97-179
//   make_workspace / compute_rhs / rk_step   src/solver.cpp:72-85, 325-492
//   compute_timestep                         src/solver.cpp:494-526
//   current_viscosity / aux_gradient         src/solver.cpp:87-91
//   random_admissible_store recipe           src/bench.cpp:22-40 (restated: it
//                                            is file-static in the reference)
#include <chrono>
#include <omp.h>

#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "cdg/curved_mesh.hpp"
#include "cdg/elasticity.hpp"
#include "cdg/meshgen.hpp"
#include "cdg/nurbs.hpp"
#include "cdg/refelem.hpp"
#include "cdg/solver.hpp"

using namespace cdg;

namespace {

struct RefMesh {
  Mesh mesh;
  std::unique_ptr<CurvedMesh> curved;  // set by ref_mesh_sphere_curved
};

struct RefLevel {
  const RefMesh* mesh = nullptr;
  std::unique_ptr<CurvedMesh> cmesh;
  std::unique_ptr<DgLevel> level;
  std::shared_ptr<RhsWorkspace> ws;
};

void copy_err(const std::exception& e, char* err, size_t n) {
  if (err && n) {
    std::strncpy(err, e.what(), n - 1);
    err[n - 1] = 0;
  }
}

int status_of(const std::exception& e) {
  if (dynamic_cast<const NumericsError*>(&e)) return 3;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  return 1;
}

}  // namespace

namespace cdg_oracle {
void make_periodic(cdg::DgLevel& level, const double period[3]);  // ref_periodic.cpp
}

extern "C" {

// Mirrors cdg_gpu_run_config in include/cdg_gpu.h (same field order).
struct ref_run_cfg {
  int riemann;  // 0 llf, 1 hllc
  double gamma;
  int visc_enabled;
  double eps0, kappa, s0_offset;
  int indicator_component;
  int jacobian_weighted;
  double cfl;
};

static RunConfig to_cfg(const ref_run_cfg* c) {
  RunConfig cfg;
  cfg.riemann = c->riemann == 1 ? "hllc" : "llf";
  cfg.gas.gamma = c->gamma;
  cfg.viscosity.enabled = c->visc_enabled != 0;
  cfg.viscosity.eps0 = c->eps0;
  cfg.viscosity.kappa = c->kappa;
  cfg.viscosity.s0_offset = c->s0_offset;
  cfg.viscosity.indicator_component = c->indicator_component;
  cfg.viscosity.jacobian_weighted = c->jacobian_weighted != 0;
  cfg.cfl = c->cfl;
  return cfg;
}

static ConservedState to_state(const double* f) {
  ConservedState s;
  s.rho = f[0];
  s.mom = {f[1], f[2], f[3]};
  s.rhoE = f[4];
  return s;
}

int ref_num_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

// ---- reference element tables (refelem.cpp:301-358) -----------------------
// sizes[0..3] = n_basis, n_cub, n_face_quad, degree
int ref_refelem_sizes(int p, int cub_override, int face_override, int* sizes) {
  try {
    auto re = get_reference_element(p, cub_override, face_override);
    sizes[0] = re->n_basis();
    sizes[1] = re->n_cub();
    sizes[2] = re->n_face_quad();
    sizes[3] = re->degree();
    return 0;
  } catch (const std::exception&) {
    return 2;
  }
}

static void put(const Eigen::MatrixXd& m, double* out) {
  // row-major export
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) out[i * m.cols() + j] = m(i, j);
}

// Row-major dumps. colloc/cub/face nodes are [n][3].
int ref_refelem_tables(int p, int cub_override, int face_override, double* colloc,
                       double* cub_nodes, double* cub_w, double* face_nodes, double* face_w,
                       double* vand, double* vand_inv, double* interp_cub,
                       double* interp_face, double* dr, double* ds, double* dt) {
  auto re = get_reference_element(p, cub_override, face_override);
  for (size_t i = 0; i < re->colloc_nodes().size(); ++i)
    for (int d = 0; d < 3; ++d) colloc[3 * i + d] = re->colloc_nodes()[i][d];
  for (size_t i = 0; i < re->cub_nodes().size(); ++i)
    for (int d = 0; d < 3; ++d) cub_nodes[3 * i + d] = re->cub_nodes()[i][d];
  for (size_t i = 0; i < re->face_nodes().size(); ++i)
    for (int d = 0; d < 3; ++d) face_nodes[3 * i + d] = re->face_nodes()[i][d];
  std::memcpy(cub_w, re->cub_weights().data(), sizeof(double) * re->cub_weights().size());
  std::memcpy(face_w, re->face_weights().data(), sizeof(double) * re->face_weights().size());
  put(re->vandermonde(), vand);
  put(re->vandermonde_inv(), vand_inv);
  put(re->interp_cub(), interp_cub);
  put(re->interp_face(), interp_face);
  put(re->deriv_r(), dr);
  put(re->deriv_s(), ds);
  put(re->deriv_t(), dt);
  return 0;
}

// ---- meshes (meshgen.cpp) ---------------------------------------------------
void* ref_mesh_cube(int n, double scale) {
  auto* m = new RefMesh;
  m->mesh = make_cube_mesh(n, "wall");
  if (scale != 1.0)
    for (auto& v : m->mesh.vertices) v = v * scale;
  return m;
}
void* ref_mesh_single_tet() {
  auto* m = new RefMesh;
  m->mesh = make_single_tet("wall");
  return m;
}
void* ref_mesh_two_tets() {
  auto* m = new RefMesh;
  m->mesh = make_two_tets("wall");
  return m;
}
// Any tet mesh from arrays (the generators of paper_1208_4772_b200/cases.py:
// cylinder, NACA0012): vertices [nv][3], tets [K][4] (positively oriented),
// boundary faces [nb] (element, local face, tag index into the comma-separated
// tag_names); connectivity by the reference's own build_connectivity
// (mesh.cpp:26-84) after validate_mesh.
void* ref_mesh_from_arrays(int nv, const double* verts, int K, const int* tets, int nb, const int* bf_elem,
                           const int* bf_face, const int* bf_tag, const char* tag_names, char* err, size_t errn) {
  try {
    auto* m = new RefMesh;
    std::vector<std::string> names;
    {
      std::string cur;
      for (const char* c = tag_names; *c; ++c) {
        if (*c == ',') names.push_back(cur), cur.clear();
        else cur += *c;
      }
      names.push_back(cur);
    }
    for (int v = 0; v < nv; ++v) m->mesh.vertices.push_back({verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]});
    for (int e = 0; e < K; ++e) m->mesh.tets.push_back({tets[4 * e], tets[4 * e + 1], tets[4 * e + 2], tets[4 * e + 3]});
    for (int i = 0; i < nb; ++i) m->mesh.boundary_faces.push_back({bf_elem[i], bf_face[i], names.at(bf_tag[i])});
    validate_mesh(m->mesh);
    build_connectivity(m->mesh);
    return m;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return nullptr;
  }
}
// Curve elements of a mesh: nodes [n][N_p(degree)][3] are the physical
// collocation nodes of element ids[i] at `degree` (CurvedMesh::set_curved,
// curved_mesh.hpp:24); levels of other degrees re-evaluate the map
// (element_nodes_for_degree).
int ref_mesh_set_curved(void* h, int degree, int n, const int* ids, const double* nodes, char* err, size_t errn) {
  try {
    auto* m = static_cast<RefMesh*>(h);
    m->curved = std::make_unique<CurvedMesh>(m->mesh, degree);
    const int np = (degree + 1) * (degree + 2) * (degree + 3) / 6;
    for (int i = 0; i < n; ++i) {
      std::vector<Vec3> x(np);
      for (int j = 0; j < np; ++j)
        x[j] = {nodes[((size_t)i * np + j) * 3], nodes[((size_t)i * np + j) * 3 + 1], nodes[((size_t)i * np + j) * 3 + 2]};
      m->curved->set_curved(ids[i], std::move(x));
    }
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return 1;
  }
}
// All boundary faces of the sphere shell get tag "wall" or "farfield" via the
// reference tags "sphere"/"farfield".
void* ref_mesh_sphere_shell(double r_in, double r_out, int subdiv, int layers) {
  auto* m = new RefMesh;
  m->mesh = make_sphere_shell_mesh(r_in, r_out, subdiv, layers, "sphere", "farfield");
  return m;
}
// The acceptance fixture pipeline (acceptance_main.cpp:82-120 / cmd_curve,
// cli_ops.cpp:16-76) in memory: sphere shell, box [-1.5,1.5]^3 sub-mesh,
// elasticity with E=1 nu=0.45 and the exact sphere displacement, curve_mesh at
// degree p_curve. Returns null on failure (err filled).
void* ref_mesh_sphere_curved(int subdiv, int layers, int p_curve, int p_fem, char* err, size_t errn) {
  try {
    auto* m = new RefMesh;
    m->mesh = make_sphere_shell_mesh(1.0, 8.0, subdiv, layers, "sphere", "farfield");
    const Box box{{-1.5, -1.5, -1.5}, {1.5, 1.5, 1.5}};
    const SubMesh sub = extract_submesh(m->mesh, box, "sphere", {});
    const Vec3 center{0, 0, 0};
    auto g = [center](const Vec3& x) { return sphere_displacement(center, 1.0, x); };
    const auto material = ElasticMaterial::from_E_nu(1.0, 0.45);
    const DeformationField field = solve_elasticity(sub, material, g, p_fem);
    auto re = get_reference_element(p_curve);
    m->curved = std::make_unique<CurvedMesh>(curve_mesh(m->mesh, sub, field, *re));
    return m;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return nullptr;
  }
}

void ref_mesh_free(void* h) { delete static_cast<RefMesh*>(h); }

// sizes: [0]=n_vertices [1]=n_elements [2]=n_boundary_faces
void ref_mesh_sizes(void* h, int* sizes) {
  const Mesh& m = static_cast<RefMesh*>(h)->mesh;
  sizes[0] = static_cast<int>(m.vertices.size());
  sizes[1] = m.n_elements();
  sizes[2] = static_cast<int>(m.boundary_faces.size());
}

// verts [nv][3]; tets [ne][4]; neighbor/neighbor_face/perm [ne][4](perm packed
// p0+3p1+9p2); bnd_tag [ne][4]: -1 interior, else index into a tag list where
// "wall"/"sphere"=0, "farfield"=1, other=2.
void ref_mesh_export(void* h, double* verts, int* tets, int* neighbor, int* neighbor_face,
                     int* perm, int* bnd_tag) {
  const Mesh& m = static_cast<RefMesh*>(h)->mesh;
  for (size_t i = 0; i < m.vertices.size(); ++i)
    for (int d = 0; d < 3; ++d) verts[3 * i + d] = m.vertices[i][d];
  for (int e = 0; e < m.n_elements(); ++e) {
    for (int k = 0; k < 4; ++k) tets[4 * e + k] = m.tets[e][k];
    for (int f = 0; f < 4; ++f) {
      const int idx = 4 * e + f;
      if (m.links[e][f]) {
        neighbor[idx] = m.links[e][f]->other.element;
        neighbor_face[idx] = m.links[e][f]->other.local_face;
        const auto& p = m.links[e][f]->perm;
        perm[idx] = p[0] + 3 * p[1] + 9 * p[2];
        bnd_tag[idx] = -1;
      } else {
        neighbor[idx] = -1;
        neighbor_face[idx] = -1;
        perm[idx] = -1;
        const std::string& tag = m.boundary_faces[m.boundary_index[e][f]].tag;
        bnd_tag[idx] = (tag == "wall" || tag == "sphere") ? 0 : (tag == "farfield" ? 1 : 2);
      }
    }
  }
}

// ---- levels (solver.cpp:97-179) ----------------------------------------------
// bc_wall / bc_far: BcKind (0 SlipWall, 1 Farfield, 2 Symmetry) for the
// "wall"/"sphere" and "farfield" tags.
void* ref_level_create(void* mesh_h, int p, int bc_wall, int bc_far, int padded,
                       int curved_quadrature, char* err, size_t errn) {
  try {
    auto* lv = new RefLevel;
    lv->mesh = static_cast<RefMesh*>(mesh_h);
    lv->cmesh = lv->mesh->curved ? std::make_unique<CurvedMesh>(*lv->mesh->curved)
                                 : std::make_unique<CurvedMesh>(lv->mesh->mesh, p);
    RunConfig cfg;
    cfg.curved_quadrature = curved_quadrature != 0;
    auto re = level_reference_element(*lv->cmesh, p, cfg);
    const BcMap bcs = {{"wall", static_cast<BcKind>(bc_wall)},
                       {"sphere", static_cast<BcKind>(bc_wall)},
                       {"farfield", static_cast<BcKind>(bc_far)},
                       {"symmetry", BcKind::Symmetry}};
    lv->level = std::make_unique<DgLevel>(*lv->cmesh, re, bcs, padded != 0);
    lv->ws = make_workspace(*lv->level);
    return lv;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return nullptr;
  }
}
void ref_level_free(void* h) { delete static_cast<RefLevel*>(h); }
// Periodic box (BASELINE config 1): link every boundary face of the level to
// its translate across the box (ref_periodic.cpp). Returns 0 / 1 (+ message).
int ref_level_make_periodic(void* h, double lx, double ly, double lz, char* err, size_t errn) {
  try {
    const double period[3] = {lx, ly, lz};
    cdg_oracle::make_periodic(*static_cast<RefLevel*>(h)->level, period);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return 1;
  }
}

// sizes: [0]=K [1]=n_basis [2]=n_cub [3]=n_face_quad [4]=block [5]=trace_block [6]=degree
void ref_level_sizes(void* h, int* sizes) {
  const DgLevel& lv = *static_cast<RefLevel*>(h)->level;
  sizes[0] = lv.n_elements();
  sizes[1] = lv.refelem().n_basis();
  sizes[2] = lv.refelem().n_cub();
  sizes[3] = lv.refelem().n_face_quad();
  const SolutionStore s = lv.make_store();
  const SolutionStore t = lv.make_trace_store();
  sizes[4] = s.block_length();
  sizes[5] = t.block_length();
  sizes[6] = lv.refelem().degree();
}

// Per-element geometry + coupling as the reference built it.
//  cub_dr [K][ncub][9], cub_jac [K][ncub], face_normal [K][nf][3],
//  face_sjac [K][nf], face_phys [K][nf][3], h [K], neighbor/nface/bc [K][4],
//  node_map [K][4][ng] (-1 on boundary faces). Any pointer may be null.
void ref_level_geometry(void* h, double* cub_dr, double* cub_jac, double* face_normal,
                        double* face_sjac, double* face_phys, double* hk, int* neighbor,
                        int* neighbor_face, int* bc, int* node_map) {
  const DgLevel& lv = *static_cast<RefLevel*>(h)->level;
  const int ne = lv.n_elements(), ncub = lv.refelem().n_cub(),
            ng = lv.refelem().n_face_quad(), nf = 4 * ng;
  for (int e = 0; e < ne; ++e) {
    const auto& g = lv.geom(e);
    for (int q = 0; q < ncub; ++q) {
      if (cub_dr)
        for (int k = 0; k < 9; ++k) cub_dr[(static_cast<size_t>(e) * ncub + q) * 9 + k] = g.cub_dr[q][k];
      if (cub_jac) cub_jac[static_cast<size_t>(e) * ncub + q] = g.cub_jac[q];
    }
    for (int q = 0; q < nf; ++q) {
      for (int d = 0; d < 3; ++d) {
        if (face_normal) face_normal[(static_cast<size_t>(e) * nf + q) * 3 + d] = g.face_normal[q][d];
        if (face_phys) face_phys[(static_cast<size_t>(e) * nf + q) * 3 + d] = g.face_phys[q][d];
      }
      if (face_sjac) face_sjac[static_cast<size_t>(e) * nf + q] = g.face_sjac[q];
    }
    if (hk) hk[e] = g.h();
    for (int f = 0; f < 4; ++f) {
      const auto& fc = lv.coupling(e, f);
      if (neighbor) neighbor[4 * e + f] = fc.neighbor;
      if (neighbor_face) neighbor_face[4 * e + f] = fc.neighbor_face;
      if (bc) bc[4 * e + f] = fc.neighbor >= 0 ? -1 : static_cast<int>(fc.bc);
      if (node_map)
        for (int gg = 0; gg < ng; ++gg)
          node_map[(static_cast<size_t>(e) * 4 + f) * ng + gg] =
              fc.neighbor >= 0 ? fc.node_map[gg] : -1;
    }
  }
}

// Element collocation nodes at the level degree (ElementGeometry::phys_nodes,
// from CurvedMesh::element_nodes_for_degree) [K][np][3] and curved flags [K].
void ref_level_nodes(void* h, double* nodes, int* curved) {
  auto* lvh = static_cast<RefLevel*>(h);
  const DgLevel& lv = *lvh->level;
  const int np = lv.refelem().n_basis();
  for (int e = 0; e < lv.n_elements(); ++e) {
    const auto& pn = lv.geom(e).phys_nodes;
    for (int i = 0; i < np; ++i)
      for (int d = 0; d < 3; ++d) nodes[(static_cast<size_t>(e) * np + i) * 3 + d] = pn[i][d];
    if (curved) curved[e] = lvh->cmesh->is_curved(e) ? 1 : 0;
  }
}

// Per-element operators (operators.cpp:123-167), row-major:
//  S [3][np][ncub], face_mass [np][nf], mass [np][np], mass_chol (column-major
//  as stored by the reference), for one element e.
void ref_level_operators(void* h, int e, double* s, double* face_mass, double* mass,
                         double* mass_chol) {
  const DgLevel& lv = *static_cast<RefLevel*>(h)->level;
  const auto& ops = lv.ops(e);
  const int np = ops.n_basis, ncub = ops.n_cub, nf = ops.n_face;
  for (int m = 0; m < 3; ++m)
    for (int i = 0; i < np; ++i)
      for (int q = 0; q < ncub; ++q) s[(static_cast<size_t>(m) * np + i) * ncub + q] = ops.s[m](i, q);
  for (int i = 0; i < np; ++i)
    for (int q = 0; q < nf; ++q) face_mass[static_cast<size_t>(i) * nf + q] = ops.face_mass(i, q);
  std::memcpy(mass, ops.mass.data(), sizeof(double) * ops.mass.size());
  std::memcpy(mass_chol, ops.mass_chol.data(), sizeof(double) * ops.mass_chol.size());
}

// Raw store access: data arrays are the SolutionStore raw() layout
// (e*5+c)*block + i, length K*5*block.
static void load_store(SolutionStore& s, const double* in) {
  std::memcpy(s.raw().data(), in, sizeof(double) * s.raw().size());
}
static void save_store(const SolutionStore& s, double* out) {
  std::memcpy(out, s.raw().data(), sizeof(double) * s.raw().size());
}

// bench.cpp:22-40 recipe (mt19937(seed), +/-0.05 jitter), restated here
// because the reference keeps it file-static.
void ref_random_admissible_store(void* h, unsigned seed, double* out) {
  const DgLevel& lv = *static_cast<RefLevel*>(h)->level;
  std::mt19937 gen(seed);
  std::uniform_real_distribution<double> jitter(-0.05, 0.05);
  SolutionStore store = lv.make_store();
  const int np = lv.refelem().n_basis();
  for (int e = 0; e < lv.n_elements(); ++e)
    for (int i = 0; i < np; ++i) {
      const double rho = 1.0 + jitter(gen);
      const Vec3 v{0.3 + jitter(gen), jitter(gen), jitter(gen)};
      const double p = 1.0 + jitter(gen);
      store.field(e, 0)[i] = rho;
      store.field(e, 1)[i] = rho * v.x;
      store.field(e, 2)[i] = rho * v.y;
      store.field(e, 3)[i] = rho * v.z;
      store.field(e, 4)[i] = p / 0.4 + 0.5 * rho * dot(v, v);
    }
  save_store(store, out);
}

int ref_compute_rhs(void* h, const ref_run_cfg* c, const double* freestream, const double* u_in,
                    double* rhs_out, char* err, size_t errn) {
  auto* lv = static_cast<RefLevel*>(h);
  try {
    SolutionStore u = lv->level->make_store();
    load_store(u, u_in);
    SolutionStore rhs = lv->level->make_store();
    compute_rhs(*lv->level, u, to_cfg(c), to_state(freestream), rhs, *lv->ws);
    save_store(rhs, rhs_out);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return status_of(e);
  }
}

int ref_interpolate_to_faces(void* h, const double* u_in, double* traces_out) {
  auto* lv = static_cast<RefLevel*>(h);
  SolutionStore u = lv->level->make_store();
  load_store(u, u_in);
  SolutionStore t = lv->level->make_trace_store();
  interpolate_to_faces(*lv->level, u, t);
  save_store(t, traces_out);
  return 0;
}

// nsteps x rk_step with the Carpenter-Kennedy scheme (rk.hpp:13-30).
int ref_rk_steps(void* h, const ref_run_cfg* c, const double* freestream, double dt, int nsteps,
                 double* u_io, double* res_io, char* err, size_t errn) {
  auto* lv = static_cast<RefLevel*>(h);
  try {
    SolutionStore u = lv->level->make_store();
    SolutionStore res = lv->level->make_store();
    load_store(u, u_io);
    load_store(res, res_io);
    const RunConfig cfg = to_cfg(c);
    const ConservedState fs = to_state(freestream);
    const RKScheme scheme = RKScheme::low_storage_rk4();
    for (int s = 0; s < nsteps; ++s) rk_step(*lv->level, u, res, cfg, fs, dt, scheme, *lv->ws);
    save_store(u, u_io);
    save_store(res, res_io);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return status_of(e);
  }
}

// The CPU baseline's timing entry: the stores are built once from u_io /
// res_io, then nsteps x rk_step run back to back and ONLY that loop is timed
// (seconds[s] = wall time of step s, steady_clock); the stores are copied
// back afterwards, outside the timed region.
int ref_rk_steps_timed(void* h, const ref_run_cfg* c, const double* freestream, double dt, int nsteps,
                       double* u_io, double* res_io, double* seconds, char* err, size_t errn) {
  auto* lv = static_cast<RefLevel*>(h);
  try {
    SolutionStore u = lv->level->make_store();
    SolutionStore res = lv->level->make_store();
    load_store(u, u_io);
    load_store(res, res_io);
    const RunConfig cfg = to_cfg(c);
    const ConservedState fs = to_state(freestream);
    const RKScheme scheme = RKScheme::low_storage_rk4();
    for (int s = 0; s < nsteps; ++s) {
      const auto t0 = std::chrono::steady_clock::now();
      rk_step(*lv->level, u, res, cfg, fs, dt, scheme, *lv->ws);
      seconds[s] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    save_store(u, u_io);
    save_store(res, res_io);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return status_of(e);
  }
}

// Viscosity + aux gradient of the last compute_rhs (solver.cpp:87-91).
// q_out [3][K*5*block] (only filled when the last RHS was viscous).
int ref_last_viscosity(void* h, double* eps_out, double* q_out) {
  auto* lv = static_cast<RefLevel*>(h);
  const auto& eps = current_viscosity(*lv->ws);
  std::memcpy(eps_out, eps.data(), sizeof(double) * eps.size());
  if (q_out) {
    const SolutionStore& q0 = aux_gradient(*lv->ws, 0);
    if (q0.n_elements() == 0) return 1;
    const size_t n = q0.raw().size();
    for (int m = 0; m < 3; ++m) save_store(aux_gradient(*lv->ws, m), q_out + m * n);
  }
  return 0;
}

int ref_compute_timestep(void* h, const ref_run_cfg* c, const double* u_in, const double* eps,
                         double* dt_out, char* err, size_t errn) {
  auto* lv = static_cast<RefLevel*>(h);
  try {
    SolutionStore u = lv->level->make_store();
    load_store(u, u_in);
    std::vector<double> ev;
    if (eps) ev.assign(eps, eps + lv->level->n_elements());
    *dt_out = compute_timestep(*lv->level, u, to_cfg(c), eps ? &ev : nullptr);
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return status_of(e);
  }
}

// run_steady (solver.cpp:594-676) on the mesh handle's CurvedMesh (the curved
// sidecar when present, else the straight mesh at the last schedule degree,
// as cmd_solve does, cli_ops.cpp:97-108). rows_out [max_rows][5] =
// (level, iteration, dt, residual, wall_seconds); u_out receives the final
// solution (capacity u_cap doubles).
int ref_run_steady(void* mesh_h, int bc_wall, int bc_far, const ref_run_cfg* c, const int* p_schedule,
                   int n_levels, const long* fixed, int n_fixed, double final_tol, double inter_tol,
                   int max_iters, int check_interval, int residual_kind, double dt_override,
                   const double* freestream, double* rows_out, int max_rows, int* n_rows, int* converged,
                   int* final_degree, double* u_out, long u_cap, char* err, size_t errn) {
  try {
    auto* m = static_cast<RefMesh*>(mesh_h);
    RunConfig cfg = to_cfg(c);
    cfg.p_schedule.assign(p_schedule, p_schedule + n_levels);
    cfg.fixed_iterations.assign(fixed, fixed + n_fixed);
    cfg.final_tolerance = final_tol;
    cfg.intermediate_tolerance = inter_tol;
    cfg.max_iterations_per_level = max_iters;
    cfg.check_interval = check_interval;
    cfg.residual_norm = residual_kind == 1 ? "l2" : "inf";
    cfg.dt_override = dt_override;
    const CurvedMesh cmesh = m->curved ? *m->curved : CurvedMesh(m->mesh, cfg.p_schedule.back());
    const BcMap bcs = {{"wall", static_cast<BcKind>(bc_wall)},
                       {"sphere", static_cast<BcKind>(bc_wall)},
                       {"farfield", static_cast<BcKind>(bc_far)},
                       {"symmetry", BcKind::Symmetry}};
    const SteadyResult r = run_steady(cmesh, bcs, cfg, to_state(freestream), nullptr);
    *n_rows = static_cast<int>(r.log.size());
    for (int i = 0; i < *n_rows && i < max_rows; ++i) {
      rows_out[5 * i + 0] = r.log[i].level;
      rows_out[5 * i + 1] = static_cast<double>(r.log[i].iteration);
      rows_out[5 * i + 2] = r.log[i].dt;
      rows_out[5 * i + 3] = r.log[i].residual;
      rows_out[5 * i + 4] = r.log[i].wall_seconds;
    }
    *converged = r.converged ? 1 : 0;
    *final_degree = r.final_degree;
    const auto& raw = r.solution.raw();
    if (static_cast<long>(raw.size()) > u_cap) throw ConfigError("ref_run_steady: u_out too small");
    std::memcpy(u_out, raw.data(), raw.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    copy_err(e, err, errn);
    return status_of(e);
  }
}

}  // extern "C"
