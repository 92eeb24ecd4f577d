/* cdg_gpu.h -- C ABI of the B200 (sm_100a) RKDG hot path.
 *
 * Drop-in boundary for the reference's solver kernels
 * (/root/reference/proj/core/include/cdg/solver.hpp:83-109). Every entry point
 * below replaces one reference interface; the C++ adapter a maintainer adds on
 * the reference side is shown in INTEGRATION.md.
 *
 *   cdg_gpu_level_create / _destroy  <- cdg::DgLevel (solver.hpp:52-79) +
 *                                       cdg::make_workspace (solver.hpp:84)
 *   cdg_gpu_set_state / _get_state   <- SolutionStore raw() layout
 *                                       (solution_store.hpp:16-77), flat copy
 *   cdg_gpu_interpolate_to_faces     <- cdg::interpolate_to_faces (solver.hpp:87-88)
 *   cdg_gpu_compute_rhs              <- cdg::compute_rhs (solver.hpp:94-96)
 *   cdg_gpu_rk_steps                 <- cdg::rk_step (solver.hpp:107-109), N steps
 *                                       device-resident
 *   cdg_gpu_viscosity                <- cdg::current_viscosity (solver.hpp:100)
 *   cdg_gpu_aux_gradient             <- cdg::aux_gradient (solver.hpp:103)
 *   cdg_gpu_timestep                 <- cdg::compute_timestep (solver.hpp:114-116)
 *   cdg_gpu_residual                 <- residual_norm (solver.cpp:572-590)
 *
 * Conventions
 *  - Plain pointers and sizes only. All arrays are row-major, float64 / int32.
 *  - Status codes mirror the reference exception types and the CLI exit codes
 *    (curveddg_main.cpp:10-31): 0 ok, 2 ConfigError, 3 NumericsError; 4 is a
 *    CUDA/runtime failure, 1 any other error. `err` (nullable) receives the
 *    reference's message text, e.g. "inadmissible state in element E at
 *    cubature node Q (rho=...)" (solver.cpp:377-379,425-426).
 *  - A level owns all device buffers; u and res stay device-resident between
 *    calls. Calls on one level are not re-entrant (the reference workspace is
 *    likewise single-caller, solver.cpp:80).
 *  - There is no CPU fallback: without a CUDA device every call fails with 4.
 */
#ifndef CDG_GPU_H
#define CDG_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDG_GPU_OK 0
#define CDG_GPU_ERR_OTHER 1
#define CDG_GPU_ERR_CONFIG 2
#define CDG_GPU_ERR_NUMERICS 3
#define CDG_GPU_ERR_CUDA 4

/* Boundary kinds: cdg::BcKind (euler.hpp:65) in declaration order. */
#define CDG_GPU_BC_SLIP_WALL 0
#define CDG_GPU_BC_FARFIELD 1
#define CDG_GPU_BC_SYMMETRY 2

/* Riemann solvers: RunConfig::riemann "llf" / "hllc" (solver.cpp:17-21). */
#define CDG_GPU_RIEMANN_LLF 0
#define CDG_GPU_RIEMANN_HLLC 1

/* The RunConfig fields the hot path reads (solver.hpp:18-36; viscosity.hpp:11-20). */
typedef struct cdg_gpu_run_config {
  int riemann;              /* CDG_GPU_RIEMANN_* */
  double gamma;             /* GasModel::gamma */
  int visc_enabled;         /* ViscosityModel::enabled */
  double eps0, kappa, s0_offset;
  int indicator_component;  /* conserved-variable index of the sensor */
  int jacobian_weighted;    /* 1: physical-space (J-weighted) indicator */
  double cfl;               /* RunConfig::cfl (timestep only) */
} cdg_gpu_run_config;

/* Everything the kernels need for one polynomial level (DgLevel). The caller
 * keeps ownership of every pointer; level_create copies what it needs. */
typedef struct cdg_gpu_level_desc {
  int degree;        /* p (1..8) */
  int n_basis;       /* N_p  = ReferenceElement::n_basis() */
  int n_cub;         /* N_cub = n_cub() */
  int n_face_quad;   /* N_g  = n_face_quad() (per face) */
  int n_elements;    /* K owned elements; rows 0..K-1 of every [K] array */
  int n_halo;        /* ghost elements K..K+n_halo-1 whose traces arrive by
                        halo exchange (multi-GPU); 0 on one GPU */
  int padded;        /* caller's SolutionStore layout: 1 = block pad16(N_p) */

  /* Reference-element tables, row-major (refelem.hpp:56-75). */
  const double *interp_cub;      /* [N_cub][N_p]  I_cub */
  const double *interp_face;     /* [4N_g][N_p]   I_g (face-major) */
  const double *deriv_r, *deriv_s, *deriv_t; /* [N_cub][N_p] D_m at cub nodes */
  const double *cub_weights;     /* [N_cub] */
  const double *face_weights;    /* [N_g]   2D rule, sums to 2 */
  const double *vandermonde_inv; /* [N_p][N_p] (sensor, viscosity.cpp:18) */

  /* Affine element geometry (ElementGeometry, operators.hpp:14-37, which is
   * constant per element/face on straight tets). */
  const double *metric;          /* [K][9]  cub_dr[q][m*3+i] = dr_m/dx_i */
  const double *jac;             /* [K]     cub_jac (det dx/dr) */
  const double *face_normal;     /* [K][4][3] outward unit normal per face */
  const double *face_sjac;       /* [K][4]  face_sjac per face */
  const double *h;               /* [K]     ElementGeometry::h() = 6V/A */

  /* Face coupling (FaceCoupling, solver.hpp:44-49). neighbor indexes
   * 0..K+n_halo-1, -1 on boundary faces. */
  const int *neighbor;           /* [K][4] */
  const int *neighbor_face;      /* [K][4] */
  const int *bc;                 /* [K][4] CDG_GPU_BC_* on boundary faces */
  const int *node_map;           /* [K][4][N_g] my g -> neighbour face node;
                                    may be NULL when face_code is given */
  const int *face_code;          /* [K][4] index into code_node_map, or NULL */
  const int *code_node_map;      /* [n_codes][N_g] */
  int n_codes;

  double freestream[5];          /* farfield ghost state (euler.cpp:157-158) */

  /* Curved (isoparametric) elements, CurvedMesh::is_curved (curved_mesh.hpp:
   * 14-51): their affine entries above are ignored; per-node geometry from
   * compute_mapping (operators.cpp:32-121) and the element mass inverse. */
  int n_curved;
  const int *curved_ids;         /* [Kc] element indices */
  const double *curved_jwr;      /* [Kc][N_cub][9] cub_jac*W*cub_dr (m*3+d) */
  const double *curved_face;     /* [Kc][4N_g][4] face_normal xyz, face_sjac*w */
  const double *curved_minv;     /* [Kc][N_p][N_p] (I_cub^T diag(JW) I_cub)^-1 */

  /* Physical-space (J-weighted) smoothness indicator, viscosity.cpp:28-45
   * (ViscosityModel::jacobian_weighted). Both may be NULL when that option is
   * never used: modal_cub defaults to I_cub * (V^-1)^-1 and curved_jac is
   * then required only for curved levels. */
  const double *modal_cub;       /* [N_cub][N_p] modal_basis_eval(p, cub_nodes) (refelem.hpp:21) */
  const double *curved_jac;      /* [Kc][N_cub] cub_jac of the curved elements */
} cdg_gpu_level_desc;

typedef struct cdg_gpu_level cdg_gpu_level;

/* Build device tables + workspace on `device`. Returns status. */
int cdg_gpu_level_create(const cdg_gpu_level_desc *desc, int device, cdg_gpu_level **out,
                         char *err, size_t errlen);
void cdg_gpu_level_destroy(cdg_gpu_level *lv);

/* Scalable setup for straight-sided meshes (replaces building the reference's
 * DgLevel, solver.cpp:97-179, ~140 KB per element): the affine geometry and
 * the perm-based face-node pairing are computed inside the library from the
 * caller's Mesh (mesh.hpp:23-57) in O(K). `tables` supplies the reference-element
 * tables, degree / sizes, padded, freestream (its geometry / coupling fields
 * are ignored); `mesh` the connectivity. Equivalent to cdg_gpu_level_create
 * with the reference's nearest-point node_map (conforming faces, symmetric
 * face rules). */
typedef struct cdg_gpu_mesh_desc {
  int n_vertices;
  const double *vertices;     /* [nv][3] Mesh::vertices */
  int n_elements;             /* K owned elements */
  int n_halo;                 /* ghost elements (multi-GPU shards), 0 otherwise */
  const int *tets;            /* [K][4] Mesh::tets (reference vertex order) */
  const int *neighbor;        /* [K][4] FaceLink.other.element, -1 on boundary faces */
  const int *neighbor_face;   /* [K][4] FaceLink.other.local_face */
  const int *face_perm;       /* [K][4][3] FaceLink.perm: other_face_vertex[perm[i]] == self_face_vertex[i] */
  const int *bc;              /* [K][4] CDG_GPU_BC_* on boundary faces (BcMap of the face's tag) */
  const double *face_nodes;   /* [N_g][3] ReferenceElement::face_nodes() of face 0 */
} cdg_gpu_mesh_desc;
int cdg_gpu_level_create_from_mesh(const cdg_gpu_level_desc *tables, const cdg_gpu_mesh_desc *mesh, int device,
                                   cdg_gpu_level **out, char *err, size_t errlen);

/* Sizes: [0]=K [1]=N_p [2]=N_cub [3]=N_g [4]=caller block [5]=caller trace
 * block [6]=device block [7]=n_halo. */
void cdg_gpu_level_sizes(const cdg_gpu_level *lv, int *sizes);

/* State transfer in the caller's SolutionStore raw() layout
 * ((e*5+c)*block + i over the K owned elements). res may be NULL (zeroed on
 * set, skipped on get). Host pointers may be pageable or pinned. */
int cdg_gpu_set_state(cdg_gpu_level *lv, const double *u, const double *res);
int cdg_gpu_get_state(cdg_gpu_level *lv, double *u, double *res);
/* Same as set_state with DEVICE source pointers (caller layout). */
int cdg_gpu_set_state_device(cdg_gpu_level *lv, const double *u, const double *res);
/* Device pointers of the resident u / res / traces buffers (device layout,
 * block = sizes[6]); lets a caller that already holds device memory skip the
 * host round trip. */
int cdg_gpu_device_buffers(cdg_gpu_level *lv, double **u, double **res, double **traces);

/* traces = I_g u for the resident state; out: [K][5][pad16(4N_g) or 4N_g]. */
int cdg_gpu_interpolate_to_faces(cdg_gpu_level *lv, double *traces_out);

/* rhs = RHS(u) for the resident state (no update). rhs_out (host, caller
 * layout) may be NULL to leave it on device. */
int cdg_gpu_compute_rhs(cdg_gpu_level *lv, const cdg_gpu_run_config *cfg, double *rhs_out,
                        char *err, size_t errlen);

/* nsteps low-storage RK steps on the resident (u, res):
 *   for stage i: res = a[i] res + dt RHS(u); u += b[i] res   (solver.cpp:469-492) */
int cdg_gpu_rk_steps(cdg_gpu_level *lv, const cdg_gpu_run_config *cfg, int nsteps, double dt,
                     const double a[5], const double b[5], char *err, size_t errlen);

/* Per-element eps of the last viscous RHS (current_viscosity). eps_out [K]. */
int cdg_gpu_viscosity(cdg_gpu_level *lv, double *eps_out);
/* q_m of the last viscous RHS (aux_gradient), caller layout; m in 0..2. */
int cdg_gpu_aux_gradient(cdg_gpu_level *lv, int m, double *q_out);

/* CFL time step for the resident u (compute_timestep, solver.cpp:494-526);
 * use_viscosity=1 applies the h^2/(eps (p+1)^4) limit with the last eps. */
int cdg_gpu_timestep(cdg_gpu_level *lv, const cdg_gpu_run_config *cfg, int use_viscosity,
                     double *dt_out, char *err, size_t errlen);

/* Snapshot u into the level's `before` buffer; then residual_norm(u, before,
 * dt, kind) with kind 0 = "inf", 1 = "l2" (solver.cpp:572-590). */
int cdg_gpu_snapshot(cdg_gpu_level *lv);
int cdg_gpu_residual(cdg_gpu_level *lv, int kind, double dt, double *out);

/* ---- device-resident run_steady (solver.cpp:594-676) --------------------------
 * The reference's per-level loop with the state on the device: RK steps run
 * back to back (graph replays) and the host synchronises only at the check
 * iterations, where it reads back one residual and one time step. */
typedef struct cdg_gpu_steady_params {
  long max_iterations;    /* RunConfig::max_iterations_per_level */
  long fixed_iterations;  /* RunConfig::fixed_iterations[level], or <= 0 */
  int check_interval;     /* RunConfig::check_interval */
  int residual_kind;      /* RunConfig::residual_norm: 0 "inf", 1 "l2" */
  double tolerance;       /* final_tolerance on the last level, else intermediate_tolerance */
  double dt_override;     /* RunConfig::dt_override (> 0 replaces the CFL formula) */
  int degree;             /* p of this level (divergence message) */
} cdg_gpu_steady_params;

/* u = freestream_store(level, freestream) (solver.cpp:559-568), res = 0. */
int cdg_gpu_fill_freestream(cdg_gpu_level *lv);
/* to.u = p_refine_embed(from.u) (solver.cpp:528-549) with the caller's
 * embedding matrix embed[np_to][np_from] = V_to[:, :np_from] V_from^-1;
 * to.res = 0. Both levels on the same device, same element count. */
int cdg_gpu_p_refine_embed(cdg_gpu_level *to, const cdg_gpu_level *from, const double *embed);
/* One level of run_steady (solver.cpp:622-668). rows receives
 * (iteration, dt, residual) for every check iteration (at most max_rows);
 * *converged = 1 when the level stopped on its tolerance. A residual above
 * 1e6 x the first one returns 3 with the reference's "run_steady: divergence
 * detected at p=P iteration I (residual R)" text. */
int cdg_gpu_run_level(cdg_gpu_level *lv, const cdg_gpu_run_config *cfg, const cdg_gpu_steady_params *sp,
                      double *rows, int max_rows, int *n_rows, int *converged, char *err, size_t errlen);

/* Same loop, with every check row also handed to on_row(user, iteration, dt,
 * residual) the moment it is computed (the reference emits rows live from
 * run_steady, solver.cpp:643-647). on_row may be NULL. */
typedef void (*cdg_gpu_row_fn)(void *user, long iteration, double dt, double residual);
int cdg_gpu_run_level_live(cdg_gpu_level *lv, const cdg_gpu_run_config *cfg, const cdg_gpu_steady_params *sp,
                           cdg_gpu_row_fn on_row, void *user, double *rows, int max_rows, int *n_rows,
                           int *converged, char *err, size_t errlen);

/* ---- multi-GPU halo plumbing (one process per GPU) --------------------------
 * send_elem_face[i] = element*4+face of an owned element whose face trace
 * (5*N_g values) is packed into row i of the caller-owned DEVICE buffer
 * send_buf [n_send][5][N_g]; recv_elem_face[i] names the ghost element
 * (K..K+n_halo-1) and face that row i of recv_buf lands in. The transport
 * (NCCL send/recv over NVLink) is driven by the caller on cdg_gpu_stream(). */
int cdg_gpu_halo_setup(cdg_gpu_level *lv, int n_send, const int *send_elem_face, int n_recv,
                       const int *recv_elem_face, double *send_buf, double *recv_buf);
int cdg_gpu_halo_pack(cdg_gpu_level *lv);
int cdg_gpu_halo_unpack(cdg_gpu_level *lv);
/* Runs one RK stage in split form for overlap: trace kernel, then (caller
 * exchanges halos) then RHS+update. phase 0 = traces + pack, phase 1 =
 * unpack + RHS + update for stage `stage`. Overlapped form: phase 2 = RHS +
 * update of the interior tiles (no ghost neighbour; launch it while the halo
 * exchange is in flight), phase 3 = unpack + RHS + update of the halo tiles
 * (after the exchange). 0,1 and 0,2,3 give bitwise identical states. */
int cdg_gpu_rk_stage_phase(cdg_gpu_level *lv, const cdg_gpu_run_config *cfg, int stage, int phase,
                           double dt, const double a[5], const double b[5], char *err,
                           size_t errlen);

/* ---- multi-rank driver (one shard per rank) -----------------------------------
 * The reference runs one process over the whole mesh (rk_step / compute_rhs /
 * compute_timestep / residual_norm / run_steady, solver.cpp:239-676); these
 * entry points run the same loop over R shards -- cdg_gpu_level's with ghost
 * elements K..K+n_halo-1 -- with one halo exchange of face traces per RK stage
 * (inviscid) or per viscous phase (U traces + sqrt(eps), then the q_m traces),
 * the interior tiles overlapping the transfer, and all-rank MIN / MAX / SUM
 * reductions for the time step, the viscous gate and the residual. Results
 * are bitwise identical to the single-level run (l2 residual: to rounding).
 *
 * cdg_gpu_halo_define: the shard's halo rows, peer by peer: rows
 * [sum(send_count[<i]), +send_count[i]) of send_elem_face go to rank
 * peer_rank[i], likewise recv. Both sides list a shared face in the same
 * (canonical) order. The library owns the transfer buffers. */
typedef struct cdg_gpu_comm cdg_gpu_comm;
int cdg_gpu_halo_define(cdg_gpu_level *lv, int n_peers, const int *peer_rank, const int *send_count,
                        const int *recv_count, const int *send_elem_face, const int *recv_elem_face);
/* NCCL transport, one process per GPU: rank 0 calls cdg_gpu_comm_unique_id and
 * the caller broadcasts the 128 bytes (MPI, torch.distributed, a file); every
 * rank then creates its communicator over its shard. libnccl.so.2 is loaded at
 * run time (status 2 when absent). */
int cdg_gpu_comm_unique_id(unsigned char id[128], char *err, size_t errlen);
int cdg_gpu_comm_create_nccl(cdg_gpu_level *shard, const unsigned char id[128], int rank, int nranks,
                             cdg_gpu_comm **out, char *err, size_t errlen);
/* In-process transport: one host thread drives all nranks shards (levels[r]
 * is rank r; on one GPU or several, peer copies over NVLink). */
int cdg_gpu_comm_create_local(int nranks, cdg_gpu_level *const *levels, cdg_gpu_comm **out, char *err,
                              size_t errlen);
void cdg_gpu_comm_destroy(cdg_gpu_comm *comm);
/* rk_steps over every shard of the communicator (viscous or not). */
int cdg_gpu_comm_rk_steps(cdg_gpu_comm *comm, const cdg_gpu_run_config *cfg, int nsteps, double dt,
                          const double a[5], const double b[5], char *err, size_t errlen);
/* global compute_timestep (MIN over ranks), snapshot, residual_norm (inf: MAX,
 * l2: SUM of squares), fill_freestream, one run_steady level. */
int cdg_gpu_comm_timestep(cdg_gpu_comm *comm, const cdg_gpu_run_config *cfg, int use_viscosity, double *dt_out,
                          char *err, size_t errlen);
int cdg_gpu_comm_snapshot(cdg_gpu_comm *comm);
int cdg_gpu_comm_residual(cdg_gpu_comm *comm, int kind, double dt, double *out);
int cdg_gpu_comm_fill_freestream(cdg_gpu_comm *comm);
int cdg_gpu_comm_run_level(cdg_gpu_comm *comm, const cdg_gpu_run_config *cfg, const cdg_gpu_steady_params *sp,
                           cdg_gpu_row_fn on_row, void *user, double *rows, int max_rows, int *n_rows,
                           int *converged, char *err, size_t errlen);
/* halo exchanges issued so far (evidence counter) */
int cdg_gpu_comm_exchange_count(const cdg_gpu_comm *comm);

/* 1 when cdg_gpu_rk_steps runs the fused-trace path (the RHS kernel's epilogue
 * writes the next stage's face traces; one trace kernel seeds each call),
 * else 0. Informational (bench roofline accounting). */
int cdg_gpu_fused_traces(const cdg_gpu_level *lv);

/* Replace the farfield ghost state (compute_rhs/rk_step take it per call,
 * solver.hpp:94-109). */
int cdg_gpu_set_freestream(cdg_gpu_level *lv, const double *freestream5);

/* Cap the grid of the persistent (grid-stride) RHS / aux kernels at max_ctas
 * CTAs (0 restores the default: SM count x resident CTAs per SM). Results do
 * not depend on the grid (each element's arithmetic is fixed); tests use a
 * small cap to drive small meshes through the many-tiles-per-CTA regime of a
 * production-size launch. */
int cdg_gpu_set_max_ctas(cdg_gpu_level *lv, int max_ctas);

/* Kernel family of a level. DEFAULT: the per-order choice compiled into the
 * kernel-set table (row-per-warp / warp-tile kernels with fused traces where
 * measured fastest; at p <= 2 on single-shard straight meshes
 * the neighbour-state kernel, which reads the neighbours' nodal states
 * instead of stored traces and so agrees with the other paths to rounding
 * only). GENERIC: the CTA kernels (k_rhs, k_rhs_curved) for every element,
 * the p >= 6 path. TRACED: DEFAULT without the neighbour-state kernel (every
 * stage through stored traces, the paths that agree bit for bit). Tests
 * cross-check the families against each other and against the reference at
 * every order. */
#define CDG_GPU_PATH_DEFAULT 0
#define CDG_GPU_PATH_GENERIC 1
#define CDG_GPU_PATH_TRACED 2
int cdg_gpu_set_kernel_path(cdg_gpu_level *lv, int path);

/* HLLC -> LLF fallbacks counted since the level was created (degenerate wave
 * speed estimates or a non-finite contact speed; RhsWorkspace::hllc_fallbacks,
 * solver.cpp:52,436, euler.cpp:99-110). */
int cdg_gpu_hllc_fallbacks(cdg_gpu_level *lv, long long *count);

/* CUDA stream (cudaStream_t) the level launches on. */
void *cdg_gpu_stream(cdg_gpu_level *lv);
/* Kernel launches issued by this level since creation (evidence counter). */
long long cdg_gpu_launch_count(const cdg_gpu_level *lv);
/* Device-time of the last rk_steps call split by kernel: [0]=trace kernel ms
 * [1]=rhs kernel ms [2]=launches, measured with cudaEvents on the level's
 * stream when profiling is enabled. */
int cdg_gpu_set_profiling(cdg_gpu_level *lv, int enabled);
int cdg_gpu_last_profile(cdg_gpu_level *lv, double *out3);

/* Name of the affine RHS + update kernel the level runs (evidence labels). */
const char *cdg_gpu_rhs_kernel(const cdg_gpu_level *lv);
/* Name of the curved-element RHS + update kernel ("" without curved elements). */
const char *cdg_gpu_curved_kernel(const cdg_gpu_level *lv);
const char *cdg_gpu_version(void);
/* FP64 roofline denominators measured on `device` (TFLOP/s): out[0] DMMA
 * m16n8k4, out[1] DFMA, out[2] DMMA m16n8k8, out[3] DMMA m16n8k16. */
int cdg_gpu_measure_fp64_peak(int device, double *out);

#ifdef __cplusplus
}
#endif

#endif /* CDG_GPU_H */
