/* ORACLE TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's
 * RK-stage hot path (parity checker; never linked into the product).
 *
 * Follows, loop by loop and in the same floating-point evaluation order:
 *   compute_mapping / build_operators / mass_solve   operators.cpp:8-167
 *   PaddedMatrix gemv / gemv_acc / gemv_sub (4-column unroll) padded.hpp:42-85
 *   DgLevel face pairing (nearest physical point)    solver.cpp:142-178
 *   interpolate_to_faces / gather_pair               solver.cpp:200-237
 *   compute_element_viscosities / compute_aux_gradient solver.cpp:239-321
 *   compute_rhs / rk_step / compute_timestep          solver.cpp:325-526
 *   pressure/admissible/flux/llf/hllc/boundary_state  euler.cpp:7-161
 *   smoothness_indicator (Parseval) / viscosity_amount viscosity.cpp:7-56
 * Reference-element tables and element nodes come from the caller.
 */
#ifndef CDG_ORACLE_H
#define CDG_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cdgo_desc {
  int p, np, ncub, ng, K, padded;
  /* row-major reference tables */
  const double *icub, *ig;             /* [ncub][np], [4ng][np] */
  const double *dr, *ds, *dt;          /* [ncub][np] */
  const double *fdr, *fds, *fdt;       /* [4ng][np] */
  const double *cub_w, *face_w;        /* [ncub], [ng] */
  const double *vinv;                  /* [np][np] */
  /* mesh */
  const double *elem_nodes;            /* [K][np][3] physical collocation nodes */
  const double *pair_scale;            /* [K] cbrt(|signed volume|) */
  const int *neighbor, *neighbor_face; /* [K][4] */
  const int *bc;                       /* [K][4] 0 wall 1 farfield 2 symmetry */
  double freestream[5];
  double period[3];                    /* > 0: periodic box length per axis (minimum-image pairing) */
} cdgo_desc;

typedef struct cdgo_cfg {
  int riemann;
  double gamma;
  int visc_enabled;
  double eps0, kappa, s0_offset;
  int indicator_component;
  int jacobian_weighted;
  double cfl;
} cdgo_cfg;

typedef struct cdgo_level cdgo_level;

int cdgo_level_create(const cdgo_desc *d, cdgo_level **out, char *err, size_t errlen);
void cdgo_level_destroy(cdgo_level *lv);
/* sizes: [0]=K [1]=block [2]=trace block */
void cdgo_level_sizes(const cdgo_level *lv, int *sizes);
/* per-element geometry exported for cross-checks: h [K], node_map [K][4][ng] */
void cdgo_level_export(const cdgo_level *lv, double *h, int *node_map);

int cdgo_interpolate_to_faces(cdgo_level *lv, const double *u, double *traces);
int cdgo_compute_rhs(cdgo_level *lv, const cdgo_cfg *cfg, const double *u, double *rhs, char *err,
                     size_t errlen);
int cdgo_rk_steps(cdgo_level *lv, const cdgo_cfg *cfg, double dt, int nsteps, const double *a,
                  const double *b, double *u, double *res, char *err, size_t errlen);
int cdgo_compute_timestep(cdgo_level *lv, const cdgo_cfg *cfg, const double *u, const double *eps,
                          double *dt, char *err, size_t errlen);
/* eps [K] and q [3][K*5*block] of the last RHS evaluation (q only if viscous) */
int cdgo_last_viscosity(cdgo_level *lv, double *eps, double *q);

#ifdef __cplusplus
}
#endif

#endif
