/* ORACLE TEST INFRASTRUCTURE ONLY -- see cdg_oracle.h for the mapping to the
 * reference sources. Single-threaded, no dependencies beyond libm. */
#include "cdg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NF5 5

struct cdgo_level {
  int p, np, ncub, ng, nf, K, block, tblock;
  double *icub, *ig, *cub_w, *face_w, *vinv;
  /* per element operators (operators.hpp:42-56) */
  double *S;      /* [K][3][np][ncub]  (i, q) */
  double *fmass;  /* [K][np][nf] */
  double *chol;   /* [K][np*np] column-major L (mass_chol[j*n+i] = L(i,j)) */
  double *normal; /* [K][nf][3] */
  double *h;      /* [K] */
  int *nb, *nbf, *bc, *nmap;
  double fs[5];
  /* workspace (RhsWorkspace, solver.cpp:43-70) */
  double *traces, *rhsbuf, *qn, *qt, *eps, *seps;
  int viscous_active, have_q;
  char errmsg[512];
  int failed;
};

static int pad16(int n) { return 16 * ((n + 15) / 16); }

static void set_err(char *err, size_t n, const char *msg) {
  if (err && n) {
    strncpy(err, msg, n - 1);
    err[n - 1] = 0;
  }
}

/* ---- PaddedMatrix gemv family (padded.hpp:42-85); A row-major [rows][cols],
 * the 4-column pass order of the reference is reproduced exactly. ---------- */
static void gemv_acc(const double *a, int rows, int cols, const double *x, double *y) {
  int j = 0;
  for (; j + 4 <= cols; j += 4) {
    const double x0 = x[j], x1 = x[j + 1], x2 = x[j + 2], x3 = x[j + 3];
    for (int i = 0; i < rows; ++i) {
      const double *r = a + (size_t)i * cols + j;
      y[i] += r[0] * x0 + r[1] * x1 + r[2] * x2 + r[3] * x3;
    }
  }
  for (; j < cols; ++j) {
    const double xj = x[j];
    for (int i = 0; i < rows; ++i) y[i] += a[(size_t)i * cols + j] * xj;
  }
}
static void gemv_sub(const double *a, int rows, int cols, const double *x, double *y) {
  int j = 0;
  for (; j + 4 <= cols; j += 4) {
    const double x0 = x[j], x1 = x[j + 1], x2 = x[j + 2], x3 = x[j + 3];
    for (int i = 0; i < rows; ++i) {
      const double *r = a + (size_t)i * cols + j;
      y[i] -= r[0] * x0 + r[1] * x1 + r[2] * x2 + r[3] * x3;
    }
  }
  for (; j < cols; ++j) {
    const double xj = x[j];
    for (int i = 0; i < rows; ++i) y[i] -= a[(size_t)i * cols + j] * xj;
  }
}
static void gemv(const double *a, int rows, int cols, const double *x, double *y) {
  for (int i = 0; i < rows; ++i) y[i] = 0.0;
  gemv_acc(a, rows, cols, x, y);
}

/* ElementOperators::mass_solve (operators.cpp:8-22) */
static void mass_solve(const double *l, int n, const double *b, double *x) {
  for (int i = 0; i < n; ++i) {
    double sum = b[i];
    for (int j = 0; j < i; ++j) sum -= l[j * n + i] * x[j];
    x[i] = sum / l[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double sum = x[i];
    for (int j = i + 1; j < n; ++j) sum -= l[i * n + j] * x[j];
    x[i] = sum / l[i * n + i];
  }
}

/* ---- Euler (euler.cpp) ----------------------------------------------------- */
typedef struct { double rho, mx, my, mz, E; } st5;
static double st_get(const st5 *s, int c) {
  return c == 0 ? s->rho : c == 1 ? s->mx : c == 2 ? s->my : c == 3 ? s->mz : s->E;
}
static double dot3(double ax, double ay, double az, double bx, double by, double bz) {
  return ax * bx + ay * by + az * bz;
}
static int admissible(const st5 *u, double g) {
  if (u->rho <= 0.0) return 0;
  return (u->E - dot3(u->mx, u->my, u->mz, u->mx, u->my, u->mz) / (2.0 * u->rho)) > 0.0 && g > 1.0;
}
static double pressure(const st5 *u, double g) {
  return (g - 1.0) * (u->E - dot3(u->mx, u->my, u->mz, u->mx, u->my, u->mz) / (2.0 * u->rho));
}
static void flux_dot_n(const st5 *u, double g, const double *n, double *f) {
  const double p = pressure(u, g);
  const double vn = dot3(u->mx, u->my, u->mz, n[0], n[1], n[2]) / u->rho;
  f[0] = u->rho * vn;
  f[1] = u->mx * vn + p * n[0];
  f[2] = u->my * vn + p * n[1];
  f[3] = u->mz * vn + p * n[2];
  f[4] = vn * (u->E + p);
}
static double max_wavespeed(const st5 *u, double g, const double *n) {
  const double p = pressure(u, g);
  const double c = sqrt(g * p / u->rho);
  return fabs(dot3(u->mx, u->my, u->mz, n[0], n[1], n[2]) / u->rho) + c;
}
static void llf_flux(const st5 *um, const st5 *up, const double *n, double g, double *out) {
  const double a = max_wavespeed(um, g, n), b = max_wavespeed(up, g, n);
  const double lambda = a > b ? a : b; /* std::max(a, b) */
  double fm[5], fp[5];
  flux_dot_n(um, g, n, fm);
  flux_dot_n(up, g, n, fp);
  for (int c = 0; c < 5; ++c) out[c] = 0.5 * (fm[c] + fp[c]) - 0.5 * lambda * (st_get(up, c) - st_get(um, c));
}
static void hllc_flux(const st5 *um, const st5 *up, const double *n, double g, double *out) {
  const double pl = pressure(um, g), pr = pressure(up, g);
  const double vl[3] = {um->mx / um->rho, um->my / um->rho, um->mz / um->rho};
  const double vr[3] = {up->mx / up->rho, up->my / up->rho, up->mz / up->rho};
  const double unl = dot3(vl[0], vl[1], vl[2], n[0], n[1], n[2]);
  const double unr = dot3(vr[0], vr[1], vr[2], n[0], n[1], n[2]);
  const double cl = sqrt(g * pl / um->rho), cr = sqrt(g * pr / up->rho);
  const double sl_ = sqrt(um->rho), sr_ = sqrt(up->rho);
  double vroe[3];
  for (int d = 0; d < 3; ++d) vroe[d] = (sl_ * vl[d] + sr_ * vr[d]) / (sl_ + sr_);
  const double hl = (um->E + pl) / um->rho, hr = (up->E + pr) / up->rho;
  const double h_roe = (sl_ * hl + sr_ * hr) / (sl_ + sr_);
  const double c2_roe = (g - 1.0) * (h_roe - 0.5 * dot3(vroe[0], vroe[1], vroe[2], vroe[0], vroe[1], vroe[2]));
  const double un_roe = dot3(vroe[0], vroe[1], vroe[2], n[0], n[1], n[2]);
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
    llf_flux(um, up, n, g, out);
    return;
  }
  const double s_star = (pr - pl + um->rho * unl * (s_left - unl) - up->rho * unr * (s_right - unr)) /
                        (um->rho * (s_left - unl) - up->rho * (s_right - unr));
  if (!isfinite(s_star)) {
    llf_flux(um, up, n, g, out);
    return;
  }
  if (0.0 <= s_left) {
    flux_dot_n(um, g, n, out);
    return;
  }
  if (0.0 >= s_right) {
    flux_dot_n(up, g, n, out);
    return;
  }
  const int left = 0.0 <= s_star;
  const st5 *u = left ? um : up;
  const double un_k = left ? unl : unr, p_k = left ? pl : pr, s_k = left ? s_left : s_right;
  const double factor = u->rho * (s_k - un_k) / (s_k - s_star);
  const double v[3] = {u->mx / u->rho, u->my / u->rho, u->mz / u->rho};
  double star[5];
  star[0] = factor;
  for (int d = 0; d < 3; ++d) star[1 + d] = factor * (v[d] + (s_star - un_k) * n[d]);
  star[4] = factor * (u->E / u->rho + (s_star - un_k) * (s_star + p_k / (u->rho * (s_k - un_k))));
  double f[5];
  flux_dot_n(u, g, n, f);
  for (int c = 0; c < 5; ++c) out[c] = f[c] + s_k * (star[c] - st_get(u, c));
}
static st5 boundary_state(const st5 *in, const double *n, int kind, const double *fs) {
  if (kind == 1) {
    st5 s = {fs[0], fs[1], fs[2], fs[3], fs[4]};
    return s;
  }
  st5 gh = *in;
  const double mn = dot3(in->mx, in->my, in->mz, n[0], n[1], n[2]);
  gh.mx = in->mx - 2.0 * mn * n[0];
  gh.my = in->my - 2.0 * mn * n[1];
  gh.mz = in->mz - 2.0 * mn * n[2];
  return gh;
}

/* ---- level construction (compute_mapping / build_operators / pairing) ---- */
static void mat3_fill(double f[3][3], const double *dxr, const double *dxs, const double *dxt) {
  for (int i = 0; i < 3; ++i) {
    f[i][0] = dxr[i];
    f[i][1] = dxs[i];
    f[i][2] = dxt[i];
  }
}
static double det3(double m[3][3]) {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}
static void inv3(double m[3][3], double det, double o[3][3]) {
  o[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
  o[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
  o[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
  o[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
  o[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
  o[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
  o[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / det;
  o[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
  o[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
}
/* out[q][3] = T[q][np] * X[np][3] */
static void tab_times_x(const double *t, int rows, int np, const double *x, double *out) {
  for (int q = 0; q < rows; ++q)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int k = 0; k < np; ++k) s += t[(size_t)q * np + k] * x[k * 3 + c];
      out[q * 3 + c] = s;
    }
}

static const double kVerts[4][3] = {{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}};
static const int kFaceVerts[4][3] = {{0, 2, 1}, {0, 1, 3}, {1, 2, 3}, {0, 3, 2}};

int cdgo_level_create(const cdgo_desc *d, cdgo_level **out, char *err, size_t errlen) {
  *out = NULL;
  cdgo_level *lv = (cdgo_level *)calloc(1, sizeof(cdgo_level));
  const int np = d->np, ncub = d->ncub, ng = d->ng, nf = 4 * ng, K = d->K;
  lv->p = d->p;
  lv->np = np;
  lv->ncub = ncub;
  lv->ng = ng;
  lv->nf = nf;
  lv->K = K;
  lv->block = d->padded ? pad16(np) : np;
  lv->tblock = d->padded ? pad16(nf) : nf;
  memcpy(lv->fs, d->freestream, sizeof(lv->fs));
#define DUP(dst, src, n)                                   \
  do {                                                     \
    dst = (double *)malloc(sizeof(double) * (size_t)(n));  \
    memcpy(dst, src, sizeof(double) * (size_t)(n));        \
  } while (0)
  DUP(lv->icub, d->icub, (size_t)ncub * np);
  DUP(lv->ig, d->ig, (size_t)nf * np);
  DUP(lv->cub_w, d->cub_w, ncub);
  DUP(lv->face_w, d->face_w, ng);
  DUP(lv->vinv, d->vinv, (size_t)np * np);
  lv->S = (double *)malloc(sizeof(double) * (size_t)K * 3 * np * ncub);
  lv->fmass = (double *)malloc(sizeof(double) * (size_t)K * np * nf);
  lv->chol = (double *)malloc(sizeof(double) * (size_t)K * np * np);
  lv->normal = (double *)malloc(sizeof(double) * (size_t)K * nf * 3);
  lv->h = (double *)malloc(sizeof(double) * K);
  double *face_phys = (double *)malloc(sizeof(double) * (size_t)K * nf * 3);
  double *cxr = malloc(sizeof(double) * ncub * 3), *cxs = malloc(sizeof(double) * ncub * 3),
         *cxt = malloc(sizeof(double) * ncub * 3);
  double *fxr = malloc(sizeof(double) * nf * 3), *fxs = malloc(sizeof(double) * nf * 3),
         *fxt = malloc(sizeof(double) * nf * 3);
  double *cub_dr = malloc(sizeof(double) * ncub * 9), *cub_jac = malloc(sizeof(double) * ncub);
  double *sjac = malloc(sizeof(double) * nf), *m = malloc(sizeof(double) * np * np);
  double *l = malloc(sizeof(double) * np * np), *tmp = malloc(sizeof(double) * np * ncub);
  int status = 0;
  char msg[512];
  for (int e = 0; e < K && !status; ++e) {
    const double *x = d->elem_nodes + (size_t)e * np * 3;
    /* compute_mapping (operators.cpp:32-121) */
    tab_times_x(d->dr, ncub, np, x, cxr);
    tab_times_x(d->ds, ncub, np, x, cxs);
    tab_times_x(d->dt, ncub, np, x, cxt);
    for (int q = 0; q < ncub; ++q) {
      double f[3][3], inv[3][3];
      mat3_fill(f, cxr + 3 * q, cxs + 3 * q, cxt + 3 * q);
      const double det = det3(f);
      if (det <= 1e-14) {
        snprintf(msg, sizeof msg, "inverted element %d: mapping Jacobian %f at quadrature node %d", e, det, q);
        status = 3;
        break;
      }
      cub_jac[q] = det;
      inv3(f, det, inv);
      for (int mm = 0; mm < 3; ++mm)
        for (int i = 0; i < 3; ++i) cub_dr[q * 9 + mm * 3 + i] = inv[mm][i];
    }
    if (status) break;
    double volume = 0.0;
    for (int q = 0; q < ncub; ++q) volume += d->cub_w[q] * cub_jac[q];
    tab_times_x(d->fdr, nf, np, x, fxr);
    tab_times_x(d->fds, nf, np, x, fxs);
    tab_times_x(d->fdt, nf, np, x, fxt);
    tab_times_x(d->ig, nf, np, x, face_phys + (size_t)e * nf * 3);
    double area = 0.0;
    for (int f = 0; f < 4; ++f) {
      const int *fv = kFaceVerts[f];
      double ra[3], rb[3];
      for (int c = 0; c < 3; ++c) {
        ra[c] = 0.5 * (kVerts[fv[1]][c] - kVerts[fv[0]][c]);
        rb[c] = 0.5 * (kVerts[fv[2]][c] - kVerts[fv[0]][c]);
      }
      for (int g = 0; g < ng; ++g) {
        const int q = f * ng + g;
        double fw[3][3];
        mat3_fill(fw, fxr + 3 * q, fxs + 3 * q, fxt + 3 * q);
        const double det = det3(fw);
        if (det <= 1e-14) {
          snprintf(msg, sizeof msg, "inverted element %d: mapping Jacobian %f at quadrature node %d", e, det, q);
          status = 3;
          break;
        }
        double xa[3], xb[3];
        for (int i = 0; i < 3; ++i) {
          xa[i] = fw[i][0] * ra[0] + fw[i][1] * ra[1] + fw[i][2] * ra[2];
          xb[i] = fw[i][0] * rb[0] + fw[i][1] * rb[1] + fw[i][2] * rb[2];
        }
        const double n0 = xa[1] * xb[2] - xa[2] * xb[1], n1 = xa[2] * xb[0] - xa[0] * xb[2],
                     n2 = xa[0] * xb[1] - xa[1] * xb[0];
        const double s = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
        if (s <= 1e-14) {
          snprintf(msg, sizeof msg, "degenerate face mapping on element %d", e);
          status = 3;
          break;
        }
        sjac[q] = s;
        double *nrm = lv->normal + ((size_t)e * nf + q) * 3;
        nrm[0] = n0 / s;
        nrm[1] = n1 / s;
        nrm[2] = n2 / s;
        area += d->face_w[g] * s;
      }
      if (status) break;
    }
    if (status) break;
    lv->h[e] = 6.0 * volume / area;
    /* build_operators (operators.cpp:123-167) */
    const double *dm[3] = {d->dr, d->ds, d->dt};
    for (int dim = 0; dim < 3; ++dim) {
      for (int i = 0; i < np * ncub; ++i) tmp[i] = 0.0;
      for (int mm = 0; mm < 3; ++mm)
        for (int i = 0; i < np; ++i)
          for (int q = 0; q < ncub; ++q) tmp[i * ncub + q] += dm[mm][(size_t)q * np + i] * cub_dr[q * 9 + mm * 3 + dim];
      double *S = lv->S + ((size_t)e * 3 + dim) * np * ncub;
      for (int i = 0; i < np; ++i)
        for (int q = 0; q < ncub; ++q) S[i * ncub + q] = tmp[i * ncub + q] * (cub_jac[q] * d->cub_w[q]);
    }
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) {
        double s = 0.0;
        for (int q = 0; q < ncub; ++q)
          s += (d->icub[(size_t)q * np + i] * (cub_jac[q] * d->cub_w[q])) * d->icub[(size_t)q * np + j];
        m[i * np + j] = s;
      }
    /* LLT lower factor, stored column-major like ElementOperators::mass_chol */
    for (int i = 0; i < np * np; ++i) l[i] = 0.0;
    for (int j = 0; j < np && !status; ++j) {
      double dd = m[j * np + j];
      for (int k = 0; k < j; ++k) dd -= l[j * np + k] * l[j * np + k];
      if (!(dd > 0.0)) {
        snprintf(msg, sizeof msg, "build_operators: mass matrix factorization failed");
        status = 3;
        break;
      }
      const double ljj = sqrt(dd);
      l[j * np + j] = ljj;
      for (int i = j + 1; i < np; ++i) {
        double s = m[i * np + j];
        for (int k = 0; k < j; ++k) s -= l[i * np + k] * l[j * np + k];
        l[i * np + j] = s / ljj;
      }
    }
    if (status) break;
    double *ch = lv->chol + (size_t)e * np * np;
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i) ch[j * np + i] = l[i * np + j];
    double *fm = lv->fmass + (size_t)e * np * nf;
    for (int i = 0; i < np; ++i)
      for (int q = 0; q < nf; ++q) fm[i * nf + q] = d->ig[(size_t)q * np + i] * (sjac[q] * d->face_w[q % ng]);
  }
  /* face pairing (solver.cpp:144-178) */
  lv->nb = (int *)malloc(sizeof(int) * K * 4);
  lv->nbf = (int *)malloc(sizeof(int) * K * 4);
  lv->bc = (int *)malloc(sizeof(int) * K * 4);
  lv->nmap = (int *)malloc(sizeof(int) * (size_t)K * 4 * ng);
  memcpy(lv->nb, d->neighbor, sizeof(int) * K * 4);
  memcpy(lv->nbf, d->neighbor_face, sizeof(int) * K * 4);
  memcpy(lv->bc, d->bc, sizeof(int) * K * 4);
  for (int e = 0; e < K && !status; ++e)
    for (int f = 0; f < 4 && !status; ++f) {
      const int nb = lv->nb[e * 4 + f];
      for (int g = 0; g < ng; ++g) {
        if (nb < 0) {
          lv->nmap[((size_t)e * 4 + f) * ng + g] = -1;
          continue;
        }
        const double *mine = face_phys + ((size_t)e * nf + f * ng + g) * 3;
        const int nface = lv->nbf[e * 4 + f];
        int match = -1;
        double best = 1e300;
        for (int h = 0; h < ng; ++h) {
          const double *th = face_phys + ((size_t)nb * nf + nface * ng + h) * 3;
          double dx = mine[0] - th[0], dy = mine[1] - th[1], dz = mine[2] - th[2];
          /* periodic boxes (BASELINE config 1, not a reference feature): the
             neighbour face is a translate, pair by minimum image */
          if (d->period[0] > 0.0) dx -= d->period[0] * nearbyint(dx / d->period[0]);
          if (d->period[1] > 0.0) dy -= d->period[1] * nearbyint(dy / d->period[1]);
          if (d->period[2] > 0.0) dz -= d->period[2] * nearbyint(dz / d->period[2]);
          const double dist = sqrt(dx * dx + dy * dy + dz * dz);
          if (dist < best) {
            best = dist;
            match = h;
          }
        }
        if (best > 1e-8 * (d->pair_scale[e] + 1e-30)) {
          snprintf(msg, sizeof msg, "face quadrature pairing failed between elements %d and %d (mismatch %f)", e,
                   nb, best);
          status = 3;
          break;
        }
        lv->nmap[((size_t)e * 4 + f) * ng + g] = match;
      }
    }
  free(face_phys);
  free(cxr), free(cxs), free(cxt), free(fxr), free(fxs), free(fxt);
  free(cub_dr), free(cub_jac), free(sjac), free(m), free(l), free(tmp);
  if (status) {
    set_err(err, errlen, msg);
    cdgo_level_destroy(lv);
    return status;
  }
  const size_t n = (size_t)K * NF5 * lv->block, nt = (size_t)K * NF5 * lv->tblock;
  lv->traces = (double *)calloc(nt, sizeof(double));
  lv->rhsbuf = (double *)calloc(n, sizeof(double));
  lv->qn = (double *)calloc(3 * n, sizeof(double));
  lv->qt = (double *)calloc(3 * nt, sizeof(double));
  lv->eps = (double *)calloc(K, sizeof(double));
  lv->seps = (double *)calloc(K, sizeof(double));
  *out = lv;
  return 0;
}

void cdgo_level_destroy(cdgo_level *lv) {
  if (!lv) return;
  free(lv->icub), free(lv->ig), free(lv->cub_w), free(lv->face_w), free(lv->vinv);
  free(lv->S), free(lv->fmass), free(lv->chol), free(lv->normal), free(lv->h);
  free(lv->nb), free(lv->nbf), free(lv->bc), free(lv->nmap);
  free(lv->traces), free(lv->rhsbuf), free(lv->qn), free(lv->qt), free(lv->eps), free(lv->seps);
  free(lv);
}

void cdgo_level_sizes(const cdgo_level *lv, int *s) {
  s[0] = lv->K;
  s[1] = lv->block;
  s[2] = lv->tblock;
}

void cdgo_level_export(const cdgo_level *lv, double *h, int *node_map) {
  if (h) memcpy(h, lv->h, sizeof(double) * lv->K);
  if (node_map) memcpy(node_map, lv->nmap, sizeof(int) * (size_t)lv->K * 4 * lv->ng);
}

/* ---- kernels -------------------------------------------------------------- */
#define FIELD(buf, blk, e, c) ((buf) + ((size_t)(e) * NF5 + (c)) * (blk))

int cdgo_interpolate_to_faces(cdgo_level *lv, const double *u, double *traces) {
  for (int e = 0; e < lv->K; ++e)
    for (int c = 0; c < NF5; ++c) gemv(lv->ig, lv->nf, lv->np, FIELD(u, lv->block, e, c), FIELD(traces, lv->tblock, e, c));
  return 0;
}

static st5 load_state(const double *buf, int blk, int e, int idx) {
  st5 s = {FIELD(buf, blk, e, 0)[idx], FIELD(buf, blk, e, 1)[idx], FIELD(buf, blk, e, 2)[idx],
           FIELD(buf, blk, e, 3)[idx], FIELD(buf, blk, e, 4)[idx]};
  return s;
}

/* gather_pair (solver.cpp:222-237) */
static int gather_pair(cdgo_level *lv, const double *traces, int e, int f, int g, const double *n, st5 *um,
                       st5 *up) {
  *um = load_state(traces, lv->tblock, e, f * lv->ng + g);
  const int nb = lv->nb[e * 4 + f];
  if (nb >= 0) {
    *up = load_state(traces, lv->tblock, nb, lv->nbf[e * 4 + f] * lv->ng + lv->nmap[((size_t)e * 4 + f) * lv->ng + g]);
    return nb;
  }
  *up = boundary_state(um, n, lv->bc[e * 4 + f], lv->fs);
  return e;
}

static void element_viscosities(cdgo_level *lv, const cdgo_cfg *cfg, const double *u) {
  const int np = lv->np, pp = lv->p;
  const int np_prev = pp * (pp + 1) * (pp + 2) / 6;
  const double s0 = log10(1.0 / pow((double)pp, 4)) + cfg->s0_offset;
  double max_eps = 0.0;
  double *modal = malloc(sizeof(double) * np);
  for (int e = 0; e < lv->K; ++e) {
    const double *f = FIELD(u, lv->block, e, cfg->indicator_component);
    double total = 0.0, top = 0.0;
    for (int j = 0; j < np; ++j) {
      double s = 0.0;
      for (int k = 0; k < np; ++k) s += lv->vinv[(size_t)j * np + k] * f[k];
      modal[j] = s;
    }
    for (int j = 0; j < np; ++j) {
      const double en = modal[j] * modal[j];
      total += en;
      if (j >= np_prev) top += en;
    }
    const double sk_val = total <= 0.0 ? 0.0 : top / total;
    double eps = 0.0;
    if (sk_val > 0.0) {
      const double sk = log10(sk_val);
      if (sk < s0 - cfg->kappa)
        eps = 0.0;
      else if (sk > s0 + cfg->kappa)
        eps = cfg->eps0;
      else
        eps = 0.5 * cfg->eps0 * (1.0 + sin(M_PI * (sk - s0) / (2.0 * cfg->kappa)));
    }
    lv->eps[e] = eps;
    lv->seps[e] = sqrt(eps);
    if (eps > max_eps) max_eps = eps;
  }
  free(modal);
  lv->viscous_active = max_eps > 0.0;
}

static void aux_gradient(cdgo_level *lv, const double *u) {
  const int np = lv->np, ncub = lv->ncub, ng = lv->ng, nf = lv->nf, blk = lv->block;
  double *ucub = malloc(sizeof(double) * NF5 * ncub), *vol = malloc(sizeof(double) * NF5 * np);
  double *fstar = malloc(sizeof(double) * NF5 * nf), *tmp = malloc(sizeof(double) * np);
  const size_t n = (size_t)lv->K * NF5 * blk, nt = (size_t)lv->K * NF5 * lv->tblock;
  for (int e = 0; e < lv->K; ++e) {
    const double se = lv->seps[e];
    for (int c = 0; c < NF5; ++c) gemv(lv->icub, ncub, np, FIELD(u, blk, e, c), ucub + c * ncub);
    for (int m = 0; m < 3; ++m) {
      const double *S = lv->S + ((size_t)e * 3 + m) * np * ncub;
      for (int c = 0; c < NF5; ++c) {
        double *v = vol + c * np;
        for (int i = 0; i < np; ++i) v[i] = 0.0;
        gemv_sub(S, np, ncub, ucub + c * ncub, v);
        for (int i = 0; i < np; ++i) v[i] *= se;
      }
      for (int f = 0; f < 4; ++f)
        for (int g = 0; g < ng; ++g) {
          const int q = f * ng + g;
          const double *nrm = lv->normal + ((size_t)e * nf + q) * 3;
          st5 um, up;
          const int nb = gather_pair(lv, lv->traces, e, f, g, nrm, &um, &up);
          const double snb = lv->seps[nb];
          for (int c = 0; c < NF5; ++c)
            fstar[c * nf + q] = 0.5 * (se * st_get(&um, c) + snb * st_get(&up, c)) * nrm[m];
        }
      for (int c = 0; c < NF5; ++c) {
        gemv_acc(lv->fmass + (size_t)e * np * nf, np, nf, fstar + c * nf, vol + c * np);
        mass_solve(lv->chol + (size_t)e * np * np, np, vol + c * np, tmp);
        double *o = lv->qn + m * n + ((size_t)e * NF5 + c) * blk;
        for (int i = 0; i < np; ++i) o[i] = tmp[i];
      }
    }
  }
  for (int e = 0; e < lv->K; ++e)
    for (int m = 0; m < 3; ++m)
      for (int c = 0; c < NF5; ++c)
        gemv(lv->ig, nf, np, lv->qn + m * n + ((size_t)e * NF5 + c) * blk,
             lv->qt + m * nt + ((size_t)e * NF5 + c) * lv->tblock);
  free(ucub), free(vol), free(fstar), free(tmp);
}

int cdgo_compute_rhs(cdgo_level *lv, const cdgo_cfg *cfg, const double *u, double *rhs, char *err, size_t errlen) {
  const int np = lv->np, ncub = lv->ncub, ng = lv->ng, nf = lv->nf, blk = lv->block, tb = lv->tblock;
  const double gm = cfg->gamma;
  if (cfg->riemann != 0 && cfg->riemann != 1) {
    set_err(err, errlen, "unknown Riemann solver (llf|hllc)");
    return 2;
  }
  int viscous = 0;
  if (cfg->visc_enabled) {
    if (cfg->jacobian_weighted) {
      set_err(err, errlen, "oracle: jacobian_weighted indicator not restated");
      return 2;
    }
    element_viscosities(lv, cfg, u);
    viscous = lv->viscous_active;
  }
  cdgo_interpolate_to_faces(lv, u, lv->traces);
  if (viscous) {
    aux_gradient(lv, u);
    lv->have_q = 1;
  }
  const size_t n = (size_t)lv->K * NF5 * blk, nt = (size_t)lv->K * NF5 * tb;
  double *ucub = malloc(sizeof(double) * NF5 * ncub), *flux = malloc(sizeof(double) * 3 * NF5 * ncub);
  double *fstar = malloc(sizeof(double) * NF5 * nf), *vol = malloc(sizeof(double) * NF5 * np);
  double *tmp = malloc(sizeof(double) * np), *qcub = malloc(sizeof(double) * 3 * NF5 * ncub);
  int status = 0;
  char msg[512];
  for (int e = 0; e < lv->K && !status; ++e) {
    const double se = viscous ? lv->seps[e] : 0.0;
    for (int c = 0; c < NF5; ++c) gemv(lv->icub, ncub, np, FIELD(u, blk, e, c), ucub + c * ncub);
    if (viscous && lv->seps[e] > 0.0)
      for (int m = 0; m < 3; ++m)
        for (int c = 0; c < NF5; ++c)
          gemv(lv->icub, ncub, np, lv->qn + m * n + ((size_t)e * NF5 + c) * blk, qcub + (m * NF5 + c) * ncub);
    for (int q = 0; q < ncub; ++q) {
      const st5 s = {ucub[q], ucub[ncub + q], ucub[2 * ncub + q], ucub[3 * ncub + q], ucub[4 * ncub + q]};
      if (!admissible(&s, gm)) {
        snprintf(msg, sizeof msg, "inadmissible state in element %d at cubature node %d (rho=%f)", e, q, s.rho);
        status = 3;
        break;
      }
      const double p = (gm - 1.0) * (s.E - dot3(s.mx, s.my, s.mz, s.mx, s.my, s.mz) / (2.0 * s.rho));
      const double v[3] = {s.mx / s.rho, s.my / s.rho, s.mz / s.rho};
      const double mom[3] = {s.mx, s.my, s.mz};
      for (int dd = 0; dd < 3; ++dd) {
        double *fd = flux + (dd * NF5) * ncub;
        const double vd = v[dd];
        fd[0 * ncub + q] = mom[dd];
        fd[1 * ncub + q] = s.mx * vd;
        fd[2 * ncub + q] = s.my * vd;
        fd[3 * ncub + q] = s.mz * vd;
        fd[(1 + dd) * ncub + q] += p;
        fd[4 * ncub + q] = vd * (s.E + p);
      }
    }
    if (status) break;
    if (viscous && lv->seps[e] > 0.0)
      for (int m = 0; m < 3; ++m)
        for (int c = 0; c < NF5; ++c) {
          double *fd = flux + (m * NF5 + c) * ncub;
          const double *qc = qcub + (m * NF5 + c) * ncub;
          for (int q = 0; q < ncub; ++q) fd[q] -= se * qc[q];
        }
    for (int c = 0; c < NF5; ++c) {
      double *v = vol + c * np;
      for (int i = 0; i < np; ++i) v[i] = 0.0;
      for (int m = 0; m < 3; ++m)
        gemv_acc(lv->S + ((size_t)e * 3 + m) * np * ncub, np, ncub, flux + (m * NF5 + c) * ncub, v);
    }
    for (int f = 0; f < 4 && !status; ++f) {
      const int nbr = lv->nb[e * 4 + f];
      for (int g = 0; g < ng; ++g) {
        const int q = f * ng + g;
        const double *nrm = lv->normal + ((size_t)e * nf + q) * 3;
        st5 um, up;
        const int nb = gather_pair(lv, lv->traces, e, f, g, nrm, &um, &up);
        if (!admissible(&um, gm) || !admissible(&up, gm)) {
          snprintf(msg, sizeof msg, "inadmissible trace state in element %d face %d node %d", e, f, g);
          status = 3;
          break;
        }
        double fs[5];
        if (cfg->riemann == 0)
          llf_flux(&um, &up, nrm, gm, fs);
        else
          hllc_flux(&um, &up, nrm, gm, fs);
        if (viscous) {
          const double snb = lv->seps[nb];
          for (int c = 0; c < NF5; ++c) {
            double visc = 0.0;
            for (int m = 0; m < 3; ++m) {
              const double qs = lv->qt[m * nt + ((size_t)e * NF5 + c) * tb + f * ng + g];
              const double qn =
                  nbr >= 0 ? lv->qt[m * nt + ((size_t)nbr * NF5 + c) * tb + lv->nbf[e * 4 + f] * ng +
                                    lv->nmap[((size_t)e * 4 + f) * ng + g]]
                           : qs;
              visc += 0.5 * (se * qs + snb * qn) * nrm[m];
            }
            fs[c] -= visc;
          }
        }
        for (int c = 0; c < NF5; ++c) fstar[c * nf + q] = fs[c];
      }
    }
    if (status) break;
    for (int c = 0; c < NF5; ++c) {
      gemv_sub(lv->fmass + (size_t)e * np * nf, np, nf, fstar + c * nf, vol + c * np);
      mass_solve(lv->chol + (size_t)e * np * np, np, vol + c * np, tmp);
      double *o = FIELD(rhs, blk, e, c);
      for (int i = 0; i < np; ++i) o[i] = tmp[i];
    }
  }
  free(ucub), free(flux), free(fstar), free(vol), free(tmp), free(qcub);
  if (status) set_err(err, errlen, msg);
  return status;
}

int cdgo_rk_steps(cdgo_level *lv, const cdgo_cfg *cfg, double dt, int nsteps, const double *a, const double *b,
                  double *u, double *res, char *err, size_t errlen) {
  const size_t n = (size_t)lv->K * NF5 * lv->block;
  for (int s = 0; s < nsteps; ++s)
    for (int stage = 0; stage < 5; ++stage) {
      const int st = cdgo_compute_rhs(lv, cfg, u, lv->rhsbuf, err, errlen);
      if (st) return st;
      const double aa = a[stage], bb = b[stage];
      for (size_t i = 0; i < n; ++i) {
        res[i] = aa * res[i] + dt * lv->rhsbuf[i];
        u[i] += bb * res[i];
      }
    }
  return 0;
}

int cdgo_compute_timestep(cdgo_level *lv, const cdgo_cfg *cfg, const double *u, const double *eps, double *dt,
                          char *err, size_t errlen) {
  if (cfg->cfl <= 0.0) {
    set_err(err, errlen, "compute_timestep: CFL must be positive");
    return 2;
  }
  const int pp = lv->p, np = lv->np;
  const double pfac = (pp + 1.0) * (pp + 1.0);
  double best = 1e300;
  char msg[256];
  for (int e = 0; e < lv->K; ++e) {
    double lambda = 0.0;
    for (int i = 0; i < np; ++i) {
      const st5 s = load_state(u, lv->block, e, i);
      if (!admissible(&s, cfg->gamma)) {
        snprintf(msg, sizeof msg, "inadmissible state in compute_timestep: rho=%f rhoE=%f", s.rho, s.E);
        set_err(err, errlen, msg);
        return 3;
      }
      const double pres = (cfg->gamma - 1.0) * (s.E - dot3(s.mx, s.my, s.mz, s.mx, s.my, s.mz) / (2.0 * s.rho));
      const double c = sqrt(cfg->gamma * pres / s.rho);
      const double w = sqrt(dot3(s.mx, s.my, s.mz, s.mx, s.my, s.mz)) / s.rho + c;
      if (w > lambda) lambda = w;
    }
    const double h = lv->h[e];
    if (h <= 0.0 || lambda <= 0.0) {
      snprintf(msg, sizeof msg, "compute_timestep: degenerate h or wavespeed in element %d", e);
      set_err(err, errlen, msg);
      return 3;
    }
    double dte = h / (lambda * pfac);
    if (eps && eps[e] > 0.0) {
      const double dv = h * h / (eps[e] * pfac * pfac);
      if (dv < dte) dte = dv;
    }
    if (dte < best) best = dte;
  }
  *dt = cfg->cfl * best;
  return 0;
}

int cdgo_last_viscosity(cdgo_level *lv, double *eps, double *q) {
  memcpy(eps, lv->eps, sizeof(double) * lv->K);
  if (q) {
    if (!lv->have_q) return 1;
    memcpy(q, lv->qn, sizeof(double) * 3 * (size_t)lv->K * NF5 * lv->block);
  }
  return 0;
}
