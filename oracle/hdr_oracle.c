/* hdr_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see hdr_oracle.h).
 *
 * Compiled with -ffp-contract=off: every a*b+c below is two roundings, as in
 * the as-shipped reference build (no -march, 0 FMAs; SURVEY.md probe P8).
 * The only fused operations are explicit fma() calls, which mirror the
 * reference's std::fma in compensated_residual (src/dense.cpp:146) and the
 * two_prod of include/hdivred/dd.hpp:35-38.
 */
#define _GNU_SOURCE
#include "hdr_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ arrays */

typedef struct {
  char name[48];
  char type; /* 'd' or 'q' */
  long long count;
  void* data;
} arr_t;

typedef struct {
  long long ni, nb, nr;
  long long *i_local, *b_local, *rows;
  double *a_ii, *a_ii_lu, *a_ib, *a_bi, *s_b, *s_b_lu, *c_b;
  long long *a_ii_piv, *s_b_piv;
} port_elem;

typedef struct {
  long long ni, nb;
  long long *i_local, *b_local;
  double *a_ii, *a_ii_lu, *a_ib, *schur, *f_s;
  long long* a_ii_piv;
  long long* b_master_ord; /* nb ordinals (single-entry P rows on the FE path) */
  double* b_master_sign;
  long long* i_global;
  double* i_sign;
} cond_elem;

struct hdo_ctx {
  int dim, k, weighted;
  long long N[3];
  double h[3];
  long long n, dpf, nint, ncells, nfaces, ndofs, face_dof_count, broken, m, nS;
  double *divdiv, *mass, *face_moments, *unit_load;
  arr_t arrs[96];
  int narr;
  port_elem* pe;
  cond_elem* ce;
  char err[256];
};

static void set_err(hdo_ctx* c, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->err, sizeof c->err, fmt, ap);
  va_end(ap);
}

static arr_t* find_arr(const hdo_ctx* c, const char* name) {
  for (int i = 0; i < c->narr; ++i)
    if (strcmp(c->arrs[i].name, name) == 0) return (arr_t*)&c->arrs[i];
  return NULL;
}

static void* put_arr(hdo_ctx* c, const char* name, char type, long long count) {
  arr_t* a = find_arr(c, name);
  if (!a) {
    if (c->narr >= 96) return NULL;
    a = &c->arrs[c->narr++];
    snprintf(a->name, sizeof a->name, "%s", name);
  } else {
    free(a->data);
  }
  a->type = type;
  a->count = count;
  a->data = calloc((size_t)(count > 0 ? count : 1), 8);
  return a->data;
}

static double* get_d(const hdo_ctx* c, const char* name) {
  arr_t* a = find_arr(c, name);
  return (a && a->type == 'd') ? (double*)a->data : NULL;
}
static long long* get_q(const hdo_ctx* c, const char* name) {
  arr_t* a = find_arr(c, name);
  return (a && a->type == 'q') ? (long long*)a->data : NULL;
}

/* -------------------------------------------------------------- RNG (§8(d)) */

typedef struct {
  uint64_t s;
} rng_t;
static uint64_t rng_next(rng_t* r) {
  r->s ^= r->s << 13;
  r->s ^= r->s >> 7;
  r->s ^= r->s << 17;
  return r->s;
}
static double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform2(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }
static double rng_log_uniform(rng_t* r, double lo, double hi) { return exp(rng_uniform2(r, log(lo), log(hi))); }

/* ---------------------------------------- 1-D polynomials, rt_space.cpp:10-65 */

static void gauss_legendre_01(int n, double* nodes, double* weights) {
  for (int i = 0; i < n; ++i) {
    double x = cos(M_PI * ((double)i + 0.75) / ((double)n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int m = 2; m <= n; ++m) {
        const double p2 = ((2.0 * m - 1.0) * x * p1 - (m - 1.0) * p0) / (double)m;
        p0 = p1;
        p1 = p2;
      }
      const double pn = p1;
      dp = (double)n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = pn / dp;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    nodes[n - 1 - i] = 0.5 * (x + 1.0);
    weights[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
  }
}

static double legendre01(int m, double s) {
  const double t = 2.0 * s - 1.0;
  double p0 = 1.0, p1 = t;
  if (m == 0) return 1.0;
  for (int i = 2; i <= m; ++i) {
    const double p2 = ((2.0 * i - 1.0) * t * p1 - (i - 1.0) * p0) / (double)i;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

static double legendre01_deriv(int m, double s) {
  if (m == 0) return 0.0;
  const double t = 2.0 * s - 1.0;
  if (m == 1) return 2.0;
  double p0 = 1.0, p1 = t;
  for (int i = 2; i <= m; ++i) {
    const double p2 = ((2.0 * i - 1.0) * t * p1 - (i - 1.0) * p0) / (double)i;
    p0 = p1;
    p1 = p2;
  }
  if (fabs(t * t - 1.0) < 1e-12) {
    const double sign = (t > 0.0) ? 1.0 : ((m % 2 == 1) ? 1.0 : -1.0);
    return 2.0 * sign * 0.5 * m * (m + 1.0);
  }
  return 2.0 * (double)m * (t * p1 - p0) / (t * t - 1.0);
}

/* ------------------------------------------- dense kernels, dense.cpp:17-163 */

/* lu_factor (dense.cpp:61-97): in place on lu (n x n row-major). Returns -1 on
 * success, else the failing pivot index. */
static long long lu_factor(double* lu, long long n, long long* piv) {
  double mx = 0.0;
  for (long long i = 0; i < n * n; ++i)
    if (fabs(lu[i]) > mx) mx = fabs(lu[i]);
  const double threshold = 1e-14 * mx;
  for (long long k = 0; k < n; ++k) {
    long long p = k;
    double pm = fabs(lu[k * n + k]);
    for (long long i = k + 1; i < n; ++i) {
      const double v = fabs(lu[i * n + k]);
      if (v > pm) {
        pm = v;
        p = i;
      }
    }
    if (!(pm > threshold) || pm == 0.0) return k;
    piv[k] = p;
    if (p != k)
      for (long long j = 0; j < n; ++j) {
        const double t = lu[k * n + j];
        lu[k * n + j] = lu[p * n + j];
        lu[p * n + j] = t;
      }
    const double inv = 1.0 / lu[k * n + k];
    for (long long i = k + 1; i < n; ++i) {
      const double l = lu[i * n + k] * inv;
      lu[i * n + k] = l;
      if (l == 0.0) continue;
      for (long long j = k + 1; j < n; ++j) lu[i * n + j] -= l * lu[k * n + j];
    }
  }
  return -1;
}

/* lu_solve (dense.cpp:99-120), x holds b on entry */
static void lu_solve(const double* lu, const long long* piv, long long n, double* x) {
  for (long long k = 0; k < n; ++k) {
    const long long p = piv[k];
    if (p != k) {
      const double t = x[k];
      x[k] = x[p];
      x[p] = t;
    }
  }
  for (long long k = 0; k < n; ++k) {
    const double xk = x[k];
    if (xk == 0.0) continue;
    for (long long i = k + 1; i < n; ++i) x[i] -= lu[i * n + k] * xk;
  }
  for (long long i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (long long j = i + 1; j < n; ++j) s -= lu[i * n + j] * x[j];
    x[i] = s / lu[i * n + i];
  }
}

/* Neumaier two-sum update (dense.cpp:125-132) */
static inline void nsum(double* sum, double* comp, double value) {
  const double t = *sum + value;
  if (fabs(*sum) >= fabs(value))
    *comp += (*sum - t) + value;
  else
    *comp += (value - t) + *sum;
  *sum = t;
}

/* compensated_residual (dense.cpp:136-152) */
static void comp_residual(const double* a, long long n, const double* x, const double* b, double* r) {
  for (long long i = 0; i < n; ++i) {
    double sum = 0.0, comp = 0.0;
    for (long long j = 0; j < n; ++j) {
      const double aij = a[i * n + j];
      const double xj = x[j];
      const double p = aij * xj;
      nsum(&sum, &comp, p);
      comp += fma(aij, xj, -p);
    }
    nsum(&sum, &comp, -b[i]);
    r[i] = -(sum + comp);
  }
}

/* lu_solve_refined (dense.cpp:154-163), steps = 2; x, b of length n */
static void lu_solve_refined(const double* a, const double* lu, const long long* piv, long long n, const double* b,
                             double* x, double* work) {
  double* r = work;
  memcpy(x, b, (size_t)n * 8);
  lu_solve(lu, piv, n, x);
  for (int it = 0; it < 2; ++it) {
    comp_residual(a, n, x, b, r);
    lu_solve(lu, piv, n, r);
    for (long long i = 0; i < n; ++i) x[i] += r[i];
  }
}

/* solve_matrix_refined (reduction.cpp:75-84): X = A^-1 B column by column */
static void solve_matrix_refined(const double* a, const double* lu, const long long* piv, long long n, const double* B,
                                 long long ncols, double* X) {
  double* col = malloc((size_t)(3 * n + 1) * 8);
  double* sol = col + n;
  double* work = sol + n;
  for (long long j = 0; j < ncols; ++j) {
    for (long long i = 0; i < n; ++i) col[i] = B[i * ncols + j];
    lu_solve_refined(a, lu, piv, n, col, sol, work);
    for (long long i = 0; i < n; ++i) X[i * ncols + j] = sol[i];
  }
  free(col);
}

/* dense_multiply (dense.cpp:17-28): C (r x c) = A (r x k) B (k x c), C zeroed */
static void dense_multiply(const double* A, const double* B, long long r, long long kk, long long c, double* C) {
  memset(C, 0, (size_t)(r * c) * 8);
  for (long long i = 0; i < r; ++i)
    for (long long k = 0; k < kk; ++k) {
      const double aik = A[i * kk + k];
      if (aik == 0.0) continue;
      for (long long j = 0; j < c; ++j) C[i * c + j] += aik * B[k * c + j];
    }
}

/* dense_apply (dense.cpp:44-53) */
static void dense_apply(const double* A, long long r, long long c, const double* x, double* y) {
  for (long long i = 0; i < r; ++i) {
    double s = 0.0;
    for (long long j = 0; j < c; ++j) s += A[i * c + j] * x[j];
    y[i] = s;
  }
}

/* symmetrize (reduction.cpp:65-72) */
static void symmetrize(double* a, long long n) {
  for (long long i = 0; i < n; ++i)
    for (long long j = i + 1; j < n; ++j) {
      const double v = 0.5 * (a[i * n + j] + a[j * n + i]);
      a[i * n + j] = v;
      a[j * n + i] = v;
    }
}

/* ---------------------------------------- reference element, rt_space.cpp */

typedef struct {
  int comp;
  int deg[3];
} spoly;

static int space_polys(int dim, int k, spoly* out) {
  int cnt = 0;
  for (int c = 0; c < dim; ++c) {
    int lim[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) lim[a] = (a == c) ? k + 1 : k;
    for (int dz = 0; dz <= lim[2]; ++dz)
      for (int dy = 0; dy <= lim[1]; ++dy)
        for (int dx = 0; dx <= lim[0]; ++dx) {
          out[cnt].comp = c;
          out[cnt].deg[0] = dx;
          out[cnt].deg[1] = dy;
          out[cnt].deg[2] = dz;
          ++cnt;
        }
  }
  return cnt;
}

static int interior_moments(int dim, int k, spoly* out) {
  int cnt = 0;
  if (k == 0) return 0;
  for (int c = 0; c < dim; ++c) {
    int lim[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) lim[a] = (a == c) ? k - 1 : k;
    for (int dz = 0; dz <= lim[2]; ++dz)
      for (int dy = 0; dy <= lim[1]; ++dy)
        for (int dx = 0; dx <= lim[0]; ++dx) {
          out[cnt].comp = c;
          out[cnt].deg[0] = dx;
          out[cnt].deg[1] = dy;
          out[cnt].deg[2] = dz;
          ++cnt;
        }
  }
  return cnt;
}

static double lpi(int p, int q) { return (p == q) ? 1.0 / (2.0 * p + 1.0) : 0.0; }
static double mweight(int m) { return sqrt(2.0 * m + 1.0); }
static void moment_degrees(int k, int dim, long long sub, int md[2]) {
  if (dim == 2) {
    md[0] = (int)sub;
    md[1] = 0;
  } else {
    md[0] = (int)(sub % (k + 1));
    md[1] = (int)(sub / (k + 1));
  }
}
static void tangent_axes(int dim, int axis, int t[2]) {
  int c = 0;
  t[0] = t[1] = -1;
  for (int a = 0; a < dim; ++a)
    if (a != axis) t[c++] = a;
}

/* basis coefficients phi (n x n, row = Legendre-product monomial q, column =
 * basis function j) = lu_inverse(lu_factor(dof_vandermonde)) (rt_space.cpp:136-189) */
static double* ref_basis(int dim, int k, spoly* polys, int* n_out) {
  spoly inter[256];
  const int n = space_polys(dim, k, polys);
  const int nint = interior_moments(dim, k, inter);
  const long long dpf = llround(pow(k + 1, dim - 1));
  *n_out = n;

  /* dof_vandermonde (rt_space.cpp:136-172) */
  double* V = calloc((size_t)(n * n), 8);
  for (int j = 0; j < n; ++j) {
    const spoly* t = &polys[j];
    for (int i = 0; i < nint; ++i) {
      const spoly* m = &inter[i];
      if (m->comp != t->comp) continue;
      double val = 1.0;
      for (int a = 0; a < dim; ++a) val *= lpi(t->deg[a], m->deg[a]) * mweight(m->deg[a]);
      V[i * n + j] = val;
    }
    for (int slot = 0; slot < 2 * dim; ++slot) {
      const int axis = slot / 2, side = slot % 2;
      if (t->comp != axis) continue;
      const double nsign = side ? 1.0 : -1.0;
      const double trace = legendre01(t->deg[axis], side ? 1.0 : 0.0);
      int tang[2];
      tangent_axes(dim, axis, tang);
      for (long long sub = 0; sub < dpf; ++sub) {
        int md[2];
        moment_degrees(k, dim, sub, md);
        double val = nsign * trace;
        for (int ti = 0; ti < dim - 1; ++ti) val *= lpi(t->deg[tang[ti]], md[ti]) * mweight(md[ti]);
        V[(nint + slot * dpf + sub) * n + j] = val;
      }
    }
  }
  /* phi = lu_inverse(lu_factor(V)) (rt_space.cpp:189; dense.cpp:165-177) */
  long long* piv = malloc((size_t)n * sizeof(long long));
  if (lu_factor(V, n, piv) >= 0) {
    free(V);
    free(piv);
    return NULL;
  }
  double* phi = calloc((size_t)(n * n), 8);
  double* col = malloc((size_t)n * 8);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i) col[i] = (i == j) ? 1.0 : 0.0;
    lu_solve(V, piv, n, col);
    for (int i = 0; i < n; ++i) phi[i * n + j] = col[i];
  }
  free(col);
  free(piv);
  free(V);
  return phi;
}

int hdo_build_reference(int dim, int k, const double h[3], int nq, double* divdiv, double* mass, double* face_moments,
                        double* unit_load) {
  spoly polys[256];
  int n = 0;
  double* phi = ref_basis(dim, k, polys, &n);
  if (!phi) return 2;
  const long long dpf = llround(pow(k + 1, dim - 1));

  double qs[16], qw[16];
  gauss_legendre_01(nq, qs, qw);
  memset(divdiv, 0, (size_t)(n * n) * 8);
  memset(mass, 0, (size_t)(n * n) * 8);
  if (unit_load) memset(unit_load, 0, (size_t)(3 * n) * 8);

  double* pval = malloc((size_t)n * 8);
  double* pdiv = malloc((size_t)n * 8);
  double* bval = malloc((size_t)(3 * n) * 8);
  double* bdiv = malloc((size_t)n * 8);
  const int nqz = (dim == 3) ? nq : 1;
  for (int iz = 0; iz < nqz; ++iz)
    for (int iy = 0; iy < nq; ++iy)
      for (int ix = 0; ix < nq; ++ix) {
        const double s[3] = {qs[ix], qs[iy], (dim == 3) ? qs[iz] : 0.0};
        double w = qw[ix] * h[0] * qw[iy] * h[1];
        if (dim == 3) w *= qw[iz] * h[2];
        for (int q = 0; q < n; ++q) {
          const spoly* t = &polys[q];
          double val = 1.0;
          for (int a = 0; a < dim; ++a) val *= legendre01(t->deg[a], s[a]);
          pval[q] = val;
          double dv = legendre01_deriv(t->deg[t->comp], s[t->comp]) / h[t->comp];
          for (int a = 0; a < dim; ++a)
            if (a != t->comp) dv *= legendre01(t->deg[a], s[a]);
          pdiv[q] = dv;
        }
        for (int j = 0; j < n; ++j) {
          bval[3 * j] = bval[3 * j + 1] = bval[3 * j + 2] = 0.0;
          double dsum = 0.0;
          for (int q = 0; q < n; ++q) {
            const double c = phi[q * n + j];
            if (c == 0.0) continue;
            bval[3 * j + polys[q].comp] += c * pval[q];
            dsum += c * pdiv[q];
          }
          bdiv[j] = dsum;
        }
        for (int i = 0; i < n; ++i) {
          const double dvi = bdiv[i];
          const double* vi = &bval[3 * i];
          for (int j = 0; j < n; ++j) {
            divdiv[i * n + j] += w * dvi * bdiv[j];
            const double* vj = &bval[3 * j];
            mass[i * n + j] += w * (vi[0] * vj[0] + vi[1] * vj[1] + vi[2] * vj[2]);
          }
          if (unit_load)
            for (int c = 0; c < dim; ++c) unit_load[c * n + i] += w * vi[c];
        }
      }

  /* face moments (rt_space.cpp:267-312) */
  if (face_moments) {
    memset(face_moments, 0, (size_t)(2 * dim * dpf * n) * 8);
    for (int slot = 0; slot < 2 * dim; ++slot) {
      const int axis = slot / 2, side = slot % 2;
      const double nsign = side ? 1.0 : -1.0;
      int tang[2];
      tangent_axes(dim, axis, tang);
      double* fm = face_moments + (long long)slot * dpf * n;
      const int nt1 = nq, nt2 = (dim == 3) ? nq : 1;
      for (int i2 = 0; i2 < nt2; ++i2)
        for (int i1 = 0; i1 < nt1; ++i1) {
          double s[3] = {0.0, 0.0, 0.0};
          s[axis] = side ? 1.0 : 0.0;
          s[tang[0]] = qs[i1];
          double w = qw[i1] * h[tang[0]];
          if (dim == 3) {
            s[tang[1]] = qs[i2];
            w *= qw[i2] * h[tang[1]];
          }
          for (int q = 0; q < n; ++q) {
            double val = 1.0;
            for (int a = 0; a < dim; ++a) val *= legendre01(polys[q].deg[a], s[a]);
            pval[q] = val;
          }
          for (int j = 0; j < n; ++j) {
            double ntr = 0.0;
            for (int q = 0; q < n; ++q) {
              if (polys[q].comp != axis) continue;
              ntr += phi[q * n + j] * pval[q];
            }
            ntr *= nsign;
            if (ntr == 0.0) continue;
            for (long long sub = 0; sub < dpf; ++sub) {
              int md[2];
              moment_degrees(k, dim, sub, md);
              double qv = legendre01(md[0], s[tang[0]]) * mweight(md[0]);
              if (dim == 3) qv *= legendre01(md[1], s[tang[1]]) * mweight(md[1]);
              fm[sub * n + j] += w * ntr * qv;
            }
          }
        }
    }
  }
  free(pval);
  free(pdiv);
  free(bval);
  free(bdiv);
  free(phi);
  return 0;
}

/* ------------------------------------------- perturbed trilinear cells (config 4)
 *
 * RESTATEMENT, NOT THE REFERENCE: the reference supports affine boxes only
 * (SURVEY.md §8(c) "Coverage gaps").  The reference's box element (basis, dofs
 * and numbering of rt_space.cpp) is mapped to the trilinear cell by the
 * contravariant Piola transform of F = X o B^-1 (B: s -> x0 + h s the box map,
 * X: s -> sum_v N_v(s) x_v the trilinear map):
 *   phi = DF phi_box / det DF,  div phi = div phi_box / det DF,
 *   DF = J J0^-1 (J = dX/ds, J0 = diag(h)),  dx = det J ds,
 * so   M_ij = sum_p w_p (det J0^2 / det J) (K phi^_i) . (K phi^_j),   K = J J0^-1
 *      D_ij = sum_p w_p (det J0^2 / det J) divh_i divh_j,   divh = sum_a d_a phi^_a / h_a
 * with the reference's (k+2)^3 Gauss points.  J = J0 (no perturbation) gives
 * the reference's divdiv / mass up to rounding (tests/test_oracle_piola.py).
 * verts: 8 x 3 physical coordinates, local vertex v = vx + 2 (vy + 2 vz). */
static void piola_accumulate(int k, const double* phi, const spoly* polys, int n, const double h[3],
                             const double* verts, int nq, double* divdiv, double* mass, double* pdiv_form,
                             double* pmass) {
  double qs[16], qw[16];
  gauss_legendre_01(nq, qs, qw);
  memset(divdiv, 0, (size_t)(n * n) * 8);
  memset(mass, 0, (size_t)(n * n) * 8);
  const int npr = (k + 1) * (k + 1) * (k + 1);
  if (pdiv_form) memset(pdiv_form, 0, (size_t)(npr * n) * 8);
  if (pmass) memset(pmass, 0, (size_t)(npr * npr) * 8);
  double* pval = malloc((size_t)n * 8);
  double* pdiv = malloc((size_t)n * 8);
  double* psi = malloc((size_t)(3 * n) * 8);
  double* bdiv = malloc((size_t)n * 8);
  double* qv = malloc((size_t)(npr + 1) * 8);
  const double det0 = h[0] * h[1] * h[2];
  for (int iz = 0; iz < nq; ++iz)
    for (int iy = 0; iy < nq; ++iy)
      for (int ix = 0; ix < nq; ++ix) {
        const double s[3] = {qs[ix], qs[iy], qs[iz]};
        /* J[c][a] = sum_v x_v[c] dN_v/ds_a */
        double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int v = 0; v < 8; ++v) {
          const int b[3] = {v & 1, (v >> 1) & 1, (v >> 2) & 1};
          double f[3], d[3];
          for (int a = 0; a < 3; ++a) {
            f[a] = b[a] ? s[a] : 1.0 - s[a];
            d[a] = b[a] ? 1.0 : -1.0;
          }
          const double dN[3] = {d[0] * f[1] * f[2], f[0] * d[1] * f[2], f[0] * f[1] * d[2]};
          for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) J[c][a] += verts[3 * v + c] * dN[a];
        }
        const double detJ = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                            J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        const double w = qw[ix] * qw[iy] * qw[iz] * (det0 * det0 / detJ);
        for (int q = 0; q < n; ++q) {
          const spoly* t = &polys[q];
          double val = 1.0;
          for (int a = 0; a < 3; ++a) val *= legendre01(t->deg[a], s[a]);
          pval[q] = val;
          double dv = legendre01_deriv(t->deg[t->comp], s[t->comp]) / h[t->comp];
          for (int a = 0; a < 3; ++a)
            if (a != t->comp) dv *= legendre01(t->deg[a], s[a]);
          pdiv[q] = dv;
        }
        for (int j = 0; j < n; ++j) {
          double bv[3] = {0.0, 0.0, 0.0}, dsum = 0.0;
          for (int q = 0; q < n; ++q) {
            const double c = phi[q * n + j];
            if (c == 0.0) continue;
            bv[polys[q].comp] += c * pval[q];
            dsum += c * pdiv[q];
          }
          for (int c = 0; c < 3; ++c) psi[3 * j + c] = J[c][0] / h[0] * bv[0] + J[c][1] / h[1] * bv[1] + J[c][2] / h[2] * bv[2];
          bdiv[j] = dsum;
        }
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) {
            divdiv[i * n + j] += w * bdiv[i] * bdiv[j];
            mass[i * n + j] += w * (psi[3 * i] * psi[3 * j] + psi[3 * i + 1] * psi[3 * j + 1] + psi[3 * i + 2] * psi[3 * j + 2]);
          }
        if (pdiv_form || pmass) {
          /* mapped pressures q = q^ det J0 / det J, q^ Legendre products of degree <= k */
          int cnt = 0;
          for (int dz = 0; dz <= k; ++dz)
            for (int dy = 0; dy <= k; ++dy)
              for (int dx = 0; dx <= k; ++dx)
                qv[cnt++] = legendre01(dx, s[0]) * legendre01(dy, s[1]) * legendre01(dz, s[2]);
          for (int p = 0; p < npr; ++p) {
            if (pdiv_form)
              for (int j = 0; j < n; ++j) pdiv_form[p * n + j] += w * qv[p] * bdiv[j];
            if (pmass)
              for (int r = 0; r < npr; ++r) pmass[p * npr + r] += w * qv[p] * qv[r];
          }
        }
      }
  free(pval);
  free(pdiv);
  free(psi);
  free(bdiv);
  free(qv);
}

int hdo_piola_element(int k, const double h[3], const double* verts, int nq, double* divdiv, double* mass,
                      double* div_form, double* pressure_mass) {
  spoly polys[256];
  int n = 0;
  double* phi = ref_basis(3, k, polys, &n);
  if (!phi) return 2;
  piola_accumulate(k, phi, polys, n, h, verts, nq, divdiv, mass, div_form, pressure_mass);
  free(phi);
  return 0;
}

/* the 8 vertices of a cell from the mesh vertex array ((N0+1)(N1+1)(N2+1) x 3) */
static void cell_vertices(const hdo_ctx* c, const double* vtx, long long cell, double* out) {
  const long long cx = cell % c->N[0], cy = (cell / c->N[0]) % c->N[1], cz = cell / (c->N[0] * c->N[1]);
  for (int v = 0; v < 8; ++v) {
    const long long ix = cx + (v & 1), iy = cy + ((v >> 1) & 1), iz = cz + ((v >> 2) & 1);
    const long long g = ix + (c->N[0] + 1) * (iy + (c->N[1] + 1) * iz);
    for (int a = 0; a < 3; ++a) out[3 * v + a] = vtx[3 * g + a];
  }
}

/* --------------------------------------------------- mesh, mesh.cpp:13-135 */

static long long nfaces_axis(const hdo_ctx* c, int axis) {
  long long n = c->N[axis] + 1;
  for (int a = 0; a < c->dim; ++a)
    if (a != axis) n *= c->N[a];
  return n;
}
static long long face_axis_offset(const hdo_ctx* c, int axis) {
  long long off = 0;
  for (int a = 0; a < axis; ++a) off += nfaces_axis(c, a);
  return off;
}
static long long face_linear(const hdo_ctx* c, int axis, const long long* co) {
  long long d[3] = {c->N[0], c->N[1], c->N[2]};
  d[axis] += 1;
  return face_axis_offset(c, axis) + co[0] + d[0] * (co[1] + d[1] * co[2]);
}
/* face(f): axis and the two cells (-1 when absent) */
static void face_info(const hdo_ctx* c, long long f, int* axis, long long* cm, long long* cp) {
  int a = 0;
  long long local = f;
  while (local >= nfaces_axis(c, a)) {
    local -= nfaces_axis(c, a);
    ++a;
  }
  long long d[3] = {c->N[0], c->N[1], c->N[2]};
  d[a] += 1;
  long long co[3];
  co[0] = local % d[0];
  local /= d[0];
  co[1] = local % d[1];
  co[2] = local / d[1];
  const long long plane = co[a];
  *axis = a;
  *cm = *cp = -1;
  if (plane > 0) {
    long long x[3] = {co[0], co[1], co[2]};
    x[a] = plane - 1;
    *cm = x[0] + c->N[0] * (x[1] + c->N[1] * x[2]);
  }
  if (plane < c->N[a]) {
    long long x[3] = {co[0], co[1], co[2]};
    x[a] = plane;
    *cp = x[0] + c->N[0] * (x[1] + c->N[1] * x[2]);
  }
}
static void cell_faces(const hdo_ctx* c, long long cell, long long* faces, double* signs) {
  long long co[3];
  co[0] = cell % c->N[0];
  long long r = cell / c->N[0];
  co[1] = r % c->N[1];
  co[2] = r / c->N[1];
  for (int a = 0; a < c->dim; ++a) {
    long long lo[3] = {co[0], co[1], co[2]}, hi[3] = {co[0], co[1], co[2]};
    hi[a] += 1;
    faces[2 * a] = face_linear(c, a, lo);
    signs[2 * a] = -1.0;
    faces[2 * a + 1] = face_linear(c, a, hi);
    signs[2 * a + 1] = 1.0;
  }
}
static void local_dof_map(const hdo_ctx* c, long long cell, long long* glob, double* sign) {
  long long faces[6];
  double fs[6];
  long long l = 0;
  for (long long i = 0; i < c->nint; ++i, ++l) {
    glob[l] = c->face_dof_count + cell * c->nint + i;
    sign[l] = 1.0;
  }
  cell_faces(c, cell, faces, fs);
  for (int s = 0; s < 2 * c->dim; ++s)
    for (long long sub = 0; sub < c->dpf; ++sub, ++l) {
      glob[l] = faces[s] * c->dpf + sub;
      sign[l] = fs[s];
    }
}

/* -------------------------------------------------------------- lifecycle */

hdo_ctx* hdo_create(int dim, const long long cells[3], int k, int weighted) {
  if ((dim != 2 && dim != 3) || k < 0 || k > 3) return NULL;
  hdo_ctx* c = calloc(1, sizeof *c);
  c->dim = dim;
  c->k = k;
  c->weighted = weighted;
  for (int a = 0; a < 3; ++a) {
    c->N[a] = (a < dim) ? cells[a] : 1;
    c->h[a] = (a < dim) ? 1.0 / (double)cells[a] : 1.0;
    if (c->N[a] < 1) {
      free(c);
      return NULL;
    }
  }
  c->dpf = llround(pow(k + 1, dim - 1));
  c->nint = (long long)(dim * k) * c->dpf;
  c->n = 2 * dim * c->dpf + c->nint;
  c->ncells = c->N[0] * c->N[1] * c->N[2];
  c->nfaces = 0;
  for (int a = 0; a < dim; ++a) c->nfaces += nfaces_axis(c, a);
  c->face_dof_count = c->nfaces * c->dpf;
  c->ndofs = c->face_dof_count + c->ncells * c->nint;
  c->broken = c->ncells * c->n;
  c->m = c->broken - c->ndofs;
  c->nS = c->face_dof_count;
  const long long n = c->n;
  c->divdiv = put_arr(c, "ref_divdiv", 'd', n * n);
  c->mass = put_arr(c, "ref_mass", 'd', n * n);
  c->face_moments = put_arr(c, "ref_face_moments", 'd', 2 * dim * c->dpf * n);
  c->unit_load = put_arr(c, "ref_unit_load", 'd', 3 * n);
  if (hdo_build_reference(dim, k, c->h, k + 2, c->divdiv, c->mass, c->face_moments, c->unit_load) != 0) {
    hdo_destroy(c);
    return NULL;
  }
  return c;
}

static void free_port(hdo_ctx* c) {
  if (c->pe) {
    for (long long e = 0; e < c->ncells; ++e) {
      port_elem* p = &c->pe[e];
      free(p->i_local);
      free(p->b_local);
      free(p->rows);
      free(p->a_ii);
      free(p->a_ii_lu);
      free(p->a_ib);
      free(p->a_bi);
      free(p->s_b);
      free(p->s_b_lu);
      free(p->c_b);
      free(p->a_ii_piv);
      free(p->s_b_piv);
    }
    free(c->pe);
    c->pe = NULL;
  }
  if (c->ce) {
    for (long long e = 0; e < c->ncells; ++e) {
      cond_elem* p = &c->ce[e];
      free(p->i_local);
      free(p->b_local);
      free(p->a_ii);
      free(p->a_ii_lu);
      free(p->a_ib);
      free(p->schur);
      free(p->f_s);
      free(p->a_ii_piv);
      free(p->b_master_ord);
      free(p->b_master_sign);
      free(p->i_global);
      free(p->i_sign);
    }
    free(c->ce);
    c->ce = NULL;
  }
}

/* Cell sizes other than the unit cube's 1/N (a z-slab sub-mesh keeps the global
   mesh's h, paper_1801_08914_b200/slab.py): the reference matrices are rebuilt
   and any per-element state dropped. */
int hdo_set_h(hdo_ctx* c, const double h[3]) {
  for (int a = 0; a < c->dim; ++a) c->h[a] = h[a];
  free_port(c);
  return hdo_build_reference(c->dim, c->k, c->h, c->k + 2, c->divdiv, c->mass, c->face_moments, c->unit_load);
}

void hdo_destroy(hdo_ctx* c) {
  if (!c) return;
  free_port(c);
  for (int i = 0; i < c->narr; ++i) free(c->arrs[i].data);
  free(c);
}

long long hdo_size(const hdo_ctx* c, const char* name) {
  if (!strcmp(name, "dim")) return c->dim;
  if (!strcmp(name, "k")) return c->k;
  if (!strcmp(name, "n")) return c->n;
  if (!strcmp(name, "dpf")) return c->dpf;
  if (!strcmp(name, "nint")) return c->nint;
  if (!strcmp(name, "ncells")) return c->ncells;
  if (!strcmp(name, "nfaces")) return c->nfaces;
  if (!strcmp(name, "ndofs")) return c->ndofs;
  if (!strcmp(name, "face_dof_count")) return c->face_dof_count;
  if (!strcmp(name, "broken")) return c->broken;
  if (!strcmp(name, "m")) return c->m;
  if (!strcmp(name, "nS")) return c->nS;
  return -1;
}

long long hdo_count(const hdo_ctx* c, const char* name) {
  arr_t* a = find_arr(c, name);
  return a ? a->count : -1;
}
int hdo_get_d(const hdo_ctx* c, const char* name, double* out) {
  arr_t* a = find_arr(c, name);
  if (!a || a->type != 'd') return 1;
  memcpy(out, a->data, (size_t)a->count * 8);
  return 0;
}
int hdo_get_q(const hdo_ctx* c, const char* name, long long* out) {
  arr_t* a = find_arr(c, name);
  if (!a || a->type != 'q') return 1;
  memcpy(out, a->data, (size_t)a->count * 8);
  return 0;
}
int hdo_set_d(hdo_ctx* c, const char* name, const double* data, long long count) {
  double* p = put_arr(c, name, 'd', count);
  if (!p) return 1;
  memcpy(p, data, (size_t)count * 8);
  return 0;
}
const char* hdo_last_error(const hdo_ctx* c) { return c->err; }

int hdo_gen_inputs(hdo_ctx* c, const char* coef, unsigned long long seed) {
  rng_t r = {seed ? seed : 0x9e3779b97f4a7c15ull};
  double* al = put_arr(c, "alpha", 'd', c->ncells);
  double* be = put_arr(c, "beta", 'd', c->ncells);
  double p0 = 0, p1 = 0;
  char kind[32] = {0};
  const char* colon = strchr(coef, ':');
  if (!colon || colon - coef >= 31) {
    set_err(c, "bad coef spec %s", coef);
    return 1;
  }
  memcpy(kind, coef, (size_t)(colon - coef));
  if (sscanf(colon + 1, "%lf:%lf", &p0, &p1) < 1) {
    set_err(c, "bad coef spec %s", coef);
    return 1;
  }
  for (long long e = 0; e < c->ncells; ++e) {
    if (!strcmp(kind, "uniform")) {
      al[e] = p0;
      be[e] = p1;
    } else if (!strcmp(kind, "logu")) {
      al[e] = rng_log_uniform(&r, p0, p1);
      be[e] = rng_log_uniform(&r, p0, p1);
    } else if (!strcmp(kind, "checker")) {
      /* mesh.cpp:49-56 cell_center; SURVEY.md §8(d) cfg5 mapping */
      long long co[3];
      co[0] = e % c->N[0];
      long long rr = e / c->N[0];
      co[1] = rr % c->N[1];
      co[2] = rr / c->N[1];
      long reg = 0;
      for (int a = 0; a < c->dim; ++a) {
        const double x = 0.0 + ((double)co[a] + 0.5) * c->h[a];
        reg += (long)floor(4.0 * x);
      }
      const double sigma = (reg % 2 == 0) ? p0 : p1;
      al[e] = 1.0;
      be[e] = 1.0 / (3.0 * sigma);
    } else if (!strcmp(kind, "softhard")) {
      /* soft_hard_coefficients (src/mesh.cpp:168-191): beta = 10^p on the cells whose
       * centre lies in [1/4, 1/2]^d or [1/2, 3/4]^d, alpha = beta = 1 elsewhere */
      long long co[3];
      co[0] = e % c->N[0];
      long long rr = e / c->N[0];
      co[1] = rr % c->N[1];
      co[2] = rr / c->N[1];
      int in_lo = 1, in_hi = 1;
      for (int a = 0; a < c->dim; ++a) {
        const double t = 0.0 + ((double)co[a] + 0.5) * c->h[a];
        in_lo = in_lo && (t >= 0.25 && t <= 0.5);
        in_hi = in_hi && (t >= 0.5 && t <= 0.75);
      }
      al[e] = 1.0;
      be[e] = (in_lo || in_hi) ? pow(10.0, (double)(int)p0) : 1.0;
    } else {
      set_err(c, "unknown coef kind %s", kind);
      return 1;
    }
  }
  double* f = put_arr(c, "f_hat", 'd', c->broken);
  for (long long i = 0; i < c->broken; ++i) f[i] = rng_uniform2(&r, -1.0, 1.0);
  double* lam = put_arr(c, "lambda", 'd', c->m);
  for (long long i = 0; i < c->m; ++i) lam[i] = rng_uniform2(&r, -1.0, 1.0);
  double* xb = put_arr(c, "x_b", 'd', c->nS);
  for (long long i = 0; i < c->nS; ++i) xb[i] = rng_uniform2(&r, -1.0, 1.0);
  /* config 4: ";perturb=f" displaces every interior vertex
   * coordinate by U[-f h, f h], vertices lexicographic (x fastest), x then y then
   * z, drawn after all other inputs; boundary vertices stay fixed */
  const char* pt = strstr(coef, ";perturb=");
  if (pt && c->dim == 3) {
    const double frac = atof(pt + 9);
    const long long nv0 = c->N[0] + 1, nv1 = c->N[1] + 1, nv2 = c->N[2] + 1;
    double* vtx = put_arr(c, "vertices", 'd', nv0 * nv1 * nv2 * 3);
    for (long long iz = 0; iz < nv2; ++iz)
      for (long long iy = 0; iy < nv1; ++iy)
        for (long long ix = 0; ix < nv0; ++ix) {
          const long long g = ix + nv0 * (iy + nv1 * iz);
          const long long idx[3] = {ix, iy, iz};
          int interior = 1;
          for (int a = 0; a < 3; ++a)
            if (idx[a] == 0 || idx[a] == c->N[a]) interior = 0;
          for (int a = 0; a < 3; ++a) {
            vtx[3 * g + a] = (double)idx[a] * c->h[a];
            if (interior) vtx[3 * g + a] += rng_uniform2(&r, -frac * c->h[a], frac * c->h[a]);
          }
        }
  }
  return 0;
}

/* A_T = fl(fl(alpha*divdiv) + fl(beta*mass)) — rt_space.cpp:356-357 through
 * dense_add (dense.cpp:37-42): c = 0 + alpha*D; c += beta*M */
int hdo_element_matrix(hdo_ctx* c, long long cell, double* a_t) {
  const double* al = get_d(c, "alpha");
  const double* be = get_d(c, "beta");
  const double* ahat = get_d(c, "a_hat");
  const long long n = c->n;
  if (ahat && hdo_count(c, "a_hat") == c->ncells * n * n) {
    memcpy(a_t, ahat + cell * n * n, (size_t)(n * n) * 8);
    return 0;
  }
  /* a_sel / a_sel_blocks: explicit blocks for a few cells (test-scale parity on
   * full-size meshes: the device's A_T of the sampled cells) */
  const double* sel = get_d(c, "a_sel");
  const double* sblk = get_d(c, "a_sel_blocks");
  if (sel && sblk) {
    const long long ns = hdo_count(c, "a_sel");
    for (long long q = 0; q < ns; ++q)
      if ((long long)sel[q] == cell && hdo_count(c, "a_sel_blocks") >= (q + 1) * n * n) {
        memcpy(a_t, sblk + q * n * n, (size_t)(n * n) * 8);
        return 0;
      }
  }
  if (!al || !be) {
    set_err(c, "alpha/beta not set");
    return 1;
  }
  const double alpha = al[cell], beta = be[cell];
  const double* vtx = get_d(c, "vertices");
  const double* D = c->divdiv;
  const double* M = c->mass;
  double* dm = NULL;
  if (vtx && c->dim == 3) { /* perturbed trilinear cell (config 4): Piola element matrices */
    dm = malloc((size_t)(2 * n * n) * 8);
    double verts[24];
    cell_vertices(c, vtx, cell, verts);
    if (hdo_piola_element(c->k, c->h, verts, c->k + 2, dm, dm + n * n, NULL, NULL) != 0) {
      free(dm);
      set_err(c, "piola element failed");
      return 1;
    }
    D = dm;
    M = dm + n * n;
  }
  for (long long i = 0; i < n * n; ++i) {
    double v = 0.0;
    v += alpha * D[i];
    v += beta * M[i];
    a_t[i] = v;
  }
  free(dm);
  return 0;
}

/* multiplier_base (reduction.cpp:88-98) */
static long long* mult_base(hdo_ctx* c) {
  long long* base = get_q(c, "mult_base");
  if (base) return base;
  base = put_arr(c, "mult_base", 'q', c->nfaces);
  long long next = 0;
  for (long long f = 0; f < c->nfaces; ++f) {
    int ax;
    long long cm, cp;
    face_info(c, f, &ax, &cm, &cp);
    if (cm >= 0 && cp >= 0) {
      base[f] = next;
      next += c->dpf;
    } else {
      base[f] = -1;
    }
  }
  return base;
}

/* build_P (reduction.cpp:136-150) and build_C (reduction.cpp:152-198); C rows
 * are emitted in sorted (row, col) order directly, equal to from_triplets. */
static int run_structure(hdo_ctx* c) {
  const long long n = c->n, dpf = c->dpf;
  long long* gl = put_arr(c, "dof_global", 'q', c->broken);
  double* sg = put_arr(c, "dof_sign", 'd', c->broken);
  for (long long e = 0; e < c->ncells; ++e) local_dof_map(c, e, gl + e * n, sg + e * n);
  long long* pr = put_arr(c, "P.row_offsets", 'q', c->broken + 1);
  long long* pc = put_arr(c, "P.col_indices", 'q', c->broken);
  double* pv = put_arr(c, "P.values", 'd', c->broken);
  for (long long r = 0; r < c->broken; ++r) {
    pr[r + 1] = r + 1;
    pc[r] = gl[r];
    pv[r] = sg[r];
  }
  long long* ps = put_arr(c, "P.shape", 'q', 2);
  ps[0] = c->broken;
  ps[1] = c->ndofs;

  long long* base = mult_base(c);
  const long long per = c->weighted ? 2 * dpf : 2;
  long long* cr = put_arr(c, "C.row_offsets", 'q', c->m + 1);
  long long* cc = put_arr(c, "C.col_indices", 'q', c->m * per);
  double* cv = put_arr(c, "C.values", 'd', c->m * per);
  long long* cs = put_arr(c, "C.shape", 'q', 2);
  cs[0] = c->m;
  cs[1] = c->broken;
  for (long long r = 0; r <= c->m; ++r) cr[r] = r * per;
  for (long long f = 0; f < c->nfaces; ++f) {
    if (base[f] < 0) continue;
    int ax;
    long long cm, cp;
    face_info(c, f, &ax, &cm, &cp);
    const int sm = 2 * ax + 1, sp = 2 * ax;
    const long long lm = c->nint + sm * dpf, lp = c->nint + sp * dpf;
    const long long offm = cm * n, offp = cp * n;
    const double* fmm = c->face_moments + (long long)sm * dpf * n;
    const double* fmp = c->face_moments + (long long)sp * dpf * n;
    for (long long r = 0; r < dpf; ++r) {
      long long pos = (base[f] + r) * per;
      if (!c->weighted) {
        cc[pos] = offm + lm + r;
        cv[pos] = 1.0;
        cc[pos + 1] = offp + lp + r;
        cv[pos + 1] = 1.0;
      } else {
        for (long long s = 0; s < dpf; ++s) {
          cc[pos + s] = offm + lm + s;
          cv[pos + s] = fmm[r * n + lm + s];
          cc[pos + dpf + s] = offp + lp + s;
          cv[pos + dpf + s] = fmp[r * n + lp + s];
        }
      }
    }
  }
  return 0;
}

/* ------------------------------------------------- triplets → CSR (csr.cpp:43-75) */

typedef struct {
  long long r, c;
  double v;
} trip_t;
static int trip_cmp(const void* a, const void* b) {
  const trip_t* x = a;
  const trip_t* y = b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return 0;
}
static void csr_from_triplets(hdo_ctx* c, const char* prefix, long long nrows, long long ncols, trip_t* t,
                              long long nt) {
  qsort(t, (size_t)nt, sizeof *t, trip_cmp);
  long long nnz = 0;
  for (long long i = 0; i < nt; ++i)
    if (i == 0 || t[i].r != t[i - 1].r || t[i].c != t[i - 1].c) ++nnz;
  char nm[64];
  snprintf(nm, sizeof nm, "%s.row_offsets", prefix);
  long long* ro = put_arr(c, nm, 'q', nrows + 1);
  snprintf(nm, sizeof nm, "%s.col_indices", prefix);
  long long* ci = put_arr(c, nm, 'q', nnz);
  snprintf(nm, sizeof nm, "%s.values", prefix);
  double* va = put_arr(c, nm, 'd', nnz);
  snprintf(nm, sizeof nm, "%s.shape", prefix);
  long long* sh = put_arr(c, nm, 'q', 2);
  sh[0] = nrows;
  sh[1] = ncols;
  long long k = -1;
  for (long long i = 0; i < nt; ++i) {
    if (i > 0 && t[i].r == t[i - 1].r && t[i].c == t[i - 1].c) {
      va[k] += t[i].v;
    } else {
      ++k;
      ci[k] = t[i].c;
      va[k] = t[i].v;
      ro[t[i].r + 1] += 1;
    }
  }
  for (long long i = 0; i < nrows; ++i) ro[i + 1] += ro[i];
}

static long long csr_find(const long long* ro, const long long* ci, long long r, long long col) {
  long long lo = ro[r], hi = ro[r + 1] - 1;
  while (lo <= hi) {
    const long long mid = (lo + hi) / 2;
    if (ci[mid] == col) return mid;
    if (ci[mid] < col)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  return -1;
}

/* ------------------------------------------------------------ port: hybridize */

static double* gather_sub(const double* a, long long n, const long long* rows, long long nr, const long long* cols,
                          long long nc) {
  double* s = malloc((size_t)(nr * nc + 1) * 8);
  for (long long i = 0; i < nr; ++i)
    for (long long j = 0; j < nc; ++j) s[i * nc + j] = a[rows[i] * n + cols[j]];
  return s;
}

/* the element's constrained local dofs and sorted multiplier rows: C columns
 * off+l with entries (constraint_slice, reduction.cpp:31-57) */
static void element_partition(hdo_ctx* c, long long e, long long* i_local, long long* ni, long long* b_local,
                              long long* nb, long long* rows, long long* nr) {
  const long long* cr = get_q(c, "C.row_offsets");
  const long long* cc = get_q(c, "C.col_indices");
  long long faces[6];
  double fs[6];
  cell_faces(c, e, faces, fs);
  long long* base = mult_base(c);
  *ni = *nb = *nr = 0;
  for (long long l = 0; l < c->nint; ++l) i_local[(*ni)++] = l;
  for (int s = 0; s < 2 * c->dim; ++s) {
    const long long mb = base[faces[s]];
    for (long long sub = 0; sub < c->dpf; ++sub) {
      const long long l = c->nint + s * c->dpf + sub;
      if (mb < 0) {
        i_local[(*ni)++] = l;
      } else {
        b_local[(*nb)++] = l;
      }
    }
    if (mb >= 0)
      for (long long sub = 0; sub < c->dpf; ++sub) rows[(*nr)++] = mb + sub;
  }
  (void)cr;
  (void)cc;
  /* rows come out ascending: slot order is ascending face order */
}

static int run_port_hybridize(hdo_ctx* c) {
  if (!get_q(c, "C.row_offsets")) run_structure(c);
  free_port(c);
  const long long n = c->n;
  const long long* cr = get_q(c, "C.row_offsets");
  const long long* cc = get_q(c, "C.col_indices");
  const double* cv = get_d(c, "C.values");
  const double* f_hat = get_d(c, "f_hat");
  if (!f_hat) {
    set_err(c, "f_hat not set");
    return 1;
  }
  c->pe = calloc((size_t)c->ncells, sizeof(port_elem));
  double* a = malloc((size_t)(n * n) * 8);
  long long max_nr = 2 * c->dim * c->dpf;
  trip_t* trips = malloc((size_t)(c->ncells * max_nr * max_nr + 1) * sizeof(trip_t));
  long long nt = 0;
  double* g = put_arr(c, "g", 'd', c->m);
  double* work = malloc((size_t)(8 * n + 8) * 8);
  for (long long e = 0; e < c->ncells; ++e) {
    port_elem* p = &c->pe[e];
    if (hdo_element_matrix(c, e, a)) return 1;
    p->i_local = malloc((size_t)(n + 1) * sizeof(long long));
    p->b_local = malloc((size_t)(n + 1) * sizeof(long long));
    p->rows = malloc((size_t)(n + 1) * sizeof(long long));
    element_partition(c, e, p->i_local, &p->ni, p->b_local, &p->nb, p->rows, &p->nr);
    const long long ni = p->ni, nb = p->nb, nr = p->nr;
    double* a_bb = gather_sub(a, n, p->b_local, nb, p->b_local, nb);
    p->a_ib = gather_sub(a, n, p->i_local, ni, p->b_local, nb);
    p->a_bi = gather_sub(a, n, p->b_local, nb, p->i_local, ni);
    p->a_ii = gather_sub(a, n, p->i_local, ni, p->i_local, ni);
    p->a_ii_lu = malloc((size_t)(ni * ni + 1) * 8);
    memcpy(p->a_ii_lu, p->a_ii, (size_t)(ni * ni) * 8);
    p->a_ii_piv = malloc((size_t)(ni + 1) * sizeof(long long));
    if (lu_factor(p->a_ii_lu, ni, p->a_ii_piv) >= 0) {
      set_err(c, "SingularBlock: element %lld A_ii", e);
      free(a_bb);
      return 2;
    }
    double* schur = a_bb;
    if (ni > 0 && nb > 0) {
      double* X = malloc((size_t)(ni * nb) * 8);
      solve_matrix_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, ni, p->a_ib, nb, X);
      double* prod = malloc((size_t)(nb * nb) * 8);
      dense_multiply(p->a_bi, X, nb, ni, nb, prod);
      for (long long i = 0; i < nb * nb; ++i) schur[i] += -1.0 * prod[i];
      symmetrize(schur, nb);
      free(X);
      free(prod);
    }
    p->s_b = schur;
    p->s_b_lu = malloc((size_t)(nb * nb + 1) * 8);
    memcpy(p->s_b_lu, schur, (size_t)(nb * nb) * 8);
    p->s_b_piv = malloc((size_t)(nb + 1) * sizeof(long long));
    if (lu_factor(p->s_b_lu, nb, p->s_b_piv) >= 0) {
      set_err(c, "SingularBlock: element %lld S_b", e);
      return 2;
    }
    /* c_b (nr x nb) */
    p->c_b = calloc((size_t)(nr * nb + 1), 8);
    for (long long r = 0; r < nr; ++r) {
      const long long row = p->rows[r];
      for (long long j = 0; j < nb; ++j) {
        const long long target = e * n + p->b_local[j];
        for (long long q = cr[row]; q < cr[row + 1]; ++q) {
          if (cc[q] == target) {
            p->c_b[r * nb + j] = cv[q];
            break;
          }
          if (cc[q] > target) break;
        }
      }
    }
  }
  /* serial fixed-order accumulation (reduction.cpp:304-337) */
  for (long long e = 0; e < c->ncells; ++e) {
    port_elem* p = &c->pe[e];
    const long long ni = p->ni, nb = p->nb, nr = p->nr;
    const long long off = e * n;
    if (nr > 0) {
      double* cbt = malloc((size_t)(nb * nr) * 8);
      for (long long r = 0; r < nr; ++r)
        for (long long j = 0; j < nb; ++j) cbt[j * nr + r] = p->c_b[r * nb + j];
      double* X = malloc((size_t)(nb * nr) * 8);
      solve_matrix_refined(p->s_b, p->s_b_lu, p->s_b_piv, nb, cbt, nr, X);
      double* he = malloc((size_t)(nr * nr) * 8);
      dense_multiply(p->c_b, X, nr, nb, nr, he);
      symmetrize(he, nr);
      for (long long r = 0; r < nr; ++r)
        for (long long q = 0; q < nr; ++q) {
          trips[nt].r = p->rows[r];
          trips[nt].c = p->rows[q];
          trips[nt].v = he[r * nr + q];
          ++nt;
        }
      free(cbt);
      free(X);
      free(he);
    }
    double* fi = work;
    double* fb = fi + n;
    double* xi0 = fb + n;
    double* corr = xi0 + n;
    double* xb = corr + n;
    double* ge = xb + n;
    double* wk = ge + n;
    for (long long i = 0; i < ni; ++i) fi[i] = f_hat[off + p->i_local[i]];
    for (long long j = 0; j < nb; ++j) fb[j] = f_hat[off + p->b_local[j]];
    lu_solve_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, ni, fi, xi0, wk);
    dense_apply(p->a_bi, nb, ni, xi0, corr);
    for (long long j = 0; j < nb; ++j) fb[j] -= corr[j];
    lu_solve_refined(p->s_b, p->s_b_lu, p->s_b_piv, nb, fb, xb, wk);
    dense_apply(p->c_b, nr, nb, xb, ge);
    for (long long r = 0; r < nr; ++r) g[p->rows[r]] += ge[r];
  }
  csr_from_triplets(c, "H", c->m, c->m, trips, nt);
  free(trips);
  free(work);
  free(a);
  return 0;
}

/* recover_hybrid (reduction.cpp:356-446), injection-P branch */
static int run_port_recover(hdo_ctx* c) {
  if (!c->pe) {
    set_err(c, "port_hybridize first");
    return 1;
  }
  const long long n = c->n;
  const double* lam = get_d(c, "lambda");
  const double* f_hat = get_d(c, "f_hat");
  if (!lam) {
    set_err(c, "lambda not set");
    return 1;
  }
  double* xh = put_arr(c, "x_hat", 'd', c->broken);
  double* work = malloc((size_t)(10 * n + 8) * 8);
  for (long long e = 0; e < c->ncells; ++e) {
    port_elem* p = &c->pe[e];
    const long long ni = p->ni, nb = p->nb, nr = p->nr, off = e * n;
    double* rhs = work;
    double* fi = rhs + n;
    double* xi0 = fi + n;
    double* corr = xi0 + n;
    double* xb = corr + n;
    double* xi = xb + n;
    double* fix = xi + n;
    double* wk = fix + n;
    for (long long j = 0; j < nb; ++j) rhs[j] = f_hat[off + p->b_local[j]];
    for (long long r = 0; r < nr; ++r) {
      const double lr = lam[p->rows[r]];
      if (lr == 0.0) continue;
      for (long long j = 0; j < nb; ++j) rhs[j] -= p->c_b[r * nb + j] * lr;
    }
    for (long long i = 0; i < ni; ++i) fi[i] = f_hat[off + p->i_local[i]];
    lu_solve_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, ni, fi, xi0, wk);
    dense_apply(p->a_bi, nb, ni, xi0, corr);
    for (long long j = 0; j < nb; ++j) rhs[j] -= corr[j];
    lu_solve_refined(p->s_b, p->s_b_lu, p->s_b_piv, nb, rhs, xb, wk);
    memcpy(xi, xi0, (size_t)ni * 8);
    if (ni > 0 && nb > 0) {
      dense_apply(p->a_ib, ni, nb, xb, corr);
      lu_solve_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, ni, corr, fix, wk);
      for (long long i = 0; i < ni; ++i) xi[i] -= fix[i];
    }
    for (long long i = 0; i < ni; ++i) xh[off + p->i_local[i]] = xi[i];
    for (long long j = 0; j < nb; ++j) xh[off + p->b_local[j]] = xb[j];
  }
  free(work);
  /* x = (P^T P)^-1 P^T x_hat; diagonal Gram for the FE P */
  const long long* gl = get_q(c, "dof_global");
  const double* sg = get_d(c, "dof_sign");
  double* x = put_arr(c, "x", 'd', c->ndofs);
  double* scale = calloc((size_t)c->ndofs, 8);
  for (long long r = 0; r < c->broken; ++r) scale[gl[r]] += sg[r] * sg[r];
  for (long long i = 0; i < c->ndofs; ++i) scale[i] = 1.0 / scale[i];
  for (long long r = 0; r < c->broken; ++r) x[gl[r]] += sg[r] * xh[r];
  for (long long i = 0; i < c->ndofs; ++i) x[i] *= scale[i];
  free(scale);
  return 0;
}

/* static_condense (reduction.cpp:448-557), marker partition i = bubbles */
static int run_port_condense(hdo_ctx* c) {
  if (!get_q(c, "dof_global")) run_structure(c);
  free_port(c);
  const long long n = c->n;
  const long long* gl = get_q(c, "dof_global");
  const double* sg = get_d(c, "dof_sign");
  const double* f_hat = get_d(c, "f_hat");
  const long long marker = c->face_dof_count;
  c->ce = calloc((size_t)c->ncells, sizeof(cond_elem));
  double* a = malloc((size_t)(n * n) * 8);
  double* work = malloc((size_t)(6 * n + 8) * 8);
  for (long long e = 0; e < c->ncells; ++e) {
    cond_elem* p = &c->ce[e];
    const long long off = e * n;
    if (hdo_element_matrix(c, e, a)) return 1;
    p->i_local = malloc((size_t)(n + 1) * sizeof(long long));
    p->b_local = malloc((size_t)(n + 1) * sizeof(long long));
    p->ni = p->nb = 0;
    for (long long l = 0; l < n; ++l) {
      if (gl[off + l] < marker)
        p->b_local[p->nb++] = l;
      else
        p->i_local[p->ni++] = l;
    }
    const long long ni = p->ni, nb = p->nb;
    double* a_bb = gather_sub(a, n, p->b_local, nb, p->b_local, nb);
    p->a_ib = gather_sub(a, n, p->i_local, ni, p->b_local, nb);
    double* a_bi = gather_sub(a, n, p->b_local, nb, p->i_local, ni);
    p->a_ii = gather_sub(a, n, p->i_local, ni, p->i_local, ni);
    p->a_ii_lu = malloc((size_t)(ni * ni + 1) * 8);
    memcpy(p->a_ii_lu, p->a_ii, (size_t)(ni * ni) * 8);
    p->a_ii_piv = malloc((size_t)(ni + 1) * sizeof(long long));
    if (lu_factor(p->a_ii_lu, ni, p->a_ii_piv) >= 0) {
      set_err(c, "SingularBlock: element %lld A_ii", e);
      return 2;
    }
    p->schur = a_bb;
    p->f_s = malloc((size_t)(nb + 1) * 8);
    for (long long j = 0; j < nb; ++j) p->f_s[j] = f_hat[off + p->b_local[j]];
    if (ni > 0) {
      if (nb > 0) {
        double* X = malloc((size_t)(ni * nb) * 8);
        solve_matrix_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, ni, p->a_ib, nb, X);
        double* prod = malloc((size_t)(nb * nb) * 8);
        dense_multiply(a_bi, X, nb, ni, nb, prod);
        for (long long i = 0; i < nb * nb; ++i) p->schur[i] += -1.0 * prod[i];
        symmetrize(p->schur, nb);
        free(X);
        free(prod);
      }
      double* fi = work;
      double* xs = fi + n;
      double* corr = xs + n;
      double* wk = corr + n;
      for (long long i = 0; i < ni; ++i) fi[i] = f_hat[off + p->i_local[i]];
      lu_solve_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, ni, fi, xs, wk);
      dense_apply(a_bi, nb, ni, xs, corr);
      for (long long j = 0; j < nb; ++j) p->f_s[j] -= corr[j];
    }
    free(a_bi);
    p->i_global = malloc((size_t)(ni + 1) * sizeof(long long));
    p->i_sign = malloc((size_t)(ni + 1) * 8);
    for (long long i = 0; i < ni; ++i) {
      p->i_global[i] = gl[off + p->i_local[i]];
      p->i_sign[i] = sg[off + p->i_local[i]];
    }
  }
  /* masters (reduction.cpp:509-521) */
  char* is_master = calloc((size_t)c->ndofs, 1);
  for (long long e = 0; e < c->ncells; ++e)
    for (long long j = 0; j < c->ce[e].nb; ++j) is_master[gl[e * n + c->ce[e].b_local[j]]] = 1;
  long long nm = 0;
  for (long long g = 0; g < c->ndofs; ++g) nm += is_master[g];
  long long* mg = put_arr(c, "master_globals", 'q', nm);
  long long* ord = malloc((size_t)c->ndofs * sizeof(long long));
  nm = 0;
  for (long long g = 0; g < c->ndofs; ++g) {
    ord[g] = -1;
    if (is_master[g]) {
      mg[nm] = g;
      ord[g] = nm++;
    }
  }
  long long nt = 0;
  for (long long e = 0; e < c->ncells; ++e) nt += c->ce[e].nb * c->ce[e].nb;
  trip_t* t = malloc((size_t)(nt + 1) * sizeof(trip_t));
  double* fs = put_arr(c, "f_s", 'd', nm);
  nt = 0;
  for (long long e = 0; e < c->ncells; ++e) {
    cond_elem* p = &c->ce[e];
    const long long nb = p->nb;
    p->b_master_ord = malloc((size_t)(nb + 1) * sizeof(long long));
    p->b_master_sign = malloc((size_t)(nb + 1) * 8);
    for (long long j = 0; j < nb; ++j) {
      p->b_master_ord[j] = ord[gl[e * n + p->b_local[j]]];
      p->b_master_sign[j] = sg[e * n + p->b_local[j]];
    }
    for (long long i = 0; i < nb; ++i) {
      for (long long j = 0; j < nb; ++j) {
        t[nt].r = p->b_master_ord[i];
        t[nt].c = p->b_master_ord[j];
        t[nt].v = p->b_master_sign[i] * p->b_master_sign[j] * p->schur[i * nb + j];
        ++nt;
      }
      fs[p->b_master_ord[i]] += p->b_master_sign[i] * p->f_s[i];
    }
  }
  csr_from_triplets(c, "S", nm, nm, t, nt);
  free(t);
  free(ord);
  free(is_master);
  free(a);
  free(work);
  return 0;
}

/* recover_condensed (reduction.cpp:559-587) */
static int run_port_recover_condensed(hdo_ctx* c) {
  if (!c->ce) {
    set_err(c, "port_condense first");
    return 1;
  }
  const long long n = c->n;
  const double* xbv = get_d(c, "x_b");
  const double* f_hat = get_d(c, "f_hat");
  const long long* mg = get_q(c, "master_globals");
  const long long nm = hdo_count(c, "master_globals");
  if (!xbv || hdo_count(c, "x_b") != nm) {
    set_err(c, "x_b not set / wrong length");
    return 1;
  }
  double* x = put_arr(c, "x_cond", 'd', c->ndofs);
  for (long long o = 0; o < nm; ++o) x[mg[o]] = xbv[o];
  double* work = malloc((size_t)(6 * n + 8) * 8);
  for (long long e = 0; e < c->ncells; ++e) {
    cond_elem* p = &c->ce[e];
    if (p->ni == 0) continue;
    const long long off = e * n;
    double* xbl = work;
    double* rhs = xbl + n;
    double* corr = rhs + n;
    double* xi = corr + n;
    double* wk = xi + n;
    for (long long j = 0; j < p->nb; ++j) {
      xbl[j] = 0.0;
      xbl[j] += p->b_master_sign[j] * xbv[p->b_master_ord[j]];
    }
    for (long long i = 0; i < p->ni; ++i) rhs[i] = f_hat[off + p->i_local[i]];
    if (p->nb > 0) {
      dense_apply(p->a_ib, p->ni, p->nb, xbl, corr);
      for (long long i = 0; i < p->ni; ++i) rhs[i] -= corr[i];
    }
    lu_solve_refined(p->a_ii, p->a_ii_lu, p->a_ii_piv, p->ni, rhs, xi, wk);
    for (long long i = 0; i < p->ni; ++i) x[p->i_global[i]] = xi[i] / p->i_sign[i];
  }
  free(work);
  return 0;
}

static int run_spmv(hdo_ctx* c, const char* pre, const char* xname, const char* yname) {
  char nm[64];
  snprintf(nm, sizeof nm, "%s.row_offsets", pre);
  const long long* ro = get_q(c, nm);
  snprintf(nm, sizeof nm, "%s.col_indices", pre);
  const long long* ci = get_q(c, nm);
  snprintf(nm, sizeof nm, "%s.values", pre);
  const double* va = get_d(c, nm);
  const double* x = get_d(c, xname);
  snprintf(nm, sizeof nm, "%s.shape", pre);
  const long long* sh = get_q(c, nm);
  if (!ro || !x) {
    set_err(c, "spmv inputs missing");
    return 1;
  }
  double* y = put_arr(c, yname, 'd', sh[0]);
  for (long long i = 0; i < sh[0]; ++i) {
    double s = 0.0;
    for (long long k = ro[i]; k < ro[i + 1]; ++k) s += va[k] * x[ci[k]];
    y[i] = s;
  }
  return 0;
}

/* ------------------------------------------- double-double (include/hdivred/dd.hpp) */

typedef struct {
  double hi, lo;
} dd;
static inline dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  dd r = {s, (a - (s - bb)) + (b - bb)};
  return r;
}
static inline dd dd_quick(double a, double b) {
  const double s = a + b;
  dd r = {s, b - (s - a)};
  return r;
}
static inline dd dd_two_prod(double a, double b) {
  const double p = a * b;
  dd r = {p, fma(a, b, -p)};
  return r;
}
static inline dd dd_add(dd x, dd y) {
  dd s = dd_two_sum(x.hi, y.hi);
  s.lo += x.lo + y.lo;
  return dd_quick(s.hi, s.lo);
}
static inline dd dd_neg(dd x) {
  dd r = {-x.hi, -x.lo};
  return r;
}
static inline dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
static inline dd dd_mul(dd x, dd y) {
  dd p = dd_two_prod(x.hi, y.hi);
  p.lo += x.hi * y.lo + x.lo * y.hi;
  return dd_quick(p.hi, p.lo);
}
static inline dd dd_from(double x) {
  dd r = {x, 0.0};
  return r;
}
static inline dd dd_div(dd x, dd y) {
  const double q1 = x.hi / y.hi;
  dd r = dd_sub(x, dd_mul(dd_from(q1), y));
  const double q2 = r.hi / y.hi;
  r = dd_sub(r, dd_mul(dd_from(q2), y));
  const double q3 = r.hi / y.hi;
  dd q = dd_quick(q1, q2);
  return dd_add(q, dd_from(q3));
}

/* dd_lu_factor / dd_lu_solve (src/reference.cpp:11-48) */
static int dd_lu_factor(dd* a, long long n, long long* piv) {
  for (long long k = 0; k < n; ++k) {
    long long p = k;
    for (long long i = k + 1; i < n; ++i)
      if (fabs(a[i * n + k].hi) > fabs(a[p * n + k].hi)) p = i;
    if (a[p * n + k].hi == 0.0) return 1;
    piv[k] = p;
    if (p != k)
      for (long long j = 0; j < n; ++j) {
        const dd t = a[k * n + j];
        a[k * n + j] = a[p * n + j];
        a[p * n + j] = t;
      }
    for (long long i = k + 1; i < n; ++i) {
      const dd l = dd_div(a[i * n + k], a[k * n + k]);
      a[i * n + k] = l;
      if (l.hi == 0.0 && l.lo == 0.0) continue;
      for (long long j = k + 1; j < n; ++j) a[i * n + j] = dd_sub(a[i * n + j], dd_mul(l, a[k * n + j]));
    }
  }
  return 0;
}
static void dd_lu_solve(const dd* lu, const long long* piv, long long n, dd* b) {
  for (long long k = 0; k < n; ++k) {
    const long long p = piv[k];
    if (p != k) {
      const dd t = b[k];
      b[k] = b[p];
      b[p] = t;
    }
  }
  for (long long k = 0; k < n; ++k) {
    const dd bk = b[k];
    if (bk.hi == 0.0 && bk.lo == 0.0) continue;
    for (long long i = k + 1; i < n; ++i) b[i] = dd_sub(b[i], dd_mul(lu[i * n + k], bk));
  }
  for (long long i = n - 1; i >= 0; --i) {
    dd s = b[i];
    for (long long j = i + 1; j < n; ++j) s = dd_sub(s, dd_mul(lu[i * n + j], b[j]));
    b[i] = dd_div(s, lu[i * n + i]);
  }
}

/* Element-wise DD on the full A_T: X = A^-1 C_T^T, H_T = C_T X, g_T = C_T A^-1 f_T,
 * x_hat_T = A^-1 (f_T - C_T^T lambda).  C_T is the element's constraint slice over
 * ALL its local dofs (rows x n), taken from the C CSR. */
static int dd_element(hdo_ctx* c, long long e, long long* rows_out, dd* h_out, dd* g_out, dd* xh_out) {
  if (!get_q(c, "C.row_offsets")) run_structure(c);
  const long long n = c->n;
  const long long* cr = get_q(c, "C.row_offsets");
  const long long* cc = get_q(c, "C.col_indices");
  const double* cv = get_d(c, "C.values");
  const double* f_hat = get_d(c, "f_hat");
  const double* lam = get_d(c, "lambda");
  long long il[512], bl[512], rows[512], ni, nb, nr;
  element_partition(c, e, il, &ni, bl, &nb, rows, &nr);
  double* a = malloc((size_t)(n * n) * 8);
  if (hdo_element_matrix(c, e, a)) {
    free(a);
    return -1;
  }
  dd* A = malloc((size_t)(n * n) * sizeof(dd));
  for (long long i = 0; i < n * n; ++i) A[i] = dd_from(a[i]);
  long long* piv = malloc((size_t)n * sizeof(long long));
  if (dd_lu_factor(A, n, piv)) {
    set_err(c, "SingularBlock: dd element %lld", e);
    free(a);
    free(A);
    free(piv);
    return -2;
  }
  /* dense C_T (nr x n) */
  double* ct = calloc((size_t)(nr * n + 1), 8);
  for (long long r = 0; r < nr; ++r)
    for (long long q = cr[rows[r]]; q < cr[rows[r] + 1]; ++q) {
      const long long col = cc[q] - e * n;
      if (col >= 0 && col < n) ct[r * n + col] = cv[q];
    }
  dd* X = malloc((size_t)(n * (nr + 2) + 1) * sizeof(dd));
  dd* col = malloc((size_t)n * sizeof(dd));
  for (long long q = 0; q < nr; ++q) {
    for (long long i = 0; i < n; ++i) col[i] = dd_from(ct[q * n + i]);
    dd_lu_solve(A, piv, n, col);
    for (long long i = 0; i < n; ++i) X[i * nr + q] = col[i];
  }
  if (h_out)
    for (long long r = 0; r < nr; ++r)
      for (long long q = 0; q < nr; ++q) {
        dd s = dd_from(0.0);
        for (long long i = 0; i < n; ++i)
          if (ct[r * n + i] != 0.0) s = dd_add(s, dd_mul(dd_from(ct[r * n + i]), X[i * nr + q]));
        h_out[r * nr + q] = s;
      }
  if (f_hat && g_out) {
    for (long long i = 0; i < n; ++i) col[i] = dd_from(f_hat[e * n + i]);
    dd_lu_solve(A, piv, n, col);
    for (long long r = 0; r < nr; ++r) {
      dd s = dd_from(0.0);
      for (long long i = 0; i < n; ++i)
        if (ct[r * n + i] != 0.0) s = dd_add(s, dd_mul(dd_from(ct[r * n + i]), col[i]));
      g_out[r] = s;
    }
  }
  if (f_hat && lam && xh_out) {
    for (long long i = 0; i < n; ++i) {
      dd s = dd_from(f_hat[e * n + i]);
      for (long long r = 0; r < nr; ++r)
        if (ct[r * n + i] != 0.0) s = dd_sub(s, dd_mul(dd_from(ct[r * n + i]), dd_from(lam[rows[r]])));
      col[i] = s;
    }
    dd_lu_solve(A, piv, n, col);
    for (long long i = 0; i < n; ++i) xh_out[i] = col[i];
  }
  for (long long r = 0; r < nr; ++r) rows_out[r] = rows[r];
  free(a);
  free(A);
  free(piv);
  free(ct);
  free(X);
  free(col);
  return (int)nr;
}

int hdo_dd_element(hdo_ctx* c, long long cell, long long* rows, double* h_t, double* g_t, double* x_hat_t) {
  const long long n = c->n;
  dd* h = malloc((size_t)(n * n + 1) * sizeof(dd));
  dd* g = malloc((size_t)(n + 1) * sizeof(dd));
  dd* xh = malloc((size_t)(n + 1) * sizeof(dd));
  const int has_lam = get_d(c, "lambda") != NULL;
  const int nr = dd_element(c, cell, rows, h, g, has_lam ? xh : NULL);
  if (nr >= 0) {
    if (h_t)
      for (long long i = 0; i < (long long)nr * nr; ++i) h_t[i] = h[i].hi + h[i].lo;
    if (g_t)
      for (int i = 0; i < nr; ++i) g_t[i] = g[i].hi + g[i].lo;
    if (x_hat_t && has_lam)
      for (long long i = 0; i < n; ++i) x_hat_t[i] = xh[i].hi + xh[i].lo;
  }
  free(h);
  free(g);
  free(xh);
  return nr;
}

static int run_dd_hybridize(hdo_ctx* c, int recover) {
  const long long* ro = get_q(c, "H.row_offsets");
  const long long* ci = get_q(c, "H.col_indices");
  if (!ro) {
    set_err(c, "dd_hybridize needs the H pattern (port_hybridize)");
    return 1;
  }
  const long long nnz = hdo_count(c, "H.col_indices");
  const long long n = c->n;
  dd* hv = calloc((size_t)(nnz + 1), sizeof(dd));
  dd* gv = calloc((size_t)(c->m + 1), sizeof(dd));
  dd* xh = recover ? calloc((size_t)(c->broken + 1), sizeof(dd)) : NULL;
  dd* h = malloc((size_t)(n * n + 1) * sizeof(dd));
  dd* g = malloc((size_t)(n + 1) * sizeof(dd));
  long long rows[512];
  for (long long e = 0; e < c->ncells; ++e) {
    const int nr = dd_element(c, e, rows, h, g, recover ? xh + e * n : NULL);
    if (nr < 0) {
      free(hv);
      free(gv);
      free(xh);
      free(h);
      free(g);
      return 2;
    }
    for (int r = 0; r < nr; ++r) {
      for (int q = 0; q < nr; ++q) {
        const long long pos = csr_find(ro, ci, rows[r], rows[q]);
        hv[pos] = dd_add(hv[pos], h[r * nr + q]);
      }
      gv[rows[r]] = dd_add(gv[rows[r]], g[r]);
    }
  }
  if (!recover) {
    double* o = put_arr(c, "H.values_dd", 'd', nnz);
    for (long long i = 0; i < nnz; ++i) o[i] = hv[i].hi + hv[i].lo;
    double* og = put_arr(c, "g_dd", 'd', c->m);
    for (long long i = 0; i < c->m; ++i) og[i] = gv[i].hi + gv[i].lo;
  } else {
    double* o = put_arr(c, "x_hat_dd", 'd', c->broken);
    for (long long i = 0; i < c->broken; ++i) o[i] = xh[i].hi + xh[i].lo;
    const long long* gl = get_q(c, "dof_global");
    const double* sg = get_d(c, "dof_sign");
    dd* x = calloc((size_t)c->ndofs, sizeof(dd));
    double* cnt = calloc((size_t)c->ndofs, 8);
    for (long long r = 0; r < c->broken; ++r) {
      x[gl[r]] = dd_add(x[gl[r]], dd_mul(dd_from(sg[r]), xh[r]));
      cnt[gl[r]] += sg[r] * sg[r];
    }
    double* ox = put_arr(c, "x_dd", 'd', c->ndofs);
    for (long long i = 0; i < c->ndofs; ++i) {
      const dd v = dd_div(x[i], dd_from(cnt[i]));
      ox[i] = v.hi + v.lo;
    }
    free(x);
    free(cnt);
  }
  free(hv);
  free(gv);
  free(xh);
  free(h);
  free(g);
  return 0;
}

/* DD static condensation per element: S_T = A_bb - A_bi A_ii^-1 A_ib,
 * f_S,T = f_b - A_bi A_ii^-1 f_i (marker partition), assembled with the P_b
 * signs in DD; plus x_i = A_ii^-1 (f_i - A_ib x_b) for recovery. */
static int run_dd_condense(hdo_ctx* c, int recover) {
  const long long* ro = get_q(c, "S.row_offsets");
  const long long* ci = get_q(c, "S.col_indices");
  if (!ro || !c->ce) {
    set_err(c, "dd_condense needs port_condense first");
    return 1;
  }
  const long long nnz = hdo_count(c, "S.col_indices");
  const long long nm = hdo_count(c, "master_globals");
  const long long n = c->n;
  const double* f_hat = get_d(c, "f_hat");
  const double* xbv = get_d(c, "x_b");
  dd* sv = calloc((size_t)(nnz + 1), sizeof(dd));
  dd* fv = calloc((size_t)(nm + 1), sizeof(dd));
  double* xo = recover ? put_arr(c, "x_cond_dd", 'd', c->ndofs) : NULL;
  if (recover) {
    const long long* mg = get_q(c, "master_globals");
    for (long long o = 0; o < nm; ++o) xo[mg[o]] = xbv[o];
  }
  double* a = malloc((size_t)(n * n) * 8);
  dd* Aii = malloc((size_t)(n * n) * sizeof(dd));
  dd* X = malloc((size_t)(n * n + 1) * sizeof(dd));
  dd* col = malloc((size_t)(n + 1) * sizeof(dd));
  long long* piv = malloc((size_t)(n + 1) * sizeof(long long));
  for (long long e = 0; e < c->ncells; ++e) {
    cond_elem* p = &c->ce[e];
    const long long ni = p->ni, nb = p->nb, off = e * n;
    hdo_element_matrix(c, e, a);
    for (long long i = 0; i < ni; ++i)
      for (long long j = 0; j < ni; ++j) Aii[i * ni + j] = dd_from(a[p->i_local[i] * n + p->i_local[j]]);
    if (ni > 0 && dd_lu_factor(Aii, ni, piv)) {
      set_err(c, "SingularBlock: dd element %lld A_ii", e);
      return 2;
    }
    if (!recover) {
      for (long long j = 0; j < nb; ++j) { /* X = A_ii^-1 A_ib (ni x nb) */
        for (long long i = 0; i < ni; ++i) col[i] = dd_from(a[p->i_local[i] * n + p->b_local[j]]);
        if (ni > 0) dd_lu_solve(Aii, piv, ni, col);
        for (long long i = 0; i < ni; ++i) X[i * nb + j] = col[i];
      }
      for (long long i = 0; i < ni; ++i) col[i] = dd_from(f_hat[off + p->i_local[i]]);
      if (ni > 0) dd_lu_solve(Aii, piv, ni, col);
      for (long long r = 0; r < nb; ++r) {
        const double sr = p->b_master_sign[r];
        for (long long q = 0; q < nb; ++q) {
          dd s = dd_from(a[p->b_local[r] * n + p->b_local[q]]);
          for (long long i = 0; i < ni; ++i)
            s = dd_sub(s, dd_mul(dd_from(a[p->b_local[r] * n + p->i_local[i]]), X[i * nb + q]));
          const long long pos = csr_find(ro, ci, p->b_master_ord[r], p->b_master_ord[q]);
          sv[pos] = dd_add(sv[pos], dd_mul(dd_from(sr * p->b_master_sign[q]), s));
        }
        dd fs = dd_from(f_hat[off + p->b_local[r]]);
        for (long long i = 0; i < ni; ++i)
          fs = dd_sub(fs, dd_mul(dd_from(a[p->b_local[r] * n + p->i_local[i]]), col[i]));
        fv[p->b_master_ord[r]] = dd_add(fv[p->b_master_ord[r]], dd_mul(dd_from(sr), fs));
      }
    } else if (ni > 0) {
      for (long long i = 0; i < ni; ++i) {
        dd s = dd_from(f_hat[off + p->i_local[i]]);
        for (long long j = 0; j < nb; ++j) {
          const double xbl = p->b_master_sign[j] * xbv[p->b_master_ord[j]];
          s = dd_sub(s, dd_mul(dd_from(a[p->i_local[i] * n + p->b_local[j]]), dd_from(xbl)));
        }
        col[i] = s;
      }
      dd_lu_solve(Aii, piv, ni, col);
      for (long long i = 0; i < ni; ++i) {
        const dd v = dd_div(col[i], dd_from(p->i_sign[i]));
        xo[p->i_global[i]] = v.hi + v.lo;
      }
    }
  }
  if (!recover) {
    double* o = put_arr(c, "S.values_dd", 'd', nnz);
    for (long long i = 0; i < nnz; ++i) o[i] = sv[i].hi + sv[i].lo;
    double* of = put_arr(c, "f_s_dd", 'd', nm);
    for (long long i = 0; i < nm; ++i) of[i] = fv[i].hi + fv[i].lo;
  }
  free(sv);
  free(fv);
  free(a);
  free(Aii);
  free(X);
  free(col);
  free(piv);
  return 0;
}

static int run_assemble(hdo_ctx* c) {
  const long long n = c->n;
  if (!get_d(c, "alpha")) {
    set_err(c, "alpha/beta not set");
    return 1;
  }
  /* drop any explicit a_hat so element_matrix assembles from alpha/beta */
  arr_t* old = find_arr(c, "a_hat");
  if (old) {
    free(old->data);
    old->data = NULL;
    old->count = 0;
  }
  double* tmp = malloc((size_t)(n * n) * 8);
  double* ah = malloc((size_t)(c->ncells * n * n) * 8);
  for (long long e = 0; e < c->ncells; ++e) {
    hdo_element_matrix(c, e, tmp);
    memcpy(ah + e * n * n, tmp, (size_t)(n * n) * 8);
  }
  hdo_set_d(c, "a_hat", ah, c->ncells * n * n);
  free(ah);
  free(tmp);
  return 0;
}

/* ------------------------------------------------ structure-only patterns
 * The CSR patterns from_triplets (csr.cpp:43-75: sorted by (row, col),
 * duplicates merged, explicit zeros kept) produces from the triplet sets of
 *   hybridize        (reduction.cpp:308-337): every pair (r, c) of an element's
 *                    sorted multiplier rows (constraint_slice, :31-57);
 *   static_condense  (reduction.cpp:509-555): every pair of master ordinals of
 *                    an element's b dofs (for FE inputs every face dof is a
 *                    master, ordinal = global face dof),
 * built row by row (a row's columns are the union of the lists of the <= 2
 * elements that reach it) without values, so full BASELINE sizes fit in memory:
 * "Hp.*" / "Sp.*" row_offsets + col_indices. */
static int cmp_ll(const void* a, const void* b) {
  const long long x = *(const long long*)a, y = *(const long long*)b;
  return x < y ? -1 : (x > y);
}
static long long merge_unique(const long long* a, long long na, const long long* b, long long nb, long long* out) {
  long long i = 0, j = 0, k = 0;
  while (i < na || j < nb) {
    long long v;
    if (j >= nb || (i < na && a[i] <= b[j])) v = a[i++];
    else v = b[j++];
    if (k == 0 || out[k - 1] != v) out[k++] = v;
  }
  return k;
}
/* the element's sorted list: multiplier rows (which = 0) or master ordinals (1) */
static long long elem_list(hdo_ctx* c, long long e, int which, long long* out) {
  long long faces[6];
  double fs[6];
  cell_faces(c, e, faces, fs);
  long long* base = mult_base(c);
  long long k = 0;
  for (int s = 0; s < 2 * c->dim; ++s) {
    if (which == 0) {
      if (base[faces[s]] < 0) continue;
      for (long long sub = 0; sub < c->dpf; ++sub) out[k++] = base[faces[s]] + sub;
    } else {
      for (long long sub = 0; sub < c->dpf; ++sub) out[k++] = faces[s] * c->dpf + sub;
    }
  }
  qsort(out, (size_t)k, sizeof *out, cmp_ll);
  return k;
}
static int run_pattern(hdo_ctx* c, int which) {
  const long long nrows = which == 0 ? c->m : c->face_dof_count;
  long long* base = mult_base(c);
  /* owner elements of each row's face */
  long long* rcell = malloc((size_t)(2 * nrows + 2) * sizeof(long long));
  for (long long r = 0; r < 2 * nrows; ++r) rcell[r] = -1;
  for (long long f = 0; f < c->nfaces; ++f) {
    int ax;
    long long cm, cp;
    face_info(c, f, &ax, &cm, &cp);
    if (which == 0 && base[f] < 0) continue;
    for (long long sub = 0; sub < c->dpf; ++sub) {
      const long long r = which == 0 ? base[f] + sub : f * c->dpf + sub;
      rcell[2 * r] = cm;
      rcell[2 * r + 1] = cp;
    }
  }
  long long la[96], lb[96], tmp[192];
  const char* pre = which == 0 ? "Hp" : "Sp";
  char nm[64];
  snprintf(nm, sizeof nm, "%s.row_offsets", pre);
  long long* ro = put_arr(c, nm, 'q', nrows + 1);
  ro[0] = 0;
  for (long long r = 0; r < nrows; ++r) {
    const long long na = rcell[2 * r] >= 0 ? elem_list(c, rcell[2 * r], which, la) : 0;
    const long long nb = rcell[2 * r + 1] >= 0 ? elem_list(c, rcell[2 * r + 1], which, lb) : 0;
    ro[r + 1] = ro[r] + merge_unique(la, na, lb, nb, tmp);
  }
  snprintf(nm, sizeof nm, "%s.col_indices", pre);
  long long* ci = put_arr(c, nm, 'q', ro[nrows]);
  for (long long r = 0; r < nrows; ++r) {
    const long long na = rcell[2 * r] >= 0 ? elem_list(c, rcell[2 * r], which, la) : 0;
    const long long nb = rcell[2 * r + 1] >= 0 ? elem_list(c, rcell[2 * r + 1], which, lb) : 0;
    merge_unique(la, na, lb, nb, ci + ro[r]);
  }
  free(rcell);
  return 0;
}

int hdo_run(hdo_ctx* c, const char* what) {
  c->err[0] = 0;
  if (!strcmp(what, "assemble")) return run_assemble(c);
  if (!strcmp(what, "structure")) return run_structure(c);
  if (!strcmp(what, "port_hybridize")) return run_port_hybridize(c);
  if (!strcmp(what, "port_recover")) return run_port_recover(c);
  if (!strcmp(what, "port_condense")) return run_port_condense(c);
  if (!strcmp(what, "port_recover_condensed")) return run_port_recover_condensed(c);
  if (!strcmp(what, "dd_hybridize")) return run_dd_hybridize(c, 0);
  if (!strcmp(what, "dd_recover")) return run_dd_hybridize(c, 1);
  if (!strcmp(what, "dd_condense")) return run_dd_condense(c, 0);
  if (!strcmp(what, "dd_recover_condensed")) return run_dd_condense(c, 1);
  if (!strcmp(what, "spmv_H")) return run_spmv(c, "H", "lambda", "H_lambda");
  if (!strcmp(what, "spmv_S")) return run_spmv(c, "S", "x_b", "S_x_b");
  if (!strcmp(what, "pattern_H")) return run_pattern(c, 0);
  if (!strcmp(what, "pattern_S")) return run_pattern(c, 1);
  set_err(c, "unknown stage %s", what);
  return 1;
}
