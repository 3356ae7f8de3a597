// Host precomputation of the fixed factors used by the structured element
// solve, once per space, in
// double-double so every factor is correctly rounded to fp64 once.
//
//   D = F F^T + E     pivoted Cholesky of the PSD rank-(k+1)^dim reference
//                     divdiv matrix (div RT_k = Q_k), E = D - F F^T exactly
//   Minv = M^-1       Cholesky of the reference mass matrix
//   U = M^-1 F,  G = F^T M^-1 F
//
// These are exact rewritings of the reference element matrices
// (src/rt_space.cpp:180-314, 356-357): no approximation enters here beyond
// one final rounding of each factor.
#include <algorithm>
#include <cmath>

#include "hdr_internal.hpp"

namespace hdr {
namespace {

struct dd {
  double hi = 0.0, lo = 0.0;
};
inline dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
inline dd quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
inline dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, std::fma(a, b, -p)};
}
inline dd operator+(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  s.lo += x.lo + y.lo;
  return quick(s.hi, s.lo);
}
inline dd operator-(dd x) { return {-x.hi, -x.lo}; }
inline dd operator-(dd x, dd y) { return x + (-y); }
inline dd operator*(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  p.lo += x.hi * y.lo + x.lo * y.hi;
  return quick(p.hi, p.lo);
}
inline dd operator/(dd x, dd y) {
  const double q1 = x.hi / y.hi;
  dd r = x - dd{q1, 0} * y;
  const double q2 = r.hi / y.hi;
  r = r - dd{q2, 0} * y;
  const double q3 = r.hi / y.hi;
  return quick(q1, q2) + dd{q3, 0};
}
inline dd dsqrt(dd x) {
  if (x.hi <= 0.0) return {0.0, 0.0};
  const double s = std::sqrt(x.hi);
  const dd r = x - two_prod(s, s);
  return dd{s, 0} + dd{r.hi / (2.0 * s), 0};
}
inline double rnd(dd x) { return x.hi + x.lo; }

}  // namespace

bool precompute_structured(const RefElement& re, int expected_rank, Structured* out, std::string* err) {
  const int n = re.n;
  const std::vector<double>& D = re.divdiv;
  const std::vector<double>& M = re.mass;
  out->n = n;

  // --- pivoted Cholesky of D in double-double
  std::vector<dd> R(static_cast<size_t>(n) * n);
  double dmax = 0.0;
  // the reference accumulates divdiv/mass entrywise (rt_space.cpp:246-253), so
  // they are symmetric only up to rounding: factor the exact symmetric parts
  auto sym = [n](const std::vector<double>& a, int i, int k) {
    return (two_sum(a[static_cast<size_t>(i) * n + k], a[static_cast<size_t>(k) * n + i])) * dd{0.5, 0.0};
  };
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      R[static_cast<size_t>(i) * n + k] = sym(D, i, k);
      dmax = std::max(dmax, std::fabs(D[static_cast<size_t>(i) * n + k]));
    }
  double diag0 = 0.0;
  for (int i = 0; i < n; ++i) diag0 = std::max(diag0, D[static_cast<size_t>(i) * n + i]);
  std::vector<char> used(n, 0);
  std::vector<std::vector<dd>> cols;
  double last_pivot = 0.0, next_pivot = 0.0;
  for (int j = 0; j < n; ++j) {
    int p = -1;
    double best = -1.0;
    for (int i = 0; i < n; ++i)
      if (!used[i] && R[static_cast<size_t>(i) * n + i].hi > best) {
        best = R[static_cast<size_t>(i) * n + i].hi;
        p = i;
      }
    if (j == expected_rank) {
      next_pivot = best;
      break;
    }
    if (p < 0 || !(best > 0.0)) break;
    last_pivot = best;
    used[p] = 1;
    const dd piv = dsqrt(R[static_cast<size_t>(p) * n + p]);
    std::vector<dd> l(n);
    for (int i = 0; i < n; ++i) l[i] = used[i] && i != p ? dd{} : R[static_cast<size_t>(i) * n + p] / piv;
    l[p] = piv;
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) R[static_cast<size_t>(i) * n + k] = R[static_cast<size_t>(i) * n + k] - l[i] * l[k];
    cols.push_back(std::move(l));
  }
  const int r = static_cast<int>(cols.size());
  if (r != expected_rank || !(last_pivot > 1e-10 * diag0) || next_pivot > 1e-12 * diag0) {
    *err = "structured precompute: reference divdiv is not numerically of rank " + std::to_string(expected_rank) +
           " (got " + std::to_string(r) + ", last pivot " + std::to_string(last_pivot / diag0) + ", next " +
           std::to_string(next_pivot / diag0) + ")";
    return false;
  }
  out->r = r;
  // DD factor columns F (n x r), D ~= F F^T
  std::vector<dd> Fd(static_cast<size_t>(n) * r);
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < n; ++i) Fd[static_cast<size_t>(i) * r + j] = cols[j][i];

  // --- M^-1 by double-double Cholesky (no pivoting keeps the block zeros exact)
  std::vector<dd> L(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j) {
    dd d = sym(M, j, j);
    for (int k = 0; k < j; ++k) d = d - L[static_cast<size_t>(j) * n + k] * L[static_cast<size_t>(j) * n + k];
    if (!(d.hi > 0.0)) {
      *err = "structured precompute: reference mass matrix is not SPD";
      return false;
    }
    const dd lj = dsqrt(d);
    L[static_cast<size_t>(j) * n + j] = lj;
    for (int i = j + 1; i < n; ++i) {
      dd s = sym(M, i, j);
      for (int k = 0; k < j; ++k) s = s - L[static_cast<size_t>(i) * n + k] * L[static_cast<size_t>(j) * n + k];
      L[static_cast<size_t>(i) * n + j] = s / lj;
    }
  }
  std::vector<dd> Minv(static_cast<size_t>(n) * n);
  std::vector<dd> y(n);
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {
      dd s{i == c ? 1.0 : 0.0, 0.0};
      for (int k = 0; k < i; ++k) s = s - L[static_cast<size_t>(i) * n + k] * y[k];
      y[i] = s / L[static_cast<size_t>(i) * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      dd s = y[i];
      for (int k = i + 1; k < n; ++k) s = s - L[static_cast<size_t>(k) * n + i] * Minv[static_cast<size_t>(k) * n + c];
      Minv[static_cast<size_t>(i) * n + c] = s / L[static_cast<size_t>(i) * n + i];
    }
  }
  out->Minv.resize(static_cast<size_t>(n) * n);
  for (int i = 0; i < n * n; ++i) out->Minv[i] = rnd(Minv[i]);
  out->block_diag = true;
  for (int i = 0; i < n && out->block_diag; ++i)
    for (int k = 0; k < n; ++k)
      if (re.comp[i] != re.comp[k] && (M[static_cast<size_t>(i) * n + k] != 0.0 ||
                                        out->Minv[static_cast<size_t>(i) * n + k] != 0.0)) {
        out->block_diag = false;
        break;
      }

  // U = M^-1 F, G = F^T U (r x r SPD)
  std::vector<dd> Ud(static_cast<size_t>(n) * r);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < r; ++j) {
      dd s{};
      for (int k = 0; k < n; ++k) s = s + Minv[static_cast<size_t>(i) * n + k] * Fd[static_cast<size_t>(k) * r + j];
      Ud[static_cast<size_t>(i) * r + j] = s;
    }
  std::vector<double> G(static_cast<size_t>(r) * r);
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      dd s{};
      for (int k = 0; k < n; ++k) s = s + Fd[static_cast<size_t>(k) * r + a] * Ud[static_cast<size_t>(k) * r + b];
      G[static_cast<size_t>(a) * r + b] = rnd(s);
    }
  for (int a = 0; a < r; ++a)
    for (int b = a + 1; b < r; ++b) {
      const double v = 0.5 * (G[static_cast<size_t>(a) * r + b] + G[static_cast<size_t>(b) * r + a]);
      G[static_cast<size_t>(a) * r + b] = G[static_cast<size_t>(b) * r + a] = v;
    }
  // cyclic Jacobi: G = P diag(sigma) P^T
  std::vector<double> P(static_cast<size_t>(r) * r, 0.0);
  for (int a = 0; a < r; ++a) P[static_cast<size_t>(a) * r + a] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, scale = 0.0;
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        const double v = std::fabs(G[static_cast<size_t>(a) * r + b]);
        if (a != b) off = std::max(off, v);
        scale = std::max(scale, v);
      }
    if (off <= 1e-18 * scale) break;
    for (int p = 0; p < r; ++p)
      for (int q = p + 1; q < r; ++q) {
        const double apq = G[static_cast<size_t>(p) * r + q];
        if (std::fabs(apq) <= 1e-300) continue;
        const double theta = (G[static_cast<size_t>(q) * r + q] - G[static_cast<size_t>(p) * r + p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < r; ++k) {
          const double gkp = G[static_cast<size_t>(k) * r + p], gkq = G[static_cast<size_t>(k) * r + q];
          G[static_cast<size_t>(k) * r + p] = c * gkp - s * gkq;
          G[static_cast<size_t>(k) * r + q] = s * gkp + c * gkq;
        }
        for (int k = 0; k < r; ++k) {
          const double gpk = G[static_cast<size_t>(p) * r + k], gqk = G[static_cast<size_t>(q) * r + k];
          G[static_cast<size_t>(p) * r + k] = c * gpk - s * gqk;
          G[static_cast<size_t>(q) * r + k] = s * gpk + c * gqk;
        }
        for (int k = 0; k < r; ++k) {
          const double pkp = P[static_cast<size_t>(k) * r + p], pkq = P[static_cast<size_t>(k) * r + q];
          P[static_cast<size_t>(k) * r + p] = c * pkp - s * pkq;
          P[static_cast<size_t>(k) * r + q] = s * pkp + c * pkq;
        }
      }
  }
  out->lambda.resize(r);
  for (int a = 0; a < r; ++a) {
    out->lambda[a] = G[static_cast<size_t>(a) * r + a];
    if (!(out->lambda[a] > 0.0)) {
      *err = "structured precompute: nonpositive generalized eigenvalue";
      return false;
    }
  }
  // X = U P diag(sigma)^-1/2, rounded once
  out->X.resize(static_cast<size_t>(n) * r);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < r; ++j) {
      dd s{};
      for (int a = 0; a < r; ++a) s = s + Ud[static_cast<size_t>(i) * r + a] * dd{P[static_cast<size_t>(a) * r + j], 0};
      out->X[static_cast<size_t>(i) * r + j] = rnd(s / dsqrt(dd{out->lambda[j], 0}));
    }
  // E = D - (M X) diag(lambda) (M X)^T, N0 = M^-1 - X X^T, both from the rounded X, lambda
  std::vector<dd> MX(static_cast<size_t>(n) * r);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < r; ++j) {
      dd s{};
      for (int k = 0; k < n; ++k)
        if (M[static_cast<size_t>(i) * n + k] != 0.0 || M[static_cast<size_t>(k) * n + i] != 0.0)
          s = s + sym(M, i, k) * dd{out->X[static_cast<size_t>(k) * r + j], 0.0};
      MX[static_cast<size_t>(i) * r + j] = s;
    }
  out->E.assign(static_cast<size_t>(n) * n, 0.0);
  out->N0.assign(static_cast<size_t>(n) * n, 0.0);
  double emax = 0.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      dd s{D[static_cast<size_t>(i) * n + k], 0.0};
      dd t = Minv[static_cast<size_t>(i) * n + k];
      for (int j = 0; j < r; ++j) {
        s = s - MX[static_cast<size_t>(i) * r + j] * dd{out->lambda[j], 0} * MX[static_cast<size_t>(k) * r + j];
        t = t - two_prod(out->X[static_cast<size_t>(i) * r + j], out->X[static_cast<size_t>(k) * r + j]);
      }
      out->E[static_cast<size_t>(i) * n + k] = rnd(s);
      out->N0[static_cast<size_t>(i) * n + k] = rnd(t);
      emax = std::max(emax, std::fabs(rnd(s)));
    }
  out->e_rel = emax / dmax;
  out->Ma.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const dd a = two_sum(M[static_cast<size_t>(i) * n + k], -M[static_cast<size_t>(k) * n + i]) * dd{0.5, 0.0};
      out->Ma[static_cast<size_t>(i) * n + k] = rnd(a);
    }
  double orth = 0.0;
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      dd s{a == b ? -1.0 : 0.0, 0.0};
      for (int k = 0; k < n; ++k) s = s + dd{out->X[static_cast<size_t>(k) * r + a], 0} * MX[static_cast<size_t>(k) * r + b];
      orth = std::max(orth, std::fabs(rnd(s)));
    }
  out->orth = orth;
  if (out->e_rel > 1e-13 || orth > 1e-13) {
    *err = "structured precompute: factorization residual too large (E " + std::to_string(out->e_rel) +
           ", orthogonality " + std::to_string(orth) + ")";
    return false;
  }

  // Neumann ratio bound: ||A0^-1 Delta|| <= (alpha/beta) ||M^-1|| (||E|| + 2u||D||) (+ O(u))
  auto inf_norm = [n](const std::vector<double>& a) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += std::fabs(a[static_cast<size_t>(i) * n + k]);
      m = std::max(m, s);
    }
    return m;
  };
  const double u = 0x1.0p-53;
  out->rho = inf_norm(out->Minv) * (inf_norm(out->E) + 2.0 * u * inf_norm(D));
  return true;
}

}  // namespace hdr
