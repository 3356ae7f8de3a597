// Reference-element matrices of the RT_k space on one axis-aligned box.
//
// Restates build_reference (/root/reference/proj/src/rt_space.cpp:180-314) and its
// helpers (gauss_legendre_01 :10-34, legendre01 :36-46, legendre01_deriv :48-65,
// space_polys :77-87, interior_moments :91-102, dof_vandermonde :136-172) with
// the same floating-point operation order, so ref_divdiv / ref_mass come out
// bit-identical to the reference's (tests/test_space.py pins this against the
// golden fixtures).  Compiled with -ffp-contract=off: the reference's as-shipped
// Release build contains no FMA.
//
// Runs once per space on the host; the per-cell work happens on the device.
#include "hdr_internal.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>

namespace hdr {
namespace {

void gauss_legendre01(int n, double* x_out, double* w_out) {
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (static_cast<double>(i) + 0.75) / (static_cast<double>(n) + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int m = 2; m <= n; ++m) {
        const double p2 = ((2.0 * m - 1.0) * x * p1 - (m - 1.0) * p0) / static_cast<double>(m);
        p0 = p1;
        p1 = p2;
      }
      dp = static_cast<double>(n) * (x * p1 - p0) / (x * x - 1.0);
      const double step = p1 / dp;
      x -= step;
      if (std::fabs(step) < 1e-15) break;
    }
    x_out[n - 1 - i] = 0.5 * (x + 1.0);
    w_out[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
  }
}

double leg(int m, double s) {
  const double t = 2.0 * s - 1.0;
  if (m == 0) return 1.0;
  double p0 = 1.0, p1 = t;
  for (int i = 2; i <= m; ++i) {
    const double p2 = ((2.0 * i - 1.0) * t * p1 - (i - 1.0) * p0) / static_cast<double>(i);
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

double leg_deriv(int m, double s) {
  if (m == 0) return 0.0;
  const double t = 2.0 * s - 1.0;
  if (m == 1) return 2.0;
  double p0 = 1.0, p1 = t;
  for (int i = 2; i <= m; ++i) {
    const double p2 = ((2.0 * i - 1.0) * t * p1 - (i - 1.0) * p0) / static_cast<double>(i);
    p0 = p1;
    p1 = p2;
  }
  if (std::fabs(t * t - 1.0) < 1e-12) {
    const double sg = (t > 0.0) ? 1.0 : ((m % 2 == 1) ? 1.0 : -1.0);
    return 2.0 * sg * 0.5 * m * (m + 1.0);
  }
  return 2.0 * static_cast<double>(m) * (t * p1 - p0) / (t * t - 1.0);
}

struct Mono {
  int comp;
  int deg[3];
};

// component-major tensor enumeration, x fastest; lim(a) = base + (a == comp ? extra : 0)
std::vector<Mono> enumerate(int dim, int k, int along, int other) {
  std::vector<Mono> out;
  for (int c = 0; c < dim; ++c) {
    int lim[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) lim[a] = (a == c) ? along : other;
    for (int z = 0; z <= lim[2]; ++z)
      for (int y = 0; y <= lim[1]; ++y)
        for (int x = 0; x <= lim[0]; ++x) out.push_back({c, {x, y, z}});
  }
  (void)k;
  return out;
}

double pair_int(int p, int q) { return (p == q) ? 1.0 / (2.0 * p + 1.0) : 0.0; }
double mom_w(int m) { return std::sqrt(2.0 * m + 1.0); }

// LU with partial pivoting + column-by-column inverse, as lu_factor / lu_inverse
// (src/dense.cpp:61-120, 165-177): the Vandermonde inverse's rounding is part
// of the reference bits.
std::vector<double> lu_inverse_ref(std::vector<double> a, int n) {
  std::vector<int> piv(n);
  double mx = 0.0;
  for (double v : a) mx = std::max(mx, std::fabs(v));
  const double thr = 1e-14 * mx;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double pm = std::fabs(a[k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(a[i * n + k]) > pm) {
        pm = std::fabs(a[i * n + k]);
        p = i;
      }
    if (!(pm > thr) || pm == 0.0) throw std::runtime_error("reference Vandermonde is singular");
    piv[k] = p;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[p * n + j]);
    const double inv = 1.0 / a[k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double l = a[i * n + k] * inv;
      a[i * n + k] = l;
      if (l == 0.0) continue;
      for (int j = k + 1; j < n; ++j) a[i * n + j] -= l * a[k * n + j];
    }
  }
  std::vector<double> inv(static_cast<size_t>(n) * n), x(n);
  for (int col = 0; col < n; ++col) {
    for (int i = 0; i < n; ++i) x[i] = (i == col) ? 1.0 : 0.0;
    for (int k = 0; k < n; ++k)
      if (piv[k] != k) std::swap(x[k], x[piv[k]]);
    for (int k = 0; k < n; ++k) {
      const double xk = x[k];
      if (xk == 0.0) continue;
      for (int i = k + 1; i < n; ++i) x[i] -= a[i * n + k] * xk;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int j = i + 1; j < n; ++j) s -= a[i * n + j] * x[j];
      x[i] = s / a[i * n + i];
    }
    for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + col] = x[i];
  }
  return inv;
}

}  // namespace

RefElement build_reference_element(int dim, int k, const double h[3]) {
  const int nq = k + 2;  // rt_space.cpp:333
  const auto polys = enumerate(dim, k, k + 1, k);
  const auto inter = (k == 0) ? std::vector<Mono>{} : enumerate(dim, k, k - 1, k);
  const int n = static_cast<int>(polys.size());
  const int ni = static_cast<int>(inter.size());
  const int dpf = static_cast<int>(std::llround(std::pow(k + 1, dim - 1)));

  RefElement re;
  re.dim = dim;
  re.k = k;
  re.n = n;
  re.dpf = dpf;
  re.nint = ni;

  // dof functionals on the monomials (dof_vandermonde)
  std::vector<double> V(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    const Mono& t = polys[j];
    for (int i = 0; i < ni; ++i) {
      const Mono& m = inter[i];
      if (m.comp != t.comp) continue;
      double v = 1.0;
      for (int a = 0; a < dim; ++a) v *= pair_int(t.deg[a], m.deg[a]) * mom_w(m.deg[a]);
      V[static_cast<size_t>(i) * n + j] = v;
    }
    for (int slot = 0; slot < 2 * dim; ++slot) {
      const int axis = slot / 2, side = slot % 2;
      if (t.comp != axis) continue;
      int tang[2] = {-1, -1}, nt = 0;
      for (int a = 0; a < dim; ++a)
        if (a != axis) tang[nt++] = a;
      const double base = (side ? 1.0 : -1.0) * leg(t.deg[axis], side ? 1.0 : 0.0);
      for (int sub = 0; sub < dpf; ++sub) {
        const int md[2] = {dim == 2 ? sub : sub % (k + 1), dim == 2 ? 0 : sub / (k + 1)};
        double v = base;
        for (int ti = 0; ti < nt; ++ti) v *= pair_int(t.deg[tang[ti]], md[ti]) * mom_w(md[ti]);
        V[static_cast<size_t>(ni + slot * dpf + sub) * n + j] = v;
      }
    }
  }
  const std::vector<double> phi = lu_inverse_ref(V, n);

  double qs[16], qw[16];
  gauss_legendre01(nq, qs, qw);
  re.divdiv.assign(static_cast<size_t>(n) * n, 0.0);
  re.mass.assign(static_cast<size_t>(n) * n, 0.0);
  re.face_moments.assign(static_cast<size_t>(2 * dim) * dpf * n, 0.0);
  re.unit_load.assign(3 * static_cast<size_t>(n), 0.0);
  const int npr = dim == 3 ? (k + 1) * (k + 1) * (k + 1) : (k + 1) * (k + 1);
  re.npr = npr;
  re.div_form.assign(static_cast<size_t>(npr) * n, 0.0);
  std::vector<double> prv(npr);

  std::vector<double> pv(n), pd(n), bv(3 * static_cast<size_t>(n)), bd(n);
  const int nqz = (dim == 3) ? nq : 1;
  re.nq = nq;
  re.qs.assign(qs, qs + nq);
  for (int iz = 0; iz < nqz; ++iz)
    for (int iy = 0; iy < nq; ++iy)
      for (int ix = 0; ix < nq; ++ix) {
        const double s[3] = {qs[ix], qs[iy], dim == 3 ? qs[iz] : 0.0};
        double w = qw[ix] * h[0] * qw[iy] * h[1];
        if (dim == 3) w *= qw[iz] * h[2];
        for (int q = 0; q < n; ++q) {
          const Mono& t = polys[q];
          double v = 1.0;
          for (int a = 0; a < dim; ++a) v *= leg(t.deg[a], s[a]);
          pv[q] = v;
          double dv = leg_deriv(t.deg[t.comp], s[t.comp]) / h[t.comp];
          for (int a = 0; a < dim; ++a)
            if (a != t.comp) dv *= leg(t.deg[a], s[a]);
          pd[q] = dv;
        }
        for (int j = 0; j < n; ++j) {
          double* vj = &bv[3 * static_cast<size_t>(j)];
          vj[0] = vj[1] = vj[2] = 0.0;
          double ds = 0.0;
          for (int q = 0; q < n; ++q) {
            const double c = phi[static_cast<size_t>(q) * n + j];
            if (c == 0.0) continue;
            vj[polys[q].comp] += c * pv[q];
            ds += c * pd[q];
          }
          bd[j] = ds;
        }
        if (dim == 3) {
          re.bq_val.insert(re.bq_val.end(), bv.begin(), bv.end());
          re.bq_div.insert(re.bq_div.end(), bd.begin(), bd.end());
          re.bq_w.push_back(qw[ix] * qw[iy] * qw[iz]);
        }
        for (int i = 0; i < n; ++i) {
          const double dvi = bd[i];
          const double* vi = &bv[3 * static_cast<size_t>(i)];
          for (int j = 0; j < n; ++j) {
            re.divdiv[static_cast<size_t>(i) * n + j] += w * dvi * bd[j];
            const double* vj = &bv[3 * static_cast<size_t>(j)];
            re.mass[static_cast<size_t>(i) * n + j] += w * (vi[0] * vj[0] + vi[1] * vj[1] + vi[2] * vj[2]);
          }
          for (int c = 0; c < dim; ++c) re.unit_load[static_cast<size_t>(c) * n + i] += w * vi[c];
        }
        // div_form (rt_space.cpp:256-259): pressure Legendre products (pressure_polys
        // :104-111, x fastest) against the basis divergence
        for (int r = 0; r < npr; ++r) {
          const int d[3] = {r % (k + 1), (r / (k + 1)) % (k + 1), r / ((k + 1) * (k + 1))};
          double v = 1.0;
          for (int a = 0; a < dim; ++a) v *= leg(d[a], s[a]);
          prv[r] = v;
        }
        for (int r = 0; r < npr; ++r)
          for (int j = 0; j < n; ++j) re.div_form[static_cast<size_t>(r) * n + j] += w * prv[r] * bd[j];
      }

  // face moment rows of the weighted constraint (rt_space.cpp:267-312)
  for (int slot = 0; slot < 2 * dim; ++slot) {
    const int axis = slot / 2, side = slot % 2;
    int tang[2] = {-1, -1}, nt = 0;
    for (int a = 0; a < dim; ++a)
      if (a != axis) tang[nt++] = a;
    double* fm = &re.face_moments[static_cast<size_t>(slot) * dpf * n];
    const int n2 = (dim == 3) ? nq : 1;
    for (int i2 = 0; i2 < n2; ++i2)
      for (int i1 = 0; i1 < nq; ++i1) {
        double s[3] = {0.0, 0.0, 0.0};
        s[axis] = side ? 1.0 : 0.0;
        s[tang[0]] = qs[i1];
        double w = qw[i1] * h[tang[0]];
        if (dim == 3) {
          s[tang[1]] = qs[i2];
          w *= qw[i2] * h[tang[1]];
        }
        for (int q = 0; q < n; ++q) {
          double v = 1.0;
          for (int a = 0; a < dim; ++a) v *= leg(polys[q].deg[a], s[a]);
          pv[q] = v;
        }
        for (int j = 0; j < n; ++j) {
          double tr = 0.0;
          for (int q = 0; q < n; ++q) {
            if (polys[q].comp != axis) continue;
            tr += phi[static_cast<size_t>(q) * n + j] * pv[q];
          }
          tr *= side ? 1.0 : -1.0;
          if (tr == 0.0) continue;
          for (int sub = 0; sub < dpf; ++sub) {
            const int md[2] = {dim == 2 ? sub : sub % (k + 1), dim == 2 ? 0 : sub / (k + 1)};
            double qv = leg(md[0], s[tang[0]]) * mom_w(md[0]);
            if (dim == 3) qv *= leg(md[1], s[tang[1]]) * mom_w(md[1]);
            fm[static_cast<size_t>(sub) * n + j] += w * tr * qv;
          }
        }
      }
  }

  // vector component of every local dof: bubbles are component-major
  // (interior_moments), face dofs follow their slot's axis.
  re.comp.resize(n);
  for (int l = 0; l < n; ++l) re.comp[l] = (l < ni) ? inter[l].comp : ((l - ni) / dpf) / 2;
  return re;
}

}  // namespace hdr
