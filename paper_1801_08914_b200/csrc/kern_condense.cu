// Static condensation (static_condense, src/reduction.cpp:448-557) and its
// recovery (recover_condensed, src/reduction.cpp:559-587) on the FE path, with
// the marker partition i = element bubbles, b = face dofs (reduction.cpp:474).
//
//   S_T   = A_FF - A_Fi A_ii^-1 A_iF        (well conditioned: fp64 Cholesky of A_ii)
//   f_S,T = f_F - A_Fi A_ii^-1 f_i          (cancellation-prone: x = A_ii^-1 f_i is
//            refined to double-double with compensated residuals, and the product
//            A_Fi x is accumulated with error-free transforms)
//   scattered with the signs of P_b into S (rows = global face dofs, which are
//   exactly the master dofs) by the red-black scheme of the hybridize kernels.
// k = 0 has no bubbles: S = P^T A_hat P and f_S = P^T f_hat, bit-identical to the
// reference (the same two-term sums).
//
// recover_condensed: x_i = A_ii^-1 (f_i - A_iF x_b,T), refined the same way;
// the master entries of x are x_b itself.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "hdr_device.cuh"
#include "kernels.hpp"

namespace hdr {
namespace {

// double-double helpers (error-free transforms, include/hdivred/dd.hpp semantics)
struct ddv {
  double hi, lo;
};
__device__ __forceinline__ ddv dd_add_d(ddv x, double y) {
  double s, e;
  two_sum(x.hi, y, s, e);
  e += x.lo;
  const double h = s + e;
  return {h, e - (h - s)};
}
__device__ __forceinline__ ddv dd_fma_sub(ddv acc, double a, double b) {  // acc - a*b, exactly rounded to dd
  double p, pe;
  two_prod(a, b, p, pe);
  double s, e;
  two_sum(acc.hi, -p, s, e);
  e += acc.lo - pe;
  const double h = s + e;
  return {h, e - (h - s)};
}

// ------------------------------------------------------------------ k = 0

template <int DIM>
__global__ void __launch_bounds__(128) k_sc_rt0(CondArgs C, int parity) {
  constexpr int N = 2 * DIM;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= parity_count(C.m)) return;
  int cc[3];
  const int e = parity_cell32(C.m, parity, static_cast<uint32_t>(t), cc);
  if (e < 0) return;
  const double a = C.alpha[e], b = C.beta[e];
  unsigned lo = 0, hi = 0;
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
    const int Nx = static_cast<int>(x == 0 ? C.m.N[0] : (x == 1 ? C.m.N[1] : C.m.N[2]));
    lo |= static_cast<unsigned>(cx > 0) << x;
    hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
  }
#pragma unroll
  for (int p = 0; p < N; ++p) {
    const int ax = p >> 1, side = p & 1;
    const bool pin = (((side) ? hi : lo) >> ax) & 1u;
    const int face = face_id32(C.m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0),
                               cc[2] + (ax == 2 ? side : 0));
    const double sp = side ? 1.0 : -1.0;
    const int ca = ax == 0 ? cc[0] : (ax == 1 ? cc[1] : cc[2]);
    const int na = static_cast<int>(ax == 0 ? C.m.N[0] : (ax == 1 ? C.m.N[1] : C.m.N[2]));
    const int64_t start = C.rowoff[face];
    const bool add = parity == 1 && pin;  // an interior face's diagonal block has two contributions
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const double sq = (q & 1) ? 1.0 : -1.0;
      const double v = sp * sq * assemble_entry(a, b, C.fx.D[p * N + q], C.fx.M[p * N + q]);
      double* dst = C.sval + start + col_rank_fast(DIM, p, q, lo, hi, ca, na, true);
      *dst = (add && p == q) ? *dst + v : v;
    }
    const double fv = sp * C.f[static_cast<int64_t>(e) * N + p];
    C.fs[face] = add ? C.fs[face] + fv : fv;
  }
}

// ------------------------------------------------------------------ k >= 1: one CTA per cell

constexpr int kNT = 128;

struct ScLayout {
  int64_t aii, aif, xh, xl, r, d, f, total;
};
__host__ __device__ inline ScLayout sc_layout(int ni, int nf, int n) {
  ScLayout L;
  int64_t o = 0;
  auto take = [&o](int64_t c) {
    const int64_t at = o;
    o += (c + 1) & ~int64_t(1);
    return at;
  };
  L.aii = take(static_cast<int64_t>(ni) * ni);
  L.aif = take(static_cast<int64_t>(ni) * nf);
  L.xh = take(ni);
  L.xl = take(ni);
  L.r = take(ni);
  L.d = take(ni);
  L.f = take(n);
  L.total = o;
  return L;
}

// Cholesky of ni x ni (row-major, lower) in place; returns false if not SPD
__device__ bool cta_cholesky(double* a, int ni, int* flag) {
  for (int k = 0; k < ni; ++k) {
    if (threadIdx.x == 0) {
      const double dkk = a[k * ni + k];
      if (!(dkk > 0.0)) *flag = 1;
      a[k * ni + k] = sqrt(fmax(dkk, 0.0));
    }
    __syncthreads();
    const double lkk = a[k * ni + k];
    for (int i = k + 1 + threadIdx.x; i < ni; i += blockDim.x) a[i * ni + k] = lkk > 0.0 ? a[i * ni + k] / lkk : 0.0;
    __syncthreads();
    const int rem = ni - k - 1;
    for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
      const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
      if (j <= i) a[i * ni + j] = fma(-a[i * ni + k], a[j * ni + k], a[i * ni + j]);
    }
    __syncthreads();
  }
  return true;
}

// x <- A^-1 x with the Cholesky factor (single thread)
__device__ void chol_solve(const double* l, int ni, double* x) {
  for (int i = 0; i < ni; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s = fma(-l[i * ni + j], x[j], s);
    x[i] = s / l[i * ni + i];
  }
  for (int i = ni - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < ni; ++j) s = fma(-l[j * ni + i], x[j], s);
    x[i] = s / l[i * ni + i];
  }
}

// (xh, xl) = A_ii^-1 rhs (rhs given as dd (rh, rl)) refined to double-double:
// 3 steps of r = rhs - A_ii x (exact products, dd accumulation), x += L^-T L^-1 r
__device__ void dd_refined_solve(const CondArgs& C, double a, double b, int ni, const double* l, const double* rh,
                                 const double* rl, double* xh, double* xl, double* r) {
  const int n = C.m.n;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ni; ++i) {
      xh[i] = rh[i];
      xl[i] = 0.0;
    }
    chol_solve(l, ni, xh);
  }
  __syncthreads();
  for (int step = 0; step < 3; ++step) {
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
      ddv acc = {rh[i], rl ? rl[i] : 0.0};
      for (int j = 0; j < ni; ++j) {
        const double aij = assemble_entry(a, b, C.fx.D[i * n + j], C.fx.M[i * n + j]);
        acc = dd_fma_sub(acc, aij, xh[j]);
        acc.lo = fma(-aij, xl[j], acc.lo);
      }
      r[i] = acc.hi + acc.lo;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      chol_solve(l, ni, r);
      for (int i = 0; i < ni; ++i) {
        ddv v = dd_add_d({xh[i], xl[i]}, r[i]);
        xh[i] = v.hi;
        xl[i] = v.lo;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kNT) k_sc_cta(CondArgs C, int parity, double* gws, int64_t stride, int use_smem) {
  extern __shared__ double smem[];
  double* ws = use_smem ? smem : gws + blockIdx.x * stride;
  const DevMesh& m = C.m;
  const int n = m.n, ni = m.nint, nf = C.nF, dpf = m.dpf, dim = m.dim, ns = 2 * dim;
  const ScLayout L = sc_layout(ni, nf, n);
  double* aii = ws + L.aii;
  double* aif = ws + L.aif;
  double* xh = ws + L.xh;
  double* xl = ws + L.xl;
  double* r = ws + L.r;
  double* fl = ws + L.f;
  __shared__ int flag;
  const uint32_t cnt = static_cast<uint32_t>(parity_count(m));
  for (uint32_t t = blockIdx.x; t < cnt; t += gridDim.x) {
    int cc[3];
    const int e = parity_cell32(m, parity, t, cc);
    if (e < 0) continue;
    const double a = C.alpha[e], b = C.beta[e];
    if (threadIdx.x == 0) flag = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) fl[i] = C.f[static_cast<int64_t>(e) * n + i];
    for (int idx = threadIdx.x; idx < ni * ni; idx += blockDim.x) {
      const int i = idx / ni, j = idx - i * ni;
      aii[idx] = assemble_entry(a, b, C.fx.D[i * n + j], C.fx.M[i * n + j]);
    }
    for (int idx = threadIdx.x; idx < ni * nf; idx += blockDim.x) {
      const int i = idx / nf, c = idx - i * nf;
      aif[idx] = assemble_entry(a, b, C.fx.D[i * n + ni + c], C.fx.M[i * n + ni + c]);
    }
    __syncthreads();
    cta_cholesky(aii, ni, &flag);
    if (flag) atomicOr(C.status, 2);
    // W = A_ii^-1 A_iF (in place, one column per thread)
    for (int c = threadIdx.x; c < nf; c += blockDim.x) {
      for (int i = 0; i < ni; ++i) {
        double s = aif[i * nf + c];
        for (int j = 0; j < i; ++j) s = fma(-aii[i * ni + j], aif[j * nf + c], s);
        aif[i * nf + c] = s / aii[i * ni + i];
      }
      for (int i = ni - 1; i >= 0; --i) {
        double s = aif[i * nf + c];
        for (int j = i + 1; j < ni; ++j) s = fma(-aii[j * ni + i], aif[j * nf + c], s);
        aif[i * nf + c] = s / aii[i * ni + i];
      }
    }
    // x = A_ii^-1 f_i to double-double
    __syncthreads();
    dd_refined_solve(C, a, b, ni, aii, fl, nullptr, xh, xl, r);
    // scatter tables (all faces: S rows are the global face dofs)
    unsigned lo = 0, hi = 0;
    for (int x = 0; x < dim; ++x) {
      const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
      const int Nx = static_cast<int>(x == 0 ? m.N[0] : (x == 1 ? m.N[1] : m.N[2]));
      lo |= static_cast<unsigned>(cx > 0) << x;
      hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
    }
    // S entries: thread per (p, q)
    for (int idx = threadIdx.x; idx < nf * (nf + 1); idx += blockDim.x) {
      const int p = idx / (nf + 1), q = idx - p * (nf + 1);
      const int ps = p / dpf, sub = p - ps * dpf;
      const int ax = ps >> 1, side = ps & 1;
      const bool pin = (((side) ? hi : lo) >> ax) & 1u;
      const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0),
                                 cc[2] + (ax == 2 ? side : 0));
      const double sp = side ? 1.0 : -1.0;
      const bool add = parity == 1 && pin;
      const int row = face * dpf + sub;
      if (q == nf) {  // f_S,p = f_F,p - A_Fi x  (x in double-double)
        ddv acc = {fl[ni + p], 0.0};
        for (int i = 0; i < ni; ++i) {
          const double api = assemble_entry(a, b, C.fx.D[(ni + p) * n + i], C.fx.M[(ni + p) * n + i]);
          acc = dd_fma_sub(acc, api, xh[i]);
          acc.lo = fma(-api, xl[i], acc.lo);
        }
        const double v = sp * (acc.hi + acc.lo);
        C.fs[row] = add ? C.fs[row] + v : v;
        continue;
      }
      double s = assemble_entry(a, b, C.fx.D[(ni + p) * n + ni + q], C.fx.M[(ni + p) * n + ni + q]);
      for (int i = 0; i < ni; ++i)
        s = fma(-assemble_entry(a, b, C.fx.D[(ni + p) * n + i], C.fx.M[(ni + p) * n + i]), aif[i * nf + q], s);
      const int qs = q / dpf, sj = q - qs * dpf;
      const double sq = (qs & 1) ? 1.0 : -1.0;
      const int ca = ax == 0 ? cc[0] : (ax == 1 ? cc[1] : cc[2]);
      const int na = static_cast<int>(ax == 0 ? m.N[0] : (ax == 1 ? m.N[1] : m.N[2]));
      const int64_t start = C.rowoff[row];
      const int rk = col_rank_fast(dim, ps, qs, lo, hi, ca, na, true);
      double* dst = C.sval + start + static_cast<int64_t>(rk) * dpf + sj;
      const double v = sp * sq * s;
      *dst = (add && ps == qs) ? *dst + v : v;
    }
    __syncthreads();
  }
  (void)ns;
}

// recover_condensed: x_i = A_ii^-1 (f_i - A_iF x_b,T) (double-double), masters copied
__global__ void __launch_bounds__(kNT) k_rc_cta(CondArgs C, double* gws, int64_t stride, int use_smem) {
  extern __shared__ double smem[];
  double* ws = use_smem ? smem : gws + blockIdx.x * stride;
  const DevMesh& m = C.m;
  const int n = m.n, ni = m.nint, nf = C.nF, dpf = m.dpf, dim = m.dim;
  const ScLayout L = sc_layout(ni, nf, n);
  double* aii = ws + L.aii;
  double* xh = ws + L.xh;
  double* xl = ws + L.xl;
  double* r = ws + L.r;
  double* rh = ws + L.d;
  double* rl = ws + L.f;  // ni <= n
  __shared__ int flag;
  for (int64_t e = blockIdx.x; e < m.ncells; e += gridDim.x) {
    const double a = C.alpha[e], b = C.beta[e];
    int cc[3];
    cell_coords32(m, static_cast<uint32_t>(e), cc);
    if (threadIdx.x == 0) flag = 0;
    for (int idx = threadIdx.x; idx < ni * ni; idx += blockDim.x) {
      const int i = idx / ni, j = idx - i * ni;
      aii[idx] = assemble_entry(a, b, C.fx.D[i * n + j], C.fx.M[i * n + j]);
    }
    // rhs_i = f_i - sum_c A_ic (sign_c x_b[global_c])  in double-double
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
      ddv acc = {C.f[e * n + i], 0.0};
      for (int c = 0; c < nf; ++c) {
        const int qs = c / dpf, sub = c - qs * dpf;
        const int ax = qs >> 1, side = qs & 1;
        const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0),
                                   cc[2] + (ax == 2 ? side : 0));
        const double xbl = (side ? 1.0 : -1.0) * C.xb[face * dpf + sub];
        acc = dd_fma_sub(acc, assemble_entry(a, b, C.fx.D[i * n + ni + c], C.fx.M[i * n + ni + c]), xbl);
      }
      rh[i] = acc.hi;
      rl[i] = acc.lo;
    }
    __syncthreads();
    cta_cholesky(aii, ni, &flag);
    if (flag) atomicOr(C.status, 2);
    dd_refined_solve(C, a, b, ni, aii, rh, rl, xh, xl, r);
    for (int i = threadIdx.x; i < ni; i += blockDim.x) C.x[m.face_dof_count + e * ni + i] = xh[i] + xl[i];
    __syncthreads();
  }
}

__global__ void k_copy_masters(const double* xb, double* x, int64_t nmaster) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < nmaster) x[i] = xb[i];
}

}  // namespace

void launch_condense(const CondArgs& c, int parity, double* gws, int64_t ws_doubles, cudaStream_t st) {
  if (c.m.nint == 0) {
    const unsigned nb = static_cast<unsigned>((parity_count(c.m) + 127) / 128);
    if (c.m.dim == 3)
      k_sc_rt0<3><<<nb, 128, 0, st>>>(c, parity);
    else
      k_sc_rt0<2><<<nb, 128, 0, st>>>(c, parity);
    count_launch();
    return;
  }
  const ScLayout L = sc_layout(c.m.nint, c.nF, c.m.n);
  const bool use_smem = L.total * 8 <= 96 * 1024;
  const size_t smem = use_smem ? static_cast<size_t>(L.total) * 8 : 0;
  if (use_smem) cudaFuncSetAttribute(k_sc_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int64_t cnt = parity_count(c.m);
  int64_t grid = use_smem ? std::min<int64_t>(cnt, 148 * 16) : std::min<int64_t>(cnt, ws_doubles / L.total);
  grid = std::max<int64_t>(grid, 1);
  k_sc_cta<<<static_cast<unsigned>(grid), kNT, smem, st>>>(c, parity, gws, L.total, use_smem ? 1 : 0);
  count_launch();
}

int64_t condense_ws_doubles(const DevMesh& m, int nF) {
  if (m.nint == 0) return 0;
  const ScLayout L = sc_layout(m.nint, nF, m.n);
  return L.total * 8 <= 96 * 1024 ? 0 : L.total * 148 * 2;
}

void launch_recover_condensed(const CondArgs& c, double* gws, int64_t ws_doubles, cudaStream_t st) {
  const int64_t nmaster = c.m.face_dof_count;
  k_copy_masters<<<static_cast<unsigned>((nmaster + 255) / 256), 256, 0, st>>>(c.xb, c.x, nmaster);
  count_launch();
  if (c.m.nint == 0) return;
  const ScLayout L = sc_layout(c.m.nint, c.nF, c.m.n);
  const bool use_smem = L.total * 8 <= 96 * 1024;
  const size_t smem = use_smem ? static_cast<size_t>(L.total) * 8 : 0;
  if (use_smem) cudaFuncSetAttribute(k_rc_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int64_t grid = use_smem ? std::min<int64_t>(c.m.ncells, 148 * 16) : std::min<int64_t>(c.m.ncells, ws_doubles / L.total);
  grid = std::max<int64_t>(grid, 1);
  k_rc_cta<<<static_cast<unsigned>(grid), kNT, smem, st>>>(c, gws, L.total, use_smem ? 1 : 0);
  count_launch();
}

}  // namespace hdr
