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
#include <cstdlib>

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
__device__ bool cta_cholesky(double* a, int ni, int* flag, int ld = 0) {
  if (ld == 0) ld = ni;
  __shared__ double colk[256];  // column k of the factor (ni <= 256)
  for (int k = 0; k < ni; ++k) {
    if (threadIdx.x == 0) {
      const double dkk = a[k * ld + k];
      if (!(dkk > 0.0)) *flag = 1;
      a[k * ld + k] = sqrt(fmax(dkk, 0.0));
    }
    __syncthreads();
    const double lkk = a[k * ld + k];
    for (int i = k + 1 + threadIdx.x; i < ni; i += blockDim.x) a[i * ld + k] = lkk > 0.0 ? a[i * ld + k] / lkk : 0.0;
    __syncthreads();
    // trailing update of the lower triangle: warps over rows i, lanes over columns j <= i
    // (contiguous in the row-major factor); column k read from a contiguous copy
    for (int i = k + 1 + threadIdx.x; i < ni; i += blockDim.x) colk[i] = a[i * ld + k];
    __syncthreads();
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = k + 1 + (threadIdx.x >> 5); i < ni; i += nw) {
      const double lik = colk[i];
      for (int j = k + 1 + lane; j <= i; j += 32) a[i * ld + j] = fma(-lik, colk[j], a[i * ld + j]);
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

// small interior blocks (ni <= 32, e.g. RT1 hexahedra): 128 threads per cell,
// column-per-thread solves in shared memory (the layout uses nF columns)
__global__ void __launch_bounds__(kNT) k_sc_small(CondArgs C, int parity, double* gws, int64_t stride, int use_smem) {
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

// ------------------------------------------------------------------ small interior blocks, one warp per cell
//
// NI <= 12 interior dofs and NF <= 24 face dofs (RT1 hexahedra, RT1 / RT2
// quadrilaterals): the whole cell fits one warp, so nothing waits on a CTA
// barrier or on a single thread:
//   * Cholesky of A_ii with lane i holding row i in registers, the pivot row
//     broadcast by shuffles (right-looking, fully unrolled);
//   * W = A_ii^-1 [A_iF | f_i]: lane c owns column c in registers, the factor read
//     as shared-memory broadcasts, right-looking substitution (independent updates);
//   * x = A_ii^-1 f_i refined to double-double (3 steps): lane i forms row i of the
//     residual with exact products, the correction L^-T L^-1 r runs lane-per-row with
//     shuffles, the factor read from shared memory;
//   * S_pq = A_Fq,p - sum_i A_Fi[p][i] W[i][q]: lane q owns column q of W in registers,
//     the row p of A_Fi is a broadcast; f_S,p by lane p with error-free accumulation;
//   * scatter by the red-black scheme with per-cell tables (row starts, block ranks).
// The arithmetic per entry is the CTA kernel's (same summation order).
template <int DIM, int NI, int NF>
struct ScWarpSm {
  static constexpr int NC = NF + 1, NS = 2 * DIM;
  double aii[NI * NI];  // A_ii as assembled (residuals)
  double l[NI * NI];    // its Cholesky factor, row-major lower
  double w[NI * NC];    // [A_iF | f_i] -> [W | x]
  double afi[NF * NI];  // A_Fi
  double ff[NF];        // f_F
  double xh[NI], xl[NI];
  double invd[NI];       // 1 / L_kk
  long long rstart[NF];  // start of the S row of face dof p
  int frow[NF];          // its row
  int rank[NS * NS];     // column-block rank of face slot qs in the rows of slot ps
};

#ifndef HDR_SC_MINB
#define HDR_SC_MINB 4  // CTAs (of 4 warps) per SM asked of ptxas
#endif
template <int DIM, int NI, int NF>
__global__ void __launch_bounds__(128, HDR_SC_MINB) k_sc_warp(CondArgs C, int parity) {
  using SM = ScWarpSm<DIM, NI, NF>;
  constexpr int N = NI + NF, NC = SM::NC, NS = SM::NS, DPF = NF / NS;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char sc_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SM& sm = reinterpret_cast<SM*>(sc_smem)[warp];
  const DevMesh& m = C.m;
  const double* __restrict__ Dg = C.fx.D;
  const double* __restrict__ Mg = C.fx.M;
  const uint32_t cnt = static_cast<uint32_t>(parity_count(m));
  const int il = lane < NI ? lane : NI - 1;  // lanes beyond the block repeat its last row
  for (uint32_t t = blockIdx.x * 4 + warp; t < cnt; t += gridDim.x * 4) {
    int cc[3];
    const int e = parity_cell32(m, parity, t, cc);
    if (e < 0) continue;  // (warp-uniform)
    if (DIM == 2) cc[2] = 0;
    const double a = __ldg(C.alpha + e), b = __ldg(C.beta + e);
    unsigned lo = 0, hi = 0;
#pragma unroll
    for (int x = 0; x < DIM; ++x) {
      const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
      const int Nx = static_cast<int>(x == 0 ? m.N[0] : (x == 1 ? m.N[1] : m.N[2]));
      lo |= static_cast<unsigned>(cx > 0) << x;
      hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
    }
    // scatter tables (their loads are in flight during the assembly)
    if (lane < NF) {
      const int ps = lane / DPF, sub = lane - ps * DPF, ax = ps >> 1, side = ps & 1;
      const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0),
                                 cc[2] + (ax == 2 ? side : 0));
      const int row = face * DPF + sub;
      sm.frow[lane] = row;
      sm.rstart[lane] = C.rowoff[row];
    }
    for (int idx = lane; idx < NS * NS; idx += 32) {
      const int ps = idx / NS, qs = idx - ps * NS, ax = ps >> 1;
      const int ca = ax == 0 ? cc[0] : (ax == 1 ? cc[1] : cc[2]);
      const int na = static_cast<int>(ax == 0 ? m.N[0] : (ax == 1 ? m.N[1] : m.N[2]));
      sm.rank[idx] = col_rank_fast(DIM, ps, qs, lo, hi, ca, na, true);
    }
    // assembly: A_ii, [A_iF | f_i], A_Fi, f_F
    const double* fe = C.f + static_cast<int64_t>(e) * N;
    for (int idx = lane; idx < NI * NI; idx += 32) {
      const int i = idx / NI, j = idx - i * NI;
      sm.aii[idx] = assemble_entry(a, b, __ldg(Dg + i * N + j), __ldg(Mg + i * N + j));
    }
    for (int idx = lane; idx < NI * NF; idx += 32) {
      const int i = idx / NF, c = idx - i * NF;
      sm.w[i * NC + c] = assemble_entry(a, b, __ldg(Dg + i * N + NI + c), __ldg(Mg + i * N + NI + c));
    }
    for (int idx = lane; idx < NF * NI; idx += 32) {
      const int p = idx / NI, i = idx - p * NI;
      sm.afi[idx] = assemble_entry(a, b, __ldg(Dg + (NI + p) * N + i), __ldg(Mg + (NI + p) * N + i));
    }
    if (lane < NI) sm.w[lane * NC + NF] = fe[lane];
    if (lane < NF) sm.ff[lane] = fe[NI + lane];
    __syncwarp();
    // ---- Cholesky, lane il = row il
    {
      double row[NI];
#pragma unroll
      for (int j = 0; j < NI; ++j) row[j] = sm.aii[il * NI + j];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const double dkk = __shfl_sync(FULL, row[k], k);
        bad = bad || !(dkk > 0.0);
        const double lkk = sqrt(fmax(dkk, 0.0));
        const double inv = lkk > 0.0 ? 1.0 / lkk : 0.0;
        if (lane == 0) sm.invd[k] = inv;
        const double lik = il == k ? lkk : row[k] * inv;
        row[k] = lik;
#pragma unroll
        for (int j = k + 1; j < NI; ++j) row[j] = fma(-lik, __shfl_sync(FULL, lik, j), row[j]);
      }
      if (bad && lane == 0) atomicOr(C.status, 2);
      if (lane < NI) {
#pragma unroll
        for (int j = 0; j < NI; ++j) sm.l[lane * NI + j] = row[j];
      }
    }
    __syncwarp();
    // ---- [W | x] = A_ii^-1 [A_iF | f_i], lane c = column c
    if (lane < NC) {
      double v[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) v[i] = sm.w[i * NC + lane];
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        v[j] *= sm.invd[j];
#pragma unroll
        for (int i = j + 1; i < NI; ++i) v[i] = fma(-sm.l[i * NI + j], v[j], v[i]);
      }
#pragma unroll
      for (int j = NI - 1; j >= 0; --j) {
        v[j] *= sm.invd[j];
#pragma unroll
        for (int i = 0; i < j; ++i) v[i] = fma(-sm.l[j * NI + i], v[j], v[i]);
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) sm.w[i * NC + lane] = v[i];
    }
    __syncwarp();
    // ---- x = A_ii^-1 f_i to double-double, lane il = entry il
    {
      double xh = sm.w[il * NC + NF], xl = 0.0;
      const double fi = fe[il];
#pragma unroll 1
      for (int step = 0; step < 3; ++step) {
        ddv acc = {fi, 0.0};
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double aij = sm.aii[il * NI + j];
          acc = dd_fma_sub(acc, aij, __shfl_sync(FULL, xh, j));
          acc.lo = fma(-aij, __shfl_sync(FULL, xl, j), acc.lo);
        }
        double r = acc.hi + acc.lo;
#pragma unroll
        for (int j = 0; j < NI; ++j) {  // L y = r
          const double vj = __shfl_sync(FULL, r, j) * sm.invd[j];
          r = il == j ? vj : (il > j ? fma(-sm.l[il * NI + j], vj, r) : r);
        }
#pragma unroll
        for (int j = NI - 1; j >= 0; --j) {  // L^T d = y
          const double vj = __shfl_sync(FULL, r, j) * sm.invd[j];
          r = il == j ? vj : (il < j ? fma(-sm.l[j * NI + il], vj, r) : r);
        }
        const ddv v = dd_add_d({xh, xl}, r);
        xh = v.hi, xl = v.lo;
      }
      if (lane < NI) sm.xh[lane] = xh, sm.xl[lane] = xl;
    }
    __syncwarp();
    // ---- S and f_S
    if (lane < NF) {
      const int q = lane, qs = q / DPF, sj = q - qs * DPF;
      const double sq = (qs & 1) ? 1.0 : -1.0;
      double wq[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) wq[i] = sm.w[i * NC + q];
#pragma unroll 2
      for (int p = 0; p < NF; ++p) {
        const int ps = p / DPF, ax = ps >> 1, side = ps & 1;
        const bool pin = ((side ? hi : lo) >> ax) & 1u;
        double s_ = assemble_entry(a, b, __ldg(Dg + (NI + p) * N + NI + q), __ldg(Mg + (NI + p) * N + NI + q));
#pragma unroll
        for (int i = 0; i < NI; ++i) s_ = fma(-sm.afi[p * NI + i], wq[i], s_);
        double* dst = C.sval + sm.rstart[p] + static_cast<int64_t>(sm.rank[ps * NS + qs]) * DPF + sj;
        const double v = (side ? sq : -sq) * s_;
        *dst = (parity == 1 && pin && ps == qs) ? *dst + v : v;
      }
      // f_S,p = f_F,p - A_Fi x  (x in double-double), p = lane
      const int ps = lane / DPF, ax = ps >> 1, side = ps & 1;
      const bool pin = ((side ? hi : lo) >> ax) & 1u;
      ddv acc = {sm.ff[lane], 0.0};
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const double api = sm.afi[lane * NI + i];
        acc = dd_fma_sub(acc, api, sm.xh[i]);
        acc.lo = fma(-api, sm.xl[i], acc.lo);
      }
      const double v = (side ? 1.0 : -1.0) * (acc.hi + acc.lo);
      const int row_ = sm.frow[lane];
      C.fs[row_] = (parity == 1 && pin) ? C.fs[row_] + v : v;
    }
    __syncwarp();
  }
}

template <int DIM, int NI, int NF>
void launch_sc_warp(const CondArgs& c, int parity, cudaStream_t st) {
  using SM = ScWarpSm<DIM, NI, NF>;
  const size_t smem = 4 * sizeof(SM);
  static const bool attr_set = [] {
    return cudaFuncSetAttribute(k_sc_warp<DIM, NI, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(4 * sizeof(SM))) == cudaSuccess;
  }();
  (void)attr_set;
  const int64_t cnt = parity_count(c.m);
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((cnt + 3) / 4, 148 * 8)));
  k_sc_warp<DIM, NI, NF><<<grid, 128, smem, st>>>(c, parity);
}

// One warp: y <- L^-T L^-1 y for CPW columns y_c (stride ys) with the
// Cholesky factor L (row-major lower, leading dimension ni) and its inverse
// diagonal.  The columns live in registers (lane owns rows lane + 32 s), y_j is
// broadcast with a shuffle: no memory round trip and no barrier on the chain;
// CPW independent columns interleave their chains.
template <int S, int CPW>
__device__ void warp_chol_solve(const double* l, int lda, const double* ld, int ni, double* const (&y)[CPW], int ys,
                                int ncol, int lane) {
  double v[CPW][S];
#pragma unroll
  for (int c = 0; c < CPW; ++c)
#pragma unroll
    for (int t = 0; t < S; ++t) {
      const int i = 32 * t + lane;
      v[c][t] = (c < ncol && i < ni) ? y[c][i * ys] : 0.0;
    }
#pragma unroll
  for (int s = 0; s < S; ++s)
    for (int jj = 0; jj < 32; ++jj) {  // forward: L z = y
      const int j = 32 * s + jj;
      if (j >= ni) break;
      const double inv = ld[j];
      double yj[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        if (lane == jj) v[c][s] *= inv;
        yj[c] = __shfl_sync(0xffffffffu, v[c][s], jj);
      }
#pragma unroll
      for (int t = s; t < S; ++t) {
        const int i = 32 * t + lane;
        if (i > j && i < ni) {
          const double lij = l[i * lda + j];
#pragma unroll
          for (int c = 0; c < CPW; ++c) v[c][t] = fma(-lij, yj[c], v[c][t]);
        }
      }
    }
#pragma unroll
  for (int s = S - 1; s >= 0; --s)
    for (int jj = 31; jj >= 0; --jj) {  // backward: L^T x = z
      const int j = 32 * s + jj;
      if (j >= ni) continue;
      const double inv = ld[j];
      double yj[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        if (lane == jj) v[c][s] *= inv;
        yj[c] = __shfl_sync(0xffffffffu, v[c][s], jj);
      }
#pragma unroll
      for (int t = 0; t <= s; ++t) {
        const int i = 32 * t + lane;
        if (i < j) {
          const double lji = l[j * lda + i];
#pragma unroll
          for (int c = 0; c < CPW; ++c) v[c][t] = fma(-lji, yj[c], v[c][t]);
        }
      }
    }
#pragma unroll
  for (int c = 0; c < CPW; ++c)
#pragma unroll
    for (int t = 0; t < S; ++t) {
      const int i = 32 * t + lane;
      if (c < ncol && i < ni) y[c][i * ys] = v[c][t];
    }
}

constexpr int kSC = 256;  // threads of the k >= 1 condensation CTA
constexpr int kSK = 16;   // K chunk of the S GEMM

// Per cell: Cholesky of A_ii; [W | x] = A_ii^-1 [A_iF | f_i] by warp-level
// sweeps (one column per warp at a time); x refined to double-double (exact
// residuals, warp sweep corrections); S = A_FF - A_Fi W as a tiled GEMM (A_Fi
// assembled into shared memory by K chunks, 4 x 4 register tiles);
// f_S = f_F - A_Fi x with error-free products; scatter as before.
template <int S>
__global__ void __launch_bounds__(kSC, 1) k_sc_cta(CondArgs C, int parity, double* gws, int64_t stride, int use_smem) {
  extern __shared__ double smem[];
  __shared__ double afs[96 * kSK];  // A_Fi chunk (p, k), nf <= 96
  __shared__ double wks[kSK * 96];  // W chunk (k, q)
  // use_smem: 1 = whole workspace in shared memory, 2 = only A_ii / its factor
  double* ws = use_smem == 1 ? smem : gws + blockIdx.x * stride;
  const DevMesh& m = C.m;
  const int n = m.n, ni = m.nint, nf = C.nF, dpf = m.dpf, dim = m.dim;
  const int nc = nf + 1;  // [W | x] columns
  const ScLayout L = sc_layout(ni, nc, n);
  double* aii = use_smem == 2 ? smem : ws + L.aii;
  const int lda = use_smem == 2 ? (ni | 1) : ni;  // odd row stride: conflict-free column reads of the factor
  double* wx = ws + L.aif;  // ni x nc: [A_iF | f_i] -> [W | x]
  double* xl = ws + L.xl;
  double* r = ws + L.r;
  double* ldi = ws + L.d;  // 1 / L_jj
  double* fl = ws + L.f;
  __shared__ int flag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cnt = static_cast<uint32_t>(parity_count(m));
  for (uint32_t t = blockIdx.x; t < cnt; t += gridDim.x) {
    int cc[3];
    const int e = parity_cell32(m, parity, t, cc);
    if (e < 0) continue;
    const double a = C.alpha[e], b = C.beta[e];
    if (tid == 0) flag = 0;
    for (int i = tid; i < n; i += kSC) fl[i] = C.f[static_cast<int64_t>(e) * n + i];
    for (int idx = tid; idx < ni * ni; idx += kSC) {
      const int i = idx / ni, j = idx - i * ni;
      aii[i * lda + j] = assemble_entry(a, b, C.fx.D[i * n + j], C.fx.M[i * n + j]);
    }
    for (int idx = tid; idx < ni * nc; idx += kSC) {
      const int i = idx / nc, c = idx - i * nc;
      wx[idx] = c < nf ? assemble_entry(a, b, C.fx.D[i * n + ni + c], C.fx.M[i * n + ni + c]) : C.f[static_cast<int64_t>(e) * n + i];
    }
    __syncthreads();
    cta_cholesky(aii, ni, &flag, lda);
    if (flag && tid == 0) atomicOr(C.status, 2);
    for (int i = tid; i < ni; i += kSC) {
      ldi[i] = 1.0 / aii[i * lda + i];  // inverse diagonal of L
      xl[i] = 0.0;
    }
    __syncthreads();
    // [W | x] = A_ii^-1 [A_iF | f_i]: two columns per warp at a time
    for (int c = 2 * warp; c < nc; c += 2 * (kSC / 32)) {
      double* const cols[2] = {wx + c, wx + c + 1};
      warp_chol_solve<S, 2>(aii, lda, ldi, ni, cols, nc, min(2, nc - c), lane);
    }
    __syncthreads();
    // x to double-double: r = f_i - A_ii (x + xl) exactly accumulated, x += A_ii^-1 r
    for (int step = 0; step < 3; ++step) {
      for (int i = tid; i < ni; i += kSC) {
        ddv acc = {fl[i], 0.0};
        for (int j = 0; j < ni; ++j) {
          const double aij = assemble_entry(a, b, C.fx.D[i * n + j], C.fx.M[i * n + j]);
          acc = dd_fma_sub(acc, aij, wx[j * nc + nf]);
          acc.lo = fma(-aij, xl[j], acc.lo);
        }
        r[i] = acc.hi + acc.lo;
      }
      __syncthreads();
      if (warp == 0) {
        double* const rc[1] = {r};
        warp_chol_solve<S, 1>(aii, lda, ldi, ni, rc, 1, 1, lane);
        for (int i = lane; i < ni; i += 32) {
          const ddv v = dd_add_d({wx[i * nc + nf], xl[i]}, r[i]);
          wx[i * nc + nf] = v.hi;
          xl[i] = v.lo;
        }
      }
      __syncthreads();
    }
    // scatter tables
    unsigned lo = 0, hi = 0;
    for (int x = 0; x < dim; ++x) {
      const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
      const int Nx = static_cast<int>(x == 0 ? m.N[0] : (x == 1 ? m.N[1] : m.N[2]));
      lo |= static_cast<unsigned>(cx > 0) << x;
      hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
    }
    // f_S,p = f_F,p - A_Fi x  (x in double-double)
    for (int p = tid; p < nf; p += kSC) {
      const int ps = p / dpf, sub = p - ps * dpf;
      const int ax = ps >> 1, side = ps & 1;
      const bool pin = (((side) ? hi : lo) >> ax) & 1u;
      const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0), cc[2] + (ax == 2 ? side : 0));
      ddv acc = {fl[ni + p], 0.0};
      for (int i = 0; i < ni; ++i) {
        const double api = assemble_entry(a, b, C.fx.D[(ni + p) * n + i], C.fx.M[(ni + p) * n + i]);
        acc = dd_fma_sub(acc, api, wx[i * nc + nf]);
        acc.lo = fma(-api, xl[i], acc.lo);
      }
      const double v = (side ? 1.0 : -1.0) * (acc.hi + acc.lo);
      const int row = face * dpf + sub;
      C.fs[row] = (parity == 1 && pin) ? C.fs[row] + v : v;
    }
    // S = A_FF - A_Fi W: 4 x 4 register tiles over (p, q), K in chunks staged in shared memory
    const int TS = (nf + 3) / 4;
    for (int tile0 = 0; tile0 < TS * TS; tile0 += kSC) {
      const int tile = tile0 + tid;
      const bool own = tile < TS * TS;
      const int p0 = own ? (tile / TS) * 4 : 0, q0 = own ? (tile % TS) * 4 : 0;
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
      for (int k0 = 0; k0 < ni; k0 += kSK) {
        const int kw = min(kSK, ni - k0);
        __syncthreads();
        for (int idx = tid; idx < nf * kSK; idx += kSC) {
          const int p = idx / kSK, kk = idx - p * kSK;
          afs[idx] = kk < kw ? assemble_entry(a, b, C.fx.D[(ni + p) * n + k0 + kk], C.fx.M[(ni + p) * n + k0 + kk]) : 0.0;
        }
        for (int idx = tid; idx < kSK * nf; idx += kSC) {
          const int kk = idx / nf, q = idx - kk * nf;
          wks[idx] = kk < kw ? wx[(k0 + kk) * nc + q] : 0.0;
        }
        __syncthreads();
        if (own)
          for (int kk = 0; kk < kw; ++kk) {
            double av[4], wv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = p0 + i < nf ? afs[(p0 + i) * kSK + kk] : 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) wv[j] = q0 + j < nf ? wks[kk * nf + q0 + j] : 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], wv[j], acc[i][j]);
          }
      }
      if (own)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int p = p0 + i;
          if (p >= nf) continue;
          const int ps = p / dpf, sub = p - ps * dpf;
          const int ax = ps >> 1, side = ps & 1;
          const bool pin = (((side) ? hi : lo) >> ax) & 1u;
          const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0),
                                     cc[2] + (ax == 2 ? side : 0));
          const double sp = side ? 1.0 : -1.0;
          const bool add = parity == 1 && pin;
          const int row = face * dpf + sub;
          const int64_t start = C.rowoff[row];
          const int ca = ax == 0 ? cc[0] : (ax == 1 ? cc[1] : cc[2]);
          const int na = static_cast<int>(ax == 0 ? m.N[0] : (ax == 1 ? m.N[1] : m.N[2]));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int q = q0 + j;
            if (q >= nf) continue;
            const double sv = assemble_entry(a, b, C.fx.D[(ni + p) * n + ni + q], C.fx.M[(ni + p) * n + ni + q]) - acc[i][j];
            const int qs = q / dpf, sj = q - qs * dpf;
            const double sq = (qs & 1) ? 1.0 : -1.0;
            const int rk = col_rank_fast(dim, ps, qs, lo, hi, ca, na, true);
            double* dst = C.sval + start + static_cast<int64_t>(rk) * dpf + sj;
            const double v = sp * sq * sv;
            *dst = (add && ps == qs) ? *dst + v : v;
          }
        }
    }
    __syncthreads();
  }
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
    if (c.host_consts && !getenv("HDR_SC_NO_PENCIL")) {  // one pass over all cells (no colours), coalesced rows
      PencilConst<3> p3;
      PencilConst<2> p2;
      if (c.m.dim == 3 ? pencil_setup<3>(c.host_consts, p3) : pencil_setup<2>(c.host_consts, p2)) {
        if (parity == 0) {
          if (c.m.dim == 3) launch_sc_pencil<3>(c, p3, st);
          else launch_sc_pencil<2>(c, p2, st);
        }
        return;
      }
    }
    const unsigned nb = static_cast<unsigned>((parity_count(c.m) + 127) / 128);
    if (c.m.dim == 3)
      k_sc_rt0<3><<<nb, 128, 0, st>>>(c, parity);
    else
      k_sc_rt0<2><<<nb, 128, 0, st>>>(c, parity);
    count_launch();
    return;
  }
  if (!getenv("HDR_SC_NO_WARP")) {  // one warp per cell where the whole block fits a warp
    const int dim = c.m.dim, ni = c.m.nint, nf = c.nF;
    bool done = true;
    if (dim == 3 && ni == 12 && nf == 24) launch_sc_warp<3, 12, 24>(c, parity, st);       // RT1 hexahedra
    else if (dim == 2 && ni == 4 && nf == 8) launch_sc_warp<2, 4, 8>(c, parity, st);      // RT1 quadrilaterals
    else if (dim == 2 && ni == 12 && nf == 12) launch_sc_warp<2, 12, 12>(c, parity, st);  // RT2 quadrilaterals
    else done = false;
    if (done) {
      count_launch();
      return;
    }
  }
  if (c.m.nint <= 32) {  // small interior blocks: the 128-thread shared-memory kernel
    const ScLayout Ls = sc_layout(c.m.nint, c.nF, c.m.n);
    const bool sm_ok = Ls.total * 8 <= 96 * 1024;
    const size_t smem_s = sm_ok ? static_cast<size_t>(Ls.total) * 8 : 0;
    if (sm_ok) cudaFuncSetAttribute(k_sc_small, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_s));
    const int64_t cnt_s = parity_count(c.m);
    int64_t grid_s = sm_ok ? std::min<int64_t>(cnt_s, 148 * 16) : std::min<int64_t>(cnt_s, ws_doubles / Ls.total);
    grid_s = std::max<int64_t>(grid_s, 1);
    k_sc_small<<<static_cast<unsigned>(grid_s), kNT, smem_s, st>>>(c, parity, gws, Ls.total, sm_ok ? 1 : 0);
    count_launch();
    return;
  }
  const ScLayout L = sc_layout(c.m.nint, c.nF + 1, c.m.n);
  const bool use_smem = L.total * 8 <= 96 * 1024;
  // otherwise keep at least the factor of A_ii on chip (the sweeps read it ni^2 times)
  const bool aii_smem = !use_smem && static_cast<int64_t>(c.m.nint) * (c.m.nint | 1) * 8 <= 190 * 1024;
  const size_t smem = use_smem ? static_cast<size_t>(L.total) * 8
                               : (aii_smem ? static_cast<size_t>(c.m.nint) * (c.m.nint | 1) * 8 : 0);
  const int mode = use_smem ? 1 : (aii_smem ? 2 : 0);
  const int64_t cnt = parity_count(c.m);
  int64_t grid = use_smem ? std::min<int64_t>(cnt, 148 * 16) : std::min<int64_t>(cnt, ws_doubles / L.total);
  grid = std::max<int64_t>(grid, 1);
  auto go = [&](auto kern) {
    if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<static_cast<unsigned>(grid), kSC, smem, st>>>(c, parity, gws, L.total, mode);
  };
  const int ni = c.m.nint;  // rows per lane in the warp-level triangular sweeps
  if (ni <= 32) go(k_sc_cta<1>);
  else if (ni <= 64) go(k_sc_cta<2>);
  else if (ni <= 96) go(k_sc_cta<3>);
  else if (ni <= 128) go(k_sc_cta<4>);
  else go(k_sc_cta<5>);
  count_launch();
}

int64_t condense_ws_doubles(const DevMesh& m, int nF) {
  if (m.nint == 0) return 0;
  const ScLayout L = sc_layout(m.nint, nF + 1, m.n);
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
