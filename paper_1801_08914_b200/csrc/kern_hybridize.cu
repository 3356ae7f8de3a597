// K2+K3+K4: fused element assembly, structured element solve and deterministic
// scatter of hybridize (src/reduction.cpp:262-354 with element_matrices,
// src/rt_space.cpp:345-374), plus the hybrid recovery (recover_hybrid,
// src/reduction.cpp:356-446).
//
// Per cell T (alpha, beta, f_T):
//   A_T   = fl(fl(alpha D) + fl(beta M))                         (bit-exact, never formed)
//   A0^-1 = (N0 + X diag(s) X^T) / beta,  s_j = beta / (beta + alpha lambda_j)
//   Delta = A_T - A0 = alpha E + beta Ma + delta(alpha, beta)     (generated on the fly)
//   V     = A0^-1 [E_F | f_T]                (face columns + load column)
//   [H_T | g_T] = E_F^T V + sum_{p>=1} (-1)^p V_F^T Y_p,  Y_1 = Delta V, Y_p = Delta A0^-1 Y_{p-1}
// H_T = C_T A_T^-1 C_T^T and g_T = C_T A_T^-1 f_T for the unit constraint rows of
// build_C (src/reduction.cpp:172-181): C_T selects the cell's interior-face dofs.
// The Neumann order P is chosen per cell from the bound rho*alpha/beta so that
// the truncation is below 1e-14 relative.
//
// Scatter: two launches, one per checkerboard colour.  Colour 0 stores, colour 1
// stores its off-diagonal face blocks and adds its same-face blocks (and g) to
// colour 0's values: every entry has at most two contributions (SURVEY.md §0
// item 7) and fl(a+b) = fl(b+a), so the result is deterministic without atomics.
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <vector>
#include <cstdlib>
#include <cstring>

#include "hdr_device.cuh"
#include "kernels.hpp"
#include "rt0_exact.cuh"

#ifndef HDR_L2HINT
#define HDR_L2HINT 1
#endif
#ifndef HDR_ROWS_MINB
#define HDR_ROWS_MINB 6
#endif

namespace hdr {

namespace {

// out-of-line form (the recovery kernel keeps its registers for the fast path)
template <int N, int NC, bool IDENT>
__device__ __noinline__ void rt0_exact_ool(const double* D, const double* M, double a, double b, unsigned bmask,
                                           const double* rh, const double* rl, double* out, int* status) {
  rt0_exact<N, NC, IDENT>(D, M, a, b, bmask, rh, rl, out, status);
}

// ------------------------------------------------------------------ k = 0

template <int N>
struct Rt0Const {
  double D[N * N], M[N * N], E[N * N], Ma[N * N], N0[N * N], X[N];
  double lam, rho;
};

// ------------------------------------------------------------------ k = 0, lane-per-row form
//
// N = 2*DIM lanes per cell (one per face / row of H_T), 32/N cells per warp.
// Pass 0 (colour-0 cells) writes [H_T | g_T] (N x (N+1)) to a per-cell staging
// slot; pass 1 (colour-1 cells) computes its own [H_T | g_T] and, for each of
// its interior faces, merges the colour-0 neighbour's row of that face from the
// staging buffer and writes the complete H row (and g entry) in one go:
// every H row is written by exactly one lane, contiguously, so sectors are
// filled whole and nothing is read back from H.
// Row k of [H_T | g_T] for one RT0 cell, lanes k = 0..N-1 of a group.
// fp64: row k of V = A0^-1 (and of [V | w]), the exact rounding errors delta_k,:
// (full error-free transform only where M_kl != 0, i.e. the two slots of k's
// axis; elsewhere A_kl = fl(alpha D_kl) and delta = -err(alpha D_kl)).
// fp32: the Neumann correction (<= 1.5e-8 |H| on BASELINE inputs):
// Y_p = Delta T_{p-1}, row k of the order-p term = sum_j V_kj (Y_p)_j,:  (A0^-1
// symmetric), T_p rows = those terms.  P is warp-uniform.
// vsh / ysh / tsh: N x (N+1) fp32, dsh: N x N fp32 warp scratch of this cell.
template <int DIM>
__device__ __forceinline__ void rt0_row_math(const HybArgs& A, const Rt0Const<2 * DIM>& c, int e, int k, int& P,
                                             bool real, float* vsh, float* ysh, float* tsh, float* dsh,
                                             double (&h)[2 * DIM + 1], bool& exact) {
  constexpr int N = 2 * DIM;
  constexpr int NC = N + 1;
  const double* Dk = A.fx.D + k * N;
  const double* Mk = A.fx.M + k * N;
  const double* Ek = A.fx.E + k * N;
  const double* Mak = A.fx.Ma + k * N;
  const double* N0k = A.fx.N0 + k * N;
  const double a = A.alpha[e], b = A.beta[e];
  const double ib = 1.0 / b;
  const double s = b / fma(a, c.lam, b);
  const double xs = __ldg(A.fx.X + k) * s;
  const double* fe = A.f + static_cast<int64_t>(e) * N;
  double vk[N];
  double wk = 0.0;  // (A0^-1 f)_k
#pragma unroll
  for (int j = 0; j < N; ++j) {
    vk[j] = fma(xs, c.X[j], __ldg(N0k + j)) * ib;
    wk = fma(vk[j], fe[j], wk);
  }
#pragma unroll
  for (int j = 0; j < N; ++j) vsh[k * NC + j] = static_cast<float>(vk[j]);
  vsh[k * NC + N] = static_cast<float>(wk);
  // Delta row k
  const int k0 = k & ~1;
#pragma unroll
  for (int j = 0; j < 2; ++j) {  // same axis: M_kl != 0
    const int l = k0 + j;
    dsh[k * N + l] = static_cast<float>(delta_entry(a, b, __ldg(Dk + l), __ldg(Mk + l), __ldg(Ek + l), __ldg(Mak + l)));
  }
#pragma unroll
  for (int j = 0; j < N - 2; ++j) {  // other axes: M_kl = Ma_kl = 0 exactly
    int l = k0 + 2 + j;
    l = l >= N ? l - N : l;
    const double d = __ldg(Dk + l);
    const double p1 = __dmul_rn(a, d);
    const double e1 = __fma_rn(a, d, -p1);
    dsh[k * N + l] = static_cast<float>(__fma_rn(a, __ldg(Ek + l), -e1));
  }
  __syncwarp();
  // order 1: y_k = Delta_k,: [V | w]
  float y[NC];
#pragma unroll
  for (int q = 0; q <= N; ++q) y[q] = 0.f;
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const float dl = dsh[k * N + l];
#pragma unroll
    for (int q = 0; q <= N; ++q) y[q] = fmaf(dl, vsh[l * NC + q], y[q]);
  }
#pragma unroll
  for (int q = 0; q <= N; ++q) ysh[k * NC + q] = y[q];
  float vk32[N];
#pragma unroll
  for (int j = 0; j < N; ++j) vk32[j] = static_cast<float>(vk[j]);
  __syncwarp();
  float corr[NC];
#pragma unroll
  for (int q = 0; q <= N; ++q) corr[q] = 0.f;
  for (int p = 1; p <= P; ++p) {
    const float sg = (p & 1) ? 1.f : -1.f;  // corr is subtracted: order p enters as (-1)^p
    float t[NC];
#pragma unroll
    for (int q = 0; q <= N; ++q) t[q] = 0.f;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int q = 0; q <= N; ++q) t[q] = fmaf(vk32[j], ysh[j * NC + q], t[q]);
#pragma unroll
    for (int q = 0; q <= N; ++q) corr[q] = fmaf(sg, t[q], corr[q]);
    if (p == 1) {
      // a-posteriori order control (as kern_warp.cu): 10 (|C| / |H0|)^2 <= 1e-12 -> order 1 suffices
      float cm = 0.f, hm = 0.f;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        cm = fmaxf(cm, fabsf(corr[q]));
        hm = fmaxf(hm, fabsf(vk32[q]));
      }
      const int lane = threadIdx.x & 31, base = lane - k;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        cm = fmaxf(cm, __shfl_sync(0xffffffffu, cm, base + j));
        hm = fmaxf(hm, __shfl_sync(0xffffffffu, hm, base + j));
      }
      const double ratio = hm > 0.f ? static_cast<double>(cm) / hm : 0.0;
      bool ex = false;
      int pc = struct_order(ratio, A.p_max, A.eps32, ex);
      ex = real && (ex || A.force_exact);
      if (ex || !real) pc = 1;
      exact = ex;
      if (real && k == 0 && A.qlog) A.qlog[e] = static_cast<float>(ratio);
      P = __reduce_max_sync(0xffffffffu, pc);
    }
    if (p == P) break;
#pragma unroll
    for (int q = 0; q <= N; ++q) tsh[k * NC + q] = t[q];
    __syncwarp();
#pragma unroll
    for (int q = 0; q <= N; ++q) y[q] = 0.f;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const float dl = dsh[k * N + l];
#pragma unroll
      for (int q = 0; q <= N; ++q) y[q] = fmaf(dl, tsh[l * NC + q], y[q]);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q <= N; ++q) ysh[k * NC + q] = y[q];
    __syncwarp();
  }
#pragma unroll
  for (int q = 0; q <= N; ++q) h[q] = (q < N ? vk[q] : wk) - static_cast<double>(corr[q]);
}

template <int DIM, int PASS>
__device__ __forceinline__ bool rt0_rows_body(const HybArgs& A, const Rt0Const<2 * DIM>& c, double* stage) {
  constexpr int N = 2 * DIM;
  constexpr int NC = N + 1;
  constexpr int G = 32 / N;  // cells per warp
  constexpr int W = 4;       // warps per block
  __shared__ float vbuf[W][G + 1][N * NC];  // group G: scratch of the spare lanes
  __shared__ float ybuf[W][G + 1][N * NC];
  __shared__ float tbuf[W][G + 1][N * NC];
  __shared__ float dbuf[W][G + 1][N * N];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / N, k = lane - grp * N;
  const uint32_t t = (blockIdx.x * W + warp) * G + grp;
  int cc[3] = {0, 0, 0};
  int e = -1;
  if (grp < G && t < static_cast<uint32_t>(parity_count(A.m))) e = parity_cell32(A.m, PASS, t, cc);
  const bool valid = e >= 0;
  // spare lanes compute on cell 0 in their own scratch group (results discarded)
  // so every lane takes part in the warp barriers, shuffles and reductions
  const int gi = grp < G ? grp : G;
  const int kk = k;
  const int ee = valid ? e : 0;
  int P = 1;
  double h[N + 1];
  bool exact = false;
  const bool& rejected = exact;
  rt0_row_math<DIM>(A, c, ee, kk, P, valid, vbuf[warp][gi], ybuf[warp][gi], tbuf[warp][gi], dbuf[warp][gi], h, exact);
  if (!valid) return rejected;
  if (exact) {  // rejected by the estimate: this lane's row from the exact solve
    if (k == 0) atomicAdd(A.xcount, 1);
    double hx[N * NC];
    rt0_exact_ool<N, NC, true>(A.fx.D, A.fx.M, A.alpha[e], A.beta[e], rt0_bmask<DIM>(A.m, cc),
                               A.f + static_cast<int64_t>(e) * N, nullptr, hx, A.status);
#pragma unroll
    for (int q = 0; q <= N; ++q) h[q] = hx[k * NC + q];
  }
  if (PASS == 0) {
    double* slot = stage + static_cast<int64_t>(t) * (N * NC) + k * NC;
    if (HDR_L2HINT >= 1) {
      const uint64_t pol = l2_policy_evict_last();
#pragma unroll
      for (int q = 0; q <= N; ++q) st_l2hint(slot + q, h[q], pol);
    } else {
#pragma unroll
      for (int q = 0; q <= N; ++q) slot[q] = h[q];
    }
    return rejected;
  }
  // pass 1: complete rows of this cell's interior faces
  const int a = k >> 1, side = k & 1;
  const int ca = a == 0 ? cc[0] : (a == 1 ? cc[1] : cc[2]);
  const int na = static_cast<int>(a == 0 ? A.m.N[0] : (a == 1 ? A.m.N[1] : A.m.N[2]));
  const bool kin = side ? (ca + 1 < na) : (ca > 0);
  if (!kin) return rejected;
  const int step = side ? 1 : -1;
  const int nc[3] = {cc[0] + (a == 0 ? step : 0), cc[1] + (a == 1 ? step : 0), cc[2] + (a == 2 ? step : 0)};
  const int kn = k ^ 1;  // the shared face's slot in the neighbour
  // issue the dependent loads first: the neighbour's row from the stage, the row start
  const uint32_t half = static_cast<uint32_t>((A.m.N[0] + 1) / 2);
  const uint32_t tn = (static_cast<uint32_t>(nc[1]) + static_cast<uint32_t>(A.m.N[1]) * nc[2]) * half + (nc[0] >> 1);
  const double* nrow_p = stage + static_cast<int64_t>(tn) * (N * NC) + kn * NC;
  double nrow[NC];
  const uint64_t pol_first = l2_policy_evict_first();
#pragma unroll
  for (int q = 0; q <= N; ++q) nrow[q] = HDR_L2HINT >= 2 ? ld_l2hint(nrow_p + q, pol_first) : nrow_p[q];
  const int face = face_id32(A.m, a, cc[0] + (a == 0 ? side : 0), cc[1] + (a == 1 ? side : 0), cc[2] + (a == 2 ? side : 0));
  const int row = A.mbase[face];
  const int64_t start = A.rowoff[row];
  // boundary flags of the cell (own faces) and the neighbour's far face along k's axis
  unsigned lo = 0, hi = 0;
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
    const int Nx = static_cast<int>(x == 0 ? A.m.N[0] : (x == 1 ? A.m.N[1] : A.m.N[2]));
    lo |= static_cast<unsigned>(cx > 0) << x;
    hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
  }
  const unsigned far = side ? static_cast<unsigned>(ca + 2 < na) : static_cast<unsigned>(ca >= 2);
  const unsigned flags = lo | (hi << DIM) | (far << (2 * DIM));
  // packed column ranks of this row (host-built table, rank_table_rt0): own slot q
  // -> bits 4q, neighbour slot q -> bits 4(N+q); 15 = absent
  const uint64_t* tab = A.rank_tab + (static_cast<size_t>(k) << (2 * DIM + 1)) * 2 + flags * 2;
  const uint64_t own = __ldg(tab), nbr = __ldg(tab + 1);
  double* out = A.hval + start;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const unsigned r = static_cast<unsigned>(own >> (4 * q)) & 15u;
    if (r == 15u) continue;
    double v = h[q];
    if (q == k) v = v + nrow_p[kn];
    if (HDR_L2HINT >= 1) st_l2hint(out + r, v, pol_first);
    else out[r] = v;
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const unsigned r = static_cast<unsigned>(nbr >> (4 * q)) & 15u;
    if (r == 15u) continue;
    if (HDR_L2HINT >= 1) st_l2hint(out + r, nrow[q], pol_first);
    else out[r] = nrow[q];
  }
  A.g[row] = h[N] + nrow[N];
  return rejected;
}

template <int DIM, int PASS>
__global__ void __launch_bounds__(128, HDR_ROWS_MINB) k_rt0_rows(HybArgs A, Rt0Const<2 * DIM> c, double* stage) {
  rt0_rows_body<DIM, PASS>(A, c, stage);
}

// ------------------------------------------------------------------ k = 0, thread-per-cell form
//
// The same arithmetic as rt0_row_math, one thread per cell: [V | w] in fp32
// registers (fp64 entries recomputed where H is formed), Delta32 and the
// correction in per-thread shared-memory columns, the Neumann terms column by
// column (C_:q = V32 (Delta32 [V|w]_:q), higher orders continue the same
// column), the order chosen per cell.  No shuffles, no warp barriers, ~1/5 of
// the lane-per-row instructions.
#ifndef HDR_CELL_CT
#define HDR_CELL_CT 64
#endif
constexpr int kCT = HDR_CELL_CT;
#ifndef HDR_CELL_MINB
#define HDR_CELL_MINB 1
#endif

// ------------------------------------------------------------------ k = 0, structured first-order correction
//
// V = A0^-1 = (N0 + s X X^T) / beta = W / beta, W = M^-1 + t X X^T (t = s - 1),
// with M^-1 block-diagonal (2 x 2 per axis: RT0 basis functions of different
// axes are orthogonal) and Delta = alpha E + beta Ma + delta, so the first-order
// correction splits as
//   C = V Delta V = [ alpha (P0 + t P1 + t^2 P2) + beta (Q0 + t Q1 + t^2 Q2)
//                     + W delta W ] / beta^2
// with P. / Q. the constant t-polynomial coefficients of W E W
// (resp. Ma), precomputed on the host, and only the per-cell rounding errors
// delta (symmetric, exact error-free transforms) multiplied per cell.  C is
// symmetric (21 entries in 3D), lives in registers, and C_w = C f.  About 380
// fp32 FMAs per cell instead of 504, no shared-memory Delta / correction
// columns.  Cells whose order control asks for P > 1 (rare) run the general
// Neumann loop (rt0_general_correction) in shared-memory scratch.
template <int N>
struct Rt0Fast {
  static constexpr int NS = N * (N + 1) / 2;
  float n0[N][2];            // M^-1 row k on its axis pair (k & ~1, k | 1)
  float x[N];                // X (rank-one direction of the divergence)
  float p[3][NS], q[3][NS];  // s-polynomial coefficients (E part, Ma part), symmetric packed
};

__host__ __device__ constexpr int sym_idx(int k, int l, int n) {
  return k <= l ? k * n - k * (k - 1) / 2 + (l - k) : l * n - l * (l - 1) / 2 + (k - l);
}

// returns max |C| (q < N); hm = max |V| (the order control's reference size)
template <int DIM>
__device__ __forceinline__ float rt0_fast_correction(const Rt0Const<2 * DIM>& c, const Rt0Fast<2 * DIM>& F, double a,
                                                     double b, double s, double ib,
                                                     float (&C)[Rt0Fast<2 * DIM>::NS], float& hm) {
  constexpr int N = 2 * DIM;
  constexpr int NS = Rt0Fast<N>::NS;
  float dl[NS];  // delta: the exact rounding error of the reference's combine
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int l = k; l < N; ++l) {
      double p1, e1;
      two_prod(a, c.D[k * N + l], p1, e1);
      if ((k >> 1) == (l >> 1)) {
        double p2, e2, s_, e3;
        two_prod(b, c.M[k * N + l], p2, e2);
        two_sum_fast(p1, p2, s_, e3);
        dl[sym_idx(k, l, N)] = static_cast<float>(-((e1 + e2) + e3));
      } else {
        dl[sym_idx(k, l, N)] = static_cast<float>(-e1);  // M_kl = 0: A_kl = fl(alpha D_kl)
      }
    }
  float u[N], nu[N], gam = 0.f;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    float acc = 0.f;
#pragma unroll
    for (int l = 0; l < N; ++l) acc = fmaf(dl[sym_idx(k, l, N)], F.x[l], acc);
    u[k] = acc;
    gam = fmaf(F.x[k], acc, gam);
  }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int k0 = k & ~1;
    nu[k] = fmaf(F.n0[k][0], u[k0], F.n0[k][1] * u[k0 + 1]);
  }
  // W = N0 + s XX^T = M^-1 + (s - 1) XX^T: F.n0 holds the block-diagonal M^-1
  const float sf = static_cast<float>(s - 1.0), af = static_cast<float>(a), bf = static_cast<float>(b);
  const float ibf = static_cast<float>(ib), ib2 = static_cast<float>(ib * ib);
  const float s2g = sf * sf * gam;
  float cm = 0.f;
  hm = 0.f;
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int l = k; l < N; ++l) {
      const int i = sym_idx(k, l, N);
      // (N0 delta N0)_kl: N0 couples only the axis pairs of k and l
      const int k0 = k & ~1, l0 = l & ~1;
      float Bkl = F.n0[k][0] * F.n0[l][0] * dl[sym_idx(k0, l0, N)];
      Bkl = fmaf(F.n0[k][0] * F.n0[l][1], dl[sym_idx(k0, l0 + 1, N)], Bkl);
      Bkl = fmaf(F.n0[k][1] * F.n0[l][0], dl[sym_idx(k0 + 1, l0, N)], Bkl);
      Bkl = fmaf(F.n0[k][1] * F.n0[l][1], dl[sym_idx(k0 + 1, l0 + 1, N)], Bkl);
      float R = fmaf(sf, fmaf(nu[k], F.x[l], F.x[k] * nu[l]), Bkl);
      R = fmaf(s2g * F.x[k], F.x[l], R);
      const float Pm = fmaf(fmaf(F.p[2][i], sf, F.p[1][i]), sf, F.p[0][i]);
      const float Qm = fmaf(fmaf(F.q[2][i], sf, F.q[1][i]), sf, F.q[0][i]);
      const float v = fmaf(af, Pm, fmaf(bf, Qm, R)) * ib2;
      C[i] = v;
      cm = fmaxf(cm, fabsf(v));
      const float n0kl = (k >> 1) == (l >> 1) ? F.n0[k][l & 1] : 0.f;
      hm = fmaxf(hm, fabsf(fmaf(sf * F.x[k], F.x[l], n0kl) * ibf));
    }
  return cm;
}

// general Neumann correction through order P (the rare cells the order control
// sends here): Delta and V (fp32, full) in per-thread shared-memory scratch
// columns (stride = threads of the block), C (symmetric) written back there
template <int DIM>
__device__ __noinline__ void rt0_general_correction(const double* Dg, const double* Mg, const double* Eg,
                                                    const double* Mag, const double* N0g, const double* Xg, double a,
                                                    double b, double s, double ib, int P, float* scr, int stride) {
  constexpr int N = 2 * DIM;
  struct {
    const double *D, *M, *E, *Ma, *N0, *X;
  } c{Dg, Mg, Eg, Mag, N0g, Xg};
  float* dm = scr;
  float* vm = scr + N * N * stride;
  float* cw = scr + 2 * N * N * stride;
#pragma unroll 1
  for (int k = 0; k < N; ++k) {
    const double xs = c.X[k] * s;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      vm[(k * N + l) * stride] = static_cast<float>(fma(xs, c.X[l], c.N0[k * N + l]) * ib);
      double d;
      if ((k >> 1) == (l >> 1)) {
        d = delta_entry(a, b, c.D[k * N + l], c.M[k * N + l], c.E[k * N + l], c.Ma[k * N + l]);
      } else {
        const double p1 = __dmul_rn(a, c.D[k * N + l]);
        const double e1 = __fma_rn(a, c.D[k * N + l], -p1);
        d = __fma_rn(a, c.E[k * N + l], -e1);
      }
      dm[(k * N + l) * stride] = static_cast<float>(d);
    }
  }
#pragma unroll 1
  for (int q = 0; q < N; ++q) {
    float t[N], acc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      t[k] = vm[(k * N + q) * stride];
      acc[k] = 0.f;
    }
#pragma unroll 1
    for (int p = 1; p <= P; ++p) {
      float y[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        float v = 0.f;
#pragma unroll
        for (int l = 0; l < N; ++l) v = fmaf(dm[(k * N + l) * stride], t[l], v);
        y[k] = v;
      }
      const float sg = (p & 1) ? 1.f : -1.f;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < N; ++j) v = fmaf(vm[(k * N + j) * stride], y[j], v);
        t[k] = v;
        acc[k] = fmaf(sg, v, acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (k <= q) cw[sym_idx(k, q, N) * stride] = acc[k];
  }
}

// the cell's correction C (registers): structured first order, general loop if needed
// returns true when the cell is rejected: then C = 0 and the caller sets 1 / beta
// = 0, so every row of [H_T | g_T] comes out exactly 0 (no branch in the row
// code); the kernel then adds the cell's exact rows (rt0_exact) where its rows
// were assembled
template <int DIM>
__device__ __forceinline__ bool rt0_correction(const HybArgs& A, const Rt0Const<2 * DIM>& c, const Rt0Fast<2 * DIM>& F,
                                               double a, double b, double s, double ib, float* scr, int stride,
                                               float (&C)[Rt0Fast<2 * DIM>::NS], int64_t e) {
  constexpr int N = 2 * DIM;
  float hm;
  const float cm = rt0_fast_correction<DIM>(c, F, a, b, s, ib, C, hm);
  // a-posteriori order control and acceptance (hdr_device.cuh struct_order)
  const double ratio = hm > 0.f ? static_cast<double>(cm) / hm : 0.0;
#ifndef HDR_AB_NOQLOG
  if (A.qlog) A.qlog[e] = static_cast<float>(ratio);
#endif
  bool exact = false;
  const int P = struct_order(ratio, A.p_max, A.eps32, exact);
#ifdef HDR_AB_NOQLOG
  if (exact) {
#else
  if (exact || A.force_exact) {
#endif  // rejected: zero contribution (the caller zeroes 1 / beta too)
#pragma unroll
    for (int i = 0; i < Rt0Fast<N>::NS; ++i) C[i] = 0.f;
    atomicAdd(A.xcount, 1);
    return true;
  }
  if (P > 1) {
    rt0_general_correction<DIM>(A.fx.D, A.fx.M, A.fx.E, A.fx.Ma, A.fx.N0, A.fx.X, a, b, s, ib, P, scr, stride);
#pragma unroll
    for (int i = 0; i < Rt0Fast<N>::NS; ++i) C[i] = scr[(2 * N * N + i) * stride];
  }
  return false;
}



// row k of [H_T | g_T] = [V | w]_k,: (fp64) - [C | C f]_k,:
template <int DIM>
__device__ __forceinline__ void rt0_hrow_c(const Rt0Const<2 * DIM>& c, double s, double ib, const double (&f)[2 * DIM],
                                           const float (&C)[Rt0Fast<2 * DIM>::NS], int k, double (&h)[2 * DIM + 1]) {
  constexpr int N = 2 * DIM;
  const double xs = c.X[k] * s;
  double wk = 0.0;
  float cw = 0.f;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double vk = fma(xs, c.X[j], c.N0[k * N + j]) * ib;
    wk = fma(vk, f[j], wk);
    const float ckj = C[sym_idx(k, j, N)];
    h[j] = vk - static_cast<double>(ckj);
    cw = fmaf(ckj, static_cast<float>(f[j]), cw);
  }
  h[N] = wk - static_cast<double>(cw);
}

template <int DIM, int PASS, bool SIDE>
__device__ __forceinline__ bool rt0_cell_body(const HybArgs& A, const Rt0Const<2 * DIM>& c, const Rt0Fast<2 * DIM>& F,
                                              double* stage) {
  constexpr int N = 2 * DIM;
  constexpr int NC = N + 1;
  __shared__ float scr[2 * N * N + Rt0Fast<N>::NS][kCT];  // general-correction scratch (rare cells)
  __shared__ longlong2 pf_rs[SIDE ? N : 1][kCT];                       // {row start, row} per slot
  __shared__ unsigned long long pf_tab[SIDE ? N : 1][kCT];             // packed column ranks
  __shared__ double2 pf_sv[(SIDE && PASS == 1) ? N : 1][kCT];          // colour 0's {diagonal, g}
  const int tid = threadIdx.x;
  const uint32_t t = blockIdx.x * kCT + tid;
  int cc[3] = {0, 0, 0};
  if (t >= static_cast<uint32_t>(parity_count(A.m))) return false;
  const int e = parity_cell32(A.m, PASS, t, cc);
  if (e < 0) return false;
  const double a = A.alpha[e], b = A.beta[e];
  // SIDE: the scatter metadata of the cell's interior faces (row start + row, the
  // packed column ranks, colour 1: colour 0's parked side slot) is fetched into
  // shared memory now, so its latency hides behind the element solve
  unsigned lo = 0, hi = 0, inmask = 0;
  if (SIDE) {
#pragma unroll
    for (int x = 0; x < DIM; ++x) {
      const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
      const int Nx = static_cast<int>(x == 0 ? A.m.N[0] : (x == 1 ? A.m.N[1] : A.m.N[2]));
      lo |= static_cast<unsigned>(cx > 0) << x;
      hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int a_ = k >> 1, side = k & 1;
      const int ca = a_ == 0 ? cc[0] : (a_ == 1 ? cc[1] : cc[2]);
      const int na = static_cast<int>(a_ == 0 ? A.m.N[0] : (a_ == 1 ? A.m.N[1] : A.m.N[2]));
      if (!(side ? (ca + 1 < na) : (ca > 0))) continue;
      inmask |= 1u << k;
      const int face = face_id32(A.m, a_, cc[0] + (a_ == 0 ? side : 0), cc[1] + (a_ == 1 ? side : 0), cc[2] + (a_ == 2 ? side : 0));
      const unsigned far = side ? static_cast<unsigned>(ca + 2 < na) : static_cast<unsigned>(ca >= 2);
      const unsigned flags = lo | (hi << DIM) | (far << (2 * DIM));
      cp_async16(&pf_rs[k][tid], A.frs + face);
      cp_async8(&pf_tab[k][tid], A.rank_tab + ((static_cast<size_t>(k) << (2 * DIM + 1)) + flags) * 2);
      if (PASS == 1) cp_async16(&pf_sv[k][tid], stage + 2 * static_cast<int64_t>(face));
    }
  }
  const double ib = 1.0 / b;
  const double s = b / fma(a, c.lam, b);
  double f[N];
#pragma unroll
  for (int j = 0; j < N; ++j) f[j] = A.f[static_cast<int64_t>(e) * N + j];
  float C[Rt0Fast<N>::NS];
  const bool rejected = rt0_correction<DIM>(A, c, F, a, b, s, ib, &scr[0][tid], kCT, C, e);
  const double ibr = rejected ? 0.0 : ib;
  auto hrow = [&](int k, double (&h)[NC]) { rt0_hrow_c<DIM>(c, s, ibr, f, C, k, h); };
  if (SIDE) {
    // both colours write their own columns of their faces' rows straight into H;
    // the two shared quantities of a row (diagonal, g) meet in a per-row side
    // slot: colour 0 parks them, colour 1 adds its own (same bits as the
    // staged merge: h(colour 1) + h(colour 0)); side slots indexed by face
    const uint64_t pol = PASS == 0 ? l2_policy_evict_last() : l2_policy_evict_first();
    cp_async_wait_all();
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if (!((inmask >> k) & 1u)) continue;
      const longlong2 rs = pf_rs[k][tid];
      const uint64_t own = pf_tab[k][tid];
      const int row = static_cast<int>(rs.y);
      double* out = A.hval + rs.x;
      double h[NC];
      hrow(k, h);
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const unsigned r = static_cast<unsigned>(own >> (4 * q)) & 15u;
        if (r == 15u || q == k) continue;
        st_l2hint(out + r, h[q], pol);
      }
      if (PASS == 0) {
        const int a_ = k >> 1, side = k & 1;
        const int face = face_id32(A.m, a_, cc[0] + (a_ == 0 ? side : 0), cc[1] + (a_ == 1 ? side : 0), cc[2] + (a_ == 2 ? side : 0));
        double* sv = stage + 2 * static_cast<int64_t>(face);
        st_l2hint(sv, h[k], l2_policy_evict_last());
        st_l2hint(sv + 1, h[N], l2_policy_evict_last());
      } else {
        const double2 sv = pf_sv[k][tid];
        out[(own >> (4 * k)) & 15u] = h[k] + sv.x;
        A.g[row] = h[N] + sv.y;
      }
    }
#ifndef HDR_AB_NOFIX
    if (rejected) {  // rare: the cell's exact rows over its zero ones (same positions, same sums)
      double hx[N * NC];
      rt0_exact_ool<N, NC, true>(A.fx.D, A.fx.M, a, b, inmask, A.f + static_cast<int64_t>(e) * N, nullptr, hx,
                                 A.status);
      for (int k = 0; k < N; ++k) {
        if (!((inmask >> k) & 1u)) continue;
        const longlong2 rs = pf_rs[k][tid];
        const uint64_t own = pf_tab[k][tid];
        double* out = A.hval + rs.x;
        for (int q = 0; q < N; ++q) {
          const unsigned r = static_cast<unsigned>(own >> (4 * q)) & 15u;
          if (r != 15u && q != k) out[r] = hx[k * NC + q];
        }
        if (PASS == 0) {
          const int a_ = k >> 1, side = k & 1;
          const int face = face_id32(A.m, a_, cc[0] + (a_ == 0 ? side : 0), cc[1] + (a_ == 1 ? side : 0),
                                     cc[2] + (a_ == 2 ? side : 0));
          stage[2 * static_cast<int64_t>(face)] = hx[k * NC + k];
          stage[2 * static_cast<int64_t>(face) + 1] = hx[k * NC + N];
        } else {
          const double2 sv = pf_sv[k][tid];
          out[(own >> (4 * k)) & 15u] = hx[k * NC + k] + sv.x;
          A.g[static_cast<int>(rs.y)] = hx[k * NC + N] + sv.y;
        }
      }
    }
#endif
    return rejected;
  }
  return rejected;  // (SIDE is the only form)
}

template <int DIM, int PASS, bool SIDE>
__global__ void __launch_bounds__(kCT, HDR_CELL_MINB) k_rt0_cell(HybArgs A, Rt0Const<2 * DIM> c, Rt0Fast<2 * DIM> F,
                                                               double* stage) {
  rt0_cell_body<DIM, PASS, SIDE>(A, c, F, stage);
}

// ------------------------------------------------------------------ k = 0, brick form (default)
//
// The thread-per-cell kernels above store each H entry as an isolated 8-byte
// write; with HBM3e ECC every partially written 32-byte sector costs a DRAM
// read-fill, and those fills, not the arithmetic, set their time (measured:
// the same kernel without its H stores runs in half the time).  Here a CTA
// owns a brick of BX x BY x BZ cells (one thread per cell, the element solve
// of rt0_cell_correction) and assembles the H rows of the brick's faces in
// shared memory.  The rows of the faces of one axis along one x-line of the
// brick are consecutive in H (faces are numbered x-fastest, rows follow the
// interior faces in face order), so each such line is one contiguous segment,
// written out with coalesced full-sector stores, together with its g entries.
// Faces on a brick boundary are shared with the neighbouring brick: bricks are
// two-coloured (bx + by + bz parity, face-adjacent bricks differ); colour 0
// parks its row of such a face in a face-indexed stage (structure of arrays,
// coalesced) and colour 1 completes and writes it.  Every H row and g entry is
// written once; the two contributions to a diagonal entry / g entry meet as
// fl(h_minus + h_plus), the reference's two-term sum.
// brick shapes: BX cells along x (64 when the mesh is at least 48 cells wide,
// else 32) by 2 x 2 (3D) / 4 (2D); 512 threads per SM either way
#ifndef HDR_BRICK_Y3
#define HDR_BRICK_Y3 2
#endif
#ifndef HDR_BRICK_Z3
#define HDR_BRICK_Z3 2
#endif
#ifndef HDR_BRICK_XW
#define HDR_BRICK_XW 64  // BX of wide meshes
#endif
template <int DIM, int BX>
struct Brick {
  static constexpr int X = BX, Y = DIM == 3 ? HDR_BRICK_Y3 : 4, Z = DIM == 3 ? HDR_BRICK_Z3 : 1;
};

template <int DIM, int BX>
struct BrickDims {
  static constexpr int X = Brick<DIM, BX>::X, Y = Brick<DIM, BX>::Y, Z = Brick<DIM, BX>::Z;
  static constexpr int CT = X * Y * Z;
  static constexpr int MINB = 512 / CT;
  static constexpr int NL0 = Y * Z, NL1 = (Y + 1) * Z, NL2 = DIM == 3 ? Y * (Z + 1) : 0;
  static constexpr int NL = NL0 + NL1 + NL2;  // x-lines of faces of each axis
  static constexpr int RL = 4 * DIM - 1;      // longest H row
  static constexpr int CAP = (X + 1) * RL;    // entries of one line segment
  static constexpr size_t line_bytes = static_cast<size_t>(NL) * (CAP + X + 1) * sizeof(double);
  static constexpr size_t scratch_bytes = static_cast<size_t>(2 * 4 * DIM * DIM + DIM * (2 * DIM + 1)) * CT * sizeof(float);
  static constexpr size_t smem_bytes() { return line_bytes > scratch_bytes ? line_bytes : scratch_bytes; }
};

// entries of the H rows of faces x in [xa, x) of one x-line of axis-ax faces
// (x-faces: x is the face index; y / z faces: the cell column): row length =
// interior faces of the face's two cells - 1, in closed form
__device__ __forceinline__ int cnt_in(int lo, int hi, int a, int b) { return max(0, min(hi, b) - max(lo, a)); }
template <int DIM>
__device__ __forceinline__ int line_entries(const DevMesh& m, int ax, int xa, int x, int y, int z) {
  const int N0 = static_cast<int>(m.N[0]), N1 = static_cast<int>(m.N[1]), N2 = DIM == 3 ? static_cast<int>(m.N[2]) : 1;
  auto f = [](int c, int n) { return (c > 0) + (c + 1 < n); };
  const int big = 1 << 30;
  const int sx = cnt_in(xa, x, 1, big) + cnt_in(xa, x, -big, N0 - 1);  // sum of f(x', N0) over [xa, x)
  const int fz = DIM == 3 ? f(z, N2) : 0;
  if (ax == 0)
    return sx + cnt_in(xa, x, 2, big) + cnt_in(xa, x, -big, N0) + (x - xa) * (2 * (f(y, N1) + fz) - 1);
  if (ax == 1) return 2 * sx + (x - xa) * (f(y - 1, N1) + f(y, N1) + 2 * fz - 1);
  return 2 * sx + (x - xa) * (2 * f(y, N1) + f(z - 1, N2) + fz - 1);
}

// interior faces of a cell (its row-length contribution)
template <int DIM>
__device__ __forceinline__ int interior_faces(const DevMesh& m, int x, int y, int z) {
  int n = (x > 0) + (x + 1 < static_cast<int>(m.N[0])) + (y > 0) + (y + 1 < static_cast<int>(m.N[1]));
  if (DIM == 3) n += (z > 0) + (z + 1 < static_cast<int>(m.N[2]));
  return n;
}

// Exact path of the brick kernels: one CTA launched after the colour-1 brick
// kernel (programmatic dependent launch: its launch overlaps colour 1's tail; it
// returns at once when no cell was rejected).  The listed cells' [H_T | g_T] by
// rt0_exact (one thread per cell, colour 0 first, then colour 1, so no two cells
// of one round share an H entry) added into H and g at the positions of the
// row-rank table: their own columns held 0, the diagonal and g the neighbour's
// term.  The list length (xcount[2]) is reset for the next call.
template <int DIM>
__global__ void __launch_bounds__(256) k_rt0_exact(HybArgs A) {
  constexpr int N = 2 * DIM, NC = N + 1;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // both colours complete, their writes visible
  const int cnt = A.xcount[2];
  const DevMesh& m = A.m;
  for (int colour = 0; colour < 2 && cnt > 0; ++colour) {
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const int e = A.xlist[i];
      int cc[3];
      cell_coords32(m, static_cast<uint32_t>(e), cc);
      if (DIM == 2) cc[2] = 0;
      if (((cc[0] + cc[1] + cc[2]) & 1) != colour) continue;
      const unsigned bm = rt0_bmask<DIM>(m, cc);
      double hx[N * NC];
      rt0_exact<N, NC, true>(A.fx.D, A.fx.M, A.alpha[e], A.beta[e], bm, A.f + static_cast<int64_t>(e) * N, nullptr,
                             hx, A.status);
      unsigned lo = 0, hi = 0;
      for (int x = 0; x < DIM; ++x) {
        lo |= ((bm >> (2 * x)) & 1u) << x;
        hi |= ((bm >> (2 * x + 1)) & 1u) << x;
      }
      for (int k = 0; k < N; ++k) {
        if (!((bm >> k) & 1u)) continue;
        const int ax = k >> 1, side = k & 1;
        const int ca = ax == 0 ? cc[0] : (ax == 1 ? cc[1] : cc[2]);
        const int na = static_cast<int>(ax == 0 ? m.N[0] : (ax == 1 ? m.N[1] : m.N[2]));
        const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0),
                                   cc[2] + (ax == 2 ? side : 0));
        const longlong2 rs = A.frs[face];  // {row start, row}
        const unsigned far = side ? static_cast<unsigned>(ca + 2 < na) : static_cast<unsigned>(ca >= 2);
        const unsigned flags = lo | (hi << DIM) | (far << (2 * DIM));
        const uint64_t own = A.rank_tab[((static_cast<size_t>(k) << (2 * DIM + 1)) + flags) * 2];
        double* out = A.hval + rs.x;
        for (int q = 0; q < N; ++q) {
          const unsigned r = static_cast<unsigned>(own >> (4 * q)) & 15u;
          if (r != 15u) out[r] += hx[k * NC + q];
        }
        A.g[rs.y] += hx[k * NC + N];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) A.xcount[2] = 0;
}

template <int DIM, int COL, int BX>
__device__ __forceinline__ bool rt0_brick_body(const HybArgs& A, const Rt0Const<2 * DIM>& c, const Rt0Fast<2 * DIM>& F,
                                               double* stage, int nbx, int nby, int nbz) {
  using B = BrickDims<DIM, BX>;
  constexpr int N = 2 * DIM;
  constexpr int NC = N + 1;
  constexpr int X = B::X, Y = B::Y, Z = B::Z, CT = B::CT, NL = B::NL, CAP = B::CAP;
  extern __shared__ double bsm[];
  double* hbuf = bsm;              // NL x CAP: H line segments
  double* gbuf = bsm + NL * CAP;   // NL x (X + 1): g of the line's faces
  // general-correction scratch of the rare P > 1 cells: dead before the segments are filled
  float* scr = reinterpret_cast<float*>(bsm) + threadIdx.x;
  __shared__ long long l_base[NL];  // H offset of the line's first row
  __shared__ int l_row0[NL], l_pa[NL], l_oa[NL], l_ob[NL], l_olo[NL], l_ohi[NL];
  const DevMesh& m = A.m;
  const int N0 = static_cast<int>(m.N[0]), N1 = static_cast<int>(m.N[1]), N2 = DIM == 3 ? static_cast<int>(m.N[2]) : 1;
  // this colour's bricks: x index alternates within a (by, bz) row
  const int by = static_cast<int>(blockIdx.y), bz = static_cast<int>(blockIdx.z);  // grid (ceil(nbx / 2), nby, nbz)
  const int bx = 2 * static_cast<int>(blockIdx.x) + ((by + bz + COL) & 1);
  if (bx >= nbx || bz >= nbz) return false;
  const int x0 = bx * X, y0 = by * Y, z0 = bz * Z;
  const int ex = min(X, N0 - x0), ey = min(Y, N1 - y0), ez = DIM == 3 ? min(Z, N2 - z0) : 1;
  const int tid = threadIdx.x;
  // programmatic dependent launch: colour 1 may start (line metadata, element
  // solves) while colour 0's last wave runs; it waits before touching the stage
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // colour 1, resp. the exact-path kernel
  // face p of line (ax, jj, kk): x = x0 + p, y = y0 + jj, z = z0 + kk (ax 1: jj in [0, ey], ax 2: kk in [0, ez])
  auto line_face = [&](int ax, int jj, int kk, int p) { return face_id32(m, ax, x0 + p, y0 + jj, z0 + kk); };
  if (tid < NL) {  // line metadata
    int ax, jj, kk;
    if (tid < B::NL0) {
      ax = 0, jj = tid % Y, kk = tid / Y;
    } else if (tid < B::NL0 + B::NL1) {
      const int u = tid - B::NL0;
      ax = 1, jj = u % (Y + 1), kk = u / (Y + 1);
    } else {
      const int u = tid - B::NL0 - B::NL1;
      ax = 2, jj = u % Y, kk = u / Y;
    }
    int pa = 0, pb = -1, oa = 0, ob = -1;
    if (ax == 0) {
      if (jj < ey && kk < ez) {
        pa = x0 == 0 ? 1 : 0;
        pb = x0 + ex == N0 ? ex - 1 : ex;
        oa = COL == 1 ? pa : 1;
        ob = COL == 1 ? pb : ex - 1;
      }
    } else if (ax == 1) {
      const int j = y0 + jj;
      if (jj <= ey && kk < ez && j > 0 && j < N1) {
        pa = 0, pb = ex - 1;
        const bool edge = jj == 0 || jj == ey;
        oa = pa, ob = (COL == 0 && edge) ? -1 : pb;
      }
    } else {
      const int k = z0 + kk;
      if (jj < ey && kk <= ez && k > 0 && k < N2) {
        pa = 0, pb = ex - 1;
        const bool edge = kk == 0 || kk == ez;
        oa = pa, ob = (COL == 0 && edge) ? -1 : pb;
      }
    }
    long long base = 0;
    int row0 = 0, lo_ = 0, hi_ = 0;
    if (pb >= pa) {
      const longlong2 fa = A.frs[line_face(ax, jj, kk, pa)];
      base = fa.x;
      row0 = static_cast<int>(fa.y);
      if (ob >= oa) {
        const int y = y0 + jj, z = z0 + kk;
        lo_ = line_entries<DIM>(m, ax, x0 + pa, x0 + oa, y, z);
        hi_ = line_entries<DIM>(m, ax, x0 + pa, x0 + ob + 1, y, z);
      }
    }
    l_base[tid] = base;
    l_row0[tid] = row0;
    l_pa[tid] = pa;
    l_oa[tid] = oa;
    l_ob[tid] = ob;
    l_olo[tid] = lo_;
    l_ohi[tid] = hi_;
  }
  // the cell
  const int lx = tid % X, ly = (tid / X) % Y, lz = tid / (X * Y);
  const int cc[3] = {x0 + lx, y0 + ly, z0 + lz};
  const bool valid = lx < ex && ly < ey && lz < ez;
  double a = 1.0, b = 1.0, s = 1.0, ib = 1.0;
  bool rejected = false;
  float C[Rt0Fast<N>::NS];
  double f[N];
#pragma unroll
  for (int j = 0; j < N; ++j) f[j] = 0.0;
  if (valid) {
    const int64_t e = cc[0] + static_cast<int64_t>(N0) * (cc[1] + static_cast<int64_t>(N1) * cc[2]);
    a = A.alpha[e];
    b = A.beta[e];
#pragma unroll
    for (int j = 0; j < N; ++j) f[j] = A.f[e * N + j];
    ib = 1.0 / b;
    s = b / fma(a, c.lam, b);
    rejected = rt0_correction<DIM>(A, c, F, a, b, s, ib, scr, CT, C, e);
    if (rejected) {  // zero rows here; k_rt0_exact adds the exact ones after both colours
      ib = 0.0;
      A.xlist[atomicAdd(A.xcount + 2, 1)] = static_cast<int>(e);
    }
  }
  auto hrow = [&](int k, double (&h)[NC]) { rt0_hrow_c<DIM>(c, s, ib, f, C, k, h); };
  __syncthreads();  // line metadata
  if (COL == 1) asm volatile("griddepcontrol.wait;" ::: "memory");  // colour 0 complete, stage visible
  unsigned lo = 0, hi = 0;
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    const int Nx = x == 0 ? N0 : (x == 1 ? N1 : N2);
    lo |= static_cast<unsigned>(cc[x] > 0) << x;
    hi |= static_cast<unsigned>(cc[x] + 1 < Nx) << x;
  }
  const int lc[3] = {lx, ly, lz}, ec[3] = {ex, ey, ez};
  const int64_t nfaces = m.nfaces;
  // pass 1: own columns; the first contribution of diagonals / g (minus cell, or
  // the completed value on a colour-1 brick boundary); colour 0 parks boundary rows
  if (valid) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int ax = k >> 1, side = k & 1;
      const int ca = cc[ax], na = ax == 0 ? N0 : (ax == 1 ? N1 : N2);
      if (!(side ? (ca + 1 < na) : (ca > 0))) continue;
      const int face = face_id32(m, ax, cc[0] + (ax == 0 ? side : 0), cc[1] + (ax == 1 ? side : 0), cc[2] + (ax == 2 ? side : 0));
      const bool bb = side ? lc[ax] == ec[ax] - 1 : lc[ax] == 0;  // neighbour in the adjacent brick
      double h[NC];
      hrow(k, h);
      if (COL == 0 && bb) {
#pragma unroll
        for (int q = 0; q <= N; ++q) stage[q * nfaces + face] = h[q];
        continue;
      }
      const int l = ax == 0 ? ly + Y * lz : (ax == 1 ? B::NL0 + (ly + side) + (Y + 1) * lz : B::NL0 + B::NL1 + ly + Y * (lz + side));
      const int p = ax == 0 ? lx + side : lx;
      const unsigned far = side ? static_cast<unsigned>(ca + 2 < na) : static_cast<unsigned>(ca >= 2);
      const unsigned flags = lo | (hi << DIM) | (far << (2 * DIM));
      const uint64_t* tab = A.rank_tab + ((static_cast<size_t>(k) << (2 * DIM + 1)) + flags) * 2;
      const uint64_t own = __ldg(tab);
      double* rowp = hbuf + l * CAP + line_entries<DIM>(m, ax, x0 + l_pa[l], x0 + p, cc[1] + (ax == 1 ? side : 0), cc[2] + (ax == 2 ? side : 0));
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const unsigned r = static_cast<unsigned>(own >> (4 * q)) & 15u;
        if (r == 15u || q == k) continue;
        rowp[r] = h[q];
      }
      const unsigned rd = static_cast<unsigned>(own >> (4 * k)) & 15u;
      if (bb) {  // colour 1: the neighbour's parked row (its slot k ^ 1)
        const uint64_t nbr = __ldg(tab + 1);
        double nv[NC];
#pragma unroll
        for (int q = 0; q <= N; ++q) nv[q] = stage[q * nfaces + face];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          const unsigned r = static_cast<unsigned>(nbr >> (4 * q)) & 15u;
          if (r != 15u) rowp[r] = nv[q];
        }
        rowp[rd] = side ? h[k] + nv[k ^ 1] : nv[k ^ 1] + h[k];
        gbuf[l * (X + 1) + p] = side ? h[N] + nv[N] : nv[N] + h[N];
      } else if (side) {  // this cell is the face's minus cell
        rowp[rd] = h[k];
        gbuf[l * (X + 1) + p] = h[N];
      }
    }
  }
  __syncthreads();
  // pass 2: the plus cell adds its diagonal / g contribution to brick-interior faces
  if (valid) {
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
      const int k = 2 * ax;  // low face of the cell
      if (!(cc[ax] > 0) || lc[ax] == 0) continue;
      const int face = face_id32(m, ax, cc[0], cc[1], cc[2]);
      const int l = ax == 0 ? ly + Y * lz : (ax == 1 ? B::NL0 + ly + (Y + 1) * lz : B::NL0 + B::NL1 + ly + Y * lz);
      const int p = lx;
      const unsigned far = static_cast<unsigned>(cc[ax] >= 2);
      const unsigned flags = lo | (hi << DIM) | (far << (2 * DIM));
      const uint64_t own = __ldg(A.rank_tab + ((static_cast<size_t>(k) << (2 * DIM + 1)) + flags) * 2);
      const unsigned rd = static_cast<unsigned>(own >> (4 * k)) & 15u;
      double h[NC];
      hrow(k, h);
      double* dp = hbuf + l * CAP + line_entries<DIM>(m, ax, x0 + l_pa[l], x0 + p, cc[1], cc[2]) + rd;
      *dp = *dp + h[k];
      gbuf[l * (X + 1) + p] = gbuf[l * (X + 1) + p] + h[N];
    }
  }
  __syncthreads();
  // write-out: one warp per line segment, coalesced
  const int lane = tid & 31, warp = tid >> 5;
  const uint64_t pol = l2_policy_evict_first();
  for (int l = warp; l < NL; l += CT / 32) {
    const int lo_ = l_olo[l], hi_ = l_ohi[l];
    double* dst = A.hval + l_base[l];
    const double* src = hbuf + l * CAP;
    for (int i = lo_ + lane; i < hi_; i += 32) st_l2hint(dst + i, src[i], pol);
    const int pa = l_pa[l], oa = l_oa[l], ob = l_ob[l];
    for (int p = oa + lane; p <= ob; p += 32) A.g[l_row0[l] + (p - pa)] = gbuf[l * (X + 1) + p];
  }
  return rejected;
}

template <int DIM, int COL, int BX>
__global__ void __launch_bounds__(BrickDims<DIM, BX>::CT, BrickDims<DIM, BX>::MINB)
    k_rt0_brick(HybArgs A, Rt0Const<2 * DIM> c, Rt0Fast<2 * DIM> F, double* stage, int nbx, int nby, int nbz) {
  rt0_brick_body<DIM, COL, BX>(A, c, F, stage, nbx, nby, nbz);
}

// ------------------------------------------------------------------ k >= 1 recovery

constexpr int kNT = 256;  // threads per CTA


// x_hat_T = A_T^-1 (f_T - C_T^T lambda) by the same structured solve (one CTA per cell):
// the Neumann series of A0^-1 Delta in fp64 with the a-priori order; every
// matrix-vector product is done warp-per-row with the lanes striding along the
// row (coalesced loads of the fixed factors) and a shuffle reduction.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double quad_sum(double v) {  // over the 4 lanes of a row
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

__global__ void __launch_bounds__(kNT) k_recover_cta(RecArgs R, double* gws, int64_t ws_stride, int use_smem) {
  extern __shared__ double smem[];
  double* ws = use_smem ? smem : gws + blockIdx.x * ws_stride;
  const DevMesh& m = R.m;
  const int n = m.n, r = R.fx.r, dpf = m.dpf, nint = m.nint;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool wide = n > 64;       // long rows: warp per row; short rows: four lanes per row
  const int row4 = threadIdx.x >> 2, part = threadIdx.x & 3, rows4 = blockDim.x >> 2;
  double* s = ws;                 // r
  double* y = ws + 64;            // n: current rhs
  double* t = y + kMaxN;          // n: current term
  double* acc = t + kMaxN;        // n: sum
  double* xty = acc + kMaxN;      // r
  for (int64_t e = blockIdx.x; e < m.ncells; e += gridDim.x) {
    const double a = R.alpha[e], b = R.beta[e];
    const double ib = 1.0 / b;
    int64_t cc[3];
    cell_coords(m, e, cc);
    for (int j = threadIdx.x; j < r; j += blockDim.x) s[j] = b / fma(a, __ldg(R.fx.lam + j), b);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double v = R.f[e * n + i];
      if (i >= nint) {
        const int p = (i - nint) / dpf, sub = (i - nint) - p * dpf;
        bool in;
        const int64_t f = slot_face(m, cc, p, &in);
        if (in) v -= R.lambda[R.mbase[f] + sub];  // unit constraint rows: C_T^T lambda
      }
      y[i] = v;
    }
    __syncthreads();
    bool exact = false;
    const int P = struct_order_apriori(R.fx.rho * a * ib, R.p_max, exact);
    if (exact || R.force_exact) {  // rejected: x_hat of this cell from the exact path (kern_exact.cu)
      if (threadIdx.x == 0) exact_push(R.xlist, R.xcount, static_cast<int>(e));
      continue;
    }
    for (int p = 0; p <= P; ++p) {
      // t = A0^-1 y = (N0 y + X diag(s) X^T y) / beta
      if (wide) {  // warp per row, lanes along the row
        for (int j = warp; j < r; j += nw) {
          double u = 0.0;
          for (int l = lane; l < n; l += 32) u = fma(__ldg(R.fx.X + static_cast<int64_t>(l) * r + j), y[l], u);
          u = warp_sum(u);
          if (lane == 0) xty[j] = u * s[j];
        }
      } else {  // small elements: four lanes per row (launched with >= 4 n threads)
        for (int j0 = 0; j0 < r; j0 += rows4) {
          const int j = j0 + row4;
          double u = 0.0;
          if (j < r)
            for (int l = part; l < n; l += 4) u = fma(__ldg(R.fx.X + static_cast<int64_t>(l) * r + j), y[l], u);
          u = quad_sum(u);
          if (j < r && part == 0) xty[j] = u * s[j];
        }
      }
      __syncthreads();
      if (wide) {
        for (int i = warp; i < n; i += nw) {
          const double* row = R.fx.N0 + static_cast<int64_t>(i) * n;
          double u = 0.0;
          for (int l = lane; l < n; l += 32) u = fma(__ldg(row + l), y[l], u);
          for (int j = lane; j < r; j += 32) u = fma(__ldg(R.fx.X + static_cast<int64_t>(i) * r + j), xty[j], u);
          u = warp_sum(u);
          if (lane == 0) {
            u *= ib;
            t[i] = u;
            acc[i] = (p == 0) ? u : ((p & 1) ? acc[i] - u : acc[i] + u);
          }
        }
      } else {
        for (int i0 = 0; i0 < n; i0 += rows4) {
          const int i = i0 + row4;
          double u = 0.0;
          if (i < n) {
            for (int l = part; l < n; l += 4) u = fma(__ldg(R.fx.N0 + static_cast<int64_t>(i) * n + l), y[l], u);
            for (int j = part; j < r; j += 4) u = fma(__ldg(R.fx.X + static_cast<int64_t>(i) * r + j), xty[j], u);
          }
          u = quad_sum(u);
          if (i < n && part == 0) {
            u *= ib;
            t[i] = u;
            acc[i] = (p == 0) ? u : ((p & 1) ? acc[i] - u : acc[i] + u);
          }
        }
      }
      __syncthreads();
      if (p == P) break;
      // y = Delta t
      if (wide) {
        for (int i = warp; i < n; i += nw) {
          double u = 0.0;
          for (int l = lane; l < n; l += 32) {
            const int64_t o = static_cast<int64_t>(i) * n + l;
            u = fma(delta_entry(a, b, __ldg(R.fx.D + o), __ldg(R.fx.M + o), __ldg(R.fx.E + o), __ldg(R.fx.Ma + o)), t[l], u);
          }
          u = warp_sum(u);
          if (lane == 0) y[i] = u;
        }
      } else {
        for (int i0 = 0; i0 < n; i0 += rows4) {
          const int i = i0 + row4;
          double u = 0.0;
          if (i < n)
            for (int l = part; l < n; l += 4) {
              const int64_t o = static_cast<int64_t>(i) * n + l;
              u = fma(delta_entry(a, b, __ldg(R.fx.D + o), __ldg(R.fx.M + o), __ldg(R.fx.E + o), __ldg(R.fx.Ma + o)), t[l], u);
            }
          u = quad_sum(u);
          if (i < n && part == 0) y[i] = u;
        }
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) R.x_hat[e * n + i] = acc[i];
    __syncthreads();
  }
}

// Long rows (RT2 / RT3 hexahedra): CB cells per CTA.  The fixed factors (N0, X and the
// Delta inputs D, M, E, Ma: 1.8 MB for RT3, far beyond L1) are streamed from L2 once per
// CTA pass and applied to all CB cells (each cell its own alpha, beta, order), which
// divides the L2 traffic that bounds the one-cell form by CB.  Per cell the arithmetic
// and the summation order are those of k_recover_cta (warp per row, lanes along the row).
template <int CB>
__global__ void __launch_bounds__(kNT) k_recover_wide(RecArgs R) {
  extern __shared__ double smem[];
  constexpr int CELL = 64 + 3 * kMaxN + 64;  // s, y, t, acc, xty of one cell
  const DevMesh& m = R.m;
  const int n = m.n, r = R.fx.r, dpf = m.dpf, nint = m.nint;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double sa[CB], sb[CB], sib[CB];
  __shared__ int sP[CB];  // the cell's Neumann order, -1: no cell / sent to the exact path
  auto S = [&](int c) { return smem + c * CELL; };
  auto Y = [&](int c) { return smem + c * CELL + 64; };
  auto T = [&](int c) { return smem + c * CELL + 64 + kMaxN; };
  auto ACC = [&](int c) { return smem + c * CELL + 64 + 2 * kMaxN; };
  auto XTY = [&](int c) { return smem + c * CELL + 64 + 3 * kMaxN; };
  const int64_t ncb = (m.ncells + CB - 1) / CB;
  for (int64_t cb = blockIdx.x; cb < ncb; cb += gridDim.x) {
    if (threadIdx.x < CB) {
      const int c = threadIdx.x;
      const int64_t e = cb * CB + c;
      int P = -1;
      double a = 1.0, b = 1.0;
      if (e < m.ncells) {
        a = R.alpha[e], b = R.beta[e];
        bool exact = false;
        P = struct_order_apriori(R.fx.rho * a / b, R.p_max, exact);
        if (exact || R.force_exact) {  // x_hat of this cell from the exact path (kern_exact.cu)
          exact_push(R.xlist, R.xcount, static_cast<int>(e));
          P = -1;
        }
      }
      sa[c] = a, sb[c] = b, sib[c] = 1.0 / b, sP[c] = P;
    }
    __syncthreads();
    int Pm = -1;
#pragma unroll
    for (int c = 0; c < CB; ++c) Pm = max(Pm, sP[c]);
    if (Pm < 0) {
      __syncthreads();
      continue;
    }
    for (int c = 0; c < CB; ++c) {
      const int64_t e = cb * CB + c;
      const bool live = e < m.ncells;
      const double a = sa[c], b = sb[c];
      int64_t cc[3] = {0, 0, 0};
      if (live) cell_coords(m, e, cc);
      for (int j = threadIdx.x; j < r; j += blockDim.x) S(c)[j] = b / fma(a, __ldg(R.fx.lam + j), b);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double v = 0.0;
        if (live) {
          v = R.f[e * n + i];
          if (i >= nint) {
            const int p = (i - nint) / dpf, sub = (i - nint) - p * dpf;
            bool in;
            const int64_t f = slot_face(m, cc, p, &in);
            if (in) v -= R.lambda[R.mbase[f] + sub];  // unit constraint rows: C_T^T lambda
          }
        }
        Y(c)[i] = v;
      }
    }
    __syncthreads();
    for (int p = 0; p <= Pm; ++p) {
      // t = A0^-1 y = (N0 y + X diag(s) X^T y) / beta
      for (int j = warp; j < r; j += nw) {
        double u[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = 0.0;
        for (int l = lane; l < n; l += 32) {
          const double xv = __ldg(R.fx.X + static_cast<int64_t>(l) * r + j);
#pragma unroll
          for (int c = 0; c < CB; ++c) u[c] = fma(xv, Y(c)[l], u[c]);
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const double w = warp_sum(u[c]);
          if (lane == 0) XTY(c)[j] = w * S(c)[j];
        }
      }
      __syncthreads();
      for (int i = warp; i < n; i += nw) {
        const double* row = R.fx.N0 + static_cast<int64_t>(i) * n;
        double u[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = 0.0;
        for (int l = lane; l < n; l += 32) {
          const double nv = __ldg(row + l);
#pragma unroll
          for (int c = 0; c < CB; ++c) u[c] = fma(nv, Y(c)[l], u[c]);
        }
        for (int j = lane; j < r; j += 32) {
          const double xv = __ldg(R.fx.X + static_cast<int64_t>(i) * r + j);
#pragma unroll
          for (int c = 0; c < CB; ++c) u[c] = fma(xv, XTY(c)[j], u[c]);
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          double w = warp_sum(u[c]);
          if (lane == 0 && p <= sP[c]) {
            w *= sib[c];
            T(c)[i] = w;
            ACC(c)[i] = (p == 0) ? w : ((p & 1) ? ACC(c)[i] - w : ACC(c)[i] + w);
          }
        }
      }
      __syncthreads();
      if (p == Pm) break;
      // y = Delta t (Delta's inputs loaded once for the CB cells)
      double ca[CB], cbeta[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) ca[c] = sa[c], cbeta[c] = sb[c];
      for (int i = warp; i < n; i += nw) {
        double u[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) u[c] = 0.0;
        for (int l = lane; l < n; l += 32) {
          const int64_t o = static_cast<int64_t>(i) * n + l;
          const double d = __ldg(R.fx.D + o), mm = __ldg(R.fx.M + o), ee = __ldg(R.fx.E + o), ma = __ldg(R.fx.Ma + o);
#pragma unroll
          for (int c = 0; c < CB; ++c) u[c] = fma(delta_entry(ca[c], cbeta[c], d, mm, ee, ma), T(c)[l], u[c]);
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const double w = warp_sum(u[c]);
          if (lane == 0) Y(c)[i] = w;
        }
      }
      __syncthreads();
    }
    for (int c = 0; c < CB; ++c) {
      if (sP[c] < 0) continue;
      const int64_t e = cb * CB + c;
      for (int i = threadIdx.x; i < n; i += blockDim.x) R.x_hat[e * n + i] = ACC(c)[i];
    }
    __syncthreads();
  }
}

// k = 0 recovery, one thread per cell: x_hat = A_T^-1 r, r = f - C_T^T lambda,
// by the structured solve in fp64 (A0^-1 = (N0 + s X X^T) / beta, Neumann
// terms with the exact rounding errors Delta; order from the a-priori bound
// rho alpha / beta as the CTA form).  Constants in the kernel-parameter bank.
template <int DIM>
__global__ void __launch_bounds__(128) k_rt0_recover(RecArgs R, Rt0Const<2 * DIM> c) {
  constexpr int N = 2 * DIM;
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= R.m.ncells) return;
  const double a = R.alpha[e], b = R.beta[e];
  const double ib = 1.0 / b;
  const double s = b / fma(a, c.lam, b);
  int cc[3];
  cell_coords32(R.m, static_cast<uint32_t>(e), cc);
  double y[N], yl[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double v = R.f[e * N + k], vl = 0.0;
    const int a_ = k >> 1, side = k & 1;
    const int ca = a_ == 0 ? cc[0] : (a_ == 1 ? cc[1] : cc[2]);
    const int na = static_cast<int>(a_ == 0 ? R.m.N[0] : (a_ == 1 ? R.m.N[1] : R.m.N[2]));
    if (side ? (ca + 1 < na) : (ca > 0)) {  // unit constraint rows: C_T^T lambda
      const int face = face_id32(R.m, a_, cc[0] + (a_ == 0 ? side : 0), cc[1] + (a_ == 1 ? side : 0),
                                 cc[2] + (a_ == 2 ? side : 0));
      two_sum(v, -R.lambda[R.mbase[face]], v, vl);  // v = fl(f - lambda), vl its rounding error
    }
    y[k] = v;
    yl[k] = vl;
  }
  bool exact = false;
  const int P = struct_order_apriori(c.rho * a * ib, R.p_max, exact);
  if (exact || R.force_exact) {  // rejected: the exact solve in this thread
    if (R.xcount) atomicAdd(R.xcount, 1);
    double xo[N];
    rt0_exact_ool<N, 1, false>(R.fx.D, R.fx.M, a, b, rt0_bmask<DIM>(R.m, cc), y, yl, xo, R.status);
#pragma unroll
    for (int k = 0; k < N; ++k) R.x_hat[e * N + k] = xo[k];
    return;
  }
  double acc[N];
  for (int p = 0; p <= P; ++p) {
    // t = A0^-1 y
    double xty = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) xty = fma(c.X[l], y[l], xty);
    xty *= s;
    double t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double u = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) u = fma(c.N0[i * N + l], y[l], u);
      u = fma(c.X[i], xty, u);
      t[i] = u * ib;
      acc[i] = (p == 0) ? t[i] : ((p & 1) ? acc[i] - t[i] : acc[i] + t[i]);
    }
    if (p == P) break;
#pragma unroll
    for (int i = 0; i < N; ++i) {  // y = Delta t
      double u = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l)
        u = fma(delta_entry(a, b, c.D[i * N + l], c.M[i * N + l], c.E[i * N + l], c.Ma[i * N + l]), t[l], u);
      y[i] = u;
    }
  }
#pragma unroll
  for (int k = 0; k < N; ++k) R.x_hat[e * N + k] = acc[k];
}

// x = (P^T P)^-1 P^T x_hat: signed average of the face copies, bubbles copied
// (src/reduction.cpp:396-404; the Gram matrix of the FE P is diagonal)
__global__ void k_average(DevMesh m, const double* x_hat, double* x) {
  const int64_t gdof = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nd = m.face_dof_count + m.ncells * m.nint;
  if (gdof >= nd) return;
  if (gdof >= m.face_dof_count) {
    const int64_t b = gdof - m.face_dof_count;
    const int64_t cell = b / m.nint, l = b - cell * m.nint;
    x[gdof] = x_hat[cell * m.n + l];
    return;
  }
  const int64_t f = gdof / m.dpf, sub = gdof - f * m.dpf;
  int64_t cm, cp, co[3];
  const int a = face_cells(m, f, &cm, &cp, co);
  double sum = 0.0, cnt = 0.0;
  if (cm >= 0) {  // +a face of cm: slot 2a+1, sign +1
    sum += x_hat[cm * m.n + m.nint + (2 * a + 1) * m.dpf + sub];
    cnt += 1.0;
  }
  if (cp >= 0) {  // -a face of cp: slot 2a, sign -1
    sum += -1.0 * x_hat[cp * m.n + m.nint + (2 * a) * m.dpf + sub];
    cnt += 1.0;
  }
  x[gdof] = sum * (1.0 / cnt);
}

}  // namespace

// Rt0Fast from the constant block; false when the structure it relies on is absent
// (M^-1 not block-diagonal per axis, or D / M / E / Ma not bitwise symmetric).
// Constant block: D, M, E, Ma, N0 (n*n each), X (n), lambda, rho, M^-1 (n*n).
template <int N>
static bool rt0_fast_setup(const double* hc, Rt0Fast<N>& F) {
  const double *D = hc, *M = hc + N * N, *E = hc + 2 * N * N, *Ma = hc + 3 * N * N, *X = hc + 5 * N * N;
  const double* N0 = hc + 5 * N * N + N + 2;  // M^-1 (named N0 below: the block-diagonal factor of W)
  for (int k = 0; k < N; ++k)
    for (int l = 0; l < N; ++l) {
      for (const double* m : {D, M, E, Ma, N0})
        if (m[k * N + l] != m[l * N + k]) return false;
      if ((k >> 1) != (l >> 1) && (N0[k * N + l] != 0.0 || M[k * N + l] != 0.0 || Ma[k * N + l] != 0.0)) return false;
    }
  // W(t) = M^-1 + t XX^T (t = s - 1, W = N0 + s XX^T);
  // W E W = Mi E Mi + t (Mi E XX^T + XX^T E Mi) + t^2 XX^T E XX^T
  auto poly = [&](const double* Em, float (*out)[Rt0Fast<N>::NS]) {
    std::vector<double> NE(N * N, 0.0), NEN(N * N, 0.0), EX(N, 0.0), NEX(N, 0.0);
    double xex = 0.0;
    for (int k = 0; k < N; ++k)
      for (int l = 0; l < N; ++l) {
        for (int j = 0; j < N; ++j) NE[k * N + l] += N0[k * N + j] * Em[j * N + l];
        EX[k] += Em[k * N + l] * X[l];
      }
    for (int k = 0; k < N; ++k) {
      for (int l = 0; l < N; ++l)
        for (int j = 0; j < N; ++j) NEN[k * N + l] += NE[k * N + j] * N0[j * N + l];
      for (int j = 0; j < N; ++j) NEX[k] += N0[k * N + j] * EX[j];
      xex += X[k] * EX[k];
    }
    for (int k = 0; k < N; ++k)
      for (int l = k; l < N; ++l) {
        const int i = sym_idx(k, l, N);
        out[0][i] = static_cast<float>(NEN[k * N + l]);
        out[1][i] = static_cast<float>(NEX[k] * X[l] + X[k] * NEX[l]);
        out[2][i] = static_cast<float>(xex * X[k] * X[l]);
      }
  };
  for (int k = 0; k < N; ++k) {
    F.n0[k][0] = static_cast<float>(N0[k * N + (k & ~1)]);
    F.n0[k][1] = static_cast<float>(N0[k * N + (k | 1)]);
    F.x[k] = static_cast<float>(X[k]);
  }
  poly(E, F.p);
  poly(Ma, F.q);
  return true;
}

void launch_hybridize_rt0_rows(const HybArgs& a, const double* hc, double* stage, cudaStream_t st) {
  const int64_t cnt = parity_count(a.m);
  auto fill = [&](auto& c, int N) {
    memcpy(c.D, hc, sizeof(double) * N * N);
    memcpy(c.M, hc + N * N, sizeof(double) * N * N);
    memcpy(c.E, hc + 2 * N * N, sizeof(double) * N * N);
    memcpy(c.Ma, hc + 3 * N * N, sizeof(double) * N * N);
    memcpy(c.N0, hc + 4 * N * N, sizeof(double) * N * N);
    memcpy(c.X, hc + 5 * N * N, sizeof(double) * N);
    c.lam = hc[5 * N * N + N];
    c.rho = hc[5 * N * N + N + 1];
  };
  // one-pass pencil kernel (kern_pencil.cu) when the element has its structure;
  // the older variants stay selectable (HDR_RT0_ROWS / _CELL / _BRICK, A/B timing)
  const bool forced = getenv("HDR_RT0_ROWS") || getenv("HDR_RT0_CELL") || getenv("HDR_RT0_BRICK") || getenv("HDR_RT0_NO_PENCIL");
  if (!forced) {
    PencilConst<3> p3;
    PencilConst<2> p2;
    const bool ok = a.m.dim == 3 ? pencil_setup<3>(hc, p3) : pencil_setup<2>(hc, p2);
    if (ok) {
      if (a.m.dim == 3) launch_rt0_pencil<3>(a, p3, st);
      else launch_rt0_pencil<2>(a, p2, st);
      // (rejected cells are solved in place by the exact path: no tail launch)
      return;
    }
  }
  // lane-per-row variant: A/B timing, or when the element lacks the structure of Rt0Fast
  bool rows = getenv("HDR_RT0_ROWS") != nullptr;
  Rt0Fast<6> f3{};
  Rt0Fast<4> f2{};
  if (!(a.m.dim == 3 ? rt0_fast_setup<6>(hc, f3) : rt0_fast_setup<4>(hc, f2))) rows = true;
  // thread-per-cell scattered-store variant: forced, or for meshes too small to
  // give each SM a few bricks per colour (e.g. 64 x 64 quads: 16 bricks a colour)
  // (HDR_RT0_BRICK forces the brick kernel at any size: tests)
  const bool cell = getenv("HDR_RT0_CELL") != nullptr || (a.m.ncells < 148 * 128 * 4 && !getenv("HDR_RT0_BRICK"));
  auto brick = [&](auto dimc, auto bxc, auto& c, auto& F) {
    constexpr int D = decltype(dimc)::value, BXv = decltype(bxc)::value;
    using B = BrickDims<D, BXv>;
    const int nbx = static_cast<int>((a.m.N[0] + B::X - 1) / B::X), nby = static_cast<int>((a.m.N[1] + B::Y - 1) / B::Y);
    const int nbz = D == 3 ? static_cast<int>((a.m.N[2] + B::Z - 1) / B::Z) : 1;
    const dim3 grid(static_cast<unsigned>((nbx + 1) / 2), static_cast<unsigned>(nby), static_cast<unsigned>(nbz));
    const size_t smem = B::smem_bytes();
    cudaFuncSetAttribute(k_rt0_brick<D, 0, BXv>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(k_rt0_brick<D, 1, BXv>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_rt0_brick<D, 0, BXv><<<grid, B::CT, smem, st>>>(a, c, F, stage, nbx, nby, nbz);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(B::CT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = getenv("HDR_NO_PDL") ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_rt0_brick<D, 1, BXv>, a, c, F, stage, nbx, nby, nbz);
    // the exact path of rejected cells (usually none: the kernel returns at once)
    cudaLaunchConfig_t xc{};
    xc.gridDim = dim3(1);
    xc.blockDim = dim3(256);
    xc.stream = st;
    xc.attrs = attr;
    xc.numAttrs = 1;
    cudaLaunchKernelEx(&xc, k_rt0_exact<D>, a);
    count_launch();
  };
  const bool wide = a.m.N[0] >= 48 && !getenv("HDR_RT0_BRICK32");
  if (a.m.dim == 3) {
    Rt0Const<6> c;
    fill(c, 6);
    if (!rows && !cell) {
      if (wide) brick(std::integral_constant<int, 3>{}, std::integral_constant<int, HDR_BRICK_XW>{}, c, f3);
      else brick(std::integral_constant<int, 3>{}, std::integral_constant<int, 32>{}, c, f3);
    } else if (rows) {
      const unsigned nb = static_cast<unsigned>((cnt + 4 * 5 - 1) / (4 * 5));
      k_rt0_rows<3, 0><<<nb, 128, 0, st>>>(a, c, stage);
      k_rt0_rows<3, 1><<<nb, 128, 0, st>>>(a, c, stage);
    } else {
      const unsigned nb = static_cast<unsigned>((cnt + kCT - 1) / kCT);
      k_rt0_cell<3, 0, true><<<nb, kCT, 0, st>>>(a, c, f3, stage);
      k_rt0_cell<3, 1, true><<<nb, kCT, 0, st>>>(a, c, f3, stage);
    }
  } else {
    Rt0Const<4> c;
    fill(c, 4);
    if (!rows && !cell) {
      if (wide) brick(std::integral_constant<int, 2>{}, std::integral_constant<int, 64>{}, c, f2);
      else brick(std::integral_constant<int, 2>{}, std::integral_constant<int, 32>{}, c, f2);
    } else if (rows) {
      const unsigned nb = static_cast<unsigned>((cnt + 4 * 8 - 1) / (4 * 8));
      k_rt0_rows<2, 0><<<nb, 128, 0, st>>>(a, c, stage);
      k_rt0_rows<2, 1><<<nb, 128, 0, st>>>(a, c, stage);
    } else {
      const unsigned nb = static_cast<unsigned>((cnt + kCT - 1) / kCT);
      k_rt0_cell<2, 0, true><<<nb, kCT, 0, st>>>(a, c, f2, stage);
      k_rt0_cell<2, 1, true><<<nb, kCT, 0, st>>>(a, c, f2, stage);
    }
  }
  count_launch(2);
}

void launch_recover_rt0(const RecArgs& a, const double* hc, cudaStream_t st) {
  auto fill = [&](auto& c, int N) {
    memcpy(c.D, hc, sizeof(double) * N * N);
    memcpy(c.M, hc + N * N, sizeof(double) * N * N);
    memcpy(c.E, hc + 2 * N * N, sizeof(double) * N * N);
    memcpy(c.Ma, hc + 3 * N * N, sizeof(double) * N * N);
    memcpy(c.N0, hc + 4 * N * N, sizeof(double) * N * N);
    memcpy(c.X, hc + 5 * N * N, sizeof(double) * N);
    c.lam = hc[5 * N * N + N];
    c.rho = hc[5 * N * N + N + 1];
  };
  const unsigned nb = static_cast<unsigned>((a.m.ncells + 127) / 128);
  if (a.m.dim == 3) {
    Rt0Const<6> c;
    fill(c, 6);
    k_rt0_recover<3><<<nb, 128, 0, st>>>(a, c);
  } else {
    Rt0Const<4> c;
    fill(c, 4);
    k_rt0_recover<2><<<nb, 128, 0, st>>>(a, c);
  }
  count_launch();
}

void launch_recover_hybrid(const RecArgs& a, double* gws, int64_t ws_doubles, cudaStream_t st) {
  (void)gws;
  (void)ws_doubles;
  const size_t smem = static_cast<size_t>(64 + 3 * kMaxN + 64) * 8;
  const int64_t grid = std::min<int64_t>(a.m.ncells, 1 << 20);
  // long rows: 128 threads (warp per row); short rows: four lanes per row, two thirds of the
  // rows per pass (measured on 48^3 RT1, n = 36: 32 / 64 / 96 / 128 / 160 threads ->
  // 1.22 / 0.92 / 0.89 / 1.00 / 0.99 ms)
  if (a.m.n > 64 && !getenv("HDR_REC_ONE_CELL")) {  // long rows: CB cells per CTA share each pass over the factors
    auto go = [&](auto cbc) {
      constexpr int CB = decltype(cbc)::value;
      const size_t smem_w = static_cast<size_t>(CB) * (64 + 3 * kMaxN + 64) * 8;
      cudaFuncSetAttribute(k_recover_wide<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_w));
      const int64_t ncb = (a.m.ncells + CB - 1) / CB;
      k_recover_wide<CB><<<static_cast<unsigned>(std::min<int64_t>(ncb, 148 * 8)), kNT, smem_w, st>>>(a);
    };
    // measured on 32^3 RT3 (cfg5): one cell per CTA 22.7 ms, four 12.8 ms, eight 11.2 ms
    if (getenv("HDR_REC_CB4")) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 8>{});
    count_launch();
    return;
  }
  int threads = a.m.n > 64 ? 128 : std::min(256, ((8 * a.m.n / 3 + 31) / 32) * 32);
  if (const char* ev = getenv("HDR_REC_THREADS")) threads = atoi(ev);  // A/B timing
  k_recover_cta<<<static_cast<unsigned>(grid), threads, smem, st>>>(a, nullptr, 0, 1);
  count_launch();
}

void launch_average_faces(const DevMesh& m, const double* x_hat, double* x, cudaStream_t st) {
  const int64_t nd = m.face_dof_count + m.ncells * m.nint;
  k_average<<<static_cast<unsigned>((nd + 255) / 256), 256, 0, st>>>(m, x_hat, x);
  count_launch();
}

}  // namespace hdr
