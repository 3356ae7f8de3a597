// Exact double-double path of one k = 0 cell in one thread, shared by the k = 0
// kernels of kern_hybridize.cu and the pencil kernel (kern_pencil.cu).
#pragma once
#include "hdr_device.cuh"

namespace hdr {
namespace {

// Exact path of one cell in one thread (k = 0 kernels; the structured
// estimate rejected the cell, hdr_device.cuh struct_order): double-double
// Gaussian elimination on the reference's A_T = fl(fl(alpha D) + fl(beta M)) in
// its [i | b] partition (bmask bit l: local dof l is an interior-face (b) dof),
// pivoting restricted to the i rows for the first n_i steps so that the
// reference's SingularBlock rule sees the pivots of A_ii and of S_b
// (src/reduction.cpp:279-302, src/dense.cpp:61-97; kern_exact.cu does the same
// for k >= 1), applied to [I | r] (IDENT, NC = N + 1: rows of A_T^-1 and
// A_T^-1 f, i.e. [H_T | g_T] rows) or to r alone (NC = 1: the recovery
// x_hat = A_T^-1 (f - C^T lambda), r given as (rh, rl)).  out: N x NC row-major
// in the local dof order, rounded once.  Local-memory arrays: only the rare
// rejected cells run this.
template <int N, int NC, bool IDENT>
__device__ __forceinline__ void rt0_exact(const double* D, const double* M, double a, double b, unsigned bmask,
                                          const double* rh, const double* rl, double* out, int* status) {
  ddr A[N][N], B[N][NC];
  int perm[N];  // partitioned position -> local dof
  int ni = 0;
  for (int l = 0; l < N; ++l)
    if (!((bmask >> l) & 1u)) perm[ni++] = l;
  for (int l = 0, q = ni; l < N; ++l)
    if ((bmask >> l) & 1u) perm[q++] = l;
  double amax = 0.0;
  for (int i = 0; i < N; ++i) {
    const int li = perm[i];
    for (int j = 0; j < N; ++j) {
      const int lj = perm[j];
      A[i][j] = dd_from(assemble_entry(a, b, D[li * N + lj], M[li * N + lj]));
      if (i < ni && j < ni) amax = fmax(amax, fabs(A[i][j].hi));
    }
    for (int c = 0; c < NC; ++c) {
      if (IDENT) B[i][c] = c < N ? dd_from(li == c ? 1.0 : 0.0) : dd_from(rh[li]);
      else B[i][c] = {rh[li], rl ? rl[li] : 0.0};
    }
  }
  for (int k = 0; k < N; ++k) {
    if (k == ni) {  // max |S_b| of the trailing block
      amax = 0.0;
      for (int i = ni; i < N; ++i)
        for (int j = ni; j < N; ++j) amax = fmax(amax, fabs(A[i][j].hi));
    }
    const int kend = k < ni ? ni : N;
    int p = k;
    for (int i = k + 1; i < kend; ++i)
      if (fabs(A[i][k].hi) > fabs(A[p][k].hi)) p = i;
    if (p != k) {
      for (int j = 0; j < N; ++j) {
        const ddr t = A[k][j];
        A[k][j] = A[p][j];
        A[p][j] = t;
      }
      for (int c = 0; c < NC; ++c) {
        const ddr t = B[k][c];
        B[k][c] = B[p][c];
        B[p][c] = t;
      }
    }
    if (!(fabs(A[k][k].hi) > 1e-14 * amax)) {
      atomicOr(status, 4);
      return;
    }
    for (int i = k + 1; i < N; ++i) {
      const ddr l = dd_div(A[i][k], A[k][k]);
      for (int j = k + 1; j < N; ++j) A[i][j] = dd_fms(A[i][j], l, A[k][j]);
      for (int c = 0; c < NC; ++c) B[i][c] = dd_fms(B[i][c], l, B[k][c]);
    }
  }
  for (int k = N - 1; k >= 0; --k) {
    for (int c = 0; c < NC; ++c) {
      ddr v = B[k][c];
      for (int j = k + 1; j < N; ++j) v = dd_fms(v, A[k][j], B[j][c]);
      B[k][c] = dd_div(v, A[k][k]);
    }
  }
  for (int i = 0; i < N; ++i)
    for (int c = 0; c < NC; ++c) out[perm[i] * NC + c] = B[i][c].hi;
}

// interior-face mask of a k = 0 cell (bit s: slot s's face is interior = a b dof)
template <int DIM>
__device__ __forceinline__ unsigned rt0_bmask(const DevMesh& m, const int (&cc)[3]) {
  unsigned mask = 0;
#pragma unroll
  for (int s = 0; s < 2 * DIM; ++s) {
    const int ax = s >> 1, side = s & 1;
    const int ca = ax == 0 ? cc[0] : (ax == 1 ? cc[1] : cc[2]);
    const int na = static_cast<int>(ax == 0 ? m.N[0] : (ax == 1 ? m.N[1] : m.N[2]));
    mask |= static_cast<unsigned>(side ? (ca + 1 < na) : (ca > 0)) << s;
  }
  return mask;
}

}  // namespace
}  // namespace hdr
