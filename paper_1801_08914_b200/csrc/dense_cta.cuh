// One-CTA dense kernels in the reference's serial operation order (src/dense.cpp):
// every matrix entry sees the same operations in the same order as the serial
// code; rows / columns / right-hand sides are the parallel axes.  Explicit _rn
// intrinsics keep nvcc from contracting into FMAs (the reference's Release
// build has none).  Shared by kern_nullspace.cu and
// kern_amg.cu (the coarsest-level LU).
#pragma once

#include <cuda_runtime.h>

namespace hdr {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// block max of a non-negative value (exact: max does not round)
__device__ inline double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < nw; ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

// lu_factor (dense.cpp:61-97) in place on a (n x n, row-major); piv[n].
// Returns false (SingularBlock) when a pivot is at or below 1e-14 max|a|.
__device__ inline bool cta_lu_factor(double* a, int n, int* piv, double* red, int* ired) {
  double mx = 0.0;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) mx = fmax(mx, fabs(a[i]));
  const double threshold = mul(1e-14, block_max(mx, red));
  for (int k = 0; k < n; ++k) {
    // pivot: the first row of the largest |lu(i, k)|, i >= k
    if (threadIdx.x == 0) {
      int p = k;
      double pm = fabs(a[k * n + k]);
      for (int i = k + 1; i < n; ++i) {
        const double v = fabs(a[i * n + k]);
        if (v > pm) {
          pm = v;
          p = i;
        }
      }
      ired[0] = p;
      red[0] = pm;
    }
    __syncthreads();
    const int p = ired[0];
    const double pm = red[0];
    __syncthreads();
    if (!(pm > threshold) || pm == 0.0) return false;
    if (threadIdx.x == 0) piv[k] = p;
    if (p != k)
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double t = a[k * n + j];
        a[k * n + j] = a[p * n + j];
        a[p * n + j] = t;
      }
    __syncthreads();
    const double inv_piv = 1.0 / a[k * n + k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) a[i * n + k] = mul(a[i * n + k], inv_piv);
    __syncthreads();
    const int w = n - k - 1;
    for (int t = threadIdx.x; t < w * w; t += blockDim.x) {
      const int i = k + 1 + t / w, j = k + 1 + t % w;
      const double l = a[i * n + k];
      if (l != 0.0) a[i * n + j] = sub(a[i * n + j], mul(l, a[k * n + j]));
    }
    __syncthreads();
  }
  return true;
}

// lu_solve_matrix (dense.cpp:99-120, 165-175): x (n x c, row-major) = A^-1 b;
// one right-hand side per thread, each in the reference's serial order.
// b == nullptr: the identity (lu_inverse).  x may not alias b.
__device__ inline void cta_lu_solve_matrix(const double* lu, const int* piv, int n, const double* b, int c, double* x) {
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    for (int i = 0; i < n; ++i) x[i * c + j] = b ? b[i * c + j] : (i == j ? 1.0 : 0.0);
    for (int k = 0; k < n; ++k) {
      const int p = piv[k];
      if (p != k) {
        const double t = x[k * c + j];
        x[k * c + j] = x[p * c + j];
        x[p * c + j] = t;
      }
    }
    for (int k = 0; k < n; ++k) {
      const double xk = x[k * c + j];
      if (xk == 0.0) continue;
      for (int i = k + 1; i < n; ++i) x[i * c + j] = sub(x[i * c + j], mul(lu[i * n + k], xk));
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i * c + j];
      for (int q = i + 1; q < n; ++q) s = sub(s, mul(lu[i * n + q], x[q * c + j]));
      x[i * c + j] = s / lu[i * n + i];
    }
  }
  __syncthreads();
}

}  // namespace hdr
