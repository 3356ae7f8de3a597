// Element elimination for symmetric positive definite FE blocks (mapped cells,
// config 4; weighted affine cells): the hybridize drop-in of
//   hybridize(const ReductionInputs&)   src/reduction.cpp:262-354
// for element blocks that are SPD (every A_T = alpha D_T + beta M_T is).
//
// One 384-thread CTA per element (persistent), everything in shared memory:
//   W   n x n, column-major (ld odd): the block in the [i | b] order, factored in
//       place as A = L D L^T (unscaled columns, one barrier per step; pivots are
//       checked with the reference's SingularBlock rule, dense.cpp:61-97: the
//       first ni pivots against 1e-14 max|A_ii|, the rest against 1e-14 max|S_b|)
//   Z   n x nc: Z = A^-1 [C_T^T | f_T]
//   R   n x nc: residuals / corrections
// The fp64 factorization is only a preconditioner: A_T is ill conditioned
// (alpha / beta up to 1e6, h^-2), so Z is refined with residuals B - A Z whose
// products are exact (two_prod) and whose sums are compensated (two_sum), until
// the correction times its observed contraction rate is below 2^-55 of |Z|.
// This gives the element-exact H_e = C_b Z, g_e like the reference's own
// double-double oracle (src/reference.cpp:137-235), at about a quarter of the
// work of kern_alg.cu's general LU + double-double solution.
#include <algorithm>

#include "hdr_device.cuh"
#include "kernels.hpp"

namespace hdr {

namespace {

constexpr int kST = 384;
constexpr int kSW = kST / 32;

struct SpdSmem {
  double* W;
  double* Z;
  double* R;
  double* dinv;
  double* red;
  int* sidx;
  int* flag;
  int ld, ldz;
};

// L (unit lower, scaled in place; the diagonal of W keeps the pivots d) ->
// L^-1 in place, by blocks of 8 columns from the right:
//   Ib = L_bb^-1;  T = L[rest, b] Ib;  Linv[rest, b] = -Linv[rest, rest] T.
// T: scratch of >= 8 (n - 8) doubles; Ib: 64 doubles.
__device__ void tri_invert(int n, double* W, int ld, double* T, double* Ib) {
  const int tid = threadIdx.x;
  for (int jb = ((n - 1) / 8) * 8; jb >= 0; jb -= 8) {
    const int je = min(jb + 8, n), w = je - jb, rest = n - je;
    if (tid < w) {  // column tid of L_bb^-1 (unit lower), forward substitution
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double v = (i == tid) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k)
          if (i > tid && k >= tid && i < w) v = fma(-W[(jb + k) * ld + jb + i], x[k], v);
        x[i] = v;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) Ib[i * 8 + tid] = x[i];
    }
    __syncthreads();
    for (int t = tid; t < rest * 8; t += kST) {  // T = L[rest, b] Ib  (w == 8 whenever rest > 0)
      const int i = je + (t >> 3), c = t & 7;
      double acc = W[(jb + c) * ld + i];
      for (int k = c + 1; k < 8; ++k) acc = fma(W[(jb + k) * ld + i], Ib[k * 8 + c], acc);
      T[t] = acc;
    }
    __syncthreads();
    for (int t = tid; t < rest * 8; t += kST) {  // Linv[rest, b] = -Linv[rest, rest] T
      const int ii = t >> 3, c = t & 7, i = je + ii;
      double acc = T[t];
      for (int kk = 0; kk < ii; ++kk) acc = fma(W[(je + kk) * ld + i], T[kk * 8 + c], acc);
      W[(jb + c) * ld + i] = -acc;
    }
    for (int t = tid; t < w * w; t += kST) {
      const int i = t / w, c = t - (t / w) * w;
      if (i > c) W[(jb + c) * ld + jb + i] = Ib[i * 8 + c];
    }
    __syncthreads();
  }
}

// Register tiles of TM rows x TN columns over n x nc outputs.  The triangular
// products are load-balanced by giving each thread the row-tile pair (t, last - t)
// (n = 108, nc = 55 -> 378 pairs).
constexpr int TM = 2, TN = 4;

// acc = Linv[r0:r0+TM, :] Y[:, c0:c0+TN]  (Linv unit lower in W)
__device__ __forceinline__ void lower_tile(int n, const double* W, int ld, const double* Y, int ldy, int r0, int c0,
                                           double (&acc)[TM][TN]) {
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;
#pragma unroll 4
  for (int k = 0; k < r0; ++k) {
    const double2 yv0 = *reinterpret_cast<const double2*>(Y + k * ldy + c0);
    const double2 yv1 = *reinterpret_cast<const double2*>(Y + k * ldy + c0 + 2);
    const double yv[TN] = {yv0.x, yv0.y, yv1.x, yv1.y};
    double lv[TM];
#pragma unroll
    for (int a = 0; a < TM; ++a) lv[a] = W[k * ld + r0 + a];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) acc[a][b] = fma(lv[a], yv[b], acc[a][b]);
  }
#pragma unroll
  for (int kk = 0; kk < TM; ++kk) {
    const int k = r0 + kk;
    if (k >= n) break;
    double yv[TN];
#pragma unroll
    for (int b = 0; b < TN; ++b) yv[b] = Y[k * ldy + c0 + b];
#pragma unroll
    for (int a = kk; a < TM; ++a) {
      const double l = (a == kk) ? 1.0 : W[k * ld + r0 + a];
#pragma unroll
      for (int b = 0; b < TN; ++b) acc[a][b] = fma(l, yv[b], acc[a][b]);
    }
  }
}

// acc = Linv^T[r0:r0+TM, :] Y[:, c0:c0+TN]
__device__ __forceinline__ void upper_tile(int n, const double* W, int ld, const double* Y, int ldy, int r0, int c0,
                                           double (&acc)[TM][TN]) {
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;
#pragma unroll
  for (int kk = 0; kk < TM; ++kk) {
    const int k = r0 + kk;
    if (k >= n) break;
    double yv[TN];
#pragma unroll
    for (int b = 0; b < TN; ++b) yv[b] = Y[k * ldy + c0 + b];
#pragma unroll
    for (int a = 0; a <= kk; ++a) {
      const double l = (a == kk) ? 1.0 : W[(r0 + a) * ld + k];
#pragma unroll
      for (int b = 0; b < TN; ++b) acc[a][b] = fma(l, yv[b], acc[a][b]);
    }
  }
#pragma unroll 4
  for (int k = r0 + TM; k < n; ++k) {
    const double2 yv0 = *reinterpret_cast<const double2*>(Y + k * ldy + c0);
    const double2 yv1 = *reinterpret_cast<const double2*>(Y + k * ldy + c0 + 2);
    const double yv[TN] = {yv0.x, yv0.y, yv1.x, yv1.y};
    double lv[TM];
#pragma unroll
    for (int a = 0; a < TM; ++a) lv[a] = W[(r0 + a) * ld + k];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) acc[a][b] = fma(lv[a], yv[b], acc[a][b]);
  }
}

// the (up to) two row tiles and the column tile of work unit u
struct PairTiles {
  int r0a, r0b, c0;  // r0b < 0: single tile
  bool ok;
};
__device__ __forceinline__ PairTiles pair_tiles(int u, int n, int nc) {
  const int tn = (nc + TN - 1) / TN, nrt = (n + TM - 1) / TM, npair = (nrt + 1) / 2;
  PairTiles p;
  p.ok = u < npair * tn;
  const int pr = u / tn;
  p.c0 = (u - pr * tn) * TN;
  p.r0a = pr * TM;
  p.r0b = (nrt - 1 - pr) != pr ? (nrt - 1 - pr) * TM : -1;
  return p;
}

template <class F>
__device__ __forceinline__ void store_tile(int n, int nc, int r0, int c0, const double (&acc)[TM][TN], F f) {
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b)
      if (r0 + a < n && c0 + b < nc) f(r0 + a, c0 + b, acc[a][b]);
}

// Y <- D^-1 Linv Y in place (two-phase: products to registers, barrier, store)
__device__ void lower_inplace(int n, int nc, const double* W, int ld, const double* dinv, double* Y, int ldy) {
  const PairTiles p = pair_tiles(threadIdx.x, n, nc);
  double acc0[TM][TN], acc1[TM][TN];
  if (p.ok) {
    lower_tile(n, W, ld, Y, ldy, p.r0a, p.c0, acc0);
    if (p.r0b >= 0) lower_tile(n, W, ld, Y, ldy, p.r0b, p.c0, acc1);
  }
  __syncthreads();
  if (p.ok) {
    auto st = [&](int i, int c, double v) { Y[i * ldy + c] = v * dinv[i]; };
    store_tile(n, nc, p.r0a, p.c0, acc0, st);
    if (p.r0b >= 0) store_tile(n, nc, p.r0b, p.c0, acc1, st);
  }
  __syncthreads();
}

// block max of two values at once
__device__ void blk_max2(double& v0, double& v1, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 = fmax(v0, __shfl_xor_sync(0xffffffffu, v0, o));
    v1 = fmax(v1, __shfl_xor_sync(0xffffffffu, v1, o));
  }
  __syncthreads();
  if (lane == 0) {
    red[warp] = v0;
    red[kSW + warp] = v1;
  }
  __syncthreads();
  v0 = red[0];
  v1 = red[kSW];
#pragma unroll
  for (int w = 1; w < kSW; ++w) {
    v0 = fmax(v0, red[w]);
    v1 = fmax(v1, red[kSW + w]);
  }
}

// R = B - A Z with exact products and compensated sums (rounded once).
// Thread tiles of TM rows x TN columns; A read through the [i | b] permutation.
__device__ void residual(int n, int nc, const double* A, const SpdSmem& s, const double* Bg) {
  constexpr int TM = 4, TN = 4;
  const int tn = (nc + TN - 1) / TN, tm = (n + TM - 1) / TM;
  for (int tile = threadIdx.x; tile < tm * tn; tile += kST) {
    const int r0 = (tile / tn) * TM, c0 = (tile % tn) * TN;
    double hi[TM][TN], lo[TM][TN];
    const double* arow[TM];
#pragma unroll
    for (int a = 0; a < TM; ++a) {
      const int r = min(r0 + a, n - 1);
      arow[a] = A + static_cast<int64_t>(s.sidx[r]) * n;
#pragma unroll
      for (int b = 0; b < TN; ++b) {
        hi[a][b] = (r0 + a < n && c0 + b < nc) ? Bg[(r0 + a) * s.ldz + c0 + b] : 0.0;
        lo[a][b] = 0.0;
      }
    }
#pragma unroll 2
    for (int j = 0; j < n; ++j) {
      const int cj = s.sidx[j];
      double av[TM], zv[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) av[a] = -__ldg(arow[a] + cj);
#pragma unroll
      for (int b = 0; b < TN; ++b) zv[b] = s.Z[j * s.ldz + c0 + b];  // padded columns hold 0
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) {
          double p, e, sm, t;
          two_prod(av[a], zv[b], p, e);
          two_sum(hi[a][b], p, sm, t);
          hi[a][b] = sm;
          lo[a][b] = lo[a][b] + (t + e);
        }
    }
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b)
        if (r0 + a < n && c0 + b < nc) s.R[(r0 + a) * s.ldz + c0 + b] = hi[a][b] + lo[a][b];
  }
}

__global__ void __launch_bounds__(kST, 1) k_spd_hyb(AlgArgs a, double* gws, int64_t slot, int nmax, int ncmax) {
  extern __shared__ __align__(16) double smem[];
  SpdSmem s;
  s.ld = nmax | 1;
  s.ldz = (ncmax + 1) & ~1;
  s.W = smem;
  s.Z = s.W + ((nmax * s.ld + 1) & ~1);
  s.R = s.Z + nmax * s.ldz;
  s.dinv = s.R + max(nmax * s.ldz, 8 * nmax + 64);
  s.red = s.dinv + nmax;
  s.sidx = reinterpret_cast<int*>(s.red + 2 * kSW);
  s.flag = s.sidx + nmax;
  double* Bg = gws + static_cast<int64_t>(blockIdx.x) * slot;  // n x ldz right-hand sides
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t e = blockIdx.x; e < a.ne; e += gridDim.x) {
    const int64_t boff = a.boff[e];
    const int n = static_cast<int>(a.boff[e + 1] - boff), ni = a.ni[e];
    const int64_t g0 = a.goff[e];
    const int nr = static_cast<int>(a.goff[e + 1] - g0), nc = nr + 1;
    const double* A = a.blocks + a.aoff[e];
    for (int i = tid; i < n; i += kST) s.sidx[i] = a.idx[boff + i];
    __syncthreads();
    // permuted block, column-major; max |A_ii|
    double mx = 0.0;
    for (int t = tid; t < n * n; t += kST) {
      const int i = t / n, k = t - i * n;  // consecutive threads: consecutive columns of row i
      const double v = __ldg(A + static_cast<int64_t>(s.sidx[i]) * n + s.sidx[k]);
      s.W[k * s.ld + i] = v;
      if (ni == 0 || (i < ni && k < ni)) mx = fmax(mx, fabs(v));
    }
    // right-hand sides [C_T^T | f_T] (global slot, row-major n x ldz, padding 0)
    for (int t = tid; t < n * s.ldz; t += kST) {
      const int i = t / s.ldz, c = t - i * s.ldz;
      Bg[t] = c == nr ? a.f[boff + s.sidx[i]] : 0.0;
    }
    double dummy0 = 0.0;
    blk_max2(mx, dummy0, s.red);
    double thr = 1e-14 * mx;
    for (int64_t q = a.cptr[g0] + tid; q < a.cptr[g0 + nr]; q += kST)
      Bg[a.cent_a[q] * s.ldz + a.cent_r[q]] = a.cent_v[q];
    // ---- A = L D L^T, right-looking by panels of <= 8 columns (a panel
    // boundary at ni, where the trailing matrix is exactly S_b):
    //   1. warp 0 factors the panel's diagonal block (pivot checks)
    //   2. rows below the block: their panel columns (one thread per row)
    //   3. trailing lower triangle -= (panel) D^-1 (panel)^T, 4 x 4 register tiles
    int fail = 0;
    for (int kb = 0; kb < n;) {
      const int ke = min(kb + 8, (kb < ni) ? ni : n);
      if (kb == ni && ni > 0) {  // Schur block S_b = trailing matrix: its own threshold
        double m2 = 0.0, dummy = 0.0;
        const int w = n - kb;
        for (int t = tid; t < w * w; t += kST) {
          const int i = t / w, j = t - i * w;
          if (j <= i) m2 = fmax(m2, fabs(s.W[(kb + j) * s.ld + kb + i]));
        }
        blk_max2(m2, dummy, s.red);
        thr = 1e-14 * m2;
      }
      if (warp == 0) {
        int f = 0;
        for (int k = kb; k < ke; ++k) {
          const double d = s.W[k * s.ld + k];
          if (!(d > thr)) {
            f = (fabs(d) > thr) ? 4 : 2;  // 4: not positive definite, 2: singular
            break;
          }
          const double dk = 1.0 / d;
          if (lane == 0) s.dinv[k] = dk;
          const int w = ke - k - 1;
          for (int t = lane; t < w * w; t += 32) {
            const int i = k + 1 + t / w, j = k + 1 + t % w;
            if (j <= i) s.W[j * s.ld + i] = fma(-s.W[k * s.ld + i], s.W[k * s.ld + j] * dk, s.W[j * s.ld + i]);
          }
          __syncwarp();
        }
        if (lane == 0) *s.flag = f;
      }
      __syncthreads();
      fail = *s.flag;
      if (fail) break;
      for (int i = ke + tid; i < n; i += kST)
        for (int k = kb; k < ke; ++k) {
          const double c = s.W[k * s.ld + i] * s.dinv[k];
          for (int j = k + 1; j < ke; ++j) s.W[j * s.ld + i] = fma(-c, s.W[k * s.ld + j], s.W[j * s.ld + i]);
        }
      __syncthreads();
      {
        const int m = n - ke, tb = (m + 3) / 4, nt = tb * (tb + 1) / 2, w = ke - kb;
        for (int t = tid; t < nt; t += kST) {
          int ti = static_cast<int>((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
          while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
          while (ti * (ti + 1) / 2 > t) --ti;
          const int tj = t - ti * (ti + 1) / 2;
          const int i0 = ke + 4 * ti, j0 = ke + 4 * tj;
          double acc[4][4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
          for (int k = kb; k < kb + w; ++k) {
            const double dk = s.dinv[k];
            double pi[4], pj[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              pi[r] = (i0 + r < n) ? s.W[k * s.ld + i0 + r] : 0.0;
              pj[r] = (j0 + r < n) ? s.W[k * s.ld + j0 + r] * dk : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[r][c] = fma(pi[r], pj[c], acc[r][c]);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (i0 + r < n && j0 + c <= i0 + r) s.W[(j0 + c) * s.ld + i0 + r] -= acc[r][c];
        }
      }
      __syncthreads();
      kb = ke;
    }
    if (fail) {
      if (tid == 0) {
        atomicOr(a.status, fail);
        atomicMin(reinterpret_cast<unsigned long long*>(a.bad_elem), static_cast<unsigned long long>(e));
      }
      __syncthreads();
      continue;
    }
    // ---- L (unit) and L^-1 in place; R is the scratch of the inversion
    for (int k = warp; k < n; k += kSW) {
      const double dk = s.dinv[k];
      for (int i = k + 1 + lane; i < n; i += 32) s.W[k * s.ld + i] *= dk;
    }
    __syncthreads();
    tri_invert(n, s.W, s.ld, s.R, s.R + 8 * nmax);
    // ---- Z = A^-1 B = Linv^T D^-1 Linv B, refined with exact residuals
    const PairTiles pt = pair_tiles(tid, n, nc);
    for (int t = tid; t < n * s.ldz; t += kST) s.Z[t] = Bg[t];
    __syncthreads();
    lower_inplace(n, nc, s.W, s.ld, s.dinv, s.Z, s.ldz);
    if (pt.ok) {  // R = Linv^T Z
      double acc[TM][TN];
      auto st = [&](int i, int c, double v) { s.R[i * s.ldz + c] = v; };
      upper_tile(n, s.W, s.ld, s.Z, s.ldz, pt.r0a, pt.c0, acc);
      store_tile(n, nc, pt.r0a, pt.c0, acc, st);
      if (pt.r0b >= 0) {
        upper_tile(n, s.W, s.ld, s.Z, s.ldz, pt.r0b, pt.c0, acc);
        store_tile(n, nc, pt.r0b, pt.c0, acc, st);
      }
    }
    __syncthreads();
    for (int t = tid; t < n * s.ldz; t += kST) s.Z[t] = (t % s.ldz < nc) ? s.R[t] : 0.0;
    __syncthreads();
    double prev = 0.0;
    for (int step = 0; step < 6; ++step) {
      residual(n, nc, A, s, Bg);
      __syncthreads();
      lower_inplace(n, nc, s.W, s.ld, s.dinv, s.R, s.ldz);
      double cm = 0.0, zm = 0.0;
      if (pt.ok) {  // Z += Linv^T R
        double acc[TM][TN];
        auto st = [&](int i, int c, double v) {
          const int o = i * s.ldz + c;
          const double z = s.Z[o] + v;
          s.Z[o] = z;
          cm = fmax(cm, fabs(v));
          zm = fmax(zm, fabs(z));
        };
        upper_tile(n, s.W, s.ld, s.R, s.ldz, pt.r0a, pt.c0, acc);
        store_tile(n, nc, pt.r0a, pt.c0, acc, st);
        if (pt.r0b >= 0) {
          upper_tile(n, s.W, s.ld, s.R, s.ldz, pt.r0b, pt.c0, acc);
          store_tile(n, nc, pt.r0b, pt.c0, acc, st);
        }
      }
      blk_max2(cm, zm, s.red);
      // the next correction is about rho * cm; rho = observed contraction (first
      // step: the relative size of the correction itself)
      const double rho = step > 0 ? fmin(1.0, prev > 0.0 ? cm / prev : 1.0) : (zm > 0.0 ? cm / zm : 0.0);
      prev = cm;
      if (!(cm * fmax(rho, 0x1p-52) > 0x1p-47 * zm)) break;
    }
    // ---- epilogue: H_e = C_b Z[:, :nr], g_e = C_b Z[:, nr]
    double* he = a.hbuf + a.hoff[e];
    double* ge = a.gbuf + g0;
    for (int t = tid; t < nr * nc; t += kST) {
      const int r = t / nc, q = t - r * nc;
      double hi = 0.0, lo = 0.0;
      for (int64_t z = a.cptr[g0 + r]; z < a.cptr[g0 + r + 1]; ++z) {
        double p, pe, sm, te;
        two_prod(a.cent_v[z], s.Z[a.cent_a[z] * s.ldz + q], p, pe);
        two_sum(hi, p, sm, te);
        hi = sm;
        lo += te + pe;
      }
      if (q < nr) he[static_cast<int64_t>(r) * nr + q] = hi + lo;
      else ge[r] = hi + lo;
    }
    __syncthreads();
  }
}

size_t spd_smem_bytes(int nmax, int ncmax) {
  const size_t ld = nmax | 1, ldz = (ncmax + 1) & ~1;
  const size_t r = std::max(nmax * ldz, 8 * static_cast<size_t>(nmax) + 64);
  return (((nmax * ld + 1) & ~size_t(1)) + nmax * ldz + r + nmax + 2 * kSW + 2) * 8 + static_cast<size_t>(nmax) * 4 + 16;
}

}  // namespace

bool spd_supported(int nmax, int ncmax) {
  const int units = (((nmax + TM - 1) / TM + 1) / 2) * ((ncmax + TN - 1) / TN);  // one row-tile pair per thread
  return units <= kST && spd_smem_bytes(nmax, ncmax) <= 227 * 1024;
}

int64_t spd_gws_doubles(int64_t ne, int nmax, int ncmax, int* grid) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  *grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ne, sms)));
  return static_cast<int64_t>(*grid) * nmax * ((ncmax + 1) & ~1);
}

void launch_spd_hyb(const AlgArgs& a, int nmax, int ncmax, double* gws, cudaStream_t st) {
  int grid = 1;
  spd_gws_doubles(a.ne, nmax, ncmax, &grid);
  const size_t smem = spd_smem_bytes(nmax, ncmax);
  cudaFuncSetAttribute(k_spd_hyb, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_spd_hyb<<<grid, kST, smem, st>>>(a, gws, static_cast<int64_t>(nmax) * ((ncmax + 1) & ~1), nmax, ncmax);
  count_launch();
}

}  // namespace hdr
