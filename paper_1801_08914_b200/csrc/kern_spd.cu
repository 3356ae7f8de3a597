// Element elimination for symmetric positive definite FE blocks (mapped cells,
// config 4; weighted affine cells): the hybridize drop-in of
//   hybridize(const ReductionInputs&)   src/reduction.cpp:262-354
// for element blocks that are SPD (every A_T = alpha D_T + beta M_T is).
//
// One 384-thread CTA per element (persistent), everything in shared memory:
//   W   n x n: the block in the [i | b] order (its lower triangle, mirrored),
//       swept in place by pivot blocks of <= 8 (block Gauss-Jordan in the
//       symmetric "sweep" form: W -> -A^-1, symmetric at every step).  The
//       scalar pivots are the LDL^T pivots and are checked with the reference's
//       SingularBlock rule (dense.cpp:61-97): the first ni against 1e-14
//       max|A_ii|, the rest against 1e-14 max|S_b| (a block boundary at ni,
//       where the unswept block is exactly S_b)
//   Z   n x nc: Z = A^-1 [C_T^T | f_T]
//   R   n x nc: right-hand sides / residuals
// The fp64 inverse is only a preconditioner: A_T is ill conditioned (alpha /
// beta up to 1e6, h^-2), so Z is refined with residuals B - A Z whose products
// are exact (two_prod) and whose sums are compensated (two_sum), until the
// correction times its observed contraction rate is below 2^-47 of |Z|.  This
// gives the element-exact H_e = C_b Z, g_e like the reference's own
// double-double oracle (src/reference.cpp:137-235).  Every product here is a
// 4 x 4 register-tiled GEMM over shared memory (128-bit loads).
#include <algorithm>

#include "hdr_device.cuh"
#include "kernels.hpp"

namespace hdr {

namespace {

#ifdef HDR_SPD_TIMING  // phase cycle counters of CTA 0 (variant builds only: make EXTRA=-DHDR_SPD_TIMING)
__device__ unsigned long long g_spd_prof[16];
#define SPD_T(slot)                                                         \
  do {                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      const long long now_ = clock64();                                     \
      g_spd_prof[slot] += static_cast<unsigned long long>(now_ - t_last_); \
      t_last_ = now_;                                                       \
    }                                                                       \
  } while (0)
#else
#define SPD_T(slot) \
  do {              \
  } while (0)
#endif

#ifndef HDR_SPD_UB
#define HDR_SPD_UB 1  // measured: 1 -> 18.9 ms, 2 -> 19.0, 4 -> 19.6 (cfg4)
#endif
constexpr int kST = 384;
constexpr int kSW = kST / 32;

struct SpdSmem {
  double* W;   // n x ld
  double* Z;   // n x ldz
  double* R;   // n x ldz
  double* T;   // 8 x ld: A_iB P^-1 of the current pivot block
  double* C;   // 8 x ld: A_iB (the block's columns before the step)
  double* P;   // 2 x 8 x 8: swept pivot blocks (-P^-1), double-buffered
  double* piv; // n scalar pivots
  double* rsum;  // n: row sums of |A| (residual anchors)
  double* red;
  int* sidx;
  int* flag;
  int ld, ldz;
};

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

// One warp: sweep the 8 x 8 block P (row-major; a w x w pivot block padded with
// the identity) in registers, P <- -P^-1.  Lane l holds (l/8, l%8) and
// (l/8 + 4, l%8).  The scalar pivots go to piv[0, w) (checked later).
__device__ void sweep8(double* P, int w, double* piv) {
  const int lane = threadIdx.x & 31, r = lane >> 3, c = lane & 7;
  double v0 = P[r * 8 + c], v1 = P[(r + 4) * 8 + c];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double akk = __shfl_sync(0xffffffffu, k < 4 ? v0 : v1, ((k & 3) << 3) | k);
    const double aik0 = __shfl_sync(0xffffffffu, v0, (r << 3) | k);
    const double aik1 = __shfl_sync(0xffffffffu, v1, (r << 3) | k);
    const double akj = __shfl_sync(0xffffffffu, k < 4 ? v0 : v1, ((k & 3) << 3) | c);
    if (lane == 0 && k < w) piv[k] = akk;
    // reciprocal for the preconditioner (refinement absorbs its last-bit error):
    // fp32 seed + two Newton steps
    double inv = static_cast<double>(__frcp_rn(static_cast<float>(akk)));
    inv = inv * fma(-akk, inv, 2.0);
    inv = inv * fma(-akk, inv, 2.0);
    auto upd = [&](int i, double v, double aik) {
      if (i == k) return c == k ? -inv : akj * inv;
      if (c == k) return aik * inv;
      return fma(-aik * inv, akj, v);
    };
    v0 = upd(r, v0, aik0);
    v1 = upd(r + 4, v1, aik1);
  }
  P[r * 8 + c] = v0;
  P[(r + 4) * 8 + c] = v1;
}

// warp 0: the pivot block [kb, kb + w) of W (padded with the identity) -> P, swept
__device__ void load_sweep(const double* W, int ld, int kb, int w, double* P, double* piv) {
  for (int t = threadIdx.x & 31; t < 64; t += 32) {
    const int r = t >> 3, c = t & 7;
    const int hi = r > c ? r : c, lo = r > c ? c : r;  // lower triangle holds the block
    P[t] = (r < w && c < w) ? W[(kb + hi) * ld + kb + lo] : (r == c ? 1.0 : 0.0);
  }
  __syncwarp();
  sweep8(P, w, piv + kb);
  __syncwarp();
}

__device__ __forceinline__ int block_end(int kb, int n, int ni) { return min(kb + 8, (kb < ni) ? ni : n); }

// lower 4 x 4 tile index t -> (ti, tj), tj <= ti
__device__ __forceinline__ void tri_tile(int t, int& ti, int& tj) {
  ti = static_cast<int>((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  tj = t - ti * (ti + 1) / 2;
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// W[i][j] -= sum_k T[k][i] C[k][j] on the 8 x 8 block (bi, bj), bi >= bj, by one
// warp on the fp64 tensor cores (two DMMA m8n8k4; fragments a = (row g, k t),
// b = (k t, col g), d = (row g, cols 2t, 2t + 1) with g = lane / 4, t = lane % 4).
// Rows / columns >= n are left alone.  Entries in the pivot block's rows or
// columns and above the diagonal are updated too: the write-back rewrites the
// former, the latter are dead until the final mirror.
template <int NB>
__device__ __forceinline__ void sweep_blocks(double* W, int ld, const double* T, const double* C, int n, int w,
                                             const int (&bi)[NB], const int (&bj)[NB]) {
  // NB independent blocks per call: their loads and MMAs interleave (latency)
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double d0[NB], d1[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int r = 8 * bi[q] + g, c = 8 * bj[q] + 2 * t;
    const bool rok = bi[q] >= 0 && r < n;
    d0[q] = rok && c < n ? W[r * ld + c] : 0.0;
    d1[q] = rok && c + 1 < n ? W[r * ld + c + 1] : 0.0;
  }
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const int k = 4 * ks + t;
    double av[NB], bv[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int i = 8 * bi[q] + g, j = 8 * bj[q] + g;
      av[q] = (bi[q] >= 0 && k < w && i < n) ? -T[k * ld + i] : 0.0;
      bv[q] = (bi[q] >= 0 && k < w && j < n) ? C[k * ld + j] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) dmma_8x8x4(d0[q], d1[q], av[q], bv[q]);
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int r = 8 * bi[q] + g, c = 8 * bj[q] + 2 * t;
    if (bi[q] < 0 || r >= n) continue;
    if (c < n) W[r * ld + c] = d0[q];
    if (c + 1 < n) W[r * ld + c + 1] = d1[q];
  }
}

__device__ __forceinline__ void sweep_block(double* W, int ld, const double* T, const double* C, int n, int w, int bi,
                                            int bj) {
  const int ri[1] = {bi}, rj[1] = {bj};
  sweep_blocks<1>(W, ld, T, C, n, w, ri, rj);
}

// acc (+)= sign * W[i0:i0+4, :] Y[:, c0:c0+4] over k < n (W symmetric: read as rows).
// Column order swizzled: acc[.][b] is column c0 + (b ^ tile_swz()) -- lanes 4..7
// of each quarter-warp read the upper half of their 32-byte Y segment first, so
// the 128-bit loads of 8 lanes at a 32-byte stride cover 32 distinct banks.
__device__ __forceinline__ int tile_swz() { return threadIdx.x & 4 ? 2 : 0; }
__device__ __forceinline__ void gemm_tile(int n, const double* W, int ld, const double* Y, int ldy, int i0, int c0,
                                          double (&acc)[4][4]) {
  const int ya = c0 + tile_swz(), yb = c0 + (tile_swz() ^ 2);
#pragma unroll 2
  for (int k = 0; k < n; ++k) {
    const double2 w0 = *reinterpret_cast<const double2*>(W + k * ld + i0);
    const double2 w1 = *reinterpret_cast<const double2*>(W + k * ld + i0 + 2);
    const double2 y0 = *reinterpret_cast<const double2*>(Y + k * ldy + ya);
    const double2 y1 = *reinterpret_cast<const double2*>(Y + k * ldy + yb);
    const double wv[4] = {w0.x, w0.y, w1.x, w1.y}, yv[4] = {y0.x, y0.y, y1.x, y1.y};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(wv[a], yv[b], acc[a][b]);
  }
}

// R = B - A Z to ~2^-99 of sum |B| + |A||Z| (rounded once), five fp64 ops per
// term instead of a double-double dot product: with a per-row anchor
// C = 1.5 * 2^q, 2^(q-1) > |B| + rowsum|A| * max|Z| (every product and partial
// sum fits below 2^(q-1)):
//   t = fma(a, z, C); p_hi = t - C (exact, Sterbenz: a z rounded to ulp(C));
//   p_lo = fma(a, z, -p_hi) (the remainder, rounded: <= u ulp(C) / 2);
//   S_hi += p_hi (exact: multiples of ulp(C) below 2^(q+1)), S_lo += p_lo.
// Thread tiles of TM rows x TN columns; A read through the [i | b] permutation.
__device__ void residual(int n, int nc, const double* A, const SpdSmem& s, const double* Bg, double bound_z,
                         double bmax) {
  constexpr int TM = 4, TN = 4;
  const int tn = (nc + TN - 1) / TN, tm = (n + TM - 1) / TM;
  for (int tile = threadIdx.x; tile < tm * tn; tile += kST) {
    const int r0 = (tile / tn) * TM, c0 = (tile % tn) * TN;
    double hi[TM][TN], lo[TM][TN], anc[TM];
    const double* arow[TM];
#pragma unroll
    for (int a = 0; a < TM; ++a) {
      const int r = min(r0 + a, n - 1);
      arow[a] = A + static_cast<int64_t>(s.sidx[r]) * n;
      const double x = fmax(s.rsum[r] * bound_z + bmax, 1e-280);
      anc[a] = scalbn(1.5, ilogb(x) + 2);
#pragma unroll
      for (int b = 0; b < TN; ++b) {
        const double bv = (r0 + a < n && c0 + b < nc) ? Bg[(r0 + a) * s.ldz + c0 + b] : 0.0;
        hi[a][b] = (bv + anc[a]) - anc[a];
        lo[a][b] = bv - hi[a][b];
      }
    }
#pragma unroll 2
    for (int j = 0; j < n; ++j) {
      const int cj = s.sidx[j];
      double av[TM], zv[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) av[a] = -__ldg(arow[a] + cj);
#pragma unroll
      for (int b = 0; b < TN; ++b) zv[b] = s.Z[j * s.ldz + c0 + b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) {
          const double t = fma(av[a], zv[b], anc[a]);
          const double ph = t - anc[a];
          hi[a][b] += ph;
          lo[a][b] += fma(av[a], zv[b], -ph);
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
  s.ld = (nmax + 1) & ~1;
  s.ldz = (ncmax + 3) & ~3;
  s.W = smem;
  s.Z = s.W + nmax * s.ld;
  s.R = s.Z + nmax * s.ldz;
  s.T = s.R + nmax * s.ldz;
  s.C = s.T + 8 * s.ld;
  s.P = s.C + 8 * s.ld;
  s.piv = s.P + 128;
  s.rsum = s.piv + nmax;
  s.red = s.rsum + nmax;
  s.sidx = reinterpret_cast<int*>(s.red + 2 * kSW);
  s.flag = s.sidx + nmax;
  double* Bg = gws + static_cast<int64_t>(blockIdx.x) * slot;  // n x ldz right-hand sides
  const int tid = threadIdx.x, warp = tid >> 5;
  const int ld = s.ld, ldz = s.ldz;
#ifdef HDR_SPD_TIMING
  long long t_last_ = clock64();
#endif
  for (int64_t e = blockIdx.x; e < a.ne; e += gridDim.x) {
    SPD_T(0);
    const int64_t boff = a.boff[e];
    const int n = static_cast<int>(a.boff[e + 1] - boff), ni = a.ni[e];
    const int64_t g0 = a.goff[e];
    const int nr = static_cast<int>(a.goff[e + 1] - g0), nc = nr + 1;
    const double* A = a.blocks + a.aoff[e];
    for (int i = tid; i < n; i += kST) s.sidx[i] = a.idx[boff + i];
    __syncthreads();
    // permuted block: lower triangle, mirrored; max |A_ii|
    double mx = 0.0;
    for (int t0 = tid; t0 < n * n; t0 += 4 * kST) {  // 4 loads in flight per thread
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * kST, i = t / n, k = t - i * n;
        v[u] = (t < n * n && k <= i) ? __ldg(A + static_cast<int64_t>(s.sidx[i]) * n + s.sidx[k]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * kST, i = t / n, k = t - i * n;
        if (t >= n * n || k > i) continue;
        s.W[i * ld + k] = v[u];
        if (ni == 0 || i < ni) mx = fmax(mx, fabs(v[u]));
      }
    }
    // right-hand sides [C_T^T | f_T] (global slot, row-major n x ldz, padding 0)
    for (int t = tid; t < n * ldz; t += kST) {
      const int i = t / ldz, c = t - i * ldz;
      Bg[t] = c == nr ? a.f[boff + s.sidx[i]] : 0.0;
    }
    double bmax = 1.0;  // max |B|: unit / weighted constraint columns and f_T
    for (int i = tid; i < n; i += kST) bmax = fmax(bmax, fabs(a.f[boff + s.sidx[i]]));
    for (int64_t q = a.cptr[g0] + tid; q < a.cptr[g0 + nr]; q += kST) bmax = fmax(bmax, fabs(a.cent_v[q]));
    blk_max2(mx, bmax, s.red);
    double thr = 1e-14 * mx;
    for (int i = tid; i < n; i += kST) {  // row sums of |A| (the block, symmetric lower triangle loaded)
      double rs = 0.0;
      for (int k = 0; k < n; ++k) rs += fabs(k <= i ? s.W[i * ld + k] : s.W[k * ld + i]);
      s.rsum[i] = rs;
    }
    for (int64_t q = a.cptr[g0] + tid; q < a.cptr[g0 + nr]; q += kST)
      Bg[a.cent_a[q] * ldz + a.cent_r[q]] = a.cent_v[q];
    SPD_T(1);
    // ---- sweep: W -> -A^-1 by pivot blocks B = [kb, kb + w).  Look-ahead:
    // warp 0 updates the next pivot block's tiles first and sweeps it while
    // the other warps finish the trailing update.  Pivots are checked at the end.
    const int nb4 = (n + 3) / 4, ntl = nb4 * (nb4 + 1) / 2;
    double thr2 = thr;
    if (warp == 0) load_sweep(s.W, ld, 0, block_end(0, n, ni), s.P, s.piv);
    __syncthreads();
    int cur = 0;
    for (int kb = 0; kb < n;) {
      const int ke = block_end(kb, n, ni), w = ke - kb;
      const int kn = ke < n ? block_end(ke, n, ni) : ke;  // next block [ke, kn)
      const double* P = s.P + 64 * cur;
      // C[m][i] = A_i,kb+m (lower triangle), T[k][i] = (A_iB P^-1)_k = -sum_m C[m][i] Sw[m][k]  (i outside B):
      // thread (i, kq) loads row i's block entries once and makes T for k in [3 kq, 3 kq + 3)
      for (int t = tid; t < 3 * n; t += kST) {
        const int kq = t / n, i = t - kq * n;
        if (i >= kb && i < ke) continue;
        double cv[8];
#pragma unroll
        for (int m = 0; m < 8; ++m)
          cv[m] = m < w ? ((i > kb + m) ? s.W[i * ld + kb + m] : s.W[(kb + m) * ld + i]) : 0.0;
        if (kq == 0)
#pragma unroll
          for (int m = 0; m < 8; ++m)
            if (m < w) s.C[m * ld + i] = cv[m];
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const int k = 3 * kq + kk;
          if (k >= w) break;
          double acc = 0.0;
#pragma unroll
          for (int m = 0; m < 8; ++m) acc = fma(cv[m], P[m * 8 + k], acc);
          s.T[k * ld + i] = -acc;
        }
      }
      __syncthreads();
      SPD_T(2);
      // trailing update on 8 x 8 blocks (fp64 tensor cores), lower triangle, blocks
      // lying fully in B's rows or columns skipped; the blocks of the next pivot
      // block go to warp 0, which then sweeps it
      const int nb8 = (n + 7) / 8, a0 = ke >> 3, a1 = (kn - 1) >> 3;
      const int sb = (kb % 8 == 0 && w == 8) ? kb >> 3 : -1;  // block row / column fully inside B
      const int nr8 = nb8 - (sb >= 0 ? 1 : 0), ntr = nr8 * (nr8 + 1) / 2;
#ifdef HDR_SPD_TIMING
      const long long tw0 = clock64();
#endif
      if (warp == 0) {
        if (kn > ke) {
          for (int bi = a0; bi <= a1; ++bi)
            for (int bj = a0; bj <= bi; ++bj) sweep_block(s.W, ld, s.T, s.C, n, w, bi, bj);
          __syncwarp();
#ifdef HDR_SPD_TIMING
          if (blockIdx.x == 0 && threadIdx.x == 0) g_spd_prof[11] += clock64() - tw0;
#endif
          load_sweep(s.W, ld, ke, kn - ke, s.P + 64 * (cur ^ 1), s.piv);
#ifdef HDR_SPD_TIMING
          if (blockIdx.x == 0 && threadIdx.x == 0) g_spd_prof[12] += clock64() - tw0;
#endif
        }
      } else {
        constexpr int UB = HDR_SPD_UB;  // blocks per warp in flight
        for (int q0 = warp - 1; q0 < ntr; q0 += UB * (kSW - 1)) {
          int bi[UB], bj[UB];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int q = q0 + u * (kSW - 1);
            bi[u] = -1;
            bj[u] = 0;
            if (q >= ntr) continue;
            int ti, tj;
            tri_tile(q, ti, tj);
            ti += (sb >= 0 && ti >= sb) ? 1 : 0;
            tj += (sb >= 0 && tj >= sb) ? 1 : 0;
            if (kn > ke && ti >= a0 && ti <= a1 && tj >= a0 && tj <= a1) continue;
            bi[u] = ti;
            bj[u] = tj;
          }
          sweep_blocks<UB>(s.W, ld, s.T, s.C, n, w, bi, bj);
        }
#ifdef HDR_SPD_TIMING
        if (blockIdx.x == 0 && threadIdx.x == 32) g_spd_prof[13] += clock64() - tw0;
#endif
      }
      __syncthreads();
      SPD_T(3);
      for (int t = tid; t < w * n; t += kST) {
        const int k = t / n, i = t - k * n, col = kb + k;
        if (i < col) s.W[col * ld + i] = (i >= kb) ? P[k * 8 + (i - kb)] : s.T[k * ld + i];
        else s.W[i * ld + col] = (i < ke) ? P[(i - kb) * 8 + k] : s.T[k * ld + i];
      }
      if (ke == ni && ni > 0) {  // the unswept block is now S_b: its own threshold
        double m2 = 0.0, dummy = 0.0;
        const int m = n - ke;
        for (int t = tid; t < m * m; t += kST) {
          const int i = t / m, j = t - i * m;
          if (j <= i) m2 = fmax(m2, fabs(s.W[(ke + i) * ld + ke + j]));
        }
        blk_max2(m2, dummy, s.red);
        thr2 = 1e-14 * m2;
      }
      __syncthreads();
      SPD_T(4);
      cur ^= 1;
      kb = ke;
    }
    for (int t = tid; t < n * n; t += kST) {  // the full matrix for the products below
      const int i = t / n, j = t - i * n;
      if (j > i) s.W[i * ld + j] = s.W[j * ld + i];
    }
    // pivot checks (the reference's SingularBlock rule)
    int fail = 0;
    for (int k = tid; k < n; k += kST) {
      const double d = s.piv[k], t2 = (k < ni || ni == 0) ? thr : thr2;
      if (!(d > t2)) fail = max(fail, (fabs(d) > t2) ? 4 : 2);
    }
    {
      double f0 = fail, dummy = 0.0;
      blk_max2(f0, dummy, s.red);
      fail = static_cast<int>(f0);
    }
    if (fail) {
      if (tid == 0) {
        atomicOr(a.status, fail);
        atomicMin(reinterpret_cast<unsigned long long*>(a.bad_elem), static_cast<unsigned long long>(e));
      }
      __syncthreads();
      continue;
    }
    SPD_T(5);
    // ---- Z = A^-1 B = -W B, refined with exact residuals; one 4 x 4 tile per thread
    const int tn = (nc + 3) / 4, ntz = nb4 * tn;
    for (int t = tid; t < n * ldz; t += kST) s.R[t] = Bg[t];
    bool unit = a.cptr[g0 + nr] - a.cptr[g0] == nr;  // one entry per row: C_T^T columns are (scaled) unit vectors
    __syncthreads();
    if (unit) {  // Z[:, r] = -W[:, a_r] v_r (exact), Z[:, nr] = -W f
      for (int t = tid; t < n * nr; t += kST) {
        const int r = t / n, i = t - r * n;
        const int64_t q = a.cptr[g0 + r];
        s.Z[i * ldz + a.cent_r[q]] = -s.W[a.cent_a[q] * ld + i] * a.cent_v[q];
      }
      for (int i = tid; i < n; i += kST) {
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc = fma(s.W[k * ld + i], s.R[k * ldz + nr], acc);
        s.Z[i * ldz + nr] = -acc;
        for (int c = nc; c < ldz; ++c) s.Z[i * ldz + c] = 0.0;
      }
    } else {
      for (int t = tid; t < ntz; t += kST) {
        const int i0 = (t / tn) * 4, c0 = (t % tn) * 4;
        double acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
        gemm_tile(n, s.W, ld, s.R, ldz, i0, c0, acc);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (i0 + r < n) s.Z[(i0 + r) * ldz + c0 + (c ^ tile_swz())] = (c0 + (c ^ tile_swz()) < nc) ? -acc[r][c] : 0.0;
      }
    }
    __syncthreads();
    SPD_T(6);
    double zb = 0.0, dummy1 = 0.0;  // max |Z|: the residual anchors' bound
    for (int t = tid; t < n * ldz; t += kST) zb = fmax(zb, fabs(s.Z[t]));
    blk_max2(zb, dummy1, s.red);
    double prev = 0.0;
    for (int step = 0; step < 6; ++step) {
      residual(n, nc, A, s, Bg, zb, bmax);
      __syncthreads();
      SPD_T(7);
#ifdef HDR_SPD_TIMING
      if (blockIdx.x == 0 && threadIdx.x == 0) g_spd_prof[15] += 1;  // residual count
#endif
      double cm = 0.0, zm = 0.0;
      for (int t = tid; t < ntz; t += kST) {  // Z -= W R
        const int i0 = (t / tn) * 4, c0 = (t % tn) * 4;
        double acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
        gemm_tile(n, s.W, ld, s.R, ldz, i0, c0, acc);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (i0 + r < n && c0 + (c ^ tile_swz()) < nc) {
              const int o = (i0 + r) * ldz + c0 + (c ^ tile_swz());
              const double z = s.Z[o] - acc[r][c];
              s.Z[o] = z;
              cm = fmax(cm, fabs(acc[r][c]));
              zm = fmax(zm, fabs(z));
            }
      }
      blk_max2(cm, zm, s.red);
      zb = zm;
      // the next correction is about rho * cm; rho = observed contraction (first
      // step: the relative size of the correction itself)
      const double rho = step > 0 ? fmin(1.0, prev > 0.0 ? cm / prev : 1.0) : (zm > 0.0 ? cm / zm : 0.0);
      prev = cm;
      SPD_T(8);
      if (!(cm * fmax(rho, 0x1p-52) > 0x1p-47 * zm)) break;
    }
    SPD_T(9);
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
    SPD_T(10);
#ifdef HDR_SPD_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) g_spd_prof[14] += 1;  // cells
#endif
  }
}

size_t spd_smem_bytes(int nmax, int ncmax) {
  const size_t ld = (nmax + 1) & ~1, ldz = (ncmax + 3) & ~3;
  return (nmax * ld + 2 * nmax * ldz + 16 * ld + 128 + 2 * nmax + 2 * kSW) * 8 + static_cast<size_t>(nmax + 2) * 4;
}

}  // namespace

#ifdef HDR_SPD_TIMING
extern "C" int hdr_debug_spd_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_spd_prof, sizeof(g_spd_prof));
  return 0;
}
#endif

bool spd_supported(int nmax, int ncmax) { return spd_smem_bytes(nmax, ncmax) <= 227 * 1024; }

int64_t spd_gws_doubles(int64_t ne, int nmax, int ncmax, int* grid) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  *grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ne, sms)));
  return static_cast<int64_t>(*grid) * nmax * ((ncmax + 3) & ~3);
}

void launch_spd_hyb(const AlgArgs& a, int nmax, int ncmax, double* gws, cudaStream_t st) {
  int grid = 1;
  spd_gws_doubles(a.ne, nmax, ncmax, &grid);
  const size_t smem = spd_smem_bytes(nmax, ncmax);
  cudaFuncSetAttribute(k_spd_hyb, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_spd_hyb<<<grid, kST, smem, st>>>(a, gws, static_cast<int64_t>(nmax) * ((ncmax + 3) & ~3), nmax, ncmax);
  count_launch();
}

}  // namespace hdr
