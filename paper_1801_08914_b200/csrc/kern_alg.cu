// Algebraic batch path: hybridize / static_condense / recoveries on a general
// ReductionInputs (arbitrary dense element blocks, arbitrary C and P), the
// drop-in for the reference's
//   hybridize(const ReductionInputs&)          src/reduction.cpp:262-354
//   recover_hybrid(op, lambda, f_hat)          src/reduction.cpp:356-446
//   static_condense(const ReductionInputs&)    src/reduction.cpp:448-557
//   recover_condensed(op, x_b, f_hat)          src/reduction.cpp:559-587
//
// One CTA per element (persistent over elements).  The element matrix is taken
// in the partitioned order [i dofs | b dofs] and factored by LU with partial
// pivoting restricted to the i rows for the first ni steps (so the first ni
// pivots are those of A_ii and the rest those of the Schur complement S_b — the
// two factorizations the reference performs, with its SingularBlock rule
// |pivot| <= 1e-14 max|block|, src/dense.cpp:61-97).  Solves are refined with
// residuals accumulated exactly (two_prod / two_sum, rounded once) until the
// correction is below the last bit, so X = M^-1 B is correctly rounded up to a
// few ulps whatever the conditioning (the reference's fixed two refinement
// steps on a rounded Schur complement are not).  Products
// with C, A_bi in the epilogues are compensated as well.
//
// Per-CTA workspace: LU (column-major d x d), X and R (row-major d x nc) in
// shared memory when they fit, else in a global slot; B0 and the low parts Xl
// (row-major d x nc) in the global slot.
#include <algorithm>

#include "hdr_device.cuh"
#include "kernels.hpp"

namespace hdr {

namespace {

constexpr int kAT = 1024;  // threads per CTA
constexpr int kAW = kAT / 32;

struct DD {
  double hi, lo;
};

__device__ __forceinline__ void dd_acc(double& hi, double& lo, double p, double pe) {
  // (hi, lo) += p + pe, p + pe an exact product
  double s, t;
  two_sum(hi, p, s, t);
  hi = s;
  lo += t + pe;
}

__device__ __forceinline__ void dd_fma(double& hi, double& lo, double a, double b) {
  double p, e;
  two_prod(a, b, p, e);
  dd_acc(hi, lo, p, e);
}

// block-wide argmax of |v| (ties: smaller index); returns (value, index) to all threads
__device__ void block_argmax(double v, int idx, double* sv, int* si, double& best, int& besti) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a = fabs(v);
  int ia = idx;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double b = __shfl_down_sync(0xffffffffu, a, o);
    const int ib = __shfl_down_sync(0xffffffffu, ia, o);
    if (b > a || (b == a && ib < ia)) {
      a = b;
      ia = ib;
    }
  }
  if (lane == 0) {
    sv[warp] = a;
    si[warp] = ia;
  }
  __syncthreads();
  if (warp == 0) {
    a = lane < kAW ? sv[lane] : -1.0;
    ia = lane < kAW ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double b = __shfl_down_sync(0xffffffffu, a, o);
      const int ib = __shfl_down_sync(0xffffffffu, ia, o);
      if (b > a || (b == a && ib < ia)) {
        a = b;
        ia = ib;
      }
    }
    if (lane == 0) {
      sv[kAW] = a;
      si[kAW] = ia;
    }
  }
  __syncthreads();
  best = sv[kAW];
  besti = si[kAW];
  __syncthreads();
}

__device__ double block_max(double v, double* sv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  if (lane == 0) sv[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kAW ? sv[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) sv[kAW] = v;
  }
  __syncthreads();
  const double r = sv[kAW];
  __syncthreads();
  return r;
}

struct Elem {
  const double* A;   // row-major n x n block
  const int* idx;    // n local dofs: [i dofs | b dofs]
  int n, ni, d;      // d = matrix order of the solve (n for hybrid modes, ni for condense modes)
  int64_t boff;      // broken offset of the block
};

__device__ __forceinline__ double Mget(const Elem& E, int i, int k) {
  return __ldg(E.A + static_cast<int64_t>(E.idx[i]) * E.n + E.idx[k]);
}

// LU with block-restricted partial pivoting (see header).  Returns false on a
// singular pivot.
__device__ bool block_lu(const Elem& E, int ni_piv, double* lu, int* piv, double* sv, int* si) {
  const int d = E.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < d; k += kAW) {
    const double* arow_k = E.A + E.idx[k];  // column idx[k] of A, stride n
    for (int i = lane; i < d; i += 32) lu[k * d + i] = __ldg(arow_k + static_cast<int64_t>(E.idx[i]) * E.n);
  }
  __syncthreads();
  double thr = 0.0;
  {
    double mx = 0.0;
    const int lim = ni_piv > 0 ? ni_piv : d;
    for (int t = threadIdx.x; t < lim * lim; t += kAT) mx = fmax(mx, fabs(lu[(t / lim) * d + t % lim]));
    thr = 1e-14 * block_max(mx, sv);
  }
  for (int j = 0; j < d; ++j) {
    if (j == ni_piv && ni_piv > 0) {  // Schur block threshold: max |S_b| of the trailing matrix
      double mx = 0.0;
      const int w = d - j;
      for (int t = threadIdx.x; t < w * w; t += kAT) mx = fmax(mx, fabs(lu[(j + t / w) * d + j + t % w]));
      thr = 1e-14 * block_max(mx, sv);
    }
    const int lim = j < ni_piv ? ni_piv : d;
    double v = 0.0;
    int vi = 0x7fffffff;
    for (int i = j + threadIdx.x; i < lim; i += kAT) {
      const double a = lu[j * d + i];
      if (vi == 0x7fffffff || fabs(a) > fabs(v)) {
        v = a;
        vi = i;
      }
    }
    double best;
    int p;
    block_argmax(vi == 0x7fffffff ? 0.0 : v, vi, sv, si, best, p);
    if (!(best > thr)) return false;  // also catches NaN
    if (threadIdx.x == 0) piv[j] = p;
    if (p != j)
      for (int k = threadIdx.x; k < d; k += kAT) {
        const double a = lu[k * d + j];
        lu[k * d + j] = lu[k * d + p];
        lu[k * d + p] = a;
      }
    __syncthreads();
    const double inv = lu[j * d + j];
    for (int i = j + 1 + threadIdx.x; i < d; i += kAT) lu[j * d + i] = lu[j * d + i] / inv;
    __syncthreads();
    for (int k = j + 1 + warp; k < d; k += kAW) {
      const double ukj = lu[k * d + j];
      for (int i = j + 1 + lane; i < d; i += 32) lu[k * d + i] = fma(-lu[j * d + i], ukj, lu[k * d + i]);
    }
    __syncthreads();
  }
  return true;
}

// Y <- LU^-1 P Y for the nc columns of Y (row-major d x nc: Y[i*nc + c]),
// blocked by kSB rows: the diagonal triangle of a block is solved column by
// column (one thread per column), the rows below / above are updated by a
// kSB-deep product (warps over rows, lanes over columns) — two barriers per
// block instead of one or two per row.
constexpr int kSB = 8;
__device__ void block_solve(int d, int nc, const double* lu, const int* piv, double* Y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < nc; c += kAT)
    for (int j = 0; j < d; ++j) {
      const int p = piv[j];
      if (p != j) {
        const double t = Y[j * nc + c];
        Y[j * nc + c] = Y[p * nc + c];
        Y[p * nc + c] = t;
      }
    }
  __syncthreads();
  for (int jb = 0; jb < d; jb += kSB) {  // forward, unit lower L
    const int je = min(jb + kSB, d);
    for (int c = threadIdx.x; c < nc; c += kAT)
      for (int j = jb; j < je; ++j) {
        const double yj = Y[j * nc + c];
        for (int i = j + 1; i < je; ++i) Y[i * nc + c] = fma(-lu[j * d + i], yj, Y[i * nc + c]);
      }
    __syncthreads();
    for (int i = je + warp; i < d; i += kAW) {
      double l[kSB];
#pragma unroll
      for (int t = 0; t < kSB; ++t) l[t] = jb + t < je ? lu[(jb + t) * d + i] : 0.0;
      for (int c = lane; c < nc; c += 32) {
        double acc = Y[i * nc + c];
#pragma unroll
        for (int t = 0; t < kSB; ++t)
          if (jb + t < je) acc = fma(-l[t], Y[(jb + t) * nc + c], acc);
        Y[i * nc + c] = acc;
      }
    }
    __syncthreads();
  }
  for (int je = d; je > 0; je -= kSB) {  // backward, upper U
    const int jb = max(0, je - kSB);
    for (int c = threadIdx.x; c < nc; c += kAT)
      for (int j = je - 1; j >= jb; --j) {
        const double yj = Y[j * nc + c] / lu[j * d + j];
        Y[j * nc + c] = yj;
        for (int i = jb; i < j; ++i) Y[i * nc + c] = fma(-lu[j * d + i], yj, Y[i * nc + c]);
      }
    __syncthreads();
    for (int i = warp; i < jb; i += kAW) {
      double u[kSB];
#pragma unroll
      for (int t = 0; t < kSB; ++t) u[t] = jb + t < je ? lu[(jb + t) * d + i] : 0.0;
      for (int c = lane; c < nc; c += 32) {
        double acc = Y[i * nc + c];
#pragma unroll
        for (int t = 0; t < kSB; ++t)
          if (jb + t < je) acc = fma(-u[t], Y[(jb + t) * nc + c], acc);
        Y[i * nc + c] = acc;
      }
    }
    __syncthreads();
  }
}

// Xg + Xlg <- M^-1 B0 (B0 = b0h + b0l; all row-major d x nc, global) as a
// double-double (Xg the rounded value, Xlg the remainder), in column chunks of
// at most ncc held in shared memory (Xs, Xls, Rs: d x cw each): residuals
// B0 - M (X + Xl) are accumulated exactly (one warp per row, lanes over the
// chunk's columns), corrections solved with the LU and folded in with two_sum.
// Stops when the correction, scaled by its observed contraction rate, is below
// tgt of the solution (tgt = 2^-100 where the epilogue cancels: f_S = f_b -
// A_bi A_ii^-1 f_i; 2^-60 elsewhere).
__device__ void refined_solve(const Elem& E, int nc, int ncc, const double* lu, const int* piv, const double* b0h,
                              const double* b0l, double* Xg, double* Xlg, double* Xs, double* Xls, double* Rs,
                              double* sv, double tgt) {
  const int d = E.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < nc; c0 += ncc) {
    const int cw = min(ncc, nc - c0);
    for (int i = warp; i < d; i += kAW)
      for (int c = lane; c < cw; c += 32) {
        Xs[i * cw + c] = b0h[i * nc + c0 + c];
        Xls[i * cw + c] = 0.0;
      }
    __syncthreads();
    block_solve(d, cw, lu, piv, Xs);
    double prev = 0.0;
    for (int step = 0; step < 8; ++step) {
      for (int i = warp; i < d; i += kAW) {
        const double* arow = E.A + static_cast<int64_t>(E.idx[i]) * E.n;
        for (int c = lane; c < cw; c += 32) {
          double hi = b0h[i * nc + c0 + c], lo = b0l ? b0l[i * nc + c0 + c] : 0.0;
          for (int k = 0; k < d; ++k) {
            const double m = -__ldg(arow + E.idx[k]);
            dd_fma(hi, lo, m, Xs[k * cw + c]);
            lo = fma(m, Xls[k * cw + c], lo);
          }
          Rs[i * cw + c] = hi + lo;
        }
      }
      __syncthreads();
      block_solve(d, cw, lu, piv, Rs);
      double cm = 0.0, xm = 0.0;
      for (int t = threadIdx.x; t < d * cw; t += kAT) {
        const double c = Rs[t];
        double hi, e;
        two_sum(Xs[t], c + Xls[t], hi, e);
        Xs[t] = hi;
        Xls[t] = e;
        cm = fmax(cm, fabs(c));
        xm = fmax(xm, fabs(hi));
      }
      cm = block_max(cm, sv);
      xm = block_max(xm, sv);
      // the next correction is about rho * cm (rho: observed contraction)
      const double rho = step > 0 && prev > 0.0 ? fmin(1.0, cm / prev) : 1.0;
      prev = cm;
      if (!(cm * fmax(rho, 0x1p-52) > tgt * xm)) break;
    }
    for (int i = warp; i < d; i += kAW)
      for (int c = lane; c < cw; c += 32) {
        Xg[i * nc + c0 + c] = Xs[i * cw + c];
        Xlg[i * nc + c0 + c] = Xls[i * cw + c];
      }
    __syncthreads();
  }
}

template <int MODE>
__global__ void __launch_bounds__(kAT) k_alg(AlgArgs a, double* gws, AlgPlan p) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double sv[kAW + 1];
  __shared__ int si[kAW + 1];
  // fast region (LU, column-chunk buffers, piv): shared memory when it fits;
  // slow region (B0h, B0l, X, Xl: element-wise traffic only) in the CTA's global slot
  const int64_t stride = p.slow + (p.smem ? 0 : p.fast);
  double* Ws = gws + static_cast<int64_t>(blockIdx.x) * stride;
  double* Wf = p.smem ? smem : Ws + p.slow;
  for (int64_t e = blockIdx.x; e < a.ne; e += gridDim.x) {
    Elem E;
    E.boff = a.boff[e];
    E.n = static_cast<int>(a.boff[e + 1] - E.boff);
    E.A = a.blocks + a.aoff[e];
    E.idx = a.idx + E.boff;
    E.ni = a.ni[e];
    const bool hyb = MODE == ALG_HYB || MODE == ALG_REC;
    E.d = hyb ? E.n : E.ni;
    const int d = E.d, nb = E.n - E.ni;
    const int nr = (MODE == ALG_HYB || MODE == ALG_REC) ? static_cast<int>(a.goff[e + 1] - a.goff[e]) : 0;
    int nc = 1;
    if (MODE == ALG_HYB) nc = nr + 1;
    if (MODE == ALG_COND) nc = nb + 1;
    const int ncc = min(nc, p.ncc);
    // workspace carve
    double* lu = Wf;
    double* Xs = lu + static_cast<int64_t>(d) * d;
    double* Xls = Xs + static_cast<int64_t>(d) * ncc;
    double* Rs = Xls + static_cast<int64_t>(d) * ncc;
    int* piv = reinterpret_cast<int*>(Rs + static_cast<int64_t>(d) * ncc);
    double* b0h = Ws;
    double* b0l = b0h + static_cast<int64_t>(d) * nc;
    double* X = b0l + static_cast<int64_t>(d) * nc;
    double* Xl = X + static_cast<int64_t>(d) * nc;
    const bool rec = MODE == ALG_REC || MODE == ALG_RECC;
    bool ok = true;
    if (d > 0) {
      ok = block_lu(E, hyb ? E.ni : 0, lu, piv, sv, si);
      if (!ok) {
        if (threadIdx.x == 0) {
          atomicOr(a.status, 2);
          atomicMin(reinterpret_cast<unsigned long long*>(a.bad_elem), static_cast<unsigned long long>(e));
        }
        __syncthreads();
        continue;
      }
      // right-hand sides
      if (MODE == ALG_HYB) {
        for (int t = threadIdx.x; t < d * nc; t += kAT) b0h[t] = 0.0;
        __syncthreads();
        // C_T^T: column r holds row r of the element's constraint slice
        for (int64_t q = a.cptr[a.goff[e]] + threadIdx.x; q < a.cptr[a.goff[e + 1]]; q += kAT)
          b0h[static_cast<int64_t>(a.cent_a[q]) * nc + a.cent_r[q]] = a.cent_v[q];
        for (int i = threadIdx.x; i < d; i += kAT) b0h[static_cast<int64_t>(i) * nc + nr] = a.f[E.boff + E.idx[i]];
      } else if (MODE == ALG_COND) {
        for (int t = threadIdx.x; t < d * nc; t += kAT) {
          const int i = t / nc, c = t % nc;
          b0h[t] = c < nb ? Mget(E, i, E.ni + c) : a.f[E.boff + E.idx[i]];
        }
      } else if (MODE == ALG_REC) {
        // f - C_T^T lambda, exactly accumulated
        for (int i = threadIdx.x; i < d; i += kAT) {
          double hi = a.f[E.boff + E.idx[i]], lo = 0.0;
          for (int64_t q = a.cptr[a.goff[e]]; q < a.cptr[a.goff[e + 1]]; ++q)
            if (a.cent_a[q] == i) dd_fma(hi, lo, -a.cent_v[q], a.lambda[a.mrows[a.goff[e] + a.cent_r[q]]]);
          b0h[i] = hi;
          b0l[i] = lo;
        }
      } else {  // ALG_RECC: f_i - A_ib x_b_local
        for (int i = threadIdx.x; i < d; i += kAT) {
          double hi = a.f[E.boff + E.idx[i]], lo = 0.0;
          for (int j = 0; j < nb; ++j) {
            const int64_t bj = a.bdof_off[e] + j;
            double xb = 0.0;
            for (int64_t q = a.bm_ptr[bj]; q < a.bm_ptr[bj + 1]; ++q) xb += a.bm_w[q] * a.xb[a.bm_ord[q]];
            dd_fma(hi, lo, -Mget(E, i, E.ni + j), xb);
          }
          b0h[i] = hi;
          b0l[i] = lo;
        }
      }
      __syncthreads();
      refined_solve(E, nc, ncc, lu, piv, b0h, rec ? b0l : nullptr, X, Xl, Xs, Xls, Rs, sv,
                    MODE == ALG_COND ? 0x1p-100 : 0x1p-60);
    }
    // epilogues
    if (MODE == ALG_HYB) {
      // H_e(r, q) = sum_(entries of row r) v X(a, q);  g_e(r) = same with column nr
      double* he = a.hbuf + a.hoff[e];
      double* ge = a.gbuf + a.goff[e];
      for (int t = threadIdx.x; t < nr * nc; t += kAT) {
        const int r = t / nc, q = t % nc;
        double hi = 0.0, lo = 0.0;
        for (int64_t z = a.cptr[a.goff[e] + r]; z < a.cptr[a.goff[e] + r + 1]; ++z)
        {
          const int64_t xi = static_cast<int64_t>(a.cent_a[z]) * nc + q;
          dd_fma(hi, lo, a.cent_v[z], X[xi]);
          lo = fma(a.cent_v[z], Xl[xi], lo);
        }
        if (q < nr) he[static_cast<int64_t>(r) * nr + q] = hi + lo;
        else ge[r] = hi + lo;
      }
      // no symmetrize(h_e) (reduction.cpp:316): the element-exact H_e is what the
      // reference's own double-double oracle defines (src/reference.cpp:195-209)
    } else if (MODE == ALG_REC) {
      for (int i = threadIdx.x; i < d; i += kAT) a.x_hat[E.boff + E.idx[i]] = X[i] + Xl[i];
    } else if (MODE == ALG_COND) {
      double* s = a.sbuf + a.soff[e];
      double* fs = a.fsbuf + a.bdof_off[e];
      for (int t = threadIdx.x; t < nb * (nb + 1); t += kAT) {
        const int j = t / (nb + 1), k = t % (nb + 1);
        double hi = k < nb ? Mget(E, E.ni + j, E.ni + k) : a.f[E.boff + E.idx[E.ni + j]], lo = 0.0;
        for (int l = 0; l < d; ++l) {
          const double m = -Mget(E, E.ni + j, l);
          dd_fma(hi, lo, m, X[static_cast<int64_t>(l) * nc + k]);
          lo = fma(m, Xl[static_cast<int64_t>(l) * nc + k], lo);
        }
        if (k < nb) s[static_cast<int64_t>(j) * nb + k] = hi + lo;
        else fs[j] = hi + lo;
      }
    } else {
      for (int i = threadIdx.x; i < d; i += kAT) {
        const int64_t gi = a.ibase[e] + i;
        a.x[a.i_global[gi]] = (X[i] + Xl[i]) / a.i_sign[gi];
      }
    }
    __syncthreads();
  }
}

// triplet keys of H (rows x rows per element) and of g (rows), element order
__global__ void k_alg_hkeys(AlgArgs a, uint64_t* hkeys, int64_t* hsrc, uint64_t* gkeys, int64_t* gsrc) {
  for (int64_t e = blockIdx.x; e < a.ne; e += gridDim.x) {
    const int64_t g0 = a.goff[e];
    const int nr = static_cast<int>(a.goff[e + 1] - g0);
    const int64_t h0 = a.hoff[e];
    for (int t = threadIdx.x; t < nr * nr; t += blockDim.x) {
      const int r = t / nr, q = t % nr;
      hkeys[h0 + t] = static_cast<uint64_t>(a.mrows[g0 + r]) * static_cast<uint64_t>(a.m) + static_cast<uint64_t>(a.mrows[g0 + q]);
      hsrc[h0 + t] = h0 + t;
    }
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
      gkeys[g0 + r] = static_cast<uint64_t>(a.mrows[g0 + r]);
      gsrc[g0 + r] = g0 + r;
    }
  }
}

// triplet keys of S = sum P_b^T S_hat P_b and of f_S (reference order: element,
// i, entry of i, j, entry of j), with the weight products w_i * w_j
__global__ void k_alg_skeys(AlgArgs a, const int64_t* trip_off, const int64_t* ftrip_off, uint64_t* skeys,
                            int64_t* ssrc, double* sw, uint64_t* fkeys, int64_t* fsrc, double* fw) {
  for (int64_t e = blockIdx.x; e < a.ne; e += gridDim.x) {
    const int nb = static_cast<int>(a.boff[e + 1] - a.boff[e]) - a.ni[e];
    const int64_t b0 = a.bdof_off[e];
    int64_t t0 = trip_off[e];
    // enumerate (i, di) pairs; each pairs with all (j, dj)
    const int64_t ent0 = a.bm_ptr[b0], ent1 = a.bm_ptr[b0 + nb];
    const int64_t nent = ent1 - ent0;
    for (int64_t u = threadIdx.x; u < nent * nent; u += blockDim.x) {
      const int64_t qi = ent0 + u / nent, qj = ent0 + u % nent;
      const int bi = a.bm_loc[qi], bj = a.bm_loc[qj];  // local b dofs of the two entries
      skeys[t0 + u] = static_cast<uint64_t>(a.bm_ord[qi]) * static_cast<uint64_t>(a.n_master) +
                      static_cast<uint64_t>(a.bm_ord[qj]);
      ssrc[t0 + u] = a.soff[e] + static_cast<int64_t>(bi) * nb + bj;
      sw[t0 + u] = a.bm_w[qi] * a.bm_w[qj];
    }
    const int64_t f0 = ftrip_off[e];
    for (int64_t u = threadIdx.x; u < nent; u += blockDim.x) {
      const int64_t qi = ent0 + u;
      const int bi = a.bm_loc[qi];
      fkeys[f0 + u] = static_cast<uint64_t>(a.bm_ord[qi]);
      fsrc[f0 + u] = b0 + bi;
      fw[f0 + u] = a.bm_w[qi];
    }
  }
}

__global__ void k_run_heads(int64_t n, const uint64_t* keys, int* head) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t < n) head[t] = (t == 0 || keys[t] != keys[t - 1]) ? 1 : 0;
}

// CSR from sorted unique keys (key = row * ncols + col): run starts, columns, row counts
__global__ void k_run_csr(int64_t n, const uint64_t* keys, const int* head, const int* pos, int64_t ncols,
                          int64_t* run_start, int64_t* cols, int64_t* row_cnt) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= n || !head[t]) return;
  const int z = pos[t];
  run_start[z] = t;
  if (cols) {
    cols[z] = static_cast<int64_t>(keys[t] % static_cast<uint64_t>(ncols));
    atomicAdd(reinterpret_cast<unsigned long long*>(row_cnt + keys[t] / static_cast<uint64_t>(ncols)), 1ull);
  } else {
    row_cnt[z] = static_cast<int64_t>(keys[t]);  // the row of run z (vectors)
  }
}

// values of run z: ordered sum of (w *) src over the run (from_triplets' summation)
__global__ void k_run_sum(int64_t nruns, const int64_t* run_start, const int64_t* src, const double* w,
                          const double* buf, double* out, const int64_t* out_index, int from_zero) {
  const int64_t z = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (z >= nruns) return;
  // from_triplets (csr.cpp:63-69) starts from the first value; the g / f_s
  // vectors start from 0.0 (reduction.cpp:335, :540)
  const int64_t t0 = run_start[z];
  double s = from_zero ? 0.0 : (w ? w[t0] * buf[src[t0]] : buf[src[t0]]);
  for (int64_t t = from_zero ? t0 : t0 + 1; t < run_start[z + 1]; ++t) {
    const double v = buf[src[t]];
    s = s + (w ? w[t] * v : v);
  }
  if (out_index) out[out_index[z]] = s;
  else out[z] = s;
}

}  // namespace

AlgPlan alg_plan(int64_t ne, int dmax, int ncmax) {
  AlgPlan p;
  const int64_t budget = 200 * 1024 / 8;  // doubles of dynamic shared memory
  const int64_t fixed = static_cast<int64_t>(dmax) * dmax + (dmax + 1) / 2 + 1;
  const int64_t per_col = 3 * static_cast<int64_t>(dmax);
  int64_t ncc = per_col > 0 ? (budget - fixed) / per_col : ncmax;
  p.smem = ncc >= 1;
  p.ncc = p.smem ? static_cast<int>(std::min<int64_t>(ncc, ncmax)) : ncmax;
  if (p.ncc < 1) p.ncc = 1;
  p.fast = fixed + per_col * p.ncc;
  p.slow = 4 * static_cast<int64_t>(dmax) * ncmax + 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  int per_sm = 2;
  if (p.smem) per_sm = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4, (226 * 1024) / (p.fast * 8 + 2048))));
  p.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ne, static_cast<int64_t>(sms) * per_sm)));
  return p;
}

int64_t alg_gws_doubles(const AlgPlan& p) { return static_cast<int64_t>(p.grid) * (p.slow + (p.smem ? 0 : p.fast)); }

void launch_alg(const AlgArgs& a, int mode, const AlgPlan& p, double* gws, cudaStream_t st) {
  const size_t dyn = p.smem ? static_cast<size_t>(p.fast) * 8 : 0;
  auto go = [&](auto kern) {
    if (p.smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
    kern<<<p.grid, kAT, dyn, st>>>(a, gws, p);
  };
  switch (mode) {
    case ALG_HYB: go(k_alg<ALG_HYB>); break;
    case ALG_REC: go(k_alg<ALG_REC>); break;
    case ALG_COND: go(k_alg<ALG_COND>); break;
    default: go(k_alg<ALG_RECC>); break;
  }
  count_launch();
}

void launch_alg_hkeys(const AlgArgs& a, uint64_t* hkeys, int64_t* hsrc, uint64_t* gkeys, int64_t* gsrc, cudaStream_t st) {
  const int grid = static_cast<int>(a.ne < 4096 ? (a.ne > 0 ? a.ne : 1) : 4096);
  k_alg_hkeys<<<grid, 128, 0, st>>>(a, hkeys, hsrc, gkeys, gsrc);
  count_launch();
}

void launch_alg_skeys(const AlgArgs& a, const int64_t* trip_off, const int64_t* ftrip_off, uint64_t* skeys,
                      int64_t* ssrc, double* sw, uint64_t* fkeys, int64_t* fsrc, double* fw, cudaStream_t st) {
  const int grid = static_cast<int>(a.ne < 4096 ? (a.ne > 0 ? a.ne : 1) : 4096);
  k_alg_skeys<<<grid, 128, 0, st>>>(a, trip_off, ftrip_off, skeys, ssrc, sw, fkeys, fsrc, fw);
  count_launch();
}

void launch_run_heads(int64_t n, const uint64_t* keys, int* head, cudaStream_t st) {
  if (n <= 0) return;
  k_run_heads<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, keys, head);
  count_launch();
}

void launch_run_csr(int64_t n, const uint64_t* keys, const int* head, const int* pos, int64_t ncols, int64_t* run_start,
                    int64_t* cols, int64_t* row_cnt, cudaStream_t st) {
  if (n <= 0) return;
  k_run_csr<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, keys, head, pos, ncols, run_start, cols, row_cnt);
  count_launch();
}

void launch_run_sum(int64_t nruns, const int64_t* run_start, const int64_t* src, const double* w, const double* buf,
                    double* out, const int64_t* out_index, int from_zero, cudaStream_t st) {
  if (nruns <= 0) return;
  k_run_sum<<<static_cast<unsigned>((nruns + 255) / 256), 256, 0, st>>>(nruns, run_start, src, w, buf, out, out_index,
                                                                        from_zero);
  count_launch();
}

}  // namespace hdr

// ------------------------------------------------------------ vector helpers
// (recover_hybrid's x = (P^T P)^-1 P^T x_hat: column sums of squares, scaling,
// and the CG of reduction.cpp:405-444 for a non-diagonal Gram matrix)
namespace hdr {
namespace {

__global__ void k_row_sumsq(int64_t nrows, const int64_t* ro, const double* v, double* out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= nrows) return;
  double s = 0.0;
  for (int64_t k = ro[r]; k < ro[r + 1]; ++k) s = s + v[k] * v[k];
  out[r] = s;
}

__global__ void k_vec_op(int64_t n, int op, double a, const double* x, const double* y, double* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  switch (op) {
    case 0: out[i] = x[i] * y[i]; break;          // elementwise product
    case 1: out[i] = out[i] + a * x[i]; break;    // axpy
    case 2: out[i] = x[i] + a * out[i]; break;    // out = x + a out
    case 3: out[i] = x[i] == 0.0 ? 0.0 : 1.0 / x[i]; break;
    default: break;
  }
}

// deterministic two-level dot product: fixed 1024 partial sums, then one block
__global__ void k_dot_partial(int64_t n, const double* x, const double* y, double* part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s = fma(x[i], y[i], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_dot_final(int nparts, const double* part, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

}  // namespace

void launch_row_sumsq(int64_t nrows, const int64_t* ro, const double* v, double* out, cudaStream_t st) {
  if (nrows <= 0) return;
  k_row_sumsq<<<static_cast<unsigned>((nrows + 255) / 256), 256, 0, st>>>(nrows, ro, v, out);
  count_launch();
}

void launch_vec_op(int64_t n, int op, double a, const double* x, const double* y, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_vec_op<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, op, a, x, y, out);
  count_launch();
}

void launch_dot(int64_t n, const double* x, const double* y, double* part, double* out, cudaStream_t st) {
  k_dot_partial<<<1024, 256, 0, st>>>(n, x, y, part);
  k_dot_final<<<1, 256, 0, st>>>(1024, part, out);
  count_launch(2);
}

}  // namespace hdr

namespace hdr {
namespace {
template <class T>
__global__ void k_gather(int64_t n, const int64_t* pos, const T* in, T* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t < n) out[t] = in[pos[t]];
}
__global__ void k_scatter(int64_t n, const int64_t* index, const double* v, double* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t < n) out[index[t]] = v[t];
}
__global__ void k_iota(int64_t n, int64_t* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t < n) out[t] = t;
}
}  // namespace

void launch_gather_i64(int64_t n, const int64_t* pos, const int64_t* in, int64_t* out, cudaStream_t st) {
  if (n <= 0) return;
  k_gather<int64_t><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, pos, in, out);
  count_launch();
}
void launch_gather_f64(int64_t n, const int64_t* pos, const double* in, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_gather<double><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, pos, in, out);
  count_launch();
}
void launch_scatter(int64_t n, const int64_t* index, const double* v, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_scatter<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, index, v, out);
  count_launch();
}
void launch_iota(int64_t n, int64_t* out, cudaStream_t st) {
  if (n <= 0) return;
  k_iota<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, out);
  count_launch();
}
}  // namespace hdr

namespace hdr {
namespace {
// a_ij = a_ji = 0.5 (a_ij + a_ji) on a structurally symmetric CSR matrix with
// sorted columns; each pair is handled by its upper-triangle entry's thread.
template <class IDX>
__global__ void k_csr_symmetrize(int64_t nrows, const int64_t* ro, const IDX* ci, double* v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nrows) return;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const int64_t j = ci[k];
    if (j <= i) continue;
    int64_t lo = ro[j], hi = ro[j + 1] - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(ci[mid]) < i) lo = mid + 1;
      else hi = mid;
    }
    if (lo > hi || static_cast<int64_t>(ci[lo]) != i) continue;  // structurally unsymmetric entry: left alone
    const double s = 0.5 * (v[k] + v[lo]);
    v[k] = s;
    v[lo] = s;
  }
}
}  // namespace

void launch_csr_symmetrize64(int64_t nrows, const int64_t* ro, const int64_t* ci, double* v, cudaStream_t st) {
  if (nrows <= 0) return;
  k_csr_symmetrize<int64_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v);
  count_launch();
}
void launch_csr_symmetrize32(int64_t nrows, const int64_t* ro, const int32_t* ci, double* v, cudaStream_t st) {
  if (nrows <= 0) return;
  k_csr_symmetrize<int32_t><<<static_cast<unsigned>((nrows + 127) / 128), 128, 0, st>>>(nrows, ro, ci, v);
  count_launch();
}
}  // namespace hdr
