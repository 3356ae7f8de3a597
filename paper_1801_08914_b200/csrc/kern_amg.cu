// Smoothed-aggregation AMG and symmetric Gauss-Seidel on the device (SURVEY.md
// §8(f) f1): amg_setup / v_cycle (src/amg.cpp:9-266) and ssgs_setup /
// gauss_seidel_forward / gauss_seidel_backward (src/solvers.cpp:60-107), the
// reference's default preconditioner of the reduced solve (driver.hpp:39).
//
// Everything with arithmetic runs on the device and rounds exactly like the
// reference, so for the same input matrix the hierarchy and every V-cycle /
// SGS application are bit-identical to it:
//  - row-local setup steps (diagonal, strength graph, filtered matrix with
//    lumping, tentative / smoothed prolongator) are one thread per row in the
//    reference's storage order;
//  - the power iteration (spectral_bound) uses the reference's xorshift start
//    vector and sequential norms (one thread: the sums are order-dependent);
//  - triple_product (csr.cpp:132-175) is exact per row: a warp collects the
//    row's column set in a shared-memory hash (symbolic pass, sorted), then
//    one thread per row accumulates every product term in the reference's
//    (kr, ia, ip) order into its sorted position;
//  - transpose places entries by atomics and sorts each row by column (the
//    reference's order), no arithmetic;
//  - Gauss-Seidel sweeps are sync-free triangular solves: warps take rows in
//    sweep order from an atomic ticket, wait (acquire) on the ready flags of the
//    rows they depend on, and lane 0 forms the row's sum in storage order;
//    old / new iterates are separate arrays, so the reference's in-place
//    semantics hold for any sparsity pattern.  A warp only ever waits on rows
//    with earlier tickets, all held by running warps: no deadlock;
//  - the coarsest level is factored / solved by the one-CTA dense LU of
//    dense_cta.cuh.
// The one serial step, aggregate() (amg.cpp:48-83: a greedy pass whose result
// depends on visiting the nodes in index order), runs on the host in C++ over
// the device-built strength graph.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "amg.hpp"
#include "capi_util.hpp"
#include "dense_cta.cuh"
#include "kernels.hpp"
#include "runs.hpp"

namespace hdr {

namespace cg = cooperative_groups;

namespace {

constexpr int kT = 256;
constexpr size_t kCtaSweepSmem = 200 * 1024;  // one-CTA sweeps: new iterate + the widest level's products

inline unsigned nblk(int64_t n, int t = kT) { return static_cast<unsigned>(std::max<int64_t>(1, (n + t - 1) / t)); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- row-local steps

// diagonal (amg.cpp:14-23): the stored a_ii (0 if absent)
__global__ void k_diag(int64_t n, const int64_t* ro, const int32_t* ci, const double* v, double* d) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double x = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k)
    if (ci[k] == i) x = v[k];
  d[i] = x;
}

// checked_inv_diag (amg.cpp:159-166) / positive_inv_diag (solvers.cpp:32-44):
// 1 / d, smallest row with d <= 0 (or NaN) into *bad
__global__ void k_inv_checked(int64_t n, double* d, unsigned long long* bad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double x = d[i];
  if (!(x > 0.0)) atomicMin(bad, static_cast<unsigned long long>(i));
  d[i] = 1.0 / x;
}

__device__ __forceinline__ bool strong(double aij, double di, double dj, double theta) {
  const double dd = __dmul_rn(di, dj);
  return dd > 0.0 && fabs(aij) >= __dmul_rn(theta, sqrt(dd));
}

// strength_graph (amg.cpp:27-44)
template <bool FILL>
__global__ void k_strength(int64_t n, const int64_t* ro, const int32_t* ci, const double* v, const double* d,
                           double theta, int64_t* cnt, const int64_t* sro, int32_t* sci) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int64_t c = 0, pos = FILL ? sro[i] : 0;
  const double di = d[i];
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const int j = ci[k];
    if (j == i || !strong(v[k], di, d[j], theta)) continue;
    if (FILL) sci[pos++] = j;
    ++c;
  }
  if (!FILL) cnt[i] = c;
}

// tentative prolongator (amg.cpp:222-232): column agg[i], 1 / sqrt(|aggregate|)
__global__ void k_agg_size(int64_t n, const int32_t* agg, int* size) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) atomicAdd(size + agg[i], 1);
}
__global__ void k_ptent(int64_t n, const int32_t* agg, const int* size, double* pv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) pv[i] = 1.0 / sqrt(static_cast<double>(size[agg[i]]));
}

// filtered_matrix (amg.cpp:116-143): diagonal + strong couplings, the weak ones
// lumped into the diagonal (row order) unless that would make it non-positive
template <bool FILL>
__global__ void k_filter(int64_t n, const int64_t* ro, const int32_t* ci, const double* v, const int64_t* sro,
                         const int32_t* sci, int64_t* cnt, const int64_t* fro, int32_t* fci, double* fv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int64_t s = sro[i];
  const int64_t se = sro[i + 1];
  int64_t pos = FILL ? fro[i] : 0, diag_pos = -1, c = 0;
  double lumped = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const int j = ci[k];
    while (s < se && sci[s] < j) ++s;  // strength row i: a sorted subset of row i's columns
    const bool keep = j == i || (s < se && sci[s] == j);
    if (keep) {
      if (FILL) {
        if (j == i) diag_pos = pos;
        fci[pos] = j;
        fv[pos] = v[k];
        ++pos;
      }
      ++c;
    } else {
      lumped = __dadd_rn(lumped, v[k]);
    }
  }
  if (FILL) {
    if (diag_pos >= 0 && __dadd_rn(fv[diag_pos], lumped) > 0.0) fv[diag_pos] = __dadd_rn(fv[diag_pos], lumped);
  } else {
    cnt[i] = c;
  }
}

__global__ void k_scale_inplace(int64_t n, double* w, const double* d) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) w[i] = __dmul_rn(w[i], d[i]);
}
__global__ void k_div_into(int64_t n, const double* w, double norm, double* v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = w[i] / norm;
}
// sequential sum of squares (the reference's loop order) and its square root:
// the CTA stages chunks of squares in shared memory (coalesced loads, the
// products in parallel), one thread adds them in order
__global__ void __launch_bounds__(1024) k_seq_norm(int64_t n, const double* w, double* out) {
  constexpr int CH = 2048;
  __shared__ double sq[2][CH];
  double s = 0.0;
  int buf = 0;
  for (int64_t i = threadIdx.x; i < CH && i < n; i += blockDim.x) sq[0][i] = __dmul_rn(w[i], w[i]);
  __syncthreads();
  for (int64_t c0 = 0; c0 < n; c0 += CH, buf ^= 1) {
    const int64_t c1 = c0 + CH;  // next chunk staged by the other threads while thread 0 adds this one
    if (threadIdx.x == 0) {
      const int m = static_cast<int>(n - c0 < CH ? n - c0 : CH);
      for (int j = 0; j < m; ++j) s = __dadd_rn(s, sq[buf][j]);
    } else {
      for (int64_t i = c1 + threadIdx.x - 1; i < c1 + CH && i < n; i += blockDim.x - 1)
        sq[buf ^ 1][i - c1] = __dmul_rn(w[i], w[i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sqrt(s);
}

// smooth_prolongator (amg.cpp:146-157): P = P_tent - omega D^-1 AP on AP's
// pattern (it contains column agg[i]: the diagonal of the filtered row);
// fl(-omega d_i) * ap, plus the tentative entry (a two-term from_triplets sum)
__global__ void k_smooth(int64_t n, const int64_t* ro, const int32_t* ci, const double* ap, const int32_t* agg,
                         const double* pt, const double* dinv, double omega, double* pv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double sc = __dmul_rn(-omega, dinv[i]);
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    double x = __dmul_rn(sc, ap[k]);
    if (ci[k] == agg[i]) x = __dadd_rn(pt[i], x);
    pv[k] = x;
  }
}

// ---------------------------------------------------------------- transpose (csr.cpp:89-107)

__global__ void k_col_count(int64_t nnz, const int32_t* ci, int64_t* cnt) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < nnz) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + ci[k]), 1ull);
}
__global__ void k_transpose_place(int64_t n, const int64_t* ro, const int32_t* ci, const double* v,
                                  unsigned long long* cursor, int32_t* tci, double* tv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const int64_t pos = static_cast<int64_t>(atomicAdd(cursor + ci[k], 1ull));
    tci[pos] = static_cast<int32_t>(i);
    tv[pos] = v[k];
  }
}
// each row of the transpose in increasing column order (insertion sort; rows are short)
__global__ void k_row_sort(int64_t n, const int64_t* ro, int32_t* ci, double* v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t a = ro[i], b = ro[i + 1];
  for (int64_t k = a + 1; k < b; ++k) {
    const int32_t c = ci[k];
    const double x = v[k];
    int64_t j = k - 1;
    while (j >= a && ci[j] > c) {
      ci[j + 1] = ci[j];
      v[j + 1] = v[j];
      --j;
    }
    ci[j + 1] = c;
    v[j + 1] = x;
  }
}

// ---------------------------------------------------------------- triple product

constexpr int kEmpty = 0x7fffffff;
constexpr int kTpWarps = 4;  // warps per CTA of the symbolic pass

// the row's candidate count (upper bound of its column count)
__global__ void k_tp_cand(int64_t nr, const int64_t* rro, const int32_t* rci, const int64_t* aro, const int32_t* aci,
                          const int64_t* pro, int64_t* cand) {
  const int64_t I = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (I >= nr) return;
  int64_t c = 0;
  for (int64_t kr = rro[I]; kr < rro[I + 1]; ++kr) {
    const int ka = rci[kr];
    for (int64_t ia = aro[ka]; ia < aro[ka + 1]; ++ia) {
      const int jp = aci[ia];
      c += pro[jp + 1] - pro[jp];
    }
  }
  cand[I] = c;
}

// gather_row (csr.cpp:113-130): the sorted column set of row I of R A P; a warp
// per row, open-addressing hash of `cap` (power of two) slots per warp (shared
// memory, or global scratch `gtab` when it does not fit), then a bitonic sort
template <bool FILL>
__global__ void k_tp_symbolic(int64_t nr, const int64_t* rro, const int32_t* rci, const int64_t* aro,
                              const int32_t* aci, const int64_t* pro, const int32_t* pci, int cap, int* gtab,
                              int64_t* cnt, const int64_t* oro, int32_t* oci) {
  extern __shared__ int stab[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = blockIdx.x * static_cast<int64_t>(kTpWarps) + wib;
  int* tab = gtab ? gtab + gw * cap : stab + wib * cap;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kTpWarps;
  for (int64_t I = gw; I < nr; I += nwarps) {
    for (int s = lane; s < cap; s += 32) tab[s] = kEmpty;
    __syncwarp();
    for (int64_t kr = rro[I]; kr < rro[I + 1]; ++kr) {
      const int ka = rci[kr];
      for (int64_t ia = aro[ka] + lane; ia < aro[ka + 1]; ia += 32) {
        const int jp = aci[ia];
        for (int64_t ip = pro[jp]; ip < pro[jp + 1]; ++ip) {
          const int c = pci[ip];
          unsigned h = (static_cast<unsigned>(c) * 2654435761u) & (cap - 1);
          while (true) {
            const int old = atomicCAS(tab + h, kEmpty, c);
            if (old == kEmpty || old == c) break;
            h = (h + 1) & (cap - 1);
          }
        }
      }
    }
    __syncwarp();
    // bitonic sort of the table (empties sort last)
    for (int k = 2; k <= cap; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = lane; t < cap; t += 32) {
          const int u = t ^ j;
          if (u > t) {
            const int x = tab[t], y = tab[u];
            const bool up = (t & k) == 0;
            if ((x > y) == up) {
              tab[t] = y;
              tab[u] = x;
            }
          }
        }
        __syncwarp();
      }
    int c = 0;
    for (int t = lane; t < cap; t += 32) c += tab[t] != kEmpty;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (FILL) {
      const int64_t base = oro[I];
      for (int t = lane; t < c; t += 32) oci[base + t] = tab[t];
    } else if (lane == 0) {
      cnt[I] = c;
    }
    __syncwarp();
  }
}

// numeric pass (csr.cpp:150-167): one thread per row, every term in the
// reference's order, accumulated at its column's sorted position
__global__ void k_tp_numeric(int64_t nr, const int64_t* rro, const int32_t* rci, const double* rv, const int64_t* aro,
                             const int32_t* aci, const double* av, const int64_t* pro, const int32_t* pci,
                             const double* pv, const int64_t* oro, const int32_t* oci, double* ov) {
  const int64_t I = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (I >= nr) return;
  const int64_t o0 = oro[I], o1 = oro[I + 1];
  for (int64_t k = o0; k < o1; ++k) ov[k] = 0.0;
  for (int64_t kr = rro[I]; kr < rro[I + 1]; ++kr) {
    const int ka = rci[kr];
    const double r = rv[kr];
    for (int64_t ia = aro[ka]; ia < aro[ka + 1]; ++ia) {
      const int jp = aci[ia];
      const double ra = __dmul_rn(r, av[ia]);
      for (int64_t ip = pro[jp]; ip < pro[jp + 1]; ++ip) {
        const int c = pci[ip];
        int64_t lo = o0, hi = o1 - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (oci[mid] < c) lo = mid + 1;
          else hi = mid;
        }
        ov[lo] = __dadd_rn(ov[lo], __dmul_rn(ra, pv[ip]));
      }
    }
  }
}

// ---------------------------------------------------------------- V-cycle pieces

// gauss_seidel_forward / _backward (solvers.cpp:75-107) as a sync-free sweep:
// zin = the iterate before the sweep (nullptr: zeros), zout = after it
template <bool FWD>
__global__ void __launch_bounds__(kT) k_gs_sweep(int64_t n, const int64_t* ro, const int32_t* ci, const double* v,
                                                 const double* r, const double* zin, double* zout, int* flags,
                                                 int epoch, unsigned long long* ticket, int* status, const int* order) {
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= static_cast<unsigned long long>(n)) return;
    const int64_t i = order[t];  // rows in level order: every dependency has a smaller ticket
    const int64_t a = ro[i], b = ro[i + 1];
    double s = r[i], diag = 0.0;
    for (int64_t base = a; base < b; base += 32) {
      const int64_t k = base + lane;
      int c = -1;
      double vk = 0.0, zk = 0.0;
      if (k < b) {
        c = ci[k];
        vk = v[k];
        const bool dep = FWD ? c < i : c > i;  // already updated in this sweep
        if (dep) {
          while (ld_acquire(flags + c) != epoch) __nanosleep(64);
          zk = __ldcg(zout + c);
        } else if (c != i) {
          zk = zin ? zin[c] : 0.0;
        }
      }
      const int m = static_cast<int>(b - base < 32 ? b - base : 32);
      for (int q = 0; q < m; ++q) {  // storage order
        const int cq = __shfl_sync(0xffffffffu, c, q);
        const double vq = __shfl_sync(0xffffffffu, vk, q);
        const double zq = __shfl_sync(0xffffffffu, zk, q);
        if (cq == i) diag = vq;
        else s = __dsub_rn(s, __dmul_rn(vq, zq));
      }
    }
    if (lane == 0) {
      if (diag == 0.0) atomicOr(status, 1);  // ZeroDiagonal (setup checks make this unreachable)
      zout[i] = s / diag;
      st_release(flags + i, epoch);
    }
    __syncwarp();
  }
}

// one row of a Gauss-Seidel sweep by one warp: lanes load 32 entries at a time
// and form the products (dependencies from znew, the rest from zold or 0),
// lane 0 subtracts them in storage order (the reference's roundings)
template <bool FWD, class ZNEW>
__device__ __forceinline__ void gs_row(int i, const int64_t* ro, const int32_t* ci, const double* v, const double* r,
                                       const double* zold, ZNEW znew_at, double* zdst, int* status) {
  const int lane = threadIdx.x & 31;
  const int64_t a = ro[i], b = ro[i + 1];
  double s = r[i], diag = 0.0;
  for (int64_t base = a; base < b; base += 32) {
    const int64_t k = base + lane;
    int c = -1;
    double p = 0.0;
    if (k < b) {
      c = ci[k];
      const double vk = v[k];
      if (c == i) {
        p = vk;  // the diagonal travels in p
      } else {
        const bool dep = FWD ? c < i : c > i;
        p = __dmul_rn(vk, dep ? znew_at(c) : (zold ? zold[c] : 0.0));
      }
    }
    const int m = static_cast<int>(b - base < 32 ? b - base : 32);
    for (int q = 0; q < m; ++q) {
      const int cq = __shfl_sync(0xffffffffu, c, q);
      const double pq = __shfl_sync(0xffffffffu, p, q);
      if (cq == i) diag = pq;
      else s = __dsub_rn(s, pq);
    }
  }
  if (lane == 0) {
    if (diag == 0.0) atomicOr(status, 1);
    *zdst = s / diag;
  }
}

// sweep of a small matrix in one CTA: the new iterate in shared memory, rows in
// level order, per level (1) every product of the level's rows formed in
// parallel into a shared buffer (the diagonal's slot holds +0: subtracting it
// leaves every sum unchanged, so the fold equals the reference's, which skips
// it), (2) one thread per row subtracts its products in storage order
template <bool FWD>
__global__ void __launch_bounds__(512) k_gs_cta(int n, const int64_t* ro, const int32_t* ci, const double* v,
                                                const double* r, const double* zin, double* zout, const int* order,
                                                const int* bat, int nbat, const int64_t* eoff, int* status) {
  extern __shared__ double zs[];  // n new values, then the products of one batch of rows
  double* pb = zs + ((n + 1) & ~1);
  __shared__ double dg[512];
  __shared__ int dpos[512];  // the row's split point: entries before it, resp. from it, are folded
  __shared__ int ntail[512];  // forward sweep from zero: some skipped term is -0 (v has its sign bit set)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // Only the terms of the dependencies need the level order.  Forward sweep from
  // zero (zin == nullptr): the terms after the diagonal are v * 0 = +-0, which
  // leave every running sum unchanged except -0 - (-0) = +0: they reduce to a
  // sign fix-up.  Backward sweep: the terms before the diagonal use zin only, so
  // their part of the ordered fold runs for every row up front, in parallel.
  const bool fwd_zero = FWD && zin == nullptr;
  if (!FWD) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double sacc = r[i];
      for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
        const int c = ci[k];
        if (c >= i) break;  // columns ascending: the rest are the diagonal and the dependencies
        sacc = __dsub_rn(sacc, __dmul_rn(v[k], zin ? zin[c] : 0.0));
      }
      zs[i] = sacc;  // the row's partial sum until the row itself is swept
    }
    __syncthreads();
  }
  // batches: rows [bat[j], bat[j + 1]) of one level, at most 512 rows and the buffer's entries
  for (int j = 0; j < nbat; ++j) {
    const int t0 = __ldg(bat + j), t1 = __ldg(bat + j + 1);
    const int64_t e0 = __ldg(eoff + t0);
    for (int t = t0 + warp; t < t1; t += nw) {  // products, warp per row
      const int i = order[t];
      const int64_t a = ro[i], b = ro[i + 1], dst = eoff[t] - e0 - a;
      bool neg = false;
      for (int64_t k = a + lane; k < b; k += 32) {
        const int c = ci[k];
        const double vk = v[k];
        double p = 0.0;
        if (c == i) {
          dg[t - t0] = vk;
          dpos[t - t0] = static_cast<int>(k - a);
        } else if (FWD ? c < i : c > i) {
          p = __dmul_rn(vk, zs[c]);
        } else if (fwd_zero) {
          neg = neg || signbit(vk);
        } else {
          p = __dmul_rn(vk, zin ? zin[c] : 0.0);
        }
        pb[dst + k] = p;
      }
      neg = __any_sync(0xffffffffu, neg);
      if (lane == 0) ntail[t - t0] = neg ? 1 : 0;
    }
    __syncthreads();
    for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {  // folds, thread per row
      const int i = order[t];
      const int64_t q0 = eoff[t] - e0, q1 = eoff[t + 1] - e0, qd = q0 + dpos[t - t0];
      double sacc;
      if (FWD) {
        sacc = r[i];
        const int64_t qe = fwd_zero ? qd : q1;  // the diagonal's slot holds +0: stopping there is exact
#pragma unroll 8
        for (int64_t q = q0; q < qe; ++q) sacc = __dsub_rn(sacc, pb[q]);
        if (fwd_zero && ntail[t - t0] && sacc == 0.0) sacc = 0.0;  // -0 - (-0) = +0
      } else {
        sacc = zs[i];  // r_i minus the terms before the diagonal
#pragma unroll 8
        for (int64_t q = qd + 1; q < q1; ++q) sacc = __dsub_rn(sacc, pb[q]);
      }
      const double d = dg[t - t0];
      if (d == 0.0) atomicOr(status, 1);
      zs[i] = sacc / d;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) zout[i] = zs[i];
}

// sweep of a larger matrix: a cooperative grid, warp per row, a grid barrier
// between levels (the new iterate in global memory, read through L2)
template <bool FWD>
__global__ void __launch_bounds__(512) k_gs_coop(int n, const int64_t* ro, const int32_t* ci, const double* v,
                                                 const double* r, const double* zin, double* zout,
                                                 const int* order, const int* lvl, int nlev, int* status) {
  cg::grid_group grid = cg::this_grid();
  const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  for (int L = 0; L < nlev; ++L) {
    for (int t = lvl[L] + gw; t < lvl[L + 1]; t += nw) {
      const int i = order[t];
      gs_row<FWD>(i, ro, ci, v, r, zin, [&](int c) { return __ldcg(zout + c); }, zout + i, status);
    }
    grid.sync();
  }
}

// dependency depth of every row in a forward (j < i) / backward (j > i) sweep:
// one Jacobi step of lev_i = max over dependencies of lev_j + 1 (monotone from
// zero; converged after as many steps as the longest chain)
template <bool FWD>
__global__ void k_level_iter(int64_t n, const int64_t* ro, const int32_t* ci, const int* lin, int* lout, int* changed) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int lv = 0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) {
    const int c = ci[k];
    if (FWD ? c < i : c > i) lv = max(lv, lin[c] + 1);
  }
  lout[i] = lv;
  if (lv != lin[i]) *changed = 1;
}

// residual = r - A z (v_cycle: spmv, then r_i - residual_i)
__global__ void k_resid(int64_t n, const int64_t* ro, const int32_t* ci, const double* v, const double* z,
                        const double* r, double* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(v[k], z[ci[k]]));
  out[i] = __dsub_rn(r[i], s);
}
// z += P cz (correction = spmv(P, coarse_z), then z_i + correction_i)
__global__ void k_prolong_add(int64_t n, const int64_t* ro, const int32_t* ci, const double* v, const double* cz,
                              double* z) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(v[k], cz[ci[k]]));
  z[i] = __dadd_rn(z[i], s);
}
__global__ void k_spmv(int64_t n, const int64_t* ro, const int32_t* ci, const double* v, const double* x, double* y) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ci[k]]));
  y[i] = s;
}

// coarsest level: to_dense + lu_factor (one CTA), then lu_solve per apply
__global__ void __launch_bounds__(256) k_coarse_factor(int64_t n, const int64_t* ro, const int32_t* ci,
                                                       const double* v, double* lu, int* piv, int* status) {
  __shared__ double red[32];
  __shared__ int ired[1];
  const int nn = static_cast<int>(n);
  for (int t = threadIdx.x; t < nn * nn; t += blockDim.x) lu[t] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < nn; i += blockDim.x)
    for (int64_t k = ro[i]; k < ro[i + 1]; ++k) lu[i * nn + ci[k]] = __dadd_rn(lu[i * nn + ci[k]], v[k]);
  __syncthreads();
  if (!cta_lu_factor(lu, nn, piv, red, ired) && threadIdx.x == 0) status[0] = 1;
}
// lu_solve (dense.cpp:99-120) with one CTA, z in shared memory: the forward
// sweep parallel over the rows below each pivot (each entry sees the serial
// sequence of updates), the back substitution row by row with the row's
// products formed in parallel and summed by one thread in the serial order
__global__ void __launch_bounds__(1024) k_coarse_solve(int n, const double* lu, const int* piv, const double* r,
                                                       double* z) {
  extern __shared__ double zs[];  // n, then n products
  double* pr = zs + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) zs[i] = r[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < n; ++k) {
      const int p = piv[k];
      if (p != k) {
        const double t = zs[k];
        zs[k] = zs[p];
        zs[p] = t;
      }
    }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double xk = zs[k];
    if (xk != 0.0)
      for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x)
        zs[i] = __dsub_rn(zs[i], __dmul_rn(lu[static_cast<int64_t>(i) * n + k], xk));
    __syncthreads();
  }
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1 + threadIdx.x; j < n; j += blockDim.x) pr[j] = __dmul_rn(lu[static_cast<int64_t>(i) * n + j], zs[j]);
    __syncthreads();
    if (threadIdx.x == 0) {
      double sacc = zs[i];
      for (int j = i + 1; j < n; ++j) sacc = __dsub_rn(sacc, pr[j]);
      zs[i] = sacc / lu[static_cast<int64_t>(i) * n + i];
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) z[i] = zs[i];
}

__global__ void k_fill_i64(int64_t n, int64_t* a, int64_t start) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) a[i] = start + i;
}
__global__ void k_i64_to_i32(int64_t n, const int64_t* a, int32_t* b) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) b[i] = static_cast<int32_t>(a[i]);
}

// ---------------------------------------------------------------- host helpers

void offsets_from_counts(DBuf<int64_t>& cnt_then_ro, int64_t n, cudaStream_t st, int64_t* total) {
  // cnt has n + 1 slots, the last one 0: the exclusive scan is the offset array
  DBuf<int64_t> out;
  out.alloc(n + 1);
  dev_scan(cnt_then_ro.p, out.p, n + 1, st);
  std::swap(cnt_then_ro.p, out.p);
  std::swap(cnt_then_ro.n, out.n);
  CK(cudaMemcpyAsync(total, cnt_then_ro.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

void dev_transpose(const DCsr& a, DCsr& t, cudaStream_t st) {
  t.n = a.ncols;
  t.ncols = a.n;
  t.nnz = a.nnz;
  t.ro.alloc(t.n + 1);
  CK(cudaMemsetAsync(t.ro.p, 0, (t.n + 1) * 8, st));
  if (a.nnz) k_col_count<<<nblk(a.nnz), kT, 0, st>>>(a.nnz, a.ci.p, t.ro.p);
  int64_t tot = 0;
  offsets_from_counts(t.ro, t.n, st, &tot);
  t.ci.alloc(a.nnz);
  t.v.alloc(a.nnz);
  DBuf<int64_t> cur;
  cur.alloc(t.n + 1);
  CK(cudaMemcpyAsync(cur.p, t.ro.p, (t.n + 1) * 8, cudaMemcpyDeviceToDevice, st));
  k_transpose_place<<<nblk(a.n), kT, 0, st>>>(a.n, a.ro.p, a.ci.p, a.v.p,
                                              reinterpret_cast<unsigned long long*>(cur.p), t.ci.p, t.v.p);
  k_row_sort<<<nblk(t.n), kT, 0, st>>>(t.n, t.ro.p, t.ci.p, t.v.p);
  count_launch(a.nnz ? 3 : 2);
}

// triple_product (csr.cpp:132-175), exact
void dev_triple(const DCsr& r, const DCsr& a, const DCsr& p, DCsr& out, cudaStream_t st) {
  if (r.ncols != a.n || a.ncols != p.n)
    throw StatusError(HDR_DIMENSION_MISMATCH, "triple_product: dimension chain R.ncols = A.nrows, A.ncols = P.nrows violated");
  out.n = r.n;
  out.ncols = p.ncols;
  DBuf<int64_t> cand;
  cand.alloc(std::max<int64_t>(1, r.n));
  int64_t maxc = 0;
  if (r.n) {
    k_tp_cand<<<nblk(r.n), kT, 0, st>>>(r.n, r.ro.p, r.ci.p, a.ro.p, a.ci.p, p.ro.p, cand.p);
    count_launch();
    std::vector<int64_t> hc(static_cast<size_t>(r.n));
    CK(cudaMemcpyAsync(hc.data(), cand.p, r.n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t x : hc) maxc = std::max(maxc, x);
  }
  const int64_t need = std::max<int64_t>(1, std::min<int64_t>(maxc, p.ncols));
  int cap = 32;
  while (cap < 2 * need) cap <<= 1;
  const size_t smem = static_cast<size_t>(cap) * kTpWarps * sizeof(int);
  const bool in_smem = smem <= 96 * 1024;
  const int64_t nwb = std::min<int64_t>(nblk(r.n, kTpWarps), 148 * 8);
  DBuf<int> gtab;
  if (!in_smem) gtab.alloc(static_cast<size_t>(nwb) * kTpWarps * cap);
  const size_t dyn = in_smem ? smem : 0;
  if (in_smem && dyn > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_tp_symbolic<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
    CK(cudaFuncSetAttribute(k_tp_symbolic<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
  }
  out.ro.alloc(out.n + 1);
  CK(cudaMemsetAsync(out.ro.p, 0, (out.n + 1) * 8, st));
  if (r.n)
    k_tp_symbolic<false><<<static_cast<unsigned>(nwb), 32 * kTpWarps, dyn, st>>>(
        r.n, r.ro.p, r.ci.p, a.ro.p, a.ci.p, p.ro.p, p.ci.p, cap, in_smem ? nullptr : gtab.p, out.ro.p, nullptr,
        nullptr);
  offsets_from_counts(out.ro, out.n, st, &out.nnz);
  out.ci.alloc(out.nnz);
  out.v.alloc(out.nnz);
  if (r.n) {
    k_tp_symbolic<true><<<static_cast<unsigned>(nwb), 32 * kTpWarps, dyn, st>>>(
        r.n, r.ro.p, r.ci.p, a.ro.p, a.ci.p, p.ro.p, p.ci.p, cap, in_smem ? nullptr : gtab.p, nullptr, out.ro.p,
        out.ci.p);
    k_tp_numeric<<<nblk(r.n, 128), 128, 0, st>>>(r.n, r.ro.p, r.ci.p, r.v.p, a.ro.p, a.ci.p, a.v.p, p.ro.p, p.ci.p,
                                                  p.v.p, out.ro.p, out.ci.p, out.v.p);
    count_launch(3);
  }
}

// aggregate (amg.cpp:48-83) on the host: the greedy pass visits nodes in index order
int64_t host_aggregate(const std::vector<int64_t>& sro, const std::vector<int32_t>& sci, std::vector<int32_t>& agg) {
  const int64_t n = static_cast<int64_t>(sro.size()) - 1;
  agg.assign(static_cast<size_t>(n), -1);
  int32_t next = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] != -1) continue;
    if (sro[i] == sro[i + 1]) continue;
    bool free = true;
    for (int64_t k = sro[i]; k < sro[i + 1]; ++k)
      if (agg[sci[k]] != -1) {
        free = false;
        break;
      }
    if (!free) continue;
    agg[i] = next;
    for (int64_t k = sro[i]; k < sro[i + 1]; ++k) agg[sci[k]] = next;
    ++next;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] != -1) continue;
    int32_t best = -1;
    for (int64_t k = sro[i]; k < sro[i + 1]; ++k) {
      const int32_t a = agg[sci[k]];
      if (a != -1 && (best == -1 || a < best)) best = a;
    }
    if (best != -1) agg[i] = best;
  }
  for (int64_t i = 0; i < n; ++i)
    if (agg[i] == -1) agg[i] = next++;
  return next;
}

// spectral_bound (amg.cpp:88-112): the reference's xorshift start vector (host,
// sequential normalisation), power steps on the device
double spectral_bound(const DCsr& a, const double* inv_diag, int iterations, cudaStream_t st) {
  const int64_t n = a.n;
  std::vector<double> hv(static_cast<size_t>(n));
  uint64_t state = 0x2545f4914f6cdd1dull;
  double norm0 = 0.0;
  for (auto& x : hv) {
    state ^= state << 13;
    state ^= state >> 7;
    state ^= state << 17;
    x = static_cast<double>(state >> 11) * 0x1.0p-53 - 0.5;
    norm0 += x * x;
  }
  norm0 = std::sqrt(norm0);
  for (auto& x : hv) x /= norm0;
  DBuf<double> v, w, nrm;
  v.upload(hv);
  w.alloc(n);
  nrm.alloc(1);
  double lambda = 1.0;
  for (int it = 0; it < iterations; ++it) {
    k_spmv<<<nblk(n), kT, 0, st>>>(n, a.ro.p, a.ci.p, a.v.p, v.p, w.p);
    k_scale_inplace<<<nblk(n), kT, 0, st>>>(n, w.p, inv_diag);
    k_seq_norm<<<1, 1024, 0, st>>>(n, w.p, nrm.p);
    count_launch(3);
    double norm = 0.0;
    CK(cudaMemcpyAsync(&norm, nrm.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (norm == 0.0) return 1.0;
    lambda = norm;
    k_div_into<<<nblk(n), kT, 0, st>>>(n, w.p, norm, v.p);
    count_launch();
  }
  return lambda;
}

void diag_of(const DCsr& a, DBuf<double>& d, cudaStream_t st) {
  d.alloc(a.n);
  if (a.n) {
    k_diag<<<nblk(a.n), kT, 0, st>>>(a.n, a.ro.p, a.ci.p, a.v.p, d.p);
    count_launch();
  }
}

// 1 / diag with the smallest non-positive row reported (-1: none)
int64_t inv_diag_checked(const DCsr& a, DBuf<double>& d, cudaStream_t st) {
  diag_of(a, d, st);
  DBuf<unsigned long long> bad;
  bad.alloc(1);
  CK(cudaMemsetAsync(bad.p, 0xff, 8, st));
  if (a.n) {
    k_inv_checked<<<nblk(a.n), kT, 0, st>>>(a.n, d.p, bad.p);
    count_launch();
  }
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return hb == ~0ull ? -1 : static_cast<int64_t>(hb);
}

}  // namespace

// ---------------------------------------------------------------- public objects

struct AmgLevel {
  DCsr A, P, R;
  DBuf<double> r, z, res, cr;  // per-level vectors of the V-cycle
  SweepState sw;               // GS flags and level orders
};

struct AmgHier {
  std::vector<std::unique_ptr<AmgLevel>> levels;
  DCsr coarse;
  DBuf<double> coarse_lu, cz, crhs;
  DBuf<int> coarse_piv, status;
  DBuf<unsigned long long> ticket;
  DBuf<double> zfwd;  // SGS / pre-smoothing output
  int epoch = 0;
  cudaStream_t st = nullptr;
};

void dcsr_from_device(int64_t n, int64_t ncols, const int64_t* ro, const int32_t* ci32, const int64_t* ci64,
                      const double* v, DCsr& out, cudaStream_t st) {
  out.n = n;
  out.ncols = ncols;
  CK(cudaMemcpyAsync(&out.nnz, ro + n, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out.ro.alloc(n + 1);
  out.ci.alloc(out.nnz);
  out.v.alloc(out.nnz);
  CK(cudaMemcpyAsync(out.ro.p, ro, (n + 1) * 8, cudaMemcpyDeviceToDevice, st));
  if (ci32) CK(cudaMemcpyAsync(out.ci.p, ci32, out.nnz * 4, cudaMemcpyDeviceToDevice, st));
  else if (out.nnz) {
    k_i64_to_i32<<<nblk(out.nnz), kT, 0, st>>>(out.nnz, ci64, out.ci.p);
    count_launch();
  }
  CK(cudaMemcpyAsync(out.v.p, v, out.nnz * 8, cudaMemcpyDeviceToDevice, st));
}

static void level_vectors(AmgLevel& L) {
  L.r.alloc(L.A.n);
  L.z.alloc(L.A.n);
  L.res.alloc(L.A.n);
  L.cr.alloc(L.P.ncols);

}

// amg_setup (amg.cpp:189-244); takes ownership of A's buffers
// HDR_AMG_PROFILE=1: phase times of the setup and the cycles on stderr (diagnostics)
static bool amg_profile() {
  static const bool on = getenv("HDR_AMG_PROFILE") != nullptr;
  return on;
}
struct PhaseClock {
  cudaStream_t st;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what, int64_t level) {
    if (!amg_profile()) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[amg] level %lld %-12s %9.3f ms\n", static_cast<long long>(level), what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

AmgHier* amg_setup_device(DCsr&& fine, const hdr_amg_options& o, cudaStream_t st) {
  if (fine.n != fine.ncols) throw StatusError(HDR_SETUP_FAILED, "amg_setup: matrix not square");
  PhaseClock pc{st};
  std::unique_ptr<AmgHier> h(new AmgHier);
  h->st = st;
  DCsr current = std::move(fine);
  for (int level = 0; level < o.max_levels; ++level) {
    const int64_t n = current.n;
    if (n < o.coarse_cap) break;
    DBuf<double> d;
    diag_of(current, d, st);
    DCsr S;
    S.n = S.ncols = n;
    std::vector<int32_t> agg;
    int64_t nc = 0;
    double theta = o.strength_threshold;
    for (int attempt = 0; attempt < 6; ++attempt) {
      S.ro.alloc(n + 1);
      CK(cudaMemsetAsync(S.ro.p, 0, (n + 1) * 8, st));
      k_strength<false><<<nblk(n), kT, 0, st>>>(n, current.ro.p, current.ci.p, current.v.p, d.p, theta, S.ro.p,
                                                nullptr, nullptr);
      offsets_from_counts(S.ro, n, st, &S.nnz);
      S.ci.alloc(S.nnz);
      k_strength<true><<<nblk(n), kT, 0, st>>>(n, current.ro.p, current.ci.p, current.v.p, d.p, theta, nullptr,
                                               S.ro.p, S.ci.p);
      count_launch(2);
      std::vector<int64_t> sro(static_cast<size_t>(n + 1));
      std::vector<int32_t> sci(static_cast<size_t>(S.nnz));
      CK(cudaMemcpyAsync(sro.data(), S.ro.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
      if (S.nnz) CK(cudaMemcpyAsync(sci.data(), S.ci.p, S.nnz * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      nc = host_aggregate(sro, sci, agg);
      if (nc > 0 && static_cast<double>(nc) <= o.stall_ratio * static_cast<double>(n)) break;
      theta *= 0.25;
    }
    pc.lap("aggregate", level);
    if (nc == 0) throw StatusError(HDR_SETUP_FAILED, "amg_setup: empty coarse level");
    if (static_cast<double>(nc) > o.stall_ratio * static_cast<double>(n)) break;  // coarsening stalled
    if (nc >= n) throw StatusError(HDR_SETUP_FAILED, "amg_setup: non-decreasing coarse size");

    // tentative prolongator
    DCsr pt;
    pt.n = n;
    pt.ncols = nc;
    pt.nnz = n;
    pt.ro.alloc(n + 1);
    k_fill_i64<<<nblk(n + 1), kT, 0, st>>>(n + 1, pt.ro.p, 0);
    pt.ci.upload(agg);
    pt.v.alloc(n);
    DBuf<int> asize;
    asize.alloc(nc);
    CK(cudaMemsetAsync(asize.p, 0, nc * sizeof(int), st));
    k_agg_size<<<nblk(n), kT, 0, st>>>(n, pt.ci.p, asize.p);
    k_ptent<<<nblk(n), kT, 0, st>>>(n, pt.ci.p, asize.p, pt.v.p);
    count_launch(3);

    std::unique_ptr<AmgLevel> L(new AmgLevel);
    {
      DBuf<double> inv;
      const int64_t bad = inv_diag_checked(current, inv, st);
      if (bad >= 0) throw StatusError(HDR_SETUP_FAILED, "amg_setup: non-positive diagonal at row " + std::to_string(bad));
    }
    // filtered matrix
    DCsr F;
    F.n = F.ncols = n;
    F.ro.alloc(n + 1);
    CK(cudaMemsetAsync(F.ro.p, 0, (n + 1) * 8, st));
    k_filter<false><<<nblk(n), kT, 0, st>>>(n, current.ro.p, current.ci.p, current.v.p, S.ro.p, S.ci.p, F.ro.p,
                                            nullptr, nullptr, nullptr);
    offsets_from_counts(F.ro, n, st, &F.nnz);
    F.ci.alloc(F.nnz);
    F.v.alloc(F.nnz);
    k_filter<true><<<nblk(n), kT, 0, st>>>(n, current.ro.p, current.ci.p, current.v.p, S.ro.p, S.ci.p, nullptr,
                                           F.ro.p, F.ci.p, F.v.p);
    count_launch(2);
    DBuf<double> finv;
    const int64_t fbad = inv_diag_checked(F, finv, st);
    if (fbad >= 0) throw StatusError(HDR_SETUP_FAILED, "amg_setup: non-positive diagonal at row " + std::to_string(fbad));
    pc.lap("filter", level);
    const double rho = spectral_bound(F, finv.p, o.power_iterations, st);
    pc.lap("power", level);
    const double omega = o.omega_factor / rho;
    // P = (I - omega D_F^-1 F) P_tent on the pattern of AP = triple_product(I, F, P_tent)
    DCsr I;
    I.n = I.ncols = n;
    I.nnz = n;
    I.ro.alloc(n + 1);
    I.ci.alloc(n);
    I.v.alloc(n);
    k_fill_i64<<<nblk(n + 1), kT, 0, st>>>(n + 1, I.ro.p, 0);
    {
      std::vector<int32_t> iota(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) iota[i] = static_cast<int32_t>(i);
      CK(cudaMemcpy(I.ci.p, iota.data(), n * 4, cudaMemcpyHostToDevice));
      std::vector<double> ones(static_cast<size_t>(n), 1.0);
      CK(cudaMemcpy(I.v.p, ones.data(), n * 8, cudaMemcpyHostToDevice));
    }
    count_launch();
    dev_triple(I, F, pt, L->P, st);
    k_smooth<<<nblk(n), kT, 0, st>>>(n, L->P.ro.p, L->P.ci.p, L->P.v.p, pt.ci.p, pt.v.p, finv.p, omega, L->P.v.p);
    count_launch();
    pc.lap("smooth P", level);
    dev_transpose(L->P, L->R, st);
    DCsr coarse;
    dev_triple(L->R, current, L->P, coarse, st);
    pc.lap("RAP", level);
    L->A = std::move(current);
    current = std::move(coarse);
    level_vectors(*L);
    h->levels.push_back(std::move(L));
  }
  h->coarse = std::move(current);
  const int64_t nc = h->coarse.n;
  if (nc * nc > 4000000)
    throw StatusError(HDR_CAP_EXCEEDED, "to_dense: " + std::to_string(nc) + "x" + std::to_string(nc) + " exceeds cap");
  h->coarse_lu.alloc(std::max<int64_t>(1, nc * nc));
  h->coarse_piv.alloc(std::max<int64_t>(1, nc));
  h->status.alloc(2);
  CK(cudaMemsetAsync(h->status.p, 0, 8, st));
  if (nc > 0) {
    k_coarse_factor<<<1, 256, 0, st>>>(nc, h->coarse.ro.p, h->coarse.ci.p, h->coarse.v.p, h->coarse_lu.p,
                                       h->coarse_piv.p, h->status.p);
    count_launch();
  }
  int hs = 0;
  CK(cudaMemcpyAsync(&hs, h->status.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (hs) throw StatusError(HDR_SINGULAR_BLOCK, "lu_factor: pivot below threshold (amg coarsest level)");
  h->cz.alloc(std::max<int64_t>(1, nc));
  h->crhs.alloc(std::max<int64_t>(1, nc));
  h->ticket.alloc(1);
  h->zfwd.alloc(std::max<int64_t>(1, h->levels.empty() ? nc : h->levels[0]->A.n));
  return h.release();
}

void amg_destroy(AmgHier* h) { delete h; }

int64_t amg_levels(const AmgHier* h) { return static_cast<int64_t>(h->levels.size()); }
const DCsr& amg_matrix(const AmgHier* h, int64_t level, int which) {
  if (level == static_cast<int64_t>(h->levels.size())) return h->coarse;
  const AmgLevel& L = *h->levels[static_cast<size_t>(level)];
  return which == 0 ? L.A : (which == 1 ? L.P : L.R);
}

// level orders of A's forward and backward sweeps (rows sorted by dependency
// depth, stable: rows of one level ascending) and the ready flags
static void sweep_prepare(const DCsr& A, SweepState& sw, cudaStream_t st) {
  const int64_t n = A.n;
  sw.flags.alloc(std::max<int64_t>(1, n));
  CK(cudaMemsetAsync(sw.flags.p, 0, std::max<int64_t>(1, n) * sizeof(int), st));
  DBuf<int> la, lb, chg, iota, keys_out;
  la.alloc(std::max<int64_t>(1, n));
  lb.alloc(std::max<int64_t>(1, n));
  chg.alloc(1);
  iota.alloc(std::max<int64_t>(1, n));
  keys_out.alloc(std::max<int64_t>(1, n));
  {
    std::vector<int> h(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int>(i);
    if (n) CK(cudaMemcpyAsync(iota.p, h.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  for (int dir = 0; dir < 2; ++dir) {
    DBuf<int>& order = dir == 0 ? sw.fwd : sw.bwd;
    order.alloc(std::max<int64_t>(1, n));
    CK(cudaMemsetAsync(la.p, 0, std::max<int64_t>(1, n) * sizeof(int), st));
    int* cur = la.p;
    int* nxt = lb.p;
    int64_t steps = 0;
    while (n > 0) {  // blocks of 16 steps; converged when a block changes nothing
      CK(cudaMemsetAsync(chg.p, 0, sizeof(int), st));
      for (int q = 0; q < 16; ++q, ++steps) {
        if (dir == 0) k_level_iter<true><<<nblk(n), kT, 0, st>>>(n, A.ro.p, A.ci.p, cur, nxt, chg.p);
        else k_level_iter<false><<<nblk(n), kT, 0, st>>>(n, A.ro.p, A.ci.p, cur, nxt, chg.p);
        std::swap(cur, nxt);
      }
      count_launch(16);
      int hc = 0;
      CK(cudaMemcpyAsync(&hc, chg.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (!hc || steps > n + 16) break;
    }
    int maxlev = 0;
    if (n > 0) {  // levels + 1 from the last block's changes bound: find the maximum on the host
      std::vector<int> hl(static_cast<size_t>(n));
      CK(cudaMemcpyAsync(hl.data(), cur, n * sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int x : hl) maxlev = std::max(maxlev, x);
      std::vector<int> off(static_cast<size_t>(maxlev) + 2, 0);  // level offsets in the sorted order
      for (int x : hl) ++off[static_cast<size_t>(x) + 1];
      for (int L = 0; L <= maxlev; ++L) off[L + 1] += off[L];
      (dir == 0 ? sw.lvl_fwd : sw.lvl_bwd).upload(off);
      int bits = 1;
      while (bits < 31 && (maxlev >> bits) != 0) ++bits;
      size_t bytes = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, cur, keys_out.p, iota.p, order.p, static_cast<int>(n), 0, bits, st));
      DBuf<unsigned char> tmp;
      tmp.alloc(bytes);
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, cur, keys_out.p, iota.p, order.p, static_cast<int>(n), 0, bits, st));
      // entry offsets of the rows in level order, and the widest level's entries / rows
      std::vector<int64_t> hro(static_cast<size_t>(n) + 1);
      std::vector<int> hord(static_cast<size_t>(n));
      CK(cudaMemcpyAsync(hro.data(), A.ro.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hord.data(), order.p, n * sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<int64_t> eo(static_cast<size_t>(n) + 1, 0);
      for (int64_t t = 0; t < n; ++t) eo[t + 1] = eo[t] + (hro[hord[t] + 1] - hro[hord[t]]);
      int64_t wide = 0, rows = 0;
      for (int64_t i = 0; i < n; ++i) sw.max_row_len = std::max(sw.max_row_len, hro[i + 1] - hro[i]);
      for (int L = 0; L <= maxlev; ++L) {
        wide = std::max(wide, eo[off[L + 1]] - eo[off[L]]);
        rows = std::max<int64_t>(rows, off[L + 1] - off[L]);
      }
      (dir == 0 ? sw.eoff_fwd : sw.eoff_bwd).upload(eo);
      (dir == 0 ? sw.h_eo_fwd : sw.h_eo_bwd) = eo;
      (dir == 0 ? sw.h_off_fwd : sw.h_off_bwd) = off;
      sw.max_level_nnz = std::max(sw.max_level_nnz, wide);
      sw.max_level_rows = std::max(sw.max_level_rows, rows);
    }
    (dir == 0 ? sw.levels_fwd : sw.levels_bwd) = maxlev + 1;
  }
  CK(cudaStreamSynchronize(st));
  sw.ready = true;
}

// one sync-free Gauss-Seidel sweep of A on (r, zin) -> zout, rows in level order
void gs_sweep(AmgHier* h, const DCsr& A, SweepState& sw, bool fwd, const double* r, const double* zin, double* zout) {
  cudaStream_t st = h->st;
  if (A.n == 0) return;
  if (!sw.ready) {
    PhaseClock pc{st};
    sweep_prepare(A, sw, st);
    if (amg_profile())
      fprintf(stderr, "[amg] matrix n %lld nnz %lld: %d forward / %d backward levels, longest row %lld, widest level %lld entries\n",
              static_cast<long long>(A.n), static_cast<long long>(A.nnz), sw.levels_fwd, sw.levels_bwd,
              static_cast<long long>(sw.max_row_len), static_cast<long long>(sw.max_level_nnz));
    pc.lap("levels", A.n);
  }
  // small (coarse) matrices: one CTA, a barrier per batch of rows within a level
  const int64_t zbytes = static_cast<int64_t>((A.n + 1) & ~1) * 8;
  const int64_t cap = (static_cast<int64_t>(kCtaSweepSmem) - zbytes) / 8;
  if (cap >= std::max<int64_t>(2048, sw.max_row_len)) {
    const int64_t capu = std::min(cap, sw.max_level_nnz);
    const size_t cta_smem = static_cast<size_t>(zbytes) + static_cast<size_t>(capu) * 8;
    if (!sw.bat_fwd.p) {  // batches: split every level into runs of <= 512 rows and <= capu entries
      for (int dir = 0; dir < 2; ++dir) {
        const std::vector<int64_t>& eo = dir == 0 ? sw.h_eo_fwd : sw.h_eo_bwd;
        const std::vector<int>& off = dir == 0 ? sw.h_off_fwd : sw.h_off_bwd;
        std::vector<int> bt{0};
        for (size_t L = 0; L + 1 < off.size(); ++L) {
          int t0 = off[L];
          while (t0 < off[L + 1]) {
            int te = t0 + 1;
            while (te < off[L + 1] && te - t0 < 512 && eo[te + 1] - eo[t0] <= capu) ++te;
            bt.push_back(te);
            t0 = te;
          }
        }
        (dir == 0 ? sw.bat_fwd : sw.bat_bwd).upload(bt);
        (dir == 0 ? sw.nbat_fwd : sw.nbat_bwd) = static_cast<int>(bt.size()) - 1;
        if (amg_profile()) fprintf(stderr, "[amg] n %lld: one-CTA sweep, %d batches (%s)\n", static_cast<long long>(A.n),
                                   static_cast<int>(bt.size()) - 1, dir == 0 ? "fwd" : "bwd");
      }
    }
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(k_gs_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCtaSweepSmem)));
      CK(cudaFuncSetAttribute(k_gs_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCtaSweepSmem)));
      attr = true;
    }
    if (fwd)
      k_gs_cta<true><<<1, 512, cta_smem, st>>>(static_cast<int>(A.n), A.ro.p, A.ci.p, A.v.p, r, zin, zout, sw.fwd.p,
                                               sw.bat_fwd.p, sw.nbat_fwd, sw.eoff_fwd.p, h->status.p);
    else
      k_gs_cta<false><<<1, 512, cta_smem, st>>>(static_cast<int>(A.n), A.ro.p, A.ci.p, A.v.p, r, zin, zout, sw.bwd.p,
                                                sw.bat_bwd.p, sw.nbat_bwd, sw.eoff_bwd.p, h->status.p);
    count_launch();
    return;
  }
  if (!getenv("HDR_GS_FLAGS")) {  // level-synchronous cooperative grid (default)
    static int coop_grid = 0;
    if (!coop_grid) {
      int dev = 0, sms = 148, per = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gs_coop<true>, 512, 0);
      coop_grid = sms * std::max(1, std::min(per, 2));
    }
    int nn = static_cast<int>(A.n);
    const int64_t* aro = A.ro.p;
    const int32_t* aci = A.ci.p;
    const double* av = A.v.p;
    const int* ord = fwd ? sw.fwd.p : sw.bwd.p;
    const int* lv = fwd ? sw.lvl_fwd.p : sw.lvl_bwd.p;
    int nlev = fwd ? sw.levels_fwd : sw.levels_bwd;
    int* stp = h->status.p;
    void* args[] = {&nn, &aro, &aci, &av, &r, &zin, &zout, &ord, &lv, &nlev, &stp};
    CK(cudaLaunchCooperativeKernel(fwd ? reinterpret_cast<void*>(k_gs_coop<true>) : reinterpret_cast<void*>(k_gs_coop<false>),
                                   dim3(coop_grid), dim3(512), args, 0, st));
    count_launch();
    return;
  }
  ++h->epoch;
  CK(cudaMemsetAsync(h->ticket.p, 0, 8, st));
  // enough warps for the widest levels, few enough that waiting warps do not crowd the flags
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nblk(A.n * 32), 148 * 2));
  if (fwd)
    k_gs_sweep<true><<<grid, kT, 0, st>>>(A.n, A.ro.p, A.ci.p, A.v.p, r, zin, zout, sw.flags.p, h->epoch, h->ticket.p,
                                          h->status.p, sw.fwd.p);
  else
    k_gs_sweep<false><<<grid, kT, 0, st>>>(A.n, A.ro.p, A.ci.p, A.v.p, r, zin, zout, sw.flags.p, h->epoch, h->ticket.p,
                                           h->status.p, sw.bwd.p);
  count_launch();
}

// v_cycle (amg.cpp:248-266): r, z device vectors of the fine size
static void v_cycle(AmgHier* h, size_t level, const double* r, double* z) {
  cudaStream_t st = h->st;
  if (level == h->levels.size()) {
    if (h->coarse.n > 0) {
      const size_t sm = static_cast<size_t>(h->coarse.n) * 16;
      if (sm > 48 * 1024) CK(cudaFuncSetAttribute(k_coarse_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
      k_coarse_solve<<<1, 1024, sm, st>>>(static_cast<int>(h->coarse.n), h->coarse_lu.p, h->coarse_piv.p, r, z);
      count_launch();
    }
    return;
  }
  AmgLevel& L = *h->levels[level];
  const int64_t n = L.A.n;
  PhaseClock pc{st};
  gs_sweep(h, L.A, L.sw, true, r, nullptr, L.z.p);  // z = 0, forward sweep
  pc.lap("fwd sweep", static_cast<int64_t>(level));
  k_resid<<<nblk(n), kT, 0, st>>>(n, L.A.ro.p, L.A.ci.p, L.A.v.p, L.z.p, r, L.res.p);
  k_spmv<<<nblk(L.R.n), kT, 0, st>>>(L.R.n, L.R.ro.p, L.R.ci.p, L.R.v.p, L.res.p, L.cr.p);
  count_launch(2);
  AmgLevel* next = level + 1 < h->levels.size() ? h->levels[level + 1].get() : nullptr;
  double* cz = next ? next->r.p : h->cz.p;  // coarse solution buffer (next level's r slot is free)
  v_cycle(h, level + 1, L.cr.p, cz);
  k_prolong_add<<<nblk(n), kT, 0, st>>>(n, L.P.ro.p, L.P.ci.p, L.P.v.p, cz, L.z.p);
  count_launch();
  pc.lap("coarser", static_cast<int64_t>(level));
  gs_sweep(h, L.A, L.sw, false, r, L.z.p, z);  // backward sweep from z
  pc.lap("bwd sweep", static_cast<int64_t>(level));
}

void amg_apply_device(AmgHier* h, const double* r, double* z) {
  PhaseClock pc{h->st};
  v_cycle(h, 0, r, z);
  pc.lap("v-cycle", 0);
}

// symmetric Gauss-Seidel (ssgs_setup's apply, solvers.cpp:60-72)
void sgs_apply_device(AmgHier* h, const DCsr& A, SweepState& sw, double* zf, const double* r, double* z) {
  gs_sweep(h, A, sw, true, r, nullptr, zf);
  gs_sweep(h, A, sw, false, r, zf, z);
}

hdr_status amg_status(AmgHier* h) {
  int hs = 0;
  CK(cudaMemcpyAsync(&hs, h->status.p, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaGetLastError());
  if (hs & 1) return fail(HDR_VALIDATION, "ZeroDiagonal: gauss_seidel: zero diagonal");
  return HDR_OK;
}

// a bare hierarchy carrying only the sweep machinery (SGS preconditioner)
AmgHier* sweep_context(int64_t n, cudaStream_t st) {
  std::unique_ptr<AmgHier> h(new AmgHier);
  h->st = st;
  h->status.alloc(2);
  CK(cudaMemsetAsync(h->status.p, 0, 8, st));
  h->ticket.alloc(1);
  h->zfwd.alloc(std::max<int64_t>(1, n));
  return h.release();
}
double* sweep_scratch(AmgHier* h) { return h->zfwd.p; }

void dcsr_from_host(int64_t n, int64_t ncols, const int64_t* ro, const int64_t* ci, const double* v, DCsr& out,
                    cudaStream_t st) {
  out.n = n;
  out.ncols = ncols;
  out.nnz = ro[n];
  if (out.nnz >= (int64_t(1) << 31) || ncols >= (int64_t(1) << 31))
    throw StatusError(HDR_UNSUPPORTED, "matrix too large for 32-bit column indices");
  out.ro.upload(ro, static_cast<size_t>(n) + 1);
  std::vector<int32_t> c32(static_cast<size_t>(out.nnz));
  for (int64_t k = 0; k < out.nnz; ++k) c32[k] = static_cast<int32_t>(ci[k]);
  out.ci.upload(c32);
  out.v.upload(v, static_cast<size_t>(out.nnz));
  (void)st;
}

void dcsr_to_host(const DCsr& a, int64_t* ro, int64_t* ci, double* v, cudaStream_t st) {
  if (ro) CK(cudaMemcpyAsync(ro, a.ro.p, (a.n + 1) * 8, cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> c32(static_cast<size_t>(a.nnz));
  if (ci && a.nnz) CK(cudaMemcpyAsync(c32.data(), a.ci.p, a.nnz * 4, cudaMemcpyDeviceToHost, st));
  if (v && a.nnz) CK(cudaMemcpyAsync(v, a.v.p, a.nnz * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ci)
    for (int64_t k = 0; k < a.nnz; ++k) ci[k] = c32[k];
}

namespace {
// max over rows of the merged |a_ij - t_ij| (max_abs_difference, csr.cpp:201-226) and of |a_ij|
__global__ void k_sym_gap(int64_t n, const int64_t* aro, const int32_t* aci, const double* av, const int64_t* tro,
                          const int32_t* tci, const double* tv, unsigned long long* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int64_t ka = aro[i], kb = tro[i];
  const int64_t ea = aro[i + 1], eb = tro[i + 1];
  double m = 0.0, mx = 0.0;
  for (int64_t k = ka; k < ea; ++k) mx = fmax(mx, fabs(av[k]));
  while (ka < ea || kb < eb) {
    if (kb == eb || (ka < ea && aci[ka] < tci[kb])) {
      m = fmax(m, fabs(av[ka++]));
    } else if (ka == ea || tci[kb] < aci[ka]) {
      m = fmax(m, fabs(tv[kb++]));
    } else {
      m = fmax(m, fabs(av[ka] - tv[kb]));
      ++ka;
      ++kb;
    }
  }
  atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));  // non-negative doubles order as integers
  atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(mx)));
}
}  // namespace

void symmetry_gap(const DCsr& a, double* diff, double* amax, cudaStream_t st) {
  DCsr t;
  dev_transpose(a, t, st);
  DBuf<unsigned long long> out;
  out.alloc(2);
  CK(cudaMemsetAsync(out.p, 0, 16, st));
  if (a.n) {
    k_sym_gap<<<nblk(a.n), kT, 0, st>>>(a.n, a.ro.p, a.ci.p, a.v.p, t.ro.p, t.ci.p, t.v.p, out.p);
    count_launch();
  }
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, out.p, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(diff, &h[0], 8);
  std::memcpy(amax, &h[1], 8);
}

int64_t positive_inv_diag(const DCsr& a, DBuf<double>& dinv, cudaStream_t st) { return inv_diag_checked(a, dinv, st); }

}  // namespace hdr

// ---------------------------------------------------------------- C ABI

struct hdr_amg_s {
  hdr::AmgHier* h = nullptr;
  int64_t n = 0;
  ~hdr_amg_s() {
    if (h) hdr::amg_destroy(h);
  }
};

using hdr::catch_all;
using hdr::CudaError;
using hdr::fail;

void hdr_amg_default_options(hdr_amg_options* o) {
  if (!o) return;
  o->strength_threshold = 0.08;
  o->omega_factor = 1.0;
  o->coarse_cap = 64;
  o->max_levels = 25;
  o->power_iterations = 10;
  o->stall_ratio = 0.9;
}

hdr_status hdr_amg_setup(int64_t n, const int64_t* ro, const int64_t* ci, const double* v, int on_device,
                         const hdr_amg_options* options, hdr_amg_t* out) {
  if (!out || n < 0 || !ro) return fail(HDR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return catch_all([&]() -> hdr_status {
    int devs = 0;
    if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) return fail(HDR_CUDA_ERROR, "no CUDA device available");
    hdr_amg_options o;
    hdr_amg_default_options(&o);
    if (options) o = *options;
    hdr::DCsr a;
    if (on_device) hdr::dcsr_from_device(n, n, ro, nullptr, ci, v, a, nullptr);
    else hdr::dcsr_from_host(n, n, ro, ci, v, a, nullptr);
    std::unique_ptr<hdr_amg_s> amg(new hdr_amg_s);
    amg->n = n;
    amg->h = hdr::amg_setup_device(std::move(a), o, nullptr);
    *out = amg.release();
    return HDR_OK;
  });
}

hdr_status hdr_amg_info(hdr_amg_t amg, int64_t* levels, int64_t* sizes, int64_t* nnz) {
  if (!amg) return fail(HDR_INVALID_ARGUMENT, "null argument");
  const int64_t L = hdr::amg_levels(amg->h);
  if (levels) *levels = L;
  for (int64_t l = 0; l <= L; ++l) {
    const hdr::DCsr& m = hdr::amg_matrix(amg->h, l, 0);
    if (sizes) sizes[l] = m.n;
    if (nnz) nnz[l] = m.nnz;
  }
  return HDR_OK;
}

hdr_status hdr_amg_level_matrix(hdr_amg_t amg, int64_t level, int which, int64_t* dims, int64_t* ro, int64_t* ci,
                                double* v) {
  if (!amg) return fail(HDR_INVALID_ARGUMENT, "null argument");
  const int64_t L = hdr::amg_levels(amg->h);
  if (level < 0 || level > L || which < 0 || which > 2 || (level == L && which != 0))
    return fail(HDR_INVALID_ARGUMENT, "amg level / matrix out of range");
  return catch_all([&]() -> hdr_status {
    const hdr::DCsr& m = hdr::amg_matrix(amg->h, level, which);
    if (dims) {
      dims[0] = m.n;
      dims[1] = m.ncols;
      dims[2] = m.nnz;
    }
    hdr::dcsr_to_host(m, ro, ci, v, nullptr);
    return HDR_OK;
  });
}

hdr_status hdr_amg_apply(hdr_amg_t amg, const double* r, double* z, int on_device) {
  if (!amg || !r || !z) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    const int64_t n = amg->n;
    hdr::DBuf<double> dr, dz;
    const double* pr = r;
    double* pz = z;
    if (!on_device) {
      dr.upload(r, static_cast<size_t>(n));
      dz.alloc(static_cast<size_t>(n));
      pr = dr.p;
      pz = dz.p;
    }
    hdr::amg_apply_device(amg->h, pr, pz);
    const hdr_status s = hdr::amg_status(amg->h);
    if (s != HDR_OK) return s;
    if (!on_device && n) CK(cudaMemcpy(z, pz, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}

void hdr_amg_destroy(hdr_amg_t amg) { delete amg; }

hdr_status hdr_csr_precond_apply_host(int64_t n, const int64_t* ro, const int64_t* ci, const double* v, int kind,
                                      const double* r, double* z) {
  if (n < 0 || !ro || !r || !z) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (kind != 1 && kind != 2) return fail(HDR_INVALID_ARGUMENT, "kind must be 1 (jacobi) or 2 (sgs)");
  return catch_all([&]() -> hdr_status {
    int devs = 0;
    if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) return fail(HDR_CUDA_ERROR, "no CUDA device available");
    hdr::DCsr a;
    hdr::dcsr_from_host(n, n, ro, ci, v, a, nullptr);
    hdr::DBuf<double> dinv, dr, dz;
    const int64_t bad = hdr::positive_inv_diag(a, dinv, nullptr);
    if (bad >= 0) return fail(HDR_VALIDATION, "ZeroDiagonal: non-positive diagonal entry at row " + std::to_string(bad));
    dr.upload(r, static_cast<size_t>(n));
    dz.alloc(static_cast<size_t>(n));
    if (kind == 1) {
      std::vector<double> d(static_cast<size_t>(n));
      if (n) CK(cudaMemcpy(d.data(), dinv.p, n * 8, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n; ++i) z[i] = d[i] * r[i];
      return HDR_OK;
    }
    std::unique_ptr<hdr::AmgHier, void (*)(hdr::AmgHier*)> ctx(hdr::sweep_context(n, nullptr), hdr::amg_destroy);
    hdr::SweepState sw;
    hdr::sgs_apply_device(ctx.get(), a, sw, hdr::sweep_scratch(ctx.get()), dr.p, dz.p);
    const hdr_status s = hdr::amg_status(ctx.get());
    if (s != HDR_OK) return s;
    if (n) CK(cudaMemcpy(z, dz.p, n * 8, cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}
