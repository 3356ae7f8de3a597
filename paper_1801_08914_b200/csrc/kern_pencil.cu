// k = 0 hybridize in one pass: the pencil kernel (hybridize, src/reduction.cpp:262-354,
// with element_matrices / assemble_from_reference, src/rt_space.cpp:345-374, and
// the from_triplets scatter, src/csr.cpp:43-75).
//
// The RT0 reference element of an axis-aligned box (build_reference,
// src/rt_space.cpp:180-314) has
//   D = c 1 1^T                  (div of every RT0 basis function is the same constant:
//                                 every entry carries the same bits, checked on the host)
//   M = blockdiag(M_0, .., M_d-1) (2 x 2 per axis, cross-axis entries exactly 0)
// so the reference's A_T = fl(fl(alpha D) + fl(beta M)) is, exactly,
//   A_T = gamma 1 1^T + P,   gamma = fl(alpha c),   P = blockdiag(P_a),
//   P_a[i][j] = A_T[i][j] - gamma   (Sterbenz / one rounding: the 2 x 2 mass blocks
//                                    are well conditioned, cond ~ 3)
// and by Sherman-Morrison, with u = P^-1 1 and sigma = 1^T u,
//   A_T^-1 = P^-1 - kappa u u^T,   kappa = gamma / (1 + gamma sigma),
//   A_T^-1 f = P^-1 f - kappa u (u . f).
// Every term is a sum of same-signed quantities or a rank-one correction whose
// size is bounded by |P^-1|, so the result is within a few ulp of max|A_T^-1|
// whatever alpha / beta: the inverse of the reference's rounded A_T, not of the
// unrounded one.  H_T = C_T A_T^-1 C_T^T is the interior-face block of A_T^-1
// (unit constraint rows of build_C, src/reduction.cpp:172-181).
//
// Acceptance (DESIGN.md §2 "Fail-safe"): a cell whose condition bound
// (1 + gamma sigma) sum_a tr(P_a) sum_a tr(P_a)/det(P_a) (at most dim^2 times the
// bound with maxima) exceeds kPencilCond, or whose blocks are not positive definite,
// contributes zeros in the fast pass; a warp with such a cell in any of its rows
// (its own cells or the cells below / behind / before them) then runs the segment
// again, out of line, with the exact double-double rows of those cells (rt0_exact,
// the reference's SingularBlock rule) and rewrites its rows: no list, no second
// launch, no ordering between CTAs.  The reference's LU pivots of an accepted SPD
// cell are >= lambda_min / G >= 1e-12 / G of the block maximum (G <= 2^(n-1) = 32 the
// partial-pivoting growth), above its 1e-14 threshold.  BASELINE config 2's worst cell
// has a bound of ~5e9; the bound grows like h^-2 alpha / beta.
//
// Scatter.  One warp per 32-cell segment of an x-line (lane = cell).  The H row of
// the interior face between cells T- and T+ (T+ the cell on the face's plus side) is
// assembled by T+'s lane: T-'s row comes from lane - 1 (x faces: a shuffle, or the
// previous warp's last lane through shared memory) or is recomputed from T-'s
// inputs (y, z faces: the cell below / behind, an L1 / L2 hit).  Rows of
// consecutive lanes are consecutive rows of H (interior faces of one line, face
// order), so a warp stages its rows in shared memory and writes them out as one
// contiguous, coalesced segment.  No staging in HBM, no colouring, one launch; every
// H entry and g entry is written exactly once (once more, complete, by the exact pass
// of a warp whose rows involve a rejected cell); the two contributions to a diagonal
// entry / g entry meet as fl(h(T-) + h(T+)), the reference's two-term sum.
#include "hdr_device.cuh"
#include "kernels.hpp"
#include "rt0_exact.cuh"

namespace hdr {

namespace {

#ifndef HDR_PENCIL_PW
#define HDR_PENCIL_PW 4
#endif
constexpr int kPW = HDR_PENCIL_PW;  // warps per CTA
#ifndef HDR_PENCIL_MINB
#define HDR_PENCIL_MINB 5               // CTAs per SM asked of ptxas: 96 registers, no spills, 20 warps per SM
#endif
constexpr double kPencilCond = 1e12;  // acceptance bound on cond(A_T)

template <int DIM>
struct PencilSol {  // A_T^-1 = P^-1 - kappa u u^T and A_T^-1 f in compact form
  double i00[DIM], i01[DIM], i11[DIM];  // P_a^-1
  double u[2 * DIM];
  double pf[2 * DIM];  // P^-1 f
  double kap, uf;      // kappa, u . f
};

__device__ __forceinline__ double rcp64(double d) {  // ~1 ulp reciprocal: MUFU seed + two Newton steps
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// the compact solution of one cell; false: not accepted (not SPD, or the condition
// bound is above kPencilCond, or non-finite); cond: the bound
template <int DIM>
__device__ __forceinline__ bool pencil_solve(const PencilConst<DIM>& pc, double a, double b, const double (&f)[2 * DIM],
                                             PencilSol<DIM>& s, double& cond) {
  const double gam = __dmul_rn(a, pc.c);  // fl(alpha D_ij), every ij
  double sig = 0.0, tsum = 0.0, rsum = 0.0, uf = 0.0;
  bool pd = gam >= 0.0;
#pragma unroll
  for (int ax = 0; ax < DIM; ++ax) {
    // the reference's A_T entries of this axis block, minus gamma (no contraction)
    const double p00 = __dsub_rn(__dadd_rn(gam, __dmul_rn(b, pc.md0[ax])), gam);
    const double p11 = __dsub_rn(__dadd_rn(gam, __dmul_rn(b, pc.md1[ax])), gam);
    const double p01 = __dsub_rn(__dadd_rn(gam, __dmul_rn(b, pc.mo[ax])), gam);
    const double det = fma(p00, p11, -(p01 * p01));
    pd = pd && p00 > 0.0 && det > 0.0;
    const double id = rcp64(det);
    s.i00[ax] = p11 * id;
    s.i11[ax] = p00 * id;
    s.i01[ax] = -p01 * id;
    s.u[2 * ax] = s.i00[ax] + s.i01[ax];
    s.u[2 * ax + 1] = s.i01[ax] + s.i11[ax];
    sig += s.u[2 * ax] + s.u[2 * ax + 1];
    const double tr = p00 + p11;
    tsum += tr;                  // >= max_a tr(P_a)  (sums: an fp64 max is several instructions)
    rsum = fma(tr, id, rsum);    // >= max_a tr(P_a) / det(P_a) >= 1 / lambda_min(P)
    const double f0 = f[2 * ax], f1 = f[2 * ax + 1];
    s.pf[2 * ax] = fma(s.i00[ax], f0, s.i01[ax] * f1);
    s.pf[2 * ax + 1] = fma(s.i01[ax], f0, s.i11[ax] * f1);
    uf = fma(s.u[2 * ax], f0, fma(s.u[2 * ax + 1], f1, uf));
  }
  const double den = fma(gam, sig, 1.0);
  s.kap = gam * rcp64(den);
  s.uf = uf;
  cond = den * tsum * rsum;
  return pd && cond <= kPencilCond && s.kap == s.kap && fabs(s.kap) < 1e300 && fabs(uf) < 1e300;
}

template <int DIM>
__device__ __forceinline__ void pencil_zero(PencilSol<DIM>& s) {
#pragma unroll
  for (int ax = 0; ax < DIM; ++ax) s.i00[ax] = s.i01[ax] = s.i11[ax] = 0.0;
#pragma unroll
  for (int i = 0; i < 2 * DIM; ++i) s.u[i] = s.pf[i] = 0.0;
  s.kap = s.uf = 0.0;
}

// row r of [A_T^-1 | A_T^-1 f]
template <int DIM>
__device__ __forceinline__ void pencil_row(const PencilSol<DIM>& s, int r, double (&h)[2 * DIM + 1]) {
  constexpr int N = 2 * DIM;
  const double kr = s.kap * s.u[r];
  const int ar = r >> 1;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double pinv = 0.0;
    if ((j >> 1) == ar) pinv = (r & 1) ? ((j & 1) ? s.i11[ar] : s.i01[ar]) : ((j & 1) ? s.i01[ar] : s.i00[ar]);
    h[j] = fma(-kr, s.u[j], pinv);
  }
  h[N] = fma(-kr, s.uf, s.pf[r]);
}

template <int DIM>
__device__ __forceinline__ void load_cell(const double* alpha, const double* beta, const double* fh, int64_t e, double& a,
                                          double& b, double (&f)[2 * DIM]) {
  a = __ldg(alpha + e);
  b = __ldg(beta + e);
  const double2* fp = reinterpret_cast<const double2*>(fh + e * (2 * DIM));
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    const double2 v = __ldg(fp + j);
    f[2 * j] = v.x;
    f[2 * j + 1] = v.y;
  }
}

// Neighbour inputs staged by cp.async: slot [0] = {alpha, beta}, [1 + j] = {f_2j, f_2j+1},
// each slot 32 double2 (one per lane: conflict-free 16-byte accesses); the copies are
// issued at kernel start and cost no registers while the own cell is solved.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}
template <int DIM>
__device__ __forceinline__ void stage_cell(const HybArgs& A, int64_t e, double2* slot) {
  cp_async8(&slot[0].x, A.alpha + e);
  cp_async8(&slot[0].y, A.beta + e);
  const double2* fp = reinterpret_cast<const double2*>(A.f + e * (2 * DIM));
#pragma unroll
  for (int j = 0; j < DIM; ++j) cp_async16(slot + 32 * (1 + j), fp + j);
}
template <int DIM>
__device__ __forceinline__ void staged_cell(const double2* slot, bool ok, double& a, double& b, double (&f)[2 * DIM]) {
  a = b = 1.0;
#pragma unroll
  for (int j = 0; j < 2 * DIM; ++j) f[j] = 0.0;
  if (ok) {
    const double2 ab = slot[0];
    a = ab.x, b = ab.y;
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      const double2 v = slot[32 * (1 + j)];
      f[2 * j] = v.x, f[2 * j + 1] = v.y;
    }
  }
}

// Row r of [A_T^-1 | A_T^-1 f] of a cell the closed form does not accept: the exact
// double-double path (rt0_exact, the reference's SingularBlock rule), out of line
// and through shared memory so that the fast path keeps its registers.  Every lane
// that needs a row of such a cell (its own lane, the lanes above / behind it)
// computes it itself: no list, no second launch, no ordering between CTAs.
template <int DIM>
__device__ __noinline__ void pencil_exact_row(const double* D, const double* M, double a, double b, unsigned bmask,
                                              const double* f, int r, int* status, double* out) {
  constexpr int N = 2 * DIM, NC = N + 1;
  double hx[N * NC];
  for (int i = 0; i < N * NC; ++i) hx[i] = 0.0;  // a singular cell raises through status; its rows stay zero
  rt0_exact<N, NC, true>(D, M, a, b, bmask, f, nullptr, hx, status);
  for (int q = 0; q < NC; ++q) out[q] = hx[r * NC + q];
}

// the solution of a neighbour cell (zero when the cell is not accepted: its own
// lane lists it for the exact path)
// (returns the kind of the cell: 0 none, 1 closed form, 2 exact path)
template <int DIM>
__device__ __forceinline__ int neighbour(const HybArgs& A, const PencilConst<DIM>& pc, int64_t e, PencilSol<DIM>& s) {
  double a, b, f[2 * DIM], cond;
  load_cell<DIM>(A.alpha, A.beta, A.f, e, a, b, f);
  if (!pencil_solve<DIM>(pc, a, b, f, s, cond) || A.force_exact) {
    pencil_zero<DIM>(s);
    return 2;
  }
  return 1;
}

// the same from prefetched inputs (zero for lanes without a cell)
template <int DIM>
__device__ __forceinline__ int solved_neighbour(const HybArgs& A, const PencilConst<DIM>& pc, bool valid, double a,
                                                double b, const double (&f)[2 * DIM], PencilSol<DIM>& s) {
  double cond;
  if (!valid || !pencil_solve<DIM>(pc, a, b, f, s, cond) || A.force_exact) {
    pencil_zero<DIM>(s);
    return valid ? 2 : 0;
  }
  return 1;
}

// Warp-collective write-out of a staged segment: stg[q] -> dst[q] for q in
// [pad, pad + total), dst 16-byte aligned (pad = the segment's 8-byte misalignment):
// aligned 16-byte streaming stores, a scalar head / tail where the ends are odd.
__device__ __forceinline__ void segment_write(double* dst, const double* stg, int pad, int total, int lane) {
  const int qe = pad + total;
  if (pad && lane == 0) __stcs(dst + 1, stg[1]);
  if ((qe & 1) && lane == 31 && qe - 1 >= 2 * pad) __stcs(dst + qe - 1, stg[qe - 1]);
  const double2* s2 = reinterpret_cast<const double2*>(stg);
  double2* d2 = reinterpret_cast<double2*>(dst);
  const int je = qe >> 1;
  int j = pad + lane;
  for (; j + 32 < je; j += 64) {  // two loads in flight, then two coalesced 16-byte stores
    const double2 v0 = s2[j], v1 = s2[j + 32];
    __stcs(d2 + j, v0);
    __stcs(d2 + j + 32, v1);
  }
  if (j < je) __stcs(d2 + j, s2[j]);
  __syncwarp();
}

// Warp-collective: the H rows (and g entries) of the lanes with `has`, faces of
// axis ax; hm = T-'s row (its slot 2 ax + 1), hp = T+'s row (slot 2 ax); c = T+'s
// coordinates.  Column order (interior faces of T- and T+ in face order; T- and
// T+ differ in coordinate ax): per axis b = 0..dim-1,
//   b == ax: [T-.lo_b], diagonal, [T+.hi_b]
//   b <  ax: T-.lo_b, T-.hi_b, T+.lo_b, T+.hi_b
//   b >  ax: T-.lo_b, T+.lo_b, T-.hi_b, T+.hi_b
// (lo_b / hi_b present when interior, the same for T- and T+ when b != ax).
template <int DIM>
__device__ __forceinline__ void emit_rows(const HybArgs& A, int ax, bool has, const int (&c)[3], const int (&nc)[3],
                                          int x0, const longlong2* fq, const double (&hm)[2 * DIM + 1],
                                          const double (&hp)[2 * DIM + 1], double* stg) {
  constexpr int N = 2 * DIM;
  const int lane = threadIdx.x & 31;
  if (__ballot_sync(0xffffffffu, has) == 0u) return;
  // the row's candidate entries in column order, each with its presence (static
  // slots: registers, no local memory)
  constexpr int RL = 4 * DIM - 1;
  double v[RL];
  bool pr[RL];
  int t = 0;
  int lfull = 0;  // entries of a row whose cell is interior along x (warp-uniform)
#pragma unroll
  for (int b = 0; b < DIM; ++b) {
    const double ml = hm[2 * b], mh = hm[2 * b + 1], pl = hp[2 * b], ph = hp[2 * b + 1];
    if (b == ax) {
      const bool far_lo = c[b] >= 2, far_hi = c[b] + 1 < nc[b];
      v[t] = ml, pr[t++] = far_lo;
      v[t] = mh + pl, pr[t++] = true;
      v[t] = ph, pr[t++] = far_hi;
      lfull += b == 0 ? 3 : 1 + (far_lo ? 1 : 0) + (far_hi ? 1 : 0);
    } else {
      const bool lo = c[b] >= 1, hi = c[b] + 2 <= nc[b];
      v[t] = ml, pr[t++] = lo;
      if (b < ax) {
        v[t] = mh, pr[t++] = hi;
        v[t] = pl, pr[t++] = lo;
      } else {
        v[t] = pl, pr[t++] = lo;
        v[t] = mh, pr[t++] = hi;
      }
      v[t] = ph, pr[t++] = hi;
      lfull += b == 0 ? 4 : 2 * ((lo ? 1 : 0) + (hi ? 1 : 0));
    }
  }
  // Row offsets in closed form (no scan): along the segment only the cells next to
  // the x boundary have shorter rows.  x faces (rows of x >= 1): the row of x = 1
  // lacks T-'s far face, the row of x = N0 - 1 T+'s; y / z faces: the rows of
  // x = 0 and x = N0 - 1 lack the two x faces beyond the boundary.
  const int n0 = nc[0], x = c[0];
  const int x1 = min(x0 + 32, n0);            // one past the segment's last cell
  const int xs = ax == 0 ? max(x0, 1) : x0;   // first cell with a row
  if (x1 <= xs) return;                       // (warp-uniform)
  const int first = xs - x0;
  int off, total;
  if (ax == 0) {
    off = (x - xs) * lfull - ((xs <= 1 && x > 1) ? 1 : 0);
    total = (x1 - xs) * lfull - ((xs <= 1 && x1 > 1) ? 1 : 0) - (x1 == n0 ? 1 : 0);
  } else {
    off = (x - xs) * lfull - ((xs == 0 && x > 0) ? 2 : 0);
    total = (x1 - xs) * lfull - (xs == 0 ? 2 : 0) - (x1 == n0 ? 2 : 0);
  }
  // {row start, row} of the first row (staged by lane `first` at kernel start)
  const longlong2 fqv = *fq;  // broadcast read of the staged pair
  const long long rs = fqv.x, row = fqv.y;
  // staged at the parity of the global position, so that the write-out moves
  // aligned 16-byte pairs: stg[q] <-> hval[rs - pad + q] (pad: the 8-byte misalignment)
  const int pad = static_cast<int>((reinterpret_cast<uintptr_t>(A.hval + rs) >> 3) & 1);  // any 8-byte aligned hval
  if (has) {
    int p = off + pad;
#pragma unroll
    for (int i = 0; i < RL; ++i)
      if (pr[i]) stg[p++] = v[i];
  }
  if (has) __stcs(A.g + row + (lane - first), hm[N] + hp[N]);
  __syncwarp();
  segment_write(A.hval + (rs - pad), stg, pad, total, lane);
}

template <int DIM>
struct PencilSmem {
  struct Args {  // the kernel arguments for the out-of-line exact pass (written only when it runs)
    HybArgs A;
    PencilConst<DIM> pc;
    FastDiv dseg;
  };
  double2 nbr[kPW][DIM - 1][DIM + 1][32];  // staged inputs of the cells below / behind
  longlong2 fq[kPW][3];                     // {row start, row} of each axis' first row
  double stg[kPW][32 * (4 * DIM - 1) + 2];  // a warp's H rows before the coalesced write-out (+ parity pad)
  double xrow[kPW][2 * DIM + 1];            // last lane's x row for the next segment's first lane
  double xr[kPW][32][2 * DIM + 1];          // exact-path rows (rare), one slot per lane
  int xkind[kPW];                           // kind of the last lane's cell
  alignas(16) unsigned char args_raw[kPW][sizeof(Args)];
  __device__ Args* args_ptr() { return reinterpret_cast<Args*>(args_raw); }
};

// row R of the cell ec = (ex, ey, ez) of kind `kind` (0 none, 1 closed form, 2 not
// accepted): the closed-form row (zeros unless kind == 1), or, in the exact pass, the
// double-double row of a cell that was not accepted
template <int DIM, bool EXACT, int R>
__device__ __forceinline__ void cell_row(const HybArgs& A, PencilSmem<DIM>& sm, const PencilSol<DIM>& sol, int kind,
                                         int64_t ec, int ex, int ey, int ez, double (&h)[2 * DIM + 1]) {
  constexpr int N = 2 * DIM, NC = N + 1;
  pencil_row<DIM>(sol, R, h);
  if (EXACT && kind == 2) {
    const int cc3[3] = {ex, ey, ez};
    double* out = sm.xr[threadIdx.x >> 5][threadIdx.x & 31];
    pencil_exact_row<DIM>(A.fx.D, A.fx.M, __ldg(A.alpha + ec), __ldg(A.beta + ec), rt0_bmask<DIM>(A.m, cc3),
                          A.f + ec * N, R, A.status, out);
#pragma unroll
    for (int q = 0; q < NC; ++q) h[q] = out[q];
  }
}

// One warp's segment.  EXACT = false: the fast pass (closed form; a cell that is not
// accepted contributes zeros and the return value tells that some row of this warp
// involves such a cell).  EXACT = true: the same segment again with the exact rows of
// those cells (rare, out of line): it rewrites the warp's rows, now complete.
template <int DIM, bool EXACT>
__device__ __forceinline__ bool pencil_warp(const HybArgs& A, const PencilConst<DIM>& pc, FastDiv dseg, uint32_t gw,
                                            bool wvalid, PencilSmem<DIM>& sm) {
  constexpr int N = 2 * DIM, NC = N + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const DevMesh& m = A.m;
  const int N0 = static_cast<int>(m.N[0]), N1 = static_cast<int>(m.N[1]), N2 = DIM == 3 ? static_cast<int>(m.N[2]) : 1;
  const uint32_t line = wvalid ? dseg.div(gw) : 0;  // multiply-shift divisions (32-bit: < 2^31 cells)
  const int seg = wvalid ? static_cast<int>(gw - line * dseg.d) : 0;
  const uint32_t zq = m.div_n1.div(line);
  const int y = static_cast<int>(line - zq * static_cast<uint32_t>(N1)), z = static_cast<int>(zq);
  const int x = seg * 32 + lane;
  const bool valid = wvalid && x < N0;
  const int c[3] = {x, y, z}, nc[3] = {N0, N1, N2};
  const int64_t e = x + static_cast<int64_t>(N0) * (y + static_cast<int64_t>(N1) * z);
  // staged by cp.async (no registers held while the own cell is solved): the {row
  // start, row} of each axis' first row (by the lane that owns it: x rows start at
  // x = 1) and the inputs of the cells below / behind
  const int xfirst = seg == 0 ? 1 : 0;
  longlong2* const fqx = &sm.fq[warp][0];
  longlong2* const fqy = &sm.fq[warp][1];
  longlong2* const fqz = &sm.fq[warp][2];
  if (valid && lane == xfirst && x >= 1) cp_async16(fqx, A.frs + face_id32(m, 0, x, y, z));
  if (valid && lane == 0 && y >= 1) cp_async16(fqy, A.frs + face_id32(m, 1, x, y, z));
  if (DIM == 3 && valid && lane == 0 && z >= 1) cp_async16(fqz, A.frs + face_id32(m, 2, x, y, z));
  auto& nbr = sm.nbr;
  if (valid && y >= 1) stage_cell<DIM>(A, e - N0, &nbr[warp][0][0][lane]);
  if (DIM == 3 && valid && z >= 1) stage_cell<DIM>(A, e - static_cast<int64_t>(N0) * N1, &nbr[warp][DIM - 2][0][lane]);
  asm volatile("cp.async.commit_group;" ::: "memory");
  PencilSol<DIM> s;
  int own = 1;
  {
    double a = 1.0, b = 1.0, f[N], cond = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) f[j] = 0.0;
    if (valid) load_cell<DIM>(A.alpha, A.beta, A.f, e, a, b, f);
    const bool ok = pencil_solve<DIM>(pc, a, b, f, s, cond);
    if (!EXACT && valid && A.qlog) A.qlog[e] = static_cast<float>(cond * 0x1p-53);
    if (!valid || !ok || A.force_exact) {
      pencil_zero<DIM>(s);
      own = valid ? 2 : 0;
      if (!EXACT && valid) atomicAdd(A.xcount, 1);  // the count hdr_hybrid_exact_cells reports
    }
  }
  bool need = own == 2;
  double* st = sm.stg[warp];
  double hm[NC], hp[NC];
  // x faces: T- = (x - 1, y, z), its row of slot 1
  cell_row<DIM, EXACT, 1>(A, sm, s, own, e, x, y, z, hp);
  if (!EXACT) {  // the next segment's first lane takes this warp's last row through shared memory
    if (lane == 31) {
#pragma unroll
      for (int q = 0; q < NC; ++q) sm.xrow[warp][q] = hp[q];
      sm.xkind[warp] = own;
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NC; ++q) hm[q] = __shfl_up_sync(0xffffffffu, hp[q], 1);
  int kx = __shfl_up_sync(0xffffffffu, own, 1);
  if (lane == 0 && seg > 0 && valid) {
    if (!EXACT && warp > 0) {  // the previous warp holds the line's previous segment
#pragma unroll
      for (int q = 0; q < NC; ++q) hm[q] = sm.xrow[warp - 1][q];
      kx = sm.xkind[warp - 1];
    } else {  // another CTA's (or, in the exact pass, any previous) segment: recompute its last cell
      PencilSol<DIM> sn;
      kx = neighbour<DIM>(A, pc, e - 1, sn);
      cell_row<DIM, EXACT, 1>(A, sm, sn, kx, e - 1, x - 1, y, z, hm);
    }
  }
  need = need || (valid && x >= 1 && kx == 2);
  cell_row<DIM, EXACT, 0>(A, sm, s, own, e, x, y, z, hp);
  asm volatile("cp.async.wait_group 0;" ::: "memory");  // neighbour inputs: own copies; row starts: another lane's
  __syncwarp();
  emit_rows<DIM>(A, 0, valid && x >= 1, c, nc, seg * 32, fqx, hm, hp, st);
  // y faces: T- = (x, y - 1, z), slot 3 (line-uniform condition)
  if (y >= 1) {
    PencilSol<DIM> sn;
    double ya, yb, yf[N];
    staged_cell<DIM>(&nbr[warp][0][0][lane], valid, ya, yb, yf);
    const int kn = solved_neighbour<DIM>(A, pc, valid, ya, yb, yf, sn);
    need = need || kn == 2;
    cell_row<DIM, EXACT, 3>(A, sm, sn, kn, e - N0, x, y - 1, z, hm);
    cell_row<DIM, EXACT, 2>(A, sm, s, own, e, x, y, z, hp);
    emit_rows<DIM>(A, 1, valid, c, nc, seg * 32, fqy, hm, hp, st);
  }
  if (DIM == 3 && z >= 1) {  // z faces: T- = (x, y, z - 1), slot 5
    PencilSol<DIM> sn;
    double za, zb, zf[N];
    staged_cell<DIM>(&nbr[warp][DIM - 2][0][lane], valid, za, zb, zf);
    const int kn = solved_neighbour<DIM>(A, pc, valid, za, zb, zf, sn);
    need = need || kn == 2;
    cell_row<DIM, EXACT, DIM == 3 ? 5 : 3>(A, sm, sn, kn, e - static_cast<int64_t>(N0) * N1, x, y, z - 1, hm);
    cell_row<DIM, EXACT, DIM == 3 ? 4 : 2>(A, sm, s, own, e, x, y, z, hp);
    emit_rows<DIM>(A, 2, valid, c, nc, seg * 32, fqz, hm, hp, st);
  }
  return need;
}

// the exact pass of one warp, out of line: its arguments come through shared memory,
// so the fast pass keeps its registers and the kernel parameters stay in the constant bank
template <int DIM>
__device__ __noinline__ void pencil_warp_exact(PencilSmem<DIM>* sm, uint32_t gw) {
  const typename PencilSmem<DIM>::Args& ar = sm->args_ptr()[threadIdx.x >> 5];
  pencil_warp<DIM, true>(ar.A, ar.pc, ar.dseg, gw, true, *sm);
}

template <int DIM>
__global__ void __launch_bounds__(kPW * 32, HDR_PENCIL_MINB) k_rt0_pencil(HybArgs A, PencilConst<DIM> pc, FastDiv dseg, uint32_t nwarps) {
  // dynamic shared memory (above the 48 KB static limit with the neighbour slots)
  extern __shared__ __align__(16) unsigned char pencil_smem[];
  using Sm = PencilSmem<DIM>;
  Sm& sm = *reinterpret_cast<Sm*>(pencil_smem);
  const int warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * kPW + warp;
  const bool need = pencil_warp<DIM, false>(A, pc, dseg, gw, gw < nwarps, sm);
  if (__any_sync(0xffffffffu, need)) {  // rare: a row of this warp involves a cell the closed form rejected
    typename Sm::Args& ar = sm.args_ptr()[warp];
    if ((threadIdx.x & 31) == 0) {
      ar.A = A;
      ar.pc = pc;
      ar.dseg = dseg;
    }
    __syncwarp();
    pencil_warp_exact<DIM>(&sm, gw);
  }
}

// ------------------------------------------------------------------ k = 0 static condensation, one pass
//
// Without bubbles S = P^T A_hat P and f_S = P^T f_hat (static_condense,
// src/reduction.cpp:448-557): the row of face F holds sp sq A_T[p][q] of its
// one or two cells over all their faces, the diagonal and f_S entry the
// two-term sums of the reference's from_triplets.  Same layout as the hybridize
// pencil kernel: one warp per 32-cell segment of an x-line, the row of a face
// assembled by the lane of its plus-side cell (T- by shuffle / from its inputs),
// the rows of the faces on the far boundary (x = N0, y = N1, z = N2) by the last
// cell / line / plane, every segment staged and written once with coalesced
// 16-byte stores.  A_T[p][q] = fl(fl(alpha c) + fl(beta M_pq)) is assemble_entry
// on the element's constants (M_pq = 0 across axes): bit-identical to the reference.
template <int DIM>
struct ScCell {  // what a row needs of a cell: gamma = fl(alpha c), beta, and the load entry of the slot
  double gam, b;
};

// row of slot p of a cell over its own slots q, signed: h[q] = sp sq A[p][q]
template <int DIM>
__device__ __forceinline__ void sc_row(const PencilConst<DIM>& pc, double gam, double b, int p, double (&h)[2 * DIM]) {
  const double sp = (p & 1) ? 1.0 : -1.0;
#pragma unroll
  for (int q = 0; q < 2 * DIM; ++q) {
    double mpq = 0.0;
    if ((q >> 1) == (p >> 1)) mpq = (p == q) ? ((p & 1) ? pc.md1[p >> 1] : pc.md0[p >> 1]) : pc.mo[p >> 1];
    const double apq = __dadd_rn(gam, __dmul_rn(b, mpq));
    h[q] = ((q & 1) ? sp : -sp) * apq;
  }
}

// Warp-collective: the S rows of one x-line of faces of axis ax.  Lane = plus-side
// cell x (hasp) with minus-side row hm (hasm); rows of lanes x0 <= x < x1; when
// `tail` the lane of x = x1 - 1 appends the row of the far x face (its own slot-1 row
// ht, T+ absent).  fm / fp: the signed load entries.  rs, frow: row start and row of the first face.
template <int DIM>
__device__ __forceinline__ void sc_emit(const CondArgs& C, int ax, bool valid, bool hasm, bool hasp, int x, int x0,
                                        int x1, bool tail, const double (&hm)[2 * DIM], const double (&hp)[2 * DIM],
                                        const double (&ht)[2 * DIM], double fm, double fp, double ft, long long rs,
                                        int frow, double* stg) {
  const int lane = threadIdx.x & 31;
  const int lm = hasm ? 2 * DIM : 0, lp = hasp ? 2 * DIM : 0;
  const int L = lm + lp - ((hasm && hasp) ? 1 : 0);
  int off, total;
  if (ax == 0) {  // only the row of x = 0 is short (no minus-side cell)
    off = (4 * DIM - 1) * (x - x0) - ((x0 == 0 && x > 0) ? 2 * DIM - 1 : 0);
    total = (4 * DIM - 1) * (x1 - x0) - (x0 == 0 ? 2 * DIM - 1 : 0);
  } else {
    off = L * (x - x0);
    total = L * (x1 - x0);
  }
  const int pad = static_cast<int>((reinterpret_cast<uintptr_t>(C.sval + rs) >> 3) & 1);
  if (valid) {
    int p = off + pad;
#pragma unroll
    for (int b = 0; b < DIM; ++b) {
      const double ml = hm[2 * b], mh = hm[2 * b + 1], pl = hp[2 * b], ph = hp[2 * b + 1];
      if (b == ax) {
        if (hasm) stg[p++] = ml;
        stg[p++] = (hasm && hasp) ? mh + pl : (hasm ? mh : pl);
        if (hasp) stg[p++] = ph;
      } else if (b < ax) {
        if (hasm) stg[p++] = ml, stg[p++] = mh;
        if (hasp) stg[p++] = pl, stg[p++] = ph;
      } else {
        if (hasm) stg[p++] = ml;
        if (hasp) stg[p++] = pl;
        if (hasm) stg[p++] = mh;
        if (hasp) stg[p++] = ph;
      }
    }
    __stcs(C.fs + frow + (x - x0), (hasm && hasp) ? fm + fp : (hasm ? fm : fp));
    if (tail && x == x1 - 1) {  // the far x face: this cell's slot-1 row alone
      int q = total + pad;
#pragma unroll
      for (int j = 0; j < 2 * DIM; ++j) stg[q++] = ht[j];
      __stcs(C.fs + frow + (x1 - x0), ft);
    }
  }
  if (tail) total += 2 * DIM;
  __syncwarp();
  segment_write(C.sval + (rs - pad), stg, pad, total, lane);
}

template <int DIM>
__global__ void __launch_bounds__(128, 5) k_sc_pencil(CondArgs C, PencilConst<DIM> pc, FastDiv dseg, uint32_t nwarps) {
  constexpr int N = 2 * DIM;
  __shared__ __align__(16) double stg_all[4][32 * (4 * DIM - 1) + 2 * DIM + 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * 4 + warp;
  if (gw >= nwarps) return;
  const DevMesh& m = C.m;
  const int N0 = static_cast<int>(m.N[0]), N1 = static_cast<int>(m.N[1]), N2 = DIM == 3 ? static_cast<int>(m.N[2]) : 1;
  const uint32_t line = dseg.div(gw);
  const int seg = static_cast<int>(gw - line * dseg.d);
  const uint32_t zq = m.div_n1.div(line);
  const int y = static_cast<int>(line - zq * static_cast<uint32_t>(N1)), z = static_cast<int>(zq);
  const int x0 = seg * 32, x1 = min(x0 + 32, N0), x = x0 + lane;
  const bool valid = x < N0;
  const int64_t e = x + static_cast<int64_t>(N0) * (y + static_cast<int64_t>(N1) * z);
  double* stg = stg_all[warp];
  // own cell, and the entries needed of the cells before / below / behind
  double a = 1.0, b = 1.0, f[N];
#pragma unroll
  for (int j = 0; j < N; ++j) f[j] = 0.0;
  if (valid) load_cell<DIM>(C.alpha, C.beta, C.f, e, a, b, f);
  double ya = 1.0, yb = 1.0, yf = 0.0, za = 1.0, zb = 1.0, zf = 0.0;
  if (valid && y >= 1) {
    const int64_t en = e - N0;
    ya = __ldg(C.alpha + en), yb = __ldg(C.beta + en), yf = __ldg(C.f + en * N + 3);
  }
  if (DIM == 3 && valid && z >= 1) {
    const int64_t en = e - static_cast<int64_t>(N0) * N1;
    za = __ldg(C.alpha + en), zb = __ldg(C.beta + en), zf = __ldg(C.f + en * N + (N - 1));
  }
  double xa = __shfl_up_sync(0xffffffffu, a, 1), xb = __shfl_up_sync(0xffffffffu, b, 1);
  double xf = __shfl_up_sync(0xffffffffu, f[1], 1);
  if (lane == 0 && seg > 0 && valid) {
    xa = __ldg(C.alpha + e - 1), xb = __ldg(C.beta + e - 1), xf = __ldg(C.f + (e - 1) * N + 1);
  }
  const double gam = __dmul_rn(a, pc.c);
  double hm[N], hp[N], ht[N];
  // x faces
  {
    sc_row<DIM>(pc, __dmul_rn(xa, pc.c), xb, 1, hm);
    sc_row<DIM>(pc, gam, b, 0, hp);
    sc_row<DIM>(pc, gam, b, 1, ht);
    const int face0 = face_id32(m, 0, x0, y, z);
    sc_emit<DIM>(C, 0, valid, x >= 1, true, x, x0, x1, x1 == N0, hm, hp, ht, xf, -f[0], f[1],
                 __ldg(C.rowoff + face0), face0, stg);
  }
  // y faces (and the far y boundary from the last line)
  {
    sc_row<DIM>(pc, __dmul_rn(ya, pc.c), yb, 3, hm);
    sc_row<DIM>(pc, gam, b, 2, hp);
    const int face0 = face_id32(m, 1, x0, y, z);
    sc_emit<DIM>(C, 1, valid, y >= 1, true, x, x0, x1, false, hm, hp, ht, yf, -f[2], 0.0, __ldg(C.rowoff + face0),
                 face0, stg);
    if (y == N1 - 1) {
      sc_row<DIM>(pc, gam, b, 3, hm);
      const int facet = face_id32(m, 1, x0, y + 1, z);
      sc_emit<DIM>(C, 1, valid, true, false, x, x0, x1, false, hm, hp, ht, f[3], 0.0, 0.0, __ldg(C.rowoff + facet),
                   facet, stg);
    }
  }
  if (DIM == 3) {
    sc_row<DIM>(pc, __dmul_rn(za, pc.c), zb, N - 1, hm);
    sc_row<DIM>(pc, gam, b, N - 2, hp);
    const int face0 = face_id32(m, 2, x0, y, z);
    sc_emit<DIM>(C, 2, valid, z >= 1, true, x, x0, x1, false, hm, hp, ht, zf, -f[N - 2], 0.0, __ldg(C.rowoff + face0),
                 face0, stg);
    if (z == N2 - 1) {
      sc_row<DIM>(pc, gam, b, N - 1, hm);
      const int facet = face_id32(m, 2, x0, y, z + 1);
      sc_emit<DIM>(C, 2, valid, true, false, x, x0, x1, false, hm, hp, ht, f[N - 1], 0.0, 0.0, __ldg(C.rowoff + facet),
                   facet, stg);
    }
  }
}

}  // namespace

// host check of the structure the pencil kernel relies on (reference D, M as
// packed by the space: D = hc[0, N^2), M = hc[N^2, 2 N^2))
template <int DIM>
bool pencil_setup(const double* hc, PencilConst<DIM>& pc) {
  constexpr int N = 2 * DIM;
  const double* D = hc;
  const double* M = hc + N * N;
  const double c = D[0];
  if (!(c > 0.0)) return false;
  for (int i = 0; i < N * N; ++i)
    if (D[i] != c) return false;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      if ((i >> 1) != (j >> 1) && M[i * N + j] != 0.0) return false;
      if (M[i * N + j] != M[j * N + i]) return false;
    }
  pc.c = c;
  for (int a = 0; a < DIM; ++a) {
    pc.md0[a] = M[(2 * a) * N + 2 * a];
    pc.md1[a] = M[(2 * a + 1) * N + 2 * a + 1];
    pc.mo[a] = M[(2 * a) * N + 2 * a + 1];
  }
  return true;
}
template bool pencil_setup<2>(const double*, PencilConst<2>&);
template bool pencil_setup<3>(const double*, PencilConst<3>&);

template <int DIM>
void launch_rt0_pencil(const HybArgs& a, const PencilConst<DIM>& pc, cudaStream_t st) {
  const int nseg = static_cast<int>((a.m.N[0] + 31) / 32);
  const int64_t nwarps = static_cast<int64_t>(nseg) * a.m.N[1] * (DIM == 3 ? a.m.N[2] : 1);
  const unsigned grid = static_cast<unsigned>((nwarps + kPW - 1) / kPW);
  static const bool attr_set = [] {  // once per instantiation
    return cudaFuncSetAttribute(k_rt0_pencil<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(PencilSmem<DIM>))) == cudaSuccess;
  }();
  (void)attr_set;
  k_rt0_pencil<DIM><<<grid, kPW * 32, sizeof(PencilSmem<DIM>), st>>>(a, pc, FastDiv(static_cast<uint32_t>(nseg)),
                                                                    static_cast<uint32_t>(nwarps));
  count_launch();
}
template void launch_rt0_pencil<2>(const HybArgs&, const PencilConst<2>&, cudaStream_t);
template void launch_rt0_pencil<3>(const HybArgs&, const PencilConst<3>&, cudaStream_t);

template <int DIM>
void launch_sc_pencil(const CondArgs& c, const PencilConst<DIM>& pc, cudaStream_t st) {
  const int nseg = static_cast<int>((c.m.N[0] + 31) / 32);
  const int64_t nwarps = static_cast<int64_t>(nseg) * c.m.N[1] * (DIM == 3 ? c.m.N[2] : 1);
  const unsigned grid = static_cast<unsigned>((nwarps + 3) / 4);
  k_sc_pencil<DIM><<<grid, 128, 0, st>>>(c, pc, FastDiv(static_cast<uint32_t>(nseg)), static_cast<uint32_t>(nwarps));
  count_launch();
}
template void launch_sc_pencil<2>(const CondArgs&, const PencilConst<2>&, cudaStream_t);
template void launch_sc_pencil<3>(const CondArgs&, const PencilConst<3>&, cudaStream_t);

}  // namespace hdr
