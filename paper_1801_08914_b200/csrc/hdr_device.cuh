// Device-side helpers: mesh numbering, error-free transforms, parameter blocks.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace hdr {

constexpr int kMaxN = 240;  // RT3 hexahedron
constexpr int kMaxR = 64;

// Unsigned 32-bit division by a runtime-invariant divisor via a precomputed
// magic multiplier (round-up method): q = (umulhi(n, m) + n) >> l.
struct FastDiv {
  uint32_t d = 1, m = 0, l = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    l = 0;
    while ((uint64_t(1) << l) < div) ++l;
    m = static_cast<uint32_t>(((uint64_t(1) << 32) * ((uint64_t(1) << l) - div)) / div + 1);
  }
  __host__ __device__ inline uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    const uint32_t hi = __umulhi(n, m);
#else
    const uint32_t hi = static_cast<uint32_t>((static_cast<uint64_t>(n) * m) >> 32);
#endif
    return static_cast<uint32_t>((static_cast<uint64_t>(hi) + n) >> l);
  }
};

// Structured mesh numbering (src/mesh.cpp:13-135): cells lexicographic x fastest;
// faces grouped by axis, lexicographic in the (N + e_axis) grid; a cell's faces
// in slot order (-x,+x,-y,+y,-z,+z) with outward signs -1,+1.
struct DevMesh {
  int dim;
  int dpf;     // dofs per face
  int n;       // element dofs
  int nint;    // interior (bubble) dofs per cell
  int64_t N[3];
  int64_t foff[3];  // first face index of each axis group
  int64_t nfaces, ncells, face_dof_count;
  FastDiv div_half, div_n0, div_n1;  // (N0+1)/2, N0, N1
};

// 32-bit fast paths (every mesh the device path accepts has < 2^31 cells and faces)
__host__ __device__ inline void cell_coords32(const DevMesh& m, uint32_t cell, int c[3]) {
  const uint32_t r = m.div_n0.div(cell);
  c[0] = static_cast<int>(cell - r * static_cast<uint32_t>(m.N[0]));
  const uint32_t z = m.div_n1.div(r);
  c[1] = static_cast<int>(r - z * static_cast<uint32_t>(m.N[1]));
  c[2] = static_cast<int>(z);
}
// parity_cell in 32-bit: t -> (cell or -1, coordinates)
__host__ __device__ inline int parity_cell32(const DevMesh& m, int parity, uint32_t t, int c[3]) {
  const uint32_t half = static_cast<uint32_t>((m.N[0] + 1) / 2);
  const uint32_t row = m.div_half.div(t);
  const uint32_t j = t - row * half;
  const uint32_t z = m.div_n1.div(row);
  const uint32_t y = row - z * static_cast<uint32_t>(m.N[1]);
  if (z >= static_cast<uint32_t>(m.N[2])) return -1;
  const uint32_t x = ((parity + y + z) & 1u) + 2u * j;
  if (x >= static_cast<uint32_t>(m.N[0])) return -1;
  c[0] = static_cast<int>(x);
  c[1] = static_cast<int>(y);
  c[2] = static_cast<int>(z);
  return static_cast<int>(x + static_cast<uint32_t>(m.N[0]) * (y + static_cast<uint32_t>(m.N[1]) * z));
}
__host__ __device__ inline int face_id32(const DevMesh& m, int axis, int x, int y, int z) {
  const int d0 = static_cast<int>(m.N[0]) + (axis == 0), d1 = static_cast<int>(m.N[1]) + (axis == 1);
  const int off = static_cast<int>(axis == 0 ? m.foff[0] : (axis == 1 ? m.foff[1] : m.foff[2]));
  return off + x + d0 * (y + d1 * z);
}

__host__ __device__ inline int64_t face_id(const DevMesh& m, int axis, int64_t x, int64_t y, int64_t z) {
  const int64_t d0 = m.N[0] + (axis == 0), d1 = m.N[1] + (axis == 1);
  return m.foff[axis] + x + d0 * (y + d1 * z);
}

__host__ __device__ inline void cell_coords(const DevMesh& m, int64_t cell, int64_t c[3]) {
  c[0] = cell % m.N[0];
  const int64_t r = cell / m.N[0];
  c[1] = r % m.N[1];
  c[2] = r / m.N[1];
}

// face of slot s of the cell at c; interior iff the cell across it exists.
// (Written without dynamic indexing of local arrays: an earlier form with
// x[a] += side miscompiled under nvcc 12.9 -O3 for sm_100a.)
__host__ __device__ inline int64_t slot_face(const DevMesh& m, const int64_t c[3], int s, bool* interior) {
  const int a = s >> 1, side = s & 1;
  const int64_t c0 = c[0], c1 = c[1], c2 = c[2];
  const int64_t x0 = c0 + (a == 0 ? side : 0), x1 = c1 + (a == 1 ? side : 0), x2 = c2 + (a == 2 ? side : 0);
  const int64_t ca = a == 0 ? c0 : (a == 1 ? c1 : c2);
  const int64_t na = a == 0 ? m.N[0] : (a == 1 ? m.N[1] : m.N[2]);
  if (interior) *interior = side ? (ca + 1 < na) : (ca > 0);
  const int64_t d0 = m.N[0] + (a == 0), d1 = m.N[1] + (a == 1);
  const int64_t off = a == 0 ? m.foff[0] : (a == 1 ? m.foff[1] : m.foff[2]);
  return off + x0 + d0 * (x1 + d1 * x2);
}

// face f -> axis and the two adjacent cells (-1 if absent)   (mesh.cpp:94-120)
__host__ __device__ inline int face_cells(const DevMesh& m, int64_t f, int64_t* cm, int64_t* cp, int64_t co[3]) {
  int a = m.dim - 1;
  for (int b = 1; b < m.dim; ++b)
    if (f < m.foff[b]) {
      a = b - 1;
      break;
    }
  int64_t local = f - m.foff[a];
  const int64_t d0 = m.N[0] + (a == 0), d1 = m.N[1] + (a == 1);
  co[0] = local % d0;
  local /= d0;
  co[1] = local % d1;
  co[2] = local / d1;
  const int64_t plane = a == 0 ? co[0] : (a == 1 ? co[1] : co[2]);
  const int64_t na = a == 0 ? m.N[0] : (a == 1 ? m.N[1] : m.N[2]);
  *cm = -1;
  *cp = -1;
  if (plane > 0) {
    const int64_t x0 = co[0] - (a == 0), x1 = co[1] - (a == 1), x2 = co[2] - (a == 2);
    *cm = x0 + m.N[0] * (x1 + m.N[1] * x2);
  }
  if (plane < na) *cp = co[0] + m.N[0] * (co[1] + m.N[1] * co[2]);
  return a;
}

// cells of one checkerboard colour: t -> cell (or -1).  Every face joins cells
// of opposite colours, so two passes give a race-free deterministic scatter.
__host__ __device__ inline int64_t parity_cell(const DevMesh& m, int parity, int64_t t) {
  const int64_t half = (m.N[0] + 1) / 2;
  const int64_t row = t / half, j = t - row * half;
  const int64_t y = row % m.N[1], z = row / m.N[1];
  if (z >= m.N[2]) return -1;
  const int64_t x = ((parity + y + z) & 1) + 2 * j;
  if (x >= m.N[0]) return -1;
  return x + m.N[0] * (y + m.N[1] * z);
}
__host__ __device__ inline int64_t parity_count(const DevMesh& m) { return ((m.N[0] + 1) / 2) * m.N[1] * m.N[2]; }

// Rank of own face slot t among the column faces of the row of the face at own
// slot s.  H rows (all_faces = false): the interior faces of this cell and of
// its neighbour across s, ascending (hybridize's from_triplets order).  S rows
// (all_faces = true): every face of the (one or two) cells of that face
// (static_condense's master ordinals are the global face dofs).
__host__ __device__ inline int col_rank(const DevMesh& m, const int64_t c[3], int s, int t, const int64_t* own_f,
                                        const bool* own_int, bool all_faces = false) {
  int r = 0;
  for (int u = 0; u < t; ++u) r += (all_faces || own_int[u]);
  if (!own_int[s]) return r;  // boundary face: the row holds this cell's faces only
  const int a = s >> 1, side = s & 1;
  const int64_t step = side ? 1 : -1;
  const int64_t nb[3] = {c[0] + (a == 0 ? step : 0), c[1] + (a == 1 ? step : 0), c[2] + (a == 2 ? step : 0)};
  const int shared = 2 * a + (1 - side);
  const int64_t ft = own_f[t];
  for (int v = 0; v < 2 * m.dim; ++v) {
    if (v == shared) continue;
    bool in;
    const int64_t f = slot_face(m, nb, v, &in);
    r += ((all_faces || in) && f < ft);
  }
  return r;
}

// Closed form of col_rank.  Face ids are grouped by axis (all x-faces < all
// y-faces < all z-faces) and, inside an axis-b group, the four b-faces of a cell
// c and its neighbour nb = c +- e_a order by the b-grid strides (s_a < s_b iff
// a < b, and s_a >= 2 s_b for a > b).  in_lo[b] / in_hi[b]: c's -b / +b faces
// are interior; the neighbour's b-faces (b != a) share those flags.  all_faces:
// count boundary faces too (S rows).  Pinned against col_rank by
// tests/test_host.py::test_closed_form_ranks.
struct CellFlags {
  bool lo[3], hi[3];
  bool far_lo, far_hi;  // c_a >= 2 / c_a + 2 < N_a: neighbour's far a-face interior
};

// Column rank from boundary flags only: lo / hi (bit x set iff the cell's -x / +x
// face is interior), own_p_in (slot p's face interior), far (the face beyond the
// neighbour across p interior).
__host__ __device__ constexpr int col_rank_flags(int p, int q, unsigned L, unsigned H, int own_p_in, int far) {
  const int a = p >> 1, sp = p & 1, b = q >> 1, sq = q & 1;
  if (!own_p_in) {  // boundary row (S only): this cell's faces in slot order
    int r = 0;
    for (int u = 0; u < q; ++u) r += ((u & 1) ? (H >> (u >> 1)) : (L >> (u >> 1))) & 1u;
    return r;
  }
  const int La = (L >> a) & 1u, Ha = (H >> a) & 1u, Lb = (L >> b) & 1u, Hb = (H >> b) & 1u;
  int r = 0;
  for (int x = 0; x < b; ++x)
    r += (x == a) ? (sp ? La + 1 + far : far + 1 + Ha) : 2 * static_cast<int>(((L >> x) & 1u) + ((H >> x) & 1u));
  if (b == a) {
    if (sp) r += sq ? La : 0;
    else r += sq ? far + 1 : far;
  } else if (sp) {
    if (sq) r += (a < b) ? 2 * Lb : Lb;
  } else {
    if (a < b) r += sq ? 2 * Lb + Hb : Lb;
    else r += sq ? 2 * Lb + Hb : Lb + Hb;
  }
  return r;
}

__host__ __device__ constexpr int col_rank_fast(int dim, int p, int q, unsigned lo, unsigned hi, int64_t ca, int64_t na,
                                             bool all_faces) {
  const int sp = p & 1;
  const int own_p_in = sp ? (ca + 1 < na) : (ca > 0);
  const unsigned L = all_faces ? 7u : lo, H = all_faces ? 7u : hi;
  const int far = all_faces ? 1 : (sp ? (ca + 2 < na) : (ca >= 2));
  (void)dim;
  return col_rank_flags(p, q, L, H, own_p_in, far);
}

// ------------------------------------------------------------ L2 eviction-priority hints
// A staged intermediate that is read back by the next launch is stored evict_last
// so the streaming output written in between does not push it out of L2; the
// streaming output itself is stored evict_first.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_l2hint(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_l2hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}

// ------------------------------------------------------------ asynchronous global -> shared copies
// (cp.async: the loads are in flight while the thread computes, no registers held)
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sdst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sdst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------ error-free transforms

__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = __fma_rn(a, b, -p);
}
// the same exact (s, e) as two_sum with 3 floating-point operations instead of 6:
// Fast2Sum on the operands ordered by magnitude (the order costs a compare and
// two selects, off the fp64 pipe's critical ops)
__device__ __forceinline__ void two_sum_fast(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const bool sw = fabs(b) > fabs(a);
  const double hi = sw ? b : a, lo = sw ? a : b;
  e = __dsub_rn(lo, __dsub_rn(s, hi));
}
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// A_T entry exactly as the reference assembles it: fl(fl(alpha D) + fl(beta M))
// (rt_space.cpp:356-357 through dense_add, dense.cpp:37-42), no contraction.
__device__ __forceinline__ double assemble_entry(double alpha, double beta, double d, double m) {
  return __dadd_rn(__dmul_rn(alpha, d), __dmul_rn(beta, m));
}

// Delta_T entry of the structured solve: A_T - A0 = alpha E + beta Ma + delta,
// delta = exact rounding error of the combine.
__device__ __forceinline__ double delta_entry(double alpha, double beta, double d, double m, double e, double ma) {
  double p1, e1, p2, e2, s, e3;
  two_prod(alpha, d, p1, e1);
  two_prod(beta, m, p2, e2);
  two_sum(p1, p2, s, e3);
  const double delta = -((e1 + e2) + e3);
  return __fma_rn(alpha, e, __fma_rn(beta, ma, delta));
}


// ------------------------------------------------------------ double-double arithmetic (exact path)
// (hi, lo) pairs with |lo| <= ulp(hi) / 2; every step through the rounding
// intrinsics so no contraction can break an error-free transform.
struct ddr {
  double hi, lo;
};
__device__ __forceinline__ ddr dd_quick(double s, double e) {
  const double h = __dadd_rn(s, e);
  return {h, __dsub_rn(e, __dsub_rn(h, s))};
}
__device__ __forceinline__ ddr dd_from(double a) { return {a, 0.0}; }
__device__ __forceinline__ ddr dd_add(ddr a, ddr b) {  // accurate sum (both parts two-summed)
  double s, e, t, f;
  two_sum(a.hi, b.hi, s, e);
  two_sum(a.lo, b.lo, t, f);
  e = __dadd_rn(e, t);
  ddr r = dd_quick(s, e);
  return dd_quick(r.hi, __dadd_rn(r.lo, f));
}
__device__ __forceinline__ ddr dd_neg(ddr a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ ddr dd_mul(ddr a, ddr b) {
  double p, e;
  two_prod(a.hi, b.hi, p, e);
  e = __fma_rn(a.hi, b.lo, e);
  e = __fma_rn(a.lo, b.hi, e);
  return dd_quick(p, e);
}
__device__ __forceinline__ ddr dd_div(ddr a, ddr b) {  // three-term long division
  const double q1 = __ddiv_rn(a.hi, b.hi);
  ddr r = dd_add(a, dd_neg(dd_mul(b, dd_from(q1))));
  const double q2 = __ddiv_rn(r.hi, b.hi);
  r = dd_add(r, dd_neg(dd_mul(b, dd_from(q2))));
  const double q3 = __ddiv_rn(r.hi, b.hi);
  return dd_add(dd_quick(q1, q2), dd_from(q3));
}
// a - b * c
__device__ __forceinline__ ddr dd_fms(ddr a, ddr b, ddr c) { return dd_add(a, dd_neg(dd_mul(b, c))); }

// ------------------------------------------------------------ structured-solve order control
// (DESIGN.md §2 "Fail-safe").  q = max|first-order term| / max|zero-order term|
// of the cell, measured a posteriori.  After P Neumann orders the remainder is
// estimated as 10 q^(P+1) (geometric tail, q < 0.25); the fp32 / TF32 evaluation
// of the correction terms adds about q * eps of |H_T| (eps: the relative
// accuracy of the correction arithmetic, set per kernel by the host,
// kStructEps*).  A cell whose estimated error exceeds kStructTol of its own
// |H_T|, or whose q is not < 0.25, is not accepted: it is marked for the exact
// path (double-double LU of A_T, kern_exact.cu) and contributes nothing here.
constexpr double kStructTol = 1e-12;
__device__ __forceinline__ int struct_order(double q, int p_max, double eps, bool& exact) {
  if (!(q < 0.25)) {
    exact = true;
    return 1;
  }
  int P = 1;
  double t = 10.0 * q * q;
  while (t > kStructTol && P < p_max) {
    ++P;
    t *= q;
  }
  exact = t > kStructTol || q * eps > kStructTol;
  return P;
}
// a-priori form (fp64 corrections: recovery): tau = rho alpha / beta bounds the
// Neumann ratio; remainder tau^(P+1)
__device__ __forceinline__ int struct_order_apriori(double tau, int p_max, bool& exact) {
  if (!(tau < 0.25)) {
    exact = true;
    return 1;
  }
  int P = 1;
  double t = tau * tau;
  while (t > 1e-14 && P < p_max) {
    ++P;
    t *= tau;
  }
  exact = t > 1e-14;
  return P;
}
// appends cell e to the exact-path list (capacity = cells of the mesh)
__device__ __forceinline__ void exact_push(int* list, int* count, int e) {
  const int s = atomicAdd(count, 1);
  list[s] = e;
}

}  // namespace hdr
