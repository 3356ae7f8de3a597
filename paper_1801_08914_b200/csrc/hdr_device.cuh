// Device-side helpers: mesh numbering, error-free transforms, parameter blocks.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace hdr {

constexpr int kMaxN = 240;  // RT3 hexahedron
constexpr int kMaxR = 64;

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
};

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

// ------------------------------------------------------------ error-free transforms

__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = __fma_rn(a, b, -p);
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

}  // namespace hdr
