// K1: analytic CSR patterns of H (hybridize) and S (static_condense), built once
// per space on the device.
//
// Reference: hybridize collects per-element triplets over the sorted multiplier
// rows of each cell (src/reduction.cpp:304-337) and from_triplets sorts them
// (src/csr.cpp:43-75); multiplier rows are interior faces in ascending face order
// times dofs_per_face (multiplier_base, src/reduction.cpp:88-98).  So the H row
// of a face F holds, ascending, the multiplier dofs of the interior faces of F's
// two cells.  static_condense's S (src/reduction.cpp:509-555) is indexed by the
// master global face dofs; its row of a face holds all faces of that face's cells.
// Both are enumerated here with the same col_rank the element kernels scatter
// with, so pattern and scatter agree by construction; tests pin the result
// against the reference bit for bit.
#include "hdr_device.cuh"
#include "kernels.hpp"

namespace hdr {

namespace {

__device__ inline int interior_faces_of(const DevMesh& m, const int64_t c[3]) {
  int k = 0;
  for (int s = 0; s < 2 * m.dim; ++s) {
    bool in;
    slot_face(m, c, s, &in);
    k += in;
  }
  return k;
}

__global__ void k_face_counts(DevMesh m, int* flag, int64_t* fnnz_h, int64_t* fnnz_s) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= m.nfaces) return;
  int64_t cm, cp, co[3];
  face_cells(m, f, &cm, &cp, co);
  const bool in = (cm >= 0 && cp >= 0);
  flag[f] = in;
  const int64_t d2 = static_cast<int64_t>(m.dpf) * m.dpf;
  if (in) {
    int64_t a[3], b[3];
    cell_coords(m, cm, a);
    cell_coords(m, cp, b);
    fnnz_h[f] = d2 * (interior_faces_of(m, a) + interior_faces_of(m, b) - 1);
    fnnz_s[f] = d2 * (4 * m.dim - 1);
  } else {
    fnnz_h[f] = 0;
    fnnz_s[f] = d2 * (2 * m.dim);
  }
}

__global__ void k_mbase(DevMesh m, const int* flag, const int* ord, int* mbase) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= m.nfaces) return;
  mbase[f] = flag[f] ? ord[f] * m.dpf : -1;
}

__global__ void k_fill_patterns(DevMesh m, const int* mbase, const int64_t* fbase_h, const int64_t* fbase_s,
                                int64_t* row_h, int32_t* col_h, int64_t* row_s, int32_t* col_s, int64_t nrows_h,
                                int64_t nnz_h, int64_t nrows_s, int64_t nnz_s) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f == 0) {
    row_h[nrows_h] = nnz_h;
    row_s[nrows_s] = nnz_s;
  }
  if (f >= m.nfaces) return;
  const int dpf = m.dpf, nsl = 2 * m.dim;
  int64_t cm, cp, co[3];
  const int a = face_cells(m, f, &cm, &cp, co);
  const bool in = (cm >= 0 && cp >= 0);
  const int64_t cells2[2] = {cm, cp};

  // S rows: every face is a master (b = face dofs, src/reduction.cpp:474)
  const int us = in ? 4 * m.dim - 1 : 2 * m.dim;
  for (int sub = 0; sub < dpf; ++sub) row_s[f * dpf + sub] = fbase_s[f] + static_cast<int64_t>(sub) * dpf * us;
  for (int w = 0; w < 2; ++w) {
    if (cells2[w] < 0) continue;
    int64_t c[3], own_f[6];
    bool own_in[6];
    cell_coords(m, cells2[w], c);
    for (int t = 0; t < nsl; ++t) own_f[t] = slot_face(m, c, t, &own_in[t]);
    const int s = 2 * a + (w == 0 ? 1 : 0);  // F is the +a face of cm, the -a face of cp
    for (int t = 0; t < nsl; ++t) {
      const int pos = col_rank(m, c, s, t, own_f, own_in, true);
      for (int sub = 0; sub < dpf; ++sub)
        for (int sj = 0; sj < dpf; ++sj)
          col_s[row_s[f * dpf + sub] + static_cast<int64_t>(pos) * dpf + sj] = static_cast<int32_t>(own_f[t] * dpf + sj);
    }
  }
  if (!in) return;
  // H rows
  const int mb = mbase[f];
  int64_t ca[3], cb[3];
  cell_coords(m, cm, ca);
  cell_coords(m, cp, cb);
  const int u = interior_faces_of(m, ca) + interior_faces_of(m, cb) - 1;
  for (int sub = 0; sub < dpf; ++sub) row_h[mb + sub] = fbase_h[f] + static_cast<int64_t>(sub) * dpf * u;
  for (int w = 0; w < 2; ++w) {
    int64_t c[3], own_f[6];
    bool own_in[6];
    cell_coords(m, cells2[w], c);
    for (int t = 0; t < nsl; ++t) own_f[t] = slot_face(m, c, t, &own_in[t]);
    const int s = 2 * a + (w == 0 ? 1 : 0);
    for (int t = 0; t < nsl; ++t) {
      if (!own_in[t]) continue;
      const int pos = col_rank(m, c, s, t, own_f, own_in, false);
      const int gb = mbase[own_f[t]];
      for (int sub = 0; sub < dpf; ++sub)
        for (int sj = 0; sj < dpf; ++sj) col_h[row_h[mb + sub] + static_cast<int64_t>(pos) * dpf + sj] = gb + sj;
    }
  }
}

// k = 0 scatter metadata: per face {start of its H row, row} in one 16-byte word
// (row = -1 and start = 0 on the boundary), so the hybridize kernel reaches a
// row with one load instead of the mbase -> rowoff chain
__global__ void k_face_rows(int64_t nfaces, const int* mbase, const int64_t* rowoff, longlong2* frs) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nfaces) return;
  const int mb = mbase[f];
  frs[f] = make_longlong2(mb >= 0 ? rowoff[mb] : 0, mb);
}

}  // namespace

void launch_face_rows(int64_t nfaces, const int* mbase, const int64_t* rowoff, longlong2* frs, cudaStream_t st) {
  k_face_rows<<<static_cast<unsigned>((nfaces + 255) / 256), 256, 0, st>>>(nfaces, mbase, rowoff, frs);
  count_launch();
}

void launch_face_counts(const DevMesh& m, int* flag, int64_t* fnnz_h, int64_t* fnnz_s, cudaStream_t st) {
  const int64_t nb = (m.nfaces + 255) / 256;
  k_face_counts<<<static_cast<unsigned>(nb), 256, 0, st>>>(m, flag, fnnz_h, fnnz_s);
  count_launch();
}
void launch_mbase(const DevMesh& m, const int* flag, const int* ord, int* mbase, cudaStream_t st) {
  const int64_t nb = (m.nfaces + 255) / 256;
  k_mbase<<<static_cast<unsigned>(nb), 256, 0, st>>>(m, flag, ord, mbase);
  count_launch();
}
void launch_fill_patterns(const DevMesh& m, const int* mbase, const int64_t* fbase_h, const int64_t* fbase_s,
                          int64_t* row_h, int32_t* col_h, int64_t* row_s, int32_t* col_s, int64_t nrows_h,
                          int64_t nnz_h, int64_t nrows_s, int64_t nnz_s, cudaStream_t st) {
  const int64_t nb = (m.nfaces + 127) / 128;
  k_fill_patterns<<<static_cast<unsigned>(nb), 128, 0, st>>>(m, mbase, fbase_h, fbase_s, row_h, col_h, row_s, col_s,
                                                              nrows_h, nnz_h, nrows_s, nnz_s);
  count_launch();
}

}  // namespace hdr

namespace hdr {

std::vector<uint64_t> rank_table_rt0(int dim) {
  const int N = 2 * dim, nflags = 1 << (2 * dim + 1);
  std::vector<uint64_t> tab(static_cast<size_t>(N) * nflags * 2, 0);
  for (int k = 0; k < N; ++k)
    for (int flags = 0; flags < nflags; ++flags) {
      const unsigned all = (1u << dim) - 1u;
      const unsigned lo = flags & all, hi = (flags >> dim) & all, far = (flags >> (2 * dim)) & 1u;
      const int a = k >> 1, side = k & 1;
      uint64_t own = ~uint64_t(0), nbr = ~uint64_t(0);
      const bool kin = side ? ((hi >> a) & 1u) : ((lo >> a) & 1u);
      if (kin) {
        // neighbour across k: same flags off axis a; along a its face k^1 is the
        // shared (interior) face and its face k is the far face
        unsigned nlo = lo, nhi = hi;
        if (side) {
          nlo |= (1u << a);
          nhi = (nhi & ~(1u << a)) | (far << a);
        } else {
          nhi |= (1u << a);
          nlo = (nlo & ~(1u << a)) | (far << a);
        }
        // the face beyond our cell, seen from the neighbour, is our face k^1
        const int nfar = side ? static_cast<int>((lo >> a) & 1u) : static_cast<int>((hi >> a) & 1u);
        for (int q = 0; q < N; ++q) {
          const bool qin = (q & 1) ? ((hi >> (q >> 1)) & 1u) : ((lo >> (q >> 1)) & 1u);
          if (qin) {
            const uint64_t r = static_cast<uint64_t>(col_rank_flags(k, q, lo, hi, 1, static_cast<int>(far)));
            own = (own & ~(uint64_t(15) << (4 * q))) | (r << (4 * q));
          }
          const bool nin = (q & 1) ? ((nhi >> (q >> 1)) & 1u) : ((nlo >> (q >> 1)) & 1u);
          if (nin && q != (k ^ 1)) {
            const uint64_t r = static_cast<uint64_t>(col_rank_flags(k ^ 1, q, nlo, nhi, 1, nfar));
            nbr = (nbr & ~(uint64_t(15) << (4 * q))) | (r << (4 * q));
          }
        }
      }
      tab[(static_cast<size_t>(k) * nflags + flags) * 2] = own;
      tab[(static_cast<size_t>(k) * nflags + flags) * 2 + 1] = nbr;
    }
  return tab;
}

}  // namespace hdr
