// Host-side launch wrappers of the device kernels (one per .cu translation unit).
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "hdr_device.cuh"

namespace hdr {

// counts every kernel this library launches (hdr_launch_count)
void count_launch(int64_t k = 1);

// ---- K1 patterns (kern_pattern.cu)
void launch_face_counts(const DevMesh& m, int* flag, int64_t* fnnz_h, int64_t* fnnz_s, cudaStream_t st);
void launch_mbase(const DevMesh& m, const int* flag, const int* ord, int* mbase, cudaStream_t st);
void launch_fill_patterns(const DevMesh& m, const int* mbase, const int64_t* fbase_h, const int64_t* fbase_s,
                          int64_t* row_h, int32_t* col_h, int64_t* row_s, int32_t* col_s, int64_t nrows_h,
                          int64_t nnz_h, int64_t nrows_s, int64_t nnz_s, cudaStream_t st);

// ---- structured element solve (kern_hybridize.cu)
struct Fixed {  // device pointers to the per-space fixed factors (see hdr_internal.hpp)
  const double *D, *M, *E, *Ma, *N0, *X, *lam;
  int r;
  double rho;
};

struct HybArgs {
  DevMesh m;
  Fixed fx;
  int nF;        // face dofs per cell = 2*dim*dpf
  int p_max;     // highest Neumann order allowed
  const double *alpha, *beta, *f;
  const int* mbase;
  const int64_t* rowoff;
  double* hval;  // H values (pattern order)
  double* g;     // reduced rhs (m)
  int* status;   // device flag: bit 0 = Neumann ratio out of range
  const uint64_t* rank_tab;  // k = 0 row-rank table (rank_table_rt0)
};

// Row-rank table of the k = 0 kernel: for row slot k and boundary flags
// (own lo bits | own hi bits << dim | neighbour far face << 2 dim), two words of
// 4-bit column ranks (own slots, then the neighbour's slots; 15 = absent).
std::vector<uint64_t> rank_table_rt0(int dim);

// Small-element path (k = 0): one thread per cell, everything in registers.
void launch_hybridize_rt0(const HybArgs& a, const double* host_consts, int parity, cudaStream_t st);
// k = 0, lane-per-row form with row-complete writes (stage: parity_count * N*(N+1) doubles)
void launch_hybridize_rt0_rows(const HybArgs& a, const double* host_consts, double* stage, cudaStream_t st);
// k >= 1 with nF + 1 <= 32 (RT1 hexes, RT1..RT3 quads): one warp per cell (kern_warp.cu)
bool hybridize_warp_supported(int dim, int k);
int64_t hybridize_warp_scratch_doubles(const HybArgs& a);
void launch_hybridize_warp(const HybArgs& a, int parity, double* gws, cudaStream_t st);
// RT2 / RT3 hexahedra: one CTA per cell (kern_cta.cu)
bool hybridize_big_supported(int dim, int k);
int64_t hybridize_big_scratch_doubles(const HybArgs& a, int k);
void launch_hybridize_big(const HybArgs& a, int k, int parity, double* gws, cudaStream_t st);
// General path (k >= 1): one CTA per cell, shared-memory or global workspace.
void launch_hybridize_cta(const HybArgs& a, int parity, double* gws, int64_t ws_doubles, cudaStream_t st);
int64_t hybridize_cta_ws_doubles(const DevMesh& m, int nF, int r, int p_max, bool* use_smem);

// ---- hybrid recovery: x_hat = A^-1 (f - C^T lambda) per cell (kern_hybridize.cu)
struct RecArgs {
  DevMesh m;
  Fixed fx;
  int nF, p_max;
  const double *alpha, *beta, *f, *lambda;
  const int* mbase;
  double* x_hat;  // broken
  double* x;      // global (ndofs): face dofs averaged, bubbles copied
  int* status;
};
void launch_recover_hybrid(const RecArgs& a, double* gws, int64_t ws_doubles, cudaStream_t st);
void launch_average_faces(const DevMesh& m, const double* x_hat, double* x, cudaStream_t st);

// ---- static condensation / recover_condensed (kern_condense.cu)
struct CondArgs {
  DevMesh m;
  Fixed fx;
  int nF;
  const double *alpha, *beta, *f;
  const int64_t* rowoff;  // S pattern
  double* sval;
  double* fs;
  const double* xb;  // recover_condensed input (nS)
  double* x;         // recover_condensed output (ndofs)
  int* status;       // bit 1: A_ii not SPD
};
void launch_condense(const CondArgs& c, int parity, double* gws, int64_t ws_doubles, cudaStream_t st);
int64_t condense_ws_doubles(const DevMesh& m, int nF);
void launch_recover_condensed(const CondArgs& c, double* gws, int64_t ws_doubles, cudaStream_t st);

// ---- spmv (kern_spmv.cu)
void launch_spmv32(int64_t nrows, const int64_t* ro, const int32_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st);
void launch_spmv64(int64_t nrows, const int64_t* ro, const int64_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st);

}  // namespace hdr
