// Device CSR + the AMG / Gauss-Seidel machinery of kern_amg.cu, shared with the
// device pcg (kern_pcg.cu) and the C ABI.
#pragma once

#include <cstdint>
#include <vector>

#include "capi_util.hpp"

namespace hdr {

struct DCsr {  // device CSR: int64 row offsets, int32 columns
  int64_t n = 0, ncols = 0, nnz = 0;
  DBuf<int64_t> ro;
  DBuf<int32_t> ci;
  DBuf<double> v;
};

struct AmgHier;  // hierarchy + sweep state (kern_amg.cu)

// Gauss-Seidel sweep state of one matrix: ready flags and the level orders
// (rows sorted by their dependency depth in the forward / backward sweep),
// built on first use
struct SweepState {
  DBuf<int> flags, fwd, bwd, lvl_fwd, lvl_bwd;  // orders and level offsets
  DBuf<int64_t> eoff_fwd, eoff_bwd;              // entry offsets of the rows in level order
  int64_t max_level_nnz = 0, max_level_rows = 0, max_row_len = 0;
  std::vector<int64_t> h_eo_fwd, h_eo_bwd;  // host copies for the one-CTA batch plan
  std::vector<int> h_off_fwd, h_off_bwd;
  DBuf<int> bat_fwd, bat_bwd;  // one-CTA sweeps: batch starts (rows of one level)
  int nbat_fwd = 0, nbat_bwd = 0;
  int levels_fwd = 0, levels_bwd = 0;
  bool ready = false;
};

// copy of a device CSR matrix (int32 or int64 columns) into a DCsr
void dcsr_from_device(int64_t n, int64_t ncols, const int64_t* ro, const int32_t* ci32, const int64_t* ci64,
                      const double* v, DCsr& out, cudaStream_t st);
void dcsr_from_host(int64_t n, int64_t ncols, const int64_t* ro, const int64_t* ci, const double* v, DCsr& out,
                    cudaStream_t st);
void dcsr_to_host(const DCsr& a, int64_t* ro, int64_t* ci, double* v, cudaStream_t st);

// amg_setup (src/amg.cpp:189-244); consumes `fine`
AmgHier* amg_setup_device(DCsr&& fine, const hdr_amg_options& o, cudaStream_t st);
void amg_destroy(AmgHier* h);
int64_t amg_levels(const AmgHier* h);
const DCsr& amg_matrix(const AmgHier* h, int64_t level, int which);  // 0 A, 1 P, 2 R (level == levels: coarse A)
// one V(1,1) cycle z = M^-1 r (device vectors of the fine size)
void amg_apply_device(AmgHier* h, const double* r, double* z);
// the sweep machinery alone (SGS): context + forward scratch
AmgHier* sweep_context(int64_t n, cudaStream_t st);
double* sweep_scratch(AmgHier* h);
// symmetric Gauss-Seidel apply of A
void sgs_apply_device(AmgHier* h, const DCsr& A, SweepState& sw, double* zf, const double* r, double* z);
// sticky device status of the sweeps (ZeroDiagonal)
hdr_status amg_status(AmgHier* h);
// check_symmetric (src/solvers.cpp:25-30): max|A - A^T| and max|A| on the device
void symmetry_gap(const DCsr& a, double* diff, double* amax, cudaStream_t st);
// positive diagonal check; returns the smallest bad row or -1
int64_t positive_inv_diag(const DCsr& a, DBuf<double>& dinv, cudaStream_t st);

}  // namespace hdr
