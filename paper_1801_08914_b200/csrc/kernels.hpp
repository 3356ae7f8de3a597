// Host-side launch wrappers of the device kernels (one per .cu translation unit).
#pragma once

#include <cstdint>

#include "../../include/hdivred_b200.h"
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
  // RT2 / RT3 hexes: Delta's inputs in the tensor-core chunk order of
  // kern_cta.cu (chunk c, row m < MP, k < 16 -> column 16 c + k; zero padded)
  const double2* dtab;  // {D, M}
  const float2* etab;   // {E, Ma} (tiny: fp32 carries them to 6e-8 relative)
  // warp-kernel spaces (RT1 hexes, RT1-3 quads): the same inputs as two sections of
  // entries, each padded to a multiple of 128 with copies of its last entry: first
  // the entries whose M and Ma are exactly zero (the mass matrix couples one vector
  // component only: delta is then the rounding error of fl(alpha D) alone), then the
  // rest; tix = (l << 16) | i of the entry (i, l), which Delta^T stores at l * ld + i
  const double2* tdm;   // {D, M}
  const float2* tem;    // {E, Ma}
  const int* tix;
  int tz, tn;           // padded length of the zero-mass section, of both sections
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
  int* status;   // device flag (bit 2: singular block on the exact path)
  const uint64_t* rank_tab;  // k = 0 row-rank table (rank_table_rt0)
  const longlong2* frs;      // k = 0: per face {rowoff[mbase[face]], mbase[face]} (launch_face_rows)
  // fail-safe (hdr_device.cuh struct_order): cells the structured solve does not
  // accept contribute nothing and are listed for the exact path (kern_exact.cu);
  // k = 0 kernels solve them in place instead (double-double, per thread)
  int* xlist;    // exact-path cells (capacity ncells)
  int* xcount;   // [0]: their number (reset before each call); [2]: k = 0 brick kernels' list length
  double eps32;  // relative accuracy of the fp32 correction arithmetic of this kernel
  double eps_tc; // same for the tcgen05 3xTF32 form (k_hyb_big)
  int force_exact;  // testing: send every cell to the exact path
  float* qlog;      // optional per-cell q (diagnostics)
};
void launch_face_rows(int64_t nfaces, const int* mbase, const int64_t* rowoff, longlong2* frs, cudaStream_t st);

// Row-rank table of the k = 0 kernel: for row slot k and boundary flags
// (own lo bits | own hi bits << dim | neighbour far face << 2 dim), two words of
// 4-bit column ranks (own slots, then the neighbour's slots; 15 = absent).
std::vector<uint64_t> rank_table_rt0(int dim);

// k = 0, one-pass pencil kernel (kern_pencil.cu): reference element with D = c 1 1^T
// and axis-block-diagonal M (checked by pencil_setup on the packed constants)
template <int DIM>
struct PencilConst {
  double c;                          // every entry of the reference divdiv
  double md0[DIM], md1[DIM], mo[DIM];  // the 2 x 2 mass block of each axis
};
template <int DIM>
bool pencil_setup(const double* host_consts, PencilConst<DIM>& pc);
template <int DIM>
void launch_rt0_pencil(const HybArgs& a, const PencilConst<DIM>& pc, cudaStream_t st);

// k = 0, lane-per-row form with row-complete writes (stage: parity_count * N*(N+1) doubles)
void launch_hybridize_rt0_rows(const HybArgs& a, const double* host_consts, double* stage, cudaStream_t st);
// k >= 1 with nF + 1 <= 32 (RT1 hexes, RT1..RT3 quads): one warp per cell (kern_warp.cu)
bool hybridize_warp_supported(int dim, int k);
int64_t hybridize_warp_scratch_doubles(const HybArgs& a);
// pre (3D RT1): (N + R) x ncells column-major [N0 f_e ; X^T f_e] (launch_gemm_f64_nn), else nullptr
void launch_hybridize_warp(const HybArgs& a, int parity, double* gws, const double* pre, cudaStream_t st);
// RT2 / RT3 hexahedra: one CTA per cell (kern_cta.cu)
bool hybridize_big_supported(int dim, int k);
int64_t hybridize_big_scratch_doubles(const HybArgs& a, int k);
// pre: (N + R) x ncells column-major [N0 f_e ; X^T f_e] (launch_gemm_f64_nn with A = [N0 ; X^T])
void launch_hybridize_big(const HybArgs& a, int k, int parity, double* gws, const double* pre, cudaStream_t st);
// C (M x Ncol) = A (M x Kd) B (Kd x Ncol), column-major fp64
void launch_gemm_f64_nn(int M, int Ncol, int Kd, const double* A, int lda, const double* B, int ldb, double* C,
                        int ldc, cudaStream_t st);

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
  int* xlist;     // exact-path cells (see HybArgs)
  int* xcount;
  int force_exact;
};
void launch_recover_hybrid(const RecArgs& a, double* gws, int64_t ws_doubles, cudaStream_t st);
// k = 0: one thread per cell (host_consts as launch_hybridize_rt0_rows)
void launch_recover_rt0(const RecArgs& a, const double* host_consts, cudaStream_t st);
void launch_average_faces(const DevMesh& m, const double* x_hat, double* x, cudaStream_t st);

// ---- exact path (kern_exact.cu): double-double LU of A_T = fl(fl(alpha D) + fl(beta M))
// for the cells the structured solve did not accept (xlist / xcount), one CTA per cell
enum { EXACT_HYB = 0, EXACT_REC = 1 };
struct ExactArgs {
  DevMesh m;
  int n, nF, mode;
  const double *D, *M;  // reference element (n x n row-major)
  const double *alpha, *beta, *f, *lambda;
  const int* mbase;
  const int64_t* rowoff;
  double *hval, *g, *x_hat;
  const int* xlist;
  const int* xcount;
  int* status;  // bit 2: singular block (the reference's rule)
  unsigned long long* bad;  // smallest singular cell
};
int exact_grid(int n);                   // CTAs of one exact launch
int64_t exact_ws_doubles(int n, int nF);  // global scratch of one launch
// HYB: adds the listed cells of colour `parity` to H, g (their fast-path contributions are zero)
// REC: writes x_hat of the listed cells (before k_average)
void launch_exact(const ExactArgs& a, int parity, double* ws, cudaStream_t st);

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
  const double* host_consts = nullptr;  // k = 0: the packed host constants (pencil_setup), else null
};
// k = 0 static condensation in one pass (kern_pencil.cu), for elements with the pencil structure
template <int DIM>
void launch_sc_pencil(const CondArgs& c, const PencilConst<DIM>& pc, cudaStream_t st);
void launch_condense(const CondArgs& c, int parity, double* gws, int64_t ws_doubles, cudaStream_t st);
int64_t condense_ws_doubles(const DevMesh& m, int nF);
void launch_recover_condensed(const CondArgs& c, double* gws, int64_t ws_doubles, cudaStream_t st);

// ---- spmv (kern_spmv.cu)
// nnz (when known) selects the form: long rows (>= 32 entries on average) go through the
// coalesced warp-tile kernel, short rows through thread-per-row; both give the same bits
void launch_spmv32(int64_t nrows, const int64_t* ro, const int32_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st, int64_t nnz = -1);
void launch_spmv64(int64_t nrows, const int64_t* ro, const int64_t* ci, const double* v, const double* x, double* y,
                   cudaStream_t st, int64_t nnz = -1);


// ---- algebraic batch path (kern_alg.cu): general ReductionInputs
enum { ALG_HYB = 0, ALG_REC = 1, ALG_COND = 2, ALG_RECC = 3 };
struct AlgArgs {
  int64_t ne;                  // elements (blocks)
  const int64_t* boff;         // ne + 1 broken offsets
  const int64_t* aoff;         // ne block offsets into blocks (sum of n_e^2)
  const double* blocks;        // row-major element blocks
  const int* idx;              // per element: its n local dofs ordered [i | b] (at boff[e])
  const int* ni;               // interior (unconstrained / marker) dof count per element
  const double* f;             // f_hat (broken)
  int* status;                 // bit 1: singular block
  unsigned long long* bad_elem;  // smallest singular element id
  // hybrid modes
  int64_t m;                   // multiplier count
  const int64_t* goff;         // ne + 1 offsets of each element's multiplier rows
  const int64_t* mrows;        // sorted global multiplier rows per element
  const int64_t* hoff;         // ne offsets of H_e (nr x nr) in hbuf
  const int64_t* cptr;         // sum(nr) + 1: entry range of each (element, local row)
  const int* cent_r;           // entry local row
  const int* cent_a;           // entry local dof position in the [i | b] order
  const double* cent_v;        // entry value (C)
  double* hbuf;                // H_e blocks
  double* gbuf;                // g_e blocks
  const double* lambda;        // recover: multipliers
  double* x_hat;               // recover: broken solution
  // condense modes
  int64_t n_master;
  const int64_t* bdof_off;     // ne + 1 offsets of each element's b dofs (sum nb)
  const int64_t* bm_ptr;       // sum(nb) + 1: P-row entries of each b dof
  const int64_t* bm_ord;       // entry master ordinal
  const double* bm_w;          // entry weight (P value)
  const int* bm_loc;           // entry's local b dof j
  const int64_t* soff;         // ne offsets of S_hat (nb x nb) in sbuf
  double* sbuf;                // S_hat blocks
  double* fsbuf;               // f_S blocks (sum nb)
  const int64_t* ibase;        // ne offsets of the element's i dofs (sum ni)
  const int64_t* i_global;     // global dof of each i dof
  const double* i_sign;        // its P value
  const double* xb;            // recover_condensed: master values
  double* x;                   // recover_condensed: global solution
};
// launch plan for elements of order <= dmax with <= ncmax right-hand sides
struct AlgPlan {
  int64_t fast = 0, slow = 0;  // doubles per CTA: LU + column-chunk buffers (+piv), and B0h/B0l/X/Xl
  int ncc = 1;                 // right-hand-side columns per chunk
  bool smem = false;           // fast region in shared memory
  int grid = 1;
};
AlgPlan alg_plan(int64_t ne, int dmax, int ncmax);
int64_t alg_gws_doubles(const AlgPlan& p);  // global scratch the plan needs
void launch_alg(const AlgArgs& a, int mode, const AlgPlan& p, double* gws, cudaStream_t st);
// SPD element blocks (kern_spd.cu): LDL^T + exact-residual refinement, hybridize mode
bool spd_supported(int nmax, int ncmax);
int64_t spd_gws_doubles(int64_t ne, int nmax, int ncmax, int* grid);
void launch_spd_hyb(const AlgArgs& a, int nmax, int ncmax, double* gws, cudaStream_t st);
void launch_alg_hkeys(const AlgArgs& a, uint64_t* hkeys, int64_t* hsrc, uint64_t* gkeys, int64_t* gsrc, cudaStream_t st);
void launch_alg_skeys(const AlgArgs& a, const int64_t* trip_off, const int64_t* ftrip_off, uint64_t* skeys,
                      int64_t* ssrc, double* sw, uint64_t* fkeys, int64_t* fsrc, double* fw, cudaStream_t st);
void launch_run_heads(int64_t n, const uint64_t* keys, int* head, cudaStream_t st);
void launch_run_csr(int64_t n, const uint64_t* keys, const int* head, const int* pos, int64_t ncols, int64_t* run_start,
                    int64_t* cols, int64_t* row_cnt, cudaStream_t st);
void launch_run_sum(int64_t nruns, const int64_t* run_start, const int64_t* src, const double* w, const double* buf,
                    double* out, const int64_t* out_index, int from_zero, cudaStream_t st);
void launch_row_sumsq(int64_t nrows, const int64_t* ro, const double* v, double* out, cudaStream_t st);
// op 0: out = x * y; 1: out += a x; 2: out = x + a out; 3: out = 1 / x (0 stays 0)
void launch_vec_op(int64_t n, int op, double a, const double* x, const double* y, double* out, cudaStream_t st);
// deterministic dot product (part: 1024 doubles of scratch), result on the device
void launch_gather_i64(int64_t n, const int64_t* pos, const int64_t* in, int64_t* out, cudaStream_t st);
void launch_gather_f64(int64_t n, const int64_t* pos, const double* in, double* out, cudaStream_t st);
void launch_scatter(int64_t n, const int64_t* index, const double* v, double* out, cudaStream_t st);
void launch_iota(int64_t n, int64_t* out, cudaStream_t st);
void launch_csr_symmetrize64(int64_t nrows, const int64_t* ro, const int64_t* ci, double* v, cudaStream_t st);
void launch_csr_symmetrize32(int64_t nrows, const int64_t* ro, const int32_t* ci, double* v, cudaStream_t st);
// ---- config 4: Piola element matrices of trilinear cells (kern_piola.cu)
struct PiolaArgs {
  int n, nq;
  int64_t ncells;
  int64_t N[3];
  const double* verts;   // (N0+1)(N1+1)(N2+1) x 3
  const double* qs;      // nq 1D Gauss points
  const double* bq_val;  // nq^3 x n x 3 reference basis values
  const double* bq_div;  // nq^3 x n
  const double* bq_w;    // nq^3 weights
  double h[3];
  double det0;
  const double *alpha, *beta;
  double* ablk;          // ncells x n x n: A_T
  double* dm;            // optional ncells x 2 x n x n: D_T, M_T
};
size_t piola_smem_bytes(int n);
// affine cells: A_T = fl(fl(alpha D) + fl(beta M)) for every cell (dm = [D | M], n x n each)
void launch_affine_assemble(int64_t ncells, int n, const double* dm, const double* alpha, const double* beta,
                            double* out, cudaStream_t st);
void launch_piola_assemble(const PiolaArgs& a, int grid, cudaStream_t st);
// GEMM form for component-separable bases (tphi / tdiv: np x n tables in the
// component-sorted dof order perm; n % 12 == 0)
bool piola_gemm_supported(int n, int np);
void launch_piola_gemm(const PiolaArgs& a, const double* tphi, const double* tdiv, const int* perm, int grid,
                       cudaStream_t st);
// device pcg (kern_pcg.cu) on a CSR matrix with int32 (ci32) or int64 (ci64) columns
hdr_status pcg_device(int64_t n, const int64_t* ro, const int32_t* ci32, const int64_t* ci64, const double* vals,
                      const double* b, double* x, double rtol, int64_t maxit, int precond, double* hist,
                      hdr_pcg_report* rep, cudaStream_t st);
void launch_dot(int64_t n, const double* x, const double* y, double* part, double* out, cudaStream_t st);

// ---- near_nullspace_check (kern_nullspace.cu)
struct RefElement;
hdr_status near_nullspace_device(const DevMesh& dm, const RefElement& re, int weighted, const int* mbase, int64_t m,
                                 const double* beta_dev, double* out, cudaStream_t st);

}  // namespace hdr
