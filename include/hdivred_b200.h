/* hdivred_b200.h — C ABI of the B200-native element-local hybridization /
 * static-condensation hot path (arXiv 1801.08914, reference: hdivred).
 *
 * Plain C: pointers, sizes, status codes.  No torch or CUDA types.  Every entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/proj).  A C++ drop-in for the reference signatures is in
 * shim/hdivred_b200_shim.cpp; ctypes/pybind bindings are shown in
 * INTEGRATION.md.
 *
 * Conventions
 *  - index width on the boundary is int64 (include/hdivred/dense.hpp:9,
 *    index_t); CSR arrays follow CsrMatrix (include/hdivred/csr.hpp:13-42):
 *    row_offsets[nrows+1], col_indices[nnz] strictly increasing per row,
 *    values[nnz]; explicit zeros kept.
 *  - dense blocks are row-major fp64 (include/hdivred/dense.hpp:12-25).
 *  - "on_device" flags: 0 = host pointers (copied through the library's
 *    stream), 1 = device pointers already resident in HBM.
 *  - every call is synchronous with respect to the host unless it says
 *    otherwise; results are bit-identical for identical inputs (the
 *    deterministic scatter has no float atomics).
 *  - errors: a non-zero hdr_status; hdr_last_error() returns a thread-local
 *    message.  The C++ shim maps HDR_SINGULAR_BLOCK → hdivred::SingularBlock,
 *    HDR_DIMENSION_MISMATCH → DimensionMismatch, HDR_VALIDATION →
 *    ValidationError (include/hdivred/errors.hpp:9-47).
 */
#ifndef HDIVRED_B200_H
#define HDIVRED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HDR_OK = 0,
  HDR_SINGULAR_BLOCK = 1,     /* hdivred::SingularBlock (errors.hpp:15) */
  HDR_DIMENSION_MISMATCH = 2, /* hdivred::DimensionMismatch (errors.hpp:9) */
  HDR_VALIDATION = 3,         /* hdivred::ValidationError (errors.hpp:44) */
  HDR_UNSUPPORTED = 4,        /* input outside what the device path implements (typed, never silent) */
  HDR_CUDA_ERROR = 5,         /* CUDA runtime failure, or no device */
  HDR_INVALID_ARGUMENT = 6,   /* std::invalid_argument in the reference */
  HDR_FORMAT_ERROR = 7,       /* hdivred::FormatError (errors.hpp:25): malformed instance file */
  HDR_CAP_EXCEEDED = 8,       /* hdivred::CapExceeded (errors.hpp:20): dense size cap */
  HDR_SETUP_FAILED = 9        /* hdivred::SetupFailed (errors.hpp:39): AMG setup */
} hdr_status;

typedef struct hdr_space_s* hdr_space_t;         /* mesh + RT_k space + device pattern + fixed factors */
typedef struct hdr_hybrid_s* hdr_hybrid_t;       /* HybridizedOperator (reduction.hpp:49-68) on the device */
typedef struct hdr_condensed_s* hdr_condensed_t; /* CondensedOperator (reduction.hpp:78-95) on the device */

/* Space information indices for hdr_space_info(). */
enum {
  HDR_INFO_DIM = 0,
  HDR_INFO_ORDER,
  HDR_INFO_NCELLS,
  HDR_INFO_NFACES,
  HDR_INFO_NDOFS,          /* RtSpace::ndofs */
  HDR_INFO_BROKEN_NDOFS,   /* RtSpace::broken_ndofs */
  HDR_INFO_ELEMENT_NDOFS,  /* n */
  HDR_INFO_DOFS_PER_FACE,  /* dpf */
  HDR_INFO_INTERIOR_DOFS,  /* per cell */
  HDR_INFO_FACE_DOF_COUNT, /* RtSpace::face_dof_count */
  HDR_INFO_M,              /* multiplier count = rows of H */
  HDR_INFO_NNZ_H,
  HDR_INFO_NS,             /* rows of S = master count */
  HDR_INFO_NNZ_S,
  HDR_INFO_DIV_RANK,       /* rank of the reference divdiv (structured path) */
  HDR_INFO_COUNT
};

/* ------------------------------------------------------------------ space */

/* Config 4: attach vertex coordinates ((N0+1)(N1+1)(N2+1) x 3, lexicographic x
 * fastest, host memory) to a 3D space; the cells become trilinear hexahedra and
 * the element matrices the contravariant Piola map of the reference element
 * (kern_piola.cu; oracle restatement hdo_piola_element — the reference has
 * affine boxes only).  Hybridize / condense / recoveries then
 * run the per-cell elimination of the algebraic path.  NULL detaches. */
hdr_status hdr_space_set_vertices(hdr_space_t space, const double* vertices);
/* The A_T blocks (ncells x n x n) of the last mapped-geometry call (host copy). */
hdr_status hdr_space_element_matrices(hdr_space_t space, double* out);

/* Builds the FE space on the device.  Replaces build_mesh (src/mesh.cpp:137)
 * + build_space (src/rt_space.cpp:318) as far as the hot path needs them.
 *  dim 2|3; cells[3]; cell sizes h[3] (cells congruent, axis aligned); order k
 *  in 0..3 (the reference allows 0..1, src/rt_space.cpp:319; 2..3 follow the
 *  guard-lifted reference).
 *  ref_divdiv / ref_mass: the reference element matrices (RtSpace::ref_divdiv /
 *  ref_mass, n*n row-major).  Pass NULL to have the library build them with
 *  its bit-exact restatement of build_reference (src/rt_space.cpp:180-314).
 *  weighted: 1 = mass-weighted constraint rows (build_C weighted=true,
 *  src/reduction.cpp:182-195); ref_face_moments (2*dim*dpf*n) is then used
 *  (NULL → built internally).
 * Builds the H and S CSR patterns (bit-exact with hybridize/static_condense's
 * from_triplets output) once, on the device. */
hdr_status hdr_space_create(int dim, const int64_t cells[3], const double h[3], int order, const double* ref_divdiv,
                            const double* ref_mass, int weighted, const double* ref_face_moments, hdr_space_t* out);
void hdr_space_destroy(hdr_space_t space);
/* out[HDR_INFO_COUNT] */
hdr_status hdr_space_info(hdr_space_t space, int64_t* out);
/* Copies the reference element matrices the space uses (n*n each; NULL skips). */
hdr_status hdr_space_reference(hdr_space_t space, double* ref_divdiv, double* ref_mass);
/* ref_unit_load (RtSpace::ref_unit_load, src/rt_space.cpp:254-255): 3*n, the load
 * of a constant unit field per component; the FE load of build_reduction_inputs
 * is sum_c g[c] * unit_load[c] (src/rt_space.cpp:361-364). */
hdr_status hdr_space_unit_load(hdr_space_t space, double* out);
/* Binds a CUDA stream (cudaStream_t passed as void*) for all later work on
 * this space and its operators; NULL = the library's own stream. */
hdr_status hdr_space_set_stream(hdr_space_t space, void* stream);
/* which = 0: H pattern (m x m); 1: S pattern (nS x nS).  Host copies, int64. */
hdr_status hdr_space_pattern(hdr_space_t space, int which, int64_t* row_offsets, int64_t* col_indices);
/* master_globals of static_condense (src/reduction.cpp:509-521), int64, nS entries. */
hdr_status hdr_space_master_globals(hdr_space_t space, int64_t* out);
/* The element matrices A_T of every cell (element_matrices, src/rt_space.cpp:345-374:
 * fl(fl(alpha D) + fl(beta M)) bit-exact; mapped cells: the Piola assembly),
 * ncells*n*n row-major, to host (on_device = 0) or device memory.  Feeds the
 * algebraic ReductionInputs of the space (build_reduction_inputs,
 * src/reduction.cpp:200-222), e.g. for eliminate_essential. */
hdr_status hdr_space_element_blocks(hdr_space_t space, const double* alpha, const double* beta, int on_device,
                                    double* out);
/* Signed local->global dof map of every cell (local_dof_map,
 * src/rt_space.cpp:383-393): global[ncells*n] int64, sign[ncells*n]. */
hdr_status hdr_space_dof_map(hdr_space_t space, int64_t* global, double* sign);

/* ------------------------------------------------------------- hybridize */

/* FE fast path of hybridize (src/reduction.cpp:262-354) fused with the
 * element assembly it consumes (build_reduction_inputs → element_matrices,
 * src/reduction.cpp:200-222, src/rt_space.cpp:345-374):
 *   A_T = fl(fl(alpha_T * ref_divdiv) + fl(beta_T * ref_mass))   (bit-exact)
 *   H   = sum_T C_T A_T^-1 C_T^T,  g = sum_T C_T A_T^-1 f_T
 * scattered into the space's H pattern without float atomics.
 * alpha, beta: ncells; f_hat: broken_ndofs (cell-major, local dof order).
 * Creates a new operator in *out (device resident; nothing is copied back). */
hdr_status hdr_hybridize_fe(hdr_space_t space, const double* alpha, const double* beta, const double* f_hat,
                            int on_device, hdr_hybrid_t* out);
/* Same, reusing an existing operator's device buffers (steady-state loop).
 * Device-resident alpha/beta are borrowed (recovery re-reads them): keep them
 * alive and unchanged until the next hybridize on this operator. */
hdr_status hdr_hybridize_fe_into(hdr_hybrid_t op, const double* alpha, const double* beta, const double* f_hat,
                                 int on_device);
/* Asynchronous form: enqueues the H2D staging (host inputs; pinned memory
 * copies asynchronously) and the kernels on the space's stream and returns.
 * Errors detected on the device are reported by the next hdr_hybrid_check. */
hdr_status hdr_hybridize_fe_enqueue(hdr_hybrid_t op, const double* alpha, const double* beta, const double* f_hat,
                                    int on_device);
/* Pipelined batch of count independent hybridizations on one space (new
 * coefficients / right-hand sides per item: parameter sweeps, time steps):
 * item i reads alpha[i], beta[i], f_hat[i] (host memory; pinned for overlap)
 * and writes its H values (nnz_H, pattern order) and g (m) to h_values[i] /
 * g[i] (host; NULL skips).  Uploads, kernels and downloads run on three
 * streams with two alternating device operators, so item i's download overlaps
 * item i+1's kernels and item i+2's upload.  Same bits as count separate
 * hdr_hybridize_fe + hdr_hybrid_values calls (reduction.cpp:262-354 each).
 * Returns after the last download; the space's stream is ordered after it. */
hdr_status hdr_hybridize_fe_batch(hdr_space_t space, int count, const double* const* alpha,
                                  const double* const* beta, const double* const* f_hat, double* const* h_values,
                                  double* const* g);
/* Synchronizes the stream and reports device-side status of enqueued work. */
hdr_status hdr_hybrid_check(hdr_hybrid_t op);
/* Fail-safe of the structured element solve: cells whose
 * a-posteriori error estimate exceeds 1e-12 of |H_T| (extreme alpha/beta
 * ratios, e.g. the reference's soft-hard preset p = -8, src/mesh.cpp:168-191)
 * are solved on the exact double-double path instead.  *count = the number of
 * such cells in the operator's last synchronous hybridize / recover call
 * (k = 0: cells since that call, enqueued calls included). */
hdr_status hdr_hybrid_exact_cells(hdr_hybrid_t op, int64_t* count);
/* Testing / tuning: force_exact = 1 sends every cell of later calls to the
 * exact path; eps32 / eps_tc (<= 0: defaults) = relative accuracy assumed for
 * the fp32 / tcgen05 correction arithmetic in the acceptance test; q_log
 * (device float[ncells] or NULL) receives each cell's measured ratio
 * q = |first-order term| / |zero-order term| on later hybridize calls. */
hdr_status hdr_space_set_exact_policy(hdr_space_t space, int force_exact, double eps32, double eps_tc, float* q_log);
/* In-place symmetrization of the operator's H values (see hdr_alg_symmetrize). */
hdr_status hdr_hybrid_symmetrize(hdr_hybrid_t op);
void hdr_hybrid_destroy(hdr_hybrid_t op);
/* Copy H values (nnz_H, in the space's pattern order) and/or g (m); NULL
 * skips.  dst_on_device selects device-to-device copies. */
hdr_status hdr_hybrid_values(hdr_hybrid_t op, double* h_values, double* g, int dst_on_device);
/* Asynchronous copy-out (enqueued on the space's stream). */
hdr_status hdr_hybrid_values_enqueue(hdr_hybrid_t op, double* h_values, double* g, int dst_on_device);
/* Device pointers of H values / g / pattern (borrowed; valid while op lives).
 * row_offsets are int64, col_indices int32 on the device. */
hdr_status hdr_hybrid_device_ptrs(hdr_hybrid_t op, const double** h_values, const double** g,
                                  const int64_t** row_offsets, const int32_t** col_indices);

/* recover_hybrid (src/reduction.cpp:356-446):
 *   x_hat = A_hat^-1 (f_hat - C^T lambda)   (broken_ndofs)
 *   x     = (P^T P)^-1 P^T x_hat            (ndofs)
 * lambda: m; f_hat: broken_ndofs.  Either output may be NULL. */
hdr_status hdr_recover_hybrid(hdr_hybrid_t op, const double* lambda, const double* f_hat, int on_device,
                              double* x_hat, double* x);

/* ---------------------------------------------------- static condensation */

/* static_condense (src/reduction.cpp:448-557) on the FE path, marker
 * partition i = element bubbles: S = sum_T P_b^T (A_bb - A_bi A_ii^-1 A_ib) P_b,
 * f_S likewise. */
hdr_status hdr_static_condense_fe(hdr_space_t space, const double* alpha, const double* beta, const double* f_hat,
                                  int on_device, hdr_condensed_t* out);
hdr_status hdr_static_condense_fe_into(hdr_condensed_t op, const double* alpha, const double* beta,
                                       const double* f_hat, int on_device);
void hdr_condensed_destroy(hdr_condensed_t op);
hdr_status hdr_condensed_values(hdr_condensed_t op, double* s_values, double* f_s, int dst_on_device);
/* recover_condensed (src/reduction.cpp:559-587): x (ndofs) from x_b (nS). */
hdr_status hdr_recover_condensed(hdr_condensed_t op, const double* x_b, const double* f_hat, int on_device,
                                 double* x);

/* ------------------------------------------------------------------ spmv */

/* spmv (src/csr.cpp:77-87) with the operator's reduced matrix: y = H x
 * (hybrid) / y = S x (condensed).  Row sums accumulate in storage order. */
hdr_status hdr_hybrid_spmv(hdr_hybrid_t op, const double* x, double* y, int on_device);
hdr_status hdr_condensed_spmv(hdr_condensed_t op, const double* x, double* y, int on_device);
/* Host-array form of spmv for a caller-owned CsrMatrix (copies in and out). */
hdr_status hdr_csr_spmv_host(int64_t nrows, int64_t ncols, const int64_t* row_offsets, const int64_t* col_indices,
                             const double* values, const double* x, double* y);
/* General CSR SpMV on device arrays (int64 offsets, int64 columns). */
hdr_status hdr_csr_spmv_device(int64_t nrows, const int64_t* row_offsets, const int64_t* col_indices,
                               const double* values, const double* x, double* y, void* stream);

/* ------------------------------------------- algebraic batch (ReductionInputs)
 *
 * Drop-in for the reference's algebraic entry points on a general
 * ReductionInputs (include/hdivred/reduction.hpp:16-33): arbitrary square dense
 * element blocks (ElementBlockOperator, block_operator.hpp:22-38), P (n_hat x n)
 * and C (m x n_hat) as CSR, f_hat, interior_global_begin.  Arrays are host
 * memory, caller-owned, read during the call only.  The handle keeps what the
 * recoveries need on the device.
 *   hdr_alg_hybridize        <- hybridize(const ReductionInputs&)        reduction.hpp:70, reduction.cpp:262-354
 *   hdr_alg_recover_hybrid   <- recover_hybrid(op, lambda, f_hat)        reduction.hpp:73-75, reduction.cpp:356-446
 *   hdr_alg_static_condense  <- static_condense(const ReductionInputs&)  reduction.hpp:97, reduction.cpp:448-557
 *   hdr_alg_recover_condensed<- recover_condensed(op, x_b, f_hat)        reduction.hpp:101-102, reduction.cpp:559-587
 * Errors: HDR_DIMENSION_MISMATCH (inconsistent sizes, as the reference's
 * DimensionMismatch), HDR_VALIDATION (P column empty; interior dof not mapped
 * to a single global), HDR_SINGULAR_BLOCK (A_ii or S_b pivot <= 1e-14 max|block|;
 * hdr_last_error names the element). */
typedef struct hdr_alg_inputs {
  int64_t nblocks;
  const int64_t* block_sizes;   /* n_e of each block (dof_map.size()) */
  const double* blocks;         /* row-major blocks, concatenated in block order */
  const int64_t* dof_global;    /* n_hat: dof_map[l].global, block order; needed when interior_global_begin >= 0 */
  int64_t p_nrows, p_ncols;
  const int64_t* p_row_offsets; /* CsrMatrix p_mat */
  const int64_t* p_col_indices;
  const double* p_values;
  int64_t c_nrows, c_ncols;
  const int64_t* c_row_offsets; /* CsrMatrix c_mat */
  const int64_t* c_col_indices;
  const double* c_values;
  int64_t f_len;
  const double* f_hat;
  int64_t interior_global_begin; /* -1: algebraic partition (zero columns of C) */
} hdr_alg_inputs;

typedef struct hdr_alg_s* hdr_alg_t;

enum {
  HDR_ALG_NROWS = 0,      /* m (hybrid) or n_master (condensed) */
  HDR_ALG_NNZ,            /* nnz of h_mat / s_mat */
  HDR_ALG_N_HAT,
  HDR_ALG_N_GLOBAL,
  HDR_ALG_DIAGONAL_GRAM,  /* HybridizedOperator::diagonal_gram */
  HDR_ALG_KIND,           /* 0 hybrid, 1 condensed */
  HDR_ALG_INFO_COUNT
};

hdr_status hdr_alg_hybridize(const hdr_alg_inputs* inputs, hdr_alg_t* out);
hdr_status hdr_alg_static_condense(const hdr_alg_inputs* inputs, hdr_alg_t* out);
/* out[HDR_ALG_INFO_COUNT] */
hdr_status hdr_alg_info(hdr_alg_t op, int64_t* out);
/* The reduced CSR matrix (h_mat / s_mat: row_offsets nrows+1, col_indices nnz,
 * values nnz) and right-hand side (g / f_s); NULL skips. */
hdr_status hdr_alg_matrix(hdr_alg_t op, int64_t* row_offsets, int64_t* col_indices, double* values, double* rhs);
/* Condensed: CondensedOperator::master_globals (nrows). */
hdr_status hdr_alg_master_globals(hdr_alg_t op, int64_t* out);
/* Hybrid: HybridizedOperator::recovery_scale = 1 / diag(P^T P) (n_global). */
hdr_status hdr_alg_recovery_scale(hdr_alg_t op, double* out);
/* x_hat (n_hat) and x (n_global); either may be NULL. */
hdr_status hdr_alg_recover_hybrid(hdr_alg_t op, const double* lambda, int64_t lambda_len, const double* f_hat,
                                  int64_t f_len, double* x_hat, double* x);
/* x (n_global) */
hdr_status hdr_alg_recover_condensed(hdr_alg_t op, const double* x_b, int64_t xb_len, const double* f_hat,
                                     int64_t f_len, double* x);
void hdr_alg_destroy(hdr_alg_t op);
/* In-place a_ij = a_ji = 0.5 (a_ij + a_ji) of h_mat / s_mat: the reference's
 * symmetrize of H_e / S_hat (reduction.cpp:65-72, 295, 316, 489) applied to the
 * assembled matrix, for consumers that require exact symmetry (its pcg checks
 * |A - A^T| <= 1e-10 max|A|, solvers.cpp:25-30).  The default output is the
 * unsymmetrized element-exact value the parity contract is stated on. */
hdr_status hdr_alg_symmetrize(hdr_alg_t op);

/* ---------------------------------------------------------- reduced solve
 *
 * pcg (src/solvers.cpp:109-163) on the device with the reference's "none"
 * (precond = 0) and Jacobi (precond = 1, positive_inv_diag :32-44) options,
 * x0 = 0, stop at ||r|| / ||b|| <= rtol or maxit iterations.
 * b: the right-hand side (NULL: the operator's own g / f_s), x: the solution,
 * both host (on_device = 0) or device arrays; residual_history: NULL or
 * maxit + 1 host doubles (relative residuals, [0] = 1).  Errors: HDR_VALIDATION
 * for a non-positive diagonal (ZeroDiagonal), <z, r> <= 0
 * (IndefinitePreconditioner) or <p, Ap> <= 0 (matrix not positive definite).
 * The reference also rejects |A - A^T| > 1e-10 max|A| before iterating; call
 * hdr_hybrid_symmetrize / hdr_alg_symmetrize first where that is wanted. */
typedef struct hdr_pcg_report {
  int64_t iterations;
  int32_t converged;
  int32_t reserved;
  double final_relative_residual;
  double wall_ms;
} hdr_pcg_report;

hdr_status hdr_hybrid_pcg(hdr_hybrid_t op, const double* b, double* x, int on_device, double rtol, int64_t maxit,
                          int precond, double* residual_history, hdr_pcg_report* report);
hdr_status hdr_condensed_pcg(hdr_condensed_t op, const double* b, double* x, int on_device, double rtol,
                             int64_t maxit, int precond, double* residual_history, hdr_pcg_report* report);
hdr_status hdr_alg_pcg(hdr_alg_t op, const double* b, double* x, int on_device, double rtol, int64_t maxit,
                       int precond, double* residual_history, hdr_pcg_report* report);
/* precond (all four of the reference's PrecondKind, include/hdivred/driver.hpp:15):
 *   0 none, 1 jacobi (jacobi_setup), 2 sgs (ssgs_setup: one forward + one backward
 *   Gauss-Seidel sweep, solvers.cpp:60-72), 3 amg (amg_setup with default
 *   AmgOptions + one V(1,1) cycle per application, amg.cpp:189-266).
 * The reference's check_symmetric (solvers.cpp:25-30) runs first on the device:
 * |A - A^T| > 1e-10 max|A| or a non-square matrix -> HDR_INVALID_ARGUMENT. */
/* Host-array form for a caller-owned CsrMatrix (copies in and out). */
hdr_status hdr_csr_pcg_host(int64_t n, const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                            const double* b, double* x, double rtol, int64_t maxit, int precond,
                            double* residual_history, hdr_pcg_report* report);

/* ------------------------------------------------------------ AMG / SGS
 *
 * Smoothed-aggregation AMG on the device (kern_amg.cu): amg_setup
 * (src/amg.cpp:189-244) and amg_apply (one V(1,1) cycle, :248-271).  Every step
 * with arithmetic rounds like the reference, so for the same matrix the levels
 * (A, P, R) and every application are bit-identical to it; the greedy
 * aggregate() pass runs on the host over the device-built strength graph. */
typedef struct hdr_amg_s* hdr_amg_t;
typedef struct hdr_amg_options { /* AmgOptions (include/hdivred/amg.hpp:12-19) */
  double strength_threshold;     /* 0.08 */
  double omega_factor;           /* 1.0 */
  int64_t coarse_cap;            /* 64 */
  int32_t max_levels;            /* 25 */
  int32_t power_iterations;      /* 10 */
  double stall_ratio;            /* 0.9 */
} hdr_amg_options;
void hdr_amg_default_options(hdr_amg_options* out);
/* CSR (row_offsets n+1, col_indices, values; int64 indices) host (on_device = 0)
 * or device arrays; options NULL = defaults.  HDR_SETUP_FAILED as SetupFailed,
 * HDR_SINGULAR_BLOCK from the coarsest LU, HDR_CAP_EXCEEDED from its to_dense. */
hdr_status hdr_amg_setup(int64_t n, const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                         int on_device, const hdr_amg_options* options, hdr_amg_t* out);
/* levels (AmgHierarchy::levels.size()); sizes / nnz: levels + 1 entries (the
 * level matrices, then the coarse matrix); NULL skips. */
hdr_status hdr_amg_info(hdr_amg_t amg, int64_t* levels, int64_t* sizes, int64_t* nnz);
/* which: 0 the level's matrix (level == levels: the coarse matrix), 1 its
 * prolongator, 2 its restriction.  dims[3] = {nrows, ncols, nnz}; the arrays
 * (host, NULL skips) must hold nrows + 1 / nnz / nnz entries. */
hdr_status hdr_amg_level_matrix(hdr_amg_t amg, int64_t level, int which, int64_t* dims, int64_t* row_offsets,
                                int64_t* col_indices, double* values);
/* z = V-cycle(r), both n, host or device */
hdr_status hdr_amg_apply(hdr_amg_t amg, const double* r, double* z, int on_device);
void hdr_amg_destroy(hdr_amg_t amg);
/* One application of the jacobi (kind 1) or sgs (kind 2) preconditioner of a
 * host CSR matrix to r (host arrays), as the reference's Preconditioner::apply. */
hdr_status hdr_csr_precond_apply_host(int64_t n, const int64_t* row_offsets, const int64_t* col_indices,
                                      const double* values, int kind, const double* r, double* z);

/* ------------------------------------------------------------ diagnostics
 *
 * near_nullspace_check (src/reduction.cpp:711-742): the ascending eigenvalues of
 * the assembled m x m matrix C Y C^T, Y_T = M^-1 - M^-1 B^T (B M^-1 B^T)^-1 B M^-1
 * (M = beta_T ref_mass, B = ref_div_form), computed on the device in the
 * reference's operation order (kern_nullspace.cu): bit-identical eigenvalues.
 * weighted: the mass-weighted constraint rows (build_C weighted).  alpha, beta:
 * ncells host (on_device = 0) or device arrays, validated > 0 like
 * element_matrices (rt_space.cpp:353-354, HDR_INVALID_ARGUMENT).  eigenvalues:
 * m host doubles (HDR_INFO_M; m = 0 writes nothing).  HDR_CAP_EXCEEDED when
 * m * m > dense_cap (the reference's default is 4,000,000). */
hdr_status hdr_near_nullspace_check(hdr_space_t space, const double* alpha, const double* beta, int on_device,
                                    int weighted, int64_t dense_cap, double* eigenvalues);

/* ------------------------------------------------- host-only introspection */

/* The reference element matrices of RT_k on an h[0] x h[1] (x h[2]) box,
 * bit-identical to build_reference (src/rt_space.cpp:180-314): divdiv, mass
 * (n*n), face_moments (2*dim*dpf*n), unit_load (3*n).  NULL skips.  Host only. */
hdr_status hdr_reference_element(int dim, int order, const double h[3], double* divdiv, double* mass,
                                 double* face_moments, double* unit_load);
/* RtSpace::ref_div_form (rt_space.cpp:197, 256-259): (k+1)^dim x n, bit-identical.  Host only. */
hdr_status hdr_reference_div_form(int dim, int order, const double h[3], double* div_form);
/* Fixed factors of the structured element solve: X (n*r), lambda
 * (r), E, N0, Ma (n*n); diag = {rho, max|E|/max|D|, max|X^T M X - I|, block
 * diagonal M}.  Host only. */
hdr_status hdr_structured_factors(int dim, int order, const double h[3], double* X, double* lambda, double* E,
                                  double* N0, double* Ma, double* diag, int64_t* rank);

/* ------------------------------------------------------------------ misc */

const char* hdr_last_error(void);
/* Build/version string: "hdivred_b200 <ver> sm_100a". */
const char* hdr_version(void);
/* Number of kernels this library launched since load (launch accounting for
 * bench.py's gpu_launches). */
int64_t hdr_launch_count(void);
/* FP64 FMA throughput of device 0 in TFLOP/s (2 flops per DFMA), measured with
 * a register-resident DFMA chain kernel; the fp64 roofline denominator. */
hdr_status hdr_measure_fp64_peak(double* tflops, double* ms);
/* fp64 tensor-core (DMMA m8n8k4) throughput of the device, TFLOP/s (the peak the
 * k >= 2 kernels' DMMA phases run against). */
hdr_status hdr_measure_dmma_peak(double* tflops, double* ms);
/* Self-test of the tcgen05 TF32 tensor-core path (kern_umma.cu): D (128 x n) =
 * A (128 x k, row-major) * B^T (B: n x k, row-major), split = 1: 3xTF32.  Host arrays. */
hdr_status hdr_umma_selftest(int n, int k, const float* a, const float* b, float* d, int split);
/* Synchronize the space's stream. */
hdr_status hdr_space_synchronize(hdr_space_t space);

/* ------------------------------------------------------------- instance I/O (host, all threads)
 * The reference's text formats (src/block_io.cpp:15-94, src/matrix_market.cpp:36-146),
 * parsed in parallel with exact rounding (values bit-identical to the reference's
 * readers) and written with its "%.17g" (byte-identical files).  threads <= 0:
 * all hardware threads.  Read results live in handles until destroyed. */
typedef struct hdr_blocks_s* hdr_blocks_t;     /* ElementBlockOperator (block_operator.hpp:22-38) */
typedef struct hdr_csr_host_s* hdr_csr_host_t; /* CsrMatrix (csr.hpp:13-42) in host memory */
/* read_block_operator (block_io.cpp:41-94) */
hdr_status hdr_io_read_block_operator(const char* path, int threads, hdr_blocks_t* out);
/* info[0..3] = nblocks, broken_dim, global_dim, total matrix entries */
hdr_status hdr_io_blocks_info(hdr_blocks_t blocks, int64_t* info);
/* copies (NULL skips): block sizes (nblocks), dof globals and signs (broken_dim), row-major entries */
hdr_status hdr_io_blocks_get(hdr_blocks_t blocks, int64_t* block_sizes, int64_t* dof_global, double* dof_sign,
                             double* entries);
void hdr_io_blocks_destroy(hdr_blocks_t blocks);
/* write_block_operator (block_io.cpp:15-39) */
hdr_status hdr_io_write_block_operator(const char* path, int64_t nblocks, int64_t broken_dim, int64_t global_dim,
                                       const int64_t* block_sizes, const int64_t* dof_global, const double* dof_sign,
                                       const double* entries, int threads);
/* read_matrix_market (matrix_market.cpp:55-97, triplets summed as from_triplets) */
hdr_status hdr_io_read_matrix_market(const char* path, int threads, hdr_csr_host_t* out);
/* read_vector_lines (matrix_market.cpp:131-146): an n x 1 handle */
hdr_status hdr_io_read_vector_lines(const char* path, int threads, hdr_csr_host_t* out);
/* info[0..2] = nrows, ncols, nnz */
hdr_status hdr_io_csr_info(hdr_csr_host_t a, int64_t* info);
hdr_status hdr_io_csr_get(hdr_csr_host_t a, int64_t* row_offsets, int64_t* col_indices, double* values);
void hdr_io_csr_destroy(hdr_csr_host_t a);
/* write_matrix_market (matrix_market.cpp:36-53) */
hdr_status hdr_io_write_matrix_market(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_offsets,
                                      const int64_t* col_indices, const double* values, int threads);
/* write_vector_lines (matrix_market.cpp:124-129) */
hdr_status hdr_io_write_vector_lines(const char* path, int64_t n, const double* v, int threads);

#ifdef __cplusplus
}
#endif
#endif
