// C++ drop-in for the reference's hot path (hdivred, include/hdivred/reduction.hpp)
// over the C ABI of libhdivred_b200.so (include/hdivred_b200.h).
//
// Compiled against the reference's own headers: the results are the reference's
// types (HybridizedOperator::h_mat, CondensedOperator::s_mat / master_globals,
// CsrMatrix), errors are the reference's exceptions (include/hdivred/errors.hpp).
// The FE fast path takes the space + coefficients + broken load that the
// reference's build_reduction_inputs (src/reduction.cpp:200-222) would have
// assembled into blocks; the element matrices are formed on the device,
// bit-identically.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "hdivred/csr.hpp"
#include "hdivred/mesh.hpp"
#include "hdivred/reduction.hpp"
#include "hdivred/rt_space.hpp"
#include "hdivred/driver.hpp"
#include "hdivred/solvers.hpp"

namespace hdivred_b200 {

// ---- operators: the reference's own types plus the device state
//
// Each derives from the reference's operator, so its public fields (h_mat,
// p_mat, block_offsets, recovery_scale, diagonal_gram / s_mat, master_globals,
// n_global) are read exactly as before, and carries a shared_ptr to the device
// handle that holds the per-element state (the reference keeps it in the private
// `elements` vector, reduction.hpp:49-68 / 78-95, which stays empty here).
// recover_hybrid / recover_condensed below take these types; an unqualified call
// `recover_hybrid(op, lambda, f_hat)` inside namespace hdivred (src/driver.cpp:244)
// finds them by argument-dependent lookup and prefers them over the reference's
// overload (exact match of the derived type), so the caller changes only the
// hybridize / static_condense line.
struct FeHybridized : hdivred::HybridizedOperator {
  std::shared_ptr<void> space, device;  // hdr_space_t, hdr_hybrid_t
};
struct FeCondensed : hdivred::CondensedOperator {
  std::shared_ptr<void> space, device;  // hdr_space_t, hdr_condensed_t
};
struct AlgHybridized : hdivred::HybridizedOperator {
  std::shared_ptr<void> device;  // hdr_alg_t
};
struct AlgCondensed : hdivred::CondensedOperator {
  std::shared_ptr<void> device;  // hdr_alg_t
};

// ---- FE fast path (the structured kernels): the space + coefficients + broken
// load that build_reduction_inputs (src/reduction.cpp:200-222) would assemble;
// the element matrices are formed on the device, bit-identically.

// hybridize (src/reduction.cpp:262-354).  symmetric = true (default) applies the
// reference's symmetrize to H (its production output is exactly symmetric and its
// pcg requires that); false returns the element-exact values the parity contract
// is stated on.
std::pair<FeHybridized, std::vector<double>> hybridize(const hdivred::RtSpace& space,
                                                       const hdivred::CellCoefficients& coeffs,
                                                       const std::vector<double>& f_hat, bool symmetric = true);
// recover_hybrid (src/reduction.cpp:356-446) on the retained device operator: (x_hat, x)
std::pair<std::vector<double>, std::vector<double>> recover_hybrid(const FeHybridized& op,
                                                                   const std::vector<double>& lambda,
                                                                   const std::vector<double>& f_hat);
// static_condense (src/reduction.cpp:448-557): s_mat, master_globals, n_global, block_offsets, f_S
std::pair<FeCondensed, std::vector<double>> static_condense(const hdivred::RtSpace& space,
                                                            const hdivred::CellCoefficients& coeffs,
                                                            const std::vector<double>& f_hat);
// recover_condensed (src/reduction.cpp:559-587) on the retained device operator
std::vector<double> recover_condensed(const FeCondensed& op, const std::vector<double>& x_b,
                                      const std::vector<double>& f_hat);

// ---- algebraic drop-ins on the reference's own ReductionInputs (reduction.hpp:16-33).
// General element blocks (any size, any C and P): double-double-refined LU per
// element (kern_alg.cu).  NOTE: FE inputs reaching this entry point do NOT use
// the structured FE kernels (the coefficients and the mesh are not part of a
// ReductionInputs); callers that hold the RtSpace and CellCoefficients should use
// the FE overloads above.

// hybridize(const ReductionInputs&)            reduction.hpp:70, reduction.cpp:262-354
std::pair<AlgHybridized, std::vector<double>> hybridize(const hdivred::ReductionInputs& inputs, bool symmetric = true);
// recover_hybrid(op, lambda, f_hat)            reduction.hpp:73-75, reduction.cpp:356-446
std::pair<std::vector<double>, std::vector<double>> recover_hybrid(const AlgHybridized& op,
                                                                   const std::vector<double>& lambda,
                                                                   const std::vector<double>& f_hat);
// static_condense(const ReductionInputs&)      reduction.hpp:97, reduction.cpp:448-557
std::pair<AlgCondensed, std::vector<double>> static_condense(const hdivred::ReductionInputs& inputs,
                                                             bool symmetric = true);
// recover_condensed(op, x_b, f_hat)            reduction.hpp:101-102, reduction.cpp:559-587
std::vector<double> recover_condensed(const AlgCondensed& op, const std::vector<double>& x_b,
                                      const std::vector<double>& f_hat);

// ---- the reduced solve on the device (run_pcg in src/driver.cpp:220-231:
// make_preconditioner + pcg, src/solvers.cpp:109-163).  All four PrecondKind
// values; amg / sgs apply bit-identically to the reference's on the same matrix
// (kern_amg.cu).  Same checks and exceptions as the reference's pcg.
std::pair<std::vector<double>, hdivred::PcgReport> pcg(const hdivred::CsrMatrix& a, hdivred::PrecondKind precond,
                                                       const std::vector<double>& b, double rtol,
                                                       hdivred::index_t maxit);
// on a device-resident H (no upload of the matrix)
std::pair<std::vector<double>, hdivred::PcgReport> pcg(const FeHybridized& op, hdivred::PrecondKind precond,
                                                       const std::vector<double>& b, double rtol,
                                                       hdivred::index_t maxit);

// near_nullspace_check (src/reduction.cpp:711-742) on the device, bit-identical.
std::vector<double> near_nullspace_check(const hdivred::RtSpace& space, const hdivred::CellCoefficients& coeffs,
                                         bool weighted = false, hdivred::index_t dense_cap = hdivred::kDefaultDenseCap);

// spmv (src/csr.cpp:77-87) on the device, bit-identical to the reference.
std::vector<double> spmv(const hdivred::CsrMatrix& a, const std::vector<double>& x);

}  // namespace hdivred_b200
