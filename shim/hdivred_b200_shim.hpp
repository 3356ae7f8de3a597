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

namespace hdivred_b200 {

// hybridize (src/reduction.cpp:262-354) of the FE inputs.  Fills h_mat,
// block_offsets and recovery_scale/diagonal_gram like the reference; the
// per-element factorizations stay on the device (HybridizedOperator::elements
// is private to reduction.cpp and left empty).
// symmetric = true (default) applies the reference's symmetrize to H (its
// production output is exactly symmetric and its pcg requires that); false
// returns the element-exact values the parity contract is stated on.
std::pair<hdivred::HybridizedOperator, std::vector<double>> hybridize(const hdivred::RtSpace& space,
                                                                      const hdivred::CellCoefficients& coeffs,
                                                                      const std::vector<double>& f_hat,
                                                                      bool symmetric = true);

// static_condense (src/reduction.cpp:448-557) of the FE inputs: s_mat,
// master_globals, n_global, block_offsets and f_S.
std::pair<hdivred::CondensedOperator, std::vector<double>> static_condense(const hdivred::RtSpace& space,
                                                                          const hdivred::CellCoefficients& coeffs,
                                                                          const std::vector<double>& f_hat);

// recover_hybrid (src/reduction.cpp:356-446): (x_hat, x)
std::pair<std::vector<double>, std::vector<double>> recover_hybrid(const hdivred::RtSpace& space,
                                                                   const hdivred::CellCoefficients& coeffs,
                                                                   const std::vector<double>& lambda,
                                                                   const std::vector<double>& f_hat);

// ---- algebraic drop-ins on the reference's own ReductionInputs (reduction.hpp:16-33)
//
// The operator handles carry the reference's public fields (h_mat, p_mat,
// block_offsets, recovery_scale, diagonal_gram / s_mat, master_globals,
// n_global); the per-element state lives on the device behind `device`.
struct AlgHybridized {
  hdivred::HybridizedOperator op;
  std::shared_ptr<void> device;
};
struct AlgCondensed {
  hdivred::CondensedOperator op;
  std::shared_ptr<void> device;
};

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

// spmv (src/csr.cpp:77-87) on the device, bit-identical to the reference.
std::vector<double> spmv(const hdivred::CsrMatrix& a, const std::vector<double>& x);

}  // namespace hdivred_b200
