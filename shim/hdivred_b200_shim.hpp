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
std::pair<hdivred::HybridizedOperator, std::vector<double>> hybridize(const hdivred::RtSpace& space,
                                                                      const hdivred::CellCoefficients& coeffs,
                                                                      const std::vector<double>& f_hat);

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

// spmv (src/csr.cpp:77-87) on the device, bit-identical to the reference.
std::vector<double> spmv(const hdivred::CsrMatrix& a, const std::vector<double>& x);

}  // namespace hdivred_b200
