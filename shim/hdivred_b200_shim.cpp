// See hdivred_b200_shim.hpp.  Maps hdr_status to the reference's exceptions.
#include "hdivred_b200_shim.hpp"

#include <array>
#include <memory>
#include <stdexcept>
#include <string>

#include "hdivred/errors.hpp"
#include "hdivred_b200.h"

namespace hdivred_b200 {
namespace {

void check(hdr_status s) {
  if (s == HDR_OK) return;
  const std::string msg = hdr_last_error();
  switch (s) {
    case HDR_SINGULAR_BLOCK: throw hdivred::SingularBlock(msg);
    case HDR_DIMENSION_MISMATCH: throw hdivred::DimensionMismatch(msg);
    case HDR_VALIDATION: throw hdivred::ValidationError(msg);
    case HDR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case HDR_CAP_EXCEEDED: throw hdivred::CapExceeded(msg);
    case HDR_SETUP_FAILED: throw hdivred::SetupFailed(msg);
    case HDR_FORMAT_ERROR: throw hdivred::FormatError(msg, 0);
    default: throw std::runtime_error("hdivred_b200: " + msg);
  }
}

struct SpaceDeleter {
  void operator()(hdr_space_s* s) const { hdr_space_destroy(s); }
};
using SpacePtr = std::unique_ptr<hdr_space_s, SpaceDeleter>;

SpacePtr make_space(const hdivred::RtSpace& sp) {
  const int64_t cells[3] = {sp.mesh.ncells_per_axis[0], sp.mesh.ncells_per_axis[1], sp.mesh.ncells_per_axis[2]};
  const double h[3] = {sp.mesh.cell_sizes[0], sp.mesh.cell_sizes[1], sp.mesh.cell_sizes[2]};
  hdr_space_t s = nullptr;
  // bind the caller's reference element matrices (their exact bits)
  check(hdr_space_create(sp.mesh.dim, cells, h, sp.order, sp.ref_divdiv.entries.data(), sp.ref_mass.entries.data(), 0,
                         nullptr, &s));
  return SpacePtr(s);
}

std::array<int64_t, HDR_INFO_COUNT> info(hdr_space_t s) {
  std::array<int64_t, HDR_INFO_COUNT> o{};
  check(hdr_space_info(s, o.data()));
  return o;
}

std::vector<hdivred::index_t> block_offsets(const hdivred::RtSpace& sp) {
  std::vector<hdivred::index_t> off(static_cast<size_t>(sp.mesh.ncells()) + 1, 0);
  for (size_t c = 0; c + 1 < off.size(); ++c) off[c + 1] = off[c] + sp.element_ndofs;
  return off;
}

void check_fe_sizes(const hdivred::RtSpace& space, const hdivred::CellCoefficients& coeffs,
                    const std::vector<double>& f_hat, const char* who) {
  if (static_cast<hdivred::index_t>(f_hat.size()) != space.broken_ndofs ||
      static_cast<hdivred::index_t>(coeffs.alpha.size()) != space.mesh.ncells() ||
      static_cast<hdivred::index_t>(coeffs.beta.size()) != space.mesh.ncells())
    throw hdivred::DimensionMismatch(std::string(who) + ": inconsistent input dimensions");
}

std::shared_ptr<void> own_space(SpacePtr s) {
  return std::shared_ptr<void>(s.release(), [](void* p) { hdr_space_destroy(static_cast<hdr_space_t>(p)); });
}

// the FE P (build_P, src/reduction.cpp:136-150): one signed entry per broken dof
hdivred::CsrMatrix fe_p_mat(hdr_space_t s, const hdivred::RtSpace& space, std::vector<int64_t>& gl,
                            std::vector<double>& sg) {
  gl.resize(static_cast<size_t>(space.broken_ndofs));
  sg.resize(static_cast<size_t>(space.broken_ndofs));
  check(hdr_space_dof_map(s, gl.data(), sg.data()));
  hdivred::CsrMatrix p(space.broken_ndofs, space.ndofs);
  p.col_indices.assign(gl.begin(), gl.end());
  p.values.assign(sg.begin(), sg.end());
  for (hdivred::index_t r = 0; r <= space.broken_ndofs; ++r) p.row_offsets[static_cast<size_t>(r)] = r;
  return p;
}

}  // namespace

std::pair<FeHybridized, std::vector<double>> hybridize(const hdivred::RtSpace& space,
                                                       const hdivred::CellCoefficients& coeffs,
                                                       const std::vector<double>& f_hat, bool symmetric) {
  check_fe_sizes(space, coeffs, f_hat, "hybridize");
  SpacePtr s = make_space(space);
  const auto in = info(s.get());
  hdr_hybrid_t op = nullptr;
  check(hdr_hybridize_fe(s.get(), coeffs.alpha.data(), coeffs.beta.data(), f_hat.data(), 0, &op));
  FeHybridized out;
  out.device = std::shared_ptr<void>(op, [](void* p) { hdr_hybrid_destroy(static_cast<hdr_hybrid_t>(p)); });
  if (symmetric) check(hdr_hybrid_symmetrize(op));
  const int64_t m = in[HDR_INFO_M], nnz = in[HDR_INFO_NNZ_H];
  out.h_mat = hdivred::CsrMatrix(m, m);
  out.h_mat.col_indices.resize(static_cast<size_t>(nnz));
  out.h_mat.values.resize(static_cast<size_t>(nnz));
  std::vector<double> g(static_cast<size_t>(m));
  check(hdr_space_pattern(s.get(), 0, out.h_mat.row_offsets.data(), out.h_mat.col_indices.data()));
  check(hdr_hybrid_values(op, out.h_mat.values.data(), g.data(), 0));
  out.block_offsets = block_offsets(space);
  // p_mat and recovery_scale = 1 / diag(P^T P) (reduction.cpp:339-352): 1 for
  // bubbles and boundary faces, 1/2 for interior faces
  std::vector<int64_t> gl;
  std::vector<double> sg;
  out.p_mat = fe_p_mat(s.get(), space, gl, sg);
  const int64_t nd = space.ndofs;
  std::vector<double> cnt(static_cast<size_t>(nd), 0.0);
  for (size_t r = 0; r < gl.size(); ++r) cnt[static_cast<size_t>(gl[r])] += sg[r] * sg[r];
  out.recovery_scale.resize(static_cast<size_t>(nd));
  for (int64_t i = 0; i < nd; ++i) out.recovery_scale[static_cast<size_t>(i)] = 1.0 / cnt[static_cast<size_t>(i)];
  out.diagonal_gram = true;
  out.space = own_space(std::move(s));  // released last: the operator borrows the space
  return {std::move(out), std::move(g)};
}

std::pair<std::vector<double>, std::vector<double>> recover_hybrid(const FeHybridized& op,
                                                                   const std::vector<double>& lambda,
                                                                   const std::vector<double>& f_hat) {
  if (!op.device) throw std::invalid_argument("recover_hybrid: operator without device state");
  if (static_cast<hdivred::index_t>(lambda.size()) != op.h_mat.nrows)
    throw hdivred::DimensionMismatch("recover_hybrid: lambda length != multiplier count");
  if (static_cast<hdivred::index_t>(f_hat.size()) != op.p_mat.nrows)
    throw hdivred::DimensionMismatch("recover_hybrid: f_hat length != broken dofs");
  std::vector<double> x_hat(static_cast<size_t>(op.p_mat.nrows)), x(static_cast<size_t>(op.p_mat.ncols));
  check(hdr_recover_hybrid(static_cast<hdr_hybrid_t>(op.device.get()), lambda.data(), f_hat.data(), 0, x_hat.data(),
                           x.data()));
  return {std::move(x_hat), std::move(x)};
}

std::pair<FeCondensed, std::vector<double>> static_condense(const hdivred::RtSpace& space,
                                                            const hdivred::CellCoefficients& coeffs,
                                                            const std::vector<double>& f_hat) {
  check_fe_sizes(space, coeffs, f_hat, "static_condense");
  SpacePtr s = make_space(space);
  const auto in = info(s.get());
  hdr_condensed_t op = nullptr;
  check(hdr_static_condense_fe(s.get(), coeffs.alpha.data(), coeffs.beta.data(), f_hat.data(), 0, &op));
  FeCondensed out;
  out.device = std::shared_ptr<void>(op, [](void* p) { hdr_condensed_destroy(static_cast<hdr_condensed_t>(p)); });
  const int64_t ns = in[HDR_INFO_NS], nnz = in[HDR_INFO_NNZ_S];
  out.s_mat = hdivred::CsrMatrix(ns, ns);
  out.s_mat.col_indices.resize(static_cast<size_t>(nnz));
  out.s_mat.values.resize(static_cast<size_t>(nnz));
  std::vector<double> f_s(static_cast<size_t>(ns));
  check(hdr_space_pattern(s.get(), 1, out.s_mat.row_offsets.data(), out.s_mat.col_indices.data()));
  check(hdr_condensed_values(op, out.s_mat.values.data(), f_s.data(), 0));
  out.master_globals.resize(static_cast<size_t>(ns));
  check(hdr_space_master_globals(s.get(), out.master_globals.data()));
  out.block_offsets = block_offsets(space);
  out.n_global = space.ndofs;
  out.space = own_space(std::move(s));
  return {std::move(out), std::move(f_s)};
}

std::vector<double> recover_condensed(const FeCondensed& op, const std::vector<double>& x_b,
                                      const std::vector<double>& f_hat) {
  if (!op.device) throw std::invalid_argument("recover_condensed: operator without device state");
  if (static_cast<hdivred::index_t>(x_b.size()) != op.s_mat.nrows)
    throw hdivred::DimensionMismatch("recover_condensed: x_b length != master count");
  if (static_cast<hdivred::index_t>(f_hat.size()) != op.block_offsets.back())
    throw hdivred::DimensionMismatch("recover_condensed: f_hat length != broken dofs");
  std::vector<double> x(static_cast<size_t>(op.n_global));
  check(hdr_recover_condensed(static_cast<hdr_condensed_t>(op.device.get()), x_b.data(), f_hat.data(), 0, x.data()));
  return x;
}

namespace {

// ReductionInputs -> hdr_alg_inputs (views into the caller's structure plus
// the concatenated blocks / dof globals kept alive in `keep`)
struct AlgView {
  std::vector<int64_t> sizes, dof_global;
  std::vector<double> blocks;
  hdr_alg_inputs in{};
};

void view_inputs(const hdivred::ReductionInputs& r, AlgView& v) {
  const auto& bl = r.a_hat.blocks;
  v.sizes.resize(bl.size());
  size_t total = 0;
  for (size_t e = 0; e < bl.size(); ++e) {
    v.sizes[e] = static_cast<int64_t>(bl[e].dof_map.size());
    total += bl[e].matrix.entries.size();
  }
  v.blocks.reserve(total);
  for (const auto& b : bl) {
    if (b.matrix.nrows != static_cast<hdivred::index_t>(b.dof_map.size()) || b.matrix.ncols != b.matrix.nrows)
      throw hdivred::DimensionMismatch("ElementBlockOperator: block matrix size != dof_map size");
    v.blocks.insert(v.blocks.end(), b.matrix.entries.begin(), b.matrix.entries.end());
    for (const auto& d : b.dof_map) v.dof_global.push_back(d.global);
  }
  hdr_alg_inputs& in = v.in;
  in.nblocks = static_cast<int64_t>(bl.size());
  in.block_sizes = v.sizes.data();
  in.blocks = v.blocks.data();
  in.dof_global = v.dof_global.data();
  in.p_nrows = r.p_mat.nrows;
  in.p_ncols = r.p_mat.ncols;
  in.p_row_offsets = r.p_mat.row_offsets.data();
  in.p_col_indices = r.p_mat.col_indices.data();
  in.p_values = r.p_mat.values.data();
  in.c_nrows = r.c_mat.nrows;
  in.c_ncols = r.c_mat.ncols;
  in.c_row_offsets = r.c_mat.row_offsets.data();
  in.c_col_indices = r.c_mat.col_indices.data();
  in.c_values = r.c_mat.values.data();
  in.f_len = static_cast<int64_t>(r.f_hat.size());
  in.f_hat = r.f_hat.data();
  in.interior_global_begin = r.interior_global_begin;
}

std::shared_ptr<void> own(hdr_alg_t h) {
  return std::shared_ptr<void>(h, [](void* p) { hdr_alg_destroy(static_cast<hdr_alg_t>(p)); });
}

std::array<int64_t, HDR_ALG_INFO_COUNT> alg_info(hdr_alg_t h) {
  std::array<int64_t, HDR_ALG_INFO_COUNT> o{};
  check(hdr_alg_info(h, o.data()));
  return o;
}

hdivred::CsrMatrix alg_matrix(hdr_alg_t h, std::vector<double>& rhs) {
  const auto o = alg_info(h);
  hdivred::CsrMatrix a(o[HDR_ALG_NROWS], o[HDR_ALG_NROWS]);
  a.col_indices.resize(static_cast<size_t>(o[HDR_ALG_NNZ]));
  a.values.resize(static_cast<size_t>(o[HDR_ALG_NNZ]));
  rhs.resize(static_cast<size_t>(o[HDR_ALG_NROWS]));
  check(hdr_alg_matrix(h, a.row_offsets.data(), a.col_indices.data(), a.values.data(), rhs.data()));
  return a;
}

std::vector<hdivred::index_t> offsets_of(const hdivred::ReductionInputs& r) {
  std::vector<hdivred::index_t> off(r.a_hat.blocks.size() + 1, 0);
  for (size_t e = 0; e < r.a_hat.blocks.size(); ++e)
    off[e + 1] = off[e] + static_cast<hdivred::index_t>(r.a_hat.blocks[e].dof_map.size());
  return off;
}

}  // namespace

std::pair<AlgHybridized, std::vector<double>> hybridize(const hdivred::ReductionInputs& inputs, bool symmetric) {
  AlgView v;
  view_inputs(inputs, v);
  hdr_alg_t h = nullptr;
  check(hdr_alg_hybridize(&v.in, &h));
  AlgHybridized out;
  out.device = own(h);
  if (symmetric) check(hdr_alg_symmetrize(h));
  std::vector<double> g;
  out.h_mat = alg_matrix(h, g);
  out.p_mat = inputs.p_mat;
  out.block_offsets = offsets_of(inputs);
  const auto o = alg_info(h);
  out.diagonal_gram = o[HDR_ALG_DIAGONAL_GRAM] != 0;
  out.recovery_scale.resize(static_cast<size_t>(o[HDR_ALG_N_GLOBAL]));
  check(hdr_alg_recovery_scale(h, out.recovery_scale.data()));
  return {std::move(out), std::move(g)};
}

std::pair<std::vector<double>, std::vector<double>> recover_hybrid(const AlgHybridized& op,
                                                                   const std::vector<double>& lambda,
                                                                   const std::vector<double>& f_hat) {
  hdr_alg_t h = static_cast<hdr_alg_t>(op.device.get());
  const auto o = alg_info(h);
  std::vector<double> x_hat(static_cast<size_t>(o[HDR_ALG_N_HAT])), x(static_cast<size_t>(o[HDR_ALG_N_GLOBAL]));
  check(hdr_alg_recover_hybrid(h, lambda.data(), static_cast<int64_t>(lambda.size()), f_hat.data(),
                               static_cast<int64_t>(f_hat.size()), x_hat.data(), x.data()));
  return {std::move(x_hat), std::move(x)};
}

std::pair<AlgCondensed, std::vector<double>> static_condense(const hdivred::ReductionInputs& inputs, bool symmetric) {
  AlgView v;
  view_inputs(inputs, v);
  hdr_alg_t h = nullptr;
  check(hdr_alg_static_condense(&v.in, &h));
  AlgCondensed out;
  out.device = own(h);
  if (symmetric) check(hdr_alg_symmetrize(h));
  std::vector<double> f_s;
  out.s_mat = alg_matrix(h, f_s);
  out.master_globals.resize(static_cast<size_t>(out.s_mat.nrows));
  check(hdr_alg_master_globals(h, out.master_globals.data()));
  out.block_offsets = offsets_of(inputs);
  out.n_global = inputs.p_mat.ncols;
  return {std::move(out), std::move(f_s)};
}

std::vector<double> recover_condensed(const AlgCondensed& op, const std::vector<double>& x_b,
                                      const std::vector<double>& f_hat) {
  hdr_alg_t h = static_cast<hdr_alg_t>(op.device.get());
  std::vector<double> x(static_cast<size_t>(op.n_global));
  check(hdr_alg_recover_condensed(h, x_b.data(), static_cast<int64_t>(x_b.size()), f_hat.data(),
                                  static_cast<int64_t>(f_hat.size()), x.data()));
  return x;
}

std::vector<double> spmv(const hdivred::CsrMatrix& a, const std::vector<double>& x) {
  if (static_cast<hdivred::index_t>(x.size()) != a.ncols) throw hdivred::DimensionMismatch("spmv: vector length != ncols");
  std::vector<double> y(static_cast<size_t>(a.nrows));
  check(hdr_csr_spmv_host(a.nrows, a.ncols, a.row_offsets.data(), a.col_indices.data(), a.values.data(), x.data(),
                          y.data()));
  return y;
}

namespace {
int precond_code(hdivred::PrecondKind p) {
  switch (p) {
    case hdivred::PrecondKind::none: return 0;
    case hdivred::PrecondKind::jacobi: return 1;
    case hdivred::PrecondKind::sgs: return 2;
    case hdivred::PrecondKind::amg: return 3;
  }
  return 0;
}

hdivred::PcgReport to_report(const hdr_pcg_report& r, const std::vector<double>& hist) {
  hdivred::PcgReport out;
  out.iterations = r.iterations;
  out.converged = r.converged != 0;
  out.relative_residuals.assign(hist.begin(), hist.begin() + static_cast<std::ptrdiff_t>(r.iterations) + 1);
  out.wall_time = r.wall_ms * 1e-3;
  return out;
}
}  // namespace

std::pair<std::vector<double>, hdivred::PcgReport> pcg(const hdivred::CsrMatrix& a, hdivred::PrecondKind precond,
                                                       const std::vector<double>& b, double rtol,
                                                       hdivred::index_t maxit) {
  if (a.nrows != a.ncols) throw std::invalid_argument("pcg: matrix not square");
  if (static_cast<hdivred::index_t>(b.size()) != a.nrows) throw hdivred::DimensionMismatch("pcg: rhs length");
  std::vector<double> x(b.size()), hist(static_cast<size_t>(maxit) + 1, 0.0);
  hdr_pcg_report rep{};
  check(hdr_csr_pcg_host(a.nrows, a.row_offsets.data(), a.col_indices.data(), a.values.data(), b.data(), x.data(),
                         rtol, maxit, precond_code(precond), hist.data(), &rep));
  return {std::move(x), to_report(rep, hist)};
}

std::pair<std::vector<double>, hdivred::PcgReport> pcg(const FeHybridized& op, hdivred::PrecondKind precond,
                                                       const std::vector<double>& b, double rtol,
                                                       hdivred::index_t maxit) {
  if (!op.device) throw std::invalid_argument("pcg: operator without device state");
  if (static_cast<hdivred::index_t>(b.size()) != op.h_mat.nrows) throw hdivred::DimensionMismatch("pcg: rhs length");
  std::vector<double> x(b.size()), hist(static_cast<size_t>(maxit) + 1, 0.0);
  hdr_pcg_report rep{};
  check(hdr_hybrid_pcg(static_cast<hdr_hybrid_t>(op.device.get()), b.data(), x.data(), 0, rtol, maxit,
                       precond_code(precond), hist.data(), &rep));
  return {std::move(x), to_report(rep, hist)};
}

std::vector<double> near_nullspace_check(const hdivred::RtSpace& space, const hdivred::CellCoefficients& coeffs,
                                         bool weighted, hdivred::index_t dense_cap) {
  if (static_cast<hdivred::index_t>(coeffs.alpha.size()) != space.mesh.ncells() ||
      static_cast<hdivred::index_t>(coeffs.beta.size()) != space.mesh.ncells())
    throw hdivred::DimensionMismatch("near_nullspace_check: coefficient count");
  SpacePtr s = make_space(space);
  const auto in = info(s.get());
  std::vector<double> ev(static_cast<size_t>(in[HDR_INFO_M]));
  check(hdr_near_nullspace_check(s.get(), coeffs.alpha.data(), coeffs.beta.data(), 0, weighted ? 1 : 0, dense_cap,
                                 ev.empty() ? nullptr : ev.data()));
  return ev;
}

}  // namespace hdivred_b200
