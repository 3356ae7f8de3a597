// Drop-in check: runs the REFERENCE (linked from oracle/_ref/libhdivred_ref.a)
// and the B200 path through the shim on the same seeded FE inputs, in one
// process, through the reference's own C++ types.  Prints one JSON line.
// TEST INFRASTRUCTURE (built by shim/Makefile; run by tests/test_dropin_gpu.py).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "hdivred/amg.hpp"
#include "hdivred/reduction.hpp"
#include "hdivred/solvers.hpp"
#include "hdivred_b200_shim.hpp"

// The reference's solve_reduction sequences (src/driver.cpp:241-254), written
// inside namespace hdivred exactly as there: the caller changes only the
// hybridize / static_condense line; the unqualified recover_* calls then reach
// the shim's overloads by argument-dependent lookup.
namespace hdivred {
template <class HybFn>
std::vector<double> solve_hybridization(const ReductionInputs& inputs, HybFn hyb_fn, index_t* its) {
  const auto [hyb, g] = hyb_fn(inputs);
  const std::unique_ptr<Preconditioner> pc = jacobi_setup(hyb.h_mat);
  auto [lambda, rep] = pcg(hyb.h_mat, pc.get(), g, 1e-12, 5000);
  *its = rep.iterations;
  return recover_hybrid(hyb, lambda, inputs.f_hat).second;
}
template <class CondFn>
std::vector<double> solve_condensation(const ReductionInputs& inputs, CondFn cond_fn, index_t* its) {
  const auto [cond, f_s] = cond_fn(inputs);
  const std::unique_ptr<Preconditioner> pc = jacobi_setup(cond.s_mat);
  auto [x_b, rep] = pcg(cond.s_mat, pc.get(), f_s, 1e-12, 5000);
  *its = rep.iterations;
  return recover_condensed(cond, x_b, inputs.f_hat);
}
// the same sequence with run_pcg's make_preconditioner + pcg replaced by the
// device solve on the device-resident H (default preconditioner: amg)
template <class HybFn, class PcgFn>
std::vector<double> solve_hybridization_pc(const ReductionInputs& inputs, HybFn hyb_fn, PcgFn pcg_fn, index_t* its) {
  const auto [hyb, g] = hyb_fn(inputs);
  auto [lambda, rep] = pcg_fn(hyb, g);
  *its = rep.iterations;
  return recover_hybrid(hyb, lambda, inputs.f_hat).second;
}
}  // namespace hdivred

using namespace hdivred;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 4;
  const int k = argc > 2 ? std::atoi(argv[2]) : 1;
  const double h = 1.0 / n;
  const CartesianMesh mesh = build_mesh(3, {n, n, n}, {h, h, h});
  const RtSpace sp = build_space(mesh, k);
  CellCoefficients co = soft_hard_coefficients(mesh, 4);
  ReductionInputs in = build_reduction_inputs(sp, co);
  std::uint64_t s = 12345;
  for (auto& v : in.f_hat) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = -1.0 + 2.0 * (static_cast<double>(s >> 11) * 0x1.0p-53);
  }
  auto [ref, g_ref] = hybridize(in);
  auto [gpu, g_gpu] = hdivred_b200::hybridize(sp, co, in.f_hat);
  const bool pattern = ref.h_mat.row_offsets == gpu.h_mat.row_offsets && ref.h_mat.col_indices == gpu.h_mat.col_indices;
  double dh = 0, mh = 0, dg = 0, mg = 0;
  for (size_t i = 0; i < ref.h_mat.values.size(); ++i) {
    dh = std::max(dh, std::fabs(ref.h_mat.values[i] - gpu.h_mat.values[i]));
    mh = std::max(mh, std::fabs(ref.h_mat.values[i]));
  }
  for (size_t i = 0; i < g_ref.size(); ++i) {
    dg = std::max(dg, std::fabs(g_ref[i] - g_gpu[i]));
    mg = std::max(mg, std::fabs(g_ref[i]));
  }
  auto [cref, fs_ref] = static_condense(in);
  auto [cgpu, fs_gpu] = hdivred_b200::static_condense(sp, co, in.f_hat);
  const bool spat = cref.s_mat.row_offsets == cgpu.s_mat.row_offsets &&
                    cref.s_mat.col_indices == cgpu.s_mat.col_indices && cref.master_globals == cgpu.master_globals;
  double ds = 0, ms = 0;
  for (size_t i = 0; i < cref.s_mat.values.size(); ++i) {
    ds = std::max(ds, std::fabs(cref.s_mat.values[i] - cgpu.s_mat.values[i]));
    ms = std::max(ms, std::fabs(cref.s_mat.values[i]));
  }
  // algebraic drop-ins on the reference's own ReductionInputs
  auto rel = [](const std::vector<double>& a, const std::vector<double>& b) {
    double d = 0, m = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      d = std::max(d, std::fabs(a[i] - b[i]));
      m = std::max(m, std::fabs(a[i]));
    }
    return d / (m > 0 ? m : 1.0);
  };
  auto [ahyb, g_alg] = hdivred_b200::hybridize(in);
  const bool apat = ref.h_mat.row_offsets == ahyb.h_mat.row_offsets &&
                    ref.h_mat.col_indices == ahyb.h_mat.col_indices;
  bool asym = true;
  {
    const CsrMatrix t = transpose(ahyb.h_mat);
    asym = t.values == ahyb.h_mat.values && t.col_indices == ahyb.h_mat.col_indices;
  }
  std::vector<double> lam(g_ref.size());
  for (auto& v : lam) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = -1.0 + 2.0 * (static_cast<double>(s >> 11) * 0x1.0p-53);
  }
  auto [xh_ref, x_ref] = recover_hybrid(ref, lam, in.f_hat);
  auto [xh_alg, x_alg] = hdivred_b200::recover_hybrid(ahyb, lam, in.f_hat);
  auto [acond, fs_alg] = hdivred_b200::static_condense(in);
  const bool acpat = cref.s_mat.row_offsets == acond.s_mat.row_offsets &&
                     cref.s_mat.col_indices == acond.s_mat.col_indices && cref.master_globals == acond.master_globals;
  std::vector<double> xb(fs_ref.size());
  for (auto& v : xb) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = -1.0 + 2.0 * (static_cast<double>(s >> 11) * 0x1.0p-53);
  }
  const std::vector<double> xc_ref = recover_condensed(cref, xb, in.f_hat);
  const std::vector<double> xc_alg = hdivred_b200::recover_condensed(acond, xb, in.f_hat);
  // FE operators: recovery on the retained device state (no re-hybridize)
  auto [xh_fe, x_fe] = hdivred_b200::recover_hybrid(gpu, lam, in.f_hat);
  const std::vector<double> xc_fe = hdivred_b200::recover_condensed(cgpu, xb, in.f_hat);
  // the solve_reduction sequences: reference, shim on ReductionInputs, shim FE path
  index_t it_ref = 0, it_alg = 0, it_fe = 0, itc_ref = 0, itc_alg = 0, itc_fe = 0;
  const std::vector<double> xs_ref = solve_hybridization(in, [](const ReductionInputs& r) { return hybridize(r); }, &it_ref);
  const std::vector<double> xs_alg = solve_hybridization(
      in, [](const ReductionInputs& r) { return hdivred_b200::hybridize(r); }, &it_alg);
  const std::vector<double> xs_fe = solve_hybridization(
      in, [&](const ReductionInputs& r) { return hdivred_b200::hybridize(sp, co, r.f_hat); }, &it_fe);
  const std::vector<double> xsc_ref =
      solve_condensation(in, [](const ReductionInputs& r) { return static_condense(r); }, &itc_ref);
  const std::vector<double> xsc_alg = solve_condensation(
      in, [](const ReductionInputs& r) { return hdivred_b200::static_condense(r); }, &itc_alg);
  const std::vector<double> xsc_fe = solve_condensation(
      in, [&](const ReductionInputs& r) { return hdivred_b200::static_condense(sp, co, r.f_hat); }, &itc_fe);
  // AMG-preconditioned solve: the reference's (host amg_setup + pcg) and the
  // device one on the FE operator's device-resident H
  index_t ita_ref = 0, ita_fe = 0;
  const std::vector<double> xa_ref = solve_hybridization_pc(
      in, [](const ReductionInputs& r) { return hybridize(r); },
      [](const HybridizedOperator& h, const std::vector<double>& g) {
        const std::unique_ptr<Preconditioner> pc = amg_preconditioner(h.h_mat);
        return pcg(h.h_mat, pc.get(), g, 1e-12, 2000);
      },
      &ita_ref);
  const std::vector<double> xa_fe = solve_hybridization_pc(
      in, [&](const ReductionInputs& r) { return hdivred_b200::hybridize(sp, co, r.f_hat); },
      [](const hdivred_b200::FeHybridized& h, const std::vector<double>& g) {
        return hdivred_b200::pcg(h, PrecondKind::amg, g, 1e-12, 2000);
      },
      &ita_fe);
  // the device pcg on the reference's own H (host CsrMatrix in, device solve)
  const std::unique_ptr<Preconditioner> pc_ref = amg_preconditioner(ref.h_mat);
  const auto ref_solve = pcg(ref.h_mat, pc_ref.get(), g_ref, 1e-12, 2000);
  const auto dev_solve = hdivred_b200::pcg(ref.h_mat, PrecondKind::amg, g_ref, 1e-12, 2000);
  // every PrecondKind through the shim's pcg on the reference's H: the same iteration counts
  bool all_kinds = true;
  for (const auto kind : {PrecondKind::none, PrecondKind::jacobi, PrecondKind::sgs, PrecondKind::amg}) {
    const std::unique_ptr<Preconditioner> pk = kind == PrecondKind::none  ? nullptr
                                               : kind == PrecondKind::jacobi ? jacobi_setup(ref.h_mat)
                                               : kind == PrecondKind::sgs    ? ssgs_setup(ref.h_mat)
                                                                             : amg_preconditioner(ref.h_mat);
    const auto rs = pcg(ref.h_mat, pk.get(), g_ref, 1e-12, 5000);
    const auto ds = hdivred_b200::pcg(ref.h_mat, kind, g_ref, 1e-12, 5000);
    all_kinds = all_kinds && std::llabs(static_cast<long long>(rs.second.iterations - ds.second.iterations)) <= 1 &&
                ds.second.converged == rs.second.converged;
  }
  // near_nullspace_check, bit-identical (small meshes: dense m x m)
  bool ns_identical = true;
  if (ref.h_mat.nrows <= 600) ns_identical = near_nullspace_check(sp, co) == hdivred_b200::near_nullspace_check(sp, co);
  const std::vector<double> y_ref = spmv(ref.h_mat, g_ref);
  const std::vector<double> y_gpu = hdivred_b200::spmv(ref.h_mat, g_ref);
  std::printf("{\"n\": %d, \"k\": %d, \"h_pattern_identical\": %s, \"h_rel\": %.3e, \"g_rel\": %.3e, "
              "\"s_pattern_identical\": %s, \"s_rel\": %.3e, \"spmv_identical\": %s, "
              "\"alg_h_pattern_identical\": %s, \"alg_h_symmetric\": %s, \"alg_h_rel\": %.3e, \"alg_g_rel\": %.3e, "
              "\"alg_x_hat_rel\": %.3e, \"alg_x_rel\": %.3e, \"alg_s_pattern_identical\": %s, \"alg_s_rel\": %.3e, "
              "\"alg_f_s_rel\": %.3e, \"alg_x_cond_rel\": %.3e, \"fe_x_hat_rel\": %.3e, \"fe_x_rel\": %.3e, "
              "\"fe_x_cond_rel\": %.3e, \"solve_hyb_alg_rel\": %.3e, \"solve_hyb_fe_rel\": %.3e, "
              "\"solve_cond_alg_rel\": %.3e, \"solve_cond_fe_rel\": %.3e, \"pcg_iterations\": [%lld, %lld, %lld, %lld, %lld, %lld], "
              "\"amg_iterations\": [%lld, %lld], \"solve_amg_fe_rel\": %.3e, \"amg_ref_matrix_iterations\": [%lld, %lld], "
              "\"amg_ref_matrix_x_rel\": %.3e, \"nullspace_identical\": %s, \"all_precond_iterations_match\": %s}\n",
              n, k, pattern ? "true" : "false", dh / mh, dg / (mg > 0 ? mg : 1), spat ? "true" : "false", ds / ms,
              y_ref == y_gpu ? "true" : "false", apat ? "true" : "false", asym ? "true" : "false",
              rel(ref.h_mat.values, ahyb.h_mat.values), rel(g_ref, g_alg), rel(xh_ref, xh_alg), rel(x_ref, x_alg),
              acpat ? "true" : "false", rel(cref.s_mat.values, acond.s_mat.values), rel(fs_ref, fs_alg),
              rel(xc_ref, xc_alg), rel(xh_ref, xh_fe), rel(x_ref, x_fe), rel(xc_ref, xc_fe), rel(xs_ref, xs_alg),
              rel(xs_ref, xs_fe), rel(xsc_ref, xsc_alg), rel(xsc_ref, xsc_fe), static_cast<long long>(it_ref),
              static_cast<long long>(it_alg), static_cast<long long>(it_fe), static_cast<long long>(itc_ref),
              static_cast<long long>(itc_alg), static_cast<long long>(itc_fe), static_cast<long long>(ita_ref),
              static_cast<long long>(ita_fe), rel(xa_ref, xa_fe), static_cast<long long>(ref_solve.second.iterations),
              static_cast<long long>(dev_solve.second.iterations), rel(ref_solve.first, dev_solve.first),
              ns_identical ? "true" : "false", all_kinds ? "true" : "false");
  return (pattern && spat && y_ref == y_gpu && apat && asym && acpat && ns_identical && all_kinds) ? 0 : 1;
}
