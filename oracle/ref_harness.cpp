// ref_harness: drives the UNMODIFIED reference library (oracle/_ref/libhdivred_ref.a,
// compiled from /root/reference/proj/src by oracle/Makefile) on the seeded synthetic
// inputs of SURVEY.md §8(d), and either dumps every hot-path output to a binary
// file (golden fixtures, oracle pinning) or times the hot path (bench.py's
// reference arm / cpu_baseline leg).
//
// TEST INFRASTRUCTURE ONLY. Nothing in the product links or executes this.
//
// Reference calls (file:line under /root/reference/proj):
//   build_mesh            src/mesh.cpp:137        build_space        src/rt_space.cpp:318
//   build_reduction_inputs src/reduction.cpp:200  hybridize          src/reduction.cpp:262
//   recover_hybrid        src/reduction.cpp:356   static_condense    src/reduction.cpp:448
//   recover_condensed     src/reduction.cpp:559   spmv               src/csr.cpp:77
//   element_matrices      src/rt_space.cpp:370    local_dof_map      src/rt_space.cpp:383
//   amg_setup / amg_apply src/amg.cpp:189, 268    ssgs_setup / pcg   src/solvers.cpp:185, 109
//
// Input generation follows SURVEY.md §8(d): xorshift64 (tests/test_support.hpp:79-92
// semantics), draw order per cell alpha then beta, then f_hat in broken order,
// then lambda (m values), then x_b (n_S values).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "hdivred/amg.hpp"
#include "hdivred/csr.hpp"
#include "hdivred/mesh.hpp"
#include "hdivred/solvers.hpp"
#include "hdivred/block_io.hpp"
#include "hdivred/matrix_market.hpp"
#include "hdivred/reduction.hpp"
#include "hdivred/rt_space.hpp"

using namespace hdivred;

namespace {

struct Rng {  // xorshift64, same recurrence and scaling as the reference test RNG
  std::uint64_t s;
  explicit Rng(std::uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  std::uint64_t next() {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double log_uniform(double lo, double hi) { return std::exp(uniform(std::log(lo), std::log(hi))); }
};

std::map<std::string, std::string> parse(int argc, char** argv) {
  std::map<std::string, std::string> kv;
  for (int i = 2; i < argc; ++i) {
    const char* eq = std::strchr(argv[i], '=');
    if (!eq) throw std::invalid_argument(std::string("bad argument ") + argv[i]);
    kv[std::string(argv[i], static_cast<std::size_t>(eq - argv[i]))] = eq + 1;
  }
  return kv;
}

std::vector<double> split_d(const std::string& s, char sep) {
  std::vector<double> out;
  std::size_t p = 0;
  while (p <= s.size()) {
    std::size_t q = s.find(sep, p);
    if (q == std::string::npos) q = s.size();
    out.push_back(std::strtod(s.substr(p, q - p).c_str(), nullptr));
    p = q + 1;
  }
  return out;
}

struct Problem {
  RtSpace space;
  CellCoefficients coeffs;
  std::vector<double> f_hat;
  Rng rng{1};
};

// coef = "uniform:a:b" | "logu:lo:hi" | "softhard:p" | "checker:sig_lo:sig_hi" (cfg5: alpha_ref = 1
// divdiv, beta_ref = 1/(3 sigma_t) mass, regions (floor(4x)+floor(4y)+floor(4z)) mod 2)
Problem make_problem(const std::map<std::string, std::string>& kv) {
  const int dim = std::stoi(kv.at("dim"));
  const auto cells_d = split_d(kv.at("cells"), ',');
  std::array<index_t, 3> cells{1, 1, 1};
  std::array<double, 3> h{1.0, 1.0, 1.0};
  for (int a = 0; a < dim; ++a) {
    cells[a] = static_cast<index_t>(cells_d.at(a));
    h[a] = 1.0 / static_cast<double>(cells[a]);
  }
  if (kv.count("h")) {  // cell sizes of a sub-mesh that keeps the full mesh's element
    const auto hs = split_d(kv.at("h"), ',');
    for (int a = 0; a < dim; ++a) h[a] = hs.at(a);
  }
  const int k = std::stoi(kv.at("k"));
  const std::uint64_t seed = std::stoull(kv.at("seed"));
  const std::string coef = kv.count("coef") ? kv.at("coef") : "uniform:1:1";

  Problem pb;
  pb.rng = Rng(seed);
  const CartesianMesh mesh = build_mesh(dim, cells, h);
  pb.space = build_space(mesh, k);
  const index_t nc = mesh.ncells();
  pb.coeffs.alpha.resize(nc);
  pb.coeffs.beta.resize(nc);
  const std::string kind = coef.substr(0, coef.find(':'));
  const auto par = split_d(coef.substr(coef.find(':') + 1), ':');
  if (kind == "uniform") {
    for (index_t c = 0; c < nc; ++c) {
      pb.coeffs.alpha[c] = par.at(0);
      pb.coeffs.beta[c] = par.at(1);
    }
  } else if (kind == "logu") {
    for (index_t c = 0; c < nc; ++c) {
      pb.coeffs.alpha[c] = pb.rng.log_uniform(par.at(0), par.at(1));
      pb.coeffs.beta[c] = pb.rng.log_uniform(par.at(0), par.at(1));
    }
  } else if (kind == "checker") {
    for (index_t c = 0; c < nc; ++c) {
      const auto x = mesh.cell_center(c);
      long reg = 0;
      for (int a = 0; a < dim; ++a) reg += static_cast<long>(std::floor(4.0 * x[a]));
      const double sigma = (reg % 2 == 0) ? par.at(0) : par.at(1);
      pb.coeffs.alpha[c] = 1.0;
      pb.coeffs.beta[c] = 1.0 / (3.0 * sigma);
    }
  } else if (kind == "softhard") {  // the reference's own preset (src/mesh.cpp:168-191)
    pb.coeffs = soft_hard_coefficients(mesh, static_cast<int>(par.at(0)));
  } else {
    throw std::invalid_argument("unknown coef kind " + kind);
  }
  pb.f_hat.resize(pb.space.broken_ndofs);
  for (auto& v : pb.f_hat) v = pb.rng.uniform(-1.0, 1.0);
  return pb;
}

struct Writer {
  std::FILE* f;
  explicit Writer(const std::string& path) : f(std::fopen(path.c_str(), "wb")) {
    if (!f) throw std::runtime_error("cannot open " + path);
    std::fwrite("HDRB0001", 1, 8, f);
  }
  ~Writer() { std::fclose(f); }
  void rec(const std::string& name, char type, const void* data, std::uint64_t count) {
    const std::uint32_t len = static_cast<std::uint32_t>(name.size());
    std::fwrite(&len, 4, 1, f);
    std::fwrite(name.data(), 1, len, f);
    std::fwrite(&type, 1, 1, f);
    std::fwrite(&count, 8, 1, f);
    if (count) std::fwrite(data, 8, count, f);
  }
  void d(const std::string& n, const std::vector<double>& v) { rec(n, 'd', v.data(), v.size()); }
  void q(const std::string& n, const std::vector<index_t>& v) { rec(n, 'q', v.data(), v.size()); }
  void csr(const std::string& n, const CsrMatrix& a) {
    q(n + ".shape", {a.nrows, a.ncols});
    q(n + ".row_offsets", a.row_offsets);
    q(n + ".col_indices", a.col_indices);
    d(n + ".values", a.values);
  }
};

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int cmd_dump(const std::map<std::string, std::string>& kv) {
  Problem pb = make_problem(kv);
  const bool weighted = kv.count("weighted") && kv.at("weighted") == "1";
  const bool blocks = !kv.count("blocks") || kv.at("blocks") == "1";
  const RtSpace& sp = pb.space;
  ReductionInputs in = build_reduction_inputs(sp, pb.coeffs, weighted);
  in.f_hat = pb.f_hat;
  Writer w(kv.at("out"));
  // essential=1: eliminate_essential (src/reduction.cpp:589-698) on every boundary
  // face, prescribed normal fluxes drawn U[-1, 1] after f_hat; everything below then
  // runs on the reduced inputs (as build_problem does, src/driver.cpp:187-195)
  if (kv.count("essential") && kv.at("essential") == "1") {
    std::vector<EssentialBc> bcs;
    std::vector<double> flux;
    for (index_t f = 0; f < sp.mesh.nfaces(); ++f)
      if (sp.mesh.face(f).is_boundary) {
        bcs.push_back({f, pb.rng.uniform(-1.0, 1.0)});
        flux.push_back(bcs.back().normal_flux);
      }
    EliminationResult el = eliminate_essential(sp, in, bcs);
    w.d("ess.flux", flux);
    w.q("ess.kept_globals", el.kept_globals);
    w.d("ess.prescribed", el.prescribed);
    w.q("ess.interior_global_begin", {el.inputs.interior_global_begin});
    std::vector<index_t> sizes;
    for (const auto& b : el.inputs.a_hat.blocks) sizes.push_back(static_cast<index_t>(b.dof_map.size()));
    w.q("ess.block_sizes", sizes);
    in = std::move(el.inputs);
  }
  w.q("meta", {sp.mesh.dim, sp.mesh.ncells_per_axis[0], sp.mesh.ncells_per_axis[1], sp.mesh.ncells_per_axis[2],
               sp.order, sp.element_ndofs, sp.dofs_per_face, sp.interior_dofs_per_cell, sp.mesh.ncells(),
               sp.mesh.nfaces(), sp.ndofs, sp.face_dof_count, sp.broken_ndofs, in.c_mat.nrows,
               weighted ? 1 : 0});
  w.d("h", {sp.mesh.cell_sizes[0], sp.mesh.cell_sizes[1], sp.mesh.cell_sizes[2]});
  w.d("ref_divdiv", sp.ref_divdiv.entries);
  w.d("ref_mass", sp.ref_mass.entries);
  {
    std::vector<double> fm;
    for (const auto& m : sp.ref_face_moments) fm.insert(fm.end(), m.entries.begin(), m.entries.end());
    w.d("ref_face_moments", fm);
    std::vector<double> ul;
    for (const auto& u : sp.ref_unit_load) ul.insert(ul.end(), u.begin(), u.end());
    w.d("ref_unit_load", ul);
  }
  w.d("ref_div_form", sp.ref_div_form.entries);
  w.d("alpha", pb.coeffs.alpha);
  w.d("beta", pb.coeffs.beta);
  w.d("f_hat", in.f_hat);
  if (blocks) {
    std::vector<double> a;
    std::vector<index_t> gl;
    std::vector<double> sg;
    for (const auto& b : in.a_hat.blocks) {
      a.insert(a.end(), b.matrix.entries.begin(), b.matrix.entries.end());
      for (const auto& d : b.dof_map) {
        gl.push_back(d.global);
        sg.push_back(d.sign);
      }
    }
    w.d("a_hat", a);
    w.q("dof_global", gl);
    w.d("dof_sign", sg);
  }
  w.csr("P", in.p_mat);
  w.csr("C", in.c_mat);

  const auto [hyb, g] = hybridize(in);
  w.csr("H", hyb.h_mat);
  // near_nullspace_check (src/reduction.cpp:711-742): eigenvalues of C Y C^T
  if (kv.count("nullspace") && kv.at("nullspace") == "1" && in.c_mat.nrows * in.c_mat.nrows <= kDefaultDenseCap)
    w.d("nullspace", near_nullspace_check(sp, pb.coeffs, weighted));
  w.d("g", g);
  // amg=1: the reduced solve of solve_reduction (src/driver.cpp:203-247) on H:
  // the AMG hierarchy, one V-cycle and one SGS application on g, and pcg
  // (rtol, maxit of RunConfig) with each preconditioner
  if (kv.count("amg") && kv.at("amg") == "1" && hyb.h_mat.nrows > 0) {
    const double rtol = kv.count("rtol") ? std::stod(kv.at("rtol")) : 1e-12;
    AmgOptions aopt;  // amg_theta / amg_cap / amg_levels / amg_omega: non-default AmgOptions
    if (kv.count("amg_theta")) aopt.strength_threshold = std::stod(kv.at("amg_theta"));
    if (kv.count("amg_cap")) aopt.coarse_cap = std::stoll(kv.at("amg_cap"));
    if (kv.count("amg_levels")) aopt.max_levels = std::stoi(kv.at("amg_levels"));
    if (kv.count("amg_omega")) aopt.omega_factor = std::stod(kv.at("amg_omega"));
    const double ts0 = now();
    const AmgHierarchy ah = amg_setup(hyb.h_mat, aopt);
    const double ts1 = now();
    std::fprintf(stderr, "{\"amg_setup_s\": %.4f}\n", ts1 - ts0);
    w.q("amg.levels", {static_cast<index_t>(ah.levels.size())});
    for (std::size_t l = 0; l < ah.levels.size(); ++l) {
      w.csr("amg.A" + std::to_string(l), ah.levels[l].matrix);
      w.csr("amg.P" + std::to_string(l), ah.levels[l].prolongator);
      w.csr("amg.R" + std::to_string(l), ah.levels[l].restriction);
    }
    w.csr("amg.coarse", ah.coarse_matrix);
    w.d("amg.z", amg_apply(ah, g));
    std::vector<double> zs;
    ssgs_setup(hyb.h_mat)->apply(g, zs);
    w.d("sgs.z", zs);
    const std::pair<const char*, std::unique_ptr<Preconditioner>> pcs[] = {
        {"amg", amg_preconditioner(hyb.h_mat)}, {"sgs", ssgs_setup(hyb.h_mat)}, {"jacobi", jacobi_setup(hyb.h_mat)}};
    for (const auto& [name, pc] : pcs) {
      auto [sol, rep] = pcg(hyb.h_mat, pc.get(), g, rtol, 2000);
      std::fprintf(stderr, "{\"pcg\": \"%s\", \"iterations\": %lld, \"wall_s\": %.4f}\n", name,
                   static_cast<long long>(rep.iterations), rep.wall_time);
      w.q(std::string("pcg.") + name + ".iterations", {rep.iterations});
      w.d(std::string("pcg.") + name + ".residuals", rep.relative_residuals);
      w.d(std::string("pcg.") + name + ".x", sol);
    }
  }
  std::vector<double> lambda(static_cast<std::size_t>(hyb.h_mat.nrows));
  for (auto& v : lambda) v = pb.rng.uniform(-1.0, 1.0);
  w.d("lambda", lambda);
  const auto [x_hat, x] = recover_hybrid(hyb, lambda, in.f_hat);
  w.d("x_hat", x_hat);
  w.d("x", x);
  w.d("H_lambda", spmv(hyb.h_mat, lambda));

  const auto [cond, f_s] = static_condense(in);
  w.csr("S", cond.s_mat);
  w.d("f_s", f_s);
  w.q("master_globals", cond.master_globals);
  std::vector<double> x_b(static_cast<std::size_t>(cond.s_mat.nrows));
  for (auto& v : x_b) v = pb.rng.uniform(-1.0, 1.0);
  w.d("x_b", x_b);
  w.d("x_cond", recover_condensed(cond, x_b, in.f_hat));
  w.d("S_x_b", spmv(cond.s_mat, x_b));
  return 0;
}

// Times the metric's assemble + eliminate + scatter (build_reduction_inputs +
// hybridize), and separately hybridize, static_condense and recover_hybrid.
// Prints one JSON object per repetition.
int cmd_bench(const std::map<std::string, std::string>& kv) {
  const int reps = kv.count("reps") ? std::stoi(kv.at("reps")) : 1;
  const bool do_sc = !kv.count("sc") || kv.at("sc") == "1";
  const bool do_rec = !kv.count("rec") || kv.at("rec") == "1";
  Problem pb = make_problem(kv);
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    ReductionInputs in = build_reduction_inputs(pb.space, pb.coeffs, false);
    const double t1 = now();
    in.f_hat = pb.f_hat;
    auto hp = hybridize(in);
    const double t2 = now();
    double t_sc = 0.0, t_rec = 0.0;
    if (do_rec) {
      std::vector<double> lambda(static_cast<std::size_t>(hp.first.h_mat.nrows), 0.25);
      const double a = now();
      auto rr = recover_hybrid(hp.first, lambda, in.f_hat);
      t_rec = now() - a;
    }
    if (do_sc) {
      const double a = now();
      auto sc = static_condense(in);
      t_sc = now() - a;
    }
    std::printf(
        "{\"cells\": %lld, \"inputs_s\": %.6f, \"hybridize_s\": %.6f, \"metric_s\": %.6f, \"static_condense_s\": %.6f, "
        "\"recover_hybrid_s\": %.6f, \"nnz_h\": %lld}\n",
        static_cast<long long>(pb.space.mesh.ncells()), t1 - t0, t2 - t1, t2 - t0, t_sc, t_rec,
        static_cast<long long>(hp.first.h_mat.nnz()));
    std::fflush(stdout);
  }
  return 0;
}

}  // namespace

// export prefix=P: the problem's ReductionInputs through the reference's own
// writers (P.blocks, P.p.mtx, P.c.mtx, P.f.mtx, P.f.txt); import prefix=P: reads
// them back with the reference's readers and prints the seconds taken.
int cmd_export(const std::map<std::string, std::string>& kv) {
  Problem pb = make_problem(kv);
  const bool weighted = kv.count("weighted") && kv.at("weighted") == "1";
  ReductionInputs in = build_reduction_inputs(pb.space, pb.coeffs, weighted);
  in.f_hat = pb.f_hat;
  const std::string pre = kv.at("prefix");
  const double t0 = now();
  write_block_operator(pre + ".blocks", in.a_hat);
  write_matrix_market(pre + ".p.mtx", in.p_mat);
  write_matrix_market(pre + ".c.mtx", in.c_mat);
  write_vector_market(pre + ".f.mtx", in.f_hat);
  write_vector_lines(pre + ".f.txt", in.f_hat);
  std::printf("{\"write_s\": %.6f}\n", now() - t0);
  return 0;
}

int cmd_import(const std::map<std::string, std::string>& kv) {
  const std::string pre = kv.at("prefix");
  const double t0 = now();
  const ElementBlockOperator a = read_block_operator(pre + ".blocks");
  const double t1 = now();
  const CsrMatrix p = read_matrix_market(pre + ".p.mtx");
  const CsrMatrix c = read_matrix_market(pre + ".c.mtx");
  const std::vector<double> f = read_vector_market(pre + ".f.mtx");
  const double t2 = now();
  std::printf("{\"blocks_s\": %.6f, \"mtx_s\": %.6f, \"nblocks\": %zu, \"c_nnz\": %lld, \"f\": %zu}\n", t1 - t0,
              t2 - t1, a.blocks.size(), static_cast<long long>(c.nnz()), f.size());
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_harness dump|bench key=value...\n");
    return 2;
  }
  try {
    const auto kv = parse(argc, argv);
    const std::string cmd = argv[1];
    if (cmd == "dump") return cmd_dump(kv);
    if (cmd == "bench") return cmd_bench(kv);
    if (cmd == "export") return cmd_export(kv);
    if (cmd == "import") return cmd_import(kv);
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_harness: %s\n", e.what());
    return 1;
  }
}
