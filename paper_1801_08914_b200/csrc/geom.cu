// Mapped-geometry FE path (config 4: perturbed trilinear hexahedra).
//
// With vertex coordinates attached to a space (hdr_space_set_vertices) every
// cell has its own element matrix, so the structured (shared-factor) element
// solve does not apply.  Per call:
//   K_A  kern_piola.cu   A_T of every cell from alpha, beta and the vertices
//   K_E  kern_alg.cu     element elimination (LU with the reference's
//                        partition and SingularBlock rule, double-double
//                        refined solves) -> H_T, g_T  (or S_hat, f_S / x_hat)
//   K_S  kern_alg.cu     from_triplets sums into the space's CSR pattern, in a
//                        precomputed deterministic order (runs.hpp)
// The per-cell descriptors (partition, multiplier rows, constraint slice) are
// the FE structure of reduction.cpp:236-258 / :31-57, built once here.
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "capi_util.hpp"
#include "geom.hpp"
#include "hdr_device.cuh"
#include "kernels.hpp"
#include "runs.hpp"

namespace hdr {

struct GeomState {
  int n = 0, nint = 0, dpf = 0, nF = 0, nq = 0;
  int64_t ncells = 0, m = 0, ndofs = 0, fdc = 0, broken = 0;
  DevMesh dm{};
  double h[3] = {1, 1, 1}, det0 = 1;
  DBuf<double> verts, qs, bq_val, bq_div, bq_w;
  bool gemm = false;            // k_piola_gemm (component-separable basis) instead of k_piola_assemble
  DBuf<double> tphi, tdiv;      // np x n tables in the component-sorted order
  DBuf<int> perm;
  bool mapped = false;   // trilinear cells (vertices attached); else the affine reference element
  DBuf<double> ref_dm;   // affine: D_ref, M_ref (n x n each)
  // hybrid descriptors
  DBuf<int64_t> boff, aoff, goff, mrows, hoff, cptr;
  DBuf<int> idx_h, ni_h, cent_r, cent_a;
  DBuf<double> cent_v;
  Runs HR, GR;
  AlgPlan plan_h;
  // condense descriptors (built on first use)
  bool cond_ready = false;
  DBuf<int64_t> bdof_off, bm_ptr, bm_ord, soff, ibase, i_global;
  DBuf<int> idx_c, ni_c, bm_loc;
  DBuf<double> bm_w, i_sign;
  Runs SR, FR;
  AlgPlan plan_c;
  // scratch
  DBuf<double> ablk, hbuf, gbuf, sbuf, fsbuf, gws;
  int64_t gws_doubles = 0;
  DBuf<int> status;
  int max_nr = 0;
  bool spd = false;  // hybridize through kern_spd.cu (SPD blocks small enough for shared memory)
  DBuf<unsigned long long> bad;
};

namespace {

int sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

void ensure_ws(GeomState* G, const AlgPlan& p) {
  const int64_t need = alg_gws_doubles(p);
  if (need > G->gws_doubles) {
    G->gws.alloc(static_cast<size_t>(need));
    G->gws_doubles = need;
  }
}

void assemble(GeomState* G, const double* alpha, const double* beta, cudaStream_t st) {
  if (!G->ablk.p) G->ablk.alloc(static_cast<size_t>(G->ncells) * G->n * G->n);
  if (!G->mapped) {  // affine cells (weighted constraint rows): A_T = fl(fl(alpha D) + fl(beta M))
    launch_affine_assemble(G->ncells, G->n, G->ref_dm.p, alpha, beta, G->ablk.p, st);
    return;
  }
  PiolaArgs P{};
  P.n = G->n;
  P.nq = G->nq;
  P.ncells = G->ncells;
  for (int a = 0; a < 3; ++a) {
    P.N[a] = G->dm.N[a];
    P.h[a] = G->h[a];
  }
  P.verts = G->verts.p;
  P.qs = G->qs.p;
  P.bq_val = G->bq_val.p;
  P.bq_div = G->bq_div.p;
  P.bq_w = G->bq_w.p;
  P.det0 = G->det0;
  P.alpha = alpha;
  P.beta = beta;
  P.ablk = G->ablk.p;
  const int grid = static_cast<int>(std::min<int64_t>(G->ncells, static_cast<int64_t>(sms())));
  if (G->gemm) launch_piola_gemm(P, G->tphi.p, G->tdiv.p, G->perm.p, grid > 0 ? grid : 1, st);
  else launch_piola_assemble(P, grid > 0 ? grid : 1, st);
}

AlgArgs hyb_args(GeomState* G, const double* f) {
  AlgArgs a{};
  a.ne = G->ncells;
  a.boff = G->boff.p;
  a.aoff = G->aoff.p;
  a.blocks = G->ablk.p;
  a.idx = G->idx_h.p;
  a.ni = G->ni_h.p;
  a.f = f;
  a.status = G->status.p;
  a.bad_elem = G->bad.p;
  a.m = G->m;
  a.goff = G->goff.p;
  a.mrows = G->mrows.p;
  a.hoff = G->hoff.p;
  a.cptr = G->cptr.p;
  a.cent_r = G->cent_r.p;
  a.cent_a = G->cent_a.p;
  a.cent_v = G->cent_v.p;
  return a;
}

hdr_status read_geom_status(GeomState* G, cudaStream_t st, const char* who) {
  int status = 0;
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&status, G->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&bad, G->bad.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (status) {
    CK(cudaMemsetAsync(G->status.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(G->bad.p, 0xff, sizeof(unsigned long long), st));
    CK(cudaStreamSynchronize(st));
    if (status & 4)
      return fail(HDR_UNSUPPORTED, std::string(who) + ": element block not positive definite (element " +
                                       std::to_string(bad) + ")");
    return fail(HDR_SINGULAR_BLOCK,
                std::string(who) + ": singular block (element " + std::to_string(bad) + ", pivot <= 1e-14 max|block|)");
  }
  return HDR_OK;
}

// local face slot of local dof l (>= nint), and its sub index
inline void slot_of(const GeomState* G, int l, int* s, int* sub) {
  *s = (l - G->nint) / G->dpf;
  *sub = (l - G->nint) % G->dpf;
}

void build_condense(GeomState* G, cudaStream_t st) {
  const int n = G->n, nint = G->nint, nF = G->nF;
  const int64_t ne = G->ncells;
  std::vector<int> idx(static_cast<size_t>(ne) * n), ni(static_cast<size_t>(ne), nint), bm_loc;
  std::vector<int64_t> bdof_off(static_cast<size_t>(ne) + 1), bm_ptr(1, 0), bm_ord, soff(static_cast<size_t>(ne) + 1),
      ibase(static_cast<size_t>(ne) + 1), i_global, trip_off(static_cast<size_t>(ne) + 1), ftrip_off(static_cast<size_t>(ne) + 1);
  std::vector<double> bm_w, i_sign;
  for (int64_t e = 0; e < ne; ++e) {
    int64_t c[3];
    cell_coords(G->dm, e, c);
    for (int l = 0; l < n; ++l) idx[e * n + l] = l;  // marker partition: bubbles first, then the faces
    for (int i = 0; i < nint; ++i) {
      i_global.push_back(G->fdc + e * nint + i);
      i_sign.push_back(1.0);
    }
    for (int j = 0; j < nF; ++j) {
      int s, sub;
      slot_of(G, nint + j, &s, &sub);
      const int64_t f = slot_face(G->dm, c, s, nullptr);
      bm_ord.push_back(f * G->dpf + sub);  // every face dof is a master; ordinal = global
      bm_w.push_back((s & 1) ? 1.0 : -1.0);
      bm_loc.push_back(j);
      bm_ptr.push_back(static_cast<int64_t>(bm_ord.size()));
    }
    bdof_off[e + 1] = bdof_off[e] + nF;
    soff[e + 1] = soff[e] + static_cast<int64_t>(nF) * nF;
    ibase[e + 1] = ibase[e] + nint;
    trip_off[e + 1] = trip_off[e] + static_cast<int64_t>(nF) * nF;
    ftrip_off[e + 1] = ftrip_off[e] + nF;
  }
  G->idx_c.upload(idx);
  G->ni_c.upload(ni);
  G->bdof_off.upload(bdof_off);
  G->bm_ptr.upload(bm_ptr);
  G->bm_ord.upload(bm_ord);
  G->bm_w.upload(bm_w);
  G->bm_loc.upload(bm_loc);
  G->soff.upload(soff);
  G->ibase.upload(ibase);
  G->i_global.upload(i_global);
  G->i_sign.upload(i_sign);
  G->plan_c = alg_plan(ne, nint, nF + 1);
  ensure_ws(G, G->plan_c);
  AlgArgs a{};
  a.ne = ne;
  a.boff = G->boff.p;
  a.ni = G->ni_c.p;
  a.n_master = G->fdc;
  a.bdof_off = G->bdof_off.p;
  a.bm_ptr = G->bm_ptr.p;
  a.bm_ord = G->bm_ord.p;
  a.bm_w = G->bm_w.p;
  a.bm_loc = G->bm_loc.p;
  a.soff = G->soff.p;
  DBuf<int64_t> d_trip, d_ftrip, ssrc, fsrc, row_cnt;
  DBuf<uint64_t> skeys, fkeys;
  DBuf<double> sw, fw;
  d_trip.upload(trip_off);
  d_ftrip.upload(ftrip_off);
  const int64_t T = trip_off.back(), F = ftrip_off.back(), nm = G->fdc;
  skeys.alloc(T);
  ssrc.alloc(T);
  sw.alloc(T);
  fkeys.alloc(F);
  fsrc.alloc(F);
  fw.alloc(F);
  launch_alg_skeys(a, d_trip.p, d_ftrip.p, skeys.p, ssrc.p, sw.p, fkeys.p, fsrc.p, fw.p, st);
  row_cnt.alloc(static_cast<size_t>(nm) + 1);
  CK(cudaMemsetAsync(row_cnt.p, 0, static_cast<size_t>(nm + 1) * 8, st));
  sort_runs(T, skeys, ssrc, &sw, static_cast<uint64_t>(nm) * static_cast<uint64_t>(nm), nm, &row_cnt, G->SR, st);
  sort_runs(F, fkeys, fsrc, &fw, static_cast<uint64_t>(nm), nm, nullptr, G->FR, st);
  G->sbuf.alloc(static_cast<size_t>(T));
  G->fsbuf.alloc(static_cast<size_t>(F));
  G->cond_ready = true;
}

AlgArgs cond_args(GeomState* G, const double* f) {
  AlgArgs a{};
  a.ne = G->ncells;
  a.boff = G->boff.p;
  a.aoff = G->aoff.p;
  a.blocks = G->ablk.p;
  a.idx = G->idx_c.p;
  a.ni = G->ni_c.p;
  a.f = f;
  a.status = G->status.p;
  a.bad_elem = G->bad.p;
  a.n_master = G->fdc;
  a.bdof_off = G->bdof_off.p;
  a.bm_ptr = G->bm_ptr.p;
  a.bm_ord = G->bm_ord.p;
  a.bm_w = G->bm_w.p;
  a.bm_loc = G->bm_loc.p;
  a.soff = G->soff.p;
  a.sbuf = G->sbuf.p;
  a.fsbuf = G->fsbuf.p;
  a.ibase = G->ibase.p;
  a.i_global = G->i_global.p;
  a.i_sign = G->i_sign.p;
  return a;
}

}  // namespace

GeomState* geom_create(const RefElement& re, const DevMesh& dm, const std::vector<int>& mbase, const double h[3],
                       int64_t m, int64_t ndofs, const double* verts_host, bool weighted, cudaStream_t st) {
  if (verts_host && (dm.dim != 3 || re.bq_w.empty())) throw StatusError(HDR_UNSUPPORTED, "mapped geometry needs a 3D space");
  auto G = std::make_unique<GeomState>();
  G->mapped = verts_host != nullptr;
  G->n = re.n;
  G->nint = re.nint;
  G->dpf = re.dpf;
  G->nF = 2 * dm.dim * re.dpf;
  G->nq = re.nq;
  G->ncells = dm.ncells;
  G->m = m;
  G->ndofs = ndofs;
  G->fdc = dm.face_dof_count;
  G->broken = dm.ncells * re.n;
  G->dm = dm;
  for (int a = 0; a < 3; ++a) G->h[a] = h[a];
  G->det0 = h[0] * h[1] * h[2];
  if (G->mapped) {
    const int64_t nv = (dm.N[0] + 1) * (dm.N[1] + 1) * (dm.N[2] + 1);
    G->verts.upload(verts_host, static_cast<size_t>(nv) * 3);
    G->qs.upload(re.qs);
    G->bq_val.upload(re.bq_val);
    G->bq_div.upload(re.bq_div);
    G->bq_w.upload(re.bq_w);
    // component-separable basis (every phi_j has one nonzero component): sorted
    // tables for the GEMM-form assembly
    const int n = re.n, np = static_cast<int>(re.bq_w.size());
    std::vector<int> comp(static_cast<size_t>(n), -1);
    bool sep = piola_gemm_supported(n, np) && !getenv("HDR_PIOLA_DIRECT");
    for (int j = 0; j < n && sep; ++j)
      for (int p = 0; p < np && sep; ++p)
        for (int c = 0; c < 3; ++c)
          if (re.bq_val[(static_cast<size_t>(p) * n + j) * 3 + c] != 0.0) {
            if (comp[j] >= 0 && comp[j] != c) sep = false;
            comp[j] = c;
          }
    std::vector<int> perm;
    for (int c = 0; c < 3 && sep; ++c)
      for (int j = 0; j < n; ++j)
        if (comp[j] == c) perm.push_back(j);
    sep = sep && static_cast<int>(perm.size()) == n;
    for (int c = 0; c < 3 && sep; ++c)
      sep = std::count(comp.begin(), comp.end(), c) == n / 3;
    if (sep) {
      std::vector<double> tp(static_cast<size_t>(np) * n), td(static_cast<size_t>(np) * n);
      for (int p = 0; p < np; ++p)
        for (int jj = 0; jj < n; ++jj) {
          const int j = perm[jj];
          tp[static_cast<size_t>(p) * n + jj] = re.bq_val[(static_cast<size_t>(p) * n + j) * 3 + comp[j]];
          td[static_cast<size_t>(p) * n + jj] = re.bq_div[static_cast<size_t>(p) * n + j];
        }
      G->tphi.upload(tp);
      G->tdiv.upload(td);
      G->perm.upload(perm);
      G->gemm = true;
    }
  } else {
    std::vector<double> dmv(re.divdiv);
    dmv.insert(dmv.end(), re.mass.begin(), re.mass.end());
    G->ref_dm.upload(dmv);
  }
  G->status.alloc(1);
  CK(cudaMemset(G->status.p, 0, sizeof(int)));
  G->bad.alloc(1);
  CK(cudaMemset(G->bad.p, 0xff, sizeof(unsigned long long)));

  // hybrid descriptors: i = bubbles + boundary-face dofs, b = interior-face
  // dofs (zero columns of C, reduction.cpp:236-258); multiplier rows = the
  // interior faces' multiplier dofs in slot order (ascending face order)
  const int n = re.n, nint = re.nint, dpf = re.dpf;
  const int64_t ne = dm.ncells;
  std::vector<int> idx(static_cast<size_t>(ne) * n), ni(static_cast<size_t>(ne)), cent_r, cent_a;
  std::vector<int64_t> boff(static_cast<size_t>(ne) + 1), aoff(static_cast<size_t>(ne)), goff(static_cast<size_t>(ne) + 1),
      hoff(static_cast<size_t>(ne) + 1), mrows, cptr;
  std::vector<double> cent_v;
  int max_nr = 0;
  for (int64_t e = 0; e < ne; ++e) {
    boff[e + 1] = boff[e] + n;
    aoff[e] = e * static_cast<int64_t>(n) * n;
    int64_t c[3];
    cell_coords(dm, e, c);
    int64_t face[6];
    bool in[6];
    for (int s = 0; s < 2 * dm.dim; ++s) face[s] = slot_face(dm, c, s, &in[s]);
    int k = 0;
    for (int l = 0; l < nint; ++l) idx[e * n + k++] = l;
    for (int s = 0; s < 2 * dm.dim; ++s)
      if (!in[s])
        for (int sub = 0; sub < dpf; ++sub) idx[e * n + k++] = nint + s * dpf + sub;
    ni[e] = k;
    int nr = 0;
    for (int s = 0; s < 2 * dm.dim; ++s)
      if (in[s]) {
        const int k0 = k;  // position of the slot's first dof in the [i | b] order
        for (int sub = 0; sub < dpf; ++sub) idx[e * n + k++] = nint + s * dpf + sub;
        for (int r = 0; r < dpf; ++r) {
          cptr.push_back(static_cast<int64_t>(cent_v.size()));
          if (!weighted) {  // unit rows: one +1 per interior-face dof (build_C, reduction.cpp:172-181)
            cent_r.push_back(nr);
            cent_a.push_back(k0 + r);
            cent_v.push_back(1.0);
          } else {  // weighted rows: face moments over the slot's dofs (reduction.cpp:182-195)
            const double* fm = re.face_moments.data() + (static_cast<size_t>(s) * dpf + r) * n;
            for (int sub = 0; sub < dpf; ++sub) {
              cent_r.push_back(nr);
              cent_a.push_back(k0 + sub);
              cent_v.push_back(fm[nint + s * dpf + sub]);
            }
          }
          mrows.push_back(static_cast<int64_t>(mbase[face[s]]) + r);
          ++nr;
        }
      }
    goff[e + 1] = goff[e] + nr;
    hoff[e + 1] = hoff[e] + static_cast<int64_t>(nr) * nr;
    max_nr = std::max(max_nr, nr);
  }
  cptr.push_back(static_cast<int64_t>(cent_v.size()));
  G->boff.upload(boff);
  G->aoff.upload(aoff);
  G->idx_h.upload(idx);
  G->ni_h.upload(ni);
  G->goff.upload(goff);
  G->hoff.upload(hoff);
  G->mrows.upload(mrows);
  G->cptr.upload(cptr);
  G->cent_r.upload(cent_r);
  G->cent_a.upload(cent_a);
  G->cent_v.upload(cent_v);
  G->plan_h = alg_plan(ne, n, max_nr + 1);
  ensure_ws(G.get(), G->plan_h);
  G->max_nr = max_nr;
  G->spd = !getenv("HDR_NO_SPD") && spd_supported(n, max_nr + 1);
  if (G->spd) {
    int grid = 1;
    const int64_t need = spd_gws_doubles(ne, n, max_nr + 1, &grid);
    if (need > G->gws_doubles) {
      G->gws.alloc(static_cast<size_t>(need));
      G->gws_doubles = need;
    }
  }
  G->hbuf.alloc(static_cast<size_t>(hoff.back()));
  G->gbuf.alloc(static_cast<size_t>(goff.back()));
  // from_triplets order of H and g, once
  AlgArgs a = hyb_args(G.get(), nullptr);
  const int64_t T = hoff.back(), Gn = goff.back();
  DBuf<uint64_t> hkeys, gkeys;
  DBuf<int64_t> hsrc, gsrc, row_cnt;
  hkeys.alloc(T);
  hsrc.alloc(T);
  gkeys.alloc(Gn);
  gsrc.alloc(Gn);
  launch_alg_hkeys(a, hkeys.p, hsrc.p, gkeys.p, gsrc.p, st);
  row_cnt.alloc(static_cast<size_t>(m) + 1);
  CK(cudaMemsetAsync(row_cnt.p, 0, static_cast<size_t>(m + 1) * 8, st));
  sort_runs(T, hkeys, hsrc, nullptr, static_cast<uint64_t>(m > 0 ? m : 1) * static_cast<uint64_t>(m > 0 ? m : 1), m,
            &row_cnt, G->HR, st);
  sort_runs(Gn, gkeys, gsrc, nullptr, static_cast<uint64_t>(m > 0 ? m : 1), m, nullptr, G->GR, st);
  CK(cudaStreamSynchronize(st));
  return G.release();
}

void geom_destroy(GeomState* G) { delete G; }

int64_t geom_nnz_h(const GeomState* G) { return G->HR.nruns; }

hdr_status geom_hybridize(GeomState* G, const double* alpha, const double* beta, const double* f, double* hval,
                          double* g, cudaStream_t st) {
  assemble(G, alpha, beta, st);
  AlgArgs a = hyb_args(G, f);
  a.hbuf = G->hbuf.p;
  a.gbuf = G->gbuf.p;
  if (G->spd) launch_spd_hyb(a, G->n, G->max_nr + 1, G->gws.p, st);
  else launch_alg(a, ALG_HYB, G->plan_h, G->gws.p, st);
  launch_run_sum(G->HR.nruns, G->HR.start.p, G->HR.src.p, nullptr, G->hbuf.p, hval, nullptr, 0, st);
  CK(cudaMemsetAsync(g, 0, static_cast<size_t>(G->m) * 8, st));
  launch_run_sum(G->GR.nruns, G->GR.start.p, G->GR.src.p, nullptr, G->gbuf.p, g, G->GR.index.p, 1, st);
  return read_geom_status(G, st, "hybridize");
}

hdr_status geom_recover_hybrid(GeomState* G, const double* alpha, const double* beta, const double* lambda,
                               const double* f, double* x_hat, double* x, cudaStream_t st) {
  assemble(G, alpha, beta, st);
  AlgArgs a = hyb_args(G, f);
  a.lambda = lambda;
  a.x_hat = x_hat;
  launch_alg(a, ALG_REC, G->plan_h, G->gws.p, st);
  launch_average_faces(G->dm, x_hat, x, st);
  return read_geom_status(G, st, "recover_hybrid");
}

hdr_status geom_condense(GeomState* G, const double* alpha, const double* beta, const double* f, double* sval,
                         double* fs, cudaStream_t st) {
  if (!G->cond_ready) build_condense(G, st);
  assemble(G, alpha, beta, st);
  AlgArgs a = cond_args(G, f);
  launch_alg(a, ALG_COND, G->plan_c, G->gws.p, st);
  launch_run_sum(G->SR.nruns, G->SR.start.p, G->SR.src.p, G->SR.w.p, G->sbuf.p, sval, nullptr, 0, st);
  CK(cudaMemsetAsync(fs, 0, static_cast<size_t>(G->fdc) * 8, st));
  launch_run_sum(G->FR.nruns, G->FR.start.p, G->FR.src.p, G->FR.w.p, G->fsbuf.p, fs, G->FR.index.p, 1, st);
  return read_geom_status(G, st, "static_condense");
}

hdr_status geom_recover_condensed(GeomState* G, const double* alpha, const double* beta, const double* x_b,
                                  const double* f, double* x, cudaStream_t st) {
  if (!G->cond_ready) build_condense(G, st);
  assemble(G, alpha, beta, st);
  CK(cudaMemsetAsync(x, 0, static_cast<size_t>(G->ndofs) * 8, st));
  CK(cudaMemcpyAsync(x, x_b, static_cast<size_t>(G->fdc) * 8, cudaMemcpyDeviceToDevice, st));  // masters = face dofs
  AlgArgs a = cond_args(G, f);
  a.xb = x_b;
  a.x = x;
  launch_alg(a, ALG_RECC, G->plan_c, G->gws.p, st);
  return read_geom_status(G, st, "recover_condensed");
}

const double* geom_element_blocks(const GeomState* G) { return G->ablk.p; }
void geom_assemble_blocks(GeomState* G, const double* alpha, const double* beta, cudaStream_t st) {
  assemble(G, alpha, beta, st);
}
bool geom_mapped(const GeomState* G) { return G->mapped; }

}  // namespace hdr
