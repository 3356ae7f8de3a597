// C ABI of the algebraic batch path (include/hdivred_b200.h, "algebraic batch"):
// hybridize / static_condense / recover_* on a general ReductionInputs.
//
// Host work here is structural only — the partition of each block's dofs
// (reduction.cpp:236-258), its multiplier rows and constraint slice
// (constraint_slice, :31-57), master numbering (:509-521) — i.e. integer index
// bookkeeping over the caller's CSR arrays.  Every floating-point operation
// (factorizations, solves, Schur complements, products with C / A_bi, the
// triplet sums of from_triplets, P^T x_hat, the Gram CG) runs on the device
// (kern_alg.cu); there is no CPU compute path.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "kernels.hpp"
#include "runs.hpp"

using namespace hdr;

struct hdr_alg_s {
  int kind = 0;  // 0 hybrid, 1 condensed
  cudaStream_t st = nullptr;
  int64_t ne = 0, n_hat = 0, n_global = 0, m = 0, nrows = 0, nnz = 0, n_master = 0;
  bool diagonal_gram = true;
  AlgPlan plan;
  // element data kept for the recoveries
  DBuf<int64_t> boff, aoff, goff, mrows, hoff, cptr, bdof_off, bm_ptr, bm_ord, soff, ibase, i_global, masters;
  DBuf<int> idx, ni, cent_r, cent_a, bm_loc;
  DBuf<double> blocks, cent_v, bm_w, i_sign;
  DBuf<int> status;
  DBuf<unsigned long long> bad;
  DBuf<double> gws;
  // results
  DBuf<int64_t> row_offsets, col_indices;
  DBuf<double> values, rhs;
  std::vector<int64_t> master_globals;
  // P and P^T (hybrid recovery)
  DBuf<int64_t> p_ro, p_ci, pt_ro, pt_ci;
  DBuf<double> p_v, pt_v, scale;
  ~hdr_alg_s() {
    if (st) cudaStreamDestroy(st);
  }
};

namespace {

int sm_count_alg() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

void check_csr(const char* what, int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci, const double* v) {
  if (nrows < 0 || ncols < 0) throw StatusError(HDR_VALIDATION, std::string(what) + ": negative dimension");
  if (!ro) throw StatusError(HDR_INVALID_ARGUMENT, std::string(what) + ": null row_offsets");
  if (ro[0] != 0) throw StatusError(HDR_VALIDATION, std::string(what) + ": row_offsets[0] != 0");
  for (int64_t r = 0; r < nrows; ++r)
    if (ro[r + 1] < ro[r]) throw StatusError(HDR_VALIDATION, std::string(what) + ": row_offsets not monotone");
  const int64_t nnz = ro[nrows];
  if (nnz > 0 && (!ci || !v)) throw StatusError(HDR_INVALID_ARGUMENT, std::string(what) + ": null column / value array");
  for (int64_t k = 0; k < nnz; ++k)
    if (ci[k] < 0 || ci[k] >= ncols) throw StatusError(HDR_VALIDATION, std::string(what) + ": column index out of range");
}

// n_hat and block offsets; dimension checks of hybridize / static_condense
std::vector<int64_t> check_inputs(const hdr_alg_inputs* in, const char* who) {
  if (!in) throw StatusError(HDR_INVALID_ARGUMENT, "null inputs");
  if (in->nblocks < 0 || (in->nblocks > 0 && (!in->block_sizes || !in->blocks)))
    throw StatusError(HDR_INVALID_ARGUMENT, std::string(who) + ": missing blocks");
  std::vector<int64_t> off(static_cast<size_t>(in->nblocks) + 1, 0);
  for (int64_t e = 0; e < in->nblocks; ++e) {
    if (in->block_sizes[e] < 0) throw StatusError(HDR_VALIDATION, std::string(who) + ": negative block size");
    if (in->block_sizes[e] > 4096) throw StatusError(HDR_UNSUPPORTED, std::string(who) + ": block larger than 4096 dofs");
    off[e + 1] = off[e] + in->block_sizes[e];
  }
  const int64_t n_hat = off.back();
  if (in->c_ncols != n_hat || in->p_nrows != n_hat || in->f_len != n_hat)
    throw StatusError(HDR_DIMENSION_MISMATCH, std::string(who) + ": inconsistent input dimensions");
  if (n_hat > 0 && !in->f_hat) throw StatusError(HDR_INVALID_ARGUMENT, std::string(who) + ": null f_hat");
  check_csr("p_mat", in->p_nrows, in->p_ncols, in->p_row_offsets, in->p_col_indices, in->p_values);
  check_csr("c_mat", in->c_nrows, in->c_ncols, in->c_row_offsets, in->c_col_indices, in->c_values);
  return off;
}

// transpose structure of a CSR matrix: for each column, its (row, position) in row order
void transpose_csr(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci, std::vector<int64_t>& tro,
                   std::vector<int64_t>& trow, std::vector<int64_t>& tpos) {
  tro.assign(static_cast<size_t>(ncols) + 1, 0);
  const int64_t nnz = ro[nrows];
  for (int64_t k = 0; k < nnz; ++k) ++tro[ci[k] + 1];
  for (int64_t c = 0; c < ncols; ++c) tro[c + 1] += tro[c];
  trow.resize(static_cast<size_t>(nnz));
  tpos.resize(static_cast<size_t>(nnz));
  std::vector<int64_t> fill(tro.begin(), tro.end() - 1);
  for (int64_t r = 0; r < nrows; ++r)
    for (int64_t k = ro[r]; k < ro[r + 1]; ++k) {
      const int64_t q = fill[ci[k]]++;
      trow[q] = r;
      tpos[q] = k;
    }
}

void finish_launch_config(hdr_alg_s* op, int dmax, int ncmax) {
  op->plan = alg_plan(op->ne, dmax, ncmax);
  op->gws.alloc(static_cast<size_t>(alg_gws_doubles(op->plan)));
}

hdr_status read_status(hdr_alg_s* op, const char* who) {
  int status = 0;
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&status, op->status.p, sizeof(int), cudaMemcpyDeviceToHost, op->st));
  CK(cudaMemcpyAsync(&bad, op->bad.p, sizeof(bad), cudaMemcpyDeviceToHost, op->st));
  CK(cudaStreamSynchronize(op->st));
  CK(cudaGetLastError());
  if (status) {
    CK(cudaMemsetAsync(op->status.p, 0, sizeof(int), op->st));
    CK(cudaMemsetAsync(op->bad.p, 0xff, sizeof(unsigned long long), op->st));
    CK(cudaStreamSynchronize(op->st));
    if (status & 2)
      return fail(HDR_SINGULAR_BLOCK, std::string(who) + ": singular block (element " + std::to_string(bad) +
                                          ", pivot <= 1e-14 max|block|)");
  }
  return HDR_OK;
}

AlgArgs base_args(hdr_alg_s* op) {
  AlgArgs a{};
  a.ne = op->ne;
  a.boff = op->boff.p;
  a.aoff = op->aoff.p;
  a.blocks = op->blocks.p;
  a.idx = op->idx.p;
  a.ni = op->ni.p;
  a.status = op->status.p;
  a.bad_elem = op->bad.p;
  a.m = op->m;
  a.goff = op->goff.p;
  a.mrows = op->mrows.p;
  a.hoff = op->hoff.p;
  a.cptr = op->cptr.p;
  a.cent_r = op->cent_r.p;
  a.cent_a = op->cent_a.p;
  a.cent_v = op->cent_v.p;
  a.n_master = op->n_master;
  a.bdof_off = op->bdof_off.p;
  a.bm_ptr = op->bm_ptr.p;
  a.bm_ord = op->bm_ord.p;
  a.bm_w = op->bm_w.p;
  a.bm_loc = op->bm_loc.p;
  a.soff = op->soff.p;
  a.ibase = op->ibase.p;
  a.i_global = op->i_global.p;
  a.i_sign = op->i_sign.p;
  return a;
}

std::unique_ptr<hdr_alg_s> new_op(const hdr_alg_inputs* in, const std::vector<int64_t>& off, int kind) {
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    throw StatusError(HDR_CUDA_ERROR, "no CUDA device available (the hot path has no CPU fallback)");
  auto op = std::make_unique<hdr_alg_s>();
  op->kind = kind;
  CK(cudaStreamCreateWithFlags(&op->st, cudaStreamNonBlocking));
  op->ne = in->nblocks;
  op->n_hat = off.back();
  op->n_global = in->p_ncols;
  op->m = in->c_nrows;
  op->boff.upload(off);
  std::vector<int64_t> aoff(static_cast<size_t>(op->ne) + 1, 0);
  for (int64_t e = 0; e < op->ne; ++e) aoff[e + 1] = aoff[e] + in->block_sizes[e] * in->block_sizes[e];
  op->aoff.upload(aoff);
  op->blocks.upload(in->blocks, static_cast<size_t>(aoff.back()));
  op->status.alloc(1);
  CK(cudaMemset(op->status.p, 0, sizeof(int)));
  op->bad.alloc(1);
  CK(cudaMemset(op->bad.p, 0xff, sizeof(unsigned long long)));
  return op;
}

}  // namespace

extern "C" {

hdr_status hdr_alg_hybridize(const hdr_alg_inputs* in, hdr_alg_t* out) {
  if (!out) return fail(HDR_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  return catch_all([&]() -> hdr_status {
    const std::vector<int64_t> off = check_inputs(in, "hybridize");
    auto op = new_op(in, off, 0);
    cudaStream_t st = op->st;
    const int64_t ne = op->ne, n_hat = op->n_hat, m = op->m;
    // C^T structure: constrained columns (reduction.cpp:253-258) and rows per broken dof
    std::vector<int64_t> tro, trow, tpos;
    transpose_csr(in->c_nrows, in->c_ncols, in->c_row_offsets, in->c_col_indices, tro, trow, tpos);
    std::vector<int> idx(static_cast<size_t>(n_hat)), ni(static_cast<size_t>(ne));
    std::vector<int64_t> goff(static_cast<size_t>(ne) + 1, 0), hoff(static_cast<size_t>(ne) + 1, 0), mrows, cptr;
    std::vector<int> cent_r, cent_a;
    std::vector<double> cent_v;
    int dmax = 1, ncmax = 1;
    std::vector<int64_t> rows;
    std::vector<int> pos_of(1, -1);
    for (int64_t e = 0; e < ne; ++e) {
      const int64_t o = off[e];
      const int n = static_cast<int>(off[e + 1] - o);
      // partition_block with marker -1 (reduction.cpp:236-251): i = unconstrained columns
      int k = 0;
      for (int l = 0; l < n; ++l)
        if (tro[o + l + 1] == tro[o + l]) idx[o + k++] = l;
      ni[e] = k;
      for (int l = 0; l < n; ++l)
        if (tro[o + l + 1] != tro[o + l]) idx[o + k++] = l;
      // multiplier rows: sorted unique rows of C over the block's columns (constraint_slice)
      rows.clear();
      for (int l = 0; l < n; ++l)
        for (int64_t q = tro[o + l]; q < tro[o + l + 1]; ++q) rows.push_back(trow[q]);
      std::sort(rows.begin(), rows.end());
      rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
      const int nr = static_cast<int>(rows.size());
      // slice entries (r, position of b dof j, C value): first match in row r, as the reference's scan
      if (static_cast<int>(pos_of.size()) < n) pos_of.assign(static_cast<size_t>(n), -1);
      for (int p = ni[e]; p < n; ++p) pos_of[idx[o + p]] = p;
      for (int r = 0; r < nr; ++r) {
        cptr.push_back(static_cast<int64_t>(cent_v.size()));
        const int64_t row = rows[r];
        for (int p = ni[e]; p < n; ++p) {
          const int64_t target = o + idx[o + p];
          for (int64_t q = in->c_row_offsets[row]; q < in->c_row_offsets[row + 1]; ++q)
            if (in->c_col_indices[q] == target) {
              cent_r.push_back(r);
              cent_a.push_back(p);
              cent_v.push_back(in->c_values[q]);
              break;
            }
        }
        mrows.push_back(row);
      }
      goff[e + 1] = goff[e] + nr;
      hoff[e + 1] = hoff[e] + static_cast<int64_t>(nr) * nr;
      dmax = std::max(dmax, n);
      ncmax = std::max(ncmax, nr + 1);
    }
    cptr.push_back(static_cast<int64_t>(cent_v.size()));
    op->idx.upload(idx);
    op->ni.upload(ni);
    op->goff.upload(goff);
    op->hoff.upload(hoff);
    op->mrows.upload(mrows);
    op->cptr.upload(cptr);
    op->cent_r.upload(cent_r);
    op->cent_a.upload(cent_a);
    op->cent_v.upload(cent_v);
    finish_launch_config(op.get(), dmax, ncmax);
    DBuf<double> f, hbuf, gbuf;
    f.upload(in->f_hat, static_cast<size_t>(n_hat));
    hbuf.alloc(static_cast<size_t>(hoff.back()));
    gbuf.alloc(static_cast<size_t>(goff.back()));
    AlgArgs a = base_args(op.get());
    a.f = f.p;
    a.hbuf = hbuf.p;
    a.gbuf = gbuf.p;
    launch_alg(a, ALG_HYB, op->plan, op->gws.p, st);
    const hdr_status s = read_status(op.get(), "hybridize");
    if (s != HDR_OK) return s;

    // from_triplets: H pattern and sums; g accumulated in element order
    const int64_t T = hoff.back(), G = goff.back();
    DBuf<uint64_t> hkeys, gkeys;
    DBuf<int64_t> hsrc, gsrc;
    hkeys.alloc(T);
    hsrc.alloc(T);
    gkeys.alloc(G);
    gsrc.alloc(G);
    launch_alg_hkeys(a, hkeys.p, hsrc.p, gkeys.p, gsrc.p, st);
    DBuf<int64_t> row_cnt;
    row_cnt.alloc(static_cast<size_t>(m) + 1);
    CK(cudaMemsetAsync(row_cnt.p, 0, static_cast<size_t>(m + 1) * 8, st));
    Runs HR, GR;
    const uint64_t mm = m > 0 ? static_cast<uint64_t>(m) * static_cast<uint64_t>(m) : 1;
    sort_runs(T, hkeys, hsrc, nullptr, mm, m, &row_cnt, HR, st);
    op->nrows = m;
    op->nnz = HR.nruns;
    op->row_offsets.alloc(static_cast<size_t>(m) + 1);
    dev_scan(row_cnt.p, op->row_offsets.p, m + 1, st);
    op->col_indices.alloc(static_cast<size_t>(op->nnz));
    if (op->nnz) CK(cudaMemcpyAsync(op->col_indices.p, HR.index.p, static_cast<size_t>(op->nnz) * 8, cudaMemcpyDeviceToDevice, st));
    op->values.alloc(static_cast<size_t>(op->nnz));
    launch_run_sum(op->nnz, HR.start.p, HR.src.p, nullptr, hbuf.p, op->values.p, nullptr, 0, st);
    sort_runs(G, gkeys, gsrc, nullptr, static_cast<uint64_t>(m > 0 ? m : 1), m, nullptr, GR, st);
    op->rhs.alloc(static_cast<size_t>(m));
    CK(cudaMemsetAsync(op->rhs.p, 0, static_cast<size_t>(m) * 8, st));
    launch_run_sum(GR.nruns, GR.start.p, GR.src.p, nullptr, gbuf.p, op->rhs.p, GR.index.p, 1, st);

    // recovery_scale = 1 / diag(P^T P) and diagonal_gram (reduction.cpp:339-352)
    const int64_t ng = in->p_ncols;
    std::vector<int64_t> ptro, ptrow, ptpos;
    transpose_csr(in->p_nrows, ng, in->p_row_offsets, in->p_col_indices, ptro, ptrow, ptpos);
    std::vector<double> ptv(ptpos.size());
    for (size_t q = 0; q < ptpos.size(); ++q) ptv[q] = in->p_values[ptpos[q]];
    for (int64_t r = 0; r < in->p_nrows; ++r)
      if (in->p_row_offsets[r + 1] - in->p_row_offsets[r] > 1) op->diagonal_gram = false;
    op->pt_ro.upload(ptro);
    op->pt_ci.upload(ptrow);
    op->pt_v.upload(ptv);
    op->p_ro.upload(in->p_row_offsets, static_cast<size_t>(in->p_nrows) + 1);
    op->p_ci.upload(in->p_col_indices, static_cast<size_t>(in->p_row_offsets[in->p_nrows]));
    op->p_v.upload(in->p_values, static_cast<size_t>(in->p_row_offsets[in->p_nrows]));
    DBuf<double> sumsq;
    sumsq.alloc(static_cast<size_t>(ng));
    op->scale.alloc(static_cast<size_t>(ng));
    launch_row_sumsq(ng, op->pt_ro.p, op->pt_v.p, sumsq.p, st);
    std::vector<double> hs(static_cast<size_t>(ng));
    if (ng) CK(cudaMemcpyAsync(hs.data(), sumsq.p, static_cast<size_t>(ng) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < ng; ++i)
      if (hs[i] == 0.0) return fail(HDR_VALIDATION, "hybridize: P has an empty column (not full column rank)");
    launch_vec_op(ng, 3, 0.0, sumsq.p, nullptr, op->scale.p, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    *out = op.release();
    return HDR_OK;
  });
}

hdr_status hdr_alg_static_condense(const hdr_alg_inputs* in, hdr_alg_t* out) {
  if (!out) return fail(HDR_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  return catch_all([&]() -> hdr_status {
    const std::vector<int64_t> off = check_inputs(in, "static_condense");
    const int64_t marker = in->interior_global_begin;
    if (marker >= 0 && off.back() > 0 && !in->dof_global)
      return fail(HDR_INVALID_ARGUMENT, "static_condense: interior_global_begin >= 0 needs dof_global");
    auto op = new_op(in, off, 1);
    cudaStream_t st = op->st;
    const int64_t ne = op->ne, n_hat = op->n_hat, ng = in->p_ncols;
    const int64_t* pro = in->p_row_offsets;
    std::vector<int64_t> tro, trow, tpos;
    transpose_csr(in->c_nrows, in->c_ncols, in->c_row_offsets, in->c_col_indices, tro, trow, tpos);
    std::vector<int> idx(static_cast<size_t>(n_hat)), ni(static_cast<size_t>(ne));
    std::vector<int64_t> bdof_off(static_cast<size_t>(ne) + 1, 0), soff(static_cast<size_t>(ne) + 1, 0),
        ibase(static_cast<size_t>(ne) + 1, 0), i_global;
    std::vector<double> i_sign;
    std::vector<char> is_master(static_cast<size_t>(ng), 0);
    int dmax = 1, ncmax = 1;
    for (int64_t e = 0; e < ne; ++e) {
      const int64_t o = off[e];
      const int n = static_cast<int>(off[e + 1] - o);
      auto iface = [&](int l) {
        return marker >= 0 ? in->dof_global[o + l] < marker : tro[o + l + 1] != tro[o + l];
      };
      int k = 0;
      for (int l = 0; l < n; ++l)
        if (!iface(l)) idx[o + k++] = l;
      ni[e] = k;
      for (int l = 0; l < n; ++l)
        if (iface(l)) idx[o + k++] = l;
      const int nb = n - ni[e];
      for (int i = 0; i < ni[e]; ++i) {  // interior rows map one-to-one onto globals (reduction.cpp:496-506)
        const int64_t row = o + idx[o + i];
        if (pro[row + 1] - pro[row] != 1 || in->p_values[pro[row]] == 0.0)
          return fail(HDR_VALIDATION, "static_condense: interior broken dof " + std::to_string(row) +
                                          " does not map to a single global dof");
        i_global.push_back(in->p_col_indices[pro[row]]);
        i_sign.push_back(in->p_values[pro[row]]);
      }
      for (int j = 0; j < nb; ++j) {
        const int64_t row = o + idx[o + ni[e] + j];
        for (int64_t q = pro[row]; q < pro[row + 1]; ++q) is_master[in->p_col_indices[q]] = 1;
      }
      bdof_off[e + 1] = bdof_off[e] + nb;
      soff[e + 1] = soff[e] + static_cast<int64_t>(nb) * nb;
      ibase[e + 1] = ibase[e] + ni[e];
      dmax = std::max(dmax, ni[e]);
      ncmax = std::max(ncmax, nb + 1);
    }
    std::vector<int64_t> ordinal(static_cast<size_t>(ng), -1);
    for (int64_t g = 0; g < ng; ++g)
      if (is_master[g]) {
        ordinal[g] = static_cast<int64_t>(op->master_globals.size());
        op->master_globals.push_back(g);
      }
    op->n_master = static_cast<int64_t>(op->master_globals.size());
    // P-row entries of every b dof: (master ordinal, weight, local j)
    std::vector<int64_t> bm_ptr(1, 0), bm_ord, trip_off(static_cast<size_t>(ne) + 1, 0), ftrip_off(static_cast<size_t>(ne) + 1, 0);
    std::vector<double> bm_w;
    std::vector<int> bm_loc;
    for (int64_t e = 0; e < ne; ++e) {
      const int64_t o = off[e];
      const int nb = static_cast<int>(off[e + 1] - o) - ni[e];
      int64_t nent = 0;
      for (int j = 0; j < nb; ++j) {
        const int64_t row = o + idx[o + ni[e] + j];
        for (int64_t q = pro[row]; q < pro[row + 1]; ++q) {
          bm_ord.push_back(ordinal[in->p_col_indices[q]]);
          bm_w.push_back(in->p_values[q]);
          bm_loc.push_back(j);
          ++nent;
        }
        bm_ptr.push_back(static_cast<int64_t>(bm_ord.size()));
      }
      trip_off[e + 1] = trip_off[e] + nent * nent;
      ftrip_off[e + 1] = ftrip_off[e] + nent;
    }
    op->idx.upload(idx);
    op->ni.upload(ni);
    op->bdof_off.upload(bdof_off);
    op->soff.upload(soff);
    op->ibase.upload(ibase);
    op->i_global.upload(i_global);
    op->i_sign.upload(i_sign);
    op->bm_ptr.upload(bm_ptr);
    op->bm_ord.upload(bm_ord);
    op->bm_w.upload(bm_w);
    op->bm_loc.upload(bm_loc);
    op->masters.upload(op->master_globals);
    finish_launch_config(op.get(), dmax, ncmax);
    DBuf<double> f, sbuf, fsbuf;
    f.upload(in->f_hat, static_cast<size_t>(n_hat));
    sbuf.alloc(static_cast<size_t>(soff.back()));
    fsbuf.alloc(static_cast<size_t>(bdof_off.back()));
    AlgArgs a = base_args(op.get());
    a.f = f.p;
    a.sbuf = sbuf.p;
    a.fsbuf = fsbuf.p;
    launch_alg(a, ALG_COND, op->plan, op->gws.p, st);
    const hdr_status s = read_status(op.get(), "static_condense");
    if (s != HDR_OK) return s;

    // S = sum P_b^T S_hat P_b and f_S through from_triplets / ordered vector sums
    const int64_t T = trip_off.back(), F = ftrip_off.back(), nm = op->n_master;
    DBuf<int64_t> d_trip_off, d_ftrip_off, ssrc, fsrc;
    DBuf<uint64_t> skeys, fkeys;
    DBuf<double> sw, fw;
    d_trip_off.upload(trip_off);
    d_ftrip_off.upload(ftrip_off);
    skeys.alloc(T);
    ssrc.alloc(T);
    sw.alloc(T);
    fkeys.alloc(F);
    fsrc.alloc(F);
    fw.alloc(F);
    launch_alg_skeys(a, d_trip_off.p, d_ftrip_off.p, skeys.p, ssrc.p, sw.p, fkeys.p, fsrc.p, fw.p, st);
    DBuf<int64_t> row_cnt;
    row_cnt.alloc(static_cast<size_t>(nm) + 1);
    CK(cudaMemsetAsync(row_cnt.p, 0, static_cast<size_t>(nm + 1) * 8, st));
    Runs SR, FR;
    const uint64_t mm = nm > 0 ? static_cast<uint64_t>(nm) * static_cast<uint64_t>(nm) : 1;
    sort_runs(T, skeys, ssrc, &sw, mm, nm, &row_cnt, SR, st);
    op->nrows = nm;
    op->nnz = SR.nruns;
    op->row_offsets.alloc(static_cast<size_t>(nm) + 1);
    dev_scan(row_cnt.p, op->row_offsets.p, nm + 1, st);
    op->col_indices.alloc(static_cast<size_t>(op->nnz));
    if (op->nnz) CK(cudaMemcpyAsync(op->col_indices.p, SR.index.p, static_cast<size_t>(op->nnz) * 8, cudaMemcpyDeviceToDevice, st));
    op->values.alloc(static_cast<size_t>(op->nnz));
    launch_run_sum(op->nnz, SR.start.p, SR.src.p, SR.w.p, sbuf.p, op->values.p, nullptr, 0, st);
    sort_runs(F, fkeys, fsrc, &fw, static_cast<uint64_t>(nm > 0 ? nm : 1), nm, nullptr, FR, st);
    op->rhs.alloc(static_cast<size_t>(nm));
    CK(cudaMemsetAsync(op->rhs.p, 0, static_cast<size_t>(nm) * 8, st));
    launch_run_sum(FR.nruns, FR.start.p, FR.src.p, FR.w.p, fsbuf.p, op->rhs.p, FR.index.p, 1, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    *out = op.release();
    return HDR_OK;
  });
}

hdr_status hdr_alg_info(hdr_alg_t op, int64_t* o) {
  if (!op || !o) return fail(HDR_INVALID_ARGUMENT, "null argument");
  o[HDR_ALG_NROWS] = op->nrows;
  o[HDR_ALG_NNZ] = op->nnz;
  o[HDR_ALG_N_HAT] = op->n_hat;
  o[HDR_ALG_N_GLOBAL] = op->n_global;
  o[HDR_ALG_DIAGONAL_GRAM] = op->diagonal_gram ? 1 : 0;
  o[HDR_ALG_KIND] = op->kind;
  return HDR_OK;
}

hdr_status hdr_alg_matrix(hdr_alg_t op, int64_t* row_offsets, int64_t* col_indices, double* values, double* rhs) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = op->st;
    if (row_offsets)
      CK(cudaMemcpyAsync(row_offsets, op->row_offsets.p, static_cast<size_t>(op->nrows + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (col_indices && op->nnz)
      CK(cudaMemcpyAsync(col_indices, op->col_indices.p, static_cast<size_t>(op->nnz) * 8, cudaMemcpyDeviceToHost, st));
    if (values && op->nnz)
      CK(cudaMemcpyAsync(values, op->values.p, static_cast<size_t>(op->nnz) * 8, cudaMemcpyDeviceToHost, st));
    if (rhs && op->nrows) CK(cudaMemcpyAsync(rhs, op->rhs.p, static_cast<size_t>(op->nrows) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HDR_OK;
  });
}

hdr_status hdr_alg_master_globals(hdr_alg_t op, int64_t* out) {
  if (!op || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (op->kind != 1) return fail(HDR_INVALID_ARGUMENT, "master_globals: not a condensed operator");
  std::copy(op->master_globals.begin(), op->master_globals.end(), out);
  return HDR_OK;
}

hdr_status hdr_alg_recovery_scale(hdr_alg_t op, double* out) {
  if (!op || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (op->kind != 0) return fail(HDR_INVALID_ARGUMENT, "recovery_scale: not a hybridized operator");
  return catch_all([&]() -> hdr_status {
    if (op->n_global)
      CK(cudaMemcpyAsync(out, op->scale.p, static_cast<size_t>(op->n_global) * 8, cudaMemcpyDeviceToHost, op->st));
    CK(cudaStreamSynchronize(op->st));
    return HDR_OK;
  });
}

hdr_status hdr_alg_recover_hybrid(hdr_alg_t op, const double* lambda, int64_t lambda_len, const double* f_hat,
                                  int64_t f_len, double* x_hat, double* x) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  if (op->kind != 0) return fail(HDR_INVALID_ARGUMENT, "recover_hybrid: not a hybridized operator");
  if (f_len != op->n_hat) return fail(HDR_DIMENSION_MISMATCH, "recover_hybrid: f_hat length");
  if (lambda_len != op->nrows) return fail(HDR_DIMENSION_MISMATCH, "recover_hybrid: lambda length");
  if ((op->n_hat && !f_hat) || (op->nrows && !lambda)) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = op->st;
    const int64_t ng = op->n_global;
    DBuf<double> dl, df, dxh, dx;
    dl.upload(lambda, static_cast<size_t>(op->nrows));
    df.upload(f_hat, static_cast<size_t>(op->n_hat));
    dxh.alloc(static_cast<size_t>(op->n_hat));
    dx.alloc(static_cast<size_t>(ng));
    AlgArgs a = base_args(op);
    a.f = df.p;
    a.lambda = dl.p;
    a.x_hat = dxh.p;
    launch_alg(a, ALG_REC, op->plan, op->gws.p, st);
    const hdr_status s = read_status(op, "recover_hybrid");
    if (s != HDR_OK) return s;
    // x = (P^T P)^-1 P^T x_hat
    launch_spmv64(ng, op->pt_ro.p, op->pt_ci.p, op->pt_v.p, dxh.p, dx.p, st);
    if (op->diagonal_gram) {
      launch_vec_op(ng, 0, 0.0, dx.p, op->scale.p, dx.p, st);
    } else {
      // CG on the Gram matrix applied matrix-free as P^T (P z) (reduction.cpp:405-444)
      DBuf<double> z, res, prec, dir, pd, q, part, sc;
      z.alloc(ng);
      res.alloc(ng);
      prec.alloc(ng);
      dir.alloc(ng);
      q.alloc(ng);
      pd.alloc(static_cast<size_t>(op->n_hat));
      part.alloc(1024);
      sc.alloc(1);
      auto dot = [&](const double* u, const double* v) {
        launch_dot(ng, u, v, part.p, sc.p, st);
        double h = 0.0;
        CK(cudaMemcpyAsync(&h, sc.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return h;
      };
      CK(cudaMemsetAsync(z.p, 0, static_cast<size_t>(ng) * 8, st));
      CK(cudaMemcpyAsync(res.p, dx.p, static_cast<size_t>(ng) * 8, cudaMemcpyDeviceToDevice, st));
      launch_vec_op(ng, 0, 0.0, op->scale.p, res.p, prec.p, st);
      CK(cudaMemcpyAsync(dir.p, prec.p, static_cast<size_t>(ng) * 8, cudaMemcpyDeviceToDevice, st));
      double rz = dot(res.p, prec.p);
      const double rhs_norm = dot(dx.p, dx.p);
      for (int it = 0; it < 200 && rz > 0.0; ++it) {
        launch_spmv64(op->n_hat, op->p_ro.p, op->p_ci.p, op->p_v.p, dir.p, pd.p, st);
        launch_spmv64(ng, op->pt_ro.p, op->pt_ci.p, op->pt_v.p, pd.p, q.p, st);
        const double dq = dot(dir.p, q.p);
        if (dq <= 0.0) break;
        const double alpha = rz / dq;
        launch_vec_op(ng, 1, alpha, dir.p, nullptr, z.p, st);
        launch_vec_op(ng, 1, -alpha, q.p, nullptr, res.p, st);
        const double res_norm = dot(res.p, res.p);
        if (res_norm <= 1e-28 * rhs_norm) break;
        launch_vec_op(ng, 0, 0.0, op->scale.p, res.p, prec.p, st);
        const double rz_new = dot(res.p, prec.p);
        const double beta = rz_new / rz;
        launch_vec_op(ng, 2, beta, prec.p, nullptr, dir.p, st);
        rz = rz_new;
      }
      CK(cudaMemcpyAsync(dx.p, z.p, static_cast<size_t>(ng) * 8, cudaMemcpyDeviceToDevice, st));
    }
    if (x_hat && op->n_hat)
      CK(cudaMemcpyAsync(x_hat, dxh.p, static_cast<size_t>(op->n_hat) * 8, cudaMemcpyDeviceToHost, st));
    if (x && ng) CK(cudaMemcpyAsync(x, dx.p, static_cast<size_t>(ng) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return HDR_OK;
  });
}

hdr_status hdr_alg_recover_condensed(hdr_alg_t op, const double* x_b, int64_t xb_len, const double* f_hat,
                                     int64_t f_len, double* x) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  if (op->kind != 1) return fail(HDR_INVALID_ARGUMENT, "recover_condensed: not a condensed operator");
  if (xb_len != op->nrows) return fail(HDR_DIMENSION_MISMATCH, "recover_condensed: x_b length");
  if (f_len != op->n_hat) return fail(HDR_DIMENSION_MISMATCH, "recover_condensed: f_hat length");
  if ((op->nrows && !x_b) || (op->n_hat && !f_hat) || !x) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = op->st;
    const int64_t ng = op->n_global;
    DBuf<double> dxb, df, dx;
    dxb.upload(x_b, static_cast<size_t>(op->nrows));
    df.upload(f_hat, static_cast<size_t>(op->n_hat));
    dx.alloc(static_cast<size_t>(ng));
    CK(cudaMemsetAsync(dx.p, 0, static_cast<size_t>(ng) * 8, st));
    launch_scatter(op->nrows, op->masters.p, dxb.p, dx.p, st);
    AlgArgs a = base_args(op);
    a.f = df.p;
    a.xb = dxb.p;
    a.x = dx.p;
    launch_alg(a, ALG_RECC, op->plan, op->gws.p, st);
    const hdr_status s = read_status(op, "recover_condensed");
    if (s != HDR_OK) return s;
    if (ng) CK(cudaMemcpyAsync(x, dx.p, static_cast<size_t>(ng) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HDR_OK;
  });
}

void hdr_alg_destroy(hdr_alg_t op) { delete op; }

hdr_status hdr_alg_pcg(hdr_alg_t op, const double* b, double* x, int on_device, double rtol, int64_t maxit,
                       int precond, double* hist, hdr_pcg_report* rep) {
  if (!op || !x) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    const int64_t n = op->nrows;
    DBuf<double> db, dx;
    const double* pb = b ? b : op->rhs.p;
    if (b && !on_device) {
      db.upload(b, static_cast<size_t>(n));
      pb = db.p;
    }
    double* px = x;
    if (!on_device) {
      dx.alloc(static_cast<size_t>(n));
      px = dx.p;
    }
    const hdr_status s = pcg_device(n, op->row_offsets.p, nullptr, op->col_indices.p, op->values.p, pb, px, rtol, maxit,
                                    precond, hist, rep, op->st);
    if (s != HDR_OK) return s;
    if (!on_device && n) CK(cudaMemcpy(x, px, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}

hdr_status hdr_alg_symmetrize(hdr_alg_t op) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status {
    launch_csr_symmetrize64(op->nrows, op->row_offsets.p, op->col_indices.p, op->values.p, op->st);
    CK(cudaStreamSynchronize(op->st));
    CK(cudaGetLastError());
    return HDR_OK;
  });
}

}  // extern "C"
