// C ABI (include/hdivred_b200.h): handles, device memory, orchestration.
//
// There is no CPU compute path behind these entry points: every per-cell
// operation runs in the kernels of kern_*.cu; the host only builds the
// reference element once per space (rt_reference.cpp), its fixed factors
// (structured.cpp) and launches.  Without a CUDA device every compute entry
// point returns HDR_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/hdivred_b200.h"
#include "capi_util.hpp"
#include "geom.hpp"
#include "hdr_internal.hpp"
#include "kernels.hpp"

namespace hdr {

static std::atomic<int64_t> g_launches{0};
void count_launch(int64_t k) { g_launches += k; }

std::string& last_error_ref() {
  thread_local std::string s;
  return s;
}

}  // namespace hdr

using namespace hdr;

struct hdr_space_s {
  int dim = 3, k = 0, n = 0, dpf = 1, nint = 0, nF = 0, r = 0;
  int64_t N[3] = {1, 1, 1};
  double h[3] = {1, 1, 1};
  int weighted = 0;
  int64_t ncells = 0, nfaces = 0, ndofs = 0, fdc = 0, broken = 0, m = 0, nnz_h = 0, ns = 0, nnz_s = 0;
  RefElement re;
  Structured st;
  DevMesh dm{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // device data
  DBuf<int> mbase;
  DBuf<int64_t> row_h, row_s;
  DBuf<int32_t> col_h, col_s;
  DBuf<double> fixed;  // D, M, E, Ma, N0 (n*n each), X (n*r), lam (r)
  std::vector<double> rt0_consts;  // packed constant block of the k = 0 kernel
  DBuf<uint64_t> rank_tab;         // k = 0 row-rank table
  DBuf<longlong2> frs;             // per-face {row start, row} (k = 0 kernels, warp kernels)
  DBuf<double> premat;             // k >= 2 (3D): [N0 ; X^T] column-major ((n + r) x n)
  DBuf<double> dtab;               // k >= 2 (3D): {D, M} in the tensor-core chunk order
  DBuf<float> etab;                // k >= 2 (3D): {E, Ma} (fp32) likewise
  DBuf<double> tdm;                // warp-kernel spaces: {D, M} transposed ((i, l) at l * n + i)
  DBuf<float> tem;                 // warp-kernel spaces: {E, Ma} (fp32) transposed
  DBuf<int> tix;                   // warp-kernel spaces: (l << 16) | i of each table entry
  Fixed fx{};
  GeomState* geom = nullptr;  // mapped (trilinear) cells: hdr_space_set_vertices
  struct BatchCtx* batch = nullptr;  // hdr_hybridize_fe_batch: streams, events, two operators
  // fail-safe of the structured solve (hdr_device.cuh struct_order, kern_exact.cu)
  DBuf<double> xws;            // exact-path scratch (exact_grid x exact_ws_doubles), on first use
  double eps32 = 0, eps_tc = 1e-6;
  int force_exact = 0;
  float* qlog = nullptr;
  ~hdr_space_s();
};

struct hdr_hybrid_s {
  hdr_space_t sp = nullptr;
  DBuf<double> hval, g, alpha, beta, f, ws, pre;
  DBuf<int> status;
  // cells sent to the exact path: xcount = [count (k >= 1: list length), -,
  // k = 0 brick kernels' list length, k = 0 recovery count]
  DBuf<int> xlist, xcount;
  int last_call = 0;  // 0: hybridize, 1: recover (which count exact_cells reports)
  DBuf<unsigned long long> xbad;  // smallest singular cell of the exact path
  int64_t ws_doubles = 0;
  const double* a_ptr = nullptr;  // coefficients used by the last hybridize (owned copy or borrowed device input)
  const double* b_ptr = nullptr;
};

// pipelined batch (hdr_hybridize_fe_batch): uploads on cs, kernels on the space's
// stream, downloads on ds; two operators alternate (double-buffered inputs and
// H values)
struct BatchCtx {
  cudaStream_t cs = nullptr, ds = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  hdr_hybrid_s op[2];
  ~BatchCtx() {
    for (int b = 0; b < 2; ++b) {
      if (ev_in[b]) cudaEventDestroy(ev_in[b]);
      if (ev_comp[b]) cudaEventDestroy(ev_comp[b]);
      if (ev_d2h[b]) cudaEventDestroy(ev_d2h[b]);
    }
    if (cs) cudaStreamDestroy(cs);
    if (ds) cudaStreamDestroy(ds);
  }
};

hdr_space_s::~hdr_space_s() {
  delete batch;
  if (geom) geom_destroy(geom);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

struct hdr_condensed_s {
  hdr_space_t sp = nullptr;
  DBuf<double> sval, fs, alpha, beta, f, ws;
  DBuf<int> status;
  int64_t ws_doubles = 0;
  const double* a_ptr = nullptr;
  const double* b_ptr = nullptr;
};

namespace {

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

template <class T>
void exclusive_scan(const T* in, T* out, int64_t count, cudaStream_t st) {
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int>(count), st));
  DBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, static_cast<int>(count), st));
  CK(cudaStreamSynchronize(st));
}

// copies host (on_device = 0) or device data into an owned device buffer
void stage(DBuf<double>& dst, const double* src, int64_t count, int on_device, cudaStream_t st) {
  if (dst.n < static_cast<size_t>(count) || !dst.p) dst.alloc(static_cast<size_t>(count));
  if (count == 0) return;
  CK(cudaMemcpyAsync(dst.p, src, static_cast<size_t>(count) * 8,
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
}

// Synchronizes the stream and reports (then clears) the sticky device status.
hdr_status check_status(int* d_status, cudaStream_t st, unsigned long long* d_bad = nullptr) {
  int status = 0;
  unsigned long long bad = ~0ull;
  CK(cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (d_bad) CK(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (status) CK(cudaMemsetAsync(d_status, 0, sizeof(int), st));
  if (d_bad && bad != ~0ull) CK(cudaMemsetAsync(d_bad, 0xff, sizeof(bad), st));
  if (status & 4)
    return fail(HDR_SINGULAR_BLOCK, "SingularBlock: element " + (bad != ~0ull ? std::to_string(bad) : std::string("?")) +
                                        " (pivot <= 1e-14 max|block| of A_ii or S_b)");
  if (status & 1) return fail(HDR_UNSUPPORTED, "structured element solve: unsupported input");
  return HDR_OK;
}

// exact-path bookkeeping of an operator (list capacity = cells) and the space's scratch
void exact_prepare(hdr_space_t sp, hdr_hybrid_s* op, cudaStream_t st) {
  if (!op->xlist.p) op->xlist.alloc(static_cast<size_t>(std::max<int64_t>(sp->ncells, 1)));
  if (!op->xcount.p) {
    op->xcount.alloc(4);
    CK(cudaMemsetAsync(op->xcount.p, 0, 4 * sizeof(int), st));
    op->xbad.alloc(1);
    CK(cudaMemsetAsync(op->xbad.p, 0xff, sizeof(unsigned long long), st));
  }
  if (sp->k > 0 && !sp->xws.p)
    sp->xws.alloc(static_cast<size_t>(exact_grid(sp->n)) * static_cast<size_t>(exact_ws_doubles(sp->n, 0)));
}

ExactArgs exact_args(hdr_space_t sp, hdr_hybrid_s* op, int mode, const double* a, const double* b, const double* f) {
  ExactArgs X{};
  X.m = sp->dm;
  X.n = sp->n;
  X.nF = sp->nF;
  X.mode = mode;
  X.D = sp->fx.D;
  X.M = sp->fx.M;
  X.alpha = a;
  X.beta = b;
  X.f = f;
  X.mbase = sp->mbase.p;
  X.rowoff = sp->row_h.p;
  X.hval = op->hval.p;
  X.g = op->g.p;
  X.xlist = op->xlist.p;
  X.xcount = op->xcount.p;
  X.status = op->status.p;
  X.bad = op->xbad.p;
  return X;
}

// Relative accuracy assumed for the correction terms in the acceptance test
// (struct_order): fp32 products of fp32-rounded operands accumulated over n terms
// in two chained GEMMs, in the probabilistic rounding-error model
// sqrt(2n) * 2^-24; the tcgen05 3xTF32 form (fp32 accumulation in TMEM,
// k_hyb_big) measured at ~1e-6 of |C|.
double default_eps32(int n) { return std::sqrt(2.0 * n) * 0x1p-24; }
constexpr double kDefaultEpsTc = 1e-6;

}  // namespace

extern "C" {

const char* hdr_last_error(void) { return last_error_ref().c_str(); }
const char* hdr_version(void) { return "hdivred_b200 0.1.0 sm_100a"; }
int64_t hdr_launch_count(void) { return g_launches.load(); }

hdr_status hdr_reference_element(int dim, int order, const double h[3], double* divdiv, double* mass,
                                 double* face_moments, double* unit_load) {
  if (dim != 2 && dim != 3) return fail(HDR_INVALID_ARGUMENT, "dim must be 2 or 3");
  if (order < 0 || order > 3) return fail(HDR_INVALID_ARGUMENT, "order must be in 0..3");
  return catch_all([&]() -> hdr_status {
    const double hh[3] = {h ? h[0] : 1.0, h ? h[1] : 1.0, (h && dim == 3) ? h[2] : 1.0};
    const RefElement re = build_reference_element(dim, order, hh);
    if (divdiv) std::memcpy(divdiv, re.divdiv.data(), re.divdiv.size() * 8);
    if (mass) std::memcpy(mass, re.mass.data(), re.mass.size() * 8);
    if (face_moments) std::memcpy(face_moments, re.face_moments.data(), re.face_moments.size() * 8);
    if (unit_load) std::memcpy(unit_load, re.unit_load.data(), re.unit_load.size() * 8);
    return HDR_OK;
  });
}

hdr_status hdr_reference_div_form(int dim, int order, const double h[3], double* div_form) {
  if (dim != 2 && dim != 3) return fail(HDR_INVALID_ARGUMENT, "dim must be 2 or 3");
  if (order < 0 || order > 3) return fail(HDR_INVALID_ARGUMENT, "order must be in 0..3");
  if (!div_form) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    const double hh[3] = {h ? h[0] : 1.0, h ? h[1] : 1.0, (h && dim == 3) ? h[2] : 1.0};
    const RefElement re = build_reference_element(dim, order, hh);
    std::memcpy(div_form, re.div_form.data(), re.div_form.size() * 8);
    return HDR_OK;
  });
}

hdr_status hdr_structured_factors(int dim, int order, const double h[3], double* X, double* lambda, double* E,
                                  double* N0, double* Ma, double* diag, int64_t* rank) {
  if (dim != 2 && dim != 3) return fail(HDR_INVALID_ARGUMENT, "dim must be 2 or 3");
  if (order < 0 || order > 3) return fail(HDR_INVALID_ARGUMENT, "order must be in 0..3");
  return catch_all([&]() -> hdr_status {
    const double hh[3] = {h ? h[0] : 1.0, h ? h[1] : 1.0, (h && dim == 3) ? h[2] : 1.0};
    const RefElement re = build_reference_element(dim, order, hh);
    Structured st;
    std::string err;
    if (!precompute_structured(re, static_cast<int>(ipow(order + 1, dim)), &st, &err)) return fail(HDR_UNSUPPORTED, err);
    if (X) std::memcpy(X, st.X.data(), st.X.size() * 8);
    if (lambda) std::memcpy(lambda, st.lambda.data(), st.lambda.size() * 8);
    if (E) std::memcpy(E, st.E.data(), st.E.size() * 8);
    if (N0) std::memcpy(N0, st.N0.data(), st.N0.size() * 8);
    if (Ma) std::memcpy(Ma, st.Ma.data(), st.Ma.size() * 8);
    if (diag) {
      diag[0] = st.rho;
      diag[1] = st.e_rel;
      diag[2] = st.orth;
      diag[3] = st.block_diag ? 1.0 : 0.0;
    }
    if (rank) *rank = st.r;
    return HDR_OK;
  });
}

hdr_status hdr_space_create(int dim, const int64_t cells[3], const double h[3], int order, const double* ref_divdiv,
                            const double* ref_mass, int weighted, const double* ref_face_moments, hdr_space_t* out) {
  if (!out || !cells) return fail(HDR_INVALID_ARGUMENT, "hdr_space_create: null argument");
  *out = nullptr;
  if (dim != 2 && dim != 3) return fail(HDR_INVALID_ARGUMENT, "build_mesh: dim must be 2 or 3");
  if (order < 0 || order > 3) return fail(HDR_INVALID_ARGUMENT, "build_space: order must be in 0..3");
  for (int a = 0; a < dim; ++a) {
    if (cells[a] < 1) return fail(HDR_INVALID_ARGUMENT, "build_mesh: cell counts must be >= 1");
    if (h && !(h[a] > 0.0)) return fail(HDR_INVALID_ARGUMENT, "build_mesh: cell sizes must be > 0");
  }
  (void)ref_face_moments;
  return catch_all([&]() -> hdr_status {
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
      return fail(HDR_CUDA_ERROR, "no CUDA device available (the hot path has no CPU fallback)");
    auto sp = std::make_unique<hdr_space_s>();
    sp->dim = dim;
    sp->k = order;
    sp->weighted = weighted ? 1 : 0;
    for (int a = 0; a < 3; ++a) {
      sp->N[a] = a < dim ? cells[a] : 1;
      sp->h[a] = a < dim ? (h ? h[a] : 1.0 / static_cast<double>(cells[a])) : 1.0;
    }
    sp->re = build_reference_element(dim, order, sp->h);
    const int n = sp->re.n;
    if (ref_divdiv) sp->re.divdiv.assign(ref_divdiv, ref_divdiv + static_cast<size_t>(n) * n);
    if (ref_mass) sp->re.mass.assign(ref_mass, ref_mass + static_cast<size_t>(n) * n);
    sp->n = n;
    sp->dpf = sp->re.dpf;
    sp->nint = sp->re.nint;
    sp->nF = 2 * dim * sp->dpf;
    std::string err;
    if (!precompute_structured(sp->re, static_cast<int>(ipow(order + 1, dim)), &sp->st, &err))
      return fail(HDR_UNSUPPORTED, err);
    sp->r = sp->st.r;
    sp->eps32 = default_eps32(n);
    sp->eps_tc = kDefaultEpsTc;

    // mesh numbering
    DevMesh& m = sp->dm;
    m.dim = dim;
    m.dpf = sp->dpf;
    m.n = n;
    m.nint = sp->nint;
    for (int a = 0; a < 3; ++a) m.N[a] = sp->N[a];
    int64_t off = 0;
    for (int a = 0; a < 3; ++a) {
      m.foff[a] = off;
      if (a < dim) {
        int64_t cnt = sp->N[a] + 1;
        for (int b = 0; b < dim; ++b)
          if (b != a) cnt *= sp->N[b];
        off += cnt;
      }
    }
    m.nfaces = off;
    m.ncells = sp->N[0] * sp->N[1] * sp->N[2];
    m.div_half = FastDiv(static_cast<uint32_t>((sp->N[0] + 1) / 2));
    m.div_n0 = FastDiv(static_cast<uint32_t>(sp->N[0]));
    m.div_n1 = FastDiv(static_cast<uint32_t>(sp->N[1]));
    m.face_dof_count = m.nfaces * sp->dpf;
    sp->ncells = m.ncells;
    sp->nfaces = m.nfaces;
    sp->fdc = m.face_dof_count;
    sp->ndofs = sp->fdc + sp->ncells * sp->nint;
    sp->broken = sp->ncells * n;
    sp->m = sp->broken - sp->ndofs;
    sp->ns = sp->fdc;

    CK(cudaStreamCreateWithFlags(&sp->stream, cudaStreamNonBlocking));
    sp->own_stream = true;
    cudaStream_t st = sp->stream;

    // K1: patterns
    const int64_t nf = m.nfaces;
    DBuf<int> flag, ord;
    DBuf<int64_t> fnnz_h, fnnz_s, fbase_h, fbase_s;
    flag.alloc(nf + 1);
    ord.alloc(nf + 1);
    fnnz_h.alloc(nf + 1);
    fnnz_s.alloc(nf + 1);
    fbase_h.alloc(nf + 1);
    fbase_s.alloc(nf + 1);
    sp->mbase.alloc(nf);
    launch_face_counts(m, flag.p, fnnz_h.p, fnnz_s.p, st);
    CK(cudaMemsetAsync(flag.p + nf, 0, sizeof(int), st));
    CK(cudaMemsetAsync(fnnz_h.p + nf, 0, sizeof(int64_t), st));
    CK(cudaMemsetAsync(fnnz_s.p + nf, 0, sizeof(int64_t), st));
    exclusive_scan(flag.p, ord.p, nf + 1, st);
    exclusive_scan(fnnz_h.p, fbase_h.p, nf + 1, st);
    exclusive_scan(fnnz_s.p, fbase_s.p, nf + 1, st);
    int n_int_faces = 0;
    CK(cudaMemcpy(&n_int_faces, ord.p + nf, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&sp->nnz_h, fbase_h.p + nf, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&sp->nnz_s, fbase_s.p + nf, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (static_cast<int64_t>(n_int_faces) * sp->dpf != sp->m)
      return fail(HDR_VALIDATION, "multiplier count mismatch (m != n_hat - n)");
    if (sp->nnz_h >= (int64_t(1) << 31) || sp->nnz_s >= (int64_t(1) << 31) || sp->fdc >= (int64_t(1) << 31))
      return fail(HDR_UNSUPPORTED, "mesh too large for int32 device column indices");
    launch_mbase(m, flag.p, ord.p, sp->mbase.p, st);
    sp->row_h.alloc(sp->m + 1);
    sp->col_h.alloc(sp->nnz_h);
    sp->row_s.alloc(sp->ns + 1);
    sp->col_s.alloc(sp->nnz_s);
    launch_fill_patterns(m, sp->mbase.p, fbase_h.p, fbase_s.p, sp->row_h.p, sp->col_h.p, sp->row_s.p, sp->col_s.p,
                         sp->m, sp->nnz_h, sp->ns, sp->nnz_s, st);

    // fixed factors
    const int r = sp->r;
    const size_t nn = static_cast<size_t>(n) * n;
    std::vector<double> pack(5 * nn + static_cast<size_t>(n) * r + r);
    std::memcpy(pack.data(), sp->re.divdiv.data(), nn * 8);
    std::memcpy(pack.data() + nn, sp->re.mass.data(), nn * 8);
    std::memcpy(pack.data() + 2 * nn, sp->st.E.data(), nn * 8);
    std::memcpy(pack.data() + 3 * nn, sp->st.Ma.data(), nn * 8);
    std::memcpy(pack.data() + 4 * nn, sp->st.N0.data(), nn * 8);
    std::memcpy(pack.data() + 5 * nn, sp->st.X.data(), static_cast<size_t>(n) * r * 8);
    std::memcpy(pack.data() + 5 * nn + static_cast<size_t>(n) * r, sp->st.lambda.data(), static_cast<size_t>(r) * 8);
    sp->fixed.alloc(pack.size());
    CK(cudaMemcpyAsync(sp->fixed.p, pack.data(), pack.size() * 8, cudaMemcpyHostToDevice, st));
    Fixed& fx = sp->fx;
    fx.D = sp->fixed.p;
    fx.M = fx.D + nn;
    fx.E = fx.M + nn;
    fx.Ma = fx.E + nn;
    fx.N0 = fx.Ma + nn;
    fx.X = fx.N0 + nn;
    fx.lam = fx.X + static_cast<size_t>(n) * r;
    fx.r = r;
    fx.rho = sp->st.rho;
    if (dim == 3 && order >= 1) {  // [N0 ; X^T] of the batched pre-GEMM (RT1..RT3 hexes)
      const int npr = n + r;
      std::vector<double> pm(static_cast<size_t>(npr) * n);
      for (int l = 0; l < n; ++l)
        for (int row = 0; row < npr; ++row)
          pm[static_cast<size_t>(l) * npr + row] =
              row < n ? sp->st.N0[static_cast<size_t>(row) * n + l] : sp->st.X[static_cast<size_t>(l) * r + (row - n)];
      sp->premat.alloc(pm.size());
      CK(cudaMemcpyAsync(sp->premat.p, pm.data(), pm.size() * 8, cudaMemcpyHostToDevice, st));
    }
    if (dim == 3 && order >= 2) {
      // chunk-ordered Delta tables of the tensor-core correction (kern_cta.cu)
      // entry order = the kernel's (chunk, iteration i, thread) order, thread
      // (warp w, lane l) -> row 8 (g / 4) + l / 4, column 16 c + 4 (g % 4) + l % 4, g = w + 16 i
      const int MP = (n + 127) / 128 * 128, KC = 16, nch = (n + 15) / 16, per = MP * KC / 512;
      std::vector<double> dt(static_cast<size_t>(nch) * MP * KC * 2, 0.0);
      std::vector<float> et(static_cast<size_t>(nch) * MP * KC * 2, 0.0f);
      for (int c = 0; c < nch; ++c)
        for (int i = 0; i < per; ++i)
          for (int tid = 0; tid < 512; ++tid) {
            const int g = tid / 32 + 16 * i, lane = tid % 32;
            const int mrow = 8 * (g / 4) + lane / 4, col = c * KC + 4 * (g % 4) + lane % 4;
            if (mrow >= n || col >= n) continue;
            const size_t q = (static_cast<size_t>(c) * per + i) * 512 + tid, o = static_cast<size_t>(mrow) * n + col;
            dt[2 * q] = sp->re.divdiv[o];
            dt[2 * q + 1] = sp->re.mass[o];
            et[2 * q] = static_cast<float>(sp->st.E[o]);
            et[2 * q + 1] = static_cast<float>(sp->st.Ma[o]);
          }
      sp->dtab.alloc(dt.size());
      sp->etab.alloc(et.size());
      CK(cudaMemcpyAsync(sp->dtab.p, dt.data(), dt.size() * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(sp->etab.p, et.data(), et.size() * 4, cudaMemcpyHostToDevice, st));
      fx.dtab = reinterpret_cast<const double2*>(sp->dtab.p);
      fx.etab = reinterpret_cast<const float2*>(sp->etab.p);
      CK(cudaStreamSynchronize(st));
    }
    if ((dim == 3 && order == 1) || (dim == 2 && order >= 1)) {  // transposed Delta inputs (kern_warp.cu)
      std::vector<double> td;
      std::vector<float> te;
      std::vector<int> tx;
      auto section = [&](bool zero_mass) {
        const size_t start = tx.size();
        for (int l = 0; l < n; ++l)
          for (int i = 0; i < n; ++i) {
            const size_t o = static_cast<size_t>(i) * n + l;
            const float ma = static_cast<float>(sp->st.Ma[o]);
            if ((sp->re.mass[o] == 0.0 && ma == 0.f) != zero_mass) continue;
            td.push_back(sp->re.divdiv[o]);
            td.push_back(sp->re.mass[o]);
            te.push_back(static_cast<float>(sp->st.E[o]));
            te.push_back(ma);
            tx.push_back((l << 16) | i);
          }
        while (tx.size() > start && tx.size() % 128 != 0) {  // benign duplicates of the last entry
          const size_t q = tx.size() - 1;
          td.push_back(td[2 * q]);
          td.push_back(td[2 * q + 1]);
          te.push_back(te[2 * q]);
          te.push_back(te[2 * q + 1]);
          tx.push_back(tx[q]);
        }
      };
      section(true);
      fx.tz = static_cast<int>(tx.size());
      section(false);
      fx.tn = static_cast<int>(tx.size());
      sp->tdm.upload(td);
      sp->tem.upload(te);
      sp->tix.upload(tx);
      fx.tdm = reinterpret_cast<const double2*>(sp->tdm.p);
      fx.tem = reinterpret_cast<const float2*>(sp->tem.p);
      fx.tix = sp->tix.p;
    }
    if (order == 0) {  // constant block for the register kernel: D, M, E, Ma, N0, X, lam, rho
      sp->rt0_consts.assign(pack.begin(), pack.begin() + 5 * nn + n + 1);
      sp->rt0_consts.push_back(sp->st.rho);
      sp->rt0_consts.insert(sp->rt0_consts.end(), sp->st.Minv.begin(), sp->st.Minv.end());  // for Rt0Fast
      const std::vector<uint64_t> tab = rank_table_rt0(dim);
      sp->rank_tab.alloc(tab.size());
      CK(cudaMemcpyAsync(sp->rank_tab.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, st));
    }
    {  // per-face {row start, row}: the k = 0 kernels and the warp kernels reach a row with one load
      sp->frs.alloc(static_cast<size_t>(sp->nfaces));
      launch_face_rows(sp->nfaces, sp->mbase.p, sp->row_h.p, sp->frs.p, st);
    }
    if (sp->weighted) {  // weighted constraint rows: the per-cell elimination path (geom.cu, affine cells)
      std::vector<int> mb(static_cast<size_t>(sp->nfaces));
      CK(cudaMemcpy(mb.data(), sp->mbase.p, mb.size() * sizeof(int), cudaMemcpyDeviceToHost));
      sp->geom = geom_create(sp->re, sp->dm, mb, sp->h, sp->m, sp->ndofs, nullptr, true, st);
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    *out = sp.release();
    return HDR_OK;
  });
}

void hdr_space_destroy(hdr_space_t sp) { delete sp; }

hdr_status hdr_space_set_vertices(hdr_space_t sp, const double* vertices) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  return catch_all([&]() -> hdr_status {
    CK(cudaStreamSynchronize(sp->stream));
    if (sp->geom) {
      geom_destroy(sp->geom);
      sp->geom = nullptr;
    }
    if (!vertices && !sp->weighted) return HDR_OK;
    if (vertices && sp->dim != 3) return fail(HDR_UNSUPPORTED, "mapped geometry: 3D spaces only");
    std::vector<int> mb(static_cast<size_t>(sp->nfaces));
    CK(cudaMemcpy(mb.data(), sp->mbase.p, mb.size() * sizeof(int), cudaMemcpyDeviceToHost));
    sp->geom = geom_create(sp->re, sp->dm, mb, sp->h, sp->m, sp->ndofs, vertices, sp->weighted != 0, sp->stream);
    if (geom_nnz_h(sp->geom) != sp->nnz_h) {
      geom_destroy(sp->geom);
      sp->geom = nullptr;
      return fail(HDR_VALIDATION, "mapped geometry: H pattern mismatch");
    }
    return HDR_OK;
  });
}

hdr_status hdr_space_element_matrices(hdr_space_t sp, double* out) {
  if (!sp || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (!sp->geom || !geom_element_blocks(sp->geom))
    return fail(HDR_INVALID_ARGUMENT, "element matrices: no mapped geometry hybridized / condensed yet");
  return catch_all([&]() -> hdr_status {
    CK(cudaStreamSynchronize(sp->stream));
    CK(cudaMemcpy(out, geom_element_blocks(sp->geom), static_cast<size_t>(sp->ncells) * sp->n * sp->n * 8,
                  cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}

hdr_status hdr_space_element_blocks(hdr_space_t sp, const double* alpha, const double* beta, int on_device,
                                    double* out) {
  if (!sp || !alpha || !beta || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    DBuf<double> da, db, dout;
    const double *pa = alpha, *pb = beta;
    if (!on_device) {
      stage(da, alpha, sp->ncells, 0, st);
      stage(db, beta, sp->ncells, 0, st);
      pa = da.p;
      pb = db.p;
    }
    const size_t cnt = static_cast<size_t>(sp->ncells) * sp->n * sp->n;
    if (sp->geom) {
      geom_assemble_blocks(sp->geom, pa, pb, st);
      CK(cudaMemcpyAsync(out, geom_element_blocks(sp->geom), cnt * 8,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    } else {
      double* po = out;
      if (!on_device) {
        dout.alloc(cnt);
        po = dout.p;
      }
      launch_affine_assemble(sp->ncells, sp->n, sp->fixed.p, pa, pb, po, st);  // fixed = [D | M | ...]
      if (!on_device) CK(cudaMemcpyAsync(out, po, cnt * 8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return HDR_OK;
  });
}

hdr_status hdr_space_info(hdr_space_t sp, int64_t* o) {
  if (!sp || !o) return fail(HDR_INVALID_ARGUMENT, "null argument");
  o[HDR_INFO_DIM] = sp->dim;
  o[HDR_INFO_ORDER] = sp->k;
  o[HDR_INFO_NCELLS] = sp->ncells;
  o[HDR_INFO_NFACES] = sp->nfaces;
  o[HDR_INFO_NDOFS] = sp->ndofs;
  o[HDR_INFO_BROKEN_NDOFS] = sp->broken;
  o[HDR_INFO_ELEMENT_NDOFS] = sp->n;
  o[HDR_INFO_DOFS_PER_FACE] = sp->dpf;
  o[HDR_INFO_INTERIOR_DOFS] = sp->nint;
  o[HDR_INFO_FACE_DOF_COUNT] = sp->fdc;
  o[HDR_INFO_M] = sp->m;
  o[HDR_INFO_NNZ_H] = sp->nnz_h;
  o[HDR_INFO_NS] = sp->ns;
  o[HDR_INFO_NNZ_S] = sp->nnz_s;
  o[HDR_INFO_DIV_RANK] = sp->r;
  return HDR_OK;
}

hdr_status hdr_space_reference(hdr_space_t sp, double* dd, double* mm) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  if (dd) std::memcpy(dd, sp->re.divdiv.data(), sp->re.divdiv.size() * 8);
  if (mm) std::memcpy(mm, sp->re.mass.data(), sp->re.mass.size() * 8);
  return HDR_OK;
}

hdr_status hdr_space_unit_load(hdr_space_t sp, double* out) {
  if (!sp || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  std::memcpy(out, sp->re.unit_load.data(), sp->re.unit_load.size() * 8);
  return HDR_OK;
}

hdr_status hdr_space_set_stream(hdr_space_t sp, void* stream) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  return catch_all([&]() -> hdr_status {
    CK(cudaStreamSynchronize(sp->stream));
    if (sp->own_stream) cudaStreamDestroy(sp->stream);
    if (stream) {
      sp->stream = static_cast<cudaStream_t>(stream);
      sp->own_stream = false;
    } else {
      CK(cudaStreamCreateWithFlags(&sp->stream, cudaStreamNonBlocking));
      sp->own_stream = true;
    }
    return HDR_OK;
  });
}

hdr_status hdr_space_synchronize(hdr_space_t sp) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  return catch_all([&]() -> hdr_status {
    CK(cudaStreamSynchronize(sp->stream));
    return HDR_OK;
  });
}

hdr_status hdr_space_pattern(hdr_space_t sp, int which, int64_t* row_offsets, int64_t* col_indices) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  return catch_all([&]() -> hdr_status {
    const int64_t nr = which == 0 ? sp->m : sp->ns;
    const int64_t nz = which == 0 ? sp->nnz_h : sp->nnz_s;
    const int64_t* ro = which == 0 ? sp->row_h.p : sp->row_s.p;
    const int32_t* ci = which == 0 ? sp->col_h.p : sp->col_s.p;
    if (row_offsets) CK(cudaMemcpy(row_offsets, ro, static_cast<size_t>(nr + 1) * 8, cudaMemcpyDeviceToHost));
    if (col_indices) {
      std::vector<int32_t> tmp(static_cast<size_t>(nz));
      if (nz) CK(cudaMemcpy(tmp.data(), ci, static_cast<size_t>(nz) * 4, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < nz; ++i) col_indices[i] = tmp[static_cast<size_t>(i)];
    }
    return HDR_OK;
  });
}

hdr_status hdr_space_master_globals(hdr_space_t sp, int64_t* out) {
  if (!sp || !out) return fail(HDR_INVALID_ARGUMENT, "null argument");
  for (int64_t i = 0; i < sp->ns; ++i) out[i] = i;  // every face dof is a master, in order
  return HDR_OK;
}

hdr_status hdr_near_nullspace_check(hdr_space_t sp, const double* alpha, const double* beta, int on_device,
                                    int weighted, int64_t dense_cap, double* eigenvalues) {
  if (!sp || !alpha || !beta) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (sp->m == 0) return HDR_OK;  // no multipliers: the reference returns {}
  if (!eigenvalues) return fail(HDR_INVALID_ARGUMENT, "null argument");
  if (sp->m * sp->m > dense_cap)
    return fail(HDR_CAP_EXCEEDED, "near_nullspace_check: m = " + std::to_string(sp->m) + " exceeds dense cap");
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    // element_matrices' coefficient check (rt_space.cpp:353-354), on a host copy
    std::vector<double> ha(static_cast<size_t>(sp->ncells)), hb(static_cast<size_t>(sp->ncells));
    CK(cudaMemcpyAsync(ha.data(), alpha, ha.size() * 8, on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, st));
    CK(cudaMemcpyAsync(hb.data(), beta, hb.size() * 8, on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, st));
    CK(cudaStreamSynchronize(st));
    for (size_t e = 0; e < ha.size(); ++e)
      if (!(ha[e] > 0.0) || !(hb[e] > 0.0))
        return fail(HDR_INVALID_ARGUMENT, "element_matrices: coefficients must be positive");
    DBuf<double> db;
    const double* pb = beta;
    if (!on_device) {
      stage(db, beta, sp->ncells, 0, st);
      pb = db.p;
    }
    return near_nullspace_device(sp->dm, sp->re, weighted, sp->mbase.p, sp->m, pb, eigenvalues, st);
  });
}

hdr_status hdr_space_dof_map(hdr_space_t sp, int64_t* global, double* sign) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  const DevMesh& m = sp->dm;
  for (int64_t e = 0; e < sp->ncells; ++e) {
    int64_t c[3];
    cell_coords(m, e, c);
    int64_t l = e * sp->n;
    for (int i = 0; i < sp->nint; ++i, ++l) {
      if (global) global[l] = sp->fdc + e * sp->nint + i;
      if (sign) sign[l] = 1.0;
    }
    for (int s = 0; s < 2 * sp->dim; ++s) {
      const int64_t f = slot_face(m, c, s, nullptr);
      for (int sub = 0; sub < sp->dpf; ++sub, ++l) {
        if (global) global[l] = f * sp->dpf + sub;
        if (sign) sign[l] = (s & 1) ? 1.0 : -1.0;
      }
    }
  }
  return HDR_OK;
}

static hdr_status run_hybridize(hdr_hybrid_t op, const double* alpha, const double* beta, const double* f_hat,
                                int on_device, bool sync) {
  hdr_space_t sp = op->sp;
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    const double *da = alpha, *db = beta, *df = f_hat;
    if (!on_device) {  // host inputs: staged into owned device buffers (pinned sources copy asynchronously)
      stage(op->alpha, alpha, sp->ncells, 0, st);
      stage(op->beta, beta, sp->ncells, 0, st);
      stage(op->f, f_hat, sp->broken, 0, st);
      da = op->alpha.p;
      db = op->beta.p;
      df = op->f.p;
    }
    // device inputs are borrowed: recovery re-reads alpha/beta from them
    op->a_ptr = da;
    op->b_ptr = db;
    if (!op->hval.p) op->hval.alloc(sp->nnz_h);
    if (!op->g.p) op->g.alloc(sp->m);
    if (!op->status.p) {
      op->status.alloc(1);
      CK(cudaMemsetAsync(op->status.p, 0, sizeof(int), st));
    }
    if (sp->geom) return geom_hybridize(sp->geom, da, db, df, op->hval.p, op->g.p, st);
    exact_prepare(sp, op, st);
    // k >= 1: the exact-path list is rebuilt every call (kern_exact.cu); k = 0: the
    // kernels solve rejected cells themselves (the brick kernels' list, xcount[2],
    // is reset by k_rt0_exact); the count is reset here for the synchronous calls
    if (sp->k > 0 || sync) CK(cudaMemsetAsync(op->xcount.p, 0, sizeof(int), st));
    op->last_call = 0;
    HybArgs A{};
    A.m = sp->dm;
    A.fx = sp->fx;
    A.nF = sp->nF;
    A.p_max = 4;
    A.xlist = op->xlist.p;
    A.xcount = op->xcount.p;
    A.eps32 = sp->eps32;
    A.eps_tc = sp->eps_tc;
    A.force_exact = sp->force_exact;
    A.qlog = sp->qlog;
    A.alpha = da;
    A.beta = db;
    A.f = df;
    A.mbase = sp->mbase.p;
    A.rowoff = sp->row_h.p;
    A.hval = op->hval.p;
    A.g = op->g.p;
    A.status = op->status.p;
    A.rank_tab = sp->rank_tab.p;
    A.frs = sp->frs.p;
    if (sp->k == 0) {
      // colour-0 staging: per cell slot (row-stage variant), per face (side slots; brick: N+1 per face)
      const int64_t need = std::max<int64_t>(parity_count(sp->dm) * sp->n * (sp->n + 1), (sp->n + 1) * sp->nfaces);
      if (op->ws_doubles < need) {
        op->ws.alloc(static_cast<size_t>(need));
        op->ws_doubles = need;
      }
      launch_hybridize_rt0_rows(A, sp->rt0_consts.data(), op->ws.p, st);
    } else if (hybridize_big_supported(sp->dim, sp->k)) {
      const int64_t need = hybridize_big_scratch_doubles(A, sp->k);
      if (op->ws_doubles < need) {
        op->ws.alloc(static_cast<size_t>(need));
        op->ws_doubles = need;
      }
      const int npr = sp->n + sp->r;  // [N0 ; X^T] f for every cell, one batched fp64 GEMM
      if (!op->pre.p || op->pre.n < static_cast<size_t>(npr) * sp->ncells) op->pre.alloc(static_cast<size_t>(npr) * sp->ncells);
      launch_gemm_f64_nn(npr, static_cast<int>(sp->ncells), sp->n, sp->premat.p, npr, df, sp->n, op->pre.p, npr, st);
      for (int parity = 0; parity < 2; ++parity) launch_hybridize_big(A, sp->k, parity, op->ws.p, op->pre.p, st);
    } else if (hybridize_warp_supported(sp->dim, sp->k)) {
      const int64_t need = hybridize_warp_scratch_doubles(A);
      if (op->ws_doubles < need) {
        op->ws.alloc(static_cast<size_t>(need));
        op->ws_doubles = need;
      }
      const double* pre = nullptr;
      if (sp->dim == 3 && sp->premat.p) {  // [N0 f ; X^T f] for every cell, one batched fp64 GEMM
        const int npr = sp->n + sp->r;
        if (!op->pre.p || op->pre.n < static_cast<size_t>(npr) * sp->ncells) op->pre.alloc(static_cast<size_t>(npr) * sp->ncells);
        launch_gemm_f64_nn(npr, static_cast<int>(sp->ncells), sp->n, sp->premat.p, npr, df, sp->n, op->pre.p, npr, st);
        pre = op->pre.p;
      }
      for (int parity = 0; parity < 2; ++parity) launch_hybridize_warp(A, parity, op->ws.p, pre, st);
    } else {
      return fail(HDR_UNSUPPORTED, "hybridize: no structured kernel for this dim / order");
    }
    if (sp->k > 0) {  // the rejected cells of each colour, after both colours' fast passes
      const ExactArgs X = exact_args(sp, op, EXACT_HYB, da, db, df);
      for (int parity = 0; parity < 2; ++parity) launch_exact(X, parity, sp->xws.p, st);
    }
    CK(cudaGetLastError());
    if (!sync) return HDR_OK;
    return check_status(op->status.p, st, op->xbad.p);
  });
}

hdr_status hdr_hybridize_fe(hdr_space_t sp, const double* alpha, const double* beta, const double* f_hat, int on_device,
                            hdr_hybrid_t* out) {
  if (!sp || !out || !alpha || !beta || !f_hat) return fail(HDR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  auto op = std::make_unique<hdr_hybrid_s>();
  op->sp = sp;
  const hdr_status s = run_hybridize(op.get(), alpha, beta, f_hat, on_device, true);
  if (s != HDR_OK) return s;
  *out = op.release();
  return HDR_OK;
}

hdr_status hdr_hybridize_fe_into(hdr_hybrid_t op, const double* alpha, const double* beta, const double* f_hat,
                                 int on_device) {
  if (!op || !alpha || !beta || !f_hat) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return run_hybridize(op, alpha, beta, f_hat, on_device, true);
}

hdr_status hdr_hybridize_fe_enqueue(hdr_hybrid_t op, const double* alpha, const double* beta, const double* f_hat,
                                   int on_device) {
  if (!op || !alpha || !beta || !f_hat) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return run_hybridize(op, alpha, beta, f_hat, on_device, false);
}

hdr_status hdr_hybridize_fe_batch(hdr_space_t sp, int count, const double* const* alpha, const double* const* beta,
                                  const double* const* f_hat, double* const* h_values, double* const* g) {
  if (!sp || count < 0 || (count > 0 && (!alpha || !beta || !f_hat))) return fail(HDR_INVALID_ARGUMENT, "null argument");
  for (int i = 0; i < count; ++i)
    if (!alpha[i] || !beta[i] || !f_hat[i]) return fail(HDR_INVALID_ARGUMENT, "null input of a batch item");
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    if (!sp->batch) {
      auto ctx = std::make_unique<BatchCtx>();
      CK(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ctx->ds, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&ctx->ev_in[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_comp[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_d2h[b], cudaEventDisableTiming));
        ctx->op[b].sp = sp;
        ctx->op[b].alpha.alloc(static_cast<size_t>(sp->ncells));
        ctx->op[b].beta.alloc(static_cast<size_t>(sp->ncells));
        ctx->op[b].f.alloc(static_cast<size_t>(sp->broken));
      }
      sp->batch = ctx.release();
    }
    BatchCtx& B = *sp->batch;
    // the previous batch (and anything else on the space's stream) completes first
    CK(cudaEventRecord(B.ev_comp[0], st));
    CK(cudaStreamWaitEvent(B.cs, B.ev_comp[0], 0));
    CK(cudaStreamWaitEvent(B.ds, B.ev_comp[0], 0));
    for (int i = 0; i < count; ++i) {
      const int b = i & 1;
      hdr_hybrid_s* op = &B.op[b];
      if (i >= 2) CK(cudaStreamWaitEvent(B.cs, B.ev_comp[b], 0));  // item i - 2's kernels done with the inputs
      CK(cudaMemcpyAsync(op->alpha.p, alpha[i], static_cast<size_t>(sp->ncells) * 8, cudaMemcpyHostToDevice, B.cs));
      CK(cudaMemcpyAsync(op->beta.p, beta[i], static_cast<size_t>(sp->ncells) * 8, cudaMemcpyHostToDevice, B.cs));
      CK(cudaMemcpyAsync(op->f.p, f_hat[i], static_cast<size_t>(sp->broken) * 8, cudaMemcpyHostToDevice, B.cs));
      CK(cudaEventRecord(B.ev_in[b], B.cs));
      CK(cudaStreamWaitEvent(st, B.ev_in[b], 0));
      if (i >= 2) CK(cudaStreamWaitEvent(st, B.ev_d2h[b], 0));  // item i - 2's download of these H values done
      const hdr_status s = run_hybridize(op, op->alpha.p, op->beta.p, op->f.p, 1, false);
      if (s != HDR_OK) return s;
      CK(cudaEventRecord(B.ev_comp[b], st));
      CK(cudaStreamWaitEvent(B.ds, B.ev_comp[b], 0));
      if (h_values && h_values[i] && sp->nnz_h)
        CK(cudaMemcpyAsync(h_values[i], op->hval.p, static_cast<size_t>(sp->nnz_h) * 8, cudaMemcpyDeviceToHost, B.ds));
      if (g && g[i] && sp->m)
        CK(cudaMemcpyAsync(g[i], op->g.p, static_cast<size_t>(sp->m) * 8, cudaMemcpyDeviceToHost, B.ds));
      CK(cudaEventRecord(B.ev_d2h[b], B.ds));
    }
    // the space's stream is ordered after the last download (callers time on it)
    if (count > 0) CK(cudaStreamWaitEvent(st, B.ev_d2h[(count - 1) & 1], 0));
    CK(cudaStreamSynchronize(B.ds));
    CK(cudaStreamSynchronize(B.cs));
    for (int b = 0; b < 2 && b < count; ++b) {
      const hdr_status s = check_status(B.op[b].status.p, st);
      if (s != HDR_OK) return s;
    }
    CK(cudaStreamSynchronize(st));
    return HDR_OK;
  });
}

hdr_status hdr_hybrid_check(hdr_hybrid_t op) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status { return check_status(op->status.p, op->sp->stream, op->xbad.p); });
}

hdr_status hdr_hybrid_exact_cells(hdr_hybrid_t op, int64_t* count) {
  if (!op || !count) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    int c = 0;
    if (op->xcount.p) {
      const int slot = (op->sp->k == 0 && op->last_call == 1) ? 3 : 0;
      CK(cudaMemcpyAsync(&c, op->xcount.p + slot, sizeof(int), cudaMemcpyDeviceToHost, op->sp->stream));
      CK(cudaStreamSynchronize(op->sp->stream));
    }
    *count = c;
    return HDR_OK;
  });
}

hdr_status hdr_space_set_exact_policy(hdr_space_t sp, int force_exact, double eps32, double eps_tc, float* q_log) {
  if (!sp) return fail(HDR_INVALID_ARGUMENT, "null space");
  sp->force_exact = force_exact ? 1 : 0;
  sp->eps32 = eps32 > 0 ? eps32 : default_eps32(sp->n);
  sp->eps_tc = eps_tc > 0 ? eps_tc : kDefaultEpsTc;
  sp->qlog = q_log;
  return HDR_OK;
}

hdr_status hdr_hybrid_symmetrize(hdr_hybrid_t op) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status {
    launch_csr_symmetrize32(op->sp->m, op->sp->row_h.p, op->sp->col_h.p, op->hval.p, op->sp->stream);
    CK(cudaStreamSynchronize(op->sp->stream));
    CK(cudaGetLastError());
    return HDR_OK;
  });
}

hdr_status hdr_hybrid_values_enqueue(hdr_hybrid_t op, double* h_values, double* g, int dst_on_device) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status {
    const cudaMemcpyKind kind = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    cudaStream_t st = op->sp->stream;
    if (h_values && op->sp->nnz_h)
      CK(cudaMemcpyAsync(h_values, op->hval.p, static_cast<size_t>(op->sp->nnz_h) * 8, kind, st));
    if (g && op->sp->m) CK(cudaMemcpyAsync(g, op->g.p, static_cast<size_t>(op->sp->m) * 8, kind, st));
    return HDR_OK;
  });
}

void hdr_hybrid_destroy(hdr_hybrid_t op) { delete op; }

hdr_status hdr_hybrid_values(hdr_hybrid_t op, double* h_values, double* g, int dst_on_device) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status {
    const cudaMemcpyKind kind = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    cudaStream_t st = op->sp->stream;
    if (h_values && op->sp->nnz_h)
      CK(cudaMemcpyAsync(h_values, op->hval.p, static_cast<size_t>(op->sp->nnz_h) * 8, kind, st));
    if (g && op->sp->m) CK(cudaMemcpyAsync(g, op->g.p, static_cast<size_t>(op->sp->m) * 8, kind, st));
    CK(cudaStreamSynchronize(st));
    return HDR_OK;
  });
}

hdr_status hdr_hybrid_device_ptrs(hdr_hybrid_t op, const double** h_values, const double** g,
                                  const int64_t** row_offsets, const int32_t** col_indices) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  if (h_values) *h_values = op->hval.p;
  if (g) *g = op->g.p;
  if (row_offsets) *row_offsets = op->sp->row_h.p;
  if (col_indices) *col_indices = op->sp->col_h.p;
  return HDR_OK;
}

hdr_status hdr_recover_hybrid(hdr_hybrid_t op, const double* lambda, const double* f_hat, int on_device, double* x_hat,
                              double* x) {
  if (!op || !lambda || !f_hat) return fail(HDR_INVALID_ARGUMENT, "null argument");
  hdr_space_t sp = op->sp;
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    DBuf<double> dl, df, dxh, dx;
    const double *pl = lambda, *pf = f_hat;
    if (!on_device) {
      stage(dl, lambda, sp->m, 0, st);
      stage(df, f_hat, sp->broken, 0, st);
      pl = dl.p;
      pf = df.p;
    }
    double* pxh = x_hat;
    double* px = x;
    if (!on_device || !x_hat) {
      dxh.alloc(sp->broken);
      pxh = dxh.p;
    }
    if (!on_device || !x) {
      dx.alloc(sp->ndofs);
      px = dx.p;
    }
    if (!op->status.p) {
      op->status.alloc(1);
      CK(cudaMemsetAsync(op->status.p, 0, sizeof(int), st));
    }
    if (sp->geom) {
      const hdr_status s = geom_recover_hybrid(sp->geom, op->a_ptr, op->b_ptr, pl, pf, pxh, px, st);
      if (s != HDR_OK) return s;
      if (!on_device) {
        if (x_hat) CK(cudaMemcpyAsync(x_hat, pxh, static_cast<size_t>(sp->broken) * 8, cudaMemcpyDeviceToHost, st));
        if (x) CK(cudaMemcpyAsync(x, px, static_cast<size_t>(sp->ndofs) * 8, cudaMemcpyDeviceToHost, st));
      }
      CK(cudaStreamSynchronize(st));
      return HDR_OK;
    }
    exact_prepare(sp, op, st);
    int* rcount = sp->k > 0 ? op->xcount.p : op->xcount.p + 3;  // k = 0 keeps the hybridize list intact
    CK(cudaMemsetAsync(rcount, 0, sizeof(int), st));
    op->last_call = 1;
    RecArgs R{};
    R.m = sp->dm;
    R.fx = sp->fx;
    R.nF = sp->nF;
    R.p_max = 8;  // fp64 Neumann terms: a-priori order control (struct_order_apriori)
    R.xlist = op->xlist.p;
    R.xcount = rcount;
    R.force_exact = sp->force_exact;
    R.alpha = op->a_ptr;
    R.beta = op->b_ptr;
    R.f = pf;
    R.lambda = pl;
    R.mbase = sp->mbase.p;
    R.x_hat = pxh;
    R.x = px;
    R.status = op->status.p;
    if (sp->k == 0) {
      launch_recover_rt0(R, sp->rt0_consts.data(), st);
    } else {
      launch_recover_hybrid(R, nullptr, 0, st);
      ExactArgs X = exact_args(sp, op, EXACT_REC, op->a_ptr, op->b_ptr, pf);
      X.lambda = pl;
      X.x_hat = pxh;
      launch_exact(X, 0, sp->xws.p, st);
    }
    launch_average_faces(sp->dm, pxh, px, st);
    CK(cudaGetLastError());
    if (!on_device) {
      if (x_hat) CK(cudaMemcpyAsync(x_hat, pxh, static_cast<size_t>(sp->broken) * 8, cudaMemcpyDeviceToHost, st));
      if (x) CK(cudaMemcpyAsync(x, px, static_cast<size_t>(sp->ndofs) * 8, cudaMemcpyDeviceToHost, st));
    }
    return check_status(op->status.p, st, op->xbad.p);
  });
}

static hdr_status check_cond_status(int* d_status, cudaStream_t st) {
  int status = 0;
  CK(cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (status) CK(cudaMemsetAsync(d_status, 0, sizeof(int), st));
  if (status & 2) return fail(HDR_SINGULAR_BLOCK, "static_condense: an interior block A_ii is not positive definite");
  return HDR_OK;
}

static hdr_status run_condense(hdr_condensed_t op, const double* alpha, const double* beta, const double* f_hat,
                               int on_device) {
  hdr_space_t sp = op->sp;
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    const double *da = alpha, *db = beta, *df = f_hat;
    if (!on_device) {
      stage(op->alpha, alpha, sp->ncells, 0, st);
      stage(op->beta, beta, sp->ncells, 0, st);
      stage(op->f, f_hat, sp->broken, 0, st);
      da = op->alpha.p;
      db = op->beta.p;
      df = op->f.p;
    }
    op->a_ptr = da;
    op->b_ptr = db;
    if (!op->sval.p) op->sval.alloc(sp->nnz_s);
    if (!op->fs.p) op->fs.alloc(sp->ns);
    if (!op->status.p) {
      op->status.alloc(1);
      CK(cudaMemsetAsync(op->status.p, 0, sizeof(int), st));
    }
    if (sp->geom) return geom_condense(sp->geom, da, db, df, op->sval.p, op->fs.p, st);
    const int64_t need = condense_ws_doubles(sp->dm, sp->nF);
    if (need > op->ws_doubles) {
      op->ws.alloc(static_cast<size_t>(need));
      op->ws_doubles = need;
    }
    CondArgs C{};
    C.m = sp->dm;
    C.fx = sp->fx;
    C.nF = sp->nF;
    C.alpha = da;
    C.beta = db;
    C.f = df;
    C.rowoff = sp->row_s.p;
    C.sval = op->sval.p;
    C.fs = op->fs.p;
    C.status = op->status.p;
    C.host_consts = (sp->k == 0 && !sp->rt0_consts.empty()) ? sp->rt0_consts.data() : nullptr;
    for (int parity = 0; parity < 2; ++parity) launch_condense(C, parity, op->ws.p, op->ws_doubles, st);
    CK(cudaGetLastError());
    return check_cond_status(op->status.p, st);
  });
}

hdr_status hdr_static_condense_fe(hdr_space_t sp, const double* alpha, const double* beta, const double* f_hat,
                                  int on_device, hdr_condensed_t* out) {
  if (!sp || !out || !alpha || !beta || !f_hat) return fail(HDR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  auto op = std::make_unique<hdr_condensed_s>();
  op->sp = sp;
  const hdr_status s = run_condense(op.get(), alpha, beta, f_hat, on_device);
  if (s != HDR_OK) return s;
  *out = op.release();
  return HDR_OK;
}

hdr_status hdr_static_condense_fe_into(hdr_condensed_t op, const double* alpha, const double* beta,
                                       const double* f_hat, int on_device) {
  if (!op || !alpha || !beta || !f_hat) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return run_condense(op, alpha, beta, f_hat, on_device);
}

void hdr_condensed_destroy(hdr_condensed_t op) { delete op; }

hdr_status hdr_condensed_values(hdr_condensed_t op, double* s_values, double* f_s, int dst_on_device) {
  if (!op) return fail(HDR_INVALID_ARGUMENT, "null operator");
  return catch_all([&]() -> hdr_status {
    const cudaMemcpyKind kind = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    cudaStream_t st = op->sp->stream;
    if (s_values && op->sp->nnz_s)
      CK(cudaMemcpyAsync(s_values, op->sval.p, static_cast<size_t>(op->sp->nnz_s) * 8, kind, st));
    if (f_s && op->sp->ns) CK(cudaMemcpyAsync(f_s, op->fs.p, static_cast<size_t>(op->sp->ns) * 8, kind, st));
    CK(cudaStreamSynchronize(st));
    return HDR_OK;
  });
}

hdr_status hdr_recover_condensed(hdr_condensed_t op, const double* x_b, const double* f_hat, int on_device,
                                 double* x) {
  if (!op || !x_b || !f_hat || !x) return fail(HDR_INVALID_ARGUMENT, "null argument");
  hdr_space_t sp = op->sp;
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    DBuf<double> dxb, df, dx;
    const double *pxb = x_b, *pf = f_hat;
    double* px = x;
    if (!on_device) {
      stage(dxb, x_b, sp->ns, 0, st);
      stage(df, f_hat, sp->broken, 0, st);
      dx.alloc(sp->ndofs);
      pxb = dxb.p;
      pf = df.p;
      px = dx.p;
    }
    if (sp->geom) {
      const hdr_status s = geom_recover_condensed(sp->geom, op->a_ptr, op->b_ptr, pxb, pf, px, st);
      if (s != HDR_OK) return s;
      if (!on_device) CK(cudaMemcpyAsync(x, px, static_cast<size_t>(sp->ndofs) * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      return HDR_OK;
    }
    const int64_t need = condense_ws_doubles(sp->dm, sp->nF);
    if (need > op->ws_doubles) {
      op->ws.alloc(static_cast<size_t>(need));
      op->ws_doubles = need;
    }
    CondArgs C{};
    C.m = sp->dm;
    C.fx = sp->fx;
    C.nF = sp->nF;
    C.alpha = op->a_ptr;
    C.beta = op->b_ptr;
    C.f = pf;
    C.xb = pxb;
    C.x = px;
    C.status = op->status.p;
    launch_recover_condensed(C, op->ws.p, op->ws_doubles, st);
    CK(cudaGetLastError());
    if (!on_device) CK(cudaMemcpyAsync(x, px, static_cast<size_t>(sp->ndofs) * 8, cudaMemcpyDeviceToHost, st));
    return check_cond_status(op->status.p, st);
  });
}

static hdr_status spmv_common(hdr_space_t sp, int which, const double* vals, const double* x, double* y,
                              int on_device) {
  return catch_all([&]() -> hdr_status {
    cudaStream_t st = sp->stream;
    const int64_t nr = which == 0 ? sp->m : sp->ns;
    DBuf<double> dx, dy;
    const double* px = x;
    double* py = y;
    if (!on_device) {
      stage(dx, x, nr, 0, st);
      dy.alloc(nr);
      px = dx.p;
      py = dy.p;
    }
    if (which == 0)
      launch_spmv32(nr, sp->row_h.p, sp->col_h.p, vals, px, py, st, sp->nnz_h);
    else
      launch_spmv32(nr, sp->row_s.p, sp->col_s.p, vals, px, py, st, sp->nnz_s);
    CK(cudaGetLastError());
    if (!on_device) CK(cudaMemcpyAsync(y, py, static_cast<size_t>(nr) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HDR_OK;
  });
}

hdr_status hdr_hybrid_spmv(hdr_hybrid_t op, const double* x, double* y, int on_device) {
  if (!op || !x || !y) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return spmv_common(op->sp, 0, op->hval.p, x, y, on_device);
}

hdr_status hdr_condensed_spmv(hdr_condensed_t op, const double* x, double* y, int on_device) {
  if (!op || !x || !y) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return spmv_common(op->sp, 1, op->sval.p, x, y, on_device);
}

static hdr_status pcg_common(int64_t n, const int64_t* ro, const int32_t* ci, const double* vals, const double* own_rhs,
                              const double* b, double* x, int on_device, double rtol, int64_t maxit, int precond,
                              double* hist, hdr_pcg_report* rep, cudaStream_t st) {
  return catch_all([&]() -> hdr_status {
    DBuf<double> db, dx;
    const double* pb = b ? b : own_rhs;
    if (b && !on_device) {
      db.upload(b, static_cast<size_t>(n));
      pb = db.p;
    }
    double* px = x;
    if (!on_device) {
      dx.alloc(static_cast<size_t>(n));
      px = dx.p;
    }
    const hdr_status s = pcg_device(n, ro, ci, nullptr, vals, pb, px, rtol, maxit, precond, hist, rep, st);
    if (s != HDR_OK) return s;
    if (!on_device && n) CK(cudaMemcpy(x, px, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}

hdr_status hdr_hybrid_pcg(hdr_hybrid_t op, const double* b, double* x, int on_device, double rtol, int64_t maxit,
                          int precond, double* hist, hdr_pcg_report* rep) {
  if (!op || !x) return fail(HDR_INVALID_ARGUMENT, "null argument");
  hdr_space_t sp = op->sp;
  return pcg_common(sp->m, sp->row_h.p, sp->col_h.p, op->hval.p, op->g.p, b, x, on_device, rtol, maxit, precond, hist,
                    rep, sp->stream);
}

hdr_status hdr_condensed_pcg(hdr_condensed_t op, const double* b, double* x, int on_device, double rtol,
                             int64_t maxit, int precond, double* hist, hdr_pcg_report* rep) {
  if (!op || !x) return fail(HDR_INVALID_ARGUMENT, "null argument");
  hdr_space_t sp = op->sp;
  return pcg_common(sp->ns, sp->row_s.p, sp->col_s.p, op->sval.p, op->fs.p, b, x, on_device, rtol, maxit, precond,
                    hist, rep, sp->stream);
}

hdr_status hdr_csr_pcg_host(int64_t n, const int64_t* ro, const int64_t* ci, const double* v, const double* b,
                            double* x, double rtol, int64_t maxit, int precond, double* hist, hdr_pcg_report* rep) {
  if (n < 0 || !ro || !b || !x || (n > 0 && ro[n] > 0 && (!ci || !v))) return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    int devs = 0;
    if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) return fail(HDR_CUDA_ERROR, "no CUDA device available");
    const int64_t nnz = ro[n];
    DBuf<int64_t> dro, dci;
    DBuf<double> dv, db, dx;
    dro.upload(ro, static_cast<size_t>(n) + 1);
    dci.upload(ci, static_cast<size_t>(nnz));
    dv.upload(v, static_cast<size_t>(nnz));
    db.upload(b, static_cast<size_t>(n));
    dx.alloc(static_cast<size_t>(n));
    const hdr_status s = pcg_device(n, dro.p, nullptr, dci.p, dv.p, db.p, dx.p, rtol, maxit, precond, hist, rep, nullptr);
    if (s != HDR_OK) return s;
    if (n) CK(cudaMemcpy(x, dx.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}

hdr_status hdr_csr_spmv_host(int64_t nrows, int64_t ncols, const int64_t* row_offsets, const int64_t* col_indices,
                             const double* values, const double* x, double* y) {
  if (nrows < 0 || ncols < 0 || !row_offsets || (nrows > 0 && (!col_indices || !values || !x || !y)))
    return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    int devs = 0;
    if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) return fail(HDR_CUDA_ERROR, "no CUDA device available");
    const int64_t nnz = row_offsets[nrows];
    DBuf<int64_t> ro, ci;
    DBuf<double> v, dx, dy;
    ro.alloc(nrows + 1);
    ci.alloc(nnz);
    v.alloc(nnz);
    dx.alloc(ncols);
    dy.alloc(nrows);
    CK(cudaMemcpy(ro.p, row_offsets, static_cast<size_t>(nrows + 1) * 8, cudaMemcpyHostToDevice));
    if (nnz) {
      CK(cudaMemcpy(ci.p, col_indices, static_cast<size_t>(nnz) * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(v.p, values, static_cast<size_t>(nnz) * 8, cudaMemcpyHostToDevice));
    }
    if (ncols) CK(cudaMemcpy(dx.p, x, static_cast<size_t>(ncols) * 8, cudaMemcpyHostToDevice));
    launch_spmv64(nrows, ro.p, ci.p, v.p, dx.p, dy.p, nullptr, nnz);
    CK(cudaGetLastError());
    if (nrows) CK(cudaMemcpy(y, dy.p, static_cast<size_t>(nrows) * 8, cudaMemcpyDeviceToHost));
    return HDR_OK;
  });
}

hdr_status hdr_csr_spmv_device(int64_t nrows, const int64_t* row_offsets, const int64_t* col_indices,
                               const double* values, const double* x, double* y, void* stream) {
  if (nrows < 0 || (nrows > 0 && (!row_offsets || !col_indices || !values || !x || !y)))
    return fail(HDR_INVALID_ARGUMENT, "null argument");
  return catch_all([&]() -> hdr_status {
    launch_spmv64(nrows, row_offsets, col_indices, values, x, y, static_cast<cudaStream_t>(stream));
    CK(cudaGetLastError());
    return HDR_OK;
  });
}

}  // extern "C"
