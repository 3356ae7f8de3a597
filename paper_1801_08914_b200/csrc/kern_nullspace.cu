// near_nullspace_check on the device: the eigenvalues of
// the assembled C Y C^T, Y_T = M^-1 - M^-1 B^T (B M^-1 B^T)^-1 B M^-1 the
// three-field flux operator of every cell (src/reduction.cpp:711-742).
//
// Bit-identical to the reference by construction:
//  - k_ns_cell: one CTA per cell runs the reference's dense sequence
//    (lu_factor / lu_solve_matrix / lu_inverse / dense_multiply / dense_add,
//    src/dense.cpp:17-177) on M = 0 + beta M_ref and B = ref_div_form; every
//    entry sees the same operations in the same order as in the serial code
//    (rows / columns / right-hand sides are the parallel axes), with explicit
//    _rn intrinsics so nothing is contracted into an FMA (the reference's
//    Release build has none).  It then forms
//    c_e (Y c_e^T) in the reference's summation order and adds it into the
//    dense m x m matrix: an entry gets at most two contributions (two distinct
//    faces share at most one cell), and fl(0 + a + b) does not depend on the
//    order of a and b, so the atomics are deterministic.
//  - k_ns_jacobi: one CTA runs the cyclic Jacobi sweeps of symmetric_eigenvalues
//    (src/dense.cpp:197-244) rotation by rotation in the reference's (p, q)
//    order; a rotation's column update and row update are parallel over k.
//    The diagonal is then sorted (rank sort: the sorted multiset is unique).
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "hdr_internal.hpp"
#include "kernels.hpp"
#include "dense_cta.cuh"

namespace hdr {
namespace {

constexpr int kNsT = 256;

// dense_multiply (dense.cpp:17-28): c (r x q) = a (r x kk) b (kk x q), zero a_ik skipped
__device__ void cta_multiply(const double* a, const double* b, int r, int kk, int q, double* c) {
  for (int t = threadIdx.x; t < r * q; t += blockDim.x) {
    const int i = t / q, j = t % q;
    double s = 0.0;
    for (int k = 0; k < kk; ++k) {
      const double aik = a[i * kk + k];
      if (aik == 0.0) continue;
      s = add(s, mul(aik, b[k * q + j]));
    }
    c[t] = s;
  }
  __syncthreads();
}

__device__ void cta_transpose(const double* a, int r, int c, double* t) {
  for (int u = threadIdx.x; u < r * c; u += blockDim.x) {
    const int i = u / c, j = u % c;
    t[j * r + i] = a[u];
  }
  __syncthreads();
}

struct NsArgs {
  DevMesh m;
  int n, npr, nint, dpf, weighted;
  const double* mass;     // n x n
  const double* bmat;     // div_form, npr x n
  const double* fm;       // face moments, 2 dim x dpf x n (weighted)
  const double* beta;
  const int* mbase;       // multiplier base per face (-1: boundary)
  int64_t mdim;           // rows of the dense matrix
  double* cyc;            // mdim x mdim (zeroed)
  double* ws;             // per-CTA workspace
  int64_t ws_stride;
  int* status;            // bit 0: singular block; bad cell in status[1] (min)
};

// c_e(row of slot s, sub-row r ; local column l)
__device__ __forceinline__ double ce_val(const NsArgs& A, int s, int r, int l) {
  const int l0 = A.nint + s * A.dpf;
  if (l < l0 || l >= l0 + A.dpf) return 0.0;
  return A.weighted ? A.fm[(static_cast<int64_t>(s) * A.dpf + r) * A.n + l] : (l - l0 == r ? 1.0 : 0.0);
}

__global__ void __launch_bounds__(kNsT) k_ns_cell(NsArgs A) {
  __shared__ double red[32];
  __shared__ int ired[1];
  const int n = A.n, npr = A.npr;
  double* w = A.ws + blockIdx.x * A.ws_stride;
  double* mlu = w;                                   // n x n
  double* minv = mlu + n * n;                        // n x n  (then y)
  double* prod = minv + n * n;                       // n x n
  double* bt = prod + n * n;                         // n x npr  (B^T)
  double* minv_bt = bt + n * npr;                    // n x npr
  double* bmbt = minv_bt + n * npr;                  // npr x npr
  double* minv_bt_t = bmbt + npr * npr;              // npr x n
  double* inner = minv_bt_t + npr * n;               // npr x n
  int* piv_m = reinterpret_cast<int*>(inner + npr * n);
  int* piv_b = piv_m + n;
  for (int64_t e = blockIdx.x; e < A.m.ncells; e += gridDim.x) {
    const double beta = A.beta[e];
    // em.m_mat = dense_add(DenseMatrix(n, n), mass, beta) (rt_space.cpp:358)
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) mlu[i] = add(0.0, mul(beta, A.mass[i]));
    cta_transpose(A.bmat, npr, n, bt);
    if (!cta_lu_factor(mlu, n, piv_m, red, ired)) {
      if (threadIdx.x == 0) {
        atomicOr(A.status, 1);
        atomicMin(A.status + 1, static_cast<int>(e));
      }
      continue;
    }
    cta_lu_solve_matrix(mlu, piv_m, n, bt, npr, minv_bt);  // M^-1 B^T
    cta_multiply(A.bmat, minv_bt, npr, n, npr, bmbt);      // B M^-1 B^T
    cta_lu_solve_matrix(mlu, piv_m, n, nullptr, n, minv);  // lu_inverse
    if (!cta_lu_factor(bmbt, npr, piv_b, red, ired)) {
      if (threadIdx.x == 0) {
        atomicOr(A.status, 1);
        atomicMin(A.status + 1, static_cast<int>(e));
      }
      continue;
    }
    cta_transpose(minv_bt, n, npr, minv_bt_t);
    cta_lu_solve_matrix(bmbt, piv_b, npr, minv_bt_t, n, inner);  // (B M^-1 B^T)^-1 B M^-1
    cta_multiply(minv_bt, inner, n, npr, n, prod);
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) minv[i] = add(minv[i], mul(-1.0, prod[i]));  // dense_add(.., -1)
    __syncthreads();
    const double* y = minv;
    // cyc_e = c_e (y c_e^T) in dense_multiply's order, scattered into the dense matrix
    int64_t c[3];
    cell_coords(A.m, e, c);
    int64_t fbase[6];
    int nsl = 2 * A.m.dim;
    for (int s = 0; s < nsl; ++s) {
      bool in = false;
      const int64_t f = slot_face(A.m, c, s, &in);
      fbase[s] = in ? A.mbase[f] : -1;
    }
    const int nr = nsl * A.dpf;
    for (int t = threadIdx.x; t < nr * nr; t += blockDim.x) {
      const int ra = t / nr, rb = t % nr;
      const int sa = ra / A.dpf, ia = ra % A.dpf, sb = rb / A.dpf, ib = rb % A.dpf;
      if (fbase[sa] < 0 || fbase[sb] < 0) continue;
      const int la0 = A.nint + sa * A.dpf, lb0 = A.nint + sb * A.dpf;
      double v = 0.0;
      for (int k = la0; k < la0 + A.dpf; ++k) {  // c_e(ra, k) nonzero only on slot sa's block
        const double cek = ce_val(A, sa, ia, k);
        if (cek == 0.0) continue;
        double tk = 0.0;  // (y c_e^T)(k, rb)
        for (int q = lb0; q < lb0 + A.dpf; ++q) {
          const double ykq = y[k * n + q];
          if (ykq == 0.0) continue;
          tk = add(tk, mul(ykq, ce_val(A, sb, ib, q)));
        }
        v = add(v, mul(cek, tk));
      }
      const int64_t R = fbase[sa] + ia, C = fbase[sb] + ib;
      atomicAdd(A.cyc + R * A.mdim + C, v);
    }
    __syncthreads();
  }
}

// symmetric_eigenvalues (dense.cpp:197-244), tol 1e-13, at most 64 sweeps
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_ns_jacobi(double* g, int n, double tol, double* ev) {
  extern __shared__ double dyn[];
  __shared__ double red[32];
  double* m = SMEM ? dyn : g;
  if (SMEM)
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) m[i] = g[i];
  __syncthreads();
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {  // symmetrize once
    const int i = t / n, j = t % n;
    if (j > i) {
      const double s = mul(0.5, add(m[i * n + j], m[j * n + i]));
      m[i * n + j] = s;
      m[j * n + i] = s;
    }
  }
  __syncthreads();
  double mx = 0.0;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) mx = fmax(mx, fabs(m[i]));
  const double scale = block_max(mx, red);
  if (scale != 0.0) {
    for (int sweep = 0; sweep < 64; ++sweep) {
      double off = 0.0;
      for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int i = t / n, j = t % n;
        if (j > i) off = fmax(off, fabs(m[t]));
      }
      if (block_max(off, red) <= mul(tol, scale)) break;
      for (int p = 0; p < n; ++p) {
        for (int q = p + 1; q < n; ++q) {
          const double apq = m[p * n + q];
          if (fabs(apq) <= 1e-300) continue;  // uniform over the CTA
          const double theta = (m[q * n + q] - m[p * n + p]) / mul(2.0, apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / add(fabs(theta), sqrt(add(mul(theta, theta), 1.0)));
          const double c = 1.0 / sqrt(add(mul(t, t), 1.0));
          const double s = mul(t, c);
          __syncthreads();  // every thread has read apq, a_pp, a_qq
          for (int k = threadIdx.x; k < n; k += blockDim.x) {
            const double akp = m[k * n + p], akq = m[k * n + q];
            m[k * n + p] = sub(mul(c, akp), mul(s, akq));
            m[k * n + q] = add(mul(s, akp), mul(c, akq));
          }
          __syncthreads();
          for (int k = threadIdx.x; k < n; k += blockDim.x) {
            const double apk = m[p * n + k], aqk = m[q * n + k];
            m[p * n + k] = sub(mul(c, apk), mul(s, aqk));
            m[q * n + k] = add(mul(s, apk), mul(c, aqk));
          }
          __syncthreads();
        }
      }
    }
  }
  __syncthreads();
  // sorted diagonal (rank sort; ties keep index order)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = scale == 0.0 ? 0.0 : m[i * n + i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double e = scale == 0.0 ? 0.0 : m[j * n + j];
      r += (e < d) || (e == d && j < i);
    }
    ev[r] = d;
  }
}

}  // namespace

// mesh / space data from the C ABI (capi.cu); eigenvalues to host `out` (m of them)
hdr_status near_nullspace_device(const DevMesh& dm, const RefElement& re, int weighted, const int* mbase, int64_t m,
                                 const double* beta_dev, double* out, cudaStream_t st) {
  if (m == 0) return HDR_OK;
  const int n = re.n, npr = re.npr;
  std::vector<double> consts;
  consts.insert(consts.end(), re.mass.begin(), re.mass.end());
  consts.insert(consts.end(), re.div_form.begin(), re.div_form.end());
  consts.insert(consts.end(), re.face_moments.begin(), re.face_moments.end());
  DBuf<double> dc, cyc, ws, ev;
  DBuf<int> status;
  dc.upload(consts);
  cyc.alloc(static_cast<size_t>(m) * m);
  ev.alloc(m);
  status.alloc(2);
  CK(cudaMemsetAsync(cyc.p, 0, static_cast<size_t>(m) * m * 8, st));
  const int init[2] = {0, 0x7fffffff};
  CK(cudaMemcpyAsync(status.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  const int grid = static_cast<int>(std::min<int64_t>(dm.ncells, 296));
  const int64_t stride = ((3 * n * n + 4 * n * npr + npr * npr + n + npr + 2) + 31) / 32 * 32;
  ws.alloc(static_cast<size_t>(grid) * stride);
  NsArgs A{};
  A.m = dm;
  A.n = n;
  A.npr = npr;
  A.nint = re.nint;
  A.dpf = re.dpf;
  A.weighted = weighted;
  A.mass = dc.p;
  A.bmat = dc.p + n * n;
  A.fm = dc.p + n * n + npr * n;
  A.beta = beta_dev;
  A.mbase = mbase;
  A.mdim = m;
  A.cyc = cyc.p;
  A.ws = ws.p;
  A.ws_stride = stride;
  A.status = status.p;
  k_ns_cell<<<grid, kNsT, 0, st>>>(A);
  count_launch();
  const size_t smem = static_cast<size_t>(m) * m * 8;
  if (smem <= 200 * 1024) {
    CK(cudaFuncSetAttribute(k_ns_jacobi<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_ns_jacobi<true><<<1, 1024, smem, st>>>(cyc.p, static_cast<int>(m), 1e-13, ev.p);
  } else {
    k_ns_jacobi<false><<<1, 1024, 0, st>>>(cyc.p, static_cast<int>(m), 1e-13, ev.p);
  }
  count_launch();
  int hs[2];
  CK(cudaMemcpyAsync(hs, status.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out, ev.p, static_cast<size_t>(m) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  if (hs[0]) return fail(HDR_SINGULAR_BLOCK, "lu_factor: pivot below threshold (near_nullspace_check, cell " +
                                                 std::to_string(hs[1]) + ")");
  return HDR_OK;
}

}  // namespace hdr
