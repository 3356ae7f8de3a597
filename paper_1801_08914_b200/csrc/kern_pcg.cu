// Preconditioned conjugate gradients on the device for the reduced systems
// (SURVEY.md §8(f) f1): the reference's pcg (src/solvers.cpp:109-163) with its
// "none" and Jacobi preconditioners (positive_inv_diag, :32-44), so a
// hybridized / condensed system can be solved where H / S already live.
//
// Per iteration: q = A p (the operator's SpMV), <p, q> (deterministic
// two-level reduction), one fused update x += a p, r -= a q, z = D^-1 r with
// the partial sums of <r, r> and <r, z>, then p = z + b p.  Two scalars come
// back to the host per iteration (the reference's control flow: breakdown
// checks, relative residual, beta).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <string>

#include "capi_util.hpp"
#include "kernels.hpp"

namespace hdr {
namespace {

constexpr int kRB = 1024;  // reduction blocks
constexpr int kRT = 256;

__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
  sh[threadIdx.x] = a;
  sh[kRT + threadIdx.x] = b;
  __syncthreads();
  for (int o = kRT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sh[threadIdx.x] += sh[threadIdx.x + o];
      sh[kRT + threadIdx.x] += sh[kRT + threadIdx.x + o];
    }
    __syncthreads();
  }
  a = sh[0];
  b = sh[kRT];
}

__global__ void k_dot2_partial(int64_t n, const double* x, const double* y, const double* u, const double* v,
                               double* part) {
  __shared__ double sh[2 * kRT];
  double s = 0.0, t = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRT) + threadIdx.x; i < n; i += static_cast<int64_t>(kRB) * kRT) {
    s = fma(x[i], y[i], s);
    if (u) t = fma(u[i], v[i], t);
  }
  block_sum2(s, t, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    part[kRB + blockIdx.x] = t;
  }
}

__global__ void k_sum2_final(const double* part, double* out) {
  __shared__ double sh[2 * kRT];
  double s = 0.0, t = 0.0;
  for (int i = threadIdx.x; i < kRB; i += kRT) {
    s += part[i];
    t += part[kRB + i];
  }
  block_sum2(s, t, sh);
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = t;
  }
}

// x += a p; r -= a q; z = dinv .* r (or r); partial sums of <r, r>, <r, z>
__global__ void k_pcg_update(int64_t n, double alpha, const double* p, const double* q, double* x, double* r,
                             const double* dinv, double* z, double* part) {
  __shared__ double sh[2 * kRT];
  double rr = 0.0, rz = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRT) + threadIdx.x; i < n; i += static_cast<int64_t>(kRB) * kRT) {
    x[i] = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    const double zi = dinv ? dinv[i] * ri : ri;
    z[i] = zi;
    rr = fma(ri, ri, rr);
    rz = fma(ri, zi, rz);
  }
  block_sum2(rr, rz, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = rr;
    part[kRB + blockIdx.x] = rz;
  }
}

__global__ void k_pcg_dir(int64_t n, double beta, const double* z, double* p) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRT) + threadIdx.x; i < n; i += static_cast<int64_t>(kRB) * kRT)
    p[i] = z[i] + beta * p[i];
}

// Jacobi: 1 / a_ii, flag (bad row + 1) where a_ii <= 0 or absent
template <class IDX>
__global__ void k_inv_diag(int64_t n, const int64_t* ro, const IDX* ci, const double* v, double* dinv,
                           unsigned long long* bad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (int64_t k = ro[i]; k < ro[i + 1]; ++k)
    if (static_cast<int64_t>(ci[k]) == i) d = v[k];
  if (!(d > 0.0)) atomicMin(bad, static_cast<unsigned long long>(i));
  dinv[i] = 1.0 / d;
}

__global__ void k_pcg_init(int64_t n, const double* b, double* x, double* r, const double* dinv, double* z,
                           double* p) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRT) + threadIdx.x; i < n; i += static_cast<int64_t>(kRB) * kRT) {
    x[i] = 0.0;
    r[i] = b[i];
    const double zi = dinv ? dinv[i] * b[i] : b[i];
    z[i] = zi;
    p[i] = zi;
  }
}

}  // namespace

hdr_status pcg_device(int64_t n, const int64_t* ro, const int32_t* ci32, const int64_t* ci64, const double* vals,
                      const double* b, double* x, double rtol, int64_t maxit, int precond, double* hist,
                      hdr_pcg_report* rep, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  hdr_pcg_report report{};
  DBuf<double> r, z, p, q, dinv, part, two;
  DBuf<unsigned long long> bad;
  r.alloc(n);
  z.alloc(n);
  p.alloc(n);
  q.alloc(n);
  part.alloc(2 * kRB);
  two.alloc(2);
  const double* dv = nullptr;
  if (precond == 1) {  // jacobi_setup (solvers.cpp:165): positive_inv_diag
    dinv.alloc(n);
    bad.alloc(1);
    CK(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    if (n > 0) {
      if (ci32) k_inv_diag<int32_t><<<g, 256, 0, st>>>(n, ro, ci32, vals, dinv.p, bad.p);
      else k_inv_diag<int64_t><<<g, 256, 0, st>>>(n, ro, ci64, vals, dinv.p, bad.p);
      count_launch();
    }
    unsigned long long hb = 0;
    CK(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hb != ~0ull) return fail(HDR_VALIDATION, "ZeroDiagonal: non-positive diagonal entry at row " + std::to_string(hb));
    dv = dinv.p;
  } else if (precond != 0) {
    return fail(HDR_INVALID_ARGUMENT, "pcg: preconditioner must be 0 (none) or 1 (jacobi)");
  }
  double h2[2];
  auto reduce = [&](const double* a1, const double* a2, const double* a3, const double* a4) {
    k_dot2_partial<<<kRB, kRT, 0, st>>>(n, a1, a2, a3, a4, part.p);
    k_sum2_final<<<1, kRT, 0, st>>>(part.p, two.p);
    count_launch(2);
    CK(cudaMemcpyAsync(h2, two.p, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  };
  auto spmv = [&](const double* in, double* out) {
    if (ci32) launch_spmv32(n, ro, ci32, vals, in, out, st);
    else launch_spmv64(n, ro, ci64, vals, in, out, st);
  };
  // x = 0, r = b, z = M^-1 r, p = z
  k_pcg_init<<<kRB, kRT, 0, st>>>(n, b, x, r.p, dv, z.p, p.p);
  count_launch();
  reduce(b, b, r.p, z.p);
  const double bnorm = std::sqrt(h2[0]);
  double rz = h2[1];
  if (hist) hist[0] = bnorm == 0.0 ? 0.0 : 1.0;
  if (bnorm == 0.0) {
    report.converged = 1;
  } else {
    if (!(rz > 0.0)) return fail(HDR_VALIDATION, "IndefinitePreconditioner: pcg: <z, r> <= 0 at setup");
    for (int64_t it = 1; it <= maxit; ++it) {
      spmv(p.p, q.p);
      reduce(p.p, q.p, nullptr, nullptr);
      const double pq = h2[0];
      if (!(pq > 0.0)) return fail(HDR_VALIDATION, "pcg: <p, Ap> <= 0, matrix is not positive definite");
      const double alpha = rz / pq;
      k_pcg_update<<<kRB, kRT, 0, st>>>(n, alpha, p.p, q.p, x, r.p, dv, z.p, part.p);
      k_sum2_final<<<1, kRT, 0, st>>>(part.p, two.p);
      count_launch(2);
      CK(cudaMemcpyAsync(h2, two.p, 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      const double rel = std::sqrt(h2[0]) / bnorm;
      if (hist) hist[it] = rel;
      report.iterations = it;
      report.final_relative_residual = rel;
      if (rel <= rtol) {
        report.converged = 1;
        break;
      }
      const double rz_new = h2[1];
      if (!(rz_new > 0.0))
        return fail(HDR_VALIDATION, "IndefinitePreconditioner: pcg: <z, r> <= 0 at iteration " + std::to_string(it));
      k_pcg_dir<<<kRB, kRT, 0, st>>>(n, rz_new / rz, z.p, p.p);
      count_launch();
      rz = rz_new;
    }
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  report.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (rep) *rep = report;
  return HDR_OK;
}

}  // namespace hdr
