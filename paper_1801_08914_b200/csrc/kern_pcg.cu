// Preconditioned conjugate gradients on the device for the reduced systems
// (SURVEY.md §8(f) f1): the reference's pcg (src/solvers.cpp:109-163) with all
// four of its preconditioners (driver.hpp:15): none, Jacobi
// (positive_inv_diag, :32-44), symmetric Gauss-Seidel (ssgs_setup, :60-72) and
// smoothed-aggregation AMG (amg_setup + V-cycle, kern_amg.cu), so a hybridized
// / condensed system is solved where H / S already live.  check_symmetric
// (:25-30) runs first, on the device.
//
// Per iteration: q = A p (the operator's SpMV), <p, q> (deterministic
// two-level reduction), one fused update x += a p, r -= a q (z = D^-1 r fused
// for Jacobi) with the partial sums of <r, r> (and <r, z>), the SGS / AMG
// application and <r, z> where the preconditioner is not diagonal, then
// p = z + b p.  Scalars come back to the host per iteration (the reference's
// control flow: breakdown checks, relative residual, beta).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <memory>
#include <string>

#include "amg.hpp"
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
    rr = fma(ri, ri, rr);
    if (z) {
      const double zi = dinv ? dinv[i] * ri : ri;
      z[i] = zi;
      rz = fma(ri, zi, rz);
    }
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
  if (precond < 0 || precond > 3)
    return fail(HDR_INVALID_ARGUMENT, "pcg: preconditioner must be 0 (none), 1 (jacobi), 2 (sgs) or 3 (amg)");
  const auto t0 = std::chrono::steady_clock::now();
  hdr_pcg_report report{};
  DBuf<double> r, z, p, q, dinv, part, two;
  // the matrix as a device CSR (int32 columns): symmetry check, SGS, AMG
  DCsr A;
  dcsr_from_device(n, n, ro, ci32, ci64, vals, A, st);
  {  // check_symmetric (solvers.cpp:25-30)
    double diff = 0.0, amax = 0.0;
    symmetry_gap(A, &diff, &amax, st);
    if (diff > 1e-10 * std::max(1e-300, amax))
      return fail(HDR_INVALID_ARGUMENT, "pcg: matrix not symmetric, max |A - A^T| = " + std::to_string(diff));
  }
  r.alloc(n);
  z.alloc(n);
  p.alloc(n);
  q.alloc(n);
  part.alloc(2 * kRB);
  two.alloc(2);
  const double* dv = nullptr;
  std::unique_ptr<AmgHier, void (*)(AmgHier*)> hier(nullptr, amg_destroy);
  SweepState sw;
  if (precond == 1 || precond == 2) {  // jacobi_setup / ssgs_setup: positive_inv_diag
    const int64_t bad = positive_inv_diag(A, dinv, st);
    if (bad >= 0) return fail(HDR_VALIDATION, "ZeroDiagonal: non-positive diagonal entry at row " + std::to_string(bad));
    if (precond == 1) dv = dinv.p;
  }
  if (precond == 2) {
    hier.reset(sweep_context(n, st));

  } else if (precond == 3) {  // amg_preconditioner with default AmgOptions
    hdr_amg_options o;
    hdr_amg_default_options(&o);
    DCsr copy;
    dcsr_from_device(n, n, A.ro.p, A.ci.p, nullptr, A.v.p, copy, st);
    hier.reset(amg_setup_device(std::move(copy), o, st));
  }
  const bool general = precond >= 2;  // z = M^-1 r is not fused into the update
  auto apply = [&](const double* in, double* out) -> hdr_status {
    if (precond == 2) sgs_apply_device(hier.get(), A, sw, sweep_scratch(hier.get()), in, out);
    else amg_apply_device(hier.get(), in, out);
    return amg_status(hier.get());
  };
  double h2[2];
  auto reduce = [&](const double* a1, const double* a2, const double* a3, const double* a4) {
    k_dot2_partial<<<kRB, kRT, 0, st>>>(n, a1, a2, a3, a4, part.p);
    k_sum2_final<<<1, kRT, 0, st>>>(part.p, two.p);
    count_launch(2);
    CK(cudaMemcpyAsync(h2, two.p, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  };
  auto spmv = [&](const double* in, double* out) { launch_spmv32(n, A.ro.p, A.ci.p, A.v.p, in, out, st, A.nnz); };
  // x = 0, r = b, z = M^-1 r, p = z
  k_pcg_init<<<kRB, kRT, 0, st>>>(n, b, x, r.p, dv, z.p, p.p);
  count_launch();
  if (general && n) {
    const hdr_status s = apply(r.p, z.p);
    if (s != HDR_OK) return s;
    CK(cudaMemcpyAsync(p.p, z.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, st));
  }
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
      k_pcg_update<<<kRB, kRT, 0, st>>>(n, alpha, p.p, q.p, x, r.p, dv, general ? nullptr : z.p, part.p);
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
      double rz_new = h2[1];
      if (general) {
        const hdr_status s = apply(r.p, z.p);
        if (s != HDR_OK) return s;
        reduce(r.p, z.p, nullptr, nullptr);
        rz_new = h2[0];
      }
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
