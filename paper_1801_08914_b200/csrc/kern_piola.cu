// Config 4: element matrices of perturbed trilinear hexahedra (contravariant
// Piola map of the reference box element, oracle/hdr_oracle.c
// hdo_piola_element — a restatement: the reference has affine boxes only).
//
//   M_ij = sum_p w_p (det J0^2 / det J_p) (K_p phi_i) . (K_p phi_j),  K = J J0^-1
//   D_ij = sum_p w_p (det J0^2 / det J_p) divh_i divh_j
//   A_T  = fl(fl(alpha D) + fl(beta M))            (rt_space.cpp:356-357)
//
// One CTA per cell (persistent).  The points are processed in chunks: the
// chunk's mapped basis (K phi, divh, weight) is formed in shared memory, then
// every thread accumulates its fixed set of (i, j) entries over the chunk in
// registers.  The arithmetic follows the oracle operation for operation with
// explicit round-to-nearest intrinsics (no FMA contraction), so the device A_T
// is bit-identical to the restatement's (tests/test_piola_gpu.py).
#include "hdr_device.cuh"
#include "kernels.hpp"

namespace hdr {

namespace {

constexpr int kPT = 512;  // threads per CTA
constexpr int kCP = 8;    // points per chunk

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

template <int EPT>
__global__ void __launch_bounds__(kPT, 1) k_piola_assemble(PiolaArgs P) {
  extern __shared__ __align__(16) double sm[];
  const int n = P.n, nq = P.nq, np = nq * nq * nq;
  double* psi = sm;                      // kCP x n x 3
  double* dvh = psi + kCP * n * 3;       // kCP x n
  double* wc = dvh + kCP * n;            // kCP
  double* Jm = wc + kCP;                 // kCP x 9
  const int nn = n * n;
  const int64_t NV0 = P.N[0] + 1, NV1 = P.N[1] + 1;
  for (int64_t cell = blockIdx.x; cell < P.ncells; cell += gridDim.x) {
    const int64_t cx = cell % P.N[0], cy = (cell / P.N[0]) % P.N[1], cz = cell / (P.N[0] * P.N[1]);
    for (int pass0 = 0; pass0 < nn; pass0 += EPT * kPT) {
      double accD[EPT], accM[EPT];
#pragma unroll
      for (int t = 0; t < EPT; ++t) accD[t] = accM[t] = 0.0;
      for (int p0 = 0; p0 < np; p0 += kCP) {
        const int cp = min(kCP, np - p0);
        // Jacobians and weights of the chunk's points
        if (threadIdx.x < cp) {
          const int p = p0 + threadIdx.x;
          const int ix = p % nq, iy = (p / nq) % nq, iz = p / (nq * nq);
          const double s[3] = {P.qs[ix], P.qs[iy], P.qs[iz]};
          double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          for (int v = 0; v < 8; ++v) {
            const int b0 = v & 1, b1 = (v >> 1) & 1, b2 = (v >> 2) & 1;
            const double f0 = b0 ? s[0] : sub(1.0, s[0]), f1 = b1 ? s[1] : sub(1.0, s[1]),
                         f2 = b2 ? s[2] : sub(1.0, s[2]);
            const double d0 = b0 ? 1.0 : -1.0, d1 = b1 ? 1.0 : -1.0, d2 = b2 ? 1.0 : -1.0;
            const double dN[3] = {mul(mul(d0, f1), f2), mul(mul(f0, d1), f2), mul(mul(f0, f1), d2)};
            const int64_t g = (cx + b0) + NV0 * ((cy + b1) + NV1 * (cz + b2));
            for (int c = 0; c < 3; ++c) {
              const double xv = P.verts[3 * g + c];
              for (int a = 0; a < 3; ++a) J[c][a] = add(J[c][a], mul(xv, dN[a]));
            }
          }
          const double det = add(sub(mul(J[0][0], sub(mul(J[1][1], J[2][2]), mul(J[1][2], J[2][1]))),
                                     mul(J[0][1], sub(mul(J[1][0], J[2][2]), mul(J[1][2], J[2][0])))),
                                 mul(J[0][2], sub(mul(J[1][0], J[2][1]), mul(J[1][1], J[2][0]))));
          wc[threadIdx.x] = mul(P.bq_w[p], __ddiv_rn(mul(P.det0, P.det0), det));
          for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) Jm[threadIdx.x * 9 + c * 3 + a] = __ddiv_rn(J[c][a], P.h[a]);
        }
        __syncthreads();
        // mapped basis of the chunk: psi = K phi (K = J / h columnwise), divh
        for (int t = threadIdx.x; t < cp * n; t += kPT) {
          const int pl = t / n, j = t % n, p = p0 + pl;
          const double* bv = P.bq_val + (static_cast<int64_t>(p) * n + j) * 3;
          const double* K = Jm + pl * 9;
          for (int c = 0; c < 3; ++c)
            psi[(pl * n + j) * 3 + c] = add(add(mul(K[c * 3 + 0], bv[0]), mul(K[c * 3 + 1], bv[1])), mul(K[c * 3 + 2], bv[2]));
          dvh[pl * n + j] = P.bq_div[static_cast<int64_t>(p) * n + j];
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < EPT; ++t) {
          const int ent = pass0 + t * kPT + threadIdx.x;
          if (ent < nn) {
            const int i = ent / n, j = ent % n;
            for (int pl = 0; pl < cp; ++pl) {
              const double w = wc[pl];
              const double* pi = psi + (pl * n + i) * 3;
              const double* pj = psi + (pl * n + j) * 3;
              accD[t] = add(accD[t], mul(mul(w, dvh[pl * n + i]), dvh[pl * n + j]));
              accM[t] = add(accM[t], mul(w, add(add(mul(pi[0], pj[0]), mul(pi[1], pj[1])), mul(pi[2], pj[2]))));
            }
          }
        }
        __syncthreads();
      }
      const double al = P.alpha[cell], be = P.beta[cell];
      double* out = P.ablk + cell * static_cast<int64_t>(nn);
#pragma unroll
      for (int t = 0; t < EPT; ++t) {
        const int ent = pass0 + t * kPT + threadIdx.x;
        if (ent < nn) {
          if (P.dm) {
            P.dm[cell * 2 * static_cast<int64_t>(nn) + ent] = accD[t];
            P.dm[cell * 2 * static_cast<int64_t>(nn) + nn + ent] = accM[t];
          }
          out[ent] = add(mul(al, accD[t]), mul(be, accM[t]));
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// GEMM form (the production kernel when the basis is component-separable, as
// the reference's is: every phi_j has exactly one nonzero component c_j).
// With the dofs sorted by component (perm), K_p = J_p diag(1/h), Q_p = K_p^T K_p,
// w'_p = w_p det0^2 / det J_p:
//   M_ij = sum_p (w'_p Q_p[c_i][c_j]) phi_i(p) phi_j(p),  D_ij = sum_p w'_p g_i(p) g_j(p)
// i.e. two K = np GEMMs per cell whose per-point coefficient depends only on the
// component pair of the 4 x 4 register tile.  The constant tables phi / g
// (np x n, sorted order) stay in shared memory for all cells of the CTA; the
// lower-triangle tiles are computed once and mirrored (A_T exactly symmetric);
// A_T = fl(fl(alpha D) + fl(beta M)) (rt_space.cpp:356-357) is staged in shared
// memory in the natural dof order and stored with coalesced rows.
constexpr int kGT = 384;  // threads per CTA (RT2: 378 lower-triangle tiles)

__device__ __forceinline__ int sym3(int a, int b) {  // (a, b) -> 0..5 for (00, 01, 02, 11, 12, 22)
  const int lo = a < b ? a : b, hi = a < b ? b : a;
  return lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
}

__global__ void __launch_bounds__(kGT, 1) k_piola_gemm(PiolaArgs P, const double* __restrict__ tphi,
                                                       const double* __restrict__ tdiv, const int* __restrict__ perm) {
  extern __shared__ __align__(16) double sm[];
  const int n = P.n, nq = P.nq, np = nq * nq * nq, nc3 = n / 3;
  double* ph = sm;               // np x n
  double* gd = ph + np * n;      // np x n
  double* cf = gd + np * n;      // np x 8: w', w' Q (00, 01, 02, 11, 12, 22), pad
  double* ao = cf + np * 8;      // n x n staging of A_T (natural order)
  int* pm = reinterpret_cast<int*>(ao + n * n);
  for (int t = threadIdx.x; t < np * n; t += kGT) {
    ph[t] = tphi[t];
    gd[t] = tdiv[t];
  }
  for (int t = threadIdx.x; t < n; t += kGT) pm[t] = perm[t];
  const int nb = n / 4, ntiles = nb * (nb + 1) / 2;
  const int64_t NV0 = P.N[0] + 1, NV1 = P.N[1] + 1;
  for (int64_t cell = blockIdx.x; cell < P.ncells; cell += gridDim.x) {
    const int64_t cx = cell % P.N[0], cy = (cell / P.N[0]) % P.N[1], cz = cell / (P.N[0] * P.N[1]);
    for (int p = threadIdx.x; p < np; p += kGT) {
      const int ix = p % nq, iy = (p / nq) % nq, iz = p / (nq * nq);
      const double sx = P.qs[ix], sy = P.qs[iy], sz = P.qs[iz];
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int b0 = v & 1, b1 = (v >> 1) & 1, b2 = (v >> 2) & 1;
        const double f0 = b0 ? sx : 1.0 - sx, f1 = b1 ? sy : 1.0 - sy, f2 = b2 ? sz : 1.0 - sz;
        const double dN0 = (b0 ? 1.0 : -1.0) * f1 * f2, dN1 = (b1 ? 1.0 : -1.0) * f0 * f2,
                     dN2 = (b2 ? 1.0 : -1.0) * f0 * f1;
        const int64_t g = (cx + b0) + NV0 * ((cy + b1) + NV1 * (cz + b2));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double xv = P.verts[3 * g + c];
          J[c][0] = fma(xv, dN0, J[c][0]);
          J[c][1] = fma(xv, dN1, J[c][1]);
          J[c][2] = fma(xv, dN2, J[c][2]);
        }
      }
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      const double w = P.bq_w[p] * (P.det0 * P.det0) / det;
      double K[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int a = 0; a < 3; ++a) K[c][a] = J[c][a] / P.h[a];
      auto q = [&](int a, int b) { return K[0][a] * K[0][b] + K[1][a] * K[1][b] + K[2][a] * K[2][b]; };
      double* c7 = cf + p * 8;
      c7[0] = w;
      c7[1] = w * q(0, 0);
      c7[2] = w * q(0, 1);
      c7[3] = w * q(0, 2);
      c7[4] = w * q(1, 1);
      c7[5] = w * q(1, 2);
      c7[6] = w * q(2, 2);
    }
    __syncthreads();
    const double al = P.alpha[cell], be = P.beta[cell];
    for (int tile = threadIdx.x; tile < ntiles; tile += kGT) {
      int ti = static_cast<int>((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
      while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
      while (ti * (ti + 1) / 2 > tile) --ti;
      const int tj = tile - ti * (ti + 1) / 2;  // tj <= ti
      const int r0 = 4 * ti, c0 = 4 * tj;
      const int cm = 1 + sym3(r0 / nc3, c0 / nc3);
      double aD[4][4], aM[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) aD[r][c] = aM[r][c] = 0.0;
#pragma unroll 2
      for (int p = 0; p < np; ++p) {
        const double wD = cf[p * 8], wM = cf[p * 8 + cm];
        const double2* prow = reinterpret_cast<const double2*>(ph + p * n);
        const double2* grow = reinterpret_cast<const double2*>(gd + p * n);
        const double2 fr0 = prow[r0 / 2], fr1 = prow[r0 / 2 + 1], gr0 = grow[r0 / 2], gr1 = grow[r0 / 2 + 1];
        const double2 fc0 = prow[c0 / 2], fc1 = prow[c0 / 2 + 1], gc0 = grow[c0 / 2], gc1 = grow[c0 / 2 + 1];
        const double fi[4] = {fr0.x, fr0.y, fr1.x, fr1.y}, gi[4] = {gr0.x, gr0.y, gr1.x, gr1.y};
        const double fj[4] = {wM * fc0.x, wM * fc0.y, wM * fc1.x, wM * fc1.y};
        const double gj[4] = {wD * gc0.x, wD * gc0.y, wD * gc1.x, wD * gc1.y};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            aD[r][c] = fma(gi[r], gj[c], aD[r][c]);
            aM[r][c] = fma(fi[r], fj[c], aM[r][c]);
          }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int i = pm[r0 + r], j = pm[c0 + c];
          const double v = add(mul(al, aD[r][c]), mul(be, aM[r][c]));
          if (ti != tj || r >= c) {
            ao[i * n + j] = v;
            ao[j * n + i] = v;
          }
        }
    }
    __syncthreads();
    double* out = P.ablk + cell * static_cast<int64_t>(n) * n;
    for (int t = threadIdx.x; t < n * n / 2; t += kGT)
      reinterpret_cast<double2*>(out)[t] = reinterpret_cast<const double2*>(ao)[t];
    __syncthreads();
  }
}

__global__ void k_affine_assemble(int64_t ncells, int n, const double* dm, const double* alpha, const double* beta,
                                  double* out) {
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < ncells * nn;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = t / nn, ij = t - e * nn;
    out[t] = add(mul(alpha[e], dm[ij]), mul(beta[e], dm[nn + ij]));
  }
}

}  // namespace

void launch_affine_assemble(int64_t ncells, int n, const double* dm, const double* alpha, const double* beta,
                            double* out, cudaStream_t st) {
  k_affine_assemble<<<148 * 8, 256, 0, st>>>(ncells, n, dm, alpha, beta, out);
  count_launch();
}

size_t piola_smem_bytes(int n) { return static_cast<size_t>(kCP * n * 4 + kCP * 10) * 8; }

size_t piola_gemm_smem_bytes(int n, int np) {
  return static_cast<size_t>(2 * np * n + 8 * np + n * n) * 8 + static_cast<size_t>(n) * 4;
}

bool piola_gemm_supported(int n, int np) {
  const int nb = n / 4;
  return n % 12 == 0 && nb * (nb + 1) / 2 <= 4 * kGT && piola_gemm_smem_bytes(n, np) <= 227 * 1024;
}

void launch_piola_gemm(const PiolaArgs& a, const double* tphi, const double* tdiv, const int* perm, int grid,
                       cudaStream_t st) {
  const size_t smem = piola_gemm_smem_bytes(a.n, a.nq * a.nq * a.nq);
  cudaFuncSetAttribute(k_piola_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_piola_gemm<<<grid, kGT, smem, st>>>(a, tphi, tdiv, perm);
  count_launch();
}

void launch_piola_assemble(const PiolaArgs& a, int grid, cudaStream_t st) {
  const size_t smem = piola_smem_bytes(a.n);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, kPT, smem, st>>>(a);
  };
  const int nn = a.n * a.n;
  if (nn <= 4 * kPT) go(k_piola_assemble<4>);
  else go(k_piola_assemble<24>);
  count_launch();
}

}  // namespace hdr
