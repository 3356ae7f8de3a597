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
