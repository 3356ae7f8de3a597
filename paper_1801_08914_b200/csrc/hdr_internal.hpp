// Internal host-side declarations shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace hdr {

// Reference element of RT_k on one box (restated build_reference).
struct RefElement {
  int dim = 3, k = 0, n = 0, dpf = 1, nint = 0;
  std::vector<double> divdiv, mass, face_moments;  // n*n, n*n, 2*dim*dpf*n
  std::vector<double> unit_load;                   // 3*n: (e_c, phi_i) per component c
  std::vector<int> comp;                           // vector component of each local dof
  int npr = 1;                                     // pressure dofs (k+1)^dim
  std::vector<double> div_form;                    // npr*n: (q_r, div phi_j) (RtSpace::ref_div_form)
  // basis at the nq^dim Gauss points (x fastest), for mapped (Piola) cells:
  // bq_val[(p*n + j)*3 + c] = phi_j,c(s_p) on the unit box coordinates s, bq_div[p*n + j]
  // = sum_a d phi_j,a / d s_a / h_a, bq_w[p] = product of the 1D weights, qs = 1D points
  int nq = 0;
  std::vector<double> bq_val, bq_div, bq_w, qs;
};
RefElement build_reference_element(int dim, int k, const double h[3]);

// Fixed factors of the structured (Woodbury + Neumann) element solve; see
// DESIGN.md "Structured element solve".  With D = ref_divdiv, M = ref_mass
// (both exact fp64 inputs) and r = rank D = (k+1)^dim:
//   X (n x r), lambda (r): M-orthonormal generalized eigenpairs of D x = l M x
//                          over range(D)  (X^T M X = I up to rounding)
//   E  = D - Ms X diag(lambda) X^T Ms      (exactly, then rounded once; tiny)
//   N0 = Ms^-1 - X X^T                     (PSD "divergence-free" inverse)
// Per cell, with A_T = fl(fl(alpha D) + fl(beta M)) and s_j = beta/(beta+alpha lambda_j):
//   (M, D are symmetric only up to rounding: Ms = (M+M^T)/2 exactly, Ma = (M-M^T)/2)
//   A0 = beta Ms + alpha Ms X diag(lambda) X^T Ms,  A_T = A0 + Delta_T,
//   Delta_T = alpha E + beta Ma + delta_T (delta_T = exact rounding error of the combine),
//   A0^-1 = (N0 + X diag(s) X^T) / beta      (no cancellation)
//   A_T^-1 = sum_p (-A0^-1 Delta_T)^p A0^-1   (Neumann; ratio <= rho*alpha/beta)
struct Structured {
  int n = 0, r = 0;
  std::vector<double> X, lambda, E, N0, Minv, Ma;  // n*r, r, n*n, n*n, n*n, n*n (row-major)
  double rho = 0.0;                            // Neumann ratio bound per unit alpha/beta
  double e_rel = 0.0;                          // max|E| / max|D| (diagnostic)
  double orth = 0.0;                           // max|X^T M X - I| (diagnostic)
  bool block_diag = false;                     // M (hence Minv) block-diagonal by component
};
// Returns false (with *err set) if the reference matrices do not have the
// expected structure (D PSD of rank (k+1)^dim numerically, M SPD).
bool precompute_structured(const RefElement& re, int expected_rank, Structured* out, std::string* err);

// Mesh numbering (src/mesh.cpp:13-135), shared by host and device code.
struct MeshDims {
  int dim;
  int64_t N[3];
  int64_t nfaces_axis[3];
  int64_t face_off[3];
  int64_t nfaces;
  int64_t ncells;
};
MeshDims make_mesh_dims(int dim, const int64_t cells[3]);

}  // namespace hdr
