/* hdr_oracle.h — CPU oracle for the element-local hybridization hot path.
 *
 * TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline leg).  The product never links, loads or calls this library.
 *
 * Two things live here, both restated from the reference (/root/reference/proj):
 *  (1) a "port": the reference's production algorithm for the FE path,
 *      restated operation-for-operation so that its bits match the reference
 *      build in oracle/_ref (tests/test_oracle_pin.py checks that):
 *        build_reference        src/rt_space.cpp:180-314 (+ helpers :10-172)
 *        assemble_from_reference src/rt_space.cpp:345-366, dense_add dense.cpp:37-42
 *        local_dof_map          src/rt_space.cpp:383-393, mesh.cpp:94-135
 *        build_P / build_C      src/reduction.cpp:136-198, multiplier_base :88-98
 *        hybridize              src/reduction.cpp:262-354
 *        recover_hybrid         src/reduction.cpp:356-446
 *        static_condense        src/reduction.cpp:448-557
 *        recover_condensed      src/reduction.cpp:559-587
 *        lu_factor/lu_solve/compensated_residual/lu_solve_refined
 *                               src/dense.cpp:61-163
 *        from_triplets / spmv   src/csr.cpp:43-87
 *  (2) the value oracle of the parity contract: element-wise
 *      double-double (include/hdivred/dd.hpp, src/reference.cpp:11-48 and
 *      137-235) on the bit-identical A_T, assembled in double-double and
 *      rounded once.
 *
 * Interface: an opaque context holding named arrays; Python reads them by
 * name through ctypes (tests/oracle.py).
 */
#ifndef HDR_ORACLE_H
#define HDR_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hdo_ctx hdo_ctx;

/* dim 2|3, cells[3] (cells[2] ignored in 2D), RT order k in 0..3,
 * weighted: 0 = unit constraint rows (build_C weighted=false). */
hdo_ctx* hdo_create(int dim, const long long cells[3], int k, int weighted);
int hdo_set_h(hdo_ctx* c, const double h[3]); /* cell sizes (default 1 / cells) */
void hdo_destroy(hdo_ctx* ctx);

/* Scalar sizes: "dim","k","n","dpf","nint","ncells","nfaces","ndofs",
 * "face_dof_count","broken","m","nS". Returns -1 for unknown names. */
long long hdo_size(const hdo_ctx* ctx, const char* name);

/* Named arrays. hdo_count returns the element count (-1 if absent); hdo_get_d /
 * hdo_get_q copy it out (double / int64).  hdo_set_d stores/overwrites one
 * (used to feed alpha, beta, f_hat, lambda, x_b, or an explicit "a_hat"). */
long long hdo_count(const hdo_ctx* ctx, const char* name);
int hdo_get_d(const hdo_ctx* ctx, const char* name, double* out);
int hdo_get_q(const hdo_ctx* ctx, const char* name, long long* out);
int hdo_set_d(hdo_ctx* ctx, const char* name, const double* data, long long count);

/* Seeded synthetic inputs: coef = "uniform:a:b" |
 * "logu:lo:hi" | "checker:sig_lo:sig_hi".  Draw order: per cell alpha then
 * beta, f_hat (broken order), lambda (m), x_b (nS).  Sets alpha, beta, f_hat,
 * lambda, x_b. */
int hdo_gen_inputs(hdo_ctx* ctx, const char* coef, unsigned long long seed);

/* Stages.  what =
 *  "assemble"        a_hat (all blocks, ncells*n*n) from alpha/beta (needs ≤ 2 GB)
 *  "structure"       P, C (csr), dof_global/dof_sign, mult_base
 *  "port_hybridize"  H.* , g        (reference algorithm restated)
 *  "port_recover"    x_hat, x       (needs lambda; after port_hybridize)
 *  "port_condense"   S.*, f_s, master_globals
 *  "port_recover_condensed"  x_cond (needs x_b; after port_condense)
 *  "dd_hybridize"    H.values_dd, g_dd on the port's H pattern (needs port_hybridize)
 *  "dd_recover"      x_hat_dd, x_dd
 *  "dd_condense"     S.values_dd, f_s_dd (needs port_condense)
 *  "dd_recover_condensed" x_cond_dd
 *  "spmv_H"          H_lambda (y = H lambda, reference spmv order)
 *  "spmv_S"          S_x_b
 *  "pattern_H"       Hp.row_offsets / Hp.col_indices: hybridize's H pattern,
 *                    structure only (no values; full BASELINE sizes)
 *  "pattern_S"       Sp.*: static_condense's S pattern likewise
 * Returns 0 on success, nonzero error code (see hdo_last_error). */
int hdo_run(hdo_ctx* ctx, const char* what);

/* Element-wise double-double result for one cell, computed on A_T (from the
 * "a_hat" array if present, else assembled on the fly): the constrained local
 * dofs' multiplier rows (sorted, like constraint_slice), H_T (nr x nr, rounded
 * from DD), g_T (nr), and x_hat_T (n) given lambda.  Returns nr, or < 0. */
int hdo_dd_element(hdo_ctx* ctx, long long cell, long long* rows, double* h_t, double* g_t, double* x_hat_t);

/* A_T for one cell, assembled exactly as assemble_from_reference. */
int hdo_element_matrix(hdo_ctx* ctx, long long cell, double* a_t);

const char* hdo_last_error(const hdo_ctx* ctx);

/* Config 4 (RESTATEMENT — the reference has no curved / trilinear cells): the
 * reference box element mapped to a trilinear hexahedron by the contravariant
 * Piola transform, with the reference's nq^3 Gauss points.  h: the unperturbed
 * cell size (the box the reference element lives on), verts: 8 x 3 vertex
 * coordinates (v = vx + 2 vy + 4 vz).  divdiv, mass: n x n; div_form ((k+1)^3 x n)
 * and pressure_mass ((k+1)^3 squared) of the Piola-mapped pressures, or NULL.
 * With the context array "vertices" ((N+1)^3 x 3, set by hdo_gen_inputs'
 * ";perturb=f" or hdo_set_d) element matrices use this map. */
int hdo_piola_element(int k, const double h[3], const double* verts, int nq, double* divdiv, double* mass,
                      double* div_form, double* pressure_mass);

/* Reference element (restates build_reference): divdiv (n*n), mass (n*n),
 * face_moments (2*dim*dpf*n), unit_load (3*n). nq = quadrature points/axis. */
int hdo_build_reference(int dim, int k, const double h[3], int nq, double* divdiv, double* mass,
                        double* face_moments, double* unit_load);

#ifdef __cplusplus
}
#endif
#endif
