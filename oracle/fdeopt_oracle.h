/* oracle/fdeopt_oracle.h — TEST INFRASTRUCTURE (CPU checker; never the product).
 *
 * Plain-C restatement of the reference hot path generalized from cubes
 * (n_t = n_x1 = n_x2, /root/reference/proj/include/fdeopt/problem.hpp:28-42)
 * to arbitrary (n_t, n_x1, n_x2) shapes, so that BASELINE configs C1, C3, C4
 * have a CPU oracle.  Every function cites the reference file:line it
 * restates.  Validated against the unchanged reference (oracle/_ref) on cubes
 * by tests/test_oracle_cpu.py.  Layout: x[(k*n1 + i)*n2 + j], time outermost.
 */
#ifndef FDEOPT_ORACLE_H
#define FDEOPT_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);
/* worker threads for the fibre / line loops (default 1; results do not
 * depend on the count: every fibre writes its own elements) */
void or_set_threads(int t);
int or_get_threads(void);

/* problem.cpp:35-45 */
int or_frac_coeffs(double order, int count, double* out);
/* toeplitz.cpp:23-42 (symmetric: row == col) */
int or_build_riesz(double beta, int n, double h, double* col);
/* toeplitz.cpp:10-21 */
int or_build_caputo(double alpha, int n, double h, double* col, double* row);
/* toeplitz.cpp:46-58: n+1 complex bins (re,im interleaved) of the 2n embedding */
int or_embed_symbol(int n, const double* col, const double* row, int transpose, double* sym);
/* circulant.cpp:10-20 + fft.cpp:111-130: T. Chan first column and eigenvalues */
int or_tchan(int n, const double* col, const double* row, double* first_col, double* eigs);

typedef struct or_op or_op;
/* toeplitz.cpp:87-101 generalized: factors of sizes nt, n1, n2 */
or_op* or_op_create(int nt, int n1, int n2, const double* tcol, const double* trow,
                    const double* c1, const double* r1, const double* c2, const double* r2,
                    double psi);
void or_op_destroy(or_op* op);
/* toeplitz.cpp:124-182 generalized (mode-wise 2n circulant embedding by FFT) */
int or_op_apply(const or_op* op, const double* x, double* out, int adjoint);
/* the same operator by direct O(n^2) fibre sums (independent algorithm) */
int or_op_apply_direct(const or_op* op, const double* x, double* out, int adjoint);

typedef struct or_pc or_pc;
/* circulant.cpp:76-90 + 28-41 generalized (lambda_S materialized, N doubles) */
or_pc* or_pc_assemble(const or_op* op, double rho, double delta, double gamma);
void or_pc_destroy(or_pc* pc);
/* circulant.cpp:49-67 generalized: complex 3-D FFT (nt x n1 x n2) */
int or_pc_solve(const or_pc* pc, const double* r, double* z);
int or_pc_lam_s(const or_pc* pc, double* out);
/* 1-D eigenvalue vectors (complex interleaved) used by assemble_precond */
int or_pc_eigs(const or_pc* pc, double* lam_t, double* lam_1, double* lam_2);

typedef struct or_admm or_admm;
/* admm.cpp:52-79 generalized; ybar may be NULL (zeros); fixed_tol > 0 fixes
 * the Krylov tolerance, else the dynamic rule admm.cpp:216-217. */
or_admm* or_admm_create(const or_op* op, const or_pc* pc, double gamma, double rho, double delta,
                        double y_lo, double y_hi, double u_lo, double u_hi, double tol_primal,
                        int max_inner, double inner_tol_floor, double inner_tol_factor,
                        double fixed_tol, int warm_start, const double* ybar);
void or_admm_destroy(or_admm* a);
size_t or_admm_size(const or_admm* a);
/* fields: 0 y,1 v,2 z_y,3 z_v,4 p,5 w_y,6 w_v,7 ybar,8 diag_j,9 diag_j2,10 m2,11 a2_inv,12 By */
int or_admm_get(const or_admm* a, int field, double* out);
int or_admm_set(or_admm* a, int field, const double* in);
/* admm.cpp:87-98 */
int or_admm_apply_S(or_admm* a, const double* x, double* out);
/* admm.cpp:100-119 */
int or_admm_build_rhs(or_admm* a, double* rhs, double* r_cache);
/* admm.cpp:121-169 on S with the circulant preconditioner; result {it, conv, relres} */
int or_admm_pcg(or_admm* a, const double* rhs, double* x, double tol, int max_inner,
                double* result);
/* admm.cpp:245-277; rec as ref_admm_step: {iter,r_eq,r_y,r_u,dual_inf,inner,inner_tol,conv} */
int or_admm_step(or_admm* a, double* rec);
/* admm.cpp:221-233 */
int or_admm_dual_inf(or_admm* a, double* out);
/* SURVEY.md §8 a19 */
int or_admm_objective(const or_admm* a, double* out);

#ifdef __cplusplus
}
#endif

#endif
