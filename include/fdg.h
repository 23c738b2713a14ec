/* include/fdg.h — C ABI of the B200 (sm_100a) fractional-diffusion PCG hot path.
 *
 * Drop-in boundary for the reference's C++ operator/plugin API
 * (/root/reference/proj/include/fdeopt/*.hpp).  Plain pointers and sizes only.
 * Each entry point names the reference interface it replaces (file:line).
 * Device pointers ("_dev") live on the context's device; "_host" variants
 * stage through pinned memory and are size-checked like the reference spans.
 *
 * Errors: every call returns fdg_status.  FDG_EINVAL replaces
 * std::invalid_argument, FDG_ENUMERIC replaces std::runtime_error (with the
 * reference's message text available from fdg_last_error()).
 * Thread model: handles are immutable after create except fdg_admm (single
 * writer, like AdmmDriver); each handle uses its context's CUDA stream.
 */
#ifndef FDG_H
#define FDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FDG_OK = 0,
  FDG_EINVAL = 1,       /* std::invalid_argument in the reference */
  FDG_ENUMERIC = 2,     /* std::runtime_error in the reference    */
  FDG_ECUDA = 3,        /* CUDA runtime failure / no device        */
  FDG_EUNSUPPORTED = 4, /* shape outside the compiled kernel set   */
  FDG_ENOMEM = 5
} fdg_status;

/* Sub-codes of FDG_ENUMERIC (fdg_last_numeric_code()). */
enum {
  FDG_NUM_NONE = 0,
  FDG_NUM_PD_LOSS = 1,            /* "pcg: operator lost positive definiteness" admm.cpp:144 */
  FDG_NUM_NONFINITE_RESIDUAL = 2, /* "pcg: non-finite residual" admm.cpp:151 */
  FDG_NUM_NONFINITE_ITERATE = 3,  /* "admm: non-finite iterate ..." admm.cpp:268 */
  FDG_NUM_STAGNATION = 4          /* "admm: PCG hit max_inner in 3 consecutive ..." admm.cpp:295 */
};

typedef struct fdg_ctx_s* fdg_ctx;
typedef struct fdg_op_s* fdg_op;
typedef struct fdg_pc_s* fdg_pc;
typedef struct fdg_admm_s* fdg_admm;

const char* fdg_last_error(void);
int fdg_last_numeric_code(void);
const char* fdg_version(void);

/* ------------------------------------------------------------- context */
/* stream == NULL: the context creates and owns a non-blocking stream. */
fdg_status fdg_ctx_create(int device, void* stream, fdg_ctx* out);
fdg_status fdg_ctx_destroy(fdg_ctx ctx);
void* fdg_ctx_stream(fdg_ctx ctx);
/* Number of kernels this library launched on the context so far. */
uint64_t fdg_ctx_launch_count(fdg_ctx ctx);
fdg_status fdg_ctx_synchronize(fdg_ctx ctx);

/* ------------------------------------------- setup (host, bit-identical) */
/* problem.cpp:35-45  frac_coeffs */
fdg_status fdg_frac_coeffs(double order, int count, double* out);
/* toeplitz.cpp:23-42 build_riesz (col == row) */
fdg_status fdg_build_riesz(double beta, int n, double h, double* col, double* row);
/* toeplitz.cpp:10-21 build_caputo */
fdg_status fdg_build_caputo(double alpha, int n, double h, double* col, double* row);
/* circulant.cpp:10-26 tchan + circulant_eigs: eigs is complex interleaved [2n] */
fdg_status fdg_tchan(int n, const double* col, const double* row, double* first_col, double* eigs);

/* ------------------------------------------------------------ operator */
/* ConstraintOperator(ToeplitzSpec1D caputo, riesz1, riesz2, psi, n)
 * toeplitz.hpp:34-35 / toeplitz.cpp:87-101, generalized to (n_t, n_x1, n_x2):
 *   B = psi (T_t (x) I (x) I - I (x) T_1 (x) I - I (x) I (x) T_2).
 * Factors are ToeplitzSpec1D (toeplitz.hpp:14-19): col[n], row[n].
 * A lower-bidiagonal time factor (implicit Euler) runs as a fused stencil;
 * any other time factor runs as an FFT pass along t. */
fdg_status fdg_op_create(fdg_ctx ctx, int n_t, int n_x1, int n_x2, const double* time_col,
                         const double* time_row, const double* x1_col, const double* x1_row,
                         const double* x2_col, const double* x2_row, double psi, fdg_op* out);
fdg_status fdg_op_destroy(fdg_op op);
size_t fdg_op_size(fdg_op op);
double fdg_op_psi(fdg_op op);
/* ConstraintOperator::apply(x, out, ws, adjoint)  toeplitz.hpp:55-56, toeplitz.cpp:174-182.
 * out is overwritten; x and out must not alias. */
fdg_status fdg_op_apply(fdg_op op, const double* x_dev, double* out_dev, int adjoint);
/* Host-span overload with the reference's size check (toeplitz.cpp:176-177). */
fdg_status fdg_op_apply_host(fdg_op op, const double* x, size_t n_x, double* out, size_t n_out,
                             int adjoint);

/* ------------------------------------------------------ preconditioner */
/* assemble_precond(op, rho, delta, gamma)  circulant.hpp:63-64, circulant.cpp:76-90 */
fdg_status fdg_pc_assemble(fdg_op op, double rho, double delta, double gamma, fdg_pc* out);
/* CirculantPreconditioner from the three 1-D eigenvalue vectors (complex
 * interleaved) of the level factors: lam_B = psi (lam_t - (lam_1 + lam_2))
 * (circulant.cpp:28-41 with lam_b in Kronecker-sum form). */
fdg_status fdg_pc_create(fdg_ctx ctx, int n_t, int n_x1, int n_x2, const double* lam_t,
                         const double* lam_x1, const double* lam_x2, double psi, double rho,
                         double delta, double gamma, fdg_pc* out);
fdg_status fdg_pc_destroy(fdg_pc pc);
/* CirculantPreconditioner::solve(r, z, ws)  circulant.hpp:43, circulant.cpp:49-67 */
fdg_status fdg_pc_solve(fdg_pc pc, const double* r_dev, double* z_dev);
fdg_status fdg_pc_solve_host(fdg_pc pc, const double* r, size_t n_r, double* z, size_t n_z);
/* lam_S materialized on the host (tests; circulant.hpp:47) */
fdg_status fdg_pc_lam_s_host(fdg_pc pc, double* out);
/* 2-level spatial T. Chan preconditioner of A = I (x) T_x + T_y (x) I applied per
 * time slice (BASELINE C1 operator microbenchmark; the reference ships only the
 * 3-level ADMM form, circulant.cpp:28-90): z = F^-1 (F r / (lam_x1[i] + lam_x2[j])),
 * any level sizes <= 1024 (Bluestein).  Eigenvalues complex interleaved and real
 * (symmetric factors).  Solved through fdg_pc_solve / fdg_pc_solve_host. */
fdg_status fdg_pc2_create(fdg_ctx ctx, int n_t, int n_x1, int n_x2, const double* lam_x1,
                          const double* lam_x2, fdg_pc* out);
/* Same, with lam from the T. Chan circulants (circulant.cpp:10-26) of the
 * operator's spatial factors. */
fdg_status fdg_pc2_assemble(fdg_op op, fdg_pc* out);

/* ---------------------------------------------------------------- ADMM */
/* AdmmConfig (admm.hpp:14-26) + ProblemSpec bounds/gamma (problem.hpp:15-26). */
typedef struct {
  double gamma, rho, delta;
  double y_lo, y_hi, u_lo, u_hi; /* +-INFINITY for unbounded */
  double tol_primal;
  int max_outer, max_inner;
  double inner_tol_floor, inner_tol_factor;
  double fixed_krylov_tol; /* > 0: fixed Krylov tolerance (BASELINE); <= 0: admm.cpp:216-217 rule */
  int warm_start;
} fdg_admm_desc;

/* IterRecord (admm.hpp:34-40) plus device timings. */
typedef struct {
  int iter;
  double r_eq, r_y, r_u;
  double dual_inf;
  int inner_iters;
  double inner_tol;
  int converged;
  int pcg_converged;
  double pcg_rel_residual;
  double pcg_ms;  /* CUDA-event time inside pcg */
  double step_ms; /* CUDA-event time of the whole step */
} fdg_iter_record;

/* PcgResult (admm.hpp:86-90) */
typedef struct {
  int iterations;
  int converged;
  double rel_residual;
  double ms; /* CUDA-event time */
} fdg_pcg_result;

/* AdmmDriver(spec, cfg, op, pc) admm.hpp:128-150 / make_admm_work admm.cpp:52-79.
 * ybar_host: desired state (AdmmWork::ybar, admm.hpp:66); NULL = zeros. */
fdg_status fdg_admm_create(fdg_op op, fdg_pc pc, const fdg_admm_desc* desc, const double* ybar_host,
                           fdg_admm* out);
fdg_status fdg_admm_destroy(fdg_admm adm);
/* AdmmDriver::step  admm.cpp:245-277 */
fdg_status fdg_admm_step(fdg_admm adm, fdg_iter_record* rec);
int fdg_admm_converged(fdg_admm adm);
int fdg_admm_stagnations(fdg_admm adm);

/* Fields of AdmmState / AdmmWork (admm.hpp:28-32, 59-71). */
enum {
  FDG_F_Y = 0, FDG_F_V, FDG_F_ZY, FDG_F_ZV, FDG_F_P, FDG_F_WY, FDG_F_WV,
  FDG_F_YBAR, FDG_F_DIAGJ, FDG_F_DIAGJ2, FDG_F_M2, FDG_F_A2INV, FDG_F_BY
};
fdg_status fdg_admm_get(fdg_admm adm, int field, double* host_out);
fdg_status fdg_admm_set(fdg_admm adm, int field, const double* host_in);
/* Device pointer of a state field (y, v, z_y, z_v, p, w_y, w_v, ybar, By). */
fdg_status fdg_admm_field_ptr(fdg_admm adm, int field, double** dev);

/* Test accessor: PCG work vector (0 r, 1 z, 2 p, 3 u, 4 w, 5 vp; N doubles)
 * or, with which = -1, the device scalar block (32 doubles). */
fdg_status fdg_admm_debug_get(fdg_admm adm, int which, double* host_out);

/* apply_S(work, x, out, ws)  admm.hpp:79-80, admm.cpp:87-98 */
fdg_status fdg_admm_apply_S(fdg_admm adm, const double* x_dev, double* out_dev);
/* build_rhs(work, state, rhs, ws) admm.cpp:100-119; r_cache_dev may be NULL */
fdg_status fdg_admm_build_rhs(fdg_admm adm, double* rhs_dev, double* r_cache_dev);
/* pcg(apply_S, pc.solve, rhs, x, tol, max_inner)  admm.hpp:97-98, admm.cpp:121-169.
 * x is in/out (x == 0 selects the reference's r = rhs start). */
fdg_status fdg_admm_pcg(fdg_admm adm, const double* rhs_dev, double* x_dev, double tol,
                        int max_inner, fdg_pcg_result* res);
/* The same with host buffers: H2D of rhs and x, solve, D2H of x (e2e path). */
fdg_status fdg_admm_pcg_host(fdg_admm adm, const double* rhs, double* x, double tol, int max_inner,
                             fdg_pcg_result* res);
/* dual_infeasibility(work, state, ws) admm.cpp:221-233 */
fdg_status fdg_admm_dual_inf(fdg_admm adm, double* out);
/* Objective 1/2 (y-ybar)^T J (y-ybar) + 1/2 v^T J2 v */
fdg_status fdg_admm_objective(fdg_admm adm, double* out);

/* Bench/roofline hook: average CUDA-event time (ms) of each kernel of one
 * PCG iteration over `reps` back-to-back launches, and its algorithmic HBM
 * bytes.  9 entries: K1 row (direction update p = z + b p fused with
 * the B row pass), K2 x1 col (S mid), K3 row (B^T + r update), P1 x2
 * Hartley, P2 x1 Hartley, P3 t filter, P4 x1 Hartley, P5 x2 Hartley (+ r.z),
 * X x += a p (once per solve; per iteration it rides in K1).
 * Clobbers the PCG scratch vectors. */
fdg_status fdg_admm_profile_passes(fdg_admm adm, int reps, double* ms, double* bytes);

/* Size threshold of the graph-driven PCG iterations (no reference
 * counterpart; a tuning knob of this library): solves with N <= nmax run
 * their steady-state iterations inside one CUDA graph launch (a WHILE node
 * over a two-iteration body, stopped by the device control step) instead of
 * host-sequenced launches.  Same kernels, same order, same results.  nmax < 0
 * leaves it unchanged; *previous (optional) receives the old value.
 * Default 2^21, or the FDG_PCG_GRAPH_NMAX environment variable. */
fdg_status fdg_set_pcg_graph_nmax(long long nmax, long long* previous);

/* --------------------------------------------------- synthetic inputs */
/* std::mt19937_64(seed) + std::normal_distribution<double> in layout order
 * (the reference tests' generator, test_toeplitz.cpp:15-20). */
fdg_status fdg_randn(uint64_t seed, size_t count, double* out);

#ifdef __cplusplus
}
#endif

#endif /* FDG_H */
