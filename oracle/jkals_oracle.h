/*
 * jkals_oracle.h — the ORACLE's own header (test infrastructure, NOT product code).
 *
 * Plain, slow, obviously-correct CPU implementation of JK-ALS (Psarras et al.,
 * arXiv 2112.03985, Alg. 2) and of the CP-ALS it calls
 * (Alg. 1). It shares no code, header, table or constant
 * with the CUDA path under paper_2112_03985_b200/ and never includes it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.
 *
 * Conventions (all 0-based here; the paper is 1-based):
 *   - tensors are dense, generalised column-major: element (i_0..i_{N-1}) is at
 *     sum_k i_k * prod_{m<k} I_m  (Eq. 3);
 *   - matrices (factors U_n, MTTKRP results M_n) are column-major I x R;
 *   - the sampled mode is mode 0 ("The samples are in the first mode").
 */
#ifndef JKALS_ORACLE_H
#define JKALS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_F_CONVERGED = 1, ORC_F_PINV = 2, ORC_F_NONFINITE = 4, ORC_F_BREAKDOWN = 8 };

/* Eq. 3: element idx -> (row i_n, column j) of T_(n). */
void orc_unfold_index(int N, const int64_t *dims, int n, const int64_t *idx,
                      int64_t *row, int64_t *col);
/* Explicit mode-n unfolding T_(n): I_n x prod_{m!=n} I_m, column-major. */
void orc_unfold(int N, const int64_t *dims, const double *T, int n, double *out);
/* Khatri-Rao product: column r of A (.) B is kron(A(:,r), B(:,r)).
 * A is I x R, B is J x R, out is (I*J) x R; out(i*J + j, r) = A(i,r) B(j,r). */
void orc_khatri_rao(const double *A, int64_t I, const double *B, int64_t J, int R, double *out);
/* MTTKRP by brute force over every tensor element (Alg. 1 line alg:als:mttkrp):
 * M(i_n, r) = sum_{all idx} T(idx) * prod_{m != n} U_m(i_m, r). */
void orc_mttkrp_brute(int N, const int64_t *dims, const double *T, const double *const *U,
                      int R, int n, double *M);
/* MTTKRP "reference path" (Eq. 1): explicit T_(n) times the explicit
 * descending-order KRP U_{N-1} (.) ... (.) U_{n+1} (.) U_{n-1} (.) ... (.) U_0. */
void orc_mttkrp_reference(int N, const int64_t *dims, const double *T, const double *const *U,
                          int R, int n, double *M);
/* Gramian U^T U (R x R, column-major) and Hadamard of Gramians over m != n. */
void orc_gramian(const double *U, int64_t I, int R, double *G);
void orc_hadamard_gramians(int N, const int64_t *dims, const double *const *U, int R, int n,
                           double *H);
/* U = M H^{-1} by textbook Cholesky H = L L^T (PAPER.md:232 with H SPD).
 * Returns 0 on success, 1 if a pivot is <= 0 or non-finite (U untouched). */
int orc_cholesky_solve(const double *H, int R, const double *M, int64_t I, double *U);
/* U = M H^+ via Jacobi symmetric eigendecomposition; eigenvalues <= rcond*lambda_max
 * are treated as zero ("pseudoinverse"). */
void orc_pinv_solve(const double *H, int R, const double *M, int64_t I, double rcond, double *U);
/* Squared Frobenius norm and mode-`mode` slice norms. */
double orc_norm_sq(int64_t n, const double *T);
void orc_slice_norms_sq(int N, const int64_t *dims, const double *T, int mode, double *out);
/* Alg. 2 line alg:jk:tensor_subsample: remove slice p of mode `mode`. */
void orc_remove_slice(int N, const int64_t *dims, const double *T, int mode, int64_t p, double *out);
/* Fast error (Alg. 1 line alg:als:error, sign corrected: SURVEY §8c A1):
 * e = ||T||^2 + sum(H_N .* (V^T V)) - 2 sum(V .* M_N), V = last-mode update (I x R). */
double orc_cp_error(double normT2, const double *H, const double *M, const double *V, int64_t I, int R);
/* Explicit ||T - [[U_0..U_{N-1}]] diag-lambda||^2 (test helper; lambda may be NULL = ones). */
double orc_explicit_residual(int N, const int64_t *dims, const double *T, const double *const *U,
                             const double *lambda, int R);

/* CP-ALS (Alg. 1) with the semantics fixed in SURVEY §8c:
 *  per sweep, for n = 0..N-1: M = MTTKRP (brute), H = Hadamard of Gramians,
 *  V = M H^{-1} (Cholesky, pinv fallback), lambda = column 2-norms of V, U_n = V / lambda;
 *  after mode N-1: e = fast error, fit = 1 - sqrt(max(e,0))/||T||; stop if tol > 0,
 *  it >= 2 and |fit - fit_prev| < tol.
 *  U: N column-major arrays (in: initial, out: fitted, unit-norm columns).
 *  lambda (R), err_hist (max_iters) outputs; returns ORC_F_* flags. */
int orc_cp_als(int N, const int64_t *dims, const double *T, int R, double *const *U,
               double *lambda, int max_iters, double tol, double *err_hist, int *iters_done);

/* JK-ALS (Alg. 2) over the left-out indices p_list (mode 0):
 * for each p: T_-p = remove slice p; U_0 = P_0 without row p; U_n = P_n (n >= 1);
 * cp_als; emit. Runs `nthreads` POSIX threads over p (each fit single-threaded).
 * Outputs, for q = 0..np-1:
 *   out_U[q*stride + off_n] : mode-n factor, column-major; mode 0 is (I_0-1) x R,
 *                             modes n >= 1 are I_n x R; off_n = R*sum_{m<n} rows_m,
 *                             stride = R*((I_0-1) + sum_{n>=1} I_n);
 *   out_lambda[q*R + r], out_err[q*max_iters + it], out_iters[q], out_flags[q]. */
int orc_jk_als(int N, const int64_t *dims, const double *T, int R, const double *const *P,
               const int64_t *p_list, int64_t np, int max_iters, double tol, int nthreads,
               double *out_U, double *out_lambda, double *out_err, int *out_iters, int *out_flags);

/* Delete-d jackknife: group g leaves out rows
 * [g*d, min(g*d + d, I_0)) of mode 0 (ceil(I_0/d) contiguous groups, the last one possibly
 * smaller); 1 <= d <= I_0/2. Same outputs as orc_jk_als, indexed by position
 * q in g_list; the mode-0 block of group q has I_0 - |group| rows (slot stride as for d = 1). */
int orc_jk_als_d(int N, const int64_t *dims, const double *T, int R, const double *const *P, int64_t d,
                 const int64_t *g_list, int64_t ng, int max_iters, double tol, int nthreads, double *out_U,
                 double *out_lambda, double *out_err, int *out_iters, int *out_flags);
void orc_remove_slices(int N, const int64_t *dims, const double *T, int mode, int64_t p0, int64_t p1,
                       double *out);

/* Alignment of one fitted submodel to the reference model (Alg. 2 alg:jk:perm_scale, PAPER.md:333;
 * scheme: DESIGN.md reading A12): congruence C(r,s) = prod_{n>=1} |cos_n(r,s)|,
 * sigma maximising sum_r C(r, sigma(r)) by exhaustive lexicographic search (R <= 10), signs so
 * that every cos_n(r, sigma(r)) >= 0 (n >= 1) with the compensating flip in mode 0, unit
 * columns in modes >= 1 and lam_r (and the removed norms) absorbed into mode 0.
 * rows[n]: rows of Uh[n] / out[n] (P[n] has rows[n] rows for n >= 1; P[0] unused);
 * lam may be NULL (ones). Outputs: out[n] column-major rows[n] x R, perm[r] = sigma(r),
 * sign[n*R + r] (n = 0 the compensating sign), cong[sigma(r)] = C(r, sigma(r)).
 * Returns -1 on bad arguments. */
int orc_align(int N, const int64_t *rows, int R, const double *const *Uh, const double *lam,
              const double *const *P, double *const *out, int *perm, int *sign, double *cong);

/* Jackknife mean and standard error over g submodels (alg:jk:std;
 * estimator reading SURVEY §8c A11): X is g blocks of len doubles;
 * std = sqrt(((g-1)/g) * sum_p (X_p - mean)^2). Returns -1 if g < 2. */
int orc_jackknife_stats(int64_t g, int64_t len, const double *X, double *mean, double *std);

#ifdef __cplusplus
}
#endif
#endif
