/*
 * jkals_oracle.c — ORACLE (test infrastructure; not part of the product path).
 *
 * A plain, slow, obviously-correct CPU implementation of what the JK-CALS hot
 * path computes: JK-ALS (Psarras, Karlsson, Bro, Bientinesi, arXiv 2112.03985,
 * Alg. 2), i.e. textbook CP-ALS (Alg. 1)
 * run independently on every explicitly sliced tensor T_-p. JK-CALS (Alg. 3)
 * reaches exactly this result ("it is possible to compute
 * M_n ... without referencing the reduced tensor"), so this is the definition
 * the GPU path is compared against, element by element.
 *
 * Rules this file follows (task ③): plain loops in fp64, no BLAS, no blocking,
 * no fusion, no reordering beyond the definitions; each function cites the
 * passage it follows. Readings of ambiguous passages are SURVEY.md §8c A1-A19
 * and are listed in DESIGN.md. Shares NO code with paper_2112_03985_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it.
 *
 * Build: gcc -O2 -std=c99 -fPIC -shared -o liborc.so jkals_oracle.c -lpthread -lm
 *        (no -ffast-math: IEEE round-to-nearest as in SURVEY §8c A18).
 */
#define _POSIX_C_SOURCE 200809L
#include "jkals_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static int64_t prod_dims(int N, const int64_t *dims) {
  int64_t p = 1;
  for (int k = 0; k < N; ++k) p *= dims[k];
  return p;
}

/* Eq. 3: j = sum_{k != n} i_k * prod_{m < k, m != n} I_m (0-based). */
void orc_unfold_index(int N, const int64_t *dims, int n, const int64_t *idx, int64_t *row,
                      int64_t *col) {
  int64_t j = 0;
  for (int k = 0; k < N; ++k) {
    if (k == n) continue;
    int64_t stride = 1;
    for (int m = 0; m < k; ++m)
      if (m != n) stride *= dims[m];
    j += idx[k] * stride;
  }
  *row = idx[n];
  *col = j;
}

/* Advance a column-major multi-index by one element (first index fastest). */
static void next_index(int N, const int64_t *dims, int64_t *idx) {
  for (int k = 0; k < N; ++k) {
    if (++idx[k] < dims[k]) return;
    idx[k] = 0;
  }
}

/* Unfolding T_(n): columns are the mode-n fibres, placed by Eq. 3. */
void orc_unfold(int N, const int64_t *dims, const double *T, int n, double *out) {
  int64_t total = prod_dims(N, dims);
  int64_t idx[16] = {0}; /* N <= 16 */
  for (int64_t lin = 0; lin < total; ++lin) {
    int64_t row, col;
    orc_unfold_index(N, dims, n, idx, &row, &col);
    out[row + dims[n] * col] = T[lin];
    next_index(N, dims, idx);
  }
}

/* Khatri-Rao product: column-wise Kronecker product. */
void orc_khatri_rao(const double *A, int64_t I, const double *B, int64_t J, int R, double *out) {
  for (int r = 0; r < R; ++r)
    for (int64_t i = 0; i < I; ++i)
      for (int64_t j = 0; j < J; ++j)
        out[(i * J + j) + I * J * r] = A[i + I * r] * B[j + J * r];
}

/* MTTKRP by definition (Alg. 1 alg:als:mttkrp): every element T(idx)
 * contributes T(idx) * prod_{m != n} U_m(i_m, r) to M(i_n, r). The KRP entry is formed
 * in the descending mode order of Eq. 1. */
void orc_mttkrp_brute(int N, const int64_t *dims, const double *T, const double *const *U, int R,
                      int n, double *M) {
  int64_t total = prod_dims(N, dims);
  int64_t In = dims[n];
  memset(M, 0, sizeof(double) * (size_t)(In * R));
  int64_t idx[16] = {0}; /* N <= 16 */
  for (int64_t lin = 0; lin < total; ++lin) {
    double t = T[lin];
    for (int r = 0; r < R; ++r) {
      double krp = 1.0;
      for (int m = N - 1; m >= 0; --m)
        if (m != n) krp *= U[m][idx[m] + dims[m] * r];
      M[idx[n] + In * r] += t * krp;
    }
    next_index(N, dims, idx);
  }
}

/* MTTKRP reference path (Eq. 1): M = T_(n) (U_{N-1} (.) ... (.) U_0),
 * mode n skipped, explicit unfolding and explicit KRP, then a plain triple loop. */
void orc_mttkrp_reference(int N, const int64_t *dims, const double *T, const double *const *U,
                          int R, int n, double *M) {
  int64_t total = prod_dims(N, dims);
  int64_t In = dims[n], J = total / In;
  double *Tn = malloc(sizeof(double) * (size_t)total);
  orc_unfold(N, dims, T, n, Tn);
  /* KRP chain: start with the lowest mode != n, then K <- U_m (.) K for ascending m,
   * which yields U_{N-1} (.) ... (.) U_0 with mode 0 varying fastest (matches Eq. 3). */
  double *K = NULL;
  int64_t rows = 0;
  for (int m = 0; m < N; ++m) {
    if (m == n) continue;
    if (!K) {
      rows = dims[m];
      K = malloc(sizeof(double) * (size_t)(rows * R));
      memcpy(K, U[m], sizeof(double) * (size_t)(rows * R));
    } else {
      double *K2 = malloc(sizeof(double) * (size_t)(rows * dims[m] * R));
      orc_khatri_rao(U[m], dims[m], K, rows, R, K2);
      free(K);
      K = K2;
      rows *= dims[m];
    }
  }
  for (int64_t i = 0; i < In; ++i)
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
      for (int64_t j = 0; j < J; ++j) s += Tn[i + In * j] * K[j + J * r];
      M[i + In * r] = s;
    }
  free(K);
  free(Tn);
}

/* Gramian U^T U. */
void orc_gramian(const double *U, int64_t I, int R, double *G) {
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      double s = 0.0;
      for (int64_t i = 0; i < I; ++i) s += U[i + I * a] * U[i + I * b];
      G[a + R * b] = s;
    }
}

/* Hadamard product of Gramians over i != n (Alg. 1 alg:als:hadamard). */
void orc_hadamard_gramians(int N, const int64_t *dims, const double *const *U, int R, int n,
                           double *H) {
  double *G = malloc(sizeof(double) * (size_t)(R * R));
  for (int k = 0; k < R * R; ++k) H[k] = 1.0;
  for (int m = 0; m < N; ++m) {
    if (m == n) continue;
    orc_gramian(U[m], dims[m], R, G);
    for (int k = 0; k < R * R; ++k) H[k] *= G[k];
  }
  free(G);
}

/* U = M H^{-1} (Alg. 1 alg:als:update; H is SPD in the generic case,
 * SURVEY §8c A3): textbook Cholesky H = L L^T without pivoting, then for each row
 * m of M solve H u = m^T by forward (L y = m) and back (L^T u = y) substitution. */
int orc_cholesky_solve(const double *H, int R, const double *M, int64_t I, double *U) {
  double *L = calloc((size_t)(R * R), sizeof(double));
  for (int j = 0; j < R; ++j) {
    double s = H[j + R * j];
    for (int k = 0; k < j; ++k) s -= L[j + R * k] * L[j + R * k];
    if (!(s > 0.0) || !isfinite(s)) {
      free(L);
      return 1;
    }
    L[j + R * j] = sqrt(s);
    for (int i = j + 1; i < R; ++i) {
      double t = H[i + R * j];
      for (int k = 0; k < j; ++k) t -= L[i + R * k] * L[j + R * k];
      L[i + R * j] = t / L[j + R * j];
    }
  }
  double *y = malloc(sizeof(double) * (size_t)R);
  for (int64_t row = 0; row < I; ++row) {
    for (int i = 0; i < R; ++i) {
      double t = M[row + I * i];
      for (int k = 0; k < i; ++k) t -= L[i + R * k] * y[k];
      y[i] = t / L[i + R * i];
    }
    for (int i = R - 1; i >= 0; --i) {
      double t = y[i];
      for (int k = i + 1; k < R; ++k) t -= L[k + R * i] * U[row + I * k];
      U[row + I * i] = t / L[i + R * i];
    }
  }
  free(y);
  free(L);
  return 0;
}

/* U = M H^+ ("pseudoinverse of H"): cyclic Jacobi eigendecomposition
 * H = Q diag(w) Q^T (Golub & Van Loan, symmetric Schur rotations), then
 * H^+ = Q diag(w_i > rcond*w_max ? 1/w_i : 0) Q^T. */
void orc_pinv_solve(const double *H, int R, const double *M, int64_t I, double rcond, double *U) {
  double *A = malloc(sizeof(double) * (size_t)(R * R));
  double *Q = calloc((size_t)(R * R), sizeof(double));
  double *Hp = calloc((size_t)(R * R), sizeof(double));
  memcpy(A, H, sizeof(double) * (size_t)(R * R));
  for (int i = 0; i < R; ++i) Q[i + R * i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        tot += A[i + R * j] * A[i + R * j];
        if (i != j) off += A[i + R * j] * A[i + R * j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < R - 1; ++p)
      for (int q = p + 1; q < R; ++q) {
        double apq = A[p + R * q];
        if (apq == 0.0) continue;
        double theta = (A[q + R * q] - A[p + R * p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        /* A <- J^T A J with J the (p,q) rotation [c s; -s c]. */
        for (int k = 0; k < R; ++k) { /* columns p, q */
          double akp = A[k + R * p], akq = A[k + R * q];
          A[k + R * p] = c * akp - s * akq;
          A[k + R * q] = s * akp + c * akq;
        }
        for (int k = 0; k < R; ++k) { /* rows p, q */
          double apk = A[p + R * k], aqk = A[q + R * k];
          A[p + R * k] = c * apk - s * aqk;
          A[q + R * k] = s * apk + c * aqk;
        }
        for (int k = 0; k < R; ++k) {
          double qkp = Q[k + R * p], qkq = Q[k + R * q];
          Q[k + R * p] = c * qkp - s * qkq;
          Q[k + R * q] = s * qkp + c * qkq;
        }
      }
  }
  double wmax = 0.0;
  for (int i = 0; i < R; ++i)
    if (A[i + R * i] > wmax) wmax = A[i + R * i];
  for (int i = 0; i < R; ++i) {
    double w = A[i + R * i];
    if (!(w > rcond * wmax) || w <= 0.0) continue;
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) Hp[a + R * b] += Q[a + R * i] * Q[b + R * i] / w;
  }
  for (int64_t row = 0; row < I; ++row)
    for (int b = 0; b < R; ++b) {
      double s = 0.0;
      for (int a = 0; a < R; ++a) s += M[row + I * a] * Hp[a + R * b];
      U[row + I * b] = s;
    }
  free(A);
  free(Q);
  free(Hp);
}

double orc_norm_sq(int64_t n, const double *T) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += T[i] * T[i];
  return s;
}

void orc_slice_norms_sq(int N, const int64_t *dims, const double *T, int mode, double *out) {
  int64_t total = prod_dims(N, dims);
  int64_t idx[16] = {0}; /* N <= 16 */
  for (int64_t p = 0; p < dims[mode]; ++p) out[p] = 0.0;
  for (int64_t lin = 0; lin < total; ++lin) {
    out[idx[mode]] += T[lin] * T[lin];
    next_index(N, dims, idx);
  }
}

/* delete-d variant: drop every element with p0 <= i_mode < p1. */
void orc_remove_slices(int N, const int64_t *dims, const double *T, int mode, int64_t p0, int64_t p1,
                       double *out) {
  int64_t total = prod_dims(N, dims), w = 0;
  int64_t idx[16] = {0}; /* N <= 16 */
  for (int64_t lin = 0; lin < total; ++lin) {
    if (idx[mode] < p0 || idx[mode] >= p1) out[w++] = T[lin];
    next_index(N, dims, idx);
  }
}

/* Alg. 2 alg:jk:tensor_subsample: drop every element with i_mode == p,
 * keeping the remaining elements in their column-major order. */
void orc_remove_slice(int N, const int64_t *dims, const double *T, int mode, int64_t p,
                      double *out) {
  int64_t total = prod_dims(N, dims), w = 0;
  int64_t idx[16] = {0}; /* N <= 16 */
  for (int64_t lin = 0; lin < total; ++lin) {
    if (idx[mode] != p) out[w++] = T[lin];
    next_index(N, dims, idx);
  }
}

/* Alg. 1 alg:als:error with the sign of the model-norm term
 * corrected to "+": e = ||T||^2 + sum(H .* V^T V) - 2 sum(V .* M). */
double orc_cp_error(double normT2, const double *H, const double *M, const double *V, int64_t I,
                    int R) {
  double quad = 0.0, cross = 0.0;
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      double g = 0.0;
      for (int64_t i = 0; i < I; ++i) g += V[i + I * a] * V[i + I * b];
      quad += H[a + R * b] * g;
    }
  for (int r = 0; r < R; ++r)
    for (int64_t i = 0; i < I; ++i) cross += V[i + I * r] * M[i + I * r];
  return normT2 + quad - 2.0 * cross;
}

double orc_explicit_residual(int N, const int64_t *dims, const double *T, const double *const *U,
                             const double *lambda, int R) {
  int64_t total = prod_dims(N, dims);
  int64_t idx[16] = {0}; /* N <= 16 */
  double res = 0.0;
  for (int64_t lin = 0; lin < total; ++lin) {
    double model = 0.0;
    for (int r = 0; r < R; ++r) {
      double t = lambda ? lambda[r] : 1.0;
      for (int m = 0; m < N; ++m) t *= U[m][idx[m] + dims[m] * r];
      model += t;
    }
    double d = T[lin] - model;
    res += d * d;
    next_index(N, dims, idx);
  }
  return res;
}

/* CP-ALS, Alg. 1, semantics per SURVEY §8c (see header). */
int orc_cp_als(int N, const int64_t *dims, const double *T, int R, double *const *U,
               double *lambda, int max_iters, double tol, double *err_hist, int *iters_done) {
  int64_t total = prod_dims(N, dims), maxI = 0;
  for (int k = 0; k < N; ++k)
    if (dims[k] > maxI) maxI = dims[k];
  double normT2 = orc_norm_sq(total, T);
  double *M = malloc(sizeof(double) * (size_t)(maxI * R));
  double *V = malloc(sizeof(double) * (size_t)(maxI * R));
  double *H = malloc(sizeof(double) * (size_t)(R * R));
  int flags = 0, it;
  double fit_prev = 0.0;
  for (it = 1; it <= max_iters; ++it) {
    for (int n = 0; n < N; ++n) {
      int64_t In = dims[n];
      orc_mttkrp_brute(N, dims, T, (const double *const *)U, R, n, M);   /* alg:als:mttkrp */
      orc_hadamard_gramians(N, dims, (const double *const *)U, R, n, H); /* alg:als:hadamard */
      if (orc_cholesky_solve(H, R, M, In, V)) {                          /* alg:als:update */
        orc_pinv_solve(H, R, M, In, 1e-12, V);
        flags |= ORC_F_PINV;
      }
      for (int r = 0; r < R; ++r) { /* column normalisation */
        double s = 0.0;
        for (int64_t i = 0; i < In; ++i) s += V[i + In * r] * V[i + In * r];
        double lam = sqrt(s);
        lambda[r] = lam;
        for (int64_t i = 0; i < In; ++i) U[n][i + In * r] = lam > 0.0 ? V[i + In * r] / lam : V[i + In * r];
      }
    }
    /* alg:als:error with the last mode's H, M and (un-normalised) update V */
    double e = orc_cp_error(normT2, H, M, V, dims[N - 1], R);
    err_hist[it - 1] = e;
    if (!isfinite(e)) {
      flags |= ORC_F_NONFINITE;
      break;
    }
    if (e < -1e-9 * normT2) flags |= ORC_F_BREAKDOWN;
    double fit = normT2 > 0.0 ? 1.0 - sqrt(e > 0.0 ? e : 0.0) / sqrt(normT2) : 0.0;
    if (tol > 0.0 && it >= 2 && fabs(fit - fit_prev) < tol) {
      flags |= ORC_F_CONVERGED;
      break;
    }
    fit_prev = fit;
  }
  *iters_done = it > max_iters ? max_iters : it;
  free(M);
  free(V);
  free(H);
  return flags;
}

/* ---- JK-ALS (Alg. 2) with a plain pthread pool over the left-out indices ---- */
typedef struct {
  int N;
  const int64_t *dims;
  const double *T;
  int R;
  const double *const *P;
  const int64_t *p_list;  /* group indices g: rows [g*d, min(g*d + d, I_0)) of mode 0 */
  int64_t np;
  int64_t d;
  int max_iters;
  double tol;
  double *out_U, *out_lambda, *out_err;
  int *out_iters, *out_flags;
  int64_t next;
  pthread_mutex_t lock;
} jk_job;

static void jk_one(jk_job *J, int64_t q) {
  int N = J->N, R = J->R;
  const int64_t *dims = J->dims;
  const int64_t p0 = J->p_list[q] * J->d;
  const int64_t p1 = (p0 + J->d < dims[0]) ? p0 + J->d : dims[0];  /* removed rows [p0, p1) */
  int64_t sub_dims[16];
  for (int k = 0; k < N; ++k) sub_dims[k] = dims[k];
  sub_dims[0] = dims[0] - (p1 - p0);
  int64_t sub_total = prod_dims(N, sub_dims);
  double *Tp = malloc(sizeof(double) * (size_t)sub_total);
  orc_remove_slices(N, dims, J->T, 0, p0, p1, Tp); /* alg:jk:tensor_subsample (delete-d) */
  double *U[16];
  int64_t stride = R * (dims[0] - 1); /* fixed slot size: mode 0 of any group has <= I_0 - 1 rows */
  for (int k = 1; k < N; ++k) stride += sub_dims[k] * R;
  double *outq = J->out_U + q * stride;
  int64_t off = 0;
  for (int k = 0; k < N; ++k) {
    U[k] = outq + off;
    off += sub_dims[k] * R;
  }
  /* alg:jk:model_subsample: U_0 = P_0 with the group's rows removed; U_n = P_n */
  for (int r = 0; r < R; ++r) {
    int64_t w = 0;
    for (int64_t i = 0; i < dims[0]; ++i)
      if (i < p0 || i >= p1) U[0][w++ + sub_dims[0] * r] = J->P[0][i + dims[0] * r];
  }
  for (int k = 1; k < N; ++k) memcpy(U[k], J->P[k], sizeof(double) * (size_t)(dims[k] * R));
  int iters = 0;
  int flags = orc_cp_als(N, sub_dims, Tp, R, U, J->out_lambda + q * R, J->max_iters, J->tol,
                         J->out_err + q * J->max_iters, &iters); /* alg:jk:fitting */
  J->out_iters[q] = iters;
  J->out_flags[q] = flags;
  free(Tp);
}

static void *jk_worker(void *arg) {
  jk_job *J = arg;
  for (;;) {
    pthread_mutex_lock(&J->lock);
    int64_t q = J->next++;
    pthread_mutex_unlock(&J->lock);
    if (q >= J->np) break;
    jk_one(J, q);
  }
  return NULL;
}

int orc_jk_als(int N, const int64_t *dims, const double *T, int R, const double *const *P,
               const int64_t *p_list, int64_t np, int max_iters, double tol, int nthreads,
               double *out_U, double *out_lambda, double *out_err, int *out_iters, int *out_flags) {
  return orc_jk_als_d(N, dims, T, R, P, 1, p_list, np, max_iters, tol, nthreads, out_U, out_lambda, out_err,
                      out_iters, out_flags);
}

int orc_jk_als_d(int N, const int64_t *dims, const double *T, int R, const double *const *P, int64_t d,
                 const int64_t *g_list, int64_t ng, int max_iters, double tol, int nthreads, double *out_U,
                 double *out_lambda, double *out_err, int *out_iters, int *out_flags) {
  if (N < 2 || N > 16 || dims[0] < 2 || R < 1 || max_iters < 1 || d < 1 || 2 * d > dims[0]) return -1;
  const int64_t ngroups = (dims[0] + d - 1) / d;
  for (int64_t q = 0; q < ng; ++q)
    if (g_list[q] < 0 || g_list[q] >= ngroups) return -1;
  for (int64_t q = 0; q < ng * max_iters; ++q) out_err[q] = NAN;
  int64_t np = ng;
  const int64_t *p_list = g_list;
  jk_job J = {N, dims, T, R, P, p_list, np, d, max_iters, tol, out_U, out_lambda, out_err,
              out_iters, out_flags, 0, PTHREAD_MUTEX_INITIALIZER};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > np) nthreads = (int)(np > 0 ? np : 1);
  pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, jk_worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  return 0;
}

/* Alg. 2 alg:jk:std: jackknife standard error, SURVEY §8c A11. */
int orc_jackknife_stats(int64_t g, int64_t len, const double *X, double *mean, double *std) {
  if (g < 2) return -1;
  for (int64_t e = 0; e < len; ++e) {
    double s = 0.0;
    for (int64_t p = 0; p < g; ++p) s += X[p * len + e];
    double mu = s / (double)g, ss = 0.0;
    for (int64_t p = 0; p < g; ++p) ss += (X[p * len + e] - mu) * (X[p * len + e] - mu);
    mean[e] = mu;
    std[e] = sqrt(((double)(g - 1) / (double)g) * ss);
  }
  return 0;
}

/* ------------------------------------------------------------------ alignment (Alg. 2 line 6)
 * "permutation and scale adjustment of P_hat_{-p}"; the paper defers the scheme
 * to its citation, so this follows the reading in DESIGN.md:
 *   cos_n(r,s) = <Uh_n(:,r), P_n(:,s)> / (||Uh_n(:,r)|| ||P_n(:,s)||)   (0 if a norm is 0), n >= 1
 *   C(r,s)     = prod_{n>=1} |cos_n(r,s)|
 *   sigma      = the permutation maximising sum_r C(r, sigma(r)); exhaustive search in
 *                lexicographic order, the first strict maximum wins (lowest-index tie-break)
 *   sign_n(r)  = -1 if cos_n(r, sigma(r)) < 0 else +1 (n >= 1); sign_0(r) = prod_{n>=1} sign_n(r)
 *   out_n(:, sigma(r)) = sign_n(r) Uh_n(:,r) / ||Uh_n(:,r)||                        (n >= 1)
 *   out_0(:, sigma(r)) = sign_0(r) lam_r prod_{n>=1} ||Uh_n(:,r)|| Uh_0(:,r)
 * so the model's tensor is unchanged and every non-sampled column has unit norm. */
static double col_dot(const double *a, const double *b, int64_t I) {
  double s = 0.0;
  for (int64_t i = 0; i < I; ++i) s += a[i] * b[i];
  return s;
}

static int next_perm(int *a, int n) { /* lexicographic successor; 0 when a is the last */
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return 0;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int t = a[i]; a[i] = a[j]; a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
  return 1;
}

int orc_align(int N, const int64_t *rows, int R, const double *const *Uh, const double *lam,
              const double *const *P, double *const *out, int *perm, int *sign, double *cong) {
  if (N < 2 || R < 1 || R > 10) return -1;
  double *cosv = malloc(sizeof(double) * (size_t)(N * R * R));
  double *C = malloc(sizeof(double) * (size_t)(R * R));
  double *nu = malloc(sizeof(double) * (size_t)(N * R));
  for (int n = 1; n < N; ++n)
    for (int r = 0; r < R; ++r) {
      const double *u = Uh[n] + rows[n] * r;
      nu[n * R + r] = sqrt(col_dot(u, u, rows[n]));
      for (int s = 0; s < R; ++s) {
        const double *p = P[n] + rows[n] * s;
        double np = sqrt(col_dot(p, p, rows[n]));
        double den = nu[n * R + r] * np;
        cosv[(n * R + r) * R + s] = den > 0.0 ? col_dot(u, p, rows[n]) / den : 0.0;
      }
    }
  for (int r = 0; r < R; ++r)
    for (int s = 0; s < R; ++s) {
      double c = 1.0;
      for (int n = 1; n < N; ++n) c *= fabs(cosv[(n * R + r) * R + s]);
      C[r * R + s] = c;
    }
  int a[16], best[16];
  for (int r = 0; r < R; ++r) a[r] = best[r] = r;
  double bestv = -1.0;
  do {
    double v = 0.0;
    for (int r = 0; r < R; ++r) v += C[r * R + a[r]];
    if (v > bestv) {
      bestv = v;
      memcpy(best, a, sizeof(int) * (size_t)R);
    }
  } while (next_perm(a, R));
  for (int r = 0; r < R; ++r) {
    const int s = best[r];
    perm[r] = s;
    cong[s] = C[r * R + s];
    int s0 = 1;
    double scale = lam ? lam[r] : 1.0;
    for (int n = 1; n < N; ++n) {
      int sg = cosv[(n * R + r) * R + s] < 0.0 ? -1 : 1;
      sign[n * R + r] = sg;
      s0 *= sg;
      double nr = nu[n * R + r];
      scale *= nr;
      for (int64_t i = 0; i < rows[n]; ++i)
        out[n][i + rows[n] * s] = nr > 0.0 ? sg * Uh[n][i + rows[n] * r] / nr : Uh[n][i + rows[n] * r];
    }
    sign[r] = s0;
    for (int64_t i = 0; i < rows[0]; ++i) out[0][i + rows[0] * s] = s0 * scale * Uh[0][i + rows[0] * r];
  }
  free(cosv);
  free(C);
  free(nu);
  return 0;
}
