/*
 * jkcals.h — C ABI of the B200-native JK-CALS hot path.
 *
 * JK-CALS (Psarras, Karlsson, Bro, Bientinesi, "Accelerating jackknife resampling for the
 * Canonical Polyadic Decomposition", arXiv 2112.03985), Alg. 3: all
 * leave-one-out (LOO) CP submodels of a dense tensor T are fitted concurrently by ALS
 * against the SAME full tensor. Submodel p's mode-0 factor carries a zero row at index p
 * (Alg. 3 alg:cals_jk:multifactor0; §4.1 Case II), so one
 * fused MTTKRP per mode (alg:cals_jk:mttkrp) serves every submodel; it is
 * followed per submodel by the Hadamard of Gramians (alg:cals_jk:hadamard),
 * the update U = M H^{-1} (alg:cals_jk:update), the re-zeroing of row p when
 * n = 0 (alg:cals_jk:multifactor), and the submodel error with ||T_-p||^2
 * (alg:cals_jk:error).
 *
 * Conventions
 *   - 0-based indices; the sampled mode is mode 0 ("The samples are in the first mode",
 *     PAPER.md:499). Submodel p leaves out slice p of mode 0.
 *   - Tensors are dense FP64, generalised column-major (first index fastest), i.e. the
 *     element (i_0..i_{N-1}) is at sum_k i_k prod_{m<k} I_m (Eq. 3).
 *   - Host factor matrices crossing this ABI are column-major, rows x rank.
 *   - Per-iteration semantics: after each update the
 *     columns are normalised to unit 2-norm (lambda kept); Cholesky solve with a Jacobi
 *     pseudoinverse fallback; error e = ||T_-p||^2 + sum(H .* V^T V) - 2 sum(V .* M)
 *     (Alg. 3 error line with its sign corrected); fit = 1 - sqrt(max(e,0))/||T_-p||;
 *     with tol > 0 a submodel stops once |fit - fit_prev| < tol (from its 2nd sweep).
 *
 * Ownership and threading
 *   - Host inputs are only read during the call; host outputs are caller buffers.
 *   - The caller owns the device WORKSPACE (e.g. a torch uint8 tensor) and the CUDA stream;
 *     the tensor is copied into the workspace at create. destroy() frees only host state,
 *     CUDA graphs and events, never the workspace.
 *   - A handle is single-owner and not thread-safe. All device work is enqueued on the
 *     handle's stream; calls that return host data synchronise that stream.
 *
 * Errors: every call returns a jkcals_status; jkcals_last_error() describes the last
 * failure on a handle. Numerical failures are PER SUBMODEL and never fail a call: a
 * failed Cholesky falls back to the pseudoinverse (JKCALS_F_PINV_FALLBACK); a non-finite
 * error freezes the submodel (JKCALS_F_NONFINITE); a negative error below -1e-9 ||T_-p||^2
 * sets JKCALS_F_BREAKDOWN.
 */
#ifndef JKCALS_H
#define JKCALS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct jkcals_s *jkcals_t;

typedef enum {
  JKCALS_OK = 0,
  JKCALS_E_ARG = -1,       /* invalid argument / precondition */
  JKCALS_E_SHAPE = -2,     /* shape unsupported by the kernels (e.g. > 2^31 elements per index) */
  JKCALS_E_STATE = -3,     /* call out of order (e.g. iterate before set_init) */
  JKCALS_E_OOM = -4,       /* workspace too small */
  JKCALS_E_CUDA = -5,      /* a CUDA runtime error (message in jkcals_last_error) */
  JKCALS_E_NONFINITE = -6  /* non-finite value in the tensor or the initial model */
} jkcals_status;

/* JKCALS_FP64_I8 (experimental): FP64 factors and epilogue, the MTTKRP from INT8
 * tcgen05 MMAs on 7 balanced base-128 digits per operand with exact integer accumulation. Each
 * (row i, slow index j') slab of T_(n) and each column c of U_q0 carries its own power-of-two scale,
 * so an operand keeps 49 bits relative to its SLAB's / COLUMN's largest magnitude and the error is
 * per-slab normwise, not elementwise as in FP64:
 *   |M - M_exact|(i, c) <~ 2^-47 sum_j' max_k |T(i, k, j')| sum_k |U_q0(k, c)| |S_j'(c)|.
 * Rows of any scale are exact to FP64 level; an entry 2^b above the rest of its slab costs those
 * entries b bits (a 1e5 scatter spike: ~1e-9 factor drift vs 1e-13 in FP64; tests/
 * test_gpu_parity.py::test_int8_sliced_*_wide_dynamic_range). A non-finite U_q0 column yields NaN
 * in M, as in FP64. Requires dims[0], dims[1] <= 65536 (padded to 64: exact int32 sums); otherwise
 * creation fails with JKCALS_E_ARG. Extra workspace: the T digits of every mode (7 x prod(dims)
 * bytes per mode, padded) and one int8 slab exponent per (i, j'). */
/* JKCALS_FP32 (north_star's "optional FP32 path", parity bar 1e-4): the MTTKRP in 3xTF32 on the
 * tcgen05 tensor cores (FP32-accurate), the epilogue in FP64. The error e is a difference of
 * O(||T||^2) terms, so an FP32-accurate M makes it unusable for a convergence test (r01: up to
 * 31 % relative error at 4-way full size). Therefore, when iterate() runs with tol > 0, the LAST
 * mode's MTTKRP of every sweep runs on the FP64 kernel: its update and the error/fit behind the
 * stop rule are FP64-accurate (reading A24). With tol <= 0 every mode runs in FP32.
 * Accuracy: FP32 accumulation chains are cut every 128 products (x 3 split terms) and summed in
 * FP64; measured at full size (every submodel, 100 sweeps) against the FP64 oracle: syn200
 * 1.6e-6, 4-way 4.1e-7, fluorescence-shaped eem R5 1.7e-5 / 2.6e-5 (factors / lambda).
 * Ill-conditioned models (e.g. R above the data's rank) can exceed 1e-4 in FP32 and should use
 * JKCALS_FP64. */
typedef enum { JKCALS_FP64 = 0, JKCALS_FP32 = 1, JKCALS_FP64_I8 = 2 } jkcals_precision;

enum {
  JKCALS_F_CONVERGED = 1,
  JKCALS_F_PINV_FALLBACK = 2,
  JKCALS_F_NONFINITE = 4,
  JKCALS_F_BREAKDOWN = 8
};

#define JKCALS_MAX_MODES 8

/* Bytes of device workspace needed by jkcals_create for these arguments on `device`.
 * ndims in [3, 8]; dims[k] >= 1, dims[0] >= 2; 1 <= rank <= 32 (ranks above 16 use the
 * streaming large-rank epilogue); n_sub = sub_end - sub_begin >= 1;
 * hist_cap >= 1 is the per-submodel error-history ring length. Returns 0 on bad arguments. */
size_t jkcals_workspace_bytes(int ndims, const int64_t *dims, int rank, int64_t n_sub,
                              jkcals_precision prec, int hist_cap, int device);

/* Create a handle for submodels p in [sub_begin, sub_end) ⊆ [0, dims[0]) (a shard; the
 * zero row of submodel p is at the GLOBAL index p). `tensor` is FP64 column-major with
 * prod(dims) elements, on the host (tensor_is_device = 0) or device (1). `cuda_stream` is a
 * cudaStream_t (NULL = legacy default stream). `workspace` is device memory of at least
 * jkcals_workspace_bytes(...) bytes, 256-byte aligned. Computes ||T||^2 and the mode-0 slice
 * norms (so ||T_-p||^2 = ||T||^2 - s_p). Errors: E_ARG, E_OOM, E_NONFINITE,
 * E_CUDA. */
/* On failure *out may still receive a handle so that jkcals_last_error() can be read; the
 * caller must then jkcals_destroy() it. */
jkcals_status jkcals_create(jkcals_t *out, int ndims, const int64_t *dims, int rank,
                            int64_t sub_begin, int64_t sub_end, const double *tensor,
                            int tensor_is_device, jkcals_precision prec, int device,
                            void *cuda_stream, void *workspace, size_t workspace_bytes,
                            int hist_cap);

/* Delete-d jackknife ("pad and periodically zero out d rows"; flop ratio
 * PAPER.md:453-476): the I_0 samples form ceil(I_0/d) contiguous groups, group g leaving out
 * rows [g*d, min(g*d + d, I_0)) of mode 0 (the last group is smaller when d does not divide
 * I_0). 1 <= d <= I_0/2 (d = 1 is jkcals_create exactly).
 * [sub_begin, sub_end) ⊆ [0, ceil(I_0/d)) are GROUP indices, and every `p` argument of the
 * calls below then names a group: its mode-0 factor has I_0 - |group| rows, its error uses
 * ||T_-g||^2 = ||T||^2 - sum_{i in group} s_i. n_sub for jkcals_workspace_bytes is
 * sub_end - sub_begin. Other arguments and errors as jkcals_create (E_ARG for a bad d). */
jkcals_status jkcals_create_d(jkcals_t *out, int ndims, const int64_t *dims, int rank, int64_t d,
                              int64_t sub_begin, int64_t sub_end, const double *tensor,
                              int tensor_is_device, jkcals_precision prec, int device,
                              void *cuda_stream, void *workspace, size_t workspace_bytes,
                              int hist_cap);

/* Multi-model pool (the paper's "All" experiment, PAPER.md:501-504 and Fig. 5 PAPER.md:590-596:
 * several fitted models of ranks R_m, e.g. {3,5,7,9} or {4,5,6}, jackknifed "simultaneously"):
 * the submodels of every model share ONE fused multi-factor per mode whose column blocks have
 * per-model widths R_m (CALS's sum_i R_i, §3.3), so one fused
 * MTTKRP per mode serves all of them. Submodel ids s in [0, nmodels * ceil(I_0/d)) enumerate
 * model m = s / ceil(I_0/d) and its group g = s % ceil(I_0/d) (d as in jkcals_create_d);
 * [sub_begin, sub_end) selects a shard of ids. Every `p` argument of the calls below is such an
 * id; factors of submodel s are rows x R_m. ranks[m] in [1, 32]. jkcals_create_d is the pool
 * with nmodels = 1. Errors as jkcals_create_d.
 * d = 0 selects plain CALS (§3.3): nothing is left out, each
 * id s in [0, nmodels) is one model fitted to the full tensor from its own initial model (e.g.
 * K random starts of one rank, or models of ranks R_m), with error ||T||^2 + ... and
 * convergence per model; the same fused sweep (a single padded-free multi-factor) serves all. */
size_t jkcals_pool_workspace_bytes(int ndims, const int64_t *dims, int nmodels, const int *ranks,
                                   int64_t d, int64_t sub_begin, int64_t sub_end,
                                   jkcals_precision prec, int hist_cap, int device);
jkcals_status jkcals_create_pool(jkcals_t *out, int ndims, const int64_t *dims, int nmodels,
                                 const int *ranks, int64_t d, int64_t sub_begin, int64_t sub_end,
                                 const double *tensor, int tensor_is_device, jkcals_precision prec,
                                 int device, void *cuda_stream, void *workspace,
                                 size_t workspace_bytes, int hist_cap);

/* Full configuration (all of the above plus spare slots). `spare` extra slots let the handle
 * later adopt submodels exported by another handle of the same problem (jkcals_import_submodel,
 * tol-mode load rebalancing across GPUs); with spare > 0 every slot can
 * hold the largest model rank. A handle has n_slots = (sub_end - sub_begin) + spare slots; the
 * per-submodel arrays of jkcals_get_status are per SLOT (n_slots long, slot q holds the id
 * jkcals_get_ids reports, -1 = free; without spare slots and migration slot q holds
 * sub_begin + q). */
typedef struct jkcals_config {
  int ndims;
  const int64_t *dims;
  int nmodels;          /* >= 1 */
  const int *ranks;     /* nmodels ranks in [1, 32] */
  int64_t d;            /* 0 = plain CALS, 1 = leave-one-out, > 1 = delete-d */
  int64_t sub_begin, sub_end;
  int spare;            /* >= 0 */
  jkcals_precision prec;
  int hist_cap;         /* >= 1 */
  int device;
} jkcals_config;
size_t jkcals_config_workspace_bytes(const jkcals_config *cfg);
jkcals_status jkcals_create_config(jkcals_t *out, const jkcals_config *cfg, const double *tensor,
                                   int tensor_is_device, void *cuda_stream, void *workspace,
                                   size_t workspace_bytes);

/* Warm start every submodel from the overall model P (Alg. 2 alg:jk:model_subsample,
 * PAPER.md:331; Alg. 3 alg:start-jk-1..alg:stop-jk-1): P[n] is a host
 * column-major dims[n] x rank array; block k of the mode-0 multi-factor gets row p_k
 * zeroed (its group's rows for delete-d). A pool takes nmodels * ndims arrays:
 * P[m * ndims + n] is model m's dims[n] x ranks[m] factor. Resets fits, histories, flags and
 * iteration counts. Errors: E_ARG, E_NONFINITE. */
jkcals_status jkcals_set_init(jkcals_t h, const double *const *P);

/* Optional per-submodel (re)initialisation, e.g. to resume: U is host column-major in the
 * get_factors layout ((dims[0]-1) x rank for mode 0, row p absent; dims[mode] x rank else;
 * delete-d: (dims[0]-|group p|) x rank for mode 0, the group's rows absent). */
jkcals_status jkcals_set_init_submodel(jkcals_t h, int64_t p, int mode, const double *U);

/* The same for every submodel on the handle at once (SURVEY §8b set_init_submodels; resume from
 * a checkpoint written with jkcals_get_all_factors): U is that call's packed layout for `mode`.
 * Errors: E_STATE (before set_init, or a submodel was compacted out), E_NONFINITE, E_ARG. */
jkcals_status jkcals_set_init_all(jkcals_t h, int mode, const double *U);

/* Run up to max_iters ALS sweeps of all active submodels (Alg. 3 repeat loop,
 * PAPER.md:432-445). tol <= 0: exactly max_iters sweeps (the §5.1 protocol);
 * tol > 0: submodels freeze as they converge and converged submodels are compacted out of
 * the fused multi-factors; returns early once all have converged. *sweeps_done (may be
 * NULL) receives the number of sweeps executed. Errors: E_STATE, E_ARG, E_CUDA. */
jkcals_status jkcals_iterate(jkcals_t h, int max_iters, double tol, int *sweeps_done);

/* Factors of submodel p (global index): mode 0 -> (dims[0]-1) x rank with row p DROPPED
 * (delete-d: (dims[0]-|group p|) x rank with the group's rows dropped),
 * mode n >= 1 -> dims[n] x rank; column-major, unit 2-norm columns. lambda (rank, may be
 * NULL) holds the column norms of the LAST updated mode (mode ndims-1 after a sweep). */
jkcals_status jkcals_get_factors(jkcals_t h, int64_t p, int mode, double *U, double *lambda);

/* Factors of ALL the submodels this handle holds, for one mode, in one call: U receives one block
 * per held submodel in slot order (= submodel order without migration), each in the get_factors
 * layout ((dims[0]-|group|) x R_p for mode 0, dims[mode] x R_p otherwise), column-major, packed
 * back to back; lambda (may be NULL) receives R_p values per submodel, packed the same way. */
jkcals_status jkcals_get_all_factors(jkcals_t h, int mode, double *U, double *lambda);

/* Debug/invariant view: submodel p's FULL block of the mode-`mode` multi-factor as it sits
 * in the fused layout, dims[mode] x R_p column-major. For mode 0 the rows of p's left-out group
 * are the padded zero rows, exactly +0.0/-0.0 after every sweep (alg:cals_jk:multifactor). */
jkcals_status jkcals_get_block(jkcals_t h, int64_t p, int mode, double *U);

/* Per-submodel status, arrays of n_slots entries in slot order (= n_sub in submodel order for a
 * handle without spare slots; any may be NULL). */
jkcals_status jkcals_get_status(jkcals_t h, double *fit, double *err, int *iters, int *flags);

/* Error history of submodel p (oldest first): up to `cap` values; *count = number written. */
jkcals_status jkcals_get_history(jkcals_t h, int64_t p, double *err, int cap, int *count);

/* Jackknife mean and standard error of U_mode over this handle's submodels (mode >= 1):
 * std = sqrt(((g-1)/g) sum_p (U_p - mean)^2), g = n_sub (Alg. 2 alg:jk:std, PAPER.md:339;
 * estimator: DESIGN.md reading A11). Column-major dims[mode] x rank. Needs n_sub >= 2. */
jkcals_status jkcals_get_jackknife_stats(jkcals_t h, int mode, double *mean, double *std);

/* Local moments for cross-shard merging (Chan et al.): per element of U_mode the count,
 * mean and sum of squared deviations M2 over this handle's submodels. mode >= 1. */
jkcals_status jkcals_get_local_moments(jkcals_t h, int mode, double *count, double *mean,
                                       double *m2);

/* Merge shard moments into the job's (the end-of-run step of a sharded jackknife, SURVEY §8e;
 * Alg. 2 alg:jk:std): folds nparts (count, mean, M2) sets of n elements each, in
 * part order, with Chan, Golub & LeVeque's pairwise update (n = n_a + n_b, d = mean_b - mean_a,
 * mean = mean_a + d n_b / n, M2 = M2_a + M2_b + d^2 n_a n_b / n; empty parts are skipped).
 * Inputs are host arrays laid out part-major (counts[k * n + e], ...); outputs count, mean, m2
 * (n each, host) may not alias them. Host computation only (no GPU needed); the std is then
 * sqrt(((g-1)/g) M2) with g the merged count. Errors: E_ARG (null pointers, nparts < 1, n < 0). */
jkcals_status jkcals_merge_moments(int nparts, int64_t n, const double *counts, const double *means,
                                   const double *m2s, double *count, double *mean, double *m2);

/* The same two calls for model `model` of a pool (over this handle's submodels of that model;
 * g = their count; dims[mode] x ranks[model]). The single-model calls above are model 0 and
 * return E_ARG on a handle with nmodels > 1. */
jkcals_status jkcals_get_model_stats(jkcals_t h, int model, int mode, double *mean, double *std);
jkcals_status jkcals_get_model_moments(jkcals_t h, int model, int mode, double *count, double *mean,
                                       double *m2);

/* Submodel alignment (Alg. 2 alg:jk:perm_scale, "permutation and scale
 * adjustment"; the scheme is DESIGN.md reading A12 since the paper defers it to its citation):
 * every local submodel is aligned to its model's reference, the warm start P given to
 * jkcals_set_init. With cos_n(r,s) the cosine between submodel column r and reference column s
 * of mode n >= 1, C(r,s) = prod_{n>=1} |cos_n(r,s)|; the permutation sigma maximises
 * sum_r C(r, sigma(r)) (exhaustive search, lowest lexicographic rank among equal maxima);
 * column r moves to sigma(r); modes n >= 1 get unit columns with sign(cos_n(r, sigma(r))),
 * mode 0 the compensating sign times lambda_r (so the model's tensor is unchanged). The result
 * goes to a separate aligned store (the fitted state is untouched) and stays valid until the
 * next iterate / set_init / set_init_submodel. Needs every rank <= 10 (E_SHAPE otherwise);
 * E_STATE before set_init. */
jkcals_status jkcals_align(jkcals_t h);

/* Alignment of submodel p: perm[r] = sigma(r) (rank values), sign[n*rank + r] the sign applied to
 * column r of mode n (n = 0: the compensating sign), congruence[sigma(r)] = C(r, sigma(r)).
 * Any output may be NULL. E_STATE if jkcals_align has not run on the current factors. */
jkcals_status jkcals_get_alignment(jkcals_t h, int64_t p, int *perm, int *sign, double *congruence);

/* Aligned factors of submodel p in the get_factors layout (mode 0 without its group's rows and
 * with lambda absorbed; modes >= 1 unit columns). E_STATE as above. */
jkcals_status jkcals_get_aligned_factors(jkcals_t h, int64_t p, int mode, double *U);

/* Full jackknife statistics of model `model`'s aligned submodels on this handle, any mode
 * (Alg. 2 alg:jk:std): per element of U_mode (column-major dims[mode] x rank)
 * count g_e, mean and M2 = sum (x - mean)^2 over the submodels in which the element exists --
 * all of them for modes >= 1; for the sampled mode 0 those whose left-out group does not
 * contain the row (reading A20) -- and std = sqrt(((g_e-1)/g_e) M2) (0 if g_e < 2).
 * The moments merge across shards with Chan's formula. E_STATE as above. */
jkcals_status jkcals_get_aligned_moments(jkcals_t h, int model, int mode, double *count,
                                         double *mean, double *m2);
jkcals_status jkcals_get_aligned_stats(jkcals_t h, int model, int mode, double *mean, double *std);

/* Slots and migration (tol-mode load rebalancing across GPUs). A live
 * (not yet converged-and-stored) submodel's whole ALS state -- its factor blocks (mode 0 with its
 * zero rows), lambda, cached Gramians, fit / error / iteration count / flags / activity and
 * error history -- is serialised into a host buffer of jkcals_state_bytes(h, p) bytes by
 * jkcals_export_submodel, which also removes it from h (its slot becomes free). Importing the
 * buffer into another handle of the same problem (same tensor, pool, d and hist_cap) with a free
 * slot continues the fit where it stopped: the sweeps that follow are those the exporting
 * handle would have run, up to the floating-point summation order of the new fused layout's
 * split-K partition (rounding-level differences). Errors: E_ARG (unknown id, foreign state,
 * small buffer), E_STATE (not live / before set_init), E_OOM (no free slot or column room). */
int jkcals_num_slots(jkcals_t h);
jkcals_status jkcals_get_ids(jkcals_t h, int64_t *ids);
size_t jkcals_state_bytes(jkcals_t h, int64_t p);
jkcals_status jkcals_export_submodel(jkcals_t h, int64_t p, void *buf, size_t bytes);
jkcals_status jkcals_import_submodel(jkcals_t h, const void *buf, size_t bytes);

/* Instrumentation: when on, iterate() launches kernels eagerly (no CUDA graph) bracketed
 * by CUDA events on the handle's stream and accumulates per-mode kernel times. */
jkcals_status jkcals_set_instrument(jkcals_t h, int on);
/* Accumulated per-mode kernel milliseconds (arrays of ndims) and launch count; resets. */
jkcals_status jkcals_get_kernel_times(jkcals_t h, double *mttkrp_ms, double *epilogue_ms,
                                      int64_t *mttkrp_launches);
/* Algorithmic MTTKRP flops of one sweep with the current fused width: 2 * C * prod(dims) per
 * mode, times ndims. */
double jkcals_sweep_flops(jkcals_t h);
/* Number of this library's kernels launched by one sweep (for bench accounting). */
int jkcals_launches_per_sweep(jkcals_t h);

const char *jkcals_last_error(jkcals_t h);
void jkcals_destroy(jkcals_t h);

/* ---- Stand-alone device operations (kernel-level parity tests and the roofline) ---- */

/* Fused MTTKRP (Eq. 1 / Alg. 3 alg:cals_jk:mttkrp) on device data:
 *   M(i, c) = sum_j T_(n)(i, j) * prod_{m != n} U_m(i_m(j), c),  c < C,
 * T device FP64 column-major; U[m] device row-major dims[m] x ldu, 16-byte aligned, ldu even and
 * ldu >= C (ldu >= C + 1 when C is odd); M device row-major dims[n] x ldm. scratch is device
 * memory of jkcals_mttkrp_scratch_bytes(...) bytes. Runs on `stream` and returns after the stream
 * has completed it (the per-call tile table is staged from pageable host memory); E_CUDA on a
 * launch or execution error. */
size_t jkcals_mttkrp_scratch_bytes(int ndims, const int64_t *dims, int n, int64_t C, int device);
jkcals_status jkcals_mttkrp(int ndims, const int64_t *dims, int n, const double *T,
                            const double *const *U, int64_t C, int64_t ldu, double *M, int64_t ldm,
                            void *scratch, size_t scratch_bytes, void *stream);

/* EXPERIMENTAL: the same MTTKRP, FP64-accurate from INT8 tcgen05 MMAs -- both
 * operands of the per-j' inner products (T per mode-n row, U_q0 per column) split into 7 balanced
 * base-128 digits with power-of-two scales, digit products accumulated exactly in int32 TMEM
 * accumulators per significance, the slow-mode row product S(j', c) applied in FP64. Same
 * arguments and blocking behaviour as jkcals_mttkrp (ldu >= C; returns after `stream` has
 * completed the op); scratch from jkcals_mttkrp_i8_scratch_bytes. The JK-CALS sweep uses the same
 * kernel under JKCALS_FP64_I8. JKCALS_E_ARG if I_q0 > 65536. Accuracy: the normwise per-slab bound
 * stated under JKCALS_FP64_I8 above. */
size_t jkcals_mttkrp_i8_scratch_bytes(int ndims, const int64_t *dims, int n, int64_t C, int device);
jkcals_status jkcals_mttkrp_i8(int ndims, const int64_t *dims, int n, const double *T,
                               const double *const *U, int64_t C, int64_t ldu, double *M, int64_t ldm,
                               void *scratch, size_t scratch_bytes, void *stream);

/* Khatri-Rao generation (descending order of Eq. 1), materialised:
 *   K(j, c) = prod_{m != n} U_m(i_m(j), c),  j in [0, prod_{m!=n} dims[m]) by Eq. 3, c < C,
 * U[m] device row-major dims[m] x ldu; K device row-major J x ldk. HBM-write-bound. */
jkcals_status jkcals_krp(int ndims, const int64_t *dims, int n, const double *const *U, int64_t C,
                         int64_t ldu, double *K, int64_t ldk, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* JKCALS_H */
