/* ckkt — condensed-KKT Newton-step solver for sm_100a (B200).
 *
 * C ABI of the per-iteration hot path of arXiv 2403.15913 (§IV-§V):
 * one interior-point iteration needs the Newton step d solving
 *
 *     K_aug d = -r                                (Eq. kkt:augmented)
 *
 *           [ W_eff  0    G^T  H^T ]        r = (r1, r2, r3, r4)
 *   K_aug = [ 0      D_s  0    I   ]        d = (dx, ds, dy, dz)
 *           [ G      0    0    0   ]
 *           [ H      I    0    0   ]        W_eff = W + diag(Sigma_x) + delta_x I  (reading R3)
 *
 * The library condenses K_aug into K_gamma = W_eff + H^T D_s H + gamma G^T G
 * (P:310), factorizes it with a supernodal Cholesky on a pattern fixed at
 * setup, and obtains d by
 *   - CKKT_LIFTED  (m_e == 0): K dx = -r1 - H^T(D_s r4 - r2)   (Eq. liftedkkt)
 *   - CKKT_HYKKT  : CG on S_gamma dy = r3 - G K_gamma^{-1} r_gamma (Eq. schurcomp),
 *                   K_gamma dx = -r_gamma - G^T dy (reading R2 of P:394)
 * followed by ds = -r4 - H dx, dz = -r2 - D_s ds and Richardson
 * refinement on K_aug (reading R7).  Readings R* are in DESIGN.md §2.
 *
 * Conventions
 *  - Indices are 0-based int32.  Matrices: W lower-triangular COO (row >= col,
 *    duplicates are summed); G (m_e x n) and H (m_i x n) in CSR with strictly
 *    increasing column indices per row.
 *  - Pattern arrays are HOST memory, read during ckkt_setup only (copied).
 *  - Value / rhs / result arrays passed to ckkt_refactor and ckkt_solve are
 *    caller-owned DEVICE pointers to contiguous FP64 (or int32) data, batch-major:
 *    instance b of a [B, len] array starts at ptr + b*len.
 *  - All device work is enqueued on the caller's stream (options.stream); calls
 *    return after enqueueing unless stated otherwise.  The library allocates all
 *    its device memory in ckkt_setup and never in refactor/solve (fixed
 *    pattern).
 *  - Errors are return codes; nothing is thrown across the ABI.  A context is
 *    used by one host thread at a time.
 */
#ifndef CKKT_H
#define CKKT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ckkt_ctx ckkt_ctx;

typedef enum {
  CKKT_OK = 0,
  CKKT_NOT_PD = 1,               /* Cholesky breakdown: wrong inertia. A result, not a failure. */
  CKKT_CG_NO_CONVERGENCE = 2,    /* CG hit cg_maxit; the last iterate is returned */
  CKKT_REFINE_NOT_CONVERGED = 3, /* refinement stopped with omega > max(ref_tol, 1e-10): the best iterate is
                                    returned; omega in (ref_tol, 1e-10] (the north-star bar) is OK */
  CKKT_PATTERN_ERROR = 4,        /* malformed pattern (index out of range, unsorted CSR, ...) */
  CKKT_INVALID_ARG = 5,
  CKKT_CUDA_ERROR = 6,
  CKKT_OUT_OF_MEMORY = 7
} ckkt_status;

enum { CKKT_LIFTED = 0, CKKT_HYKKT = 1 };

typedef struct {
  int32_t n;                   /* number of primal variables x */
  int32_t m_e;                 /* equality rows (G); must be 0 for CKKT_LIFTED */
  int32_t m_i;                 /* inequality / relaxed rows (H), each with one slack */
  int64_t w_nnz;               /* entries of W (lower COO) */
  const int32_t *w_row, *w_col;
  const int32_t *g_rowptr;     /* [m_e+1] (may be NULL when m_e == 0) */
  const int32_t *g_col;        /* [g_rowptr[m_e]] */
  const int32_t *h_rowptr;     /* [m_i+1] (may be NULL when m_i == 0) */
  const int32_t *h_col;
} ckkt_pattern;

typedef struct {
  int32_t strategy;            /* CKKT_LIFTED or CKKT_HYKKT */
  double gamma;                /* HyKKT augmentation, default 1e7; ignored by Lifted */
  double cg_rtol;              /* CG stop ||r_k||_2 <= cg_rtol ||b||_2, default 1e-10 (reading R6); finite, > 0 */
  int32_t cg_maxit;            /* default 200 */
  double ref_tol;              /* refinement stop on the componentwise backward error, default 1e-10 (R7:
                                  the north-star relative KKT residual) */
  int32_t ref_maxit;           /* default 10; 0 = no refinement */
  int32_t batch;               /* B >= 1 independent instances sharing the pattern */
  int32_t leaf;                /* nested-dissection leaf size, default 64 */
  const int32_t *perm;         /* optional host [n] caller ordering (new -> old); NULL = built-in ND */
  int32_t device;              /* CUDA device ordinal; -1 = host-only analysis (no device resources) */
  void *stream;                /* cudaStream_t owned by the caller; NULL = legacy default stream */
  double cg_rtol_corr;         /* CG stop of the refinement passes' corrections (HyKKT), default 1e-6:
                                  the refinement test ref_tol still decides the final accuracy (R6).
                                  0 = the default (a zero-initialised struct); negative / non-finite
                                  values, like non-positive cg_rtol, ref_tol or (HyKKT) gamma and
                                  negative caps, make ckkt_setup return CKKT_INVALID_ARG.  (Appended
                                  to the struct in round 1: callers must use this header's layout.) */
} ckkt_options;

typedef struct {
  int32_t status;              /* ckkt_status of this instance */
  int32_t k_cg;                /* CG iterations of the unrefined solve (HyKKT) */
  int32_t k_cg_total;          /* CG iterations summed over refinement passes */
  int32_t n_ref;               /* Richardson corrections applied */
  double rel_res;              /* componentwise backward error of the returned step (R7) */
  double rel_res_unrefined;    /* same, before refinement */
  double res_inf;              /* ||K_aug d + r||_inf of the returned step */
} ckkt_info;

typedef struct {
  int32_t n, m_e, m_i, batch;
  int64_t nnz_k;               /* lower-triangular entries of the K pattern (incl. diagonal) */
  int64_t nnz_l;               /* entries of the exact L pattern (incl. diagonal), R11 */
  int64_t l_storage;           /* doubles of supernodal factor storage per instance */
  int32_t n_supernodes;
  int32_t n_levels;            /* supernodal elimination-tree levels */
  double flops_factor;         /* sum over columns of colcount^2 (algorithmic factor flops) */
  int64_t device_bytes;        /* device memory owned by the context */
} ckkt_sizes;

/* Fill *opt with the defaults listed above (strategy HyKKT, batch 1, device 0). */
void ckkt_default_options(ckkt_options *opt);

/* Symbolic setup, once per pattern: K pattern = W ∪ G^T G ∪ H^T H ∪ diag,
 * fill-reducing ordering, elimination tree, column counts, L pattern, supernodes,
 * condensation maps; then device allocation and upload (unless device == -1).
 * Returns CKKT_PATTERN_ERROR / CKKT_INVALID_ARG / CKKT_OUT_OF_MEMORY / CKKT_CUDA_ERROR. */
ckkt_status ckkt_setup(const ckkt_pattern *pattern, const ckkt_options *opt, ckkt_ctx **out);

/* Serialized analysis (the symbolic analysis depends on the pattern only, "can be done
 * offline" and reused across processes).  ckkt_export_analysis writes the analysis of ctx to buf
 * (host memory): with buf == NULL it only stores the required size in *size; otherwise *size is the
 * capacity of buf on entry and the bytes written on exit (CKKT_INVALID_ARG if too small).  The blob
 * records a hash of the pattern, the leaf size, whether a caller ordering was used and the amalgamation
 * parameters.  ckkt_setup_from_analysis = ckkt_setup without the analysis: the blob must come from the
 * same pattern and settings (else CKKT_INVALID_ARG); the context is identical to a freshly analysed
 * one (same arrays, bit-exact results).  The blob is not referenced after the call. */
ckkt_status ckkt_export_analysis(const ckkt_ctx *ctx, void *buf, int64_t *size);
ckkt_status ckkt_setup_from_analysis(const ckkt_pattern *pattern, const ckkt_options *opt, const void *blob,
                                     int64_t size, ckkt_ctx **out);

/* Sizes of the analysis (host call, no synchronisation). */
ckkt_status ckkt_get_sizes(const ckkt_ctx *ctx, ckkt_sizes *sizes);

/* Copy the exact symbolic arrays (host memory, for bit-exact checks, R8/R11):
 * perm[n] (new -> old), parent[n] (elimination tree of P K P^T, -1 = root),
 * colcount[n], l_colptr[n+1] and l_rowind[nnz_l] (rows ascending, diagonal first).
 * Any pointer may be NULL to skip that array. */
ckkt_status ckkt_export_symbolic(const ckkt_ctx *ctx, int32_t *perm, int32_t *parent, int32_t *colcount,
                                 int64_t *l_colptr, int32_t *l_rowind);

/* Copy the internal elimination order (host memory): order[k] = original index of the column the
 * numeric factorization eliminates k-th.  It is perm composed with a postorder of its elimination
 * tree (same fill, contiguous supernodes; reading R11) and is the order in which min_bad_pivot is
 * defined (reading R9 of P:347-350): a sequential Cholesky of K_gamma permuted by `order` first
 * fails at position k* with min_bad_pivot == order[k*].  order: [n].  CKKT_INVALID_ARG on NULL. */
ckkt_status ckkt_export_elimination_order(const ckkt_ctx *ctx, int32_t *order);

/* Numeric refactorization of K_gamma from the values of one IPM iterate.
 *   w_val [B, w_nnz], g_val [B, nnz(G)], h_val [B, nnz(H)], sigma_x [B, n], d_s [B, m_i] (> 0),
 *   delta_x [B]  -- device FP64 (g_val/h_val/d_s may be NULL when the block is empty;
 *   delta_x may be NULL = 0).
 *   not_pd [B] (device int32, may be NULL): set to 1 where some pivot is <= 0 or not finite;
 *   min_bad_pivot [B] (device int32, may be NULL): ORIGINAL index of the failing column that comes
 *   first in the internal elimination order (ckkt_export_elimination_order), -1 if none (reading R9).
 * Asynchronous: the flags are valid once the stream reaches this point.
 * Zero-copy: the value arrays are read again by ckkt_solve (condensed rhs, SpMVs with G/H,
 * K_aug residual), so they must stay valid and unmodified until the last ckkt_solve that
 * uses this factorization has completed on the stream. */
ckkt_status ckkt_refactor(ckkt_ctx *ctx, const double *w_val, const double *g_val, const double *h_val,
                          const double *sigma_x, const double *d_s, const double *delta_x,
                          int32_t *not_pd, int32_t *min_bad_pivot);

/* Inertia correction around the refactorization ("(delta_x, delta_c) are computed so as
 * the regularized system satisfies (8)"; Cholesky success <=> In(K_k) = (n,0,0); for
 * HyKKT the congruence of reading R9).  delta_c is not a parameter (reading R4).  Schedule
 * (reading R15, from SPEC inertia_correction): per instance b, trial 0 with delta = 0; on
 * NOT_PD the first nonzero delta is 1e-4 * max(1, ||W_b||_inf) (symmetric W, max row sum of |W_ij|)
 * if delta_last[b] == 0, else max(1e-20, delta_last[b] / 3); each further failure multiplies delta
 * by 8; a delta above 1e40 gives up on that instance.
 *   Values as for ckkt_refactor.  delta_last [B] HOST (may be NULL = all 0): the previous IPM
 *   iteration's accepted deltas.  delta_x [B] DEVICE, library-written: the deltas of the final
 *   factorization; it stays referenced (zero-copy) like the value arrays until the last ckkt_solve.
 *   delta_out [B], trials_out [B] HOST (may be NULL): accepted delta and number of factorizations
 *   the instance needed (>= 1).  not_pd [B] DEVICE (may be NULL): final flags.
 * Synchronous (one stream synchronisation per trial).  Every trial refactors the whole batch with
 * the current per-instance deltas, so accepted instances are refactored to bit-identical factors.
 * Returns CKKT_OK when every instance is positive definite, CKKT_NOT_PD when some instance gave up
 * (its delta_out is the last delta tried), or the errors of ckkt_refactor. */
ckkt_status ckkt_refactor_inertia(ckkt_ctx *ctx, const double *w_val, const double *g_val, const double *h_val,
                                  const double *sigma_x, const double *d_s, const double *delta_last,
                                  double *delta_x, double *delta_out, int32_t *trials_out, int32_t *not_pd);

/* Fraction-to-boundary rule ("computed using a fraction-to-boundary rule"; SPEC
 * fraction_to_boundary): for each of `batch` instances, the largest alpha in (0, 1] with
 * s + alpha ds >= (1 - tau) s, i.e. alpha[b] = min(1, min over ds_i < 0 of (tau s_i) / (-ds_i)).
 *   s, ds [batch, len] DEVICE FP64 (s > 0 is the caller's precondition); 0 < tau < 1;
 *   alpha [batch] DEVICE FP64 out; stream = cudaStream_t (NULL = default stream).  Entries whose
 *   ratio is NaN are skipped.  Asynchronous, stateless (no context), deterministic (bit-exact).
 * Returns CKKT_INVALID_ARG for tau outside (0, 1), negative sizes or missing pointers. */
ckkt_status ckkt_fraction_to_boundary(int32_t batch, int64_t len, const double *s, const double *ds, double tau,
                                      double *alpha, void *stream);

/* Newton step for the last refactorization: r1 [B,n], r2 [B,m_i], r3 [B,m_e], r4 [B,m_i] in;
 * dx [B,n], ds [B,m_i], dy [B,m_e], dz [B,m_i] out (device FP64; empty blocks may be NULL).
 * info: HOST array [B] or NULL.  With info != NULL the call synchronises the stream,
 * fills info and returns the worst per-instance status (NOT_PD instances get NaN steps
 * and status CKKT_NOT_PD).  With NULL the call may still synchronise for its
 * convergence tests but does not report. */
ckkt_status ckkt_solve(ckkt_ctx *ctx, const double *r1, const double *r2, const double *r3, const double *r4,
                       double *dx, double *ds, double *dy, double *dz, ckkt_info *info);

/* End-to-end iteration from HOST buffers (pinned recommended): copies the values and
 * right-hand sides to the device, refactorizes, solves and copies the step back.
 * Same array shapes as ckkt_refactor / ckkt_solve, all host pointers. Synchronous.
 * The right-hand sides travel on a context-owned second stream after the values, while the
 * factorization runs (overlap needs pinned buffers; pageable ones are copied synchronously). */
ckkt_status ckkt_iterate_host(ckkt_ctx *ctx, const double *w_val, const double *g_val, const double *h_val,
                              const double *sigma_x, const double *d_s, const double *delta_x,
                              const double *r1, const double *r2, const double *r3, const double *r4,
                              double *dx, double *ds, double *dy, double *dz, int32_t *not_pd, ckkt_info *info);

/* Phase profiling (telemetry for the roofline report): when enabled, CUDA events are recorded on
 * the context's stream around every launch of the phases
 *   0 = condensation (k_condense), 1 = numeric factorization, 2 = forward sweeps, 3 = backward sweeps,
 *   4 = vector work of the solve (right-hand side, SpMVs with G / G^T, CG dots and updates, recovery,
 *       K_aug residuals and refinement updates).
 * ckkt_phase_times synchronises the stream, returns the accumulated device milliseconds and launch
 * counts per phase since the previous call (or since enabling), and resets them. */
ckkt_status ckkt_profile(ckkt_ctx *ctx, int32_t enable);
#define CKKT_NPHASES 5
ckkt_status ckkt_phase_times(ckkt_ctx *ctx, double *ms /* [CKKT_NPHASES] */, int64_t *count /* [CKKT_NPHASES] */);

/* Number of CUDA kernel launches enqueued by this context since creation (telemetry). */
int64_t ckkt_launch_count(const ckkt_ctx *ctx);

/* Model evaluation on the GPU (P:418-430 evaluates the model derivatives on the GPU
 * with ExaModels): the distillation-column NLP of P:489-530 (reading A of DESIGN.md R12, gradient scaling
 * R14), one warp per stage.  For `batch` instances (batch-major arrays, all DEVICE FP64):
 *   v [B, 67(N+1)] the primal point (stage-major x_1..x_32, y_1..y_32, u, L, V);
 *   lam [B, 66(N+1)] the equality multipliers (NULL = 0), row_scale [B, 66(N+1)] (NULL = 1), obj_scale;
 *   xbar0 [32] the initial state (needed for c);
 * out (any may be NULL): j_val [B, 288N+100] = row_scale * dg/dv in the CSR order of the pattern
 * (inputs/distillation.build_pattern: rows stage-major, columns increasing), w_val [B, 96N+32] = the
 * lower triangle of obj_scale grad^2 f + sum_r lam_r row_scale_r grad^2 g_r in the pattern's (row, col)
 * order, c [B, 66(N+1)] = row_scale * g(v), grad_f [B, 67(N+1)] = obj_scale grad f(v).
 * Asynchronous on `stream`; CKKT_INVALID_ARG for N < 1, batch < 1, a missing v / params, a feed tray
 * outside 2..31, non-positive holdups or horizon. */
typedef struct {
  double alpha, D, F;      /* relative volatility, distillate and feed flows */
  double w_x, rho;         /* objective weights on (x_1 - xbar_1)^2 and (u - ubar)^2 (w_x renamed, R12) */
  double horizon;          /* dt = horizon / N */
  double x_f, xbar1, ubar; /* feed composition, setpoints (unstated in the paper: SURVEY C14 fills) */
  int32_t feed_tray;       /* 1-based feed tray */
  double M[32];            /* tray holdups (C14: M_1 = M_32 = 5, else 1) */
} ckkt_distillation_params;
ckkt_status ckkt_distillation_eval(int32_t N, int32_t batch, const ckkt_distillation_params *params,
                                   const double *xbar0, const double *v, const double *lam, const double *row_scale,
                                   double obj_scale, double *j_val, double *w_val, double *c, double *grad_f,
                                   void *stream);

void ckkt_destroy(ckkt_ctx *ctx);
const char *ckkt_status_str(ckkt_status s);

#ifdef __cplusplus
}
#endif
#endif /* CKKT_H */
