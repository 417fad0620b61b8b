/*
 * tsf.h -- C-ABI of the B200-native per-time-level solver for the implicit difference
 * scheme of Gu, Huang, Ji, Carpentieri, Alikhanov (arXiv 1603.00279).
 *
 * Citations "P:nnn" are lines of the paper's LaTeX source.
 *
 * Problem (eq:lin): d^alpha_t u = gamma(t) u_x + d+(t) aD^beta_x u + d-(t) xD^beta_b u + f
 * on [a,b] x (0,T], u(x,0) = phi(x), u(a,t) = u(b,t) = 0, alpha in (0,1], beta in (1,2].
 * Grid: n interior nodes x_i = a + i h, i = 1..n, h = (b-a)/(n+1);
 *                   t_j = j tau, tau = T/M; coefficients and f are taken at
 *                   t_{j+sigma} = (j+sigma) tau, sigma = 1 - alpha/2.
 * Per level j = 0..M-1 (alg1; eq3.3):
 *     A^{(j+sigma)} u^{j+1} = B^{(j+sigma)} u^j - kappa sum_{s<j} c_{j-s}^{(j)} (u^{s+1}-u^s) + f^{j+sigma}
 * solved by right-preconditioned BiCGSTAB, CGNR (CGLS on A P^{-1}) or PCGS with a Strang
 * or T. Chan circulant preconditioner, x0 = 0, stop at ||r||_2/||r_0||_2 < tol
 * (P:922-925).  A and B are applied through a 2n circulant embedding and FP64 FFTs.
 *
 * Conventions
 *  - All floating point is IEEE double.  All vectors are contiguous, natural order
 *    (element i <-> node x_{i+1}).  "host" pointers are CPU memory, "device" pointers are
 *    CUDA device memory of the handle's device.
 *  - Every function returns TSF_OK (0) or a negative TSF_E_* code; tsf_last_error()
 *    returns a thread-local message describing the last failure.
 *  - n must be a power of two in [64, 1048576]; M >= 1.  B (instances per handle) >= 1.
 *    n <= 2^17 keeps every local FFT in shared memory; n = 2^18..2^20 (FFT lengths up to 2^21
 *    real) runs the multi-pass regime on 16-CTA clusters (plan exchange 3).
 *  - The caller owns the device workspace (e.g. a torch uint8 tensor) and every output
 *    buffer.  All input arrays are copied during tsf_init; nothing is borrowed.
 *  - A handle is bound to one device and one CUDA stream and is not thread-safe.
 *    tsf_step / tsf_solve only enqueue work; tsf_sync waits and reports status.
 */
#ifndef TSF_H
#define TSF_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------------------- */
#define TSF_OK 0
#define TSF_E_ARG (-1)            /* invalid argument (range, size, null pointer)          */
#define TSF_E_WORKSPACE (-2)      /* workspace too small or misaligned (256 B)             */
#define TSF_E_CUDA (-3)           /* CUDA runtime error (message in tsf_last_error)        */
#define TSF_E_SINGULAR_PREC (-4)  /* |lambda_P| < 1e-14 max|lambda_P|         */
#define TSF_E_BREAKDOWN (-5)      /* Krylov denominator |.| < 1e-300          */
#define TSF_E_DIVERGED (-6)       /* NaN/Inf in the iterates                  */
#define TSF_W_MAXIT 1             /* level stopped at maxit; result stored and flagged     */
#define TSF_E_STATE (-7)          /* all M levels already done / handle misuse             */

/* per-level status words stored by the device (tsf_get_stats) */
#define TSF_LEVEL_OK 0
#define TSF_LEVEL_MAXIT 1
#define TSF_LEVEL_BREAKDOWN 2
#define TSF_LEVEL_DIVERGED 3
#define TSF_LEVEL_SINGULAR_PREC 4

/* TSF_PCGS: preconditioned CGS, the paper's own Krylov method (MATLAB pcgs, P:778-779,
 * P:917-925), right-preconditioned so the stopping test uses the unpreconditioned residual. */
/* TSF_GSF: NEXT-2, the constant-coefficient path of alg2: level 0 by BiCGSTAB, levels
 * j >= 1 by u = A^{-1} g through the Gohberg-Semencul formula (alg1x) built
 * at tsf_init from A x = e_1, A y = e_n (eq3.4) solved by BiCGSTAB.  Requires gamma, d+, d- to
 * be the same at every level (else TSF_E_ARG).  Per-level stats: iterations 0, relres = the
 * true residual ||A u - g|| / ||g||. */
typedef enum { TSF_BICGSTAB = 0, TSF_CGNR = 1, TSF_PCGS = 2, TSF_GSF = 3 } tsf_method;
typedef enum { TSF_STRANG = 0, TSF_TCHAN = 1, TSF_NOPREC = 2 } tsf_precond;
typedef enum { TSF_SRC_ZERO = 0, TSF_SRC_SEPARABLE = 1, TSF_SRC_TABLE = 2, TSF_SRC_CALLBACK = 3 } tsf_src_kind;

/* host scalar function of time or space; evaluated on the host during tsf_init only */
typedef double (*tsf_fn_t)(double arg, void *ctx);
/* host source callback (general f of eq:lin): out[i] = f(x[i], t) for the n interior
 * nodes x at time t = t_{j+sigma}; called once per level during tsf_init (slow path). */
typedef void (*tsf_src_cb)(const double *x, int64_t n, double t, double *out, void *ctx);

/* One problem instance (eq:lin).  Coefficients: for each of gamma, d+, d- give EITHER a
 * host array of M samples at t_{j+sigma} (the points tsf_sample_points returns) OR a host
 * callback (array wins when both are set).  d+- must be >= 0 at every sample.
 * Initial data: host array phi[n] at the interior nodes, or callback phi_fn(x).
 * Source f^{j+sigma}_i = f(x_i, t_{j+sigma}):
 *   TSF_SRC_ZERO      f = 0
 *   TSF_SRC_SEPARABLE f^{j+sigma} = sum_{k<K} scal[j*K+k] * basis[k*n+i], 1 <= K <= 4
 *   TSF_SRC_TABLE     f^{j+sigma}_i = f_table[j*n+i]  (M x n, natural order): a host array
 *                     (copied at init on the handle's stream, directly from this buffer:
 *                     pinned memory makes it one DMA per instance; the copy has completed when
 *                     tsf_init returns), or with f_table_on_device = 1 a device array of the
 *                     handle's device that is BORROWED (read every level; must stay valid and
 *                     unchanged until tsf_destroy; all instances of a handle agree on the flag)
 *   TSF_SRC_CALLBACK  f^{j+sigma} = f_cb(x, n, t_{j+sigma}) evaluated on the host once per level
 *                     during tsf_init into the instance's device table; a non-finite value
 *                     makes tsf_init fail with TSF_E_ARG                                    */
typedef struct {
  double alpha, beta;
  int64_t n;
  int64_t M;
  double a, b, T;
  const double *gamma_t, *dplus_t, *dminus_t;   /* host [M] or NULL */
  tsf_fn_t gamma_fn, dplus_fn, dminus_fn;       /* used when the array is NULL */
  void *coef_ctx;
  const double *phi;                            /* host [n] or NULL */
  tsf_fn_t phi_fn;
  void *phi_ctx;
  int32_t src_kind;
  int32_t K;
  const double *basis;                          /* host [K][n] */
  const double *scal;                           /* host [M][K] */
  const double *f_table;                        /* [M][n], host (or device, see below) */
  int32_t f_table_on_device;                    /* 1: f_table is borrowed device memory  */
  tsf_src_cb f_cb;                              /* TSF_SRC_CALLBACK                      */
  void *f_ctx;
} tsf_problem;

/* Solver settings.  tol = 1e-12 and x0 = 0 follow P:922-925.  cluster: CTAs cooperating
 * on one instance (thread-block cluster), 0 = planner's choice, else 1/2/4/8/16.
 * x0_warm (NEXT-3, SPEC open question S:321): 0 = the paper's x0 = 0 with the stop
 * ||r_k|| < tol ||r_0|| = tol ||g||; 1 = initial guess u^j (one extra A application per level,
 * r_0 = g - A u^j) with the same g-relative stop ||r_k|| < tol ||g||.  Not for TSF_GSF.
 * true_residual: 1 = at every level exit also compute ||g - A u^{j+1}|| / ||g|| with a fresh
 * operator application (tsf_get_true_residuals; SURVEY reading c13), 0 = skip it.
 * pipelined (NEXT-3, BiCGSTAB and the GSF path's setup/level-0 solves only): 1 = two cluster
 * reductions per iteration instead of four -- r^.v, r.v, v.v, r.r in one, t.s, t.t, r^.s, r^.t
 * in the other; ||s||^2 = ||r||^2 - 2 alpha r.v + alpha^2 v.v, ||r'||^2 = ||s||^2 - 2 omega t.s +
 * omega^2 t.t and rho' = r^.s - omega r^.t by expansion (exact reduction as a fallback when the
 * expansion cancels), and the x, r and p updates in one vector pass.  Same iterates as 0 in
 * exact arithmetic; the stopping test reads the expanded norms.
 * hist_block (NEXT-3, blocked time convolution of the memory term of eq3.1): 0 = every level
 * sums its whole history (j rows, O(M^2) row reads per run); b in {2,4,...,64} = at each block
 * start J0 = kb one pass over the rows d^0..d^{J0-1} forms the partial sums of all b levels of
 * the block (kappa e_j d^0 + sum_{s=1}^{J0-1} kappa chat_{j-s} d^s, j = J0..J0+b-1), and level j
 * adds only its < b rows since J0: ~(J0/b + j - J0 + 2) row reads per level instead of j.  Same
 * terms, grouped differently (rounding only).  Disables the history-helper clusters. */
typedef struct {
  int32_t method;     /* tsf_method  */
  int32_t precond;    /* tsf_precond */
  double tol;         /* > 0 */
  int32_t maxit;      /* > 0; 1000 BiCGSTAB / PCGS, 5000 CGNR */
  int32_t cluster;
  int32_t x0_warm;
  int32_t true_residual;
  int32_t pipelined;
  int32_t hist_block;
} tsf_solver;

/* Plan summary (host only, no GPU needed). */
typedef struct {
  int32_t cluster;            /* CTAs per instance                                     */
  int32_t threads;            /* threads per CTA                                       */
  int64_t smem_bytes;         /* dynamic shared memory per CTA                         */
  int64_t embed_len;          /* complex FFT length of the 2n real embedding (= n)     */
  int64_t precond_len;        /* complex FFT length of the n-point preconditioner (n/2)*/
  size_t workspace_bytes;     /* device workspace required                             */
  int32_t exchange;           /* cross-CTA column stage: 0 none (cluster 1), 1 staged
                                 DSMEM push (local length <= 4096), 2 chunked through L2,
                                 3 multi-pass (local length > 8192: R x S rows through the
                                 global apply buffer, then chunked through L2)              */
  int32_t chunk;              /* exchange 2: column pairs per chunk                     */
  int32_t vsmem;              /* 1: Krylov vectors kept in shared memory, 0: in HBM     */
  int32_t resident;           /* 1: per-level multiplier/twiddle tables in shared memory*/
} tsf_plan_info;

typedef struct tsf_handle tsf_handle;

/* ---- host-only helpers (no GPU) ------------------------------------------------------- */
/* Interior nodes x[n] (x_i = a + (i+1) h) and level times t[M] (t_{j+sigma}).  Either
 * output may be NULL.  Errors: TSF_E_ARG on invalid alpha/beta/n/M/[a,b]/T.          */
int tsf_sample_points(const tsf_problem *p, double *x, double *t);
/* Validate p[0..B) and s; fill *info.  Errors: TSF_E_ARG. */
int tsf_plan(const tsf_problem *p, int32_t B, const tsf_solver *s, tsf_plan_info *info);
/* Workspace size in bytes for tsf_init with the same arguments. */
int tsf_workspace_bytes(const tsf_problem *p, int32_t B, const tsf_solver *s, size_t *bytes);

/* ---- lifecycle (GPU) ------------------------------------------------------------------ */
/* Build a handle for B instances (all with the same n and M) on `device`, enqueueing
 * work on `cuda_stream` (a cudaStream_t; NULL = legacy default stream).  d_workspace:
 * device memory of >= tsf_workspace_bytes, 256-byte aligned, owned by the caller and
 * kept alive until tsf_destroy.  Runs the one-time setup (WSGD weights, circulant
 * spectra, source upload) and synchronizes the stream before returning.
 * Errors: TSF_E_ARG, TSF_E_WORKSPACE, TSF_E_CUDA, TSF_E_SINGULAR_PREC.               */
int tsf_init(const tsf_problem *p, int32_t B, const tsf_solver *s, void *d_workspace,
             size_t workspace_bytes, int device, void *cuda_stream, tsf_handle **out);
/* Enqueue level j -> j+1 for every instance (one CUDA-graph launch).  Async.
 * Errors: TSF_E_STATE if all M levels are done, TSF_E_CUDA.                           */
int tsf_step(tsf_handle *h);
/* Enqueue all remaining levels (one kernel launch).  Async. */
int tsf_solve(tsf_handle *h);
/* Reset to level 0 (u = phi, history cleared).  Async. */
int tsf_reset(tsf_handle *h);
/* Wait for the stream.  Returns TSF_OK, TSF_W_MAXIT, or the first fatal per-level
 * status of the completed levels mapped to TSF_E_BREAKDOWN / TSF_E_DIVERGED /
 * TSF_E_SINGULAR_PREC; TSF_E_CUDA on a CUDA error.                                    */
int tsf_sync(tsf_handle *h);
/* Current level index j (number of completed levels, 0..M), host-side counter. */
int64_t tsf_level(const tsf_handle *h);
/* Current solution u^j of instance `inst` (natural order, n doubles) into `out` (host
 * pointer if out_on_device == 0, else device pointer).  Synchronizes the stream.      */
int tsf_get_solution(tsf_handle *h, int32_t inst, double *out, int32_t out_on_device);
/* All instances: out[B][n]. */
int tsf_get_solutions(tsf_handle *h, double *out, int32_t out_on_device);
/* Per-level statistics of all instances, host arrays [B][M] (any may be NULL):
 * iters_half = Krylov iterations x 2 (a BiCGSTAB half-step exit counts 1), relres = final
 * recurrence ||r||/||r0||, status = TSF_LEVEL_*.  Entries of levels not yet run are 0.  */
int tsf_get_stats(tsf_handle *h, int32_t *iters_half, double *relres, int32_t *status);
/* True relative residuals ||g^{j+1} - A u^{j+1}|| / ||g^{j+1}|| of every level, host array
 * [B][M] (0 for levels not yet run or when the solver's true_residual was 0; the GSF path
 * always stores it).  Synchronizes the stream. */
int tsf_get_true_residuals(tsf_handle *h, double *true_relres);
/* Plan actually used by the handle. */
int tsf_handle_info(const tsf_handle *h, tsf_plan_info *info);
/* Release host resources (the workspace belongs to the caller). */
int tsf_destroy(tsf_handle *h);
/* Thread-local description of the last error ("" if none). */
const char *tsf_last_error(void);

/* ---- test hooks ----------------------------------------------------------------------- */
/* Canonical FFT tables of the local transform of complex length L (power of two, <= 2^20),
 * the tables the kernels are planned from (DESIGN.md R-fft): plan[<=20] radices
 * (returns the stage count via *stages), perm[L] gather digit reversal, twiddle
 * exponents of stage s concatenated in tw[] (k-major, q-minor; sum over stages of
 * m_s entries, at most 2L).  Host only.                                               */
int tsf_debug_fft_tables(int64_t L, int32_t *plan, int32_t *stages, int32_t *perm,
                         int32_t *tw);
/* Run the device in-place local FFT of length L (one CTA) on host data x[2L]
 * (interleaved complex): y = raw slot-order output of the forward DIF transform
 * (y[p] = X[perm[p]]) when inverse == 0; when inverse == 1, x is taken in slot order and
 * y is the unnormalized inverse transform in natural order.                            */
int tsf_debug_local_fft(int64_t L, const double *x, double *y, int32_t inverse);
/* WSGD weights g[0..K], omega[0..K] from the device generator (K <= 2^21). */
int tsf_debug_weights(double beta, int64_t K, double *g, double *omega);
/* Apply one operator of instance `inst` at level j to host x[n] -> host y[n] with the
 * solve's own fused device path.  which: 0 = A, 1 = B, 2 = A^T, 3 = P^{-1}, 4 = P^{-T}. */
int tsf_debug_apply(tsf_handle *h, int32_t inst, int64_t j, int32_t which, const double *x,
                    double *y);
/* Timing hook: one kernel launch running reps (>= 2) operator applications of instance inst
 * at level j, alternating P^{-1} and A as in a Krylov iteration, on a device buffer; *ms =
 * CUDA-event time of the launch (after one warm-up launch).  Needs a preconditioner. */
int tsf_debug_apply_bench(tsf_handle *h, int32_t inst, int64_t j, int32_t reps, float *ms);
/* Per-level spectra of instance `inst` in natural bin order (interleaved complex):
 * lamA[n+1] = bins 0..n of the 2n embedding of A^{(j+sigma)};
 * lamP[n/2+1] = bins 0..n/2 of the preconditioner.  Either may be NULL.              */
int tsf_debug_spectra(tsf_handle *h, int32_t inst, int64_t j, double *lamA, double *lamP);
/* Right-hand side g^{(j+1)} the device would build at the handle's current level for
 * instance `inst` (host out[n]).                                                       */
int tsf_debug_rhs(tsf_handle *h, int32_t inst, double *out);
/* Overwrite the solution history of instance `inst` with host U[(j+1)][n] = u^0..u^j and
 * set the handle to level j (teacher forcing).  Every instance is moved to level j.    */
int tsf_debug_set_history(tsf_handle *h, int32_t inst, int64_t j, const double *U);
/* History-helper handshake words of the last solve (out[8] host): [0] solver CTA-levels done,
 * [1..2] ready[J&1], [3..4] helper counters, [5] 1 if a bounded wait timed out and the solver
 * summed the history itself. */
int tsf_debug_helper_state(tsf_handle *h, int64_t *out);
/* Section cycle counters of the profiling build (libtsf_prof.so; zeros otherwise):
 * out[32] host, then cleared when reset != 0.                                          */
int tsf_debug_prof(tsf_handle *h, uint64_t *out, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* TSF_H */
