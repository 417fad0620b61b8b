/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the per-time-level solve of
 * Gu et al., arXiv 1603.00279 ("Fast iterative method with a second order implicit
 * difference scheme for time-space fractional convection-diffusion equations").
 * Citations "P:nnn" are lines of /root/reference/PAPER.md (LaTeX source).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1603_00279_b200/) never does.
 * The oracle shares no code, header, table or constant generator with the CUDA path.
 *
 * Every floating-point quantity is IEEE double (the paper's precision).
 */
#ifndef TSF_ORACLE_H
#define TSF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- coefficient-function shapes: c(t) = scale * shape(t) ---------------------------- */
enum { ORC_CONST = 0, ORC_ONE_PLUS_T = 1, ORC_ONE_PLUS_T2 = 2, ORC_COS = 3, ORC_SIN = 4, ORC_T = 5 };
typedef struct { int32_t shape; double scale; } orc_fn;

/* ---- initial data / source kinds ------------------------------------------------------ */
enum { ORC_PHI_ARRAY = 0, ORC_PHI_X2 = 1 };          /* X(x) = x^2 (1-x)^2          */
enum { ORC_SRC_ZERO = 0, ORC_SRC_TABLE = 1,          /* f[j][i] = f(x_i, t_{j+sigma})       */
       ORC_SRC_EXA = 2,                              /* u=(t^{2+a}+1)X, Examples 1/2 P:937  */
       ORC_SRC_MMS3 = 3 };                           /* u=(t^3+1)X             */

typedef struct {
  double alpha, beta;       /* alpha in (0,1], beta in (1,2]            */
  int64_t n;                /* interior unknowns; h = (b-a)/(n+1)      */
  int64_t M;                /* time levels; tau = T/M                  */
  double a, b, T;
  orc_fn gamma, dplus, dminus;
  int32_t phi_kind; const double *phi;      /* phi[n] when ORC_PHI_ARRAY        */
  int32_t src_kind; const double *f_table;  /* f_table[M][n] when ORC_SRC_TABLE */
} orc_problem;

/* Lemma 3: g_k = (1 - (beta+1)/k) g_{k-1}, g_0 = 1.  g[0..K]. */
void orc_grunwald(double beta, int64_t K, double *g);
/* Lemma 2: WSGD weights omega[0..K] (K >= 1). */
void orc_wsgd(double beta, int64_t K, double *omega);
/* Lemma 1: a[0..M], b[0..M] (b[0] = 0, unused). */
void orc_time_ab(double alpha, int64_t M, double *a, double *b);
/* Lemma 1: c^{(alpha,sigma,j)}_m for m = 0..j into c[0..j]. */
void orc_c_row(double alpha, int64_t j, double *c);
/* eta_j of eq3.1 and kappa = tau^{-alpha}/Gamma(2-alpha). */
double orc_eta(double alpha, double tau, int64_t j);
double orc_eval_fn(orc_fn f, double t);

/* Dense assembly of A^{(j+sigma)}, B^{(j+sigma)} (eq3.3), row-major n x n. */
int orc_assemble(const orc_problem *p, int64_t j, double *A, double *B);
/* Right-hand side g^{(j+1)} of alg1 step 2 from the history U[0..j][n]. */
int orc_rhs(const orc_problem *p, int64_t j, const double *U, double *g);
/* Source f(x_i, t) at interior nodes (closed forms; EXA transcribes P:937-942). */
int orc_source(const orc_problem *p, int64_t j, double t, double *f);
/* Exact solution u(x_i, t) for EXA / MMS3. */
int orc_exact(const orc_problem *p, double t, double *u);
/* Gaussian elimination with partial pivoting; A destroyed. */
int orc_ge_solve(int64_t n, double *A, double *x_inout);
/* Matrix-free A (which=0) / B (which=1) product and RHS for large n (O(n) memory). */
int orc_matvec(const orc_problem *p, int64_t j, int which, const double *x, double *y);
/* The same product at the rows rows[0..nr) only: y[k] = (A x)[rows[k]] (O(n) per row). */
int orc_matvec_rows(const orc_problem *p, int64_t j, int which, const double *x, const int64_t *rows,
                    int64_t nr, double *y);
/* Toeplitz generator of A (which=0) / B (which=1): col[i] = M[i][0], row[m] = M[0][m]. */
int orc_generator(const orc_problem *p, int64_t j, int which, double *col, double *row);
int orc_rhs_nodense(const orc_problem *p, int64_t j, const double *U, double *g);
/* Rows rows[0..nr) of the same RHS (same arithmetic order per row). */
int orc_rhs_rows(const orc_problem *p, int64_t j, const double *U, const int64_t *rows, int64_t nr,
                 double *g);
/* Full IDS run (alg1) with a direct solve per level: U[(M+1)][n]. */
int orc_solve(const orc_problem *p, double *U);
/* Same, but solve level j only from a given history (teacher forcing): out[n]. */
int orc_solve_level(const orc_problem *p, int64_t j, const double *U, double *out);

/* Timing sample at full n for bench.py (see oracle.c): t[3] = assembly, first kmax columns of
 * the elimination, one level's RHS + solve + refinement at history length j.  U[(j+1)][n]. */
int orc_time_sample(const orc_problem *p, int64_t j, int64_t kmax, const double *U, double *t);

/* Discrete L2 norm: sqrt(h sum v_i^2). */
double orc_l2(int64_t n, double h, const double *v);

/* Brute-force O(L^2) DFT, interleaved complex; inverse carries 1/L. */
void orc_dft(int64_t L, const double *x, double *X, int inverse);
/* Canonical FFT integer tables (reading R-fft): radix plan, gather
 * digit-reversal permutation, stage twiddle exponents.  Returns number of stages. */
int orc_fft_plan(int64_t L, int32_t *plan);
void orc_fft_perm(int64_t L, int32_t *perm);
/* twiddle exponents of stage s: tw[k*r_s + q] for k < m_s/r_s, q < r_s */
int64_t orc_fft_twiddles(int64_t L, int32_t s, int32_t *tw);

/* Strang and T. Chan circulant first columns of a Toeplitz (col,row). */
void orc_strang_col(int64_t n, const double *col, const double *row, double *c);
void orc_tchan_col(int64_t n, const double *col, const double *row, double *c);

#ifdef __cplusplus
}
#endif
#endif
