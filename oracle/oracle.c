/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow CPU implementation of what the hot path computes, written from
 * PAPER.md in the paper's order and notation.  Each function cites the passage it
 * follows.  Dense matrices, Gaussian elimination, direct sums, brute-force DFT: no
 * blocking, fusion or reordering beyond what the paper's definitions state.
 *
 * Built with -O2 -ffp-contract=off (reading R-fma): IEEE round-to-nearest,
 * no fused multiply-add, so results are reproducible across hosts.  -fopenmp splits the
 * independent ROWS of the dense loops (assembly, products, the GE row updates, refinement
 * residuals) across threads; every row's arithmetic and summation order is unchanged, so
 * results are bitwise identical for any OMP_NUM_THREADS (tests/test_oracle.py checks it).
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------- */
/* Lemma 3: g_k = (1 - (beta+1)/k) g_{k-1}, with g_0 = 1.                 */
void orc_grunwald(double beta, int64_t K, double *g) {
  g[0] = 1.0;
  for (int64_t k = 1; k <= K; ++k) g[k] = (1.0 - (beta + 1.0) / (double)k) * g[k - 1];
}

/* Lemma 2: lambda_1 = (b^2+3b+2)/12, lambda_0 = (4-b^2)/6,
 * lambda_{-1} = (b^2-3b+2)/12;  omega_0 = l1 g0, omega_1 = l1 g1 + l0 g0,
 * omega_k = l1 g_k + l0 g_{k-1} + l-1 g_{k-2}  (k >= 2).                              */
void orc_wsgd(double beta, int64_t K, double *omega) {
  double *g = (double *)malloc(sizeof(double) * (size_t)(K + 1));
  orc_grunwald(beta, K, g);
  const double l1 = (beta * beta + 3.0 * beta + 2.0) / 12.0;
  const double l0 = (4.0 - beta * beta) / 6.0;
  const double lm1 = (beta * beta - 3.0 * beta + 2.0) / 12.0;
  omega[0] = l1 * g[0];
  if (K >= 1) omega[1] = l1 * g[1] + l0 * g[0];
  for (int64_t k = 2; k <= K; ++k) omega[k] = l1 * g[k] + l0 * g[k - 1] + lm1 * g[k - 2];
  free(g);
}

/* Lemma 1: sigma = 1 - alpha/2, a_0 = sigma^{1-alpha},
 * a_l = (l+sigma)^{1-alpha} - (l-1+sigma)^{1-alpha},
 * b_l = [(l+sigma)^{2-alpha} - (l-1+sigma)^{2-alpha}]/(2-alpha)
 *       - [(l+sigma)^{1-alpha} + (l-1+sigma)^{1-alpha}]/2.                             */
void orc_time_ab(double alpha, int64_t M, double *a, double *b) {
  const double s = 1.0 - alpha / 2.0;
  a[0] = pow(s, 1.0 - alpha);
  b[0] = 0.0;
  for (int64_t l = 1; l <= M; ++l) {
    const double hi = (double)l + s, lo = (double)(l - 1) + s;
    a[l] = pow(hi, 1.0 - alpha) - pow(lo, 1.0 - alpha);
    b[l] = (pow(hi, 2.0 - alpha) - pow(lo, 2.0 - alpha)) / (2.0 - alpha) -
           0.5 * (pow(hi, 1.0 - alpha) + pow(lo, 1.0 - alpha));
  }
}

/* Lemma 1: c_0^{(0)} = a_0 for j = 0; for j >= 1
 * c_0 = a_0 + b_1, c_m = a_m + b_{m+1} - b_m (1 <= m <= j-1), c_j = a_j - b_j.        */
void orc_c_row(double alpha, int64_t j, double *c) {
  double *a = (double *)malloc(sizeof(double) * (size_t)(j + 2));
  double *b = (double *)malloc(sizeof(double) * (size_t)(j + 2));
  orc_time_ab(alpha, j + 1, a, b);
  if (j == 0) {
    c[0] = a[0];
  } else {
    c[0] = a[0] + b[1];
    for (int64_t m = 1; m <= j - 1; ++m) c[m] = a[m] + b[m + 1] - b[m];
    c[j] = a[j] - b[j];
  }
  free(a);
  free(b);
}

/* eta_j: c_0^{(alpha,sigma,j)} / (tau^alpha Gamma(2-alpha)). */
double orc_eta(double alpha, double tau, int64_t j) {
  double *c = (double *)malloc(sizeof(double) * (size_t)(j + 1));
  orc_c_row(alpha, j, c);
  const double c0 = c[0];
  free(c);
  return c0 / (pow(tau, alpha) * tgamma(2.0 - alpha));
}

double orc_eval_fn(orc_fn f, double t) {
  switch (f.shape) {
    case ORC_CONST: return f.scale;
    case ORC_ONE_PLUS_T: return f.scale * (1.0 + t);
    case ORC_ONE_PLUS_T2: return f.scale * (1.0 + t * t);
    case ORC_COS: return f.scale * cos(t);
    case ORC_SIN: return f.scale * sin(t);
    case ORC_T: return f.scale * t;
  }
  return NAN;
}

static int grid_ok(const orc_problem *p) {
  if (!(p->alpha > 0.0 && p->alpha <= 1.0)) return 0;
  if (!(p->beta > 1.0 && p->beta <= 2.0)) return 0;
  if (p->n < 1 || p->M < 1 || !(p->b > p->a) || !(p->T > 0.0)) return 0;
  return 1;
}

/* ---------------------------------------------------------------------------------- */
/* eq3.2 read as the pure Toeplitz W[i][m] = omega_{i-m+1} (i-m+1 >= 0)
 * (reading R-W), Q[i][i+1] = +1, Q[i+1][i] = -1, and
 * L_j = gamma/(2h) Q + D+/h^beta W + D-/h^beta W^T at t_{j+sigma}.
 * A = eta_j I - sigma L_j,  B = eta_j I + (1-sigma) L_j   (eq3.3).          */
static void dense_L(const orc_problem *p, int64_t j, double *L) {
  const int64_t n = p->n;
  const double h = (p->b - p->a) / (double)(n + 1);
  const double tau = p->T / (double)p->M;
  const double sigma = 1.0 - p->alpha / 2.0;
  const double t = ((double)j + sigma) * tau;
  const double gam = orc_eval_fn(p->gamma, t);
  const double dp = orc_eval_fn(p->dplus, t), dm = orc_eval_fn(p->dminus, t);
  const double hb = pow(h, p->beta);
  double *omega = (double *)malloc(sizeof(double) * (size_t)(n + 2));
  orc_wsgd(p->beta, n + 1, omega);
#pragma omp parallel for schedule(static) if (n > 256)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t m = 0; m < n; ++m) {
      double W = (i - m + 1 >= 0) ? omega[i - m + 1] : 0.0;   /* W[i][m]   */
      double WT = (m - i + 1 >= 0) ? omega[m - i + 1] : 0.0;  /* W^T[i][m] */
      double Q = (m == i + 1) ? 1.0 : ((m == i - 1) ? -1.0 : 0.0);
      L[i * n + m] = gam / (2.0 * h) * Q + dp / hb * W + dm / hb * WT;
    }
  free(omega);
}

int orc_assemble(const orc_problem *p, int64_t j, double *A, double *B) {
  if (!grid_ok(p) || j < 0 || j >= p->M) return -1;
  const int64_t n = p->n;
  const double tau = p->T / (double)p->M;
  const double sigma = 1.0 - p->alpha / 2.0;
  const double eta = orc_eta(p->alpha, tau, j);
  dense_L(p, j, A);
#pragma omp parallel for schedule(static) if (n > 256)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t m = 0; m < n; ++m) {
      const double Lim = A[i * n + m];
      const double I = (i == m) ? 1.0 : 0.0;
      if (B) B[i * n + m] = eta * I + (1.0 - sigma) * Lim;
      A[i * n + m] = eta * I - sigma * Lim;
    }
  return 0;
}

/* ---------------------------------------------------------------------------------- */
/* X(x) = x^2(1-x)^2 and the Riemann-Liouville derivatives of the manufactured solutions
 * (P:937-942 for u = (t^{2+alpha}+1) X; same structure with t^3 for SURVEY c25):
 *   aD^beta_x x^p = Gamma(p+1)/Gamma(p+1-beta) x^{p-beta}  (a = 0)
 *   xD^beta_b (1-x)^p = Gamma(p+1)/Gamma(p+1-beta) (1-x)^{p-beta}  (b = 1).           */
static double Xfun(double x) { return x * x * (1.0 - x) * (1.0 - x); }

int orc_source(const orc_problem *p, int64_t j, double t, double *f) {
  const int64_t n = p->n;
  const double h = (p->b - p->a) / (double)(n + 1);
  if (p->src_kind == ORC_SRC_ZERO) {
    for (int64_t i = 0; i < n; ++i) f[i] = 0.0;
    return 0;
  }
  if (p->src_kind == ORC_SRC_TABLE) {
    for (int64_t i = 0; i < n; ++i) f[i] = p->f_table[j * n + i];
    return 0;
  }
  if (p->a != 0.0 || p->b != 1.0) return -1;
  const double al = p->alpha, be = p->beta;
  const double gam = orc_eval_fn(p->gamma, t);
  const double dp = orc_eval_fn(p->dplus, t), dm = orc_eval_fn(p->dminus, t);
  double time_caputo, time_u;
  if (p->src_kind == ORC_SRC_EXA) {
    /* Gamma(3+alpha)/2 x^2(1-x)^2 t^2  (Caputo of t^{2+alpha}) */
    time_caputo = tgamma(3.0 + al) / 2.0 * t * t;
    time_u = pow(t, 2.0 + al) + 1.0;
  } else if (p->src_kind == ORC_SRC_MMS3) {
    time_caputo = tgamma(4.0) / tgamma(4.0 - al) * pow(t, 3.0 - al);
    time_u = t * t * t + 1.0;
  } else {
    return -1;
  }
  const double G3 = tgamma(3.0) / tgamma(3.0 - be);
  const double G4 = 2.0 * tgamma(4.0) / tgamma(4.0 - be);
  const double G5 = tgamma(5.0) / tgamma(5.0 - be);
  for (int64_t i = 0; i < n; ++i) {
    const double x = p->a + (double)(i + 1) * h;
    const double y = 1.0 - x;
    /* P:937-942 bracket: gamma*2x(1-x)(1-2x) + G3[d+ x^{2-b} + d- (1-x)^{2-b}]
     *   - 2G(4)/G(4-b)[d+ x^{3-b} + d-(1-x)^{3-b}] + G5[d+ x^{4-b} + d-(1-x)^{4-b}] */
    const double br = gam * 2.0 * x * (1.0 - x) * (1.0 - 2.0 * x) +
                      G3 * (dp * pow(x, 2.0 - be) + dm * pow(y, 2.0 - be)) -
                      G4 * (dp * pow(x, 3.0 - be) + dm * pow(y, 3.0 - be)) +
                      G5 * (dp * pow(x, 4.0 - be) + dm * pow(y, 4.0 - be));
    f[i] = time_caputo * Xfun(x) - time_u * br;
  }
  return 0;
}

int orc_exact(const orc_problem *p, double t, double *u) {
  const int64_t n = p->n;
  const double h = (p->b - p->a) / (double)(n + 1);
  double tu;
  if (p->src_kind == ORC_SRC_EXA) tu = pow(t, 2.0 + p->alpha) + 1.0;
  else if (p->src_kind == ORC_SRC_MMS3) tu = t * t * t + 1.0;
  else return -1;
  for (int64_t i = 0; i < n; ++i) u[i] = tu * Xfun(p->a + (double)(i + 1) * h);
  return 0;
}

/* ---------------------------------------------------------------------------------- */
/* Gaussian elimination with partial pivoting, row-major, factors kept for reuse
 * ("[L,U]=lu(A); x = U\(L\b)").                                           */
static int lu_factor_k(int64_t n, double *A, int64_t *piv, int64_t kmax) {
  for (int64_t k = 0; k < kmax; ++k) {
    int64_t pr = k;
    double best = fabs(A[k * n + k]);
    for (int64_t i = k + 1; i < n; ++i)
      if (fabs(A[i * n + k]) > best) { best = fabs(A[i * n + k]); pr = i; }
    piv[k] = pr;
    if (best == 0.0) return -2;
    if (pr != k)
      for (int64_t m = 0; m < n; ++m) {
        double tmp = A[k * n + m]; A[k * n + m] = A[pr * n + m]; A[pr * n + m] = tmp;
      }
    const double inv = 1.0 / A[k * n + k];
    /* rows are independent: OpenMP splits them across threads, each row's arithmetic is
     * unchanged, so the factors are bitwise identical to the single-threaded loop */
#pragma omp parallel for schedule(static) if (n - k > 256)
    for (int64_t i = k + 1; i < n; ++i) {
      const double l = A[i * n + k] * inv;
      A[i * n + k] = l;
      double *ri = A + i * n;
      const double *rk = A + k * n;
      for (int64_t m = k + 1; m < n; ++m) ri[m] -= l * rk[m];
    }
  }
  return 0;
}

static int lu_factor(int64_t n, double *A, int64_t *piv) { return lu_factor_k(n, A, piv, n); }

static void lu_solve(int64_t n, const double *LU, const int64_t *piv, double *x) {
  for (int64_t k = 0; k < n; ++k) {
    if (piv[k] != k) { double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
  }
  for (int64_t i = 0; i < n; ++i) {                 /* L y = P b (unit lower) */
    double s = x[i];
    for (int64_t m = 0; m < i; ++m) s -= LU[i * n + m] * x[m];
    x[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {            /* U x = y */
    double s = x[i];
    for (int64_t m = i + 1; m < n; ++m) s -= LU[i * n + m] * x[m];
    x[i] = s / LU[i * n + i];
  }
}

/* Iterative refinement (DESIGN.md R-refine): the per-level result is defined as the exact
 * solution of A u = g (eq3.3); plain GE has forward error ~cond(A) eps (1e-8 relative at
 * cond ~ 1e7, e.g. beta -> 2 with small alpha).  r = b - A x is accumulated in x87 extended
 * precision (long double, 64-bit mantissa) from the unfactored A0, the correction solved
 * with the LU factors, x += d; this converges to the correctly rounded solution while
 * cond(A) * eps << 1.                                                                   */
static void refine(int64_t n, const double *A0, const double *LU, const int64_t *piv,
                   const double *b, double *x, int steps) {
  double *d = (double *)malloc(sizeof(double) * (size_t)n);
  for (int it = 0; it < steps; ++it) {
#pragma omp parallel for schedule(static) if (n > 256)
    for (int64_t i = 0; i < n; ++i) {
      long double s = (long double)b[i];
      const double *ai = A0 + i * n;
      for (int64_t m = 0; m < n; ++m) s -= (long double)ai[m] * (long double)x[m];
      d[i] = (double)s;
    }
    lu_solve(n, LU, piv, d);
    for (int64_t i = 0; i < n; ++i) x[i] += d[i];
  }
  free(d);
}

int orc_ge_solve(int64_t n, double *A, double *x) {
  int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  double *A0 = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *b = (double *)malloc(sizeof(double) * (size_t)n);
  memcpy(A0, A, sizeof(double) * (size_t)(n * n));
  memcpy(b, x, sizeof(double) * (size_t)n);
  int rc = lu_factor(n, A, piv);
  if (rc == 0) {
    lu_solve(n, A, piv, x);
    refine(n, A0, A, piv, b, x, 3);
  }
  free(piv);
  free(A0);
  free(b);
  return rc;
}

/* ---------------------------------------------------------------------------------- */
/* alg1 step 2 with eq3.1:
 *   g = B^{(j+sigma)} u^j - tau^{-alpha}/Gamma(2-alpha) sum_{s=0}^{j-1} c_{j-s}^{(j)} (u^{s+1}-u^s)
 *       + f^{j+sigma}                                        (sign: DESIGN.md R-sign)    */
static void rhs_with_B(const orc_problem *p, int64_t j, const double *U, const double *B,
                       double *g) {
  const int64_t n = p->n;
  const double tau = p->T / (double)p->M;
  const double sigma = 1.0 - p->alpha / 2.0;
  const double kappa = pow(tau, -p->alpha) / tgamma(2.0 - p->alpha);
  const double *uj = U + j * n;
#pragma omp parallel for schedule(static) if (n > 256)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t m = 0; m < n; ++m) s += B[i * n + m] * uj[m];
    g[i] = s;
  }
  if (j >= 1) {
    double *c = (double *)malloc(sizeof(double) * (size_t)(j + 1));
    orc_c_row(p->alpha, j, c);
    for (int64_t s = 0; s <= j - 1; ++s) {
      const double w = kappa * c[j - s];
      for (int64_t i = 0; i < n; ++i) g[i] -= w * (U[(s + 1) * n + i] - U[s * n + i]);
    }
    free(c);
  }
  double *f = (double *)malloc(sizeof(double) * (size_t)n);
  orc_source(p, j, ((double)j + sigma) * tau, f);
  for (int64_t i = 0; i < n; ++i) g[i] += f[i];
  free(f);
}

int orc_rhs(const orc_problem *p, int64_t j, const double *U, double *g) {
  if (!grid_ok(p) || j < 0 || j >= p->M) return -1;
  const int64_t n = p->n;
  double *A = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *B = (double *)malloc(sizeof(double) * (size_t)(n * n));
  orc_assemble(p, j, A, B);
  rhs_with_B(p, j, U, B, g);
  free(A);
  free(B);
  return 0;
}

/* Matrix-free products with A^{(j+sigma)} (which = 0) or B^{(j+sigma)} (which = 1): the
 * same entries as orc_assemble (eq3.2-eq3.3) generated row by row, O(n^2) time and O(n)
 * memory, for sampled checks at sizes where the dense matrix does not fit.  Each row sum is
 * accumulated in x87 extended precision, as the refinement residuals are (R-refine): at
 * n = 2^17 the entries reach h^{-beta} ~ 1e10 and cancel to O(1), so a double accumulator
 * would add its own ~1e-6 relative error to a residual check of that size.              */
/* Level-j scalars of the literal operator (eq3.3): A = eta I - sigma L, B = eta I +
 * (1 - sigma) L, L = gamma/(2h) Q + d+/h^beta W + d-/h^beta W^T, with omega the WSGD weights. */
typedef struct { double eta, mu, q, dph, dmh; int64_t n; double *omega; } mv_ctx;

static int mv_setup(const orc_problem *p, int64_t j, int which, mv_ctx *c) {
  if (!grid_ok(p) || j < 0 || j >= p->M || (which != 0 && which != 1)) return -1;
  const int64_t n = p->n;
  const double h = (p->b - p->a) / (double)(n + 1);
  const double tau = p->T / (double)p->M;
  const double sigma = 1.0 - p->alpha / 2.0;
  const double t = ((double)j + sigma) * tau;
  const double hb = pow(h, p->beta);
  c->n = n;
  c->eta = orc_eta(p->alpha, tau, j);
  c->mu = (which == 0) ? -sigma : (1.0 - sigma);
  c->q = orc_eval_fn(p->gamma, t) / (2.0 * h);
  c->dph = orc_eval_fn(p->dplus, t) / hb;
  c->dmh = orc_eval_fn(p->dminus, t) / hb;
  c->omega = (double *)malloc(sizeof(double) * (size_t)(n + 2));
  orc_wsgd(p->beta, n + 1, c->omega);
  return 0;
}

/* L[i][m] written out: W[i][m] = omega_{i-m+1}, W^T[i][m] = omega_{m-i+1} (zero for negative
 * index), Q[i][i+1] = 1, Q[i][i-1] = -1 (central difference of the convection term). */
static double mv_L(const mv_ctx *c, int64_t i, int64_t m) {
  const double W = (i - m + 1 >= 0) ? c->omega[i - m + 1] : 0.0;
  const double WT = (m - i + 1 >= 0) ? c->omega[m - i + 1] : 0.0;
  const double Q = (m == i + 1) ? 1.0 : ((m == i - 1) ? -1.0 : 0.0);
  return c->q * Q + c->dph * W + c->dmh * WT;
}

/* row i of the product, the row sum in extended precision (reading R-refine) */
static double mv_row(const mv_ctx *c, int64_t i, const double *x) {
  long double s = 0.0L;
  for (int64_t m = 0; m < c->n; ++m) s += (long double)mv_L(c, i, m) * (long double)x[m];
  return (double)((long double)c->eta * (long double)x[i] + (long double)c->mu * s);
}

int orc_matvec(const orc_problem *p, int64_t j, int which, const double *x, double *y) {
  mv_ctx c;
  if (mv_setup(p, j, which, &c)) return -1;
  const int64_t n = c.n;
#pragma omp parallel for schedule(static) if (n > 256)
  for (int64_t i = 0; i < n; ++i) y[i] = mv_row(&c, i, x);
  free(c.omega);
  return 0;
}

int orc_matvec_rows(const orc_problem *p, int64_t j, int which, const double *x, const int64_t *rows,
                    int64_t nr, double *y) {
  mv_ctx c;
  if (mv_setup(p, j, which, &c)) return -1;
  for (int64_t k = 0; k < nr; ++k)
    if (rows[k] < 0 || rows[k] >= c.n) { free(c.omega); return -1; }
#pragma omp parallel for schedule(static) if (nr > 4)
  for (int64_t k = 0; k < nr; ++k) y[k] = mv_row(&c, rows[k], x);
  free(c.omega);
  return 0;
}

int orc_generator(const orc_problem *p, int64_t j, int which, double *col, double *row) {
  mv_ctx c;
  if (mv_setup(p, j, which, &c)) return -1;
  for (int64_t i = 0; i < c.n; ++i) {
    col[i] = (i == 0 ? c.eta : 0.0) + c.mu * mv_L(&c, i, 0);
    row[i] = (i == 0 ? c.eta : 0.0) + c.mu * mv_L(&c, 0, i);
  }
  free(c.omega);
  return 0;
}

/* RHS of alg1 step 2 without dense storage (same arithmetic order as orc_rhs's sums). */
int orc_rhs_nodense(const orc_problem *p, int64_t j, const double *U, double *g) {
  if (!grid_ok(p) || j < 0 || j >= p->M) return -1;
  const int64_t n = p->n;
  const double tau = p->T / (double)p->M;
  const double sigma = 1.0 - p->alpha / 2.0;
  const double kappa = pow(tau, -p->alpha) / tgamma(2.0 - p->alpha);
  orc_matvec(p, j, 1, U + j * n, g);
  if (j >= 1) {
    double *c = (double *)malloc(sizeof(double) * (size_t)(j + 1));
    orc_c_row(p->alpha, j, c);
    for (int64_t s = 0; s <= j - 1; ++s) {
      const double w = kappa * c[j - s];
      for (int64_t i = 0; i < n; ++i) g[i] -= w * (U[(s + 1) * n + i] - U[s * n + i]);
    }
    free(c);
  }
  double *f = (double *)malloc(sizeof(double) * (size_t)n);
  orc_source(p, j, ((double)j + sigma) * tau, f);
  for (int64_t i = 0; i < n; ++i) g[i] += f[i];
  free(f);
  return 0;
}

/* Rows rows[0..nr) of the same RHS (alg1 step 2, eq3.1): B u^j - kappa sum_{s<j} c_{j-s}
 * (u^{s+1} - u^s) + f^{j+sigma}, each row O(n + j). */
int orc_rhs_rows(const orc_problem *p, int64_t j, const double *U, const int64_t *rows, int64_t nr,
                 double *g) {
  if (!grid_ok(p) || j < 0 || j >= p->M) return -1;
  const int64_t n = p->n;
  const double tau = p->T / (double)p->M;
  const double sigma = 1.0 - p->alpha / 2.0;
  const double kappa = pow(tau, -p->alpha) / tgamma(2.0 - p->alpha);
  if (orc_matvec_rows(p, j, 1, U + j * n, rows, nr, g)) return -1;
  if (j >= 1) {
    double *c = (double *)malloc(sizeof(double) * (size_t)(j + 1));
    orc_c_row(p->alpha, j, c);
    for (int64_t s = 0; s <= j - 1; ++s) {
      const double w = kappa * c[j - s];
      for (int64_t k = 0; k < nr; ++k) g[k] -= w * (U[(s + 1) * n + rows[k]] - U[s * n + rows[k]]);
    }
    free(c);
  }
  double *f = (double *)malloc(sizeof(double) * (size_t)n);
  orc_source(p, j, ((double)j + sigma) * tau, f);
  for (int64_t k = 0; k < nr; ++k) g[k] += f[rows[k]];
  free(f);
  return 0;
}

int orc_solve_level(const orc_problem *p, int64_t j, const double *U, double *out) {
  if (!grid_ok(p) || j < 0 || j >= p->M) return -1;
  const int64_t n = p->n;
  double *A = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *B = (double *)malloc(sizeof(double) * (size_t)(n * n));
  orc_assemble(p, j, A, B);
  rhs_with_B(p, j, U, B, out);
  int rc = orc_ge_solve(n, A, out);
  free(A);
  free(B);
  return rc;
}

static int coefficients_constant(const orc_problem *p) {
  return p->gamma.shape == ORC_CONST && p->dplus.shape == ORC_CONST &&
         p->dminus.shape == ORC_CONST;
}

/* alg1: for j = 0..M-1, g = B u^j + delta u^j + f; solve A u^{j+1} = g.
 * The direct solve is GE; when gamma, d+- are constant A is level-invariant for j >= 1
 * (eqgux) and its LU factors are reused.                        */
int orc_solve(const orc_problem *p, double *U) {
  if (!grid_ok(p)) return -1;
  const int64_t n = p->n, M = p->M;
  const double h = (p->b - p->a) / (double)(n + 1);
  for (int64_t i = 0; i < n; ++i) {
    const double x = p->a + (double)(i + 1) * h;
    U[i] = (p->phi_kind == ORC_PHI_X2) ? Xfun(x) : p->phi[i];
  }
  double *A = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *A0 = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *B = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *rhs = (double *)malloc(sizeof(double) * (size_t)n);
  int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  const int reuse = coefficients_constant(p);
  int have_factor = 0;
  int rc = 0;
  for (int64_t j = 0; j < M && rc == 0; ++j) {
    double *g = U + (j + 1) * n;
    if (!(reuse && have_factor && j >= 1)) {
      orc_assemble(p, j, A, B);
      memcpy(A0, A, sizeof(double) * (size_t)(n * n));
      rhs_with_B(p, j, U, B, g);
      rc = lu_factor(n, A, piv);
      if (rc) break;
      if (j >= 1) have_factor = 1;
    } else {
      rhs_with_B(p, j, U, B, g);   /* B is level-invariant too for j >= 1 */
    }
    memcpy(rhs, g, sizeof(double) * (size_t)n);
    lu_solve(n, A, piv, g);
    refine(n, A0, A, piv, rhs, g, 3);
  }
  free(A);
  free(A0);
  free(B);
  free(rhs);
  free(piv);
  return rc;
}

double orc_l2(int64_t n, double h, const double *v) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(h * s);
}

/* ---------------------------------------------------------------------------------- */
/* DFT, SURVEY c18 / SPEC S:170: X_k = sum_m x_m e^{-2 pi i k m / L}; inverse 1/L.    */
void orc_dft(int64_t L, const double *x, double *X, int inverse) {
  const double sgn = inverse ? 1.0 : -1.0;
  for (int64_t k = 0; k < L; ++k) {
    double re = 0.0, im = 0.0;
    for (int64_t m = 0; m < L; ++m) {
      const int64_t e = (k * m) % L;
      const double ang = sgn * 2.0 * M_PI * (double)e / (double)L;
      const double c = cos(ang), s = sin(ang);
      re += x[2 * m] * c - x[2 * m + 1] * s;
      im += x[2 * m] * s + x[2 * m + 1] * c;
    }
    if (inverse) { re /= (double)L; im /= (double)L; }
    X[2 * k] = re;
    X[2 * k + 1] = im;
  }
}

/* Canonical tables (DESIGN.md R-fft, SURVEY 8c "Canonical integer tables"):
 * plan = [4]*(l//2) + ([2] if l odd), stages s = 0..S-1 applied first-to-last (DIT).
 * perm (gather): position p = sum_s d_s prod_{t<s} r_t holds input index
 *                perm[p] = sum_s d_s prod_{t>s} r_t.
 * tw_s[k][q] = (k q L/m_s) mod L, k < m_s/r_s, q < r_s, m_s = prod_{t<=s} r_t.          */
int orc_fft_plan(int64_t L, int32_t *plan) {
  int l = 0;
  while ((1LL << l) < L) ++l;
  int S = 0;
  for (int i = 0; i < l / 2; ++i) plan[S++] = 4;
  if (l % 2) plan[S++] = 2;
  return S;
}

void orc_fft_perm(int64_t L, int32_t *perm) {
  int32_t plan[64];
  const int S = orc_fft_plan(L, plan);
  for (int64_t p = 0; p < L; ++p) {
    int64_t rem = p, idx = 0;
    for (int s = 0; s < S; ++s) {           /* digit d_s of p (weight prod_{t<s} r_t) */
      const int64_t d = rem % plan[s];
      rem /= plan[s];
      int64_t w = 1;
      for (int t = s + 1; t < S; ++t) w *= plan[t];
      idx += d * w;
    }
    perm[p] = (int32_t)idx;
  }
}

int64_t orc_fft_twiddles(int64_t L, int32_t s, int32_t *tw) {
  int32_t plan[64];
  const int S = orc_fft_plan(L, plan);
  if (s < 0 || s >= S) return 0;
  int64_t ms = 1;
  for (int t = 0; t <= s; ++t) ms *= plan[t];
  const int64_t r = plan[s];
  int64_t cnt = 0;
  for (int64_t k = 0; k < ms / r; ++k)
    for (int64_t q = 0; q < r; ++q) tw[cnt++] = (int32_t)((k * q * (L / ms)) % L);
  return cnt;
}

/* Strang: c_k = col[k] for k <= n/2, row[n-k] otherwise.
 * T. Chan: c_k = ((n-k) col[k] + k row[n-k]) / n, row[0] = col[0].          */
void orc_strang_col(int64_t n, const double *col, const double *row, double *c) {
  for (int64_t k = 0; k < n; ++k) c[k] = (k <= n / 2) ? col[k] : row[n - k];
}

void orc_tchan_col(int64_t n, const double *col, const double *row, double *c) {
  c[0] = col[0];
  for (int64_t k = 1; k < n; ++k)
    c[k] = ((double)(n - k) * col[k] + (double)k * row[n - k]) / (double)n;
}

/* ---------------------------------------------------------------------------------- */
/* Timing sample of orc_solve's own steps at the full size n (bench.py cpu_baseline): wall
 * seconds of (t[0]) the dense assembly of A and B, (t[1]) the first kmax column steps of
 * lu_factor, (t[2]) one level's remaining work at history length j: the RHS (dense B u^j,
 * memory term over j rows, source), lu_solve and 3 refinement steps.  The level work is timed on
 * the partially eliminated matrix: its cost does not depend on the values.  U[(j+1)][n].  */
#include <time.h>
static double wall_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
int orc_time_sample(const orc_problem *p, int64_t j, int64_t kmax, const double *U, double *t) {
  if (!grid_ok(p) || j < 0 || j >= p->M || kmax < 1 || kmax > p->n) return -1;
  const int64_t n = p->n;
  double *A = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *A0 = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *B = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *g = (double *)malloc(sizeof(double) * (size_t)n);
  double *rhs = (double *)malloc(sizeof(double) * (size_t)n);
  int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!A || !A0 || !B || !g || !rhs || !piv) return -2;
  double t0 = wall_s();
  orc_assemble(p, j, A, B);
  memcpy(A0, A, sizeof(double) * (size_t)(n * n));
  t[0] = wall_s() - t0;
  t0 = wall_s();
  int rc = lu_factor_k(n, A, piv, kmax);
  t[1] = wall_s() - t0;
  for (int64_t k = kmax; k < n; ++k) piv[k] = k;
  t0 = wall_s();
  rhs_with_B(p, j, U, B, g);
  memcpy(rhs, g, sizeof(double) * (size_t)n);
  lu_solve(n, A, piv, g);
  refine(n, A0, A, piv, rhs, g, 3);
  t[2] = wall_s() - t0;
  free(A); free(A0); free(B); free(g); free(rhs); free(piv);
  return rc;
}
