// tsf_plan.cpp -- host planner (see tsf_plan.h).  Pure C++; no CUDA calls.
#include "tsf_plan.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace tsf {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
const char *last_error() { return g_err.c_str(); }

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

static int fail(const char *fmt, double a = 0, double b = 0) {
  char buf[256];
  std::snprintf(buf, sizeof(buf), fmt, a, b);
  set_error(buf);
  return TSF_E_ARG;
}

static double coef(const double *arr, tsf_fn_t fn, void *ctx, int64_t j, double t, bool *ok) {
  if (arr) return arr[j];
  if (fn) return fn(t, ctx);
  *ok = false;
  return 0.0;
}

int sample_points(const tsf_problem &p, double *x, double *t) {
  // grid of P:221-223 with n interior nodes; t_{j+sigma} = (j + sigma) tau
  const double h = (p.b - p.a) / double(p.n + 1);
  const double sigma = 1.0 - p.alpha / 2.0;
  const double tau = p.T / double(p.M);
  if (x)
    for (int64_t i = 0; i < p.n; ++i) x[i] = p.a + double(i + 1) * h;
  if (t)
    for (int64_t j = 0; j < p.M; ++j) t[j] = (double(j) + sigma) * tau;
  return TSF_OK;
}

static int validate_one(const tsf_problem *p) {
  if (!(p->alpha > 0.0 && p->alpha <= 1.0)) return fail("alpha=%g outside (0,1] (P:74)", p->alpha);
  if (!(p->beta > 1.0 && p->beta <= 2.0)) return fail("beta=%g outside (1,2] (P:74)", p->beta);
  if (!is_pow2(p->n) || p->n < 64 || p->n > kMaxN)
    return fail("n=%g must be a power of two in [64, 1048576]", double(p->n));
  if (p->M < 1) return fail("M=%g must be >= 1", double(p->M));
  if (!(p->b > p->a) || !std::isfinite(p->a) || !std::isfinite(p->b))
    return fail("need a < b (got a=%g, b=%g)", p->a, p->b);
  if (!(p->T > 0.0) || !std::isfinite(p->T)) return fail("T=%g must be > 0", p->T);
  if (!p->phi && !p->phi_fn) return fail("phi: need an array or a callback");
  if (p->src_kind == TSF_SRC_SEPARABLE) {
    if (p->K < 1 || p->K > 4) return fail("separable source needs 1 <= K <= 4 (got %g)", p->K);
    if (!p->basis || !p->scal) return fail("separable source needs basis and scal arrays");
  } else if (p->src_kind == TSF_SRC_TABLE) {
    if (!p->f_table) return fail("table source needs f_table");
  } else if (p->src_kind == TSF_SRC_CALLBACK) {
    if (!p->f_cb) return fail("callback source needs f_cb");
  } else if (p->src_kind != TSF_SRC_ZERO) {
    return fail("unknown src_kind %g", p->src_kind);
  }
  std::vector<double> t(static_cast<size_t>(p->M));
  sample_points(*p, nullptr, t.data());
  for (int64_t j = 0; j < p->M; ++j) {
    bool ok = true;
    const double g = coef(p->gamma_t, p->gamma_fn, p->coef_ctx, j, t[j], &ok);
    const double dp = coef(p->dplus_t, p->dplus_fn, p->coef_ctx, j, t[j], &ok);
    const double dm = coef(p->dminus_t, p->dminus_fn, p->coef_ctx, j, t[j], &ok);
    if (!ok) return fail("gamma/dplus/dminus: need an array or a callback each");
    if (!std::isfinite(g) || !std::isfinite(dp) || !std::isfinite(dm))
      return fail("non-finite coefficient at level %g", double(j));
    if (dp < 0.0 || dm < 0.0)
      return fail("d+- must be >= 0 (P:75-77); got %g at t=%g", std::min(dp, dm), t[j]);
  }
  return TSF_OK;
}

int validate(const tsf_problem *p, int32_t B, const tsf_solver *s) {
  if (!p || !s) return fail("null problem or solver");
  if (B < 1) return fail("B=%g must be >= 1", B);
  for (int32_t b = 0; b < B; ++b) {
    int rc = validate_one(p + b);
    if (rc) return rc;
    if (p[b].n != p[0].n || p[b].M != p[0].M || p[b].src_kind != p[0].src_kind ||
        (p[0].src_kind == TSF_SRC_SEPARABLE && p[b].K != p[0].K) ||
        (p[0].src_kind == TSF_SRC_TABLE && (p[b].f_table_on_device != 0) != (p[0].f_table_on_device != 0)))
      return fail("instance %g: all instances must share n, M, source kind, K and f table residency", b);
    if (p[b].f_table_on_device && p[b].src_kind != TSF_SRC_TABLE)
      return fail("instance %g: f_table_on_device needs the table source", b);
  }
  if (s->method != TSF_BICGSTAB && s->method != TSF_CGNR && s->method != TSF_PCGS && s->method != TSF_GSF) return fail("unknown method %g", s->method);
  if (s->method == TSF_GSF) {
    // alg2 / eqgux: A is level-invariant for j >= 1 only with constant coefficients
    for (int32_t b = 0; b < B; ++b) {
      const tsf_problem &q = p[b];
      std::vector<double> t(static_cast<size_t>(q.M));
      sample_points(q, nullptr, t.data());
      bool ok = true;
      const double g0 = coef(q.gamma_t, q.gamma_fn, q.coef_ctx, 0, t[0], &ok);
      const double p0 = coef(q.dplus_t, q.dplus_fn, q.coef_ctx, 0, t[0], &ok);
      const double m0 = coef(q.dminus_t, q.dminus_fn, q.coef_ctx, 0, t[0], &ok);
      for (int64_t j = 1; j < q.M; ++j)
        if (coef(q.gamma_t, q.gamma_fn, q.coef_ctx, j, t[size_t(j)], &ok) != g0 ||
            coef(q.dplus_t, q.dplus_fn, q.coef_ctx, j, t[size_t(j)], &ok) != p0 ||
            coef(q.dminus_t, q.dminus_fn, q.coef_ctx, j, t[size_t(j)], &ok) != m0)
          return fail("method GSF needs constant gamma, d+, d- (alg2, P:863); instance %g varies at level %g",
                      double(b), double(j));
    }
    if (s->precond == TSF_NOPREC) return fail("method GSF solves eq3.4 with a preconditioner (eqx2xzz, P:893)");
  }
  if (s->precond != TSF_STRANG && s->precond != TSF_TCHAN && s->precond != TSF_NOPREC)
    return fail("unknown preconditioner %g", s->precond);
  if (!(s->tol > 0.0)) return fail("tol=%g must be > 0", s->tol);
  if (s->hist_block != 0 && (!is_pow2(s->hist_block) || s->hist_block < 2 || s->hist_block > 64))
    return fail("hist_block=%g must be 0 or a power of two in [2, 64]", s->hist_block);
  if (s->maxit < 1) return fail("maxit=%g must be >= 1", s->maxit);
  return TSF_OK;
}

// Feasible cluster sizes: local embed FFT fits 128 KiB of shared memory (n/C <= 8192);
// every CTA owns >= 1 preconditioner column pair (n >= 4 C^2); for C > 1 one column-pair
// task per thread (n/(2 C^2) <= 256).
static bool cluster_ok(int64_t n, int C) {
  // local transforms longer than kMaxLocal: the multi-pass regime, on 16-CTA clusters only
  if (n / C > kMaxLocal) return C == 16 && n <= kMaxN;
  if (n < 4LL * C * C) return false;
  // C > 1: staged exchange (local length <= 4096) or one column-pair task per thread
  if (C > 1 && n / C > 4096 && n / (2LL * C * C) > kThreads) return false;
  return true;
}

static size_t up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

int make_plan(const tsf_problem *p, int32_t B, const tsf_solver *s, Plan *pl) {
  int rc = validate(p, B, s);
  if (rc) return rc;
  Plan P;
  P.n = p[0].n;
  P.M = p[0].M;
  P.B = B;
  P.K = p[0].src_kind == TSF_SRC_SEPARABLE ? p[0].K : 0;
  // a callback source is evaluated at tsf_init into the instance's table (slow path)
  P.src_kind = p[0].src_kind == TSF_SRC_CALLBACK ? int32_t(TSF_SRC_TABLE) : p[0].src_kind;
  P.method = s->method;
  P.precond = s->precond;
  P.maxit = s->maxit;
  P.tol = s->tol;
  P.ftab_dev = (p[0].src_kind == TSF_SRC_TABLE && p[0].f_table_on_device) ? 1 : 0;
  P.x0_warm = s->x0_warm ? 1 : 0;
  P.true_res = s->true_residual ? 1 : 0;
  P.pipelined = s->pipelined ? 1 : 0;
  if (const char *ef = std::getenv("TSF_NO_FUSE")) P.fuse = std::atoi(ef) ? 0 : 1;
  P.hblock = s->hist_block;
  const int64_t n = P.n;
  int C = s->cluster;
  if (C == 0) {
    const int cands[5] = {1, 2, 4, 8, 16};
    C = -1;
    for (int c : cands) {
      if (!cluster_ok(n, c)) continue;
      if (C < 0) { C = c; continue; }            // smallest feasible cluster
      // a larger cluster only while the GPU is not yet full and each CTA keeps >= 256 local
      // FFT points (measured at n = 1024: C = 2 / 4 / 8 -> 7.1k / 8.4k / 6.8k levels/s)
      if (int64_t(B) * c <= 148 && n / c >= 256) C = c;
    }
    if (C < 0) return fail("no feasible cluster size for n=%g", double(n));
  } else {
    if (!(C == 1 || C == 2 || C == 4 || C == 8 || C == 16)) return fail("cluster=%g not in {1,2,4,8,16}", C);
    if (!cluster_ok(n, C)) return fail("cluster=%g infeasible for n=%g", C, double(n));
  }
  P.C = C;
  P.L1e = int32_t(n / C);
  P.L1p = int32_t(n / (2 * C));
  P.npe = P.L1e / (2 * C);
  P.npp = P.L1p / (2 * C);
  // staged cross-CTA exchange when three local buffers fit (L1e <= 4096); constant tables
  // resident in SMEM when they fit too (L1e <= 1024)
  P.staged = (C > 1 && P.L1e <= 4096) ? 1 : 0;
  if (const char *es = std::getenv("TSF_STAGED")) P.staged = (C > 1) ? std::atoi(es) : 0;
  P.resident = (P.staged && P.L1e <= 1024) ? 1 : 0;
  if (const char *er = std::getenv("TSF_RESIDENT")) P.resident = P.staged ? std::atoi(er) : 0;
  // multi-pass regime (n > 2^17): each local transform of L1 = R x S points (S <= kMaxLocal)
  // runs as R-point DFTs over stride S and R SMEM FFTs of S points, through the global apply
  // buffer; the column stage is the chunked one through L2.  Vectors live in HBM.
  if (P.L1e > kMaxLocal) {
    P.big = 1;
    P.staged = 0;
    P.resident = 0;
    auto lg = [](int64_t v) { int l = 0; while ((int64_t(1) << l) < v) ++l; return l; };
    P.lre = lg(P.L1e / kMaxLocal);
    P.lrp = P.L1p > kMaxLocal ? lg(P.L1p / kMaxLocal) : 0;
  }
  // Krylov vectors in SMEM when they fit next to the transform buffers (one CTA per SM for
  // clusters; single-CTA instances keep two CTAs per SM)
  {
    const int64_t with = smem_bytes(P.L1e, P.L1p, P.staged, P.resident, 1);
    P.vsmem = (with <= (C > 1 ? kMaxSmem : kMaxSmem / 2 - 1024)) ? 1 : 0;
    if (const char *ev = std::getenv("TSF_VSMEM")) P.vsmem = (with <= kMaxSmem) ? std::atoi(ev) : 0;
    if (P.big) P.vsmem = 0;
  }
  P.smem = smem_bytes(P.L1e, P.L1p, P.staged, P.resident, P.vsmem);
  if (C > 1 && !P.staged) {      // chunk buffer [2 chunk C] + 3 prefetched pair tables [chunk C]:
    int chunk = P.npe;             // the largest power-of-two pair count that fits
    while (chunk > 1 && P.smem + int64_t(5) * chunk * C * 16 > kMaxSmem) chunk /= 2;
    if (const char *ec = std::getenv("TSF_CHUNK")) chunk = std::min(chunk, std::max(1, std::atoi(ec)));
    P.chunk = chunk;
    P.smem = smem_bytes(P.L1e, P.L1p, P.staged, P.resident, P.vsmem, int64_t(5) * chunk * C);
  }
  if (const char *ef = std::getenv("TSF_FUSE_MIN")) P.fuse_min = std::atoi(ef);

  // shared tables
  size_t o = 0;
  P.off_tw = o;      o = up(o + size_t(2 * n) * 16);
  P.off_slot_e = o;  o = up(o + size_t(P.L1e) * 4);
  P.off_slot_p = o;  o = up(o + size_t(P.L1p) * 4);
  P.off_sq_e = o;    o = up(o + size_t(n) * 8);
  P.off_sq_p = o;    o = up(o + size_t(n / 2) * 8);
  P.off_level = o;   o = up(o + 64);
  P.off_sync = o;    o = up(o + 64);
  P.off_pre = o;     o = up(o + (B == 1 ? size_t(2) * size_t(n) * 8 : 0));
  P.off_prof = o;    o = up(o + 32 * 8);
  P.off_fptr = o;    o = up(o + size_t(B) * 8);
  // init scratch (batched spectra FFTs): per instance 2 x (2n + n) complex
  const size_t per = size_t(3 * n) * 16 * 2;
  int32_t batch = int32_t(std::max<int64_t>(1, std::min<int64_t>(B, (256LL << 20) / int64_t(per))));
  P.scratch_batch = batch;
  P.off_scratch = o; P.scratch_bytes = per * size_t(batch); o = up(o + P.scratch_bytes);
  P.off_inst = o;
  // per-instance block
  // host-provided inputs first ([0, o_omega) is one contiguous host image per instance,
  // uploaded for all instances by a single pitched copy), then device-computed tables
  size_t q = 0;
  P.o_par = q;   q = up(q + 128);
  P.o_lev = q;   q = up(q + size_t(P.M) * 32);
  P.o_hwc = q;   q = up(q + size_t(P.M) * 8);
  P.o_hwe = q;   q = up(q + size_t(P.M) * 8);
  P.o_scal = q;  q = up(q + size_t(P.M) * size_t(std::max(P.K, 1)) * 8);
  P.o_basis = q; q = up(q + size_t(std::max(P.K, 1)) * size_t(n) * 8);
  P.o_ftab = q;  q = up(q + (P.src_kind == TSF_SRC_TABLE && !P.ftab_dev ? size_t(P.M) * size_t(n) * 8 : 0));
  P.o_phi = q;   q = up(q + size_t(n) * 8);
  P.o_omega = q; q = up(q + size_t(n + 2) * 8);
  P.o_lwe = q;   q = up(q + size_t(n + 1) * 16);
  P.o_lwp = q;   q = up(q + size_t(n / 2 + 1) * 16);
  P.o_vec = q;   q = up(q + size_t(kNumVec) * size_t(n) * 8);
  P.o_hist = q;  q = up(q + size_t(P.M) * size_t(n) * 8);
  P.o_it = q;    q = up(q + size_t(P.M) * 4);
  P.o_rr = q;    q = up(q + size_t(P.M) * 8);
  P.o_trr = q;   q = up(q + size_t(P.M) * 8);
  P.o_st = q;    q = up(q + size_t(P.M) * 4);
  P.o_mul = q;   q = up(q + size_t(n + n / 2) * 16);
  P.o_gsf = q;   q = up(q + (s->method == TSF_GSF ? size_t(4) * size_t(n + 1) * 16 : 0));
  P.o_xg = q;    q = up(q + (C > 1 && !P.staged ? size_t(n) * 16 : 0));   // L2 exchange (unstaged)
  P.o_xa = q;    q = up(q + (P.big ? size_t(n) * 16 : 0));                 // apply buffer (multi-pass)
  P.o_hb = q;    q = up(q + size_t(P.hblock) * size_t(n) * 8);             // blocked history sums
  P.stride = q;
  P.total = P.off_inst + P.stride * size_t(B);
  *pl = P;
  return TSF_OK;
}

int inst_tables(const tsf_problem &p, InstTables *out) {
  const int64_t M = p.M;
  const double alpha = p.alpha, sigma = 1.0 - alpha / 2.0;
  const double tau = p.T / double(M);
  const double h = (p.b - p.a) / double(p.n + 1);
  // Lemma 1
  std::vector<double> a(static_cast<size_t>(M + 2)), b(size_t(M + 2), 0.0);
  a[0] = std::pow(sigma, 1.0 - alpha);
  for (int64_t l = 1; l <= M + 1; ++l) {
    const double hi = double(l) + sigma, lo = double(l - 1) + sigma;
    a[size_t(l)] = std::pow(hi, 1.0 - alpha) - std::pow(lo, 1.0 - alpha);
    b[size_t(l)] = (std::pow(hi, 2.0 - alpha) - std::pow(lo, 2.0 - alpha)) / (2.0 - alpha) -
                   0.5 * (std::pow(hi, 1.0 - alpha) + std::pow(lo, 1.0 - alpha));
  }
  const double kappa = std::pow(tau, -alpha) / std::tgamma(2.0 - alpha);
  out->sigma = sigma;
  out->kappa = kappa;
  out->h = h;
  out->tau = tau;
  out->lev.assign(size_t(4 * M), 0.0);
  out->hwc.assign(size_t(M), 0.0);
  out->hwe.assign(size_t(M), 0.0);
  std::vector<double> t(static_cast<size_t>(M));
  sample_points(p, nullptr, t.data());
  const double hb = std::pow(h, p.beta);
  for (int64_t j = 0; j < M; ++j) {
    bool ok = true;
    const double g = coef(p.gamma_t, p.gamma_fn, p.coef_ctx, j, t[size_t(j)], &ok);
    const double dp = coef(p.dplus_t, p.dplus_fn, p.coef_ctx, j, t[size_t(j)], &ok);
    const double dm = coef(p.dminus_t, p.dminus_fn, p.coef_ctx, j, t[size_t(j)], &ok);
    // eta_j: c_0^{(j)} kappa with c_0^{(0)} = a_0, c_0^{(j>=1)} = a_0 + b_1
    const double eta = (j == 0 ? a[0] : a[0] + b[1]) * kappa;
    out->lev[size_t(4 * j + 0)] = eta;
    out->lev[size_t(4 * j + 1)] = g / (2.0 * h);
    out->lev[size_t(4 * j + 2)] = dp / hb;
    out->lev[size_t(4 * j + 3)] = dm / hb;
    // history weights (Lemma 1): c_m^{(j)} = a_m + b_{m+1} - b_m for
    // 1 <= m <= j-1 (independent of j) and c_j^{(j)} = a_j - b_j for the d^0 term.
    if (j >= 1) {
      out->hwc[size_t(j)] = kappa * (a[size_t(j)] + b[size_t(j + 1)] - b[size_t(j)]);
      out->hwe[size_t(j)] = kappa * (a[size_t(j)] - b[size_t(j)]);
    }
  }
  return TSF_OK;
}

// ---- FFT tables (DESIGN.md R-fft) -------------------------------------------------------
int fft_plan_radices(int64_t L, int32_t *plan) {
  int l = 0;
  while ((int64_t(1) << l) < L) ++l;
  int S = 0;
  for (int i = 0; i < l / 2; ++i) plan[S++] = 4;
  if (l & 1) plan[S++] = 2;
  return S;
}

void fft_perm(int64_t L, int32_t *perm) {
  // gather digit reversal: buffer position p = sum_s d_s prod_{t<s} r_t holds input
  // index sum_s d_s prod_{t>s} r_t.  Built by digit recursion over the stages.
  int32_t plan[32];
  const int S = fft_plan_radices(L, plan);
  std::vector<int64_t> wt(size_t(S) + 1, 1);     // wt[s] = prod_{t>s} r_t
  for (int s = S - 1; s >= 0; --s) wt[size_t(s)] = (s + 1 < S ? wt[size_t(s + 1)] * plan[s + 1] : 1);
  for (int64_t p = 0; p < L; ++p) {
    int64_t rem = p, idx = 0;
    for (int s = 0; s < S; ++s) {
      idx += (rem % plan[s]) * wt[size_t(s)];
      rem /= plan[s];
    }
    perm[p] = int32_t(idx);
  }
}

int64_t fft_stage_twiddles(int64_t L, int s, int32_t *tw) {
  int32_t plan[32];
  const int S = fft_plan_radices(L, plan);
  if (s < 0 || s >= S) return 0;
  int64_t ms = 1;
  for (int t = 0; t <= s; ++t) ms *= plan[t];
  const int64_t r = plan[s], stride = L / ms;
  int64_t c = 0;
  for (int64_t k = 0; k < ms / r; ++k)
    for (int64_t q = 0; q < r; ++q) tw[c++] = int32_t(((k * q) % L) * stride % L);
  return c;
}

DevParams dev_params(const Plan &pl, char *ws) {
  DevParams d;
  std::memset(&d, 0, sizeof(d));
  d.n = pl.n; d.M = pl.M; d.B = pl.B; d.C = pl.C; d.K = pl.K; d.src_kind = pl.src_kind;
  d.method = pl.method; d.precond = pl.precond; d.maxit = pl.maxit;
  d.L1e = pl.L1e; d.L1p = pl.L1p; d.npe = pl.npe; d.npp = pl.npp;
  d.staged = pl.staged; d.resident = pl.resident; d.vsmem = pl.vsmem; d.fuse_min = pl.fuse_min; d.chunk = pl.chunk;
  d.big = pl.big; d.lre = pl.lre; d.lrp = pl.lrp; d.o_xa = pl.o_xa;
  d.tol = pl.tol;
  d.scale_e = 1.0 / (4.0 * double(pl.n));
  d.scale_p = 1.0 / (4.0 * double(pl.n / 2));
  d.qscale_p = pl.precond == TSF_TCHAN ? double(pl.n - 1) / double(pl.n) : 1.0;
  d.strang = pl.precond == TSF_STRANG;
  d.twN = int32_t(2 * pl.n);
  d.tw = ws + pl.off_tw;
  d.slot_e = reinterpret_cast<const int32_t *>(ws + pl.off_slot_e);
  d.slot_p = reinterpret_cast<const int32_t *>(ws + pl.off_slot_p);
  d.sq_e = reinterpret_cast<const double *>(ws + pl.off_sq_e);
  d.sq_p = reinterpret_cast<const double *>(ws + pl.off_sq_p);
  d.level = reinterpret_cast<int64_t *>(ws + pl.off_level);
  d.sync = reinterpret_cast<int64_t *>(ws + pl.off_sync);
  d.pre = reinterpret_cast<double *>(ws + pl.off_pre);
  d.helpers = 0;
  d.prof = reinterpret_cast<unsigned long long *>(ws + pl.off_prof);
  d.inst = ws + pl.off_inst;
  d.stride = int64_t(pl.stride);
  d.o_par = pl.o_par; d.o_omega = pl.o_omega; d.o_lwe = pl.o_lwe; d.o_lwp = pl.o_lwp;
  d.o_lev = pl.o_lev; d.o_hwc = pl.o_hwc; d.o_hwe = pl.o_hwe; d.o_scal = pl.o_scal;
  d.o_basis = pl.o_basis; d.o_ftab = pl.o_ftab; d.o_vec = pl.o_vec; d.o_hist = pl.o_hist;
  d.o_it = pl.o_it; d.o_rr = pl.o_rr; d.o_trr = pl.o_trr; d.o_st = pl.o_st; d.o_phi = pl.o_phi;
  d.fptr = reinterpret_cast<const double *const *>(ws + pl.off_fptr);
  d.ftab_dev = pl.ftab_dev;
  d.x0_warm = pl.x0_warm;
  d.true_res = pl.true_res;
  d.pipelined = pl.pipelined;
  d.fuse = pl.fuse;
  d.hblock = pl.hblock; d.o_hb = pl.o_hb; d.o_mul = pl.o_mul; d.o_gsf = pl.o_gsf; d.o_xg = pl.o_xg;
  return d;
}

}  // namespace tsf
