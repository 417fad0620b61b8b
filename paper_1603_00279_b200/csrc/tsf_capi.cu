// tsf_capi.cu -- C-ABI (include/tsf.h) of the B200 per-level solver: one-time setup
// kernels (WSGD weights, circulant spectra), launches of the fused solve kernel, CUDA-graph
// level step, statistics and test hooks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tsf_kernels.cuh"
#include "tsf_plan.h"

using namespace tsf;

namespace tsf {
__global__ void k_advance(int64_t *level, int64_t by, int64_t M) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t v = *level + by;
    *level = v < M ? v : M;
  }
}
}  // namespace tsf

struct tsf_handle {
  Plan pl;
  DevParams dp;
  char *ws = nullptr;
  int device = 0;
  cudaStream_t st = nullptr;
  cudaGraphExec_t step_exec = nullptr;
  cudaGraph_t step_graph = nullptr;
  int64_t level = 0;
};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
      return TSF_E_CUDA;                                                                 \
    }                                                                                    \
  } while (0)

namespace {

// ---------------------------------------------------------------------- setup kernels
__global__ void k_twiddle(double2 *tw, int twN) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < twN; e += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(2.0 * double(e) / double(twN), &s, &c);
    tw[e] = make_double2(c, -s);                 // exp(-2 pi i e / twN)
  }
}

// sine tables of Lambda_Q in task order: sin(fac * pi * bin / n)
__global__ void k_sq(double *sq, int L1, int C, int np, int64_t n, double fac) {
  const int total = C * C * 2 * np;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int i = idx % np, ab = (idx / np) % 2, k2 = (idx / (2 * np)) % C, r = idx / (2 * np * C);
    const int64_t bin = task_bin(L1, C, r, i, k2, ab);
    sq[idx] = sinpi(fac * double(bin) / double(n));
  }
}

// WSGD weights (Lemma 2) from the Grunwald recurrence (Lemma 3):
// g_0 = 1, g_k = (1 - (beta+1)/k) g_{k-1}; omega_0 = l1 g_0, omega_1 = l1 g_1 + l0 g_0,
// omega_k = l1 g_k + l0 g_{k-1} + l-1 g_{k-2}.
__device__ void wsgd_gen(double beta, int64_t K, double *g, double *omega) {
  const double l1 = (beta * beta + 3.0 * beta + 2.0) / 12.0;
  const double l0 = (4.0 - beta * beta) / 6.0;
  const double lm1 = (beta * beta - 3.0 * beta + 2.0) / 12.0;
  double gm2 = 0.0, gm1 = 0.0, gk = 1.0;
  for (int64_t k = 0; k <= K; ++k) {
    if (k > 0) {
      gm2 = gm1;
      gm1 = gk;
      gk = (1.0 - (beta + 1.0) / double(k)) * gm1;
    }
    if (g) g[k] = gk;
    double w = l1 * gk;
    if (k >= 1) w += l0 * gm1;
    if (k >= 2) w += lm1 * gm2;
    omega[k] = w;
  }
}

__global__ void k_weights(DevParams P) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P.B) return;
  Inst I = inst_view(P, b);
  wsgd_gen(I.par[1], P.n + 1, nullptr, I.omega);
  I.par[2] = I.omega[P.n / 2 + 1];
}

__global__ void k_dbg_weights(double beta, int64_t K, double *g, double *omega) {
  if (blockIdx.x == 0 && threadIdx.x == 0) wsgd_gen(beta, K, g, omega);
}

// Generators (first columns) of the circulants whose spectra are needed once:
//  embedding of W (2n): [w1 .. wn, 0, 0 .. 0, w0]   (eq3.2)
//  Strang s(W) (n): c_k = t_k (k <= n/2), t_{k-n} (k > n/2)
//  T. Chan c(W) (n): c_k = ((n-k) t_k + k t_{k-n}) / n
// with t_k = omega_{k+1} (k >= -1), t_{-k} = 0 (k >= 2).
__global__ void k_cols(DevParams P, int b0, int nb, double2 *emb, double2 *pre) {
  const int64_t n = P.n;
  const int64_t total = int64_t(nb) * 2 * n;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int bb = int(id / (2 * n));
    const int64_t m = id % (2 * n);
    const Inst I = inst_view(P, b0 + bb);
    const double *w = I.omega;
    double e = 0.0;
    if (m < n) e = w[m + 1];
    else if (m == 2 * n - 1) e = w[0];
    emb[id] = make_double2(e, 0.0);
    if (m < n && P.precond != TSF_NOPREC) {
      const int64_t k = m;
      double c = 0.0;
      if (P.precond == TSF_STRANG) {
        if (k <= n / 2) c = w[k + 1];
        else if (k == n - 1) c = w[0];
      } else {
        c = (double(n - k) * w[k + 1] + (k == n - 1 ? double(k) * w[0] : 0.0)) / double(n);
      }
      pre[int64_t(bb) * n + k] = make_double2(c, 0.0);
    }
  }
}

// Radix-2 Stockham autosort pass (natural order in and out after all passes), batched.
__global__ void k_stockham(const double2 *in, double2 *out, int64_t L, int lNs, int nb,
                           const double2 *tw, int twN) {
  const int64_t half = L / 2;
  const int64_t total = half * nb;
  const int64_t Ns = int64_t(1) << lNs;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = id / half, j = id % half;
    const double2 *x = in + b * L;
    double2 *y = out + b * L;
    const int64_t k = j & (Ns - 1);
    const double2 w = tw[k * (twN / (2 * Ns))];
    const double2 v0 = x[j], v1 = cmul(x[j + half], w);
    const int64_t d = ((j >> lNs) << (lNs + 1)) + k;
    y[d] = cadd(v0, v1);
    y[d + Ns] = csub(v0, v1);
  }
}

__global__ void k_scatter_spec(DevParams P, int b0, int nb, const double2 *emb, const double2 *pre) {
  const int64_t n = P.n;
  const int C = P.C;
  const int64_t total = int64_t(nb) * (n + 1 + n / 2 + 1);
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int bb = int(id / (n + 1 + n / 2 + 1));
    int64_t idx = id % (n + 1 + n / 2 + 1);
    Inst I = inst_view(P, b0 + bb);
    if (idx <= n) {
      int64_t bin = n;
      if (idx < n) {
        const int np = P.npe;
        const int i = int(idx % np), ab = int((idx / np) % 2), k2 = int((idx / (2 * np)) % C);
        const int r = int(idx / (2 * np * C));
        bin = task_bin(P.L1e, C, r, i, k2, ab);
      }
      I.lwe[idx] = emb[int64_t(bb) * 2 * n + bin];
    } else if (P.precond != TSF_NOPREC) {
      idx -= n + 1;
      int64_t bin = n / 2;
      if (idx < n / 2) {
        const int np = P.npp;
        const int i = int(idx % np), ab = int((idx / np) % 2), k2 = int((idx / (2 * np)) % C);
        const int r = int(idx / (2 * np * C));
        bin = task_bin(P.L1p, C, r, i, k2, ab);
      }
      I.lwp[idx] = pre[int64_t(bb) * n + bin];
    }
  }
}

__global__ void k_reset(DevParams P) {
  const int64_t n = P.n;
  const int64_t per = n + 4 * P.M;
  const int64_t total = per * P.B;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(id / per);
    const int64_t k = id % per;
    Inst I = inst_view(P, b);
    if (k < n) I.vec[V_U * n + k] = I.phi[k];
    else if (k < n + P.M) I.it[k - n] = 0;
    else if (k < n + 2 * P.M) I.rr[k - n - P.M] = 0.0;
    else if (k < n + 3 * P.M) I.trr[k - n - 2 * P.M] = 0.0;
    else I.st[k - n - 3 * P.M] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *P.level = 0;
}

// Host source table (eq3.1 f^{j+sigma}): rows arrive in natural order (staged in the
// instance's still-unused history block) and are stored in the chunk order of the kernels.
__global__ void k_permute_rows(const double *__restrict__ nat, double *__restrict__ out, int64_t n, int64_t M, int C) {
  const int64_t total = n * M;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = id / n, e = id % n;
    out[j * n + perm_pos(n, C, e)] = nat[id];
  }
}

// Nonsingularity guard of the circulant preconditioner (themx2 P:831-848 proves
// P nonsingular in exact arithmetic): for every (instance, level) block, min and max |lambda_P|
// over the n/2 + 1 bins of the level's spectrum; |lambda_P| < 1e-14 max |lambda_P| marks the
// level TSF_LEVEL_SINGULAR_PREC (tsf_init then fails with TSF_E_SINGULAR_PREC).
__global__ void k_prec_guard(DevParams P) {
  const int b = int(blockIdx.x / P.M);
  const int64_t j = blockIdx.x % P.M;
  const Inst I = inst_view(P, b);
  const Smem none = {};
  const SpecOp op = make_op(P, I, j, OP_PINV, 0, none);
  const int64_t half = P.n / 2;
  const int C = P.C, np = P.npp;
  double lo = INFINITY, hi = 0.0;
  for (int64_t q = threadIdx.x; q <= half; q += blockDim.x) {
    double2 l;
    if (q == half) {
      l = op.nyquist_lam(int(half));
    } else {
      const int i = int(q % np), ab = int((q / np) % 2), k2 = int((q / (2 * np)) % C);
      const int r = int(q / (2 * np * C));
      l = op.lam_idx(int(q), int(task_bin(P.L1p, C, r, i, k2, ab)));
    }
    const double m2 = l.x * l.x + l.y * l.y;
    lo = fmin(lo, m2);
    hi = fmax(hi, m2);
  }
  __shared__ double slo[32], shi[32];
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) { lo = fmin(lo, slo[w]); hi = fmax(hi, shi[w]); }
    lo = fmin(lo, slo[0]);
    hi = fmax(hi, shi[0]);
    if (!(lo >= 1e-28 * hi) || !(hi > 0.0)) I.st[j] = TSF_LEVEL_SINGULAR_PREC;   // |l| < 1e-14 max|l|
  }
}

// u^j of instances [b0, b0 + nb) in natural order (device output of tsf_get_solution(s))
__global__ void k_gather_u(DevParams P, int b0, int nb, double *out) {
  const int64_t n = P.n;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < int64_t(nb) * n;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(id / n);
    const int64_t e = id % n;
    const Inst I = inst_view(P, b0 + b);
    out[id] = I.vec[V_U * n + perm_pos(n, P.C, e)];
  }
}

__global__ void k_set_level(int64_t *level, int64_t v) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *level = v;
}

__global__ void k_dbg_fft(double2 *buf, int L, const double2 *tw, int twN, int inverse) {
  extern __shared__ __align__(16) unsigned char raw[];
  const Smem sm = smem_view(raw, L, L / 2, false, false, false, nullptr);
  const int f = twN / L;
  for (int i = threadIdx.x; i < tw_lo_len(L); i += blockDim.x) sm.tlo[i] = tw[i * f];
  for (int i = threadIdx.x; i < tw_hi_len(L); i += blockDim.x) sm.thi[i] = tw[(i << 6) * f];
  for (int e = threadIdx.x; e < L; e += blockDim.x) sm.A[pidx(e)] = buf[e];
  __syncthreads();
  if (inverse) local_fft<true>(sm.A, L, sm, L);
  else local_fft<false>(sm.A, L, sm, L);
  for (int e = threadIdx.x; e < L; e += blockDim.x) buf[e] = sm.A[pidx(e)];
}

// per-level spectra of one instance in natural bin order
__global__ void k_dbg_spectra(DevParams P, int b, int64_t j, double2 *lamA, double2 *lamP) {
  const Inst I = inst_view(P, b);
  const int64_t n = P.n;
  const int C = P.C;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx <= n + n / 2 + 1;
       idx += int64_t(gridDim.x) * blockDim.x) {
    if (idx <= n && lamA) {
      const Smem none = {};
      SpecOp op = make_op(P, I, j, OP_A, 0, none);
      if (idx == n) { lamA[n] = op.nyquist_lam(int(n)); continue; }
      const int np = P.npe;
      const int i = int(idx % np), ab = int((idx / np) % 2), k2 = int((idx / (2 * np)) % C);
      const int r = int(idx / (2 * np * C));
      const int64_t bin = task_bin(P.L1e, C, r, i, k2, ab);
      lamA[bin] = op.lam_idx(int(idx), int(bin));
    } else if (idx > n && lamP && P.precond != TSF_NOPREC) {
      const int64_t q = idx - n - 1;
      const Smem none = {};
      SpecOp op = make_op(P, I, j, OP_PINV, 0, none);
      if (q == n / 2) { lamP[n / 2] = op.nyquist_lam(int(n / 2)); continue; }
      const int np = P.npp;
      const int i = int(q % np), ab = int((q / np) % 2), k2 = int((q / (2 * np)) % C);
      const int r = int(q / (2 * np * C));
      const int64_t bin = task_bin(P.L1p, C, r, i, k2, ab);
      lamP[bin] = op.lam_idx(int(q), int(bin));
    }
  }
}

// ---------------------------------------------------------------------- launch helpers
cudaError_t launch_solve(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st, int32_t mode = 0) {
  switch (pl.C) {
    case 1: return launch_solve_c<1>(pl, dp, nlev, st, mode);
    case 2: return launch_solve_c<2>(pl, dp, nlev, st, mode);
    case 4: return launch_solve_c<4>(pl, dp, nlev, st, mode);
    case 8: return launch_solve_c<8>(pl, dp, nlev, st, mode);
    case 16: return launch_solve_c<16>(pl, dp, nlev, st, mode);
  }
  return cudaErrorInvalidValue;
}

// NEXT-2: 2n circulant embeddings (R-emb) of the four triangular Toeplitz factors of the
// Gohberg-Semencul formula from x = A^{-1} e_1 (V_GX) and y = A^{-1} e_n (V_GY),
// natural element e stored at perm_pos(n, C, e):
//   k = 0  R_p^0 upper, first row [0, x_{n-1}, .., x_1]   c[n+t] = x_t      (t = 1..n-1)
//   k = 1  R_p   upper, first row [y_{n-1}, .., y_0]      c[0] = y_{n-1}, c[n+t] = y_{t-1}
//   k = 2  L_p^0 lower, first col [0, y_0, .., y_{n-2}]   c[m] = y_{m-1}    (m = 1..n-1)
//   k = 3  L_p   lower, first col [x_0, .., x_{n-1}]      c[m] = x_m        (m < n)
// and 1/xi_0 = 1/x_0 into par[7].
__global__ void k_gsf_cols(DevParams P, int b0, int nb, int k, double2 *emb) {
  const int64_t n = P.n;
  const int64_t total = int64_t(nb) * 2 * n;
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int bb = int(id / (2 * n));
    const int64_t m = id % (2 * n);
    const Inst I = inst_view(P, b0 + bb);
    const double *x = I.vec + int64_t(V_GX) * n, *y = I.vec + int64_t(V_GY) * n;
    auto X = [&](int64_t e) { return x[perm_pos(n, P.C, e)]; };
    auto Y = [&](int64_t e) { return y[perm_pos(n, P.C, e)]; };
    double c = 0.0;
    if (k == 0) c = (m > n) ? X(m - n) : 0.0;
    else if (k == 1) c = (m == 0) ? Y(n - 1) : ((m > n) ? Y(m - n - 1) : 0.0);
    else if (k == 2) c = (m >= 1 && m < n) ? Y(m - 1) : 0.0;
    else c = (m < n) ? X(m) : 0.0;
    emb[id] = make_double2(c, 0.0);
    if (k == 0 && m == 0) I.par[7] = 1.0 / X(0);
  }
}

// spectrum (natural bins 0..n of a length-2n transform) -> task order table k of I.gsf
__global__ void k_gsf_scatter(DevParams P, int b0, int nb, int k, const double2 *spec) {
  const int64_t n = P.n;
  const int C = P.C;
  const int64_t total = int64_t(nb) * (n + 1);
  for (int64_t id = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; id < total;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int bb = int(id / (n + 1));
    const int64_t idx = id % (n + 1);
    Inst I = inst_view(P, b0 + bb);
    int64_t bin = n;
    if (idx < n) {
      const int np = P.npe;
      const int i = int(idx % np), ab = int((idx / np) % 2), k2 = int((idx / (2 * np)) % C);
      const int r = int(idx / (2 * np * C));
      bin = task_bin(P.L1e, C, r, i, k2, ab);
    }
    I.gsf[int64_t(k) * (n + 1) + idx] = spec[int64_t(bb) * 2 * n + bin];
  }
}

cudaError_t launch_dbg_apply(const Plan &pl, const DevParams &dp, int b, int64_t j, int which,
                             const double *in, double *out, cudaStream_t st, int32_t reps = 0) {
  switch (pl.C) {
    case 1: return launch_dbg_apply_c<1>(pl, dp, b, j, which, in, out, st, reps);
    case 2: return launch_dbg_apply_c<2>(pl, dp, b, j, which, in, out, st, reps);
    case 4: return launch_dbg_apply_c<4>(pl, dp, b, j, which, in, out, st, reps);
    case 8: return launch_dbg_apply_c<8>(pl, dp, b, j, which, in, out, st, reps);
    case 16: return launch_dbg_apply_c<16>(pl, dp, b, j, which, in, out, st, reps);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_dbg_rhs(const Plan &pl, const DevParams &dp, cudaStream_t st) {
  switch (pl.C) {
    case 1: return launch_dbg_rhs_c<1>(pl, dp, st);
    case 2: return launch_dbg_rhs_c<2>(pl, dp, st);
    case 4: return launch_dbg_rhs_c<4>(pl, dp, st);
    case 8: return launch_dbg_rhs_c<8>(pl, dp, st);
    case 16: return launch_dbg_rhs_c<16>(pl, dp, st);
  }
  return cudaErrorInvalidValue;
}

int grid_for(int64_t work) {
  int64_t g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return int(g);
}

void permute_host(int64_t n, int C, const double *nat, double *perm) {
  for (int64_t e = 0; e < n; ++e) perm[perm_pos(n, C, e)] = nat[e];
}
void unpermute_host(int64_t n, int C, const double *perm, double *nat) {
  for (int64_t e = 0; e < n; ++e) nat[e] = perm[perm_pos(n, C, e)];
}

double *inst_ptr(tsf_handle *h, int b, int64_t off) {
  return reinterpret_cast<double *>(h->ws + h->pl.off_inst + size_t(b) * h->pl.stride + size_t(off));
}

int level_status_to_rc(int32_t s) {
  switch (s) {
    case TSF_LEVEL_OK: return TSF_OK;
    case TSF_LEVEL_MAXIT: return TSF_W_MAXIT;
    case TSF_LEVEL_BREAKDOWN: return TSF_E_BREAKDOWN;
    case TSF_LEVEL_DIVERGED: return TSF_E_DIVERGED;
    case TSF_LEVEL_SINGULAR_PREC: return TSF_E_SINGULAR_PREC;
  }
  return TSF_E_DIVERGED;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char *tsf_last_error(void) { return last_error(); }

int tsf_sample_points(const tsf_problem *p, double *x, double *t) {
  if (!p) { set_error("null problem"); return TSF_E_ARG; }
  if (!(p->alpha > 0.0 && p->alpha <= 1.0) || p->n < 1 || p->M < 1 || !(p->b > p->a) || !(p->T > 0.0)) {
    set_error("invalid alpha/n/M/[a,b]/T");
    return TSF_E_ARG;
  }
  return sample_points(*p, x, t);
}

int tsf_plan(const tsf_problem *p, int32_t B, const tsf_solver *s, tsf_plan_info *info) {
  Plan pl;
  int rc = make_plan(p, B, s, &pl);
  if (rc) return rc;
  if (info) {
    info->cluster = pl.C;
    info->threads = kThreads;
    info->smem_bytes = pl.smem;
    info->embed_len = pl.n;
    info->precond_len = pl.n / 2;
    info->workspace_bytes = pl.total;
    info->exchange = pl.C == 1 ? 0 : (pl.staged ? 1 : (pl.big ? 3 : 2));
    info->chunk = pl.chunk;
    info->vsmem = pl.vsmem;
    info->resident = pl.resident;
  }
  return TSF_OK;
}

int tsf_workspace_bytes(const tsf_problem *p, int32_t B, const tsf_solver *s, size_t *bytes) {
  tsf_plan_info info;
  int rc = tsf_plan(p, B, s, &info);
  if (rc) return rc;
  if (!bytes) { set_error("null bytes"); return TSF_E_ARG; }
  *bytes = info.workspace_bytes;
  return TSF_OK;
}

int tsf_init(const tsf_problem *p, int32_t B, const tsf_solver *s, void *d_ws, size_t ws_bytes,
             int device, void *cuda_stream, tsf_handle **out) {
  if (!out) { set_error("null out"); return TSF_E_ARG; }
  *out = nullptr;
  Plan pl;
  int rc = make_plan(p, B, s, &pl);
  if (rc) return rc;
  if (!d_ws || ws_bytes < pl.total || (reinterpret_cast<uintptr_t>(d_ws) % kAlign) != 0) {
    set_error("workspace: need " + std::to_string(pl.total) + " bytes, 256-byte aligned");
    return TSF_E_WORKSPACE;
  }
  CK(cudaSetDevice(device));
  tsf_handle *h = new tsf_handle();
  h->pl = pl;
  h->ws = static_cast<char *>(d_ws);
  h->device = device;
  h->st = static_cast<cudaStream_t>(cuda_stream);
  h->dp = dev_params(pl, h->ws);
  const DevParams &dp = h->dp;
  const int64_t n = pl.n, M = pl.M;
  cudaStream_t st = h->st;
  auto bail = [&](int code) { delete h; return code; };
#define CKH(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
      return bail(TSF_E_CUDA);                                                           \
    }                                                                                    \
  } while (0)

  // shared integer tables: slot[k1] = inverse of the gather digit reversal (R-fft)
  {
    std::vector<int32_t> perm(static_cast<size_t>(pl.L1e)), slot(static_cast<size_t>(pl.L1e));
    fft_perm(pl.L1e, perm.data());
    for (int32_t p2 = 0; p2 < pl.L1e; ++p2) slot[size_t(perm[size_t(p2)])] = p2;
    CKH(cudaMemcpyAsync(h->ws + pl.off_slot_e, slot.data(), size_t(pl.L1e) * 4, cudaMemcpyHostToDevice, st));
    std::vector<int32_t> permp(static_cast<size_t>(pl.L1p)), slotp(static_cast<size_t>(pl.L1p));
    fft_perm(pl.L1p, permp.data());
    for (int32_t p2 = 0; p2 < pl.L1p; ++p2) slotp[size_t(permp[size_t(p2)])] = p2;
    CKH(cudaMemcpyAsync(h->ws + pl.off_slot_p, slotp.data(), size_t(pl.L1p) * 4, cudaMemcpyHostToDevice, st));
  }
  CKH(cudaMemsetAsync(h->ws + pl.off_inst, 0, pl.stride * size_t(B), st));
  CKH(cudaMemsetAsync(h->ws + pl.off_level, 0, 64, st));
  k_twiddle<<<grid_for(2 * n), 256, 0, st>>>(reinterpret_cast<double2 *>(h->ws + pl.off_tw), int(2 * n));
  k_sq<<<grid_for(n), 256, 0, st>>>(reinterpret_cast<double *>(h->ws + pl.off_sq_e), pl.L1e, pl.C, pl.npe, n, 1.0);
  k_sq<<<grid_for(n / 2), 256, 0, st>>>(reinterpret_cast<double *>(h->ws + pl.off_sq_p), pl.L1p, pl.C, pl.npp, n, 2.0);
  CKH(cudaGetLastError());

  // Per-instance inputs.  Every host-provided field of an instance block lies in [0, o_omega)
  // (par, level tables, history weights, source, phi): they are written into ONE host image per
  // instance (permuted chunks where the kernels want them) and uploaded by pitched copies on the
  // handle's stream, ordered after the zeroing memset above (pageable source: cudaMemcpy2DAsync
  // returns once the image is staged, so it may be freed after).  A host f table (the bulk of
  // the input: M x n doubles) is left out of the image: it goes straight from the caller's
  // buffer (one DMA per instance when that buffer is pinned) into the instance's history
  // block, which nothing reads before level 1, and k_permute_rows moves it into the table in
  // chunk order; the history block is zeroed again afterwards.  u^0 = phi is then set on the
  // device by k_reset.  A device f table is borrowed (R-ftab).
  {
    const bool tab_host = pl.src_kind == TSF_SRC_TABLE && !pl.ftab_dev && p[0].src_kind == TSF_SRC_TABLE;
    const int64_t gap = tab_host ? int64_t(pl.o_phi) - int64_t(pl.o_ftab) : 0;   // table bytes left out
    const size_t img = size_t(int64_t(pl.o_omega) - gap);
    std::vector<char> himg(img * size_t(B), 0);
    std::vector<double> tmp(static_cast<size_t>(std::max<int64_t>(n, 8))), xs(static_cast<size_t>(n));
    std::vector<double> tl(static_cast<size_t>(M));
    for (int32_t b = 0; b < B; ++b) {
      const tsf_problem &q = p[b];
      char *base = himg.data() + size_t(b) * img;
      auto at = [&](int64_t off) { return reinterpret_cast<double *>(base + (off >= int64_t(pl.o_phi) ? off - gap : off)); };
      InstTables T;
      inst_tables(q, &T);
      double par[16] = {T.sigma, q.beta, 0.0, T.kappa, T.h, T.tau, 0.0, 0.0};
      std::memcpy(at(pl.o_par), par, sizeof(par));
      std::memcpy(at(pl.o_lev), T.lev.data(), T.lev.size() * 8);
      std::memcpy(at(pl.o_hwc), T.hwc.data(), T.hwc.size() * 8);
      std::memcpy(at(pl.o_hwe), T.hwe.data(), T.hwe.size() * 8);
      sample_points(q, xs.data(), tl.data());
      if (q.phi) {
        std::memcpy(tmp.data(), q.phi, size_t(n) * 8);
      } else {
        for (int64_t i = 0; i < n; ++i) tmp[size_t(i)] = q.phi_fn(xs[size_t(i)], q.phi_ctx);
      }
      permute_host(n, pl.C, tmp.data(), at(pl.o_phi));
      if (q.src_kind == TSF_SRC_SEPARABLE) {
        std::memcpy(at(pl.o_scal), q.scal, size_t(M) * size_t(pl.K) * 8);
        for (int k = 0; k < pl.K; ++k) permute_host(n, pl.C, q.basis + int64_t(k) * n, at(pl.o_basis) + int64_t(k) * n);
      } else if (q.src_kind == TSF_SRC_TABLE) {
        // host table: uploaded below from the caller's buffer; device table: borrowed
      } else if (q.src_kind == TSF_SRC_CALLBACK) {
        // slow path: the host callback is evaluated once per level at
        // t_{j+sigma} here, into the instance's source table (same kernel path as a table)
        for (int64_t j = 0; j < M; ++j) {
          q.f_cb(xs.data(), n, tl[size_t(j)], tmp.data(), q.f_ctx);
          for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(tmp[size_t(i)])) {
              set_error("f callback returned a non-finite value at level " + std::to_string(j));
              return bail(TSF_E_ARG);
            }
          permute_host(n, pl.C, tmp.data(), at(pl.o_ftab) + j * n);
        }
      }
    }
    if (!tab_host) {
      CKH(cudaMemcpy2DAsync(h->ws + pl.off_inst, pl.stride, himg.data(), img, img, size_t(B),
                            cudaMemcpyHostToDevice, st));
    } else {
      CKH(cudaMemcpy2DAsync(h->ws + pl.off_inst, pl.stride, himg.data(), img, size_t(pl.o_ftab), size_t(B),
                            cudaMemcpyHostToDevice, st));
      CKH(cudaMemcpy2DAsync(h->ws + pl.off_inst + pl.o_phi, pl.stride, himg.data() + size_t(pl.o_ftab), img,
                            size_t(pl.o_omega - pl.o_phi), size_t(B), cudaMemcpyHostToDevice, st));
      const size_t tab = size_t(M) * size_t(n) * 8;
      for (int32_t b = 0; b < B; ++b) {
        char *blk = h->ws + pl.off_inst + size_t(b) * pl.stride;
        CKH(cudaMemcpyAsync(blk + pl.o_hist, p[b].f_table, tab, cudaMemcpyHostToDevice, st));
        k_permute_rows<<<grid_for(M * n), 256, 0, st>>>(reinterpret_cast<const double *>(blk + pl.o_hist),
                                                        reinterpret_cast<double *>(blk + pl.o_ftab), n, M, pl.C);
        CKH(cudaMemsetAsync(blk + pl.o_hist, 0, tab, st));
      }
      CKH(cudaGetLastError());
    }
    if (pl.ftab_dev) {
      std::vector<const double *> ptrs(static_cast<size_t>(B));
      for (int32_t b = 0; b < B; ++b) ptrs[size_t(b)] = p[b].f_table;
      CKH(cudaMemcpyAsync(h->ws + pl.off_fptr, ptrs.data(), size_t(B) * sizeof(double *), cudaMemcpyHostToDevice, st));
    }
  }
  k_reset<<<grid_for((n + 4 * M) * B), 256, 0, st>>>(h->dp);     // u = phi, stats cleared
  CKH(cudaGetLastError());
  // weights and one-time spectra (batched Stockham FFTs in the scratch region)
  k_weights<<<(B + 127) / 128, 128, 0, st>>>(dp);
  CKH(cudaGetLastError());
  const double2 *tw = reinterpret_cast<const double2 *>(h->ws + pl.off_tw);
  for (int b0 = 0; b0 < B; b0 += pl.scratch_batch) {
    const int nb = std::min(pl.scratch_batch, B - b0);
    double2 *bufA = reinterpret_cast<double2 *>(h->ws + pl.off_scratch);
    double2 *bufB = bufA + int64_t(nb) * 3 * n;
    double2 *embA = bufA, *preA = bufA + int64_t(nb) * 2 * n;
    double2 *embB = bufB, *preB = bufB + int64_t(nb) * 2 * n;
    k_cols<<<grid_for(int64_t(nb) * 2 * n), 256, 0, st>>>(dp, b0, nb, embA, preA);
    int le = 0;
    while ((int64_t(1) << le) < 2 * n) ++le;
    double2 *src = embA, *dst = embB;
    for (int ps = 0; ps < le; ++ps) {
      k_stockham<<<grid_for(int64_t(nb) * n), 256, 0, st>>>(src, dst, 2 * n, ps, nb, tw, int(2 * n));
      std::swap(src, dst);
    }
    const double2 *embS = src;
    const double2 *preS = preA;
    if (pl.precond != TSF_NOPREC) {
      double2 *ps_src = preA, *ps_dst = preB;
      for (int ps = 0; ps < le - 1; ++ps) {
        k_stockham<<<grid_for(int64_t(nb) * n / 2), 256, 0, st>>>(ps_src, ps_dst, n, ps, nb, tw, int(2 * n));
        std::swap(ps_src, ps_dst);
      }
      preS = ps_src;
    }
    k_scatter_spec<<<grid_for(int64_t(nb) * (2 * n)), 256, 0, st>>>(dp, b0, nb, embS, preS);
    CKH(cudaGetLastError());
  }
  if (pl.precond != TSF_NOPREC) {
    k_prec_guard<<<unsigned(int64_t(B) * M), 256, 0, st>>>(dp);
    CKH(cudaGetLastError());
    std::vector<int32_t> stv(size_t(B) * size_t(M));
    CKH(cudaMemcpy2DAsync(stv.data(), size_t(M) * 4, h->ws + pl.off_inst + pl.o_st, pl.stride, size_t(M) * 4,
                          size_t(B), cudaMemcpyDeviceToHost, st));
    CKH(cudaStreamSynchronize(st));
    for (size_t k = 0; k < stv.size(); ++k)
      if (stv[k] == TSF_LEVEL_SINGULAR_PREC) {
        set_error("preconditioner singular: |lambda_P| < 1e-14 max|lambda_P| (S:257) at instance " +
                  std::to_string(k / size_t(M)) + ", level " + std::to_string(k % size_t(M)));
        return bail(TSF_E_SINGULAR_PREC);
      }
  }
  CKH(cudaStreamSynchronize(st));

  // NEXT-2 setup: x = A^{-1} e_1, y = A^{-1} e_n by BiCGSTAB (eq3.4), then the spectra of the
  // four Gohberg-Semencul factors (same batched Stockham FFTs as the one-time spectra)
  if (pl.method == TSF_GSF && M >= 2) {
    CKH(launch_solve(pl, dp, 1, st, 1));
    CKH(launch_solve(pl, dp, 1, st, 2));
    for (int b0 = 0; b0 < B; b0 += pl.scratch_batch) {
      const int nb = std::min(pl.scratch_batch, B - b0);
      double2 *bufA = reinterpret_cast<double2 *>(h->ws + pl.off_scratch);
      double2 *bufB = bufA + int64_t(nb) * 3 * n;
      int le = 0;
      while ((int64_t(1) << le) < 2 * n) ++le;
      for (int k = 0; k < 4; ++k) {
        k_gsf_cols<<<grid_for(int64_t(nb) * 2 * n), 256, 0, st>>>(dp, b0, nb, k, bufA);
        double2 *src = bufA, *dst = bufB;
        for (int ps = 0; ps < le; ++ps) {
          k_stockham<<<grid_for(int64_t(nb) * n), 256, 0, st>>>(src, dst, 2 * n, ps, nb, tw, int(2 * n));
          std::swap(src, dst);
        }
        k_gsf_scatter<<<grid_for(int64_t(nb) * (n + 1)), 256, 0, st>>>(dp, b0, nb, k, src);
      }
      CKH(cudaGetLastError());
    }
    CKH(cudaStreamSynchronize(st));
    for (int32_t b = 0; b < B; ++b) {
      double par[16];
      CKH(cudaMemcpyAsync(par, inst_ptr(h, b, pl.o_par), sizeof(par), cudaMemcpyDeviceToHost, st));
      CKH(cudaStreamSynchronize(st));
      if (par[8] < 0 || par[9] < 0 || !std::isfinite(par[7])) {
        set_error("GSF setup (A x = e_1, A y = e_n) failed for instance " + std::to_string(b));
        return bail(TSF_E_BREAKDOWN);
      }
      // GSF applicability (eq. 3.5 "if xi_0 != 0"; |xi_0| < 1e-12 ||x||_inf is singular)
      std::vector<double> xv(static_cast<size_t>(n));
      CKH(cudaMemcpyAsync(xv.data(), inst_ptr(h, b, pl.o_vec + int64_t(V_GX) * n * 8), size_t(n) * 8,
                          cudaMemcpyDeviceToHost, st));
      CKH(cudaStreamSynchronize(st));
      double xinf = 0.0;
      for (double v : xv) xinf = std::max(xinf, std::fabs(v));
      const double xi0 = 1.0 / par[7];
      if (!(std::fabs(xi0) >= 1e-12 * xinf)) {
        set_error("GSF inapplicable: |xi_0| < 1e-12 ||x||_inf (S:255) for instance " + std::to_string(b));
        return bail(TSF_E_SINGULAR_PREC);
      }
    }
  }

  // CUDA graph of one level step: fused solve kernel (1 level) + level counter advance
  {
    cudaStream_t cs;
    CKH(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CKH(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    cudaError_t e1 = launch_solve(pl, dp, 1, cs);
    k_advance<<<1, 32, 0, cs>>>(dp.level, 1, M);
    cudaError_t e2 = cudaStreamEndCapture(cs, &h->step_graph);
    cudaStreamDestroy(cs);
    CKH(e1);
    CKH(e2);
    CKH(cudaGraphInstantiate(&h->step_exec, h->step_graph, 0));
  }
#undef CKH
  *out = h;
  return TSF_OK;
}

int tsf_step(tsf_handle *h) {
  if (!h) { set_error("null handle"); return TSF_E_ARG; }
  if (h->level >= h->pl.M) { set_error("all levels done"); return TSF_E_STATE; }
  CK(cudaSetDevice(h->device));
  CK(cudaGraphLaunch(h->step_exec, h->st));
  h->level += 1;
  return TSF_OK;
}

int tsf_solve(tsf_handle *h) {
  if (!h) { set_error("null handle"); return TSF_E_ARG; }
  if (h->level >= h->pl.M) { set_error("all levels done"); return TSF_E_STATE; }
  CK(cudaSetDevice(h->device));
  const int64_t nlev = h->pl.M - h->level;
  CK(launch_solve(h->pl, h->dp, int32_t(nlev), h->st));
  k_advance<<<1, 32, 0, h->st>>>(h->dp.level, nlev, h->pl.M);
  CK(cudaGetLastError());
  h->level = h->pl.M;
  return TSF_OK;
}

int tsf_reset(tsf_handle *h) {
  if (!h) { set_error("null handle"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  k_reset<<<grid_for((h->pl.n + 4 * h->pl.M) * h->pl.B), 256, 0, h->st>>>(h->dp);
  CK(cudaGetLastError());
  h->level = 0;
  return TSF_OK;
}

int64_t tsf_level(const tsf_handle *h) { return h ? h->level : -1; }

int tsf_sync(tsf_handle *h) {
  if (!h) { set_error("null handle"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  if (h->level == 0) return TSF_OK;
  const int64_t M = h->pl.M;
  std::vector<int32_t> stv(size_t(h->pl.B) * size_t(M));
  CK(cudaMemcpy2D(stv.data(), size_t(M) * 4, h->ws + h->pl.off_inst + h->pl.o_st, h->pl.stride,
                  size_t(M) * 4, size_t(h->pl.B), cudaMemcpyDeviceToHost));
  int rc = TSF_OK;
  for (int32_t b = 0; b < h->pl.B; ++b)
    for (int64_t j = 0; j < h->level; ++j) {
      const int32_t s = stv[size_t(b) * size_t(M) + size_t(j)];
      if (s == TSF_LEVEL_OK) continue;
      const int code = level_status_to_rc(s);
      if (code < 0) {
        set_error("instance " + std::to_string(b) + " level " + std::to_string(j) + ": status " + std::to_string(s));
        return code;
      }
      rc = code;
    }
  return rc;
}

// u^j of instances [b0, b0 + nb) -> out[nb][n] in natural order.  Host: one pitched D2H copy
// of the permuted vectors on the handle's stream, then the host unpermute; device: a gather
// kernel on the stream.  Synchronizes the stream.
static int get_solutions_range(tsf_handle *h, int32_t b0, int32_t nb, double *out, int32_t out_on_device) {
  CK(cudaSetDevice(h->device));
  const int64_t n = h->pl.n;
  const char *src = h->ws + h->pl.off_inst + size_t(b0) * h->pl.stride + size_t(h->pl.o_vec + int64_t(V_U) * n * 8);
  if (out_on_device) {
    k_gather_u<<<grid_for(int64_t(nb) * n), 256, 0, h->st>>>(h->dp, b0, nb, out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->st));
    return TSF_OK;
  }
  std::vector<double> pv(size_t(nb) * size_t(n));
  CK(cudaMemcpy2DAsync(pv.data(), size_t(n) * 8, src, h->pl.stride, size_t(n) * 8, size_t(nb),
                       cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  for (int32_t b = 0; b < nb; ++b) unpermute_host(n, h->pl.C, pv.data() + size_t(b) * n, out + int64_t(b) * n);
  return TSF_OK;
}

int tsf_get_solution(tsf_handle *h, int32_t inst, double *out, int32_t out_on_device) {
  if (!h || !out || inst < 0 || inst >= h->pl.B) { set_error("bad arguments"); return TSF_E_ARG; }
  return get_solutions_range(h, inst, 1, out, out_on_device);
}

int tsf_get_solutions(tsf_handle *h, double *out, int32_t out_on_device) {
  if (!h || !out) { set_error("bad arguments"); return TSF_E_ARG; }
  return get_solutions_range(h, 0, h->pl.B, out, out_on_device);
}

static int get_rows(tsf_handle *h, int64_t off, size_t esz, void *dst) {
  const size_t M = size_t(h->pl.M), B = size_t(h->pl.B);
  CK(cudaMemcpy2DAsync(dst, M * esz, h->ws + h->pl.off_inst + off, h->pl.stride, M * esz, B,
                       cudaMemcpyDeviceToHost, h->st));
  return TSF_OK;
}

int tsf_get_stats(tsf_handle *h, int32_t *iters_half, double *relres, int32_t *status) {
  if (!h) { set_error("null handle"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  int rc = TSF_OK;
  if (iters_half && (rc = get_rows(h, h->pl.o_it, 4, iters_half))) return rc;
  if (relres && (rc = get_rows(h, h->pl.o_rr, 8, relres))) return rc;
  if (status && (rc = get_rows(h, h->pl.o_st, 4, status))) return rc;
  CK(cudaStreamSynchronize(h->st));
  return TSF_OK;
}

int tsf_get_true_residuals(tsf_handle *h, double *true_relres) {
  if (!h || !true_relres) { set_error("bad arguments"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  int rc = get_rows(h, h->pl.o_trr, 8, true_relres);
  if (rc) return rc;
  CK(cudaStreamSynchronize(h->st));
  return TSF_OK;
}

int tsf_handle_info(const tsf_handle *h, tsf_plan_info *info) {
  if (!h || !info) { set_error("bad arguments"); return TSF_E_ARG; }
  info->cluster = h->pl.C;
  info->threads = kThreads;
  info->smem_bytes = h->pl.smem;
  info->embed_len = h->pl.n;
  info->precond_len = h->pl.n / 2;
  info->workspace_bytes = h->pl.total;
  info->exchange = h->pl.C == 1 ? 0 : (h->pl.staged ? 1 : (h->pl.big ? 3 : 2));
  info->chunk = h->pl.chunk;
  info->vsmem = h->pl.vsmem;
  info->resident = h->pl.resident;
  return TSF_OK;
}

int tsf_destroy(tsf_handle *h) {
  if (!h) return TSF_OK;
  cudaSetDevice(h->device);
  // the caller may free the workspace right after: let every enqueued launch finish first
  cudaStreamSynchronize(h->st);
  if (h->step_exec) cudaGraphExecDestroy(h->step_exec);
  if (h->step_graph) cudaGraphDestroy(h->step_graph);
  delete h;
  return TSF_OK;
}

// ---------------------------------------------------------------------- test hooks
int tsf_debug_fft_tables(int64_t L, int32_t *plan, int32_t *stages, int32_t *perm, int32_t *tw) {
  if (!is_pow2(L) || L > (int64_t(1) << 20)) { set_error("L must be a power of two <= 2^20"); return TSF_E_ARG; }
  int32_t pl[32];
  const int S = fft_plan_radices(L, pl);
  if (plan) for (int s = 0; s < S; ++s) plan[s] = pl[s];
  if (stages) *stages = S;
  if (perm) fft_perm(L, perm);
  if (tw) {
    int64_t o = 0;
    for (int s = 0; s < S; ++s) o += fft_stage_twiddles(L, s, tw + o);
  }
  return TSF_OK;
}

int tsf_debug_local_fft(int64_t L, const double *x, double *y, int32_t inverse) {
  if (!is_pow2(L) || L < 2 || L > kMaxLocal || !x || !y) { set_error("bad arguments"); return TSF_E_ARG; }
  double2 *buf = nullptr, *tw = nullptr;
  CK(cudaMalloc(&buf, size_t(L) * 16));
  CK(cudaMalloc(&tw, size_t(2 * L) * 16));
  CK(cudaMemcpy(buf, x, size_t(L) * 16, cudaMemcpyHostToDevice));
  k_twiddle<<<grid_for(2 * L), 256>>>(tw, int(2 * L));
  const size_t dsm = size_t(L + L / 16) * 16 + 16 * size_t(L / 64 + 64) + 1024;
  CK(cudaFuncSetAttribute(k_dbg_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dsm)));
  k_dbg_fft<<<1, kThreads, dsm>>>(buf, int(L), tw, int(2 * L), inverse);
  CK(cudaGetLastError());
  CK(cudaMemcpy(y, buf, size_t(L) * 16, cudaMemcpyDeviceToHost));
  cudaFree(buf);
  cudaFree(tw);
  return TSF_OK;
}

int tsf_debug_weights(double beta, int64_t K, double *g, double *omega) {
  if (K < 0 || K > (int64_t(1) << 21) || !g || !omega) { set_error("bad arguments"); return TSF_E_ARG; }
  double *dg = nullptr, *dw = nullptr;
  CK(cudaMalloc(&dg, size_t(K + 1) * 8));
  CK(cudaMalloc(&dw, size_t(K + 1) * 8));
  k_dbg_weights<<<1, 1>>>(beta, K, dg, dw);
  CK(cudaGetLastError());
  CK(cudaMemcpy(g, dg, size_t(K + 1) * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(omega, dw, size_t(K + 1) * 8, cudaMemcpyDeviceToHost));
  cudaFree(dg);
  cudaFree(dw);
  return TSF_OK;
}

int tsf_debug_apply(tsf_handle *h, int32_t inst, int64_t j, int32_t which, const double *x, double *y) {
  if (!h || !x || !y || inst < 0 || inst >= h->pl.B || j < 0 || j >= h->pl.M || which < 0 || which > 4) {
    set_error("bad arguments");
    return TSF_E_ARG;
  }
  if (which >= 3 && h->pl.precond == TSF_NOPREC) {
    std::memcpy(y, x, size_t(h->pl.n) * 8);
    return TSF_OK;
  }
  CK(cudaSetDevice(h->device));
  const int64_t n = h->pl.n;
  std::vector<double> pv(static_cast<size_t>(n)), po(static_cast<size_t>(n));
  permute_host(n, h->pl.C, x, pv.data());
  double *din = nullptr, *dout = nullptr;
  CK(cudaMalloc(&din, size_t(n) * 8));
  CK(cudaMalloc(&dout, size_t(n) * 8));
  { CK(cudaMemcpyAsync(din, pv.data(), size_t(n) * 8, cudaMemcpyHostToDevice, h->st)); CK(cudaStreamSynchronize(h->st)); }
  CK(launch_dbg_apply(h->pl, h->dp, inst, j, which, din, dout, h->st));
  CK(cudaStreamSynchronize(h->st));
  { CK(cudaMemcpyAsync(po.data(), dout, size_t(n) * 8, cudaMemcpyDeviceToHost, h->st)); CK(cudaStreamSynchronize(h->st)); }
  unpermute_host(n, h->pl.C, po.data(), y);
  cudaFree(din);
  cudaFree(dout);
  return TSF_OK;
}

int tsf_debug_apply_bench(tsf_handle *h, int32_t inst, int64_t j, int32_t reps, float *ms) {
  if (!h || !ms || inst < 0 || inst >= h->pl.B || j < 0 || j >= h->pl.M || reps < 2 ||
      h->pl.precond == TSF_NOPREC) {
    set_error("bad arguments");
    return TSF_E_ARG;
  }
  CK(cudaSetDevice(h->device));
  const int64_t n = h->pl.n;
  std::vector<double> x(static_cast<size_t>(n), 1.0);
  double *din = nullptr, *dout = nullptr;
  CK(cudaMalloc(&din, size_t(n) * 8));
  CK(cudaMalloc(&dout, size_t(n) * 8));
  { CK(cudaMemcpyAsync(din, x.data(), size_t(n) * 8, cudaMemcpyHostToDevice, h->st)); CK(cudaStreamSynchronize(h->st)); }
  CK(launch_dbg_apply(h->pl, h->dp, inst, j, OP_A, din, dout, h->st, reps));   // warm-up
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, h->st));
  CK(launch_dbg_apply(h->pl, h->dp, inst, j, OP_A, din, dout, h->st, reps));
  CK(cudaEventRecord(e1, h->st));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(din);
  cudaFree(dout);
  return TSF_OK;
}

int tsf_debug_spectra(tsf_handle *h, int32_t inst, int64_t j, double *lamA, double *lamP) {
  if (!h || inst < 0 || inst >= h->pl.B || j < 0 || j >= h->pl.M) { set_error("bad arguments"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  const int64_t n = h->pl.n;
  double2 *dA = nullptr, *dP = nullptr;
  CK(cudaMalloc(&dA, size_t(n + 1) * 16));
  CK(cudaMalloc(&dP, size_t(n / 2 + 1) * 16));
  CK(cudaMemset(dP, 0, size_t(n / 2 + 1) * 16));
  k_dbg_spectra<<<grid_for(2 * n), 256, 0, h->st>>>(h->dp, inst, j, dA, dP);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->st));
  if (lamA) { CK(cudaMemcpyAsync(lamA, dA, size_t(n + 1) * 16, cudaMemcpyDeviceToHost, h->st)); CK(cudaStreamSynchronize(h->st)); }
  if (lamP) { CK(cudaMemcpyAsync(lamP, dP, size_t(n / 2 + 1) * 16, cudaMemcpyDeviceToHost, h->st)); CK(cudaStreamSynchronize(h->st)); }
  cudaFree(dA);
  cudaFree(dP);
  return TSF_OK;
}

int tsf_debug_rhs(tsf_handle *h, int32_t inst, double *out) {
  if (!h || !out || inst < 0 || inst >= h->pl.B) { set_error("bad arguments"); return TSF_E_ARG; }
  if (h->level >= h->pl.M) { set_error("all levels done"); return TSF_E_STATE; }
  CK(cudaSetDevice(h->device));
  CK(launch_dbg_rhs(h->pl, h->dp, h->st));
  CK(cudaStreamSynchronize(h->st));
  const int64_t n = h->pl.n;
  std::vector<double> pv(static_cast<size_t>(n));
  { CK(cudaMemcpyAsync(pv.data(), inst_ptr(h, inst, h->pl.o_vec + int64_t(V_R) * n * 8), size_t(n) * 8, cudaMemcpyDeviceToHost, h->st)); CK(cudaStreamSynchronize(h->st)); }
  unpermute_host(n, h->pl.C, pv.data(), out);
  return TSF_OK;
}

int tsf_debug_set_history(tsf_handle *h, int32_t inst, int64_t j, const double *U) {
  if (!h || !U || inst < 0 || inst >= h->pl.B || j < 0 || j > h->pl.M) { set_error("bad arguments"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  const int64_t n = h->pl.n;
  std::vector<double> d(static_cast<size_t>(n)), pv(static_cast<size_t>(n));
  for (int64_t s = 0; s < j; ++s) {
    for (int64_t i = 0; i < n; ++i) d[size_t(i)] = U[(s + 1) * n + i] - U[s * n + i];
    permute_host(n, h->pl.C, d.data(), pv.data());
    { CK(cudaMemcpyAsync(inst_ptr(h, inst, h->pl.o_hist + s * n * 8), pv.data(), size_t(n) * 8, cudaMemcpyHostToDevice, h->st)); CK(cudaStreamSynchronize(h->st)); }
  }
  permute_host(n, h->pl.C, U + j * n, pv.data());
  { CK(cudaMemcpyAsync(inst_ptr(h, inst, h->pl.o_vec + int64_t(V_U) * n * 8), pv.data(), size_t(n) * 8, cudaMemcpyHostToDevice, h->st)); CK(cudaStreamSynchronize(h->st)); }
  k_set_level<<<1, 32, 0, h->st>>>(h->dp.level, j);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->st));
  h->level = j;
  return TSF_OK;
}

}  // extern "C"

extern "C" int tsf_debug_helper_state(tsf_handle *h, int64_t *out) {
  if (!h || !out) { set_error("bad arguments"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(out, h->dp.sync, 8 * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return TSF_OK;
}

extern "C" int tsf_debug_prof(tsf_handle *h, uint64_t *out, int32_t reset) {
  if (!h || !out) { set_error("bad arguments"); return TSF_E_ARG; }
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaMemcpy(out, h->dp.prof, 32 * 8, cudaMemcpyDeviceToHost));
  if (reset) CK(cudaMemset(h->dp.prof, 0, 32 * 8));
  return TSF_OK;
}
