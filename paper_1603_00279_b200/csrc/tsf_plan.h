// tsf_plan.h -- host planner of the per-level solver (no CUDA types; compiled by g++/nvcc).
//
// The planner validates problems, computes the O(M) scalar tables of the scheme
// (Lemma 1 weights, eta_j, kappa), picks the thread-block-cluster
// size, builds the integer FFT/task tables and lays out the caller's device workspace.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tsf.h"

namespace tsf {

constexpr int kThreads = 256;          // threads per CTA
constexpr int kMaxLocal = 8192;        // max complex elements of an SMEM-resident local FFT (128 KiB)
constexpr int64_t kMaxN = 1 << 20;     // largest n (multi-pass regime above n = 2^17)
constexpr int kNumVec = 13;            // u, Krylov work vectors, phi copy, GSF generators x, y
constexpr int kSmemVec = 9;            // vectors kept in SMEM when they fit (u, x, r, r^, p, v, s, p^, s^);
                                       // g (read once per level) always lives in HBM
constexpr int64_t kMaxSmem = 232448;   // opt-in dynamic shared memory per CTA (227 KiB)
constexpr size_t kAlign = 256;
#ifdef TSF_PAD
constexpr int kPadBuf = 1;             // padded transform buffers (one pad per 16 elements)
#else
constexpr int kPadBuf = 0;             // XOR-swizzled transform buffers need no padding
#endif

// Vector slots inside the per-instance vector block (each n doubles).
enum Vec { V_U = 0, V_X, V_R, V_RH, V_P, V_V, V_S, V_T, V_PH, V_SH, V_G, V_GX, V_GY };

// Plain-old-data parameters handed to every kernel by value.
struct DevParams {
  int64_t n, M;
  int32_t B, C, K, src_kind, method, precond, maxit;
  int32_t L1e, L1p, npe, npp;      // local FFT lengths and column-pair tasks per CTA
  int32_t staged, resident;        // exchange / SMEM-table modes (see Plan)
  int32_t vsmem;                   // Krylov vectors in SMEM (else in the instance's HBM block)
  int32_t fuse_min;                // local FFT length from which radix-16 passes are used
  int32_t chunk;                   // column pairs per chunk of the unstaged column stage
  int32_t big;                     // multi-pass regime: local transforms longer than kMaxLocal
  int32_t lre, lrp;                // log2 of the row count R = L1 / S of the embedding / preconditioner
                                   // local transform (S = min(L1, kMaxLocal); 0 unless big)
  double tol;
  double scale_e, scale_p;         // 1/(4L) folding of the real-FFT split and 1/L
  double qscale_p;                 // Lambda_Q scale of the preconditioner: 1 or (n-1)/n
  int32_t strang;                  // Strang midpoint correction active
  int32_t twN;                     // twiddle table length (2n)
  // shared tables
  const void *tw;                  // double2[2n]: e^{-2 pi i e/(2n)}
  const int32_t *slot_e, *slot_p;  // k1 -> slot of the local DIF output
  const double *sq_e, *sq_p;       // sin tables in task order
  int64_t *level;                  // device level counter
  int64_t *sync;                   // history helpers: [0] solver CTA-levels done, [1..2] ready[J&1], [3] counters
  double *pre;                     // history pre-sums P^J, two n-vectors (J & 1), single-instance plans
  int32_t helpers;                 // history-helper CTAs of this launch (0: the solver sums the history)
  unsigned long long *prof;        // 32 cycle counters (profiling build only)
  // per-instance block
  char *inst;                      // base of instance 0
  int64_t stride;                  // bytes between instances
  int64_t o_par, o_omega, o_lwe, o_lwp, o_lev, o_hwc, o_hwe, o_scal, o_basis, o_ftab;
  int64_t o_vec, o_hist, o_it, o_rr, o_trr, o_st, o_mul, o_gsf, o_xg, o_phi;
  int64_t o_xa;                    // multi-pass regime: the apply buffer [C][L1e] (global)
  const double *const *fptr;       // borrowed device f tables (natural order), one per instance
  int32_t ftab_dev;                // 1: the source table is read through fptr
  int32_t x0_warm;                 // NEXT-3: Krylov initial guess u^j (else 0)
  int32_t true_res;                // compute ||g - A u^{j+1}|| / ||g|| at every level exit
  int32_t pipelined;               // NEXT-3: BiCGSTAB with two cluster reductions per iteration
  int32_t hblock;                  // NEXT-3: blocked history sum, block length (0 = direct)
  int32_t fuse;                    // fused BiCGSTAB vector updates on the first/last FFT stages (C3 shape)
  int64_t o_hb;                    // blocked history: partial sums of the block's levels [hblock][n]
};

struct Plan {
  int64_t n = 0, M = 0;
  int32_t B = 0, C = 1, K = 0, src_kind = 0;
  int32_t method = 0, precond = 0, maxit = 0;
  double tol = 0;
  int32_t L1e = 0, L1p = 0, npe = 0, npp = 0;
  int32_t vsmem = 0;    // Krylov vectors of a CTA's chunk resident in SMEM (else HBM)
  int32_t staged = 0;   // cross-CTA step staged through SMEM buffers B (staging) and O (output)
  int32_t resident = 0; // per-instance constant tables cached in SMEM (small local length)
  int32_t fuse_min = 1024;   // radix-16 passes from L1 = 1024 (measured, tools/fft_ubench.cu)
  int32_t chunk = 0;         // unstaged clusters: column pairs per chunk (chunk buffer 2 chunk C complex)
  int32_t big = 0;           // multi-pass regime (n / C > kMaxLocal; C = 16): see DESIGN.md
  int32_t lre = 0, lrp = 0;  // log2 rows of the embedding / preconditioner local transforms
  int64_t smem = 0;
  // workspace layout (byte offsets from the workspace base)
  size_t off_tw = 0, off_slot_e = 0, off_slot_p = 0, off_sq_e = 0, off_sq_p = 0;
  size_t off_level = 0, off_prof = 0, off_scratch = 0, scratch_bytes = 0, off_inst = 0;
  size_t off_sync = 0, off_pre = 0, off_fptr = 0;
  int32_t x0_warm = 0, true_res = 0, pipelined = 0, hblock = 0;
  int32_t fuse = 1;          // developer knob TSF_NO_FUSE=1 disables (bitwise A/B test)
  int64_t o_hb = 0;
  int32_t scratch_batch = 0;
  size_t stride = 0, total = 0;
  int64_t o_par, o_omega, o_lwe, o_lwp, o_lev, o_hwc, o_hwe, o_scal, o_basis, o_ftab;
  int64_t o_vec, o_hist, o_it, o_rr, o_trr, o_st, o_mul, o_gsf, o_xg, o_phi;
  int64_t o_xa = 0;
  int32_t ftab_dev = 0;      // source table borrowed from device memory (not copied)
};

// Per-instance host tables (all doubles).
struct InstTables {
  double sigma = 0, kappa = 0, h = 0, tau = 0;
  std::vector<double> lev;   // [M][4]: eta_j, gamma_j/(2h), d+_j/h^beta, d-_j/h^beta
  std::vector<double> hwc;   // [M]: kappa * chat_m, chat_m = a_m + b_{m+1} - b_m (m >= 1)
  std::vector<double> hwe;   // [M]: kappa * e_j,    e_j = a_j - b_j             (j >= 1)
};

// Error reporting shared with the C-ABI (thread-local message).
void set_error(const std::string &msg);
const char *last_error();

bool is_pow2(int64_t v);
int validate(const tsf_problem *p, int32_t B, const tsf_solver *s);
int make_plan(const tsf_problem *p, int32_t B, const tsf_solver *s, Plan *plan);
int sample_points(const tsf_problem &p, double *x, double *t);
int inst_tables(const tsf_problem &p, InstTables *out);

// FFT integer tables (DESIGN.md R-fft).
int fft_plan_radices(int64_t L, int32_t *plan);
void fft_perm(int64_t L, int32_t *perm);
int64_t fft_stage_twiddles(int64_t L, int s, int32_t *tw);

#ifdef __CUDACC__
#define TSF_HD __host__ __device__
#else
#define TSF_HD
#endif

// Column-pair task geometry: CTA r owns the column pairs
// pi = r + i C (i < L1/(2C)) of the L1 x C four-step grid, pair (k1a, k1b) = (pi, L1 - pi),
// or (0, L1/2) for pi = 0.  Bin of (task i, row k2, column ab) is k1 + L1 k2.
TSF_HD inline int64_t task_bin(int64_t L1, int C, int r, int i, int k2, int ab) {
  const int64_t pi = int64_t(r) + int64_t(i) * C;
  const int64_t k1a = pi == 0 ? 0 : pi;
  const int64_t k1b = pi == 0 ? L1 / 2 : L1 - pi;
  return (ab ? k1b : k1a) + L1 * int64_t(k2);
}
// Task-order storage index of (r, k2, ab, i) for np tasks per CTA.
TSF_HD inline int64_t task_index(int C, int np, int r, int k2, int ab, int i) {
  return ((int64_t(r) * C + k2) * 2 + ab) * np + i;
}
// Permuted chunk layout: element e (natural order) of an n-vector lives at
// r (n/C) + 2 m1 + (e & 1) with m = e/2 = C m1 + r, so CTA r owns a contiguous chunk of
// packed complex values z_m = (x_{2m}, x_{2m+1}) with m = r mod C.
TSF_HD inline int64_t perm_pos(int64_t n, int C, int64_t e) {
  const int64_t m = e >> 1, r = m % C, m1 = m / C;
  return r * (n / C) + 2 * m1 + (e & 1);
}

DevParams dev_params(const Plan &pl, char *ws);

// Shared-memory carve-up of the solve kernel (must match smem_view in tsf_kernels.cuh):
// A [L1e], B [L1e] and O [L1e] if staged, twiddles (direct [L1e] if resident, else two-level
// [L1e/64 + 64]), resident tables: column twiddles [L1e + L1p], per-level multipliers
// [L1e + L1p], pair twiddles [L1e + L1p] (double2), Krylov vectors [kSmemVec x L1p] (double2) if
// vsmem; 48 doubles of reduction scratch, 128 doubles of pushed CTA partials and 4 mbarriers.
// Per-stage twiddle table of the compile-time local FFTs (resident, L1e = 1024 or 256): stage
// tables of W_m^k (k < m/4) for m = 4 .. L1e, then W_{L1e/2}^b (b < L1e/4).
TSF_HD inline int tws_len(int64_t L1e) { return (L1e == 1024 || L1e == 256) ? int((L1e - 1) / 3 + L1e / 4) : 0; }
TSF_HD inline int64_t smem_bytes(int64_t L1e, int64_t L1p, int staged, int resident, int vsmem,
                                 int64_t chunk_cplx = 0) {
  // A holds one row of at most kMaxLocal points (multi-pass regime: L1e > kMaxLocal)
  const int64_t la = L1e > kMaxLocal ? kMaxLocal : L1e;
  int64_t c2 = (staged ? 3 * la : la) + (staged ? 2 : 1) * kPadBuf * (la / 16);   // A (+ B, O)
  if (resident) c2 += L1e + 3 * (L1e + L1p);      // twiddles, column twiddles, multipliers, pair twiddles
  if (resident) c2 += tws_len(L1e);                // per-stage twiddles of the compile-time FFTs
  else c2 += (L1e >= 64 ? L1e / 64 : 1) + (L1e >= 64 ? 64 : L1e);
  if (vsmem) c2 += kSmemVec * L1p;
  if (!staged) c2 += chunk_cplx;                   // chunk buffer of the unstaged column stage
  int64_t d = 48 + 128 + 4 + 2 + 32;               // reductions, push buffers, mbarriers, flag, W_C table
  return 16 * c2 + 8 * d + 64;
}

}  // namespace tsf
