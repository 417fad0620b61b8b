// tsf_kernels.cuh -- sm_100a FP64 device code of the per-level Toeplitz Krylov solver.
//
// One thread-block cluster of C CTAs owns one problem instance for a whole run of levels.
// Per level (alg1):
//   RHS   g = B u^j - kappa sum_s c_{j-s} d^s + f^{j+sigma}          (eq3.1)
//   Krylov solve A u^{j+1} = g, right-preconditioned BiCGSTAB or CGNR (CGLS on A P^{-1})
//   finalize d^j = u^{j+1} - u^j (history), u^j <- u^{j+1}, per-level stats.
// A, B are applied through the 2n circulant embedding of their Toeplitz generators (P:765-767,
// P:775-776) and the preconditioner is a circulant solve; each is
// FFT -> per-bin spectral op -> inverse FFT, fused in shared memory:
//   * the n real unknowns are packed as n/2 complex values z_m = x_{2m} + i x_{2m+1}
//     (real-FFT packing); CTA r of the cluster owns z_m for m = r mod C;
//   * a length-L complex transform (L = n: embedding, L = n/2: preconditioner) is a
//     four-step split L = C x L1: an in-place radix-4/2 FFT of length L1 per CTA in SMEM
//     (DIF forward into digit-reversed slots, DIT inverse back), a length-C DFT across the
//     cluster through distributed shared memory, and the per-bin real split + spectral
//     scaling on bin pairs (k, L-k) that the column-pair ownership keeps inside one CTA;
//   * per-level spectra are formed on the fly from one-time base spectra:
//     lambda = eta + mu (c Lambda_Q + p Lambda_W + q conj Lambda_W).
// Krylov vectors live in registers when a CTA's chunk is small (VPT complex values per
// thread and vector), else in global memory.  Reductions are deterministic (fixed-order warp
// shuffles, CTA, cluster).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "tsf_plan.h"

namespace cg = cooperative_groups;

#ifndef TSF_C1_BLOCKS
#define TSF_C1_BLOCKS 2   // resident CTAs per SM of single-CTA instances
#endif
#ifndef TSF_BATCH
#define TSF_BATCH 1       // elements per thread per batch of the HBM vector loops
#endif
namespace tsf {

// ------------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 mul_i(double2 a) { return make_double2(-a.y, a.x); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 caxpy(double s, double2 x, double2 y) {  // y + s x
  return make_double2(fma(s, x.x, y.x), fma(s, x.y, y.y));
}
__device__ __forceinline__ double cdot(double2 a, double2 b) { return a.x * b.x + a.y * b.y; }
__device__ __forceinline__ double2 zero2() { return make_double2(0.0, 0.0); }

// ------------------------------------------------------------------------ instance view
struct Inst {
  double *par;           // [0] sigma [1] beta [2] omega_{n/2+1}
  double *omega;
  double2 *lwe, *lwp;    // base spectra, task order (+ Nyquist at the end)
  const double *lev, *hwc, *hwe, *scal, *basis, *ftab;
  double *vec, *hist;
  double2 *mul;          // per-level multiplier tables [n + n/2] (task order), HBM variant
  double2 *gsf;          // NEXT-2: spectra of the 4 triangular GSF factors [4][n+1] (task order)
  double2 *xg;           // unstaged clusters: L2 exchange buffer [C][L1e] of the local FFT outputs
  double2 *xa;           // multi-pass regime: apply input/output buffer [C][L1e] (natural local order)
  double *hb;            // blocked history: partial sums of the current block's levels [hblock][n]
  const double *phi;     // u^0 (permuted chunks)
  const double *fdev;    // borrowed device source table (natural order) or nullptr
  int32_t *it, *st;
  double *rr, *trr;
};

__device__ __forceinline__ Inst inst_view(const DevParams &P, int b) {
  char *base = P.inst + int64_t(b) * P.stride;
  Inst I;
  I.par = reinterpret_cast<double *>(base + P.o_par);
  I.omega = reinterpret_cast<double *>(base + P.o_omega);
  I.lwe = reinterpret_cast<double2 *>(base + P.o_lwe);
  I.lwp = reinterpret_cast<double2 *>(base + P.o_lwp);
  I.lev = reinterpret_cast<const double *>(base + P.o_lev);
  I.hwc = reinterpret_cast<const double *>(base + P.o_hwc);
  I.hwe = reinterpret_cast<const double *>(base + P.o_hwe);
  I.scal = reinterpret_cast<const double *>(base + P.o_scal);
  I.basis = reinterpret_cast<const double *>(base + P.o_basis);
  I.ftab = reinterpret_cast<const double *>(base + P.o_ftab);
  I.vec = reinterpret_cast<double *>(base + P.o_vec);
  I.hist = reinterpret_cast<double *>(base + P.o_hist);
  I.mul = reinterpret_cast<double2 *>(base + P.o_mul);
  I.gsf = reinterpret_cast<double2 *>(base + P.o_gsf);
  I.xg = reinterpret_cast<double2 *>(base + P.o_xg);
  I.xa = reinterpret_cast<double2 *>(base + P.o_xa);
  I.hb = reinterpret_cast<double *>(base + P.o_hb);
  I.it = reinterpret_cast<int32_t *>(base + P.o_it);
  I.rr = reinterpret_cast<double *>(base + P.o_rr);
  I.trr = reinterpret_cast<double *>(base + P.o_trr);
  I.st = reinterpret_cast<int32_t *>(base + P.o_st);
  I.phi = reinterpret_cast<const double *>(base + P.o_phi);
  I.fdev = P.ftab_dev ? P.fptr[b] : nullptr;
  return I;
}

// ------------------------------------------------------------------------ sync helpers
template <int C>
__device__ __forceinline__ void csync() {
  if constexpr (C == 1) __syncthreads();
  else cg::this_cluster().sync();
}
template <int C>
__device__ __forceinline__ uint32_t crank() {
  if constexpr (C == 1) return 0;
  else return cg::this_cluster().block_rank();
}
template <int C, class T>
__device__ __forceinline__ T *remote(T *p, uint32_t q) {
  if constexpr (C == 1) return p;
  else return cg::this_cluster().map_shared_rank(p, q);
}

// ------------------------------------------------------------------------ async DSMEM push
// Cross-CTA data moves are pushes: the producer writes straight into the consumer's shared
// memory with st.async, which signals the consumer's mbarrier with the byte count; the consumer
// waits on its own mbarrier only.  No cluster-wide barrier, no GPU-scope fence (measured on
// B200: cluster.sync ~390 cycles + MEMBAR.ALL.GPU; a 16 KB all-to-all push ~1.4k cycles vs ~2.6k
// for pull-after-cluster.sync).  Buffers are reused only after a causal chain of exchanges
// (DESIGN.md "Exchange protocol"), so no extra barrier protects them.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *m, uint32_t bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p; TSF_W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra TSF_W; }" ::"r"(
          smem_u32(m)),
      "r"(parity)
      : "memory");
}
// 16-byte push of v to the shared::cluster address dst, completing 16 bytes on mbarrier mb
__device__ __forceinline__ void push2(uint32_t dst, double2 v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "d"(v.x), "d"(v.y), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void push1(uint32_t dst, double v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(dst), "d"(v),
               "r"(mb)
               : "memory");
}
__device__ __forceinline__ int64_t ld_acquire(const int64_t *p) {
  int64_t v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int64_t *p, int64_t v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// 16-byte asynchronous global -> shared copy through L2 (LDGSTS): no register staging, so a
// thread can keep many loads in flight without raising register pressure
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// History-helper handshake bounds: the solver waits at most
// kHelperWaitNs for a pre-sum, helpers at most kHelperIdleNs for solver progress; on a timeout
// the shared flag sync[5] is raised, helpers exit and the solver sums the history itself (same
// summation order, same bits), so a launch that is only partly resident cannot deadlock.
constexpr uint64_t kHelperWaitNs = 2000000;     // 2 ms
constexpr uint64_t kHelperIdleNs = 200000000;   // 200 ms

// Exchange state of one CTA: counts of operator exchanges and reductions so far (identical in
// every thread of the cluster, since control flow is uniform); they select mbarrier phases.
struct Xch {
  uint32_t nap = 0, ncs = 0;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------------ shared memory
// Carve-up (smem_bytes in tsf_plan.h): A (apply input), B (staging) and O (apply output) when
// staged; local-FFT twiddles (direct W_{L1e}^e table if resident, else two-level); resident
// per-CTA constant tables: column twiddles W_L^{q k1}, base spectra and pair twiddles
// W_{2L}^{bin} in task order, sine tables; reduction scratch.
struct Smem {
  double2 *A, *B, *O;
  double2 *twd, *thi, *tlo;          // twd != nullptr: direct table
  double2 *tws;                      // per-stage twiddles of the compile-time FFTs (L1e = 1024 / 256), tws_len
  double2 *ctwe, *ctwp;              // column twiddles (resident)
  double2 *mule, *mulp, *pwe, *pwp;  // per-level multipliers lambda_A, 1/lambda_P / pair twiddles (resident)
  double2 *vs;                       // Krylov vectors of this CTA's chunk (kSmemVec x L1p), or null
  double *wred, *cred;
  double *red;                       // push reductions: [2][16][4] CTA partials (double-buffered)
  uint64_t *mbar;                    // mbarriers: [0] exchange-in B, [1] exchange-back O, [2..3] red
  double2 *twc;                      // W_C^e, e < C (column-DFT twiddles of the staged column stage)
  int *flag;                         // CTA-wide broadcast word.  NOTE: the solve kernels declare NO
                                     // static __shared__ variable: one would shift the dynamic buffers
                                     // off their 128-byte alignment and break the bank-conflict-free
                                     // swizzle (measured -9% at C3 for a single 4-byte static int)
  int fuse_min;                      // local FFTs of at least this length use radix-16 passes
  int chunk;                         // column pairs per chunk of the unstaged column stage (B = chunk buffer)
  unsigned long long *prof;
};

// Section timers (profiling build, -DTSF_PROFILE): thread 0 of block 0 accumulates clock64
// cycles per section into P.prof[slot]; the wait at a barrier is charged to the section
// that ends with it.
#ifndef TSF_PROF_CTA
#define TSF_PROF_CTA 0   // the CTA whose section times are recorded (profiling build)
#endif
#ifdef TSF_PROFILE
#define TSF_PT0() long long tsf_pt_ = clock64()
#define TSF_PTR() tsf_pt_ = clock64()
#define TSF_PACC(sm, slot)                                                                    \
  do {                                                                                      \
    const long long t_ = clock64();                                                         \
    if (threadIdx.x == 0 && blockIdx.x == TSF_PROF_CTA) (sm).prof[slot] += (unsigned long long)(t_ - tsf_pt_); \
    tsf_pt_ = t_;                                                                           \
  } while (0)
#else
#define TSF_PT0() do {} while (0)
#define TSF_PTR() do {} while (0)
#define TSF_PACC(sm, slot) do {} while (0)
#endif
enum ProfSlot { PS_FFT_F = 0, PS_BAR1, PS_GATHER, PS_COLF, PS_PAIRS, PS_COLI, PS_BAR2, PS_SCATTER,
                PS_BAR3, PS_FFT_I, PS_CSUM, PS_VEC, PS_RHS_HIST, PS_LEVEL, PS_APPLIES, PS_ITERS };
__device__ __forceinline__ int tw_hi_len(int L1e) { return L1e >= 64 ? L1e / 64 : 1; }
__device__ __forceinline__ int tw_lo_len(int L1e) { return L1e >= 64 ? 64 : L1e; }

__device__ __forceinline__ Smem smem_view(unsigned char *raw, int L1e, int L1p, bool staged,
                                          bool resident, bool vsmem, unsigned long long *prof,
                                          int fuse_min = 16 * kThreads, int chunk = 0, int C = 1) {
  Smem s = {};
  s.prof = prof;
  s.fuse_min = fuse_min;
  s.chunk = chunk;
  double2 *c = reinterpret_cast<double2 *>(raw);
  const int la = L1e > kMaxLocal ? kMaxLocal : L1e;   // one row in the multi-pass regime
  s.A = c; c += la + kPadBuf * (la / 16);
  if (staged) { s.B = c; c += L1e; s.O = c; c += L1e + kPadBuf * (L1e / 16); }
  else if (chunk > 0) { s.B = c; c += 5 * chunk * C; }   // chunk buffer [2 chunk C] + 3 prefetched tables
  if (resident) {
    s.twd = c; c += L1e;
    s.ctwe = c; c += L1e; s.ctwp = c; c += L1p;
    s.mule = c; c += L1e; s.mulp = c; c += L1p;
    s.pwe = c; c += L1e; s.pwp = c; c += L1p;
  } else {
    s.thi = c; c += tw_hi_len(L1e);
    s.tlo = c; c += tw_lo_len(L1e);
  }
  if (resident && (L1e == 1024 || L1e == 256)) { s.tws = c; c += tws_len(L1e); }
  if (vsmem) { s.vs = c; c += kSmemVec * L1p; }
  double *d = reinterpret_cast<double *>(c);
  s.wred = d;
  s.cred = d + 40;
  s.red = d + 48;
  s.mbar = reinterpret_cast<uint64_t *>(d + 48 + 128);
  s.flag = reinterpret_cast<int *>(d + 48 + 128 + 4);
  s.twc = reinterpret_cast<double2 *>(d + 48 + 128 + 4 + 2);
  return s;
}

__device__ __forceinline__ double2 twid(const Smem &sm, int e) {
  if (sm.twd) return sm.twd[e];
  return cmul(sm.thi[e >> 6], sm.tlo[e & 63]);
}

__device__ __forceinline__ int col_k1(int L1, int C, uint32_t r, int col);
__device__ __forceinline__ int dperm(int p, int l);

#ifndef TSF_COL_T16
#define TSF_COL_T16 4      // lanes per column at C = 16 (4: 4 points per lane; 1: whole column)
#endif
// Resident column twiddle W_L^{q k1} of column (i, ab), row q, in the order the lane groups of
// the staged column stage read them (T = 4: the 8 lanes of a 16-byte phase are one group, rows
// s + 4m of both columns; T = 1: four groups, one row).
template <int C>
__device__ __forceinline__ int ctw_idx(int q, int i, int ab, int np) {
  if constexpr (C >= 16 && TSF_COL_T16 == 4) return (i * C + q) * 2 + ab;
  else if constexpr (C >= 16) return (q * np + i) * 2 + ab;
  else return q * (2 * np) + 2 * i + ab;          // C < 16: [q][column 2i+ab] (cross_push)
}

// Kernel prologue: local-FFT twiddles and (resident mode) this CTA's constant tables, copied
// from the accurate global tables (twiddles tw[x] = exp(-2 pi i x / twN)).
__device__ __forceinline__ void load_constants(const DevParams &P, const double2 *lwe, const double2 *lwp,
                                               const Smem &sm, uint32_t r) {
  const double2 *tw = reinterpret_cast<const double2 *>(P.tw);
  const int L1e = P.L1e, L1p = P.L1p, C = P.C;
  const int f = P.twN / L1e;
  if (sm.twd) {
    for (int i = threadIdx.x; i < L1e; i += kThreads) sm.twd[i] = tw[i * f];
  } else {
    for (int i = threadIdx.x; i < tw_lo_len(L1e); i += kThreads) sm.tlo[i] = tw[i * f];
    for (int i = threadIdx.x; i < tw_hi_len(L1e); i += kThreads) sm.thi[i] = tw[(i << 6) * f];
  }
  if (C > 1)
    for (int e = threadIdx.x; e < C; e += kThreads) sm.twc[e] = tw[e * (P.twN / C)];
  if (sm.tws) {
    // per-stage tables (conflict-free: a stage's lanes read consecutive entries): stage m = 2^LM
    // holds W_m^k, k < m / 4, at (L1e - m) / 3; then W_{L1e/2}^b, b < L1e / 4 (the radix-2 stage)
    const int nst = (L1e - 1) / 3;
    for (int u = threadIdx.x; u < tws_len(L1e); u += kThreads) {
      if (u >= nst) { sm.tws[u] = tw[(u - nst) * (P.twN / (L1e / 2))]; continue; }
      int lm = __ffs(L1e) - 1;
      while (u >= (L1e - (1 << (lm - 2))) / 3) lm -= 2;
      sm.tws[u] = tw[(u - (L1e - (1 << lm)) / 3) * (P.twN >> lm)];
    }
  }
  if (sm.ctwe) {
    // resident tables in the layouts of the staged column stage (cross_push): column twiddles
    // W_L^{q k1} at ctw_idx(q, i, ab), pair twiddles W_{2L}^{bin} of the a-side bins
    // (k2a, column (i, 0)) at i C + k2a
    const int64_t n = P.n;
    const int twL_e = P.twN / int(n), twL_p = P.twN / int(n / 2);
    const int lC = __ffs(C) - 1;
    for (int u = threadIdx.x; u < L1e; u += kThreads) {      // u = (q, i, ab) row-major
      const int ab = u & 1, i = (u >> 1) % P.npe, q = (u >> 1) / P.npe;
      const int idx = C == 16 ? ctw_idx<16>(q, i, ab, P.npe) : ctw_idx<8>(q, i, ab, P.npe);
      sm.ctwe[idx] = tw[q * col_k1(L1e, C, r, 2 * i + ab) * twL_e];
    }
    for (int u = threadIdx.x; u < L1p; u += kThreads) {
      const int ab = u & 1, i = (u >> 1) % P.npp, q = (u >> 1) / P.npp;
      const int idx = C == 16 ? ctw_idx<16>(q, i, ab, P.npp) : ctw_idx<8>(q, i, ab, P.npp);
      sm.ctwp[idx] = tw[q * col_k1(L1p, C, r, 2 * i + ab) * twL_p];
    }
    if (C == 16) {
      for (int u = threadIdx.x; u < L1e / 2; u += kThreads)
        sm.pwe[u] = tw[task_bin(L1e, C, int(r), u >> lC, u & (C - 1), 0) * (P.twN / int(2 * n))];
      for (int u = threadIdx.x; u < L1p / 2; u += kThreads)
        sm.pwp[u] = tw[task_bin(L1p, C, int(r), u >> lC, u & (C - 1), 0) * (P.twN / int(n))];
    } else {                       // task order ((k2 2 + ab) np + i), SpecOp::wtw
      for (int u = threadIdx.x; u < L1e; u += kThreads) {
        const int np = P.npe, i = u % np, ab = (u / np) & 1, k2 = u / (2 * np);
        sm.pwe[u] = tw[task_bin(L1e, C, int(r), i, k2, ab) * (P.twN / int(2 * n))];
      }
      for (int u = threadIdx.x; u < L1p; u += kThreads) {
        const int np = P.npp, i = u % np, ab = (u / np) & 1, k2 = u / (2 * np);
        sm.pwp[u] = tw[task_bin(L1p, C, int(r), i, k2, ab) * (P.twN / int(n))];
      }
    }
  }
}

// Deterministic cluster-wide sum of NV <= 4 scalars: warp butterflies (exactly commutative,
// so every lane holds the same bits) -> 8 warps in order -> CTA partial; for C > 1 warp 0 pushes
// the partial to every CTA of the cluster (slot red[par][r]) and every CTA adds the C partials
// in rank order after its mbarrier completes -> identical bits in every CTA.
template <int C, int NV>
__device__ __forceinline__ void csum(double (&v)[NV], const Smem &sm, Xch &xs) {
  TSF_PT0();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  const int par = int(xs.ncs & 1);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sm.wred[warp * 4 + k] = v[k];
  }
  __syncthreads();
  if constexpr (C == 1) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) s += sm.wred[w * 4 + k];
        sm.cred[par * 4 + k] = s;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = sm.cred[par * 4 + k];
  } else {
    double *red = sm.red + par * 64;
    uint64_t *mb = sm.mbar + 2 + par;
    if (warp == 0) {
      if (lane == 0) mbar_expect(mb, uint32_t(C * NV * 8));
      if (lane < C) {
        double s[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          s[k] = 0.0;
#pragma unroll
          for (int w = 0; w < kThreads / 32; ++w) s[k] += sm.wred[w * 4 + k];
        }
        const uint32_t r = crank<C>();
        const uint32_t dst = mapa_u32(smem_u32(red + r * 4), uint32_t(lane));
        const uint32_t mbr = mapa_u32(smem_u32(mb), uint32_t(lane));
        if constexpr (NV == 1) push1(dst, s[0], mbr);
        else {
#pragma unroll
          for (int k = 0; k + 1 < NV; k += 2) push2(dst + 8 * k, make_double2(s[k], s[k + 1]), mbr);
          if constexpr (NV & 1) push1(dst + 8 * (NV - 1), s[NV - 1], mbr);
        }
      }
    }
    mbar_wait(mb, (xs.ncs >> 1) & 1);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < C; ++q) s += red[q * 4 + k];
      v[k] = s;
    }
  }
  xs.ncs += 1;
  TSF_PACC(sm, PS_CSUM);
}

// mbarrier setup of a cluster kernel (before any push): init, make it visible cluster-wide.
template <int C>
__device__ __forceinline__ void xinit(const Smem &sm) {
  if constexpr (C > 1) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < 4; ++i) mbar_init(sm.mbar + i, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    csync<C>();
  }
}

// Digit-reversal maps of the local FFT plan (DESIGN.md R-fft) in closed form, l = log2(L1):
// slot p of the forward (DIF) output holds bin dperm(p); bin k sits in slot dslot(k).
__device__ __forceinline__ uint32_t rev4(uint32_t x, int m) {   // reverse m base-4 digits
  if (m == 0) return 0;
  uint32_t y = __brev(x) >> (32 - 2 * m);
  return ((y & 0x55555555u) << 1) | ((y >> 1) & 0x55555555u);
}
__device__ __forceinline__ int dperm(int p, int l) {
  const int s4 = l >> 1;
  if (!(l & 1)) return int(rev4(uint32_t(p), s4));
  return int(2 * rev4(uint32_t(p) & ((1u << (2 * s4)) - 1), s4) + (uint32_t(p) >> (2 * s4)));
}
__device__ __forceinline__ int dslot(int k, int l) {
  const int s4 = l >> 1;
  if (!(l & 1)) return int(rev4(uint32_t(k), s4));
  return int(rev4(uint32_t(k) >> 1, s4) + ((uint32_t(k) & 1u) << (2 * s4)));
}

// ------------------------------------------------------------------------ local FFT (SMEM)
// Plan (DESIGN.md R-fft): DIT stages s = 0..S-1 with radix 4 (s < floor(l/2)) and a final
// radix 2 when l = log2(L1) is odd; m_s = prod_{t<=s} r_t.  The forward transform runs the
// transposed stages (DIF, S-1..0) in place: natural input -> slot order, slot p holding
// X[perm[p]] with perm the gather digit reversal.  The inverse runs the conjugated DIT stages
// 0..S-1 in place: slot order -> natural order (unnormalized).
template <bool INV>
__device__ __forceinline__ void bfly4(double2 &a0, double2 &a1, double2 &a2, double2 &a3) {
  const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3);
  double2 t3 = csub(a1, a3);
  t3 = INV ? mul_i(t3) : mul_mi(t3);
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

// Swizzled SMEM index of element p of a transform buffer (A, O): bits 0..2 of p XOR
// (p>>2 ^ p>>5 ^ p>>9).  High bits are kept, so it permutes every aligned block of 8 and is a
// bijection on every power-of-two range.  For 16-byte elements (8 lanes per wavefront) it
// makes every radix-4 / radix-2 stage, every fused radix-16 pass and the linear loops free of
// shared-memory bank conflicts, and keeps the digit-reversed pair reads <= ~2.3-way
// (tools/smem_conflicts.py, L1 = 2^8..2^13).
#ifdef TSF_PAD
__device__ __forceinline__ int pidx(int p) { return p + (p >> 4); }
#else
__device__ __forceinline__ int pidx(int p) { return p ^ (((p >> 2) ^ (p >> 5) ^ (p >> 9)) & 7); }
#endif

// one stage: m = 2^lm, twiddle W_m^{kq} = W_{L1e}^{kq (L1e/m)}
// Twiddles W^e, W^{2e}, W^{3e} of a radix-4 butterfly from ONE table read: the local FFTs are
// bound by shared-memory bandwidth (16 B per complex per access, 128 B/clk/SM), and three table
// reads per butterfly were 27% of it; the two extra complex products are free on the idle FP64
// pipe (measured: 1024-point fwd+inv 7.5k -> 4.4k cycles, tools/fft_ubench.cu).  W^0 = 1 exactly,
// so no k == 0 branch is needed.
__device__ __forceinline__ void tw3(const Smem &sm, int e, double2 &w1, double2 &w2, double2 &w3) {
  w1 = twid(sm, e);
  w2 = cmul(w1, w1);
  w3 = cmul(w2, w1);
}

template <bool INV, int RADIX>
__device__ __forceinline__ void fft_stage(double2 *A, int L1, int lm, const Smem &sm, int L1e) {
  const int lmp = lm - (RADIX == 4 ? 2 : 1);
  const int mprev = 1 << lmp;
  const int tstep = L1e >> lm;
  const int nb = L1 / RADIX;
  for (int b = threadIdx.x; b < nb; b += kThreads) {
    const int k = b & (mprev - 1);
    const int base = ((b >> lmp) << lm) + k;
    if constexpr (RADIX == 4) {
      const int p0 = pidx(base), p1 = pidx(base + mprev), p2 = pidx(base + 2 * mprev), p3 = pidx(base + 3 * mprev);
      double2 a0 = A[p0], a1 = A[p1], a2 = A[p2], a3 = A[p3];
      double2 w1, w2, w3;
      tw3(sm, k * tstep, w1, w2, w3);
      if (INV) {
        a1 = cmulc(a1, w1); a2 = cmulc(a2, w2); a3 = cmulc(a3, w3);
        bfly4<true>(a0, a1, a2, a3);
      } else {
        bfly4<false>(a0, a1, a2, a3);
        a1 = cmul(a1, w1); a2 = cmul(a2, w2); a3 = cmul(a3, w3);
      }
      A[p0] = a0; A[p1] = a1; A[p2] = a2; A[p3] = a3;
    } else {
      const int p0 = pidx(base), p1 = pidx(base + mprev);
      double2 a0 = A[p0], a1 = A[p1];
      const double2 w = twid(sm, k * tstep);
      if (INV) {
        a1 = cmulc(a1, w);
        A[p0] = cadd(a0, a1); A[p1] = csub(a0, a1);
      } else {
        A[p0] = cadd(a0, a1); A[p1] = cmul(csub(a0, a1), w);
      }
    }
  }
}

// Two consecutive radix-4 stages s (m = 2^lm) and s-1 (m/4) fused in registers: a thread owns
// the 16 positions g m + j (m/4) + j' (m/16) + k'' and applies exactly the butterflies of both
// stages (DIF: s then s-1; DIT: s-1 then s), so the data placement equals the unfused plan.
template <bool INV>
__device__ __forceinline__ void fft_pass16(double2 *A, int L1, int lm, const Smem &sm, int L1e) {
  const int lmpp = lm - 4;
  const int mp = 1 << (lm - 2), mpp = 1 << lmpp;
  const int ts = L1e >> lm;          // W_m^x   = W_{L1e}^{x ts}
  const int tsp = L1e >> (lm - 2);   // W_{m/4}^x = W_{L1e}^{x tsp}
  const int nsb = L1 >> 4;
  for (int u = threadIdx.x; u < nsb; u += kThreads) {
    const int kpp = u & (mpp - 1);
    const int base = ((u >> lmpp) << lm) + kpp;
    double2 x[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) x[j][jp] = A[pidx(base + j * mp + jp * mpp)];
    if (!INV) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {            // stage s: butterfly k = jp mpp + kpp
        bfly4<false>(x[0][jp], x[1][jp], x[2][jp], x[3][jp]);
        double2 v1, v2, v3;
        tw3(sm, (jp * mpp + kpp) * ts, v1, v2, v3);
        x[1][jp] = cmul(x[1][jp], v1);
        x[2][jp] = cmul(x[2][jp], v2);
        x[3][jp] = cmul(x[3][jp], v3);
      }
      double2 w1, w2, w3;
      tw3(sm, kpp * tsp, w1, w2, w3);
#pragma unroll
      for (int j = 0; j < 4; ++j) {               // stage s-1: butterfly k = kpp in group 4g + j
        bfly4<false>(x[j][0], x[j][1], x[j][2], x[j][3]);
        x[j][1] = cmul(x[j][1], w1);
        x[j][2] = cmul(x[j][2], w2);
        x[j][3] = cmul(x[j][3], w3);
      }
    } else {
      double2 w1, w2, w3;
      tw3(sm, kpp * tsp, w1, w2, w3);
#pragma unroll
      for (int j = 0; j < 4; ++j) {               // DIT stage s-1
        x[j][1] = cmulc(x[j][1], w1);
        x[j][2] = cmulc(x[j][2], w2);
        x[j][3] = cmulc(x[j][3], w3);
        bfly4<true>(x[j][0], x[j][1], x[j][2], x[j][3]);
      }
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {            // DIT stage s
        double2 v1, v2, v3;
        tw3(sm, (jp * mpp + kpp) * ts, v1, v2, v3);
        x[1][jp] = cmulc(x[1][jp], v1);
        x[2][jp] = cmulc(x[2][jp], v2);
        x[3][jp] = cmulc(x[3][jp], v3);
        bfly4<true>(x[0][jp], x[1][jp], x[2][jp], x[3][jp]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) A[pidx(base + j * mp + jp * mpp)] = x[j][jp];
  }
}

// Compile-time-specialised radix-4 plan for the resident (direct twiddle table) lengths of the
// C3 cluster kernels: all index arithmetic folds to shifts/masks of constants (same data
// placement as local_fft).
template <bool INV, int LM>
__device__ __forceinline__ void st4_ct(double2 *A, int L1, const double2 *twd, int L1e) {
  constexpr int lmp = LM - 2, mprev = 1 << lmp;
  const int nb = L1 >> 2;
  for (int b = threadIdx.x; b < nb; b += kThreads) {
    const int k = b & (mprev - 1);
    const int base = ((b >> lmp) << LM) + k;
    const int p0 = pidx(base), p1 = pidx(base + mprev), p2 = pidx(base + 2 * mprev), p3 = pidx(base + 3 * mprev);
    double2 a0 = A[p0], a1 = A[p1], a2 = A[p2], a3 = A[p3];
    const double2 w1 = twd[(L1e - (1 << LM)) / 3 + k];   // per-stage table (tws)
    const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
    if (INV) {
      a1 = cmulc(a1, w1); a2 = cmulc(a2, w2); a3 = cmulc(a3, w3);
      bfly4<true>(a0, a1, a2, a3);
    } else {
      bfly4<false>(a0, a1, a2, a3);
      a1 = cmul(a1, w1); a2 = cmul(a2, w2); a3 = cmul(a3, w3);
    }
    A[p0] = a0; A[p1] = a1; A[p2] = a2; A[p3] = a3;
  }
}
template <bool INV, int L, int S>   // radix-4 stages S-1 .. 0 (DIF) or 0 .. S-1 (DIT)
struct Ct4 {
  __device__ __forceinline__ static void run(double2 *A, const double2 *twd, int L1e) {
    if constexpr (S > 0) {
      if constexpr (!INV) {
        st4_ct<false, 2 * S>(A, L, twd, L1e);
        __syncthreads();
        Ct4<INV, L, S - 1>::run(A, twd, L1e);
      } else {
        Ct4<INV, L, S - 1>::run(A, twd, L1e);
        st4_ct<true, 2 * S>(A, L, twd, L1e);
        __syncthreads();
      }
    }
  }
};
template <bool INV, int L>
__device__ __forceinline__ void local_fft_ct(double2 *A, const double2 *twd, int L1e) {
  constexpr int l = __builtin_ctz(L), S4 = l / 2;
  constexpr bool r2 = l & 1;
  if constexpr (!INV) {
    if constexpr (r2) {
      for (int b = threadIdx.x; b < L / 2; b += kThreads) {
        const int p0 = pidx(b), p1 = pidx(b + L / 2);
        const double2 a0 = A[p0], a1 = A[p1];
        A[p0] = cadd(a0, a1);
        A[p1] = cmul(csub(a0, a1), twd[(L1e - 1) / 3 + b]);
      }
      __syncthreads();
    }
    Ct4<false, L, S4>::run(A, twd, L1e);
  } else {
    Ct4<true, L, S4>::run(A, twd, L1e);
    if constexpr (r2) {
      for (int b = threadIdx.x; b < L / 2; b += kThreads) {
        const int p0 = pidx(b), p1 = pidx(b + L / 2);
        const double2 a0 = A[p0];
        const double2 a1 = cmulc(A[p1], twd[(L1e - 1) / 3 + b]);
        A[p0] = cadd(a0, a1);
        A[p1] = csub(a0, a1);
      }
      __syncthreads();
    }
  }
}

template <int L, int S>   // forward radix-4 stages S-1 .. 1 (all but the last), each followed by a barrier
struct Ct4Top {
  __device__ __forceinline__ static void run(double2 *A, const double2 *twd, int L1e) {
    if constexpr (S > 1) {
      st4_ct<false, 2 * S>(A, L, twd, L1e);
      __syncthreads();
      Ct4Top<L, S - 1>::run(A, twd, L1e);
    }
  }
};
// Last forward DIF stage (radix 4, m = 4, twiddle-free) handing its outputs to `out`.  Below
// 4 kThreads points several threads share a butterfly (each loads it, pushes a subset of its
// outputs), so every thread takes part in the push-in.
template <int L, class OUT>
__device__ __forceinline__ void last_stage_out(const double2 *A, const OUT &out) {
  constexpr int NB = L / 4;
  if constexpr (NB >= kThreads) {
    for (int b = threadIdx.x; b < NB; b += kThreads) {
      double2 a0 = A[pidx(4 * b)], a1 = A[pidx(4 * b + 1)], a2 = A[pidx(4 * b + 2)], a3 = A[pidx(4 * b + 3)];
      bfly4<false>(a0, a1, a2, a3);
      out(4 * b, a0); out(4 * b + 1, a1); out(4 * b + 2, a2); out(4 * b + 3, a3);
    }
  } else {
    constexpr int R = kThreads / NB;
    const int b = threadIdx.x % NB, h = threadIdx.x / NB;
    if (h < 4) {
      double2 a[4] = {A[pidx(4 * b)], A[pidx(4 * b + 1)], A[pidx(4 * b + 2)], A[pidx(4 * b + 3)]};
      bfly4<false>(a[0], a[1], a[2], a[3]);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j % R == h) out(4 * b + j, a[j]);
    }
  }
}

// Forward compile-time FFT whose last DIF stage (radix 4, m = 4, twiddle-free) hands every output
// slot to a functor instead of storing it (cross_push's push-in).  No trailing barrier.
template <int L, class OUT>
__device__ __forceinline__ void local_fft_ct_fwd_out(double2 *A, const double2 *twd, int L1e, const OUT &out) {
  constexpr int l = __builtin_ctz(L), S4 = l / 2;
  constexpr bool r2 = l & 1;
  if constexpr (r2) {
    for (int b = threadIdx.x; b < L / 2; b += kThreads) {
      const int p0 = pidx(b), p1 = pidx(b + L / 2);
      const double2 a0 = A[p0], a1 = A[p1];
      A[p0] = cadd(a0, a1);
      A[p1] = cmul(csub(a0, a1), twd[(L1e - 1) / 3 + b]);
    }
    __syncthreads();
  }
  Ct4Top<L, S4>::run(A, twd, L1e);
  last_stage_out<L>(A, out);
}

// Requires the input to be visible to all threads (caller synchronizes); ends synchronized.
// Radix-4 stages are fused pairwise into radix-16 register passes from the bottom (stages
// (1,0), (3,2), ...); a leftover top radix-4 stage and the radix-2 stage run alone.
template <bool INV>
__device__ __forceinline__ void local_fft(double2 *A, int L1, const Smem &sm, int L1e) {
#ifndef TSF_NO_CT_FFT
  if (sm.tws != nullptr && L1e == 1024) {       // C3's resident cluster kernels (n = 2^14, C = 16)
    if (L1 == 1024) { local_fft_ct<INV, 1024>(A, sm.tws, L1e); return; }
    if (L1 == 512) { local_fft_ct<INV, 512>(A, sm.tws, L1e); return; }
  }
  if (sm.tws != nullptr && L1e == 256) {        // C2's (n = 2^10, C = 4)
    if (L1 == 256) { local_fft_ct<INV, 256>(A, sm.tws, L1e); return; }
    if (L1 == 128) { local_fft_ct<INV, 128>(A, sm.tws, L1e); return; }
  }
#endif
  const int l = __ffs(L1) - 1;
  const int S4 = l >> 1;
  const bool r2 = l & 1;
  // fuse when the local length reaches sm.fuse_min (default: every thread owns a 16-point
  // super-butterfly); the data placement is the same either way
  const bool fuse = L1 >= sm.fuse_min && L1 >= 256;
  const int npair = fuse ? (S4 >> 1) : 0;   // fused pairs (2i+1, 2i), i < npair
  if (!fuse) {
    if (!INV) {
      if (r2) { fft_stage<false, 2>(A, L1, l, sm, L1e); __syncthreads(); }
      for (int s = S4 - 1; s >= 0; --s) { fft_stage<false, 4>(A, L1, 2 * (s + 1), sm, L1e); __syncthreads(); }
    } else {
      for (int s = 0; s < S4; ++s) { fft_stage<true, 4>(A, L1, 2 * (s + 1), sm, L1e); __syncthreads(); }
      if (r2) { fft_stage<true, 2>(A, L1, l, sm, L1e); __syncthreads(); }
    }
    return;
  }
  const bool lone = S4 & 1;           // stage S4-1 alone
  if (!INV) {
    if (r2) { fft_stage<false, 2>(A, L1, l, sm, L1e); __syncthreads(); }
    if (lone) { fft_stage<false, 4>(A, L1, 2 * S4, sm, L1e); __syncthreads(); }
    for (int i = npair - 1; i >= 0; --i) {
      fft_pass16<false>(A, L1, 4 * i + 4, sm, L1e);   // stages 2i+1 (m = 4^{2i+2}) and 2i
      __syncthreads();
    }
  } else {
    for (int i = 0; i < npair; ++i) {
      fft_pass16<true>(A, L1, 4 * i + 4, sm, L1e);
      __syncthreads();
    }
    if (lone) { fft_stage<true, 4>(A, L1, 2 * S4, sm, L1e); __syncthreads(); }
    if (r2) { fft_stage<true, 2>(A, L1, l, sm, L1e); __syncthreads(); }
  }
}

// ------------------------------------------------------------------------ register DFT_C
__device__ __forceinline__ double2 w16(int e) {  // exp(-2 pi i e / 16), e in [0,16)
  const double c[16] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
                        0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
                        -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977,
                        0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674};
  return make_double2(c[e & 15], -c[(e + 12) & 15]);
}

template <int N>
__host__ __device__ constexpr int brev(int i) {
  int r = 0;
  for (int b = 1; b < N; b <<= 1) r = (r << 1) | ((i & b) ? 1 : 0);
  return r;
}

// In-register radix-2 FFT of N <= 16 points: forward X_k = sum x_q W_N^{qk}; INV uses W^{-1}.
template <int N, bool INV>
__device__ __forceinline__ void fft_reg(double2 (&x)[N]) {
  if constexpr (N == 2) {
    const double2 a = x[0];
    x[0] = cadd(a, x[1]);
    x[1] = csub(a, x[1]);
  } else if constexpr (N == 4) {
    bfly4<INV>(x[0], x[1], x[2], x[3]);     // natural-order 4-point DFT, no products by 0 / 1
  } else if constexpr (N > 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = brev<N>(i);
      if (j > i) { const double2 t = x[i]; x[i] = x[j]; x[j] = t; }
    }
#pragma unroll
    for (int m = 2; m <= N; m <<= 1) {
#pragma unroll
      for (int k = 0; k < m / 2; ++k) {
        double2 w = w16(k * (16 / m));
        if (INV) w = cconj(w);
#pragma unroll
        for (int g = 0; g < N; g += m) {
          const double2 a = x[g + k];
          const double2 b = cmul(x[g + k + m / 2], w);
          x[g + k] = cadd(a, b);
          x[g + k + m / 2] = csub(a, b);
        }
      }
    }
  }
}

// ------------------------------------------------------------------------ spectral op
// lambda(bin) = eta + mu * [ (p+q) Re L_W + q corr (-1)^bin + i ((p-q) Im L_W + c2 s(bin)) ]
// for L_W the base spectrum of W (embedding, Strang or T. Chan), s the sine table of Lambda_Q,
// optionally conjugated (A^T, P^T).  Multiply (A, B, A^T) or divide (P^{-1}, P^{-T}).
// Explicit shared-memory loads for pointers the compiler cannot prove to be shared.
__device__ __forceinline__ double2 lds2(const double2 *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ double lds1(const double *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

struct SpecOp {
  const double2 *lam;   // task-order base spectrum of this instance (global)
  const double *sq;     // task-order sine table (global)
  const double2 *mul;   // per-level effective multipliers (task order) or nullptr: then formed
                        // from lam/sq on the fly (the once-per-level B operator)
  const double2 *pw;    // resident: pair twiddles W_{2L}^{bin} of this CTA's slice, else nullptr
  double2 nyq;          // base spectrum at the Nyquist bin L
  double2 nyqe;         // effective multiplier at the Nyquist bin (formed once by make_op)
  int np;               // column-pair tasks per CTA
  int rC;               // r * C: task-order index base of this CTA in the global tables
  bool mul_sh;          // mul is this CTA's slice in SMEM (else the global task-order table)
  double eta, mu, ppq, pmq, c2, qcorr, scale;
  bool conj;
  bool div;             // apply 1/lambda (circulant solve) instead of lambda
  // multiplier of a bin: lambda, or 1/lambda = conj(lambda)/|lambda|^2 for a solve
  __device__ __forceinline__ double2 eff(double2 l) const {
    if (!div) return l;
    const double inv = 1.0 / (l.x * l.x + l.y * l.y);
    return make_double2(l.x * inv, -l.y * inv);
  }
  // W_{2L}^{bin} of bin (k2, ab, i): resident table or the global twiddle table
  __device__ __forceinline__ double2 wtw(int k2, int ab, int i, int bin, const double2 *tw,
                                         int tw2L) const {
    return pw ? lds2(pw + (k2 * 2 + ab) * np + i) : tw[bin * tw2L];
  }
  __device__ __forceinline__ double2 lam_idx(int idx, int bin) const {
    const double2 b = lam[idx];
    const double s = sq[idx];
    const double re = ppq * b.x + ((bin & 1) ? -qcorr : qcorr);
    const double im = pmq * b.y + c2 * s;
    return make_double2(eta + mu * re, conj ? -(mu * im) : mu * im);
  }
  // effective multiplier (lambda or 1/lambda) of bin (k2, ab, i)
  __device__ __forceinline__ double2 get(int k2, int ab, int i, int bin) const {
    if (mul) {
      const double2 m = mul_sh ? lds2(mul + (k2 * 2 + ab) * np + i) : mul[((rC + k2) * 2 + ab) * np + i];
      return conj ? cconj(m) : m;
    }
    return eff(lam_idx(((rC + k2) * 2 + ab) * np + i, bin));
  }
  __device__ __forceinline__ double2 nyquist_lam(int Lbin) const {
    const double re = ppq * nyq.x + ((Lbin & 1) ? -qcorr : qcorr);
    const double im = pmq * nyq.y;
    return make_double2(eta + mu * re, conj ? -(mu * im) : mu * im);
  }
  __device__ __forceinline__ double2 nyquist(int Lbin) const { return eff(nyquist_lam(Lbin)); }
};

// Real-FFT split for the pair of bins (k, L-k) of a length-L complex transform z of a
// 2L-point real sequence x (z_m = x_{2m} + i x_{2m+1}), apply Y = X * la (bin k) and
// Y = X * lb (bin L-k), la/lb the effective multipliers (lambda or 1/lambda), and merge back to
// Z' such that the unnormalized inverse DFT of Z' returns y packed the same way.
// w = exp(-i pi k / L); s = 1/(4L) folds the halves and 1/L.
__device__ __forceinline__ void pair_apply(double2 &Za, double2 &Zb, double2 la, double2 lb,
                                           double2 w, double s) {
  const double2 cZb = cconj(Zb);
  const double2 Ep = cadd(Za, cZb);               // 2 E_k
  const double2 Op = mul_mi(csub(Za, cZb));       // 2 O_k
  const double2 wO = cmul(w, Op);
  const double2 Xa = cadd(Ep, wO);                // 2 X_k
  const double2 Xb = cconj(csub(Ep, wO));         // 2 X_{L-k}
  const double2 Ya = cmul(Xa, la);
  const double2 Yb = cmul(Xb, lb);
  const double2 cYb = cconj(Yb);
  const double2 E2 = cadd(Ya, cYb);               // 4 E'_k
  const double2 O2 = cmulc(csub(Ya, cYb), w);     // 4 O'_k
  Za = cscale(cadd(E2, mul_i(O2)), s);
  Zb = cscale(cadd(cconj(E2), mul_i(cconj(O2))), s);
}

__device__ __forceinline__ void pair_self(double2 &Z, double2 la, double2 lb, double2 w, double s) {
  double2 a = Z, b = Z;
  pair_apply(a, b, la, lb, w, s);
  Z = a;
}

struct Geo {
  int L1, L, np, twL, tw2L;   // twL = twN/L (W_L factor), tw2L = twN/(2L)
  int l1;                     // log2(L1)
  int lr, ls;                 // multi-pass regime: L1 = R x S, lr = log2 R, ls = log2 S (else 0, l1)
  int lnp;                    // log2(np): task indices split by shifts, not integer division
  const int32_t *slot;
  const double2 *ctw;         // resident column twiddles W_L^{q k1(col)} [q ncol + col]
};

// C == 1: the whole transform is local; column pairs are bin pairs (k, L-k).  Slots come from
// the exported slot table (L1-resident; measured faster here than the closed-form dslot).  Two
// pairs per thread and step, their table loads issued together (the loop is latency bound).
__device__ __forceinline__ void pointwise_local(double2 *A, const Geo &g, const SpecOp &op,
                                             const double2 *__restrict__ tw) {
  if (threadIdx.x == 0) {
    const int sa = pidx(g.slot[0]), sb = pidx(g.slot[g.L1 / 2]);
    double2 a = A[sa], b = A[sb];
    pair_self(a, op.get(0, 0, 0, 0), op.nyqe, tw[0], op.scale);
    const double2 lm = op.get(0, 1, 0, g.L / 2);
    pair_self(b, lm, lm, tw[(g.L / 2) * g.tw2L], op.scale);
    A[sa] = a; A[sb] = b;
  }
  for (int i0 = threadIdx.x + 1; i0 < g.np; i0 += 2 * kThreads) {
    const int i1 = i0 + kThreads;
    const bool h1 = i1 < g.np;
    const int j1 = h1 ? i1 : i0;
    const double2 la0 = op.get(0, 0, i0, i0), lb0 = op.get(0, 1, i0, g.L - i0);
    const double2 la1 = op.get(0, 0, j1, j1), lb1 = op.get(0, 1, j1, g.L - j1);
    const double2 w0 = tw[i0 * g.tw2L], w1 = tw[j1 * g.tw2L];
    const int sa0 = pidx(g.slot[i0]), sb0 = pidx(g.slot[g.L1 - i0]);
    const int sa1 = pidx(g.slot[j1]), sb1 = pidx(g.slot[g.L1 - j1]);
    double2 a0 = A[sa0], b0 = A[sb0], a1 = A[sa1], b1 = A[sb1];
    pair_apply(a0, b0, la0, lb0, w0, op.scale);
    pair_apply(a1, b1, la1, lb1, w1, op.scale);
    A[sa0] = a0; A[sb0] = b0;
    if (h1) { A[sa1] = a1; A[sb1] = b1; }
  }
}

// column pair i of CTA r: (k1a, k1b) = (pi, L1 - pi) with pi = r + i C, or (0, L1/2) for pi = 0
__device__ __forceinline__ int col_k1(int L1, int C, uint32_t r, int col) {
  const int pi = int(r) + (col >> 1) * C;
  if (pi == 0) return (col & 1) ? L1 / 2 : 0;
  return (col & 1) ? L1 - pi : pi;
}

// Slot of local bin k1 in a CTA's staged transform output (xg row): the SMEM DIF FFT puts bin k
// in slot dslot(k); in the multi-pass regime row rho' = k1 mod R holds the S-point spectrum of
// bins rho' + R k (see apply_big), so k1 sits at rho' S + dslot(k1 / R).
__device__ __forceinline__ int gslot(const Geo &g, int k1) {
  return ((k1 & ((1 << g.lr) - 1)) << g.ls) + dslot(k1 >> g.lr, g.ls);
}

// ------------------------------------------------------------------------ staged column stage
// Thread split of the length-C column DFTs (C = T x Q): T lanes per column, Q points per lane,
// a column PAIR (i, 0) / (i, 1) on G = 2T consecutive lanes, so both columns of every real-split
// bin pair sit in one lane group and the whole stage runs in registers with shuffles.
#ifndef TSF_COL_T16
#define TSF_COL_T16 4      // lanes per column at C = 16 (4: 4 points per lane; 1: whole column)
#endif
template <int C> struct ColSplit {
  static constexpr int T = C >= 16 ? TSF_COL_T16 : 1;   // C <= 8: a whole column per lane
  static constexpr int Q = C / T;
  static constexpr int G = 2 * T;
  static constexpr int LT = T == 4 ? 2 : (T == 2 ? 1 : 0);
  static constexpr int SH = 2 - LT;          // log2(8 / G): XOR key shift of the B swizzle
};

// Receive-buffer index of row q (source CTA) of column t = ab np + i.  The column stage reads,
// per lane group, rows q = s + T m of both columns of pair i; the XOR key (s, ab) << SH spreads
// the 8 lanes of each 16-byte-access phase over 8 distinct bank groups (np >= 8).
template <int C>
__device__ __forceinline__ int bix(int q, int t, int ncol, int lnp) {
  using S = ColSplit<C>;
  if (C < 16 || lnp < 3) return q * ncol + t;   // C < 16: the column-per-thread stage reads rows
  const int key = ((q & (S::T - 1)) | (((t >> lnp) & 1) << S::LT)) << S::SH;
  return q * ncol + (t ^ key);
}

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m, unsigned mask) {
  return make_double2(__shfl_xor_sync(mask, v.x, m), __shfl_xor_sync(mask, v.y, m));
}

// x[k] *= W_C^{s k} (k < N compile-time slots, s < T runtime) from the SMEM table W_C^e
template <int C, int N>
__device__ __forceinline__ void twiddle_tab(double2 (&x)[N], int s, const double2 *twc) {
#pragma unroll
  for (int k = 1; k < N; ++k) x[k] = cmul(x[k], lds2(twc + ((s * k) & (C - 1))));
}

// In-group transposition (T lanes): lane s holds slots sigma; round b moves every slot whose
// bit b differs from the lane's bit b to lane s ^ b, at slot sigma ^ b (an involution, so the
// inverse runs the rounds in reverse order).
template <int T, int Q>
__device__ __forceinline__ void group_transpose(double2 (&x)[Q], int s, unsigned mask, bool rev) {
#pragma unroll
  for (int bi = 0; bi < 2; ++bi) {
    const int b = rev ? (T >> 1) >> bi : 1 << bi;
    if (b >= T || b == 0) continue;
    const bool hi = s & b;
#pragma unroll
    for (int s0 = 0; s0 < Q; ++s0) {
      if (s0 & b) continue;
      const int s1 = s0 | b;
      const double2 send = hi ? x[s0] : x[s1];
      const double2 recv = shfl_xor2(send, b, mask);
      if (hi) x[s0] = recv; else x[s1] = recv;
    }
  }
}

// Push of local DIF output slot p (bin k1 = dperm(p)) into row r of the B buffer of the CTA that
// owns k1's column pair (cross_push); callable from the last forward FFT stage.
template <int C>
struct PushIn {
  uint32_t bB, aB;
  int L1, l1, np, ncol, lnp, r;
  __device__ __forceinline__ PushIn(double2 *B, uint64_t *mbB, const Geo &g, uint32_t rr)
      : bB(smem_u32(B)), aB(smem_u32(mbB)), L1(g.L1), l1(g.l1), np(g.np), ncol(g.L1 / C), lnp(g.lnp),
        r(int(rr)) {}
  __device__ __forceinline__ void operator()(int p, double2 v) const {
    const int k1 = dperm(p, l1);
    int pi, ab;
    if (k1 == 0) { pi = 0; ab = 0; }
    else if (k1 == L1 / 2) { pi = 0; ab = 1; }
    else if (k1 < L1 / 2) { pi = k1; ab = 0; }
    else { pi = L1 - k1; ab = 1; }
    const uint32_t q = uint32_t(pi) & (C - 1);
    const int idx = bix<C>(r, ab * np + pi / C, ncol, lnp);
    push2(mapa_u32(bB + 16u * idx, q), v, mapa_u32(aB, q));
  }
};

// C > 1, staged: the four-step column stage through the receive buffer B and the output O,
// both filled by pushes.  Steps: push the local DIF output (slot
// p holds bin dperm(p)) into row r of the owner's B (layout bix); per column pair, on its lane
// group: column DFT_C (twiddles W_L^{q k1}, Q-point DFTs in registers, in-group transposition,
// T-point DFTs), the real split + spectral op of every bin pair (k2, (i,0)) <-> (C-1-k2, (i,1))
// with the partner lane (lane ^ (2T-1), slot Q-1-sigma), the inverse column DFT, conjugate
// twiddles, and push row q back to CTA q's O at the slot of k1.  The pseudo column pair
// (0, L1/2) of CTA 0 pairs bins inside each column and is redone by warp 0 through B.
// Returns with O complete and visible.
template <int C>
__device__ __forceinline__ void cross_push(double2 *A, double2 *B, double2 *O, const Geo &g,
                                           const SpecOp &op, const double2 *__restrict__ tw, uint32_t r,
                                           const Smem &sm, Xch &xs, bool prepushed = false) {
  using S = ColSplit<C>;
  constexpr int T = S::T, Q = S::Q, G = S::G;
  TSF_PT0();
  const int L1 = g.L1, l1 = g.l1, ncol = L1 / C, np = g.np, lnp = g.lnp;
  uint64_t *mbB = sm.mbar, *mbO = sm.mbar + 1;
  const uint32_t ph = xs.nap & 1;
  if (threadIdx.x == 0) {
    mbar_expect(mbB, uint32_t(L1 * 16));
    mbar_expect(mbO, uint32_t(L1 * 16));
  }
  if (!prepushed) {
    const PushIn<C> pin(B, mbB, g, r);
#pragma unroll 4
    for (int p = threadIdx.x; p < L1; p += kThreads) pin(p, A[pidx(p)]);
  }
  // pseudo column pair items of CTA 0 (warp 0, one pair per lane): twiddles prefetched
  constexpr int NPS = C / 2 + 1 + (C + 1) / 2;
  const int lane32 = threadIdx.x & 31;
  double2 wps = make_double2(1.0, 0.0);
  if (r == 0 && threadIdx.x < NPS) {
    const bool c0 = lane32 <= C / 2;
    const int k2 = c0 ? lane32 : lane32 - (C / 2 + 1);
    const int bin = c0 ? L1 * k2 : L1 / 2 + L1 * k2;
    wps = tw[bin * g.tw2L];
  }
  mbar_wait(mbB, ph);
  TSF_PACC(sm, PS_GATHER);
  if constexpr (C < 16) {
    // C <= 8: one thread per column (rows in registers), the bin pairs on all threads through B,
    // one thread per column for the inverse (measured faster than lane groups at C = 2, 4)
  for (int t = threadIdx.x; t < ncol; t += kThreads) {        // column DFT_C
    const int ab = t >> g.lnp, i = t & (np - 1), colo = 2 * i + ab;
    const int k1 = col_k1(L1, C, r, colo);
    double2 z[C];
#pragma unroll
    for (int q = 0; q < C; ++q) z[q] = B[q * ncol + t];
    if (g.ctw) {
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmul(z[q], g.ctw[q * ncol + colo]);
    } else {
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmul(z[q], tw[q * k1 * g.twL]);
    }
    fft_reg<C, false>(z);
#pragma unroll
    for (int q = 0; q < C; ++q) B[q * ncol + t] = z[q];
  }
  __syncthreads();
  TSF_PACC(sm, PS_COLF);
  // bin pairs: item u = k2 * np + i; regular pair (row k2, col (i,0)) <-> (row C-1-k2, col (i,1)).
  // The pseudo column pair (0, L1/2) of CTA 0 is done afterwards by warp 0, one pair per lane:
  // inside the item loop its branch diverged from the regular lanes in every warp and made
  // CTA 0's stage ~2.4x longer than its peers' (measured), which all of them then waited for.
  for (int u = threadIdx.x; u < np * C; u += kThreads) {
    const int k2 = u >> g.lnp, i = u & (np - 1);
    const int pi = int(r) + i * C;
    if (pi == 0) continue;
    const int bin = pi + L1 * k2;
    double2 &za = B[k2 * ncol + i];
    double2 &zb = B[(C - 1 - k2) * ncol + np + i];
    double2 a = za, b = zb;
    pair_apply(a, b, op.get(k2, 0, i, bin), op.get(C - 1 - k2, 1, i, g.L - bin),
               op.wtw(k2, 0, i, bin, tw, g.tw2L), op.scale);
    za = a;
    zb = b;
  }
  if (r == 0 && threadIdx.x < C / 2 + 1 + (C + 1) / 2) {
    // one bin pair per lane, branch-free (operands selected, a single pair_apply):
    // column 0 (bins L1 k2): k2 <-> (C - k2) mod C, k2 = 0 with the Nyquist bin;
    // column L1/2 (bins L1/2 + L1 k2): k2 <-> C - 1 - k2
    const int o = threadIdx.x;
    const bool c0 = o <= C / 2;
    const int k2 = c0 ? o : o - (C / 2 + 1);
    const int kp = c0 ? (C - k2) % C : C - 1 - k2;
    const int ab = c0 ? 0 : 1;
    const int cof = c0 ? 0 : np;
    const int bin = c0 ? L1 * k2 : L1 / 2 + L1 * k2;
    const bool self = kp == k2;
    const double2 la = op.get(k2, ab, 0, bin);
    const double2 lp = op.get(kp, ab, 0, g.L - bin);
    const double2 lb = self ? ((c0 && k2 == 0) ? op.nyqe : la) : lp;
    const double2 w = op.wtw(k2, ab, 0, bin, tw, g.tw2L);
    double2 &za = B[k2 * ncol + cof];
    double2 a = za, b = self ? za : B[kp * ncol + cof];
    pair_apply(a, b, la, lb, w, op.scale);
    za = a;
    if (!self) B[kp * ncol + cof] = b;
  }
  __syncthreads();
  TSF_PACC(sm, PS_PAIRS);
  {
    const uint32_t bO = smem_u32(O), aO = smem_u32(mbO);
    for (int t = threadIdx.x; t < ncol; t += kThreads) {      // inverse column DFT_C + push back
      const int ab = t >> g.lnp, i = t & (np - 1), colo = 2 * i + ab;
      const int k1 = col_k1(L1, C, r, colo);
      double2 z[C];
#pragma unroll
      for (int q = 0; q < C; ++q) z[q] = B[q * ncol + t];
      fft_reg<C, true>(z);
      if (g.ctw) {
#pragma unroll
        for (int q = 1; q < C; ++q) z[q] = cmulc(z[q], g.ctw[q * ncol + colo]);
      } else {
#pragma unroll
        for (int q = 1; q < C; ++q) z[q] = cmulc(z[q], tw[q * k1 * g.twL]);
      }
      const uint32_t dst = bO + 16u * uint32_t(pidx(dslot(k1, l1)));
#pragma unroll
      for (int q = 0; q < C; ++q) push2(mapa_u32(dst, uint32_t(q)), z[q], mapa_u32(aO, uint32_t(q)));
    }
  }
  } else {
  const int lane = threadIdx.x & (G - 1), ab = lane >> S::LT, s = lane & (T - 1);
  const unsigned gmask = ((1u << G) - 1u) << (lane32 & ~(G - 1));
  const uint32_t bO = smem_u32(O), aO = smem_u32(mbO);
  const int nsh = np * C;                     // offset of the b-side multipliers (SMEM layout)
  const bool msh = op.mul != nullptr && op.mul_sh;   // per-level table in SMEM (B forms lambda)
  for (int i = threadIdx.x / G; i < np; i += kThreads / G) {
    const int t = ab * np + i, colo = 2 * i + ab;
    const int k1 = col_k1(L1, C, r, colo);
    const int pi = int(r) + i * C;
    double2 x[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m) {             // column DFT_C, rows q = s + T m
      const int q = s + T * m;
      x[m] = cmul(B[bix<C>(q, t, ncol, lnp)], g.ctw ? lds2(g.ctw + ctw_idx<C>(q, i, ab, np)) : tw[q * k1 * g.twL]);
    }
    fft_reg<Q, false>(x);
    if constexpr (T > 1) twiddle_tab<C, Q>(x, s, sm.twc);
    group_transpose<T, Q>(x, s, gmask, false);
#pragma unroll
    for (int j = 0; j < Q / T; ++j) {         // slot j T + kb holds bin k2 = s + T j + Q kb
      double2 y[T];
#pragma unroll
      for (int kb = 0; kb < T; ++kb) y[kb] = x[j * T + kb];
      fft_reg<T, false>(y);
#pragma unroll
      for (int kb = 0; kb < T; ++kb) x[j * T + kb] = y[kb];
    }
    const bool pseudo = (r == 0) && (i == 0);
    if (pseudo) {                             // pre-pair values for warp 0's pseudo pass
#pragma unroll
      for (int sg = 0; sg < Q; ++sg) B[bix<C>(s + T * (sg / T) + Q * (sg % T), t, ncol, lnp)] = x[sg];
    }
    {                                         // regular bin pairs with the partner lane
      double2 y[Q / 2];
#pragma unroll
      for (int jj = 0; jj < Q / 2; ++jj) y[jj] = shfl_xor2(x[Q - 1 - jj], G - 1, gmask);
#pragma unroll
      for (int jj = 0; jj < Q / 2; ++jj) {
        const int k2m = s + T * (jj / T) + Q * (jj % T);
        const int k2a = ab ? C - 1 - k2m : k2m;
        const int bin = pi + L1 * k2a;
        double2 la, lb, w;
        if (msh) {
          la = lds2(op.mul + i * C + k2a);
          lb = lds2(op.mul + nsh + i * C + k2a);
          if (op.conj) { la = cconj(la); lb = cconj(lb); }
        } else {
          la = op.get(k2a, 0, i, bin);
          lb = op.get(C - 1 - k2a, 1, i, g.L - bin);
        }
        w = op.pw ? lds2(op.pw + i * C + k2a) : tw[bin * g.tw2L];
        double2 a = ab ? y[jj] : x[jj], b = ab ? x[jj] : y[jj];
        pair_apply(a, b, la, lb, w, op.scale);
        x[jj] = ab ? b : a;
        y[jj] = ab ? a : b;
      }
#pragma unroll
      for (int jj = 0; jj < Q / 2; ++jj) x[Q - 1 - jj] = shfl_xor2(y[jj], G - 1, gmask);
    }
    if (r == 0 && threadIdx.x < 32 && i < 32 / G) {
      // warp 0, first pass: the pseudo column pair (0, L1/2), one bin pair per lane, branch-free:
      // column 0 (bins L1 k2): k2 <-> (C - k2) mod C, k2 = 0 with the Nyquist bin; column L1/2
      // (bins L1/2 + L1 k2): k2 <-> C - 1 - k2
      const int nact = np * G >= 32 ? 32 : np * G;
      const unsigned am = nact >= 32 ? 0xffffffffu : ((1u << nact) - 1u);
      __syncwarp(am);
      for (int o = lane32; o < NPS; o += nact) {
        const bool c0 = o <= C / 2;
        const int k2 = c0 ? o : o - (C / 2 + 1);
        const int kp = c0 ? (C - k2) % C : C - 1 - k2;
        const int abp = c0 ? 0 : 1;
        const int cof = c0 ? 0 : np;
        const int bin = c0 ? L1 * k2 : L1 / 2 + L1 * k2;
        const bool self = kp == k2;
        double2 la, lp;
        if (msh) {
          la = lds2(op.mul + (abp ? nsh + (C - 1 - k2) : k2));
          lp = lds2(op.mul + (abp ? nsh + (C - 1 - kp) : kp));
          if (op.conj) { la = cconj(la); lp = cconj(lp); }
        } else {
          la = op.get(k2, abp, 0, bin);
          lp = op.get(kp, abp, 0, g.L - bin);
        }
        const double2 lb = self ? ((c0 && k2 == 0) ? op.nyqe : la) : lp;
        const double2 w = o == lane32 ? wps : tw[bin * g.tw2L];
        double2 &za = B[bix<C>(k2, cof, ncol, lnp)];
        double2 a = za, b = self ? za : B[bix<C>(kp, cof, ncol, lnp)];
        pair_apply(a, b, la, lb, w, op.scale);
        za = a;
        if (!self) B[bix<C>(kp, cof, ncol, lnp)] = b;
      }
      __syncwarp(am);
      if (pseudo) {
#pragma unroll
        for (int sg = 0; sg < Q; ++sg) x[sg] = B[bix<C>(s + T * (sg / T) + Q * (sg % T), t, ncol, lnp)];
      }
    }
    // inverse column DFT_C: T-point inverse DFTs over kb, W_C^{-s' ka}, transposition back,
    // Q-point inverse DFTs -> row q = s + T m at slot m
#pragma unroll
    for (int j = 0; j < Q / T; ++j) {
      double2 y[T];
#pragma unroll
      for (int kb = 0; kb < T; ++kb) y[kb] = x[j * T + kb];
      fft_reg<T, true>(y);
      // slot j T + s' times W_C^{-s' (j T + s)}
      x[j * T] = y[0];
#pragma unroll
      for (int sp = 1; sp < T; ++sp) x[j * T + sp] = cmulc(y[sp], lds2(sm.twc + ((sp * (j * T + s)) & (C - 1))));
    }
    group_transpose<T, Q>(x, s, gmask, true);
    fft_reg<Q, true>(x);
    const uint32_t dst = bO + 16u * uint32_t(pidx(dslot(k1, l1)));
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      const int q = s + T * m;
      const double2 w = g.ctw ? lds2(g.ctw + ctw_idx<C>(q, i, ab, np)) : tw[q * k1 * g.twL];
      push2(mapa_u32(dst, uint32_t(q)), cmulc(x[m], w), mapa_u32(aO, uint32_t(q)));
    }
  }
  }
  TSF_PACC(sm, PS_COLI);
  mbar_wait(mbO, ph);
  xs.nap += 1;
  TSF_PACC(sm, PS_BAR3);
}

// Column twiddles W^{q k1}, q < C, from the single table value w = W^{k1}: products in a binary
// tree (depth log2 C), so each power carries at most log2(C) rounding steps; one global load
// per column instead of C - 1.
template <int C>
__device__ __forceinline__ void col_twiddles(double2 w, double2 (&wq)[C]) {
  wq[0] = make_double2(1.0, 0.0);
  if constexpr (C > 1) wq[1] = w;
#pragma unroll
  for (int p = 2; p < C; p *= 2) {
    wq[p] = cmul(wq[p / 2], wq[p / 2]);
#pragma unroll
    for (int q = 1; q < p && p + q < C; ++q) wq[p + q] = cmul(wq[p], wq[q]);
  }
}

// C > 1 without room for B and O (L1 = 8192, C5): the column stage in chunks of CP column
// pairs through a chunk buffer Bc (layout Bc[q * 2CP + 2 il + ab], conflict-free column reads).
// Per chunk: pull the rows of its columns from every CTA's A (DSMEM), column DFT_C, bin pairs,
// inverse column DFT_C and push the results straight back into the owners' A at the same slots.
// Slots of a column pair are read and written only by the pair's owner, so chunks need no
// cluster barrier; the caller's barriers order the local FFTs before the first pull and every
// push before the local inverse FFTs.
template <int C>
__device__ __forceinline__ void cross_chunked(double2 *A, double2 *Bc, int CP, const Geo &g, const SpecOp &op,
                                              const double2 *__restrict__ tw, uint32_t r, const Smem &sm,
                                              double2 *__restrict__ xg) {
  TSF_PT0();
  const int L1 = g.L1, np = g.np;
  const int W = 2 * CP;                       // columns per chunk
  // Every global (L2) access below is latency bound (~600-900 cycles per dependent round trip):
  // each thread issues a batch of independent loads before using any of them (memory-level
  // parallelism; one load in flight per thread gave ~7 B/clk/SM for the 128 KiB pull).
  const bool pre = op.mul != nullptr && !op.mul_sh && op.pw == nullptr;
  double2 *Ta = Bc + 2 * CP * C, *Tb = Ta + CP * C, *Tw = Tb + CP * C;
  for (int c0 = 0; c0 < np; c0 += CP) {
    const int cp = np - c0 < CP ? np - c0 : CP;
    // pull: item u -> (row q, chunk column col); the rows come from the peers' local FFT outputs
    // staged in L2 (xg[q][slot], written by the caller before its cluster barrier); async
    // copies, all of a thread's in flight at once
    const int tot = C * 2 * cp;
    for (int u = threadIdx.x; u < tot; u += kThreads) {
      const int q = u / (2 * cp), col = u - q * (2 * cp);
      const int k1 = col_k1(L1, C, r, 2 * c0 + col);
      cp_async16(Bc + q * W + col, xg + q * L1 + gslot(g, k1));
    }
    // the bin-pair stage's multipliers (task-order table, contiguous in i) and split twiddles,
    // prefetched with the pull so their L2 latency overlaps it
    if (pre) {
      for (int u = threadIdx.x; u < C * cp; u += kThreads) {
        const int k2 = u / cp, i = c0 + (u - k2 * cp);
        cp_async16(Ta + u, op.mul + ((op.rC + k2) * 2 + 0) * np + i);
        cp_async16(Tb + u, op.mul + ((op.rC + C - 1 - k2) * 2 + 1) * np + i);
        cp_async16(Tw + u, tw + int64_t(int(r) + i * C + L1 * k2) * g.tw2L);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    TSF_PACC(sm, PS_GATHER);
    for (int col = threadIdx.x; col < 2 * cp; col += kThreads) {   // column DFT_C
      const int k1 = col_k1(L1, C, r, 2 * c0 + col);
      double2 z[C];
#pragma unroll
      for (int q = 0; q < C; ++q) z[q] = Bc[q * W + col];
      double2 wq[C];
      col_twiddles<C>(tw[k1 * g.twL], wq);
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmul(z[q], wq[q]);
      fft_reg<C, false>(z);
#pragma unroll
      for (int q = 0; q < C; ++q) Bc[q * W + col] = z[q];
    }
    __syncthreads();
    TSF_PACC(sm, PS_COLF);
    // bin pairs: item u = k2 * cp + il; (row k2, col (il,0)) <-> (row C-1-k2, col (il,1)); the
    // multiplier / twiddle table loads of PU items are issued together.  The pseudo column pair
    // pi = 0 (CTA 0, first chunk) is done afterwards, one row per thread.
    constexpr int PU = 1;            // more items per batch spilled the 255-register kernel
    const int nit = C * cp;
    for (int u0 = threadIdx.x; u0 < nit; u0 += PU * kThreads) {
      double2 la[PU], lb[PU], w[PU];
      int ia[PU], ib[PU];
#pragma unroll
      for (int k = 0; k < PU; ++k) {
        const int u = u0 + k * kThreads;
        ia[k] = -1;
        if (u < nit) {
          const int k2 = u / cp, il = u - k2 * cp, i = c0 + il;
          const int pi = int(r) + i * C;
          if (pi != 0) {
            const int bin = pi + L1 * k2;
            if (pre) {
              la[k] = op.conj ? cconj(Ta[u]) : Ta[u];
              lb[k] = op.conj ? cconj(Tb[u]) : Tb[u];
              w[k] = Tw[u];
            } else {
              la[k] = op.get(k2, 0, i, bin);
              lb[k] = op.get(C - 1 - k2, 1, i, g.L - bin);
              w[k] = op.wtw(k2, 0, i, bin, tw, g.tw2L);
            }
            ia[k] = k2 * W + 2 * il;
            ib[k] = (C - 1 - k2) * W + 2 * il + 1;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < PU; ++k) {
        if (ia[k] < 0) continue;
        double2 a = Bc[ia[k]], b = Bc[ib[k]];
        pair_apply(a, b, la[k], lb[k], w[k], op.scale);
        Bc[ia[k]] = a;
        Bc[ib[k]] = b;
      }
    }
    if (r == 0 && c0 == 0 && threadIdx.x < C) {
      const int k2 = threadIdx.x;
      const int kk = (C - k2) % C;
      if (k2 <= C / 2) {                      // column 0: bins L1 k2 <-> L1 (C - k2)
        const int bin = L1 * k2;
        const double2 la = op.get(k2, 0, 0, bin);
        const double2 w = op.wtw(k2, 0, 0, bin, tw, g.tw2L);
        double2 &za = Bc[k2 * W];
        if (kk == k2) {
          double2 a = za;
          pair_self(a, la, k2 == 0 ? op.nyqe : la, w, op.scale);
          za = a;
        } else {
          double2 &zb = Bc[kk * W];
          double2 a = za, b = zb;
          pair_apply(a, b, la, op.get(kk, 0, 0, g.L - bin), w, op.scale);
          za = a;
          zb = b;
        }
      }
      const int km = C - 1 - k2;
      if (k2 < (C + 1) / 2) {                 // column L1/2: bins L1/2 + L1 k2 <-> k2' = C-1-k2
        const int bin = L1 / 2 + L1 * k2;
        const double2 la = op.get(k2, 1, 0, bin);
        const double2 w = op.wtw(k2, 1, 0, bin, tw, g.tw2L);
        double2 &za = Bc[k2 * W + 1];
        if (km == k2) {
          double2 a = za;
          pair_self(a, la, la, w, op.scale);
          za = a;
        } else {
          double2 &zb = Bc[km * W + 1];
          double2 a = za, b = zb;
          pair_apply(a, b, la, op.get(km, 1, 0, g.L - bin), w, op.scale);
          za = a;
          zb = b;
        }
      }
    }
    __syncthreads();
    TSF_PACC(sm, PS_PAIRS);
    for (int col = threadIdx.x; col < 2 * cp; col += kThreads) {   // inverse column DFT_C + push
      const int k1 = col_k1(L1, C, r, 2 * c0 + col);
      double2 z[C];
#pragma unroll
      for (int q = 0; q < C; ++q) z[q] = Bc[q * W + col];
      fft_reg<C, true>(z);
      double2 wq[C];
      col_twiddles<C>(tw[k1 * g.twL], wq);
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmulc(z[q], wq[q]);
      // back into the L2 staging rows, in place: the slots of a column pair are read and written
      // only by the pair's owner (L2 stores run at ~10x the per-SM rate of DSMEM stores)
      const int sl = gslot(g, k1);
#pragma unroll
      for (int q = 0; q < C; ++q) __stcg(xg + q * L1 + sl, z[q]);
    }
    __syncthreads();                            // Bc is refilled by the next chunk
    TSF_PACC(sm, PS_COLI);
  }
}

// ------------------------------------------------------------------------ multi-pass regime
// n > 2^17 (local transforms of L1 = R x S points, S = kMaxLocal, R = 2..8): the CTA's apply
// buffer X = xa + r L1e (global, natural local order) replaces the SMEM buffer A.  Forward
// (m = s + S rho, k1 = rho' + R k):
//   F1  Y[rho'][s] = W_{L1}^{s rho'} sum_rho x[s + S rho] W_R^{rho rho'}   (R-point DFTs, in place)
//   F2  row rho' -> SMEM, S-point DIF FFT, staged into xg at row rho' (slot p holds bin
//       rho' + R dperm(p), gslot), then the chunked column stage of the cluster (cross_chunked);
// inverse: I2 row rho' of xg -> SMEM, S-point DIT FFT, times conj W_{L1}^{s rho'} back into X;
//   I1  inverse R-point DFTs over stride S.  Every element of X is read and written by the same
// thread in F1, F2's copies, I2's stores and I1 (S is a multiple of kThreads), and the vector
// loops touch element e from thread e mod kThreads too, so only SMEM reuse needs barriers.
template <int R, bool INV>
__device__ __forceinline__ void rows_dft(double2 *__restrict__ X, int S, const Smem &sm, int tf) {
  for (int s = threadIdx.x; s < S; s += kThreads) {
    double2 x[R];
    if (!INV) {
#pragma unroll
      for (int q = 0; q < R; ++q) x[q] = X[s + q * S];
      fft_reg<R, false>(x);
#pragma unroll
      for (int q = 0; q < R; ++q) X[q * S + s] = q ? cmul(x[q], twid(sm, s * q * tf)) : x[q];
    } else {
#pragma unroll
      for (int q = 0; q < R; ++q) x[q] = X[q * S + s];
      fft_reg<R, true>(x);
#pragma unroll
      for (int q = 0; q < R; ++q) X[s + q * S] = x[q];
    }
  }
}
template <bool INV>
__device__ __forceinline__ void rows_dft_any(double2 *X, int lr, int S, const Smem &sm, int tf) {
  if (lr == 1) rows_dft<2, INV>(X, S, sm, tf);
  else if (lr == 2) rows_dft<4, INV>(X, S, sm, tf);
  else if (lr == 3) rows_dft<8, INV>(X, S, sm, tf);
}

template <int C>
__device__ __noinline__ double2 *apply_big(const Smem &sm, int L1e, const Geo &g, const SpecOp &op,
                                           const double2 *__restrict__ tw, uint32_t r,
                                           double2 *__restrict__ xg, double2 *__restrict__ xa) {
  TSF_PT0();
  const int L1 = g.L1, R = 1 << g.lr, S = 1 << g.ls;
  const int tf = L1e / L1;                    // W_{L1}^x = W_{L1e}^{x tf}
  double2 *X = xa + int64_t(r) * L1e;
  double2 *xr = xg + int64_t(r) * L1;
  if (R > 1) rows_dft_any<false>(X, g.lr, S, sm, tf);       // F1 (same-thread elements)
  for (int rho = 0; rho < R; ++rho) {                        // F2
    for (int p = threadIdx.x; p < S; p += kThreads) cp_async16(sm.A + pidx(p), X + rho * S + p);
    cp_async_wait_all();
    __syncthreads();
    local_fft<false>(sm.A, S, sm, L1e);
    for (int p = threadIdx.x; p < S; p += kThreads) __stcg(xr + rho * S + p, sm.A[pidx(p)]);
    __syncthreads();                          // A is refilled by the next row
  }
  TSF_PACC(sm, PS_FFT_F);
  csync<C>();                                 // every row of every CTA staged in L2
  TSF_PACC(sm, PS_BAR1);
  cross_chunked<C>(sm.A, sm.B, sm.chunk, g, op, tw, r, sm, xg);
  TSF_PTR();
  csync<C>();                                 // every column result back in L2
  TSF_PACC(sm, PS_BAR3);
  for (int rho = 0; rho < R; ++rho) {                        // I2
    for (int p = threadIdx.x; p < S; p += kThreads) cp_async16(sm.A + pidx(p), xr + rho * S + p);
    cp_async_wait_all();
    __syncthreads();
    local_fft<true>(sm.A, S, sm, L1e);
    for (int s = threadIdx.x; s < S; s += kThreads) {
      const double2 v = sm.A[pidx(s)];
      X[rho * S + s] = rho ? cmulc(v, twid(sm, s * rho * tf)) : v;
    }
    __syncthreads();
  }
  if (R > 1) rows_dft_any<true>(X, g.lr, S, sm, tf);        // I1
  TSF_PACC(sm, PS_FFT_I);
#ifdef TSF_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == TSF_PROF_CTA) sm.prof[PS_APPLIES] += 1;
#endif
  return X;
}

// y = op(x) for the CTA's local data already in A[0..L1) (natural order, visible).
// Returns the buffer that holds this CTA's part of the result (natural order, visible):
// O in the staged mode, A otherwise.  The caller writes the next input into A.
// Inlined at each call site (a __noinline__ variant, -DTSF_APPLY_NOINLINE, shrinks the SASS
// ~5x but measured 20% slower at C3: its arguments travel through the stack).
#ifdef TSF_APPLY_NOINLINE
#define TSF_APPLY_ATTR __noinline__
#else
#define TSF_APPLY_ATTR __forceinline__
#endif
template <int C, bool STG>
__device__ TSF_APPLY_ATTR double2 *apply_smem(const Smem &sm, int L1e, const Geo &g, const SpecOp &op,
                                            const double2 *__restrict__ tw, uint32_t r, Xch &xs,
                                            double2 *xg) {
  TSF_PT0();
  bool pre = false;               // forward FFT already pushed its outputs (staged, compile-time FFT)
  if constexpr (C > 1 && STG) {
#ifndef TSF_NO_CT_FFT
    if (sm.tws != nullptr && L1e == 1024 && (g.L1 == 1024 || g.L1 == 512)) {
      const PushIn<C> pin(sm.B, sm.mbar, g, r);
      if (g.L1 == 1024) local_fft_ct_fwd_out<1024>(sm.A, sm.tws, L1e, pin);
      else local_fft_ct_fwd_out<512>(sm.A, sm.tws, L1e, pin);
      pre = true;
    } else if (sm.tws != nullptr && L1e == 256 && (g.L1 == 256 || g.L1 == 128)) {
      const PushIn<C> pin(sm.B, sm.mbar, g, r);
      if (g.L1 == 256) local_fft_ct_fwd_out<256>(sm.A, sm.tws, L1e, pin);
      else local_fft_ct_fwd_out<128>(sm.A, sm.tws, L1e, pin);
      pre = true;
    }
#endif
  }
  if (!pre) local_fft<false>(sm.A, g.L1, sm, L1e);
  TSF_PACC(sm, PS_FFT_F);
  double2 *Y = sm.A;
  if constexpr (C == 1) {
    pointwise_local(sm.A, g, op, tw);
    __syncthreads();
    TSF_PACC(sm, PS_PAIRS);
  } else {
    if constexpr (STG) {
      cross_push<C>(sm.A, sm.B, sm.O, g, op, tw, r, sm, xs, pre);
      Y = sm.O;
    } else {
      for (int p = threadIdx.x; p < g.L1; p += kThreads) __stcg(xg + int64_t(r) * g.L1 + p, sm.A[pidx(p)]);
      csync<C>();                // every local transform staged in L2 before the gathers
      TSF_PACC(sm, PS_BAR1);
      cross_chunked<C>(sm.A, sm.B, sm.chunk, g, op, tw, r, sm, xg);
      TSF_PTR();
      csync<C>();                // every column result back in L2 before the row reads
      TSF_PACC(sm, PS_BAR3);
      {                          // this CTA's row back from L2 (async copies, all in flight)
        const double2 *xr = xg + int64_t(r) * g.L1;
        for (int p = threadIdx.x; p < g.L1; p += kThreads) cp_async16(sm.A + pidx(p), xr + p);
        cp_async_wait_all();
      }
      __syncthreads();
      TSF_PACC(sm, PS_SCATTER);
    }
    TSF_PTR();
  }
  local_fft<true>(Y, g.L1, sm, L1e);
  TSF_PACC(sm, PS_FFT_I);
#ifdef TSF_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == TSF_PROF_CTA) sm.prof[PS_APPLIES] += 1;
#endif
  return Y;
}

// Operator application: the SMEM four-step (n <= 2^17) or the multi-pass regime (BIG).
template <int C, bool STG, bool BIG = false>
__device__ __forceinline__ double2 *apply(const Smem &sm, int L1e, const Geo &g, const SpecOp &op,
                                         const double2 *__restrict__ tw, uint32_t r, Xch &xs,
                                         double2 *xg = nullptr, double2 *xa = nullptr) {
  if constexpr (BIG) return apply_big<C>(sm, L1e, g, op, tw, r, xg, xa);
  else return apply_smem<C, STG>(sm, L1e, g, op, tw, r, xs, xg);
}

// ------------------------------------------------------------------------ operator setup
enum Which { OP_A = 0, OP_B = 1, OP_AT = 2, OP_PINV = 3, OP_PTINV = 4 };

__device__ __forceinline__ Geo geo_embed(const DevParams &P, const Smem &sm) {
  Geo g;
  g.L1 = P.L1e; g.L = int(P.n); g.np = P.npe; g.twL = P.twN / int(P.n); g.tw2L = P.twN / int(2 * P.n);
  g.slot = P.slot_e;
  g.ctw = sm.ctwe;
  g.l1 = __ffs(g.L1) - 1;
  g.lnp = __ffs(g.np) - 1;
  g.lr = P.lre;
  g.ls = g.l1 - g.lr;
  return g;
}
__device__ __forceinline__ Geo geo_prec(const DevParams &P, const Smem &sm) {
  Geo g;
  g.L1 = P.L1p; g.L = int(P.n / 2); g.np = P.npp; g.twL = P.twN / int(P.n / 2); g.tw2L = P.twN / int(P.n);
  g.slot = P.slot_p;
  g.ctw = sm.ctwp;
  g.l1 = __ffs(g.L1) - 1;
  g.lnp = __ffs(g.np) - 1;
  g.lr = P.lrp;
  g.ls = g.l1 - g.lr;
  return g;
}

// Level-j operator: which in {A, B, A^T} uses the embedding spectrum, {P^-1, P^-T} the
// preconditioner spectrum.  A = eta I - sigma L_j, B = eta I + (1-sigma) L_j (eq3.3), P the
// circulant of (preku) with s(.) replaced by the chosen circulant approximation.
__device__ __forceinline__ SpecOp make_op(const DevParams &P, const Inst &I, int64_t j, int which,
                                          uint32_t r, const Smem &sm) {
  const double *lv = I.lev + 4 * j;
  const double eta = lv[0], c = lv[1], p = lv[2], q = lv[3];
  const double sigma = I.par[0];
  SpecOp op;
  const bool res = sm.mule != nullptr;
  op.rC = int(r) * P.C;
  op.mul_sh = res;
  op.eta = eta;
  op.ppq = p + q;
  op.pmq = p - q;
  if (which <= OP_AT) {
    op.lam = I.lwe;
    op.sq = P.sq_e;
    op.mul = (which == OP_B) ? nullptr : (res ? sm.mule : I.mul);
    op.pw = res ? sm.pwe : nullptr;
    op.np = P.npe; op.nyq = I.lwe[P.n];
    op.mu = (which == OP_B) ? (1.0 - sigma) : -sigma;
    op.c2 = 2.0 * c;
    op.qcorr = 0.0;
    op.scale = P.scale_e;
    op.conj = (which == OP_AT);
    op.div = false;
  } else {
    op.lam = I.lwp;
    op.sq = P.sq_p;
    op.mul = res ? sm.mulp : I.mul + P.n;
    op.pw = res ? sm.pwp : nullptr;
    op.np = P.npp; op.nyq = I.lwp[P.n / 2];
    op.mu = -sigma;
    op.c2 = 2.0 * c * P.qscale_p;
    op.qcorr = P.strang ? -q * I.par[2] : 0.0;   // Strang s(W^T) midpoint fix (R-strang)
    op.scale = P.scale_p;
    op.conj = (which == OP_PTINV);
    op.div = true;
  }
  op.nyqe = op.nyquist(which <= OP_AT ? int(P.n) : int(P.n / 2));
  return op;
}

// Per-level multiplier tables (task order, this CTA's slice): lambda_A of the embedding and
// 1/lambda_P of the preconditioner, formed once per level from the base spectra so the per-bin
// work of every operator application is a single table read (A^T, P^{-T} conjugate it).
// Written to SMEM (resident) or the instance's HBM table; the caller synchronizes.
__device__ __forceinline__ void fill_mul(const DevParams &P, const Inst &I, int64_t j, uint32_t r,
                                         const Smem &sm) {
  const Smem none = {};
  SpecOp a = make_op(P, I, j, OP_A, r, none), pinv = make_op(P, I, j, OP_PINV, r, none);
  const bool res = sm.mule != nullptr;
  const int L1e = P.L1e, L1p = P.L1p, C = P.C;
  // resident (SMEM) tables in the staged column stage's layout: a-side bins (k2a, column (i, 0))
  // at i C + k2a, b-side bins (C-1-k2a, column (i, 1)) at np C + i C + k2a; the HBM tables in
  // task order
  const int lC = __ffs(C) - 1;
  auto slot_task = [&](int u, int np, int &k2, int &ab, int &i) {
    const int lnp = __ffs(np) - 1;
    if (res && C == 16) {
      ab = u >> (lnp + lC);
      const int k2a = u & (C - 1);
      i = (u >> lC) & (np - 1);
      k2 = ab ? C - 1 - k2a : k2a;
    } else {
      i = u & (np - 1); ab = (u >> lnp) & 1; k2 = u >> (lnp + 1);
    }
  };
  for (int u = threadIdx.x; u < L1e; u += kThreads) {
    int k2, ab, i;
    slot_task(u, P.npe, k2, ab, i);
    const double2 v = a.lam_idx(int(task_index(C, P.npe, int(r), k2, ab, i)), 0);
    if (res) sm.mule[u] = v; else I.mul[int64_t(r) * L1e + u] = v;
  }
  if (P.precond == TSF_NOPREC) return;
  const int np = P.npp;
  for (int u = threadIdx.x; u < L1p; u += kThreads) {
    int k2, ab, i;
    slot_task(u, np, k2, ab, i);
    const int bin = int(task_bin(L1p, C, int(r), i, k2, ab));
    const double2 v = pinv.eff(pinv.lam_idx(int(task_index(C, np, int(r), k2, ab, i)), bin));
    if (res) sm.mulp[u] = v; else I.mul[P.n + int64_t(r) * L1p + u] = v;
  }
}

// NEXT-2 (alg1x): product with one triangular Toeplitz factor of the Gohberg-Semencul
// formula through its 2n circulant embedding.  The factor's spectrum table is multiplied raw:
// eta = 0, mu = ppq = pmq = 1, c2 = qcorr = 0 make the Nyquist formula return the stored value
// exactly.  k: 0 = R_p^0, 1 = R_p, 2 = L_p^0, 3 = L_p (tsf_capi.cu k_gsf_cols).
__device__ __forceinline__ SpecOp make_gsf_op(const DevParams &P, const Inst &I, int k, uint32_t r,
                                              const Smem &sm) {
  SpecOp op;
  op.lam = I.lwe;
  op.sq = P.sq_e;
  op.mul = I.gsf + int64_t(k) * (P.n + 1);
  op.mul_sh = false;
  op.pw = sm.mule != nullptr ? sm.pwe : nullptr;
  op.nyq = op.mul[P.n];
  op.np = P.npe;
  op.rC = int(r) * P.C;
  op.eta = 0.0; op.mu = 1.0; op.ppq = 1.0; op.pmq = 1.0; op.c2 = 0.0; op.qcorr = 0.0;
  op.scale = P.scale_e;
  op.conj = false;
  op.div = false;
  op.nyqe = op.nyq;
  return op;
}

// ------------------------------------------------------------------------ apply buffer view
// The operator input/output of this CTA, element e of the local chunk: the swizzled SMEM buffer
// (A, or O in the staged mode), or in the multi-pass regime the global apply buffer (linear).
template <bool BIG>
struct ABuf {
  double2 *p;
  __device__ __forceinline__ double2 &operator[](int e) const {
    if constexpr (BIG) return p[e];
    else return p[pidx(e)];
  }
};
template <bool BIG>
__device__ __forceinline__ ABuf<BIG> abuf_in(const DevParams &P, const Inst &I, const Smem &sm, uint32_t r) {
  if constexpr (BIG) return ABuf<BIG>{I.xa + int64_t(r) * P.L1e};
  else return ABuf<BIG>{sm.A};
}

// ------------------------------------------------------------------------ vector storage
// Krylov vectors of this CTA's chunk (npc = L1p complex values): SMEM slots when the plan
// keeps them on chip (P.vsmem), else the instance's HBM vector block (permuted chunks).
// Every vector loop visits element e = tid + q T, so each element is only ever touched by
// the same thread and vector updates need no barrier.
struct Vecs {
  double2 *U, *X, *R, *RH, *P, *V, *S, *PH, *SH, *G;
};

// VS (compile time) = vectors in SMEM, so every vector access compiles to LDS/STS or LDG/STG
// rather than generic loads.
template <bool VS>
__device__ __forceinline__ Vecs vec_view(const DevParams &P, const Inst &I, const Smem &sm, uint32_t r) {
  Vecs v;
  const int npc = P.L1p;
  auto g = [&](int slot) { return reinterpret_cast<double2 *>(I.vec + slot * P.n) + r * npc; };
  if constexpr (VS) {
    double2 *b = sm.vs;
    v.U = b; v.X = b + npc; v.R = b + 2 * npc; v.RH = b + 3 * npc; v.P = b + 4 * npc;
    v.V = b + 5 * npc; v.S = b + 6 * npc; v.PH = b + 7 * npc; v.SH = b + 8 * npc; v.G = g(V_G);
  } else {
    v.U = g(V_U); v.X = g(V_X); v.R = g(V_R); v.RH = g(V_RH); v.P = g(V_P);
    v.V = g(V_V); v.S = g(V_S); v.PH = g(V_PH); v.SH = g(V_SH); v.G = g(V_G);
  }
  return v;
}

#define TSF_FOR_E(npc) for (int e = threadIdx.x; e < (npc); e += kThreads)

// Element loop in batches of U elements per thread: every load of the batch (ld) is issued
// before any store (op), so HBM-resident vectors get U x (loads per element) requests in flight
// per thread.  Elements are visited in the same per-thread order as TSF_FOR_E, so per-thread
// partial sums (and therefore the reductions) are bit-identical to the unbatched loop.
template <int U, class T, class LD, class OP>
__device__ __forceinline__ void batched(int npc, LD &&ld, OP &&op) {
  for (int e0 = threadIdx.x; e0 < npc; e0 += U * kThreads) {
    T t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kThreads;
      if (e < npc) ld(e, t[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kThreads;
      if (e < npc) op(e, t[u]);
    }
  }
}
struct T1 { double2 a; };
struct T2 { double2 a, b; };
struct T3 { double2 a, b, c; };
struct T5 { double2 a, b, c, d, f; };

// ------------------------------------------------------------------------ RHS (alg1 step 2)
// NEXT-3 blocked history sum (tsf.h hist_block).  Levels J0 = kb .. J0+b-1 form a block.  At the
// block start one pass over the rows d^0..d^{J0-1} (each row read once, HU rows in flight per
// thread) forms for every level of the block
//   HB[q] = kappa e_{J0+q} d^0 + sum_{s=1}^{J0-1} kappa chat_{J0+q-s} d^s        (q < b),
// and level j adds its rows since the block start: Hs = HB[j-J0] + sum_{s=max(1,J0)}^{j-1}
// kappa chat_{j-s} d^s (+ kappa e_j d^0 in block 0, where HB is not used).  Element e is only
// ever touched by thread e mod kThreads (same thread writes HB and reads it later).
template <int QB>
__device__ __forceinline__ void hist_block_pass(const Inst &I, int64_t J0, int64_t M, uint32_t r, int npc,
                                                const double2 *__restrict__ H, double2 *__restrict__ HB,
                                                int64_t hstride) {
  constexpr int HU = 4;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    double2 acc[QB];
    const double2 d0 = H[e];
#pragma unroll
    for (int q = 0; q < QB; ++q) acc[q] = (J0 + q < M) ? cscale(d0, I.hwe[J0 + q]) : zero2();
    int64_t s = 1;
    for (; s + HU - 1 <= J0 - 1; s += HU) {
      double2 v[HU];
#pragma unroll
      for (int u = 0; u < HU; ++u) v[u] = H[(s + u) * hstride + e];
#pragma unroll
      for (int u = 0; u < HU; ++u)
#pragma unroll
        for (int q = 0; q < QB; ++q) acc[q] = caxpy(I.hwc[min(J0 + q - s - u, M - 1)], v[u], acc[q]);
    }
    for (; s <= J0 - 1; ++s) {
      const double2 v = H[s * hstride + e];
#pragma unroll
      for (int q = 0; q < QB; ++q) acc[q] = caxpy(I.hwc[min(J0 + q - s, M - 1)], v, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < QB; ++q) HB[q * hstride + e] = acc[q];
  }
}

__device__ __forceinline__ void hist_blocked(const DevParams &P, const Inst &I, int64_t j, uint32_t r,
                                             const double2 *__restrict__ H, double2 *__restrict__ Hs, int b) {
  const int npc = P.L1p;
  const int64_t hstride = P.n / 2;
  const int64_t J0 = j - j % b;
  double2 *HB = reinterpret_cast<double2 *>(I.hb) + r * npc;
  if (j == J0 && J0 > 0) {
    // the block's partial sums, in sub-blocks of at most 16 levels (register budget)
    for (int q0 = 0; q0 < b; q0 += 16) {
      const int qb = b - q0 < 16 ? b - q0 : 16;
      double2 *dst = HB + q0 * hstride;
      if (qb == 16) hist_block_pass<16>(I, J0 + q0, P.M, r, npc, H, dst, hstride);
      else if (qb == 8) hist_block_pass<8>(I, J0 + q0, P.M, r, npc, H, dst, hstride);
      else if (qb == 4) hist_block_pass<4>(I, J0 + q0, P.M, r, npc, H, dst, hstride);
      else hist_block_pass<2>(I, J0 + q0, P.M, r, npc, H, dst, hstride);
    }
  }
  const int64_t s0 = J0 > 1 ? J0 : 1;
  const double2 *Bj = HB + (j - J0) * hstride;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    double2 a = J0 > 0 ? Bj[e] : cscale(H[e], I.hwe[j]);
    double2 c = zero2();
    int64_t s = s0;
    for (; s + 1 <= j - 1; s += 2) {
      const double2 v0 = H[s * hstride + e], v1 = H[(s + 1) * hstride + e];
      a = caxpy(I.hwc[j - s], v0, a);
      c = caxpy(I.hwc[j - s - 1], v1, c);
    }
    if (s <= j - 1) a = caxpy(I.hwc[j - s], H[s * hstride + e], a);
    Hs[e] = cadd(a, c);
  }
}

// g = B u^j - [kappa e_j d^0 + sum_{s=1}^{j-1} kappa chat_{j-s} d^s] + f^{j+sigma}
// First half: the memory term into Hsum and u^j (zero-padded) into A; the caller applies B.
template <int C, bool BIG>
__device__ __forceinline__ void rhs_pre(const DevParams &P, const Smem &sm, const Inst &I, int64_t j, uint32_t r,
                                        const double2 *U, double2 *Hsum, bool use_pre, int hblock = 0) {
  // (use_pre is dropped below when the helpers do not deliver in time)
  const int npc = P.L1p;
  const int64_t n = P.n;
  TSF_PT0();
  const ABuf<BIG> AX = abuf_in<BIG>(P, I, sm, r);
  const double2 *H = reinterpret_cast<const double2 *>(I.hist) + r * npc;
  const int64_t hstride = n / 2;  // double2 per history row
  // history term kappa (e_j d^0 + sum_{s=1}^{j-1} chat_{j-s} d^s) into Hs (the X slot, zeroed after
  // the RHS anyway): two elements per thread and HU rows per batch, all loads of a batch issued
  // before the FMAs (HU x 2 loads in flight per thread; the sum streams j rows of the CTA chunk)
  double2 *Hs = Hsum;
  if (use_pre) {
    // history pre-sum P^j = kappa (e_j d^0 + sum_{s=1}^{j-2} chat_{j-s} d^s) from the helper CTAs
    // (computed during level j-1); bounded wait, else this CTA sums its slice itself below
    if (threadIdx.x == 0) {
      int ok = 0;
      if (ld_acquire(P.sync + 5) == 0) {
        const uint64_t t0 = gtimer_ns();
        for (;;) {
          if (ld_acquire(P.sync + 1 + (j & 1)) == j) { ok = 1; break; }
          if (gtimer_ns() - t0 > kHelperWaitNs) { st_release(P.sync + 5, 1); break; }
          __nanosleep(64);
        }
      }
      *sm.flag = ok;
    }
    __syncthreads();
    use_pre = *sm.flag != 0;
    __syncthreads();              // the flag word is reused
  }
  if (use_pre) {
    const double2 *Pj = reinterpret_cast<const double2 *>(P.pre) + (j & 1) * hstride + r * npc;
    const double w1 = I.hwc[1];
    TSF_FOR_E(npc) { Hs[e] = caxpy(w1, H[(j - 1) * hstride + e], __ldcg(Pj + e)); }
  } else if (j >= 1 && hblock > 0) {
    hist_blocked(P, I, j, r, H, Hs, hblock);
  } else if (j >= 1) {
    // the same summation order as the helpers (P^j over rows 1..j-2 with HU-row batches and two
    // accumulators, then + chat_1 d^{j-1}), so step-wise and helper-assisted runs agree bitwise;
    // two elements per thread, all loads of a batch issued before the FMAs
    constexpr int HU = C == 1 ? 4 : 8;
    const double w1 = I.hwc[1];
    for (int e0 = threadIdx.x; e0 < npc; e0 += 2 * kThreads) {
      const int e1 = e0 + kThreads;
      const bool has1 = e1 < npc;
      const double wj = I.hwe[j];
      double2 a0 = cscale(H[e0], wj), a1 = has1 ? cscale(H[e1], wj) : zero2();
      double2 b0 = zero2(), b1 = zero2();
      int64_t s = 1;
      for (; s + HU - 1 <= j - 2; s += HU) {
        double2 v0[HU], v1[HU];
        double w[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
          v0[u] = H[(s + u) * hstride + e0];
          v1[u] = has1 ? H[(s + u) * hstride + e1] : zero2();
          w[u] = I.hwc[j - s - u];
        }
#pragma unroll
        for (int u = 0; u < HU; u += 2) {
          a0 = caxpy(w[u], v0[u], a0);
          a1 = caxpy(w[u], v1[u], a1);
          b0 = caxpy(w[u + 1], v0[u + 1], b0);
          b1 = caxpy(w[u + 1], v1[u + 1], b1);
        }
      }
      for (; s <= j - 2; ++s) {
        const double w = I.hwc[j - s];
        a0 = caxpy(w, H[s * hstride + e0], a0);
        if (has1) a1 = caxpy(w, H[s * hstride + e1], a1);
      }
      if (j >= 2) {
        Hs[e0] = caxpy(w1, H[(j - 1) * hstride + e0], cadd(a0, b0));
        if (has1) Hs[e1] = caxpy(w1, H[(j - 1) * hstride + e1], cadd(a1, b1));
      } else {
        Hs[e0] = a0;
        if (has1) Hs[e1] = a1;
      }
    }
  }
  TSF_PACC(sm, PS_RHS_HIST);
  TSF_FOR_E(npc) {
    AX[e] = U[e];
    AX[e + npc] = zero2();
  }
}

// Second half of the RHS: g = Y - Hs + f from the product Y = B u^j; g into A[0..npc)
// (A[npc..2npc) zero).  Returns the local partial ||g||^2.
template <bool BIG>
__device__ __forceinline__ double rhs_post(const DevParams &P, const Smem &sm, const Inst &I, int64_t j,
                                           uint32_t r, const ABuf<BIG> Y, const double2 *Hs) {
  const ABuf<BIG> AX = abuf_in<BIG>(P, I, sm, r);
  const int npc = P.L1p;
  const int64_t n = P.n, hstride = n / 2;
  const int C = P.C;
  double acc = 0.0;
  TSF_FOR_E(npc) {
    double2 g = Y[e];
    if (j >= 1) g = csub(g, Hs[e]);
    if (P.src_kind == TSF_SRC_SEPARABLE) {
      const double2 *Bs = reinterpret_cast<const double2 *>(I.basis) + r * npc;
      for (int k = 0; k < P.K; ++k) g = caxpy(I.scal[j * P.K + k], Bs[k * hstride + e], g);
    } else if (P.src_kind == TSF_SRC_TABLE) {
      if (I.fdev) {          // borrowed natural-order table: packed value m = C e + r
        const double2 *F = reinterpret_cast<const double2 *>(I.fdev + j * n);
        g = cadd(g, __ldg(F + int64_t(e) * C + r));
      } else {
        const double2 *F = reinterpret_cast<const double2 *>(I.ftab) + r * npc;
        g = cadd(g, F[j * hstride + e]);
      }
    }
    AX[e] = g;
    AX[e + npc] = zero2();
    acc += cdot(g, g);
  }
  return acc;
}

// Whole RHS (debug hook): history, B u^j, g.
template <int C, bool STG, bool BIG>
__device__ __forceinline__ double rhs_phase(const DevParams &P, const Smem &sm, const Inst &I, const Geo &ge,
                                            const SpecOp &opB, int64_t j, uint32_t r, const double2 *U,
                                            double2 *Hsum, Xch &xs) {
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  rhs_pre<C, BIG>(P, sm, I, j, r, U, Hsum, false);
  __syncthreads();
  const ABuf<BIG> Y{apply<C, STG, BIG>(sm, P.L1e, ge, opB, tw, r, xs, I.xg, I.xa)};
  return rhs_post<BIG>(P, sm, I, j, r, Y, Hsum);
}

// ------------------------------------------------------------------------ one level
// All control flow is uniform over the cluster (every CTA reduces to identical scalars).
// NEXT-2, alg2 for j >= 1 with constant coefficients: u^{j+1} = A^{-1} g^{j+1} by the
// Gohberg-Semencul formula and alg1x:
//   z1 = R_p^0 g, z2 = R_p g, z3 = L_p^0 z1, z4 = L_p z2, u = (z4 - z3) / xi_0,
// each factor applied through its 2n circulant embedding (four fused FFT applications), then
// the true residual ||A u - g|| / ||g|| (one more application) is stored as the level's relres.
// g arrives in A[0..npc) (rhs_phase) with ||g||^2 local partial g2loc.
template <int C, bool STG, bool BIG>
__device__ __forceinline__ void gsf_level(const DevParams &P, const Inst &I, const Smem &sm, const Vecs &V,
                                          int64_t j, uint32_t r, Xch &xs, double g2loc) {
  const int npc = P.L1p;
  const int64_t n = P.n;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  const Geo ge = geo_embed(P, sm);
  double2 *G = V.R, *Z1 = V.S, *Z2 = V.PH, *X = V.X;
  const ABuf<BIG> AX = abuf_in<BIG>(P, I, sm, r);
  ABuf<BIG> Y = AX;
  TSF_FOR_E(npc) { G[e] = AX[e]; }
  double g2[1] = {g2loc};
  csum<C, 1>(g2, sm, xs);
  const double inv_xi0 = I.par[7];
  // z1 = R_p^0 g, z2 = R_p g
  for (int k = 0; k < 2; ++k) {
    TSF_FOR_E(npc) {
      AX[e] = G[e];
      AX[e + npc] = zero2();
    }
    __syncthreads();
    const SpecOp op = make_gsf_op(P, I, k, r, sm);
    Y.p = apply<C, STG, BIG>(sm, P.L1e, ge, op, tw, r, xs, I.xg, I.xa);
    double2 *Z = k == 0 ? Z1 : Z2;
    TSF_FOR_E(npc) { Z[e] = Y[e]; }
  }
  // z3 = L_p^0 z1 (kept in X), z4 = L_p z2, u = (z4 - z3) / xi_0
  for (int k = 2; k < 4; ++k) {
    const double2 *Z = k == 2 ? Z1 : Z2;
    TSF_FOR_E(npc) {
      AX[e] = Z[e];
      AX[e + npc] = zero2();
    }
    __syncthreads();
    const SpecOp op = make_gsf_op(P, I, k, r, sm);
    Y.p = apply<C, STG, BIG>(sm, P.L1e, ge, op, tw, r, xs, I.xg, I.xa);
    if (k == 2) {
      TSF_FOR_E(npc) { X[e] = Y[e]; }
    } else {
      TSF_FOR_E(npc) { X[e] = cscale(csub(Y[e], X[e]), inv_xi0); }
    }
  }
  // true residual of the level: ||A u - g|| / ||g||
  TSF_FOR_E(npc) {
    AX[e] = X[e];
    AX[e + npc] = zero2();
  }
  __syncthreads();
  const SpecOp opA = make_op(P, I, j, OP_A, r, sm);
  Y.p = apply<C, STG, BIG>(sm, P.L1e, ge, opA, tw, r, xs, I.xg, I.xa);
  double rs[1] = {0.0};
  TSF_FOR_E(npc) {
    const double2 d = csub(Y[e], G[e]);
    rs[0] += cdot(d, d);
  }
  csum<C, 1>(rs, sm, xs);
  const double relres = g2[0] > 0.0 ? sqrt(rs[0] / g2[0]) : 0.0;
  // finalize as the Krylov levels: d^j = u^{j+1} - u^j, u^j <- u^{j+1}
  double2 *Hj = reinterpret_cast<double2 *>(I.hist + j * n) + r * npc;
  TSF_FOR_E(npc) {
    const double2 x = X[e], u = V.U[e];
    Hj[e] = csub(x, u);
    V.U[e] = x;
  }
  if (r == 0 && threadIdx.x == 0) {
    I.it[j] = 0;
    I.rr[j] = relres;
    I.trr[j] = relres;
    I.st[j] = isfinite(relres) ? TSF_LEVEL_OK : TSF_LEVEL_DIVERGED;
  }
  __syncthreads();
  if (P.helpers > 0 && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(reinterpret_cast<unsigned long long *>(P.sync), 1ull);
  }
}

// Views (carve-up, instance, vectors) are computed by every thread from the kernel's own
// pointers, so the compiler keeps SMEM accesses as LDS/STS (a view copied through shared memory
// turned them into generic LD/ST and was measured slower).
// mode 0: level j of the scheme.  mode 1 / 2 (NEXT-2 setup, TSF_GSF): solve A x = e_1 / A y = e_n
// (eq3.4) with the level-j operators and store the solution in V_GX / V_GY; no RHS,
// history or statistics.
//
// Code shape: exactly two inlined operator applications per level, as measured fastest: the
// Krylov loop's single site (every quarter step selects its operator) and one "cold" site shared
// by the once-per-level products: S_RHS (B u^j), S_WARM (A u^j, warm start), S_TRUE
// (A u^{j+1}, true residual).  Each inlined site adds the whole fused transform (~8k
// instructions); a separate site per cold product, or an out-of-line copy, measured slower, and
// a single state machine for everything cost ~6% at C3 against this shape.
enum LevelState { S_RHS = 0, S_WARM = 1, S_TRUE = 2, S_KRYLOV = 3 };

// ------------------------------------------------------------------------ fused BiCGSTAB (C3 shape)
// For the C3 geometry (C = 16 CTAs, local lengths L1e = 1024 / L1p = 512, staged exchange,
// resident twiddles) the first forward and the last inverse radix stage of every application
// touch exactly the elements e = tid, tid + 256 that thread tid owns in the vector loops.  The
// BiCGSTAB vector updates therefore ride on those stages: the update that produces an
// application's input feeds its first stage from registers, the last stage of P^{-1} feeds the
// first stage of A directly (phat / shat are only stored for the x update), and the last stage
// of A yields v / t with their dot products.  Same arithmetic and summation order as the
// unfused loop (R-fuse); one barrier and one shared-memory round trip fewer per stage boundary.
namespace fz {
constexpr int kH = kThreads;        // e = b and b + kH (npc = 512)
// P^{-1} forward, first stage (radix 2, L = 512, twiddle W_512^b = tws[341 + b]); twd below is sm.tws
__device__ __forceinline__ void p_first(double2 *A, int b, double2 a0, double2 a1, const double2 *twd) {
  A[pidx(b)] = cadd(a0, a1);
  A[pidx(b + kH)] = cmul(csub(a0, a1), twd[341 + b]);   // tws: W_512^b
}
// A forward, first stage (radix 4, m = 1024) on the zero-padded input (a2 = a3 = 0)
__device__ __forceinline__ void a_first(double2 *A, int b, double2 a0, double2 a1, const double2 *twd) {
  double2 a2 = zero2(), a3 = zero2();
  const double2 w1 = twd[b];
  const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
  bfly4<false>(a0, a1, a2, a3);
  a1 = cmul(a1, w1); a2 = cmul(a2, w2); a3 = cmul(a3, w3);
  A[pidx(b)] = a0; A[pidx(b + kH)] = a1; A[pidx(b + 2 * kH)] = a2; A[pidx(b + 3 * kH)] = a3;
}
// P^{-1} inverse, last stage (radix 2): elements b, b + 256
__device__ __forceinline__ void p_last(const double2 *O, int b, const double2 *twd, double2 &o0, double2 &o1) {
  const double2 a0 = O[pidx(b)];
  const double2 a1 = cmulc(O[pidx(b + kH)], twd[341 + b]);
  o0 = cadd(a0, a1);
  o1 = csub(a0, a1);
}
// A inverse, last stage (radix 4, m = 1024): the kept (unpadded) elements b, b + 256
__device__ __forceinline__ void a_last(const double2 *O, int b, const double2 *twd, double2 &o0, double2 &o1) {
  double2 a0 = O[pidx(b)], a1 = O[pidx(b + kH)], a2 = O[pidx(b + 2 * kH)], a3 = O[pidx(b + 3 * kH)];
  const double2 w1 = twd[b];
  const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
  a1 = cmulc(a1, w1); a2 = cmulc(a2, w2); a3 = cmulc(a3, w3);
  bfly4<true>(a0, a1, a2, a3);
  o0 = a0;
  o1 = a1;
}
}  // namespace fz

// One operator application after its first forward stage (caller: stage written, then barrier):
// the remaining forward stages with the push-in fused into the last, the column stage, and the
// inverse stages but the last (its caller does it).
template <int C, int L>
__device__ __forceinline__ void apply_mid(const Smem &sm, const Geo &g, const SpecOp &op,
                                          const double2 *__restrict__ tw, uint32_t r, Xch &xs) {
  TSF_PT0();
  const PushIn<C> pin(sm.B, sm.mbar, g, r);
  Ct4Top<L, 4>::run(sm.A, sm.tws, 1024);
  last_stage_out<L>(sm.A, pin);
  TSF_PACC(sm, PS_FFT_F);
  cross_push<C>(sm.A, sm.B, sm.O, g, op, tw, r, sm, xs, true);
  TSF_PTR();
  Ct4<true, L, 4>::run(sm.O, sm.tws, 1024);
  TSF_PACC(sm, PS_FFT_I);
#ifdef TSF_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == TSF_PROF_CTA) sm.prof[PS_APPLIES] += 1;
#endif
}

// The BiCGSTAB iterations of level_solve (default variant: x0 given by R/PV/RH/X, four reductions
// merged to three: ||s||^2 travels with t.s and t.t, the half-step exit test follows them).
// Half iteration hh = 0 (p -> phat -> v) and hh = 1 (s -> shat -> t) share ONE site of each
// application (instruction-cache footprint); their vector work is dispatched on hh.
template <int C>
__device__ __forceinline__ void bicg_fused(const DevParams &P, const Smem &sm, const Vecs &V, const Geo &ge,
                                           const Geo &gp, const SpecOp &opA, const SpecOp &opP,
                                           const double2 *__restrict__ tw, uint32_t r, Xch &xs, double rr0,
                                           double rn0, int &hs, double &relres, int &status) {
  using namespace fz;
  double2 *__restrict__ X = V.X, *__restrict__ R = V.R, *__restrict__ RH = V.RH, *__restrict__ PV = V.P;
  double2 *__restrict__ VV = V.V, *__restrict__ S = V.S, *__restrict__ PH = V.PH, *__restrict__ SH = V.SH;
  const double2 *twd = sm.tws;
  double2 *A = sm.A, *O = sm.O;
  const int b = threadIdx.x, b1 = threadIdx.x + kH;
  double rho = rr0, alpha = 0.0, omega = 0.0, beta = 0.0, ssp = 0.0;
  double2 v0 = zero2(), v1 = zero2();
  bool first = true;
  for (;;) {
#pragma unroll 1
    for (int hh = 0; hh < 2; ++hh) {
      TSF_PT0();
      double2 i0, i1;             // input of P^{-1}: p (first iteration: r0) or s = r - alpha v
      if (hh == 0) {
        if (first) {
          i0 = PV[b]; i1 = PV[b1];
        } else {
          i0 = caxpy(beta, caxpy(-omega, VV[b], PV[b]), R[b]);
          i1 = caxpy(beta, caxpy(-omega, VV[b1], PV[b1]), R[b1]);
          PV[b] = i0; PV[b1] = i1;
        }
      } else {
        i0 = caxpy(-alpha, v0, R[b]);
        i1 = caxpy(-alpha, v1, R[b1]);
        S[b] = i0; S[b1] = i1;
        ssp = 0.0;
        ssp += cdot(i0, i0);
        ssp += cdot(i1, i1);
      }
      __syncthreads();            // every thread done with A / O of the last application
      p_first(A, b, i0, i1, twd);
      TSF_PACC(sm, PS_VEC);
      __syncthreads();
      apply_mid<C, 512>(sm, gp, opP, tw, r, xs);
      TSF_PTR();
      {                           // phat / shat, and the first stage of A on it
        double2 o0, o1;
        p_last(O, b, twd, o0, o1);
        double2 *H = hh == 0 ? PH : SH;
        H[b] = o0; H[b1] = o1;
        a_first(A, b, o0, o1, twd);
      }
      TSF_PACC(sm, PS_VEC);
      __syncthreads();
      apply_mid<C, 1024>(sm, ge, opA, tw, r, xs);
      TSF_PTR();
      double2 y0, y1;
      a_last(O, b, twd, y0, y1);
      if (hh == 0) {              // v; alpha = rho / (r^.v)
        v0 = y0; v1 = y1;
        VV[b] = y0; VV[b1] = y1;
        double d[1] = {0.0};
        d[0] += cdot(RH[b], y0);
        d[0] += cdot(RH[b1], y1);
        TSF_PACC(sm, PS_VEC);
        csum<C, 1>(d, sm, xs);
        if (!(fabs(d[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; return; }
        alpha = rho / d[0];
        continue;
      }
      // t: omega = t.s / t.t (with ||s||^2 in the same reduction); x, r updates
      double tt[3] = {0.0, 0.0, ssp};
      const double2 s0 = S[b], s1 = S[b1];
      tt[0] += cdot(y0, s0);
      tt[1] += cdot(y0, y0);
      tt[0] += cdot(y1, s1);
      tt[1] += cdot(y1, y1);
      TSF_PACC(sm, PS_VEC);
      csum<C, 3>(tt, sm, xs);
      TSF_PTR();
      if (sqrt(tt[2]) < P.tol * rn0) {        // half-step exit on ||s||
        X[b] = caxpy(alpha, PH[b], X[b]);
        X[b1] = caxpy(alpha, PH[b1], X[b1]);
        hs += 1;
        relres = sqrt(tt[2]) / rn0;
        return;
      }
      if (!(tt[1] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; return; }
      omega = tt[0] / tt[1];
      double rr[2] = {0.0, 0.0};
      X[b] = caxpy(omega, SH[b], caxpy(alpha, PH[b], X[b]));
      const double2 r0 = caxpy(-omega, y0, s0);
      R[b] = r0;
      rr[0] += cdot(RH[b], r0);
      rr[1] += cdot(r0, r0);
      X[b1] = caxpy(omega, SH[b1], caxpy(alpha, PH[b1], X[b1]));
      const double2 r1 = caxpy(-omega, y1, s1);
      R[b1] = r1;
      rr[0] += cdot(RH[b1], r1);
      rr[1] += cdot(r1, r1);
      TSF_PACC(sm, PS_VEC);
      csum<C, 2>(rr, sm, xs);
      hs += 2;
      relres = sqrt(rr[1]) / rn0;
      if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; return; }
      if (relres < P.tol) return;
      if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; return; }
      if (!(fabs(rr[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; return; }
      beta = (rr[0] / rho) * (alpha / omega);
      rho = rr[0];
      first = false;
    }
  }
}

template <int C, int METHOD, bool STG, bool BIG>
__device__ __forceinline__ void level_solve(const DevParams &P, const Inst &I, const Smem &sm, const Vecs &V,
                                            int64_t j, uint32_t r, Xch &xs, int mode = 0, int64_t j0 = 0) {
  const int npc = P.L1p;
  const int64_t n = P.n;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  const bool prec = P.precond != TSF_NOPREC;
  const Geo ge = geo_embed(P, sm), gp = geo_prec(P, sm);
  fill_mul(P, I, j, r, sm);      // visible after the first barrier below
  const SpecOp opA = make_op(P, I, j, OP_A, r, sm);
  const SpecOp opP = make_op(P, I, j, OP_PINV, r, sm);
  double2 *__restrict__ X = V.X, *__restrict__ R = V.R, *__restrict__ RH = V.RH, *__restrict__ PV = V.P;
  double2 *__restrict__ VV = V.V, *__restrict__ S = V.S, *__restrict__ PH = V.PH, *__restrict__ SH = V.SH;
  double2 *__restrict__ G = V.G;
#ifdef TSF_PROFILE
  const long long tlev0 = clock64();
#endif
  const bool warm = P.x0_warm && mode == 0;
  const bool tres = P.true_res && mode == 0;
  int hs = 0, status = TSF_LEVEL_OK;
  double relres = 0.0, gg = 0.0, rr0 = 0.0;
  const ABuf<BIG> AX = abuf_in<BIG>(P, I, sm, r);   // operator input of this CTA
  ABuf<BIG> Y = AX;              // output buffer of the last operator application

  double g2[1] = {0.0};
  int ph;
  if (mode == 0) {
    rhs_pre<C, BIG>(P, sm, I, j, r, V.U, V.X, P.helpers > 0 && j >= 2 && j >= j0 + 1, P.hblock);
    ph = S_RHS;
  } else {
    // e_1: packed z_0 = (1, 0) on CTA 0; e_n: z_{n/2-1} = (0, 1) on CTA (n/2-1) mod C
    const int64_t m = mode == 1 ? 0 : n / 2 - 1;
    TSF_FOR_E(npc) {
      const bool hit = (int64_t(r) == m % C) && (int64_t(e) == m / C);
      const double2 g = hit ? (mode == 1 ? make_double2(1.0, 0.0) : make_double2(0.0, 1.0)) : zero2();
      AX[e] = g;
      AX[e + npc] = zero2();
      R[e] = g;
      G[e] = g;
      if (METHOD == TSF_BICGSTAB || METHOD == TSF_GSF) { RH[e] = g; PV[e] = g; }
      if (METHOD == TSF_PCGS) RH[e] = g;
      X[e] = zero2();
      g2[0] += cdot(g, g);
    }
    csum<C, 1>(g2, sm, xs);
    gg = rr0 = g2[0];
    ph = S_KRYLOV;
  }

  for (;;) {
    if (ph != S_KRYLOV) {
      // ---- the cold application site: B u^j, A u^j (warm start) or A u^{j+1} (true residual)
      {
        const SpecOp op = ph == S_RHS ? make_op(P, I, j, OP_B, r, sm) : opA;
        __syncthreads();
        Y.p = apply<C, STG, BIG>(sm, P.L1e, ge, op, tw, r, xs, I.xg, I.xa);
      }
      if (ph == S_TRUE) {
        // true residual at exit (SURVEY reading c13): ||g - A u^{j+1}|| / ||g||
        double tr[1] = {0.0};
        TSF_FOR_E(npc) {
          const double2 d = csub(G[e], Y[e]);
          tr[0] += cdot(d, d);
        }
        csum<C, 1>(tr, sm, xs);
        if (r == 0 && threadIdx.x == 0) I.trr[j] = gg > 0.0 ? sqrt(tr[0] / gg) : 0.0;
        break;
      }
      if (ph == S_RHS) {
        g2[0] = rhs_post<BIG>(P, sm, I, j, r, Y, V.X);
        if constexpr (METHOD == TSF_GSF) {
          if (j >= 1) {          // NEXT-2: the level by the Gohberg-Semencul formula
            gsf_level<C, STG, BIG>(P, I, sm, V, j, r, xs, g2[0]);
            return;
          }
        }
        if (warm) {
          // NEXT-3 warm start x0 = u^j: r0 = g - A u^j, stop on ||r|| < tol ||g||
          TSF_FOR_E(npc) {
            G[e] = AX[e];
            AX[e] = V.U[e];
            AX[e + npc] = zero2();
          }
          ph = S_WARM;
          continue;
        }
        TSF_FOR_E(npc) {
          const double2 g = AX[e];
          R[e] = g;
          G[e] = g;
          if (METHOD == TSF_BICGSTAB || METHOD == TSF_GSF) { RH[e] = g; PV[e] = g; }
          if (METHOD == TSF_PCGS) RH[e] = g;
          X[e] = zero2();
        }
        csum<C, 1>(g2, sm, xs);
        gg = rr0 = g2[0];
      } else {                   // S_WARM
        double w2[2] = {g2[0], 0.0};
        TSF_FOR_E(npc) {
          const double2 r0 = csub(G[e], Y[e]);
          R[e] = r0;
          if (METHOD == TSF_BICGSTAB || METHOD == TSF_GSF) { RH[e] = r0; PV[e] = r0; }
          if (METHOD == TSF_PCGS) RH[e] = r0;
          X[e] = V.U[e];
          w2[1] += cdot(r0, r0);
        }
        __syncthreads();         // Y may alias A
        TSF_FOR_E(npc) {
          AX[e] = R[e];
          AX[e + npc] = zero2();
        }
        csum<C, 2>(w2, sm, xs);
        gg = w2[0];
        rr0 = w2[1];
      }
    }
    // ---- Krylov solve from r_0 (in R and A), ||r_0||^2 = rr0, stop on ||r|| < tol ||g||
    const double rn0 = sqrt(gg);
    relres = rn0 > 0.0 ? sqrt(rr0) / rn0 : 0.0;
    const bool iterate = rr0 > 0.0 && !(warm && sqrt(rr0) < P.tol * rn0);

    bool fused = false;
    if constexpr (METHOD == TSF_BICGSTAB && C == 16 && STG && !BIG) {
      if (iterate && P.fuse && prec && !P.pipelined && sm.tws != nullptr && sm.vs != nullptr &&
          P.L1e == 1024 && P.L1p == 512) {
        bicg_fused<C>(P, sm, V, ge, gp, opA, opP, tw, r, xs, rr0, rn0, hs, relres, status);
        fused = true;
      }
    }
    if (!fused && iterate && (METHOD == TSF_BICGSTAB || METHOD == TSF_GSF)) {
      // One BiCGSTAB iteration = four operator applications, h = 0..3: phat = P^{-1} p,
      // v = A phat, shat = P^{-1} s, t = A shat.  They go through ONE inlined apply (the operator
      // and geometry are selected per h) so the hot loop's code stays small for the instruction
      // cache; the vector work before/after each application is dispatched on h.
      double rho = rr0, alpha = 0.0, omega = 0.0, beta = 0.0, ss_est = 0.0;
      for (int h = 0;; h = (h + 1) & 3) {
        const bool isP = !(h & 1);
        if (isP && !prec) {
          Y = AX;
        } else {
          __syncthreads();
          const SpecOp op = isP ? opP : opA;
          const Geo g = isP ? gp : ge;
          Y.p = apply<C, STG, BIG>(sm, P.L1e, g, op, tw, r, xs, I.xg, I.xa);
        }
        if (isP) {
          // h = 0: phat = Y; h = 2: shat = Y.  Either becomes the (padded) input of A.
          double2 *const Dst = h == 0 ? PH : SH;
          TSF_FOR_E(npc) {
            const double2 z = Y[e];
            Dst[e] = z;
            AX[e] = z;
            AX[e + npc] = zero2();
          }
          continue;
        }
        if (h == 1 && P.pipelined) {
          // NEXT-3 (two reductions per iteration): r^.v, r.v, v.v, r.r in one cluster sum;
          // ||s||^2 = ||r||^2 - 2 alpha r.v + alpha^2 v.v (exact reduction if it cancels)
          double d[4] = {0.0, 0.0, 0.0, 0.0};
          TSF_FOR_E(npc) {
            const double2 v = Y[e], rv = R[e];
            VV[e] = v;
            d[0] += cdot(RH[e], v);
            d[1] += cdot(rv, v);
            d[2] += cdot(v, v);
            d[3] += cdot(rv, rv);
          }
          csum<C, 4>(d, sm, xs);
          if (!(fabs(d[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
          alpha = rho / d[0];
          ss_est = d[3] - 2.0 * alpha * d[1] + alpha * alpha * d[2];
          const bool exact = !(ss_est > 1e-10 * d[3]);
          double ss[1] = {0.0};
          if (!exact && sqrt(ss_est) < P.tol * rn0) {
            TSF_FOR_E(npc) { X[e] = caxpy(alpha, PH[e], X[e]); }
            hs += 1;
            relres = sqrt(ss_est) / rn0;
            break;
          }
          TSF_FOR_E(npc) {
            const double2 sv = caxpy(-alpha, VV[e], R[e]);
            S[e] = sv;
            AX[e] = sv;
            if (exact) ss[0] += cdot(sv, sv);
          }
          if (exact) {
            csum<C, 1>(ss, sm, xs);
            ss_est = ss[0];
            if (sqrt(ss[0]) < P.tol * rn0) {
              TSF_FOR_E(npc) { X[e] = caxpy(alpha, PH[e], X[e]); }
              hs += 1;
              relres = sqrt(ss[0]) / rn0;
              break;
            }
          }
          continue;
        }
        if (h == 3 && P.pipelined) {
          // t.s, t.t, r^.s, r^.t in one cluster sum; omega; ||r'||^2 and rho' = r^.r' by
          // expansion; then x, r and the next p in one pass
          double tt[4] = {0.0, 0.0, 0.0, 0.0};
          TSF_FOR_E(npc) {
            const double2 t = Y[e], sv = S[e], rh = RH[e];
            tt[0] += cdot(t, sv);
            tt[1] += cdot(t, t);
            tt[2] += cdot(rh, sv);
            tt[3] += cdot(rh, t);
          }
          csum<C, 4>(tt, sm, xs);
          if (!(tt[1] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
          omega = tt[0] / tt[1];
          double rn2 = ss_est - 2.0 * omega * tt[0] + omega * omega * tt[1];
          const double rho_n = tt[2] - omega * tt[3];
          hs += 2;
          bool exact = !(rn2 > 1e-10 * ss_est);
          bool done = false;
          if (!exact) {
            relres = sqrt(rn2) / rn0;
            if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
            done = relres < P.tol || hs >= 2 * P.maxit || !(fabs(rho_n) > 1e-300);
          }
          if (!exact && !done) {
            beta = (rho_n / rho) * (alpha / omega);
            rho = rho_n;
            TSF_FOR_E(npc) {
              X[e] = caxpy(omega, SH[e], caxpy(alpha, PH[e], X[e]));
              const double2 rn = caxpy(-omega, Y[e], S[e]);
              R[e] = rn;
              const double2 pv = caxpy(beta, caxpy(-omega, VV[e], PV[e]), rn);
              PV[e] = pv;
              AX[e] = pv;
            }
            continue;
          }
          // convergence, a limit, or a cancelled expansion: the plain update with exact norms
          double rr[2] = {0.0, 0.0};
          TSF_FOR_E(npc) {
            X[e] = caxpy(omega, SH[e], caxpy(alpha, PH[e], X[e]));
            const double2 rn = caxpy(-omega, Y[e], S[e]);
            R[e] = rn;
            rr[0] += cdot(RH[e], rn);
            rr[1] += cdot(rn, rn);
          }
          csum<C, 2>(rr, sm, xs);
          relres = sqrt(rr[1]) / rn0;
          if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
          if (relres < P.tol) break;
          if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
          if (!(fabs(rr[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
          beta = (rr[0] / rho) * (alpha / omega);
          rho = rr[0];
          TSF_FOR_E(npc) {
            const double2 pv = caxpy(beta, caxpy(-omega, VV[e], PV[e]), R[e]);
            PV[e] = pv;
            AX[e] = pv;
          }
          continue;
        }
        if (h == 1) {
          // v = Y; alpha = rho / (r^.v); s = r - alpha v; half-step exit on ||s||
          double d[1] = {0.0};
          TSF_FOR_E(npc) {
            const double2 v = Y[e];
            VV[e] = v;
            d[0] += cdot(RH[e], v);
          }
          csum<C, 1>(d, sm, xs);
          if (!(fabs(d[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
          alpha = rho / d[0];
          double ss[1] = {0.0};
          TSF_FOR_E(npc) {
            const double2 sv = caxpy(-alpha, VV[e], R[e]);
            S[e] = sv;
            AX[e] = sv;
            ss[0] += cdot(sv, sv);
          }
          csum<C, 1>(ss, sm, xs);
          if (sqrt(ss[0]) < P.tol * rn0) {
            TSF_FOR_E(npc) { X[e] = caxpy(alpha, PH[e], X[e]); }
            hs += 1;
            relres = sqrt(ss[0]) / rn0;
            break;
          }
          continue;
        }
        // h == 3: t = Y; omega = t.s / t.t; x += alpha phat + omega shat; r = s - omega t
        double tt[2] = {0.0, 0.0};
        TSF_FOR_E(npc) {
          const double2 t = Y[e];
          const double2 sv = S[e];
          tt[0] += cdot(t, sv);
          tt[1] += cdot(t, t);
        }
        csum<C, 2>(tt, sm, xs);
        if (!(tt[1] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
        omega = tt[0] / tt[1];
        double rr[2] = {0.0, 0.0};
        TSF_FOR_E(npc) {
          X[e] = caxpy(omega, SH[e], caxpy(alpha, PH[e], X[e]));
          const double2 rn = caxpy(-omega, Y[e], S[e]);
          R[e] = rn;
          rr[0] += cdot(RH[e], rn);
          rr[1] += cdot(rn, rn);
        }
        csum<C, 2>(rr, sm, xs);
        hs += 2;
        relres = sqrt(rr[1]) / rn0;
        if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
        if (relres < P.tol) break;
        if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
        if (!(fabs(rr[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
        beta = (rr[0] / rho) * (alpha / omega);
        rho = rr[0];
        // next p = r + beta (p - omega v) into A
        TSF_FOR_E(npc) {
          const double2 pv = caxpy(beta, caxpy(-omega, VV[e], PV[e]), R[e]);
          PV[e] = pv;
          AX[e] = pv;
        }
      }
    } else if (iterate && METHOD == TSF_PCGS) {
      // Preconditioned CGS (the paper's PCGS; MATLAB pcgs), right-preconditioned:
      // shadow rt = r0, u = r + beta q, p = u + beta (q + beta p), phat = P^{-1} p, vhat = A phat,
      // alpha = rho / (rt.vhat), q = u - alpha vhat, uhat = P^{-1}(u + q), x += alpha uhat,
      // r -= alpha A uhat.  Vector slots: u -> S, p -> PV, q -> VV, phat -> PH.  As for BiCGSTAB,
      // the four applications of an iteration (h = 0..3: P^{-1}, A, P^{-1}, A) share one inlined
      // apply.
      double rho = rr0, alpha = 0.0;
      TSF_FOR_E(npc) {                           // u_0 = p_0 = r_0
        const double2 rv = R[e];
        S[e] = rv;
        PV[e] = rv;
      }
      for (int h = 0;; h = (h + 1) & 3) {
        const bool isP = !(h & 1);
        if (isP && !prec) {
          Y = AX;
        } else {
          __syncthreads();
          const SpecOp op = isP ? opP : opA;
          const Geo g = isP ? gp : ge;
          Y.p = apply<C, STG, BIG>(sm, P.L1e, g, op, tw, r, xs, I.xg, I.xa);
        }
        if (h == 0) {                            // phat
          TSF_FOR_E(npc) {
            const double2 phv = Y[e];
            PH[e] = phv;
            AX[e] = phv;
            AX[e + npc] = zero2();
          }
          continue;
        }
        if (h == 1) {                            // vhat: alpha, q = u - alpha vhat, A <- u + q
          double sg[1] = {0.0};
          TSF_FOR_E(npc) { sg[0] += cdot(RH[e], Y[e]); }
          csum<C, 1>(sg, sm, xs);
          if (!(fabs(sg[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
          alpha = rho / sg[0];
          TSF_FOR_E(npc) {                       // Y may alias A: read before the write
            const double2 u = S[e];
            const double2 q = caxpy(-alpha, Y[e], u);
            VV[e] = q;
            AX[e] = cadd(u, q);
          }
          continue;
        }
        if (h == 2) {                            // uhat: x += alpha uhat, A <- uhat
          TSF_FOR_E(npc) {
            const double2 uh = Y[e];
            X[e] = caxpy(alpha, uh, X[e]);
            AX[e] = uh;
            AX[e + npc] = zero2();
          }
          continue;
        }
        // h == 3: A uhat: r -= alpha A uhat; rho' = rt.r; ||r||
        double rr[2] = {0.0, 0.0};
        TSF_FOR_E(npc) {
          const double2 rn = caxpy(-alpha, Y[e], R[e]);
          R[e] = rn;
          rr[0] += cdot(RH[e], rn);
          rr[1] += cdot(rn, rn);
        }
        csum<C, 2>(rr, sm, xs);
        hs += 2;
        relres = sqrt(rr[1]) / rn0;
        if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
        if (relres < P.tol) break;
        if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
        if (!(fabs(rr[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
        const double beta = rr[0] / rho;
        rho = rr[0];
        TSF_FOR_E(npc) {                         // u = r + beta q; p = u + beta (q + beta p)
          const double2 q = VV[e];
          const double2 u = caxpy(beta, q, R[e]);
          const double2 pv = caxpy(beta, caxpy(beta, PV[e], q), u);
          S[e] = u;
          PV[e] = pv;
          AX[e] = pv;
        }
      }
    } else if (iterate && METHOD == TSF_CGNR) {
      // CGLS on K = A P^{-1} (DESIGN.md R-cgnr): y0 = 0, r = b, z = K^T r = P^{-T} A^T r, p = z;
      // per iteration phat = P^{-1} p, q = A phat, a = gamma/||q||^2, x += a phat, r -= a q,
      // z = P^{-T} A^T r, beta = ||z||^2 / gamma, p = z + beta p.  The four applications
      // (h = 2: A^T, 3: P^{-T}, 0: P^{-1}, 1: A) share one inlined apply; the loop enters at h = 2
      // with r already in A.
      const SpecOp opAT = make_op(P, I, j, OP_AT, r, sm);
      const SpecOp opPT = make_op(P, I, j, OP_PTINV, r, sm);
      double gam = 0.0, a = 0.0;
      bool first = true;
      for (int h = 2;; h = (h + 1) & 3) {
        const bool isPre = h == 0 || h == 3;
        if (isPre && !prec) {
          Y = AX;
        } else {
          __syncthreads();
          const SpecOp op = h == 0 ? opP : (h == 1 ? opA : (h == 2 ? opAT : opPT));
          const Geo g = isPre ? gp : ge;
          Y.p = apply<C, STG, BIG>(sm, P.L1e, g, op, tw, r, xs, I.xg, I.xa);
        }
        if (h == 2) {                            // A^T r -> first npc values into A for P^{-T}
          TSF_FOR_E(npc) { AX[e] = Y[e]; }
          continue;
        }
        if (h == 3) {                            // z = P^{-T} A^T r; gamma, beta; p = z + beta p
          double zz[1] = {0.0};
          TSF_FOR_E(npc) { zz[0] += cdot(Y[e], Y[e]); }
          csum<C, 1>(zz, sm, xs);
          const double beta = first ? 0.0 : zz[0] / gam;
          gam = zz[0];
          TSF_FOR_E(npc) {
            const double2 z = Y[e];
            const double2 pv = first ? z : caxpy(beta, PV[e], z);
            PV[e] = pv;
            AX[e] = pv;
          }
          first = false;
          continue;
        }
        if (h == 0) {                            // phat
          TSF_FOR_E(npc) {
            const double2 phv = Y[e];
            PH[e] = phv;
            AX[e] = phv;
            AX[e + npc] = zero2();
          }
          continue;
        }
        // h == 1: q = A phat; a = gamma / ||q||^2; x += a phat; r -= a q; ||r||
        double qq[1] = {0.0};
        TSF_FOR_E(npc) { qq[0] += cdot(Y[e], Y[e]); }
        csum<C, 1>(qq, sm, xs);
        if (!(qq[0] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
        a = gam / qq[0];
        double rl[1] = {0.0};
        TSF_FOR_E(npc) {
          X[e] = caxpy(a, PH[e], X[e]);
          const double2 rn = caxpy(-a, Y[e], R[e]);
          R[e] = rn;
          AX[e] = rn;
          AX[e + npc] = zero2();
          rl[0] += cdot(rn, rn);
        }
        csum<C, 1>(rl, sm, xs);
        hs += 2;
        relres = sqrt(rl[0] / gg);
        if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
        if (relres < P.tol) break;
        if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
      }
    }
    if (!tres) break;
    // true residual next, through the cold site: A <- x
    __syncthreads();             // every thread done with the last Y
    TSF_FOR_E(npc) {
      AX[e] = X[e];
      AX[e + npc] = zero2();
    }
    ph = S_TRUE;
  }

  if (mode != 0) {               // GSF setup: keep the solution of eq3.4
    double2 *Gx = reinterpret_cast<double2 *>(I.vec + (mode == 1 ? V_GX : V_GY) * n) + r * npc;
    TSF_FOR_E(npc) { Gx[e] = X[e]; }
    if (r == 0 && threadIdx.x == 0) I.par[mode == 1 ? 8 : 9] = double(status == TSF_LEVEL_OK ? hs : -1 - status);
    __syncthreads();
    return;
  }
  // finalize (alg1 step 3 result): d^j = u^{j+1} - u^j, u^j <- u^{j+1}
  double2 *Hj = reinterpret_cast<double2 *>(I.hist + j * n) + r * npc;
  TSF_FOR_E(npc) {
    const double2 x = X[e], u = V.U[e];
    Hj[e] = csub(x, u);
    V.U[e] = x;
  }
  if (r == 0 && threadIdx.x == 0) {
    I.it[j] = hs;
    I.rr[j] = relres;
    I.st[j] = status;
  }
  __syncthreads();
  if (P.helpers > 0 && threadIdx.x == 0) {   // this CTA's slice of d^j is written
    __threadfence();
    atomicAdd(reinterpret_cast<unsigned long long *>(P.sync), 1ull);
  }
#ifdef TSF_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    sm.prof[PS_LEVEL] += (unsigned long long)(clock64() - tlev0);
    sm.prof[PS_ITERS] += (unsigned long long)hs;
  }
#endif
}

// ------------------------------------------------------------------------ history helpers
// Single-instance solves occupy one cluster (C3: 16 of 148 SMs).  Extra clusters of the same
// launch ("helpers", all co-resident: the launcher checks cudaOccupancyMaxActiveClusters) stream
// the history while the solver iterates: during level J-1 they form the pre-sum
//   P^J = kappa (e_J d^0 + sum_{s=1}^{J-2} chat_{J-s} d^s)
// (eq3.1's memory term without its newest row) into pre[J & 1]; the solver then needs only
// kappa chat_1 d^{J-1}.  Protocol: solver CTAs count finished levels in sync[0] (release by
// fence + atomic); helpers wait for C (J - 1 - j0) of them, write their slice, count themselves
// in sync[3 + (J & 1)], and the last one publishes ready[J & 1] = J (release store).
template <int C>
__device__ void hist_helper(const DevParams &P, int32_t nlev, int *quit) {
  const Inst I = inst_view(P, 0);
  const int h = int(blockIdx.x) - P.B * C, nh = P.helpers;
  const int64_t n = P.n, half = n / 2;
  const int64_t j0 = *P.level, jend = (j0 + nlev < P.M) ? j0 + nlev : P.M;
  const double2 *Hd = reinterpret_cast<const double2 *>(I.hist);
  for (int64_t J = (j0 + 1 > 2 ? j0 + 1 : 2); J < jend; ++J) {
    if (threadIdx.x == 0) {
      // wait for the solver to finish level J-2 (its CTAs count levels in sync[0]); give up when
      // it makes no progress for kHelperIdleNs or the solver stopped relying on the helpers
      int q = 0;
      int64_t last = -1;
      uint64_t t0 = gtimer_ns();
      for (;;) {
        if (ld_acquire(P.sync + 5) != 0) { q = 1; break; }
        const int64_t v = ld_acquire(P.sync);
        if (v >= int64_t(C) * (J - 1 - j0)) break;
        if (v != last) { last = v; t0 = gtimer_ns(); }
        else if (gtimer_ns() - t0 > kHelperIdleNs) { st_release(P.sync + 5, 1); q = 1; break; }
        __nanosleep(256);
      }
      *quit = q;
    }
    __syncthreads();
    if (*quit) return;
    __syncthreads();
    double2 *Pj = reinterpret_cast<double2 *>(P.pre) + (J & 1) * half;
    const double wJ = I.hwe[J];
    for (int64_t e = int64_t(h) * kThreads + threadIdx.x; e < half; e += int64_t(nh) * kThreads) {
      double2 a = cscale(__ldcg(Hd + e), wJ), b = zero2();
      int64_t s = 1;
      for (; s + 7 <= J - 2; s += 8) {
        double2 v[8];
        double w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = __ldcg(Hd + (s + u) * half + e);
          w[u] = I.hwc[J - s - u];
        }
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          a = caxpy(w[u], v[u], a);
          b = caxpy(w[u + 1], v[u + 1], b);
        }
      }
      for (; s <= J - 2; ++s) a = caxpy(I.hwc[J - s], __ldcg(Hd + s * half + e), a);
      Pj[e] = cadd(a, b);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned long long *cnt = reinterpret_cast<unsigned long long *>(P.sync + 3 + (J & 1));
      if (atomicAdd(cnt, 1ull) == (unsigned long long)(nh - 1)) {
        *cnt = 0ull;
        __threadfence();
        st_release(P.sync + 1 + (J & 1), J);
      }
    }
  }
}

// ------------------------------------------------------------------------ kernels
template <int C, int METHOD, bool STG, bool VS, bool BIG = false>
__global__ void __launch_bounds__(kThreads, C == 1 ? TSF_C1_BLOCKS : 1)
    k_solve(DevParams P, int32_t nlev, int32_t mode) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (int(blockIdx.x) >= P.B * C) {   // history-helper clusters (single-instance launches)
    if constexpr (C > 1) hist_helper<C>(P, nlev, reinterpret_cast<int *>(smem_raw));
    return;
  }
  const int b = blockIdx.x / C;
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
#ifdef TSF_PROFILE
  // section counters accumulate in SMEM (a global read-modify-write per section would stall
  // warp 0 by an L2 round trip and inflate every section it times); flushed at the end
  __shared__ unsigned long long prof_s[32];
  if (threadIdx.x < 32) prof_s[threadIdx.x] = 0;
  __syncthreads();
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.vsmem != 0, prof_s, P.fuse_min, P.chunk, P.C);
#else
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.vsmem != 0, P.prof, P.fuse_min, P.chunk, P.C);
#endif
  const Vecs V = vec_view<VS>(P, I, sm, r);
  load_constants(P, I.lwe, P.precond != TSF_NOPREC ? I.lwp : nullptr, sm, r);
  const int npc = P.L1p;
  double2 *Ug = reinterpret_cast<double2 *>(I.vec + V_U * P.n) + r * npc;
  if constexpr (VS) TSF_FOR_E(npc) { V.U[e] = Ug[e]; }
  __syncthreads();
  xinit<C>(sm);
  Xch xs;
  const int64_t j0 = *P.level;
  if (mode != 0) {               // NEXT-2 setup solve with the level-1 operators
    level_solve<C, METHOD, STG, BIG>(P, I, sm, V, 1, r, xs, mode);
  } else {
    for (int64_t j = j0; j < j0 + nlev && j < P.M; ++j) level_solve<C, METHOD, STG, BIG>(P, I, sm, V, j, r, xs, 0, j0);
  }
  if constexpr (VS) TSF_FOR_E(npc) { Ug[e] = V.U[e]; }
#ifdef TSF_PROFILE
  __syncthreads();
  if (blockIdx.x == TSF_PROF_CTA && threadIdx.x < 32) P.prof[threadIdx.x] += prof_s[threadIdx.x];
#endif
  csync<C>();                    // no CTA leaves while a peer may still push into it
}

__global__ void k_advance(int64_t *level, int64_t by, int64_t M);

// Debug: one operator application of instance b at level j: in/out are permuted chunks.
// reps > 1 (timing): reps applications alternating P^{-1} and A (as in a Krylov iteration),
// each feeding the next; out holds the last result.
template <int C, bool STG, bool BIG = false>
__global__ void __launch_bounds__(kThreads, 1) k_debug_apply(DevParams P, int32_t reps, int b, int64_t j,
                                                              int which, const double *in, double *out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
#ifdef TSF_PROFILE
  __shared__ unsigned long long prof_s[32];
  if (threadIdx.x < 32) prof_s[threadIdx.x] = 0;
  __syncthreads();
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.vsmem != 0, prof_s, P.fuse_min, P.chunk, P.C);
#else
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.vsmem != 0, P.prof, P.fuse_min, P.chunk, P.C);
#endif
  load_constants(P, I.lwe, P.precond != TSF_NOPREC ? I.lwp : nullptr, sm, r);
  const int npc = P.L1p;
  const double2 *X = reinterpret_cast<const double2 *>(in) + r * npc;
  double2 *Y = reinterpret_cast<double2 *>(out) + r * npc;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  const ABuf<BIG> AX = abuf_in<BIG>(P, I, sm, r);
  for (int e = threadIdx.x; e < npc; e += kThreads) AX[e] = X[e];
  __syncthreads();
  xinit<C>(sm);
  Xch xs;
  fill_mul(P, I, j, r, sm);
  __syncthreads();
  ABuf<BIG> Z = AX;
  const int nrep = reps > 1 ? reps : 1;
  for (int rep = 0; rep < nrep; ++rep) {
    const int wh = reps > 1 ? ((rep & 1) ? OP_A : OP_PINV) : which;
    const bool embed = wh <= OP_AT;
    for (int e = threadIdx.x; e < npc; e += kThreads) {
      const double2 v = Z[e];
      AX[e] = v;
      if (embed) AX[e + npc] = zero2();
    }
    __syncthreads();
    const SpecOp op = make_op(P, I, j, wh, r, sm);
    Z.p = apply<C, STG, BIG>(sm, P.L1e, embed ? geo_embed(P, sm) : geo_prec(P, sm), op, tw, r, xs, I.xg, I.xa);
  }
  for (int e = threadIdx.x; e < npc; e += kThreads) Y[e] = Z[e];
#ifdef TSF_PROFILE
  __syncthreads();
  if (blockIdx.x == TSF_PROF_CTA && threadIdx.x < 32) P.prof[threadIdx.x] += prof_s[threadIdx.x];
#endif
  csync<C>();
}

// Debug: RHS of the current level for every instance into V_R.
template <int C, bool STG, bool BIG = false>
__global__ void __launch_bounds__(kThreads, 1) k_debug_rhs(DevParams P, int32_t) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int b = blockIdx.x / C;
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.vsmem != 0, P.prof, P.fuse_min, P.chunk, P.C);
  load_constants(P, I.lwe, P.precond != TSF_NOPREC ? I.lwp : nullptr, sm, r);
  const int64_t j = *P.level;
  const int npc = P.L1p;
  __syncthreads();
  if (j >= P.M) return;
  xinit<C>(sm);
  Xch xs;
  const SpecOp opB = make_op(P, I, j, OP_B, r, sm);
  const double2 *U = reinterpret_cast<const double2 *>(I.vec + V_U * P.n) + r * npc;
  double2 *Hs = reinterpret_cast<double2 *>(I.vec + V_X * P.n) + r * npc;
  rhs_phase<C, STG, BIG>(P, sm, I, geo_embed(P, sm), opB, j, r, U, Hs, xs);
  double2 *R = reinterpret_cast<double2 *>(I.vec + V_R * P.n) + r * npc;
  const ABuf<BIG> AX = abuf_in<BIG>(P, I, sm, r);
  for (int e = threadIdx.x; e < npc; e += kThreads) R[e] = AX[e];
  csync<C>();
}

// ------------------------------------------------------------------------ launch API
// Implemented per cluster size in tsf_solve_c<C>.cu (parallel compilation).
template <int C>
cudaError_t launch_solve_c(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st, int32_t mode);
template <int C>
cudaError_t launch_dbg_apply_c(const Plan &pl, const DevParams &dp, int b, int64_t j, int which,
                               const double *in, double *out, cudaStream_t st, int32_t reps);
template <int C>
cudaError_t launch_dbg_rhs_c(const Plan &pl, const DevParams &dp, cudaStream_t st);

// Cluster launch with the plan's dynamic shared memory.
template <class K, class... Args>
cudaError_t launch_cluster(K kern, const Plan &pl, int grid, cudaStream_t st, Args... args) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
  if (e != cudaSuccess) return e;
  if (pl.C > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = size_t(pl.smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(pl.C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Launch of a solve kernel, with history-helper clusters for multi-level single-instance
// cluster solves when the GPU can keep them all resident at once (they spin on each other).
template <class K>
cudaError_t launch_solve_k(K kern, const Plan &pl, const DevParams &dp0, int32_t nlev, cudaStream_t st,
                           int32_t mode) {
  DevParams dp = dp0;
  dp.helpers = 0;
  int grid = pl.B * pl.C;
  if (pl.B == 1 && pl.C > 1 && nlev >= 3 && mode == 0 && pl.hblock == 0 &&
      std::getenv("TSF_NO_HELPERS") == nullptr) {
    const int64_t cta_need = (pl.n / 2 + kThreads - 1) / kThreads;
    int hcl = int((cta_need + pl.C - 1) / pl.C);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) return e;
    if (pl.C > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((1 + hcl) * pl.C));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = size_t(pl.smem);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(pl.C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) == cudaSuccess) {
      if (hcl > active - 1) hcl = active - 1;
      if (hcl > 0) {
        dp.helpers = hcl * pl.C;
        grid = (1 + hcl) * pl.C;
        e = cudaMemsetAsync(dp.sync, 0, 8, st);                 // solver CTA-levels done
        if (e == cudaSuccess) e = cudaMemsetAsync(dp.sync + 1, 0xff, 16, st);   // ready[] = -1
        if (e == cudaSuccess) e = cudaMemsetAsync(dp.sync + 3, 0, 24, st);      // counters, gave-up flag
        if (e != cudaSuccess) return e;
      }
    } else {
      (void)cudaGetLastError();
    }
  }
  return launch_cluster(kern, pl, grid, st, dp, nlev, mode);
}

// Staged exchange (STG) exists for C > 1 only.
#define TSF_STG_OF(CC, pl) ((CC) > 1 && (pl).staged)
// Solve-kernel launchers per (cluster size, method), each instantiated in its own translation unit
// tsf_solve_c<C>_m<M>.cu (parallel compilation); launch_solve_c<C> dispatches on the method.
template <int C, int METHOD>
cudaError_t launch_solve_cm(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st, int32_t mode);
// Multi-pass regime kernels exist for 16-CTA clusters only.
template <int CC, int MM, bool ON = (CC == 16)>
struct BigK {
  static cudaError_t solve(const Plan &, const DevParams &, int32_t, cudaStream_t, int32_t) {
    return cudaErrorInvalidValue;
  }
  static cudaError_t apply(const Plan &, const DevParams &, int, int64_t, int, const double *, double *,
                           cudaStream_t, int32_t) {
    return cudaErrorInvalidValue;
  }
  static cudaError_t rhs(const Plan &, const DevParams &, cudaStream_t) { return cudaErrorInvalidValue; }
};
template <int CC, int MM>
struct BigK<CC, MM, true> {
  static cudaError_t solve(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st, int32_t z) {
    return launch_solve_k(k_solve<CC, MM, false, false, true>, pl, dp, nlev, st, z);
  }
  static cudaError_t apply(const Plan &pl, const DevParams &dp, int b, int64_t j, int which, const double *in,
                           double *out, cudaStream_t st, int32_t reps) {
    return launch_cluster(k_debug_apply<CC, false, true>, pl, CC, st, dp, reps, b, j, which, in, out);
  }
  static cudaError_t rhs(const Plan &pl, const DevParams &dp, cudaStream_t st) {
    return launch_cluster(k_debug_rhs<CC, false, true>, pl, pl.B * CC, st, dp, int32_t(0));
  }
};
#define TSF_INSTANTIATE_METHOD(CC, MM)                                                          \
  template <>                                                                                   \
  cudaError_t launch_solve_cm<CC, MM>(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st, \
                                      int32_t z) {                                              \
    constexpr bool S1 = (CC) > 1;                                                               \
    if (pl.big) return BigK<CC, MM>::solve(pl, dp, nlev, st, z);                                \
    const bool stg = TSF_STG_OF(CC, pl), vs = pl.vsmem != 0;                                    \
    if (stg && vs) return launch_solve_k(k_solve<CC, MM, S1, true>, pl, dp, nlev, st, z);       \
    if (stg) return launch_solve_k(k_solve<CC, MM, S1, false>, pl, dp, nlev, st, z);            \
    if (vs && CC == 1) return launch_solve_k(k_solve<CC, MM, false, CC == 1>, pl, dp, nlev, st, z); \
    return launch_solve_k(k_solve<CC, MM, false, false>, pl, dp, nlev, st, z);                  \
  }
#define TSF_INSTANTIATE_CLUSTER(CC)                                                             \
  template <>                                                                                   \
  cudaError_t launch_solve_c<CC>(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st, \
                                 int32_t z) {                                                   \
    switch (pl.method) {                                                                        \
      case TSF_BICGSTAB: return launch_solve_cm<CC, TSF_BICGSTAB>(pl, dp, nlev, st, z);         \
      case TSF_CGNR: return launch_solve_cm<CC, TSF_CGNR>(pl, dp, nlev, st, z);                 \
      case TSF_PCGS: return launch_solve_cm<CC, TSF_PCGS>(pl, dp, nlev, st, z);                 \
      case TSF_GSF: return launch_solve_cm<CC, TSF_GSF>(pl, dp, nlev, st, z);                   \
    }                                                                                           \
    return cudaErrorInvalidValue;                                                               \
  }                                                                                             \
  template <>                                                                                   \
  cudaError_t launch_dbg_apply_c<CC>(const Plan &pl, const DevParams &dp, int b, int64_t j,     \
                                     int which, const double *in, double *out, cudaStream_t st,  \
                                     int32_t reps) {                                             \
    if (pl.big) return BigK<CC, 0>::apply(pl, dp, b, j, which, in, out, st, reps);              \
    if (TSF_STG_OF(CC, pl))                                                                     \
      return launch_cluster(k_debug_apply<CC, true>, pl, CC, st, dp, reps, b, j, which, in, out); \
    return launch_cluster(k_debug_apply<CC, false>, pl, CC, st, dp, reps, b, j, which, in, out); \
  }                                                                                             \
  template <>                                                                                   \
  cudaError_t launch_dbg_rhs_c<CC>(const Plan &pl, const DevParams &dp, cudaStream_t st) {      \
    if (pl.big) return BigK<CC, 0>::rhs(pl, dp, st);                                            \
    if (TSF_STG_OF(CC, pl)) return launch_cluster(k_debug_rhs<CC, true>, pl, pl.B * CC, st, dp, int32_t(0)); \
    return launch_cluster(k_debug_rhs<CC, false>, pl, pl.B * CC, st, dp, int32_t(0));           \
  }

}  // namespace tsf
