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

#include "tsf_plan.h"

namespace cg = cooperative_groups;

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
  int32_t *it, *st;
  double *rr;
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
  I.it = reinterpret_cast<int32_t *>(base + P.o_it);
  I.rr = reinterpret_cast<double *>(base + P.o_rr);
  I.st = reinterpret_cast<int32_t *>(base + P.o_st);
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
  double2 *ctwe, *ctwp;              // column twiddles (resident)
  double2 *lame, *lamp, *pwe, *pwp;  // base spectra / pair twiddles (resident)
  double *sqe, *sqp;                 // sine tables (resident)
  double *wred, *cred;
  unsigned long long *prof;
};

// Section timers (profiling build, -DTSF_PROFILE): thread 0 of block 0 accumulates clock64
// cycles per section into P.prof[slot]; the wait at a barrier is charged to the section
// that ends with it.
#ifdef TSF_PROFILE
#define TSF_PT0() long long tsf_pt_ = clock64()
#define TSF_PACC(sm, slot)                                                                    \
  do {                                                                                      \
    const long long t_ = clock64();                                                         \
    if (threadIdx.x == 0 && blockIdx.x == 0) (sm).prof[slot] += (unsigned long long)(t_ - tsf_pt_); \
    tsf_pt_ = t_;                                                                           \
  } while (0)
#else
#define TSF_PT0() do {} while (0)
#define TSF_PACC(sm, slot) do {} while (0)
#endif
enum ProfSlot { PS_FFT_F = 0, PS_BAR1, PS_GATHER, PS_COLF, PS_PAIRS, PS_COLI, PS_BAR2, PS_SCATTER,
                PS_BAR3, PS_FFT_I, PS_CSUM, PS_VEC, PS_RHS_HIST, PS_LEVEL, PS_APPLIES, PS_ITERS };
__device__ __forceinline__ int tw_hi_len(int L1e) { return L1e >= 64 ? L1e / 64 : 1; }
__device__ __forceinline__ int tw_lo_len(int L1e) { return L1e >= 64 ? 64 : L1e; }

__device__ __forceinline__ Smem smem_view(unsigned char *raw, int L1e, int L1p, bool staged,
                                          bool resident, unsigned long long *prof) {
  Smem s = {};
  s.prof = prof;
  double2 *c = reinterpret_cast<double2 *>(raw);
  const int L1pad = L1e + L1e / 16;
  s.A = c; c += L1pad;
  if (staged) { s.B = c; c += L1e; s.O = c; c += L1pad; }
  if (resident) {
    s.twd = c; c += L1e;
    s.ctwe = c; c += L1e; s.ctwp = c; c += L1p;
    s.lame = c; c += L1e; s.lamp = c; c += L1p;
    s.pwe = c; c += L1e; s.pwp = c; c += L1p;
  } else {
    s.thi = c; c += tw_hi_len(L1e);
    s.tlo = c; c += tw_lo_len(L1e);
  }
  double *d = reinterpret_cast<double *>(c);
  if (resident) { s.sqe = d; d += L1e; s.sqp = d; d += L1p; }
  s.wred = d;
  s.cred = d + 40;
  return s;
}

__device__ __forceinline__ double2 twid(const Smem &sm, int e) {
  if (sm.twd) return sm.twd[e];
  return cmul(sm.thi[e >> 6], sm.tlo[e & 63]);
}

__device__ __forceinline__ int col_k1(int L1, int C, uint32_t r, int col);

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
  if (sm.ctwe) {
    const int64_t n = P.n;
    const int twL_e = P.twN / int(n), twL_p = P.twN / int(n / 2);
    const int nce = L1e / C, ncp = L1p / C;
    for (int u = threadIdx.x; u < L1e; u += kThreads) {     // column twiddles W_L^{q k1}
      const int q = u / nce, col = u - q * nce;
      sm.ctwe[u] = tw[q * col_k1(L1e, C, r, col) * twL_e];
    }
    for (int u = threadIdx.x; u < L1p; u += kThreads) {
      const int q = u / ncp, col = u - q * ncp;
      sm.ctwp[u] = tw[q * col_k1(L1p, C, r, col) * twL_p];
    }
    // task-order slices of CTA r: index ((r C + k2) 2 + ab) np + i = r L1 + local
    for (int u = threadIdx.x; u < L1e; u += kThreads) {
      const int np = P.npe;
      const int i = u % np, ab = (u / np) & 1, k2 = u / (2 * np);
      sm.lame[u] = lwe[int64_t(r) * L1e + u];
      sm.sqe[u] = P.sq_e[int64_t(r) * L1e + u];
      sm.pwe[u] = tw[task_bin(L1e, C, int(r), i, k2, ab) * (P.twN / int(2 * n))];
    }
    for (int u = threadIdx.x; u < L1p; u += kThreads) {
      const int np = P.npp;
      const int i = u % np, ab = (u / np) & 1, k2 = u / (2 * np);
      if (lwp) sm.lamp[u] = lwp[int64_t(r) * L1p + u];
      sm.sqp[u] = P.sq_p[int64_t(r) * L1p + u];
      sm.pwp[u] = tw[task_bin(L1p, C, int(r), i, k2, ab) * (P.twN / int(n))];
    }
  }
}

// Deterministic cluster-wide sum of NV <= 4 scalars: warp butterflies (exactly commutative,
// so every lane holds the same bits) -> 8 warps in order -> C CTA partials through a
// 32-lane butterfly in warp 0 (lanes >= C add 0) -> broadcast.
template <int C, int NV>
__device__ __forceinline__ void csum(double (&v)[NV], const Smem &sm, int &par) {
  TSF_PT0();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sm.wred[warp * 4 + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) s += sm.wred[w * 4 + k];
      sm.cred[par * 4 + k] = s;
    }
  }
  if constexpr (C == 1) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = sm.cred[par * 4 + k];
  } else {
    csync<C>();
    if (warp == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double s = lane < C ? remote<C>(sm.cred, uint32_t(lane))[par * 4 + k] : 0.0;
        s = warp_sum(s);
        if (lane == 0) sm.wred[32 + k] = s;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = sm.wred[32 + k];
  }
  par ^= 1;
  TSF_PACC(sm, PS_CSUM);
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

// Padded SMEM index of element p of a transform buffer (A, O): one pad slot per 16 elements
// makes the stride-4 and stride-16 accesses of the early DIT / late DIF stages bank-conflict
// free.  Buffers hold L1 + L1/16 complex values.
__device__ __forceinline__ int pidx(int p) { return p + (p >> 4); }

// one stage: m = 2^lm, twiddle W_m^{kq} = W_{L1e}^{kq (L1e/m)}
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
      if (k != 0) {
        const double2 w1 = twid(sm, k * tstep), w2 = twid(sm, 2 * k * tstep), w3 = twid(sm, 3 * k * tstep);
        if (INV) {
          a1 = cmulc(a1, w1); a2 = cmulc(a2, w2); a3 = cmulc(a3, w3);
          bfly4<true>(a0, a1, a2, a3);
        } else {
          bfly4<false>(a0, a1, a2, a3);
          a1 = cmul(a1, w1); a2 = cmul(a2, w2); a3 = cmul(a3, w3);
        }
      } else {
        bfly4<INV>(a0, a1, a2, a3);
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
        const int k = jp * mpp + kpp;
        if (k != 0) {
          x[1][jp] = cmul(x[1][jp], twid(sm, k * ts));
          x[2][jp] = cmul(x[2][jp], twid(sm, 2 * k * ts));
          x[3][jp] = cmul(x[3][jp], twid(sm, 3 * k * ts));
        }
      }
      double2 w1 = zero2(), w2 = zero2(), w3 = zero2();
      if (kpp != 0) { w1 = twid(sm, kpp * tsp); w2 = twid(sm, 2 * kpp * tsp); w3 = twid(sm, 3 * kpp * tsp); }
#pragma unroll
      for (int j = 0; j < 4; ++j) {               // stage s-1: butterfly k = kpp in group 4g + j
        bfly4<false>(x[j][0], x[j][1], x[j][2], x[j][3]);
        if (kpp != 0) {
          x[j][1] = cmul(x[j][1], w1);
          x[j][2] = cmul(x[j][2], w2);
          x[j][3] = cmul(x[j][3], w3);
        }
      }
    } else {
      double2 w1 = zero2(), w2 = zero2(), w3 = zero2();
      if (kpp != 0) { w1 = twid(sm, kpp * tsp); w2 = twid(sm, 2 * kpp * tsp); w3 = twid(sm, 3 * kpp * tsp); }
#pragma unroll
      for (int j = 0; j < 4; ++j) {               // DIT stage s-1
        if (kpp != 0) {
          x[j][1] = cmulc(x[j][1], w1);
          x[j][2] = cmulc(x[j][2], w2);
          x[j][3] = cmulc(x[j][3], w3);
        }
        bfly4<true>(x[j][0], x[j][1], x[j][2], x[j][3]);
      }
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {            // DIT stage s
        const int k = jp * mpp + kpp;
        if (k != 0) {
          x[1][jp] = cmulc(x[1][jp], twid(sm, k * ts));
          x[2][jp] = cmulc(x[2][jp], twid(sm, 2 * k * ts));
          x[3][jp] = cmulc(x[3][jp], twid(sm, 3 * k * ts));
        }
        bfly4<true>(x[0][jp], x[1][jp], x[2][jp], x[3][jp]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) A[pidx(base + j * mp + jp * mpp)] = x[j][jp];
  }
}

// Requires the input to be visible to all threads (caller synchronizes); ends synchronized.
// Radix-4 stages are fused pairwise into radix-16 register passes from the bottom (stages
// (1,0), (3,2), ...); a leftover top radix-4 stage and the radix-2 stage run alone.
template <bool INV>
__device__ __forceinline__ void local_fft(double2 *A, int L1, const Smem &sm, int L1e) {
  const int l = __ffs(L1) - 1;
  const int S4 = l >> 1;
  const bool r2 = l & 1;
  // fuse only when every thread owns a 16-point super-butterfly (else radix-4 stages keep
  // all threads busy); the data placement is the same either way
  const bool fuse = L1 >= 16 * kThreads;
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
  if constexpr (N > 1) {
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
struct SpecOp {
  const double2 *lam;   // task-order base spectrum of this instance (SMEM slice if resident)
  const double *sq;     // task-order sine table
  const double2 *pw;    // resident: pair twiddles W_{2L}^{bin} in task order, else nullptr
  double2 nyq;          // base spectrum at the Nyquist bin L
  int np;               // column-pair tasks per CTA
  int rC;               // r * C (0 for resident slices)
  double eta, mu, ppq, pmq, c2, qcorr, scale;
  bool conj;
  // W_{2L}^{bin} of bin (k2, ab, i): resident table or the global twiddle table
  __device__ __forceinline__ double2 wtw(int k2, int ab, int i, int bin, const double2 *tw,
                                         int tw2L) const {
    return pw ? pw[((rC + k2) * 2 + ab) * np + i] : tw[bin * tw2L];
  }
  __device__ __forceinline__ double2 lam_idx(int idx, int bin) const {
    const double2 b = lam[idx];
    const double s = sq[idx];
    const double re = ppq * b.x + ((bin & 1) ? -qcorr : qcorr);
    const double im = pmq * b.y + c2 * s;
    return make_double2(eta + mu * re, conj ? -(mu * im) : mu * im);
  }
  __device__ __forceinline__ double2 get(int k2, int ab, int i, int bin) const {
    return lam_idx(((rC + k2) * 2 + ab) * np + i, bin);
  }
  __device__ __forceinline__ double2 nyquist(int Lbin) const {
    const double re = ppq * nyq.x + ((Lbin & 1) ? -qcorr : qcorr);
    const double im = pmq * nyq.y;
    return make_double2(eta + mu * re, conj ? -(mu * im) : mu * im);
  }
};

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  const double inv = 1.0 / d;
  return make_double2((a.x * b.x + a.y * b.y) * inv, (a.y * b.x - a.x * b.y) * inv);
}

// Real-FFT split for the pair of bins (k, L-k) of a length-L complex transform z of a
// 2L-point real sequence x (z_m = x_{2m} + i x_{2m+1}), apply Y = X * lambda (or X / lambda)
// to X_k and X_{L-k}, and merge back to Z' such that the unnormalized inverse DFT of Z'
// returns y packed the same way.  w = exp(-i pi k / L); s = 1/(4L) folds the halves and 1/L.
template <bool DIV>
__device__ __forceinline__ void pair_apply(double2 &Za, double2 &Zb, double2 la, double2 lb,
                                           double2 w, double s) {
  const double2 cZb = cconj(Zb);
  const double2 Ep = cadd(Za, cZb);               // 2 E_k
  const double2 Op = mul_mi(csub(Za, cZb));       // 2 O_k
  const double2 wO = cmul(w, Op);
  const double2 Xa = cadd(Ep, wO);                // 2 X_k
  const double2 Xb = cconj(csub(Ep, wO));         // 2 X_{L-k}
  const double2 Ya = DIV ? cdiv(Xa, la) : cmul(Xa, la);
  const double2 Yb = DIV ? cdiv(Xb, lb) : cmul(Xb, lb);
  const double2 cYb = cconj(Yb);
  const double2 E2 = cadd(Ya, cYb);               // 4 E'_k
  const double2 O2 = cmulc(csub(Ya, cYb), w);     // 4 O'_k
  Za = cscale(cadd(E2, mul_i(O2)), s);
  Zb = cscale(cadd(cconj(E2), mul_i(cconj(O2))), s);
}

template <bool DIV>
__device__ __forceinline__ void pair_self(double2 &Z, double2 la, double2 lb, double2 w, double s) {
  double2 a = Z, b = Z;
  pair_apply<DIV>(a, b, la, lb, w, s);
  Z = a;
}

struct Geo {
  int L1, L, np, twL, tw2L;   // twL = twN/L (W_L factor), tw2L = twN/(2L)
  const int32_t *slot;
  const double2 *ctw;         // resident column twiddles W_L^{q k1(col)} [q ncol + col]
};

// C == 1: the whole transform is local; column pairs are bin pairs (k, L-k).
template <bool DIV>
__device__ __forceinline__ void pointwise_local(double2 *A, const Geo &g, const SpecOp &op,
                                             const double2 *__restrict__ tw) {
  for (int i = threadIdx.x; i < g.np; i += kThreads) {
    if (i == 0) {
      const int sa = pidx(g.slot[0]), sb = pidx(g.slot[g.L1 / 2]);
      double2 a = A[sa], b = A[sb];
      pair_self<DIV>(a, op.get(0, 0, 0, 0), op.nyquist(g.L), tw[0], op.scale);
      const double2 lm = op.get(0, 1, 0, g.L / 2);
      pair_self<DIV>(b, lm, lm, tw[(g.L / 2) * g.tw2L], op.scale);
      A[sa] = a; A[sb] = b;
    } else {
      const int sa = pidx(g.slot[i]), sb = pidx(g.slot[g.L1 - i]);
      double2 a = A[sa], b = A[sb];
      pair_apply<DIV>(a, b, op.get(0, 0, i, i), op.get(0, 1, i, g.L - i), tw[i * g.tw2L], op.scale);
      A[sa] = a; A[sb] = b;
    }
  }
}

// column pair i of CTA r: (k1a, k1b) = (pi, L1 - pi) with pi = r + i C, or (0, L1/2) for pi = 0
__device__ __forceinline__ int col_k1(int L1, int C, uint32_t r, int col) {
  const int pi = int(r) + (col >> 1) * C;
  if (pi == 0) return (col & 1) ? L1 / 2 : 0;
  return (col & 1) ? L1 - pi : pi;
}

// C > 1, staged through the local buffer B (layout B[q * ncol + col], ncol = L1/C):
//   gather A_q[slot(k1)] from every CTA -> per column: twiddle W_L^{q k1}, DFT_C -> per bin
//   pair: spectral op -> per column: inverse DFT_C, conj twiddle -> scatter to O_{m2}.
// The result lands in the output buffers O, so no CTA can still be gathering from the
// buffer being written: two cluster barriers per application (before the gather, after the
// scatter).
template <int C, bool DIV>
__device__ __forceinline__ void cross_staged(double2 *A, double2 *B, double2 *O, const Geo &g,
                                          const SpecOp &op, const double2 *__restrict__ tw, uint32_t r,
                                          const Smem &sm) {
  TSF_PT0();
  const int ncol = g.L1 / C;
#pragma unroll 4
  for (int u = threadIdx.x; u < g.L1; u += kThreads) {       // DSMEM gather
    const int q = u / ncol, col = u - q * ncol;
    B[u] = remote<C>(A, uint32_t(q))[pidx(g.slot[col_k1(g.L1, C, r, col)])];
  }
  __syncthreads();
  TSF_PACC(sm, PS_GATHER);
  for (int col = threadIdx.x; col < ncol; col += kThreads) {  // column DFT_C
    const int k1 = col_k1(g.L1, C, r, col);
    double2 z[C];
#pragma unroll
    for (int q = 0; q < C; ++q) z[q] = B[q * ncol + col];
    if (g.ctw) {
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmul(z[q], g.ctw[q * ncol + col]);
    } else {
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmul(z[q], tw[q * k1 * g.twL]);
    }
    fft_reg<C, false>(z);
#pragma unroll
    for (int q = 0; q < C; ++q) B[q * ncol + col] = z[q];
  }
  __syncthreads();
  TSF_PACC(sm, PS_COLF);
  // bin pairs: item u = k2 * np + i; regular pair (col 2i row k2) <-> (col 2i+1 row C-1-k2)
  for (int u = threadIdx.x; u < g.np * C; u += kThreads) {
    const int k2 = u / g.np, i = u - k2 * g.np;
    const int pi = int(r) + i * C;
    if (pi != 0) {
      const int bin = pi + g.L1 * k2;
      double2 &za = B[k2 * ncol + 2 * i];
      double2 &zb = B[(C - 1 - k2) * ncol + 2 * i + 1];
      double2 a = za, b = zb;
      pair_apply<DIV>(a, b, op.get(k2, 0, i, bin), op.get(C - 1 - k2, 1, i, g.L - bin),
                      op.wtw(k2, 0, i, bin, tw, g.tw2L), op.scale);
      za = a;
      zb = b;
    } else {
      // column 0 (bins L1 k2) pairs k2 <-> (C - k2) mod C; k2 = 0 pairs with the Nyquist bin
      const int kk = (C - k2) % C;
      if (k2 <= C / 2) {
        const int bin = g.L1 * k2;
        const double2 la = op.get(k2, 0, 0, bin);
        const double2 w = op.wtw(k2, 0, 0, bin, tw, g.tw2L);
        double2 &za = B[k2 * ncol];
        if (kk == k2) {
          double2 a = za;
          pair_self<DIV>(a, la, k2 == 0 ? op.nyquist(g.L) : la, w, op.scale);
          za = a;
        } else {
          double2 &zb = B[kk * ncol];
          double2 a = za, b = zb;
          pair_apply<DIV>(a, b, la, op.get(kk, 0, 0, g.L - bin), w, op.scale);
          za = a;
          zb = b;
        }
      }
      // column L1/2 (bins L1/2 + L1 k2) pairs k2 <-> C-1-k2
      const int km = C - 1 - k2;
      if (k2 < (C + 1) / 2) {
        const int bin = g.L1 / 2 + g.L1 * k2;
        const double2 la = op.get(k2, 1, 0, bin);
        const double2 w = op.wtw(k2, 1, 0, bin, tw, g.tw2L);
        double2 &za = B[k2 * ncol + 1];
        if (km == k2) {
          double2 a = za;
          pair_self<DIV>(a, la, la, w, op.scale);
          za = a;
        } else {
          double2 &zb = B[km * ncol + 1];
          double2 a = za, b = zb;
          pair_apply<DIV>(a, b, la, op.get(km, 1, 0, g.L - bin), w, op.scale);
          za = a;
          zb = b;
        }
      }
    }
  }
  __syncthreads();
  TSF_PACC(sm, PS_PAIRS);
  for (int col = threadIdx.x; col < ncol; col += kThreads) {  // inverse column DFT_C
    const int k1 = col_k1(g.L1, C, r, col);
    double2 z[C];
#pragma unroll
    for (int q = 0; q < C; ++q) z[q] = B[q * ncol + col];
    fft_reg<C, true>(z);
    if (g.ctw) {
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmulc(z[q], g.ctw[q * ncol + col]);
    } else {
#pragma unroll
      for (int q = 1; q < C; ++q) z[q] = cmulc(z[q], tw[q * k1 * g.twL]);
    }
#pragma unroll
    for (int q = 0; q < C; ++q) B[q * ncol + col] = z[q];
  }
  __syncthreads();
  TSF_PACC(sm, PS_COLI);
#pragma unroll 4
  for (int u = threadIdx.x; u < g.L1; u += kThreads) {       // DSMEM scatter into O
    const int q = u / ncol, col = u - q * ncol;
    remote<C>(O, uint32_t(q))[pidx(g.slot[col_k1(g.L1, C, r, col)])] = B[u];
  }
  TSF_PACC(sm, PS_SCATTER);
  csync<C>();                    // scatters landed
}

// C > 1 without a staging buffer (shared memory full): one thread per column pair keeps the
// 2C values in registers across the barrier.  Requires np <= kThreads.
template <int C, bool DIV>
__device__ __noinline__ void cross_reg(double2 *A, const Geo &g, const SpecOp &op,
                                       const double2 *__restrict__ tw, uint32_t r) {
  double2 za[C], zb[C];
  const int i = threadIdx.x;
  const bool act = i < g.np;
  const int pi = int(r) + i * C;
  const bool pseudo = (pi == 0);
  const int k1a = pseudo ? 0 : pi;
  const int k1b = pseudo ? g.L1 / 2 : g.L1 - pi;
  int sa = 0, sb = 0;
  if (act) {
    sa = pidx(g.slot[k1a]);
    sb = pidx(g.slot[k1b]);
#pragma unroll
    for (int q = 0; q < C; ++q) {
      const double2 *Aq = remote<C>(A, uint32_t(q));
      za[q] = Aq[sa];
      zb[q] = Aq[sb];
    }
#pragma unroll
    for (int q = 1; q < C; ++q) {
      za[q] = cmul(za[q], tw[q * k1a * g.twL]);
      zb[q] = cmul(zb[q], tw[q * k1b * g.twL]);
    }
    fft_reg<C, false>(za);
    fft_reg<C, false>(zb);
    if (!pseudo) {
#pragma unroll
      for (int k2 = 0; k2 < C; ++k2) {
        const int bin = k1a + g.L1 * k2;
        pair_apply<DIV>(za[k2], zb[C - 1 - k2], op.get(k2, 0, i, bin),
                        op.get(C - 1 - k2, 1, i, g.L - bin), tw[bin * g.tw2L], op.scale);
      }
    } else {
#pragma unroll
      for (int k2 = 0; k2 <= C / 2; ++k2) {
        const int kk = (C - k2) % C;
        const int bin = g.L1 * k2;
        const double2 la = op.get(k2, 0, 0, bin);
        if (kk == k2) {
          const double2 lb = (k2 == 0) ? op.nyquist(g.L) : la;
          pair_self<DIV>(za[k2], la, lb, tw[bin * g.tw2L], op.scale);
        } else {
          pair_apply<DIV>(za[k2], za[kk], la, op.get(kk, 0, 0, g.L - bin), tw[bin * g.tw2L], op.scale);
        }
      }
#pragma unroll
      for (int k2 = 0; k2 < (C + 1) / 2; ++k2) {
        const int kk = C - 1 - k2;
        const int bin = g.L1 / 2 + g.L1 * k2;
        const double2 la = op.get(k2, 1, 0, bin);
        if (kk == k2) pair_self<DIV>(zb[k2], la, la, tw[bin * g.tw2L], op.scale);
        else pair_apply<DIV>(zb[k2], zb[kk], la, op.get(kk, 1, 0, g.L - bin), tw[bin * g.tw2L], op.scale);
      }
    }
    fft_reg<C, true>(za);
    fft_reg<C, true>(zb);
#pragma unroll
    for (int q = 1; q < C; ++q) {
      za[q] = cmulc(za[q], tw[q * k1a * g.twL]);
      zb[q] = cmulc(zb[q], tw[q * k1b * g.twL]);
    }
  }
  csync<C>();
  if (act) {
#pragma unroll
    for (int q = 0; q < C; ++q) {
      double2 *Aq = remote<C>(A, uint32_t(q));
      Aq[sa] = za[q];
      Aq[sb] = zb[q];
    }
  }
  csync<C>();
}

// y = op(x) for the CTA's local data already in A[0..L1) (natural order, visible).
// Returns the buffer that holds this CTA's part of the result (natural order, visible):
// O in the staged mode, A otherwise.  The caller writes the next input into A.
template <int C, bool DIV, bool STG>
__device__ __forceinline__ double2 *apply(const Smem &sm, int L1e, const Geo &g, const SpecOp &op,
                                          const double2 *__restrict__ tw, uint32_t r) {
  TSF_PT0();
  local_fft<false>(sm.A, g.L1, sm, L1e);
  TSF_PACC(sm, PS_FFT_F);
  double2 *Y = sm.A;
  if constexpr (C == 1) {
    pointwise_local<DIV>(sm.A, g, op, tw);
    __syncthreads();
    TSF_PACC(sm, PS_PAIRS);
  } else {
    csync<C>();                  // every local transform done before remote gathers
    TSF_PACC(sm, PS_BAR1);
    if constexpr (STG) {
      cross_staged<C, DIV>(sm.A, sm.B, sm.O, g, op, tw, r, sm);
      Y = sm.O;
    } else {
      cross_reg<C, DIV>(sm.A, g, op, tw, r);
    }
    TSF_PACC(sm, PS_BAR3);
  }
  local_fft<true>(Y, g.L1, sm, L1e);
  TSF_PACC(sm, PS_FFT_I);
#ifdef TSF_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == 0) sm.prof[PS_APPLIES] += 1;
#endif
  return Y;
}

// ------------------------------------------------------------------------ operator setup
enum Which { OP_A = 0, OP_B = 1, OP_AT = 2, OP_PINV = 3, OP_PTINV = 4 };

__device__ __forceinline__ Geo geo_embed(const DevParams &P, const Smem &sm) {
  Geo g;
  g.L1 = P.L1e; g.L = int(P.n); g.np = P.npe; g.twL = P.twN / int(P.n); g.tw2L = P.twN / int(2 * P.n);
  g.slot = P.slot_e;
  g.ctw = sm.ctwe;
  return g;
}
__device__ __forceinline__ Geo geo_prec(const DevParams &P, const Smem &sm) {
  Geo g;
  g.L1 = P.L1p; g.L = int(P.n / 2); g.np = P.npp; g.twL = P.twN / int(P.n / 2); g.tw2L = P.twN / int(P.n);
  g.slot = P.slot_p;
  g.ctw = sm.ctwp;
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
  const bool res = sm.lame != nullptr;
  op.rC = res ? 0 : int(r) * P.C;
  op.eta = eta;
  op.ppq = p + q;
  op.pmq = p - q;
  if (which <= OP_AT) {
    op.lam = res ? sm.lame : I.lwe;
    op.sq = res ? sm.sqe : P.sq_e;
    op.pw = res ? sm.pwe : nullptr;
    op.np = P.npe; op.nyq = I.lwe[P.n];
    op.mu = (which == OP_B) ? (1.0 - sigma) : -sigma;
    op.c2 = 2.0 * c;
    op.qcorr = 0.0;
    op.scale = P.scale_e;
    op.conj = (which == OP_AT);
  } else {
    op.lam = res ? sm.lamp : I.lwp;
    op.sq = res ? sm.sqp : P.sq_p;
    op.pw = res ? sm.pwp : nullptr;
    op.np = P.npp; op.nyq = I.lwp[P.n / 2];
    op.mu = -sigma;
    op.c2 = 2.0 * c * P.qscale_p;
    op.qcorr = P.strang ? -q * I.par[2] : 0.0;   // Strang s(W^T) midpoint fix (R-strang)
    op.scale = P.scale_p;
    op.conj = (which == OP_PTINV);
  }
  return op;
}

// ------------------------------------------------------------------------ vector storage
// VPT > 0: this thread's VPT complex elements e = tid + q T in registers; VPT == 0: global.
template <int VPT>
struct VecT {
  double2 d[VPT > 0 ? VPT : 1];
  double2 *p;
  __device__ __forceinline__ double2 &operator()(int q, int e) {
    if constexpr (VPT > 0) return d[q];
    else return p[e];
  }
};

template <int VPT, class F>
__device__ __forceinline__ void for_elems(int npc, F &&f) {
  if constexpr (VPT > 0) {
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int e = threadIdx.x + q * kThreads;
      if (e < npc) f(q, e);
    }
  } else {
    for (int e = threadIdx.x; e < npc; e += kThreads) f(0, e);
  }
}

template <int VPT>
__device__ __forceinline__ void bind(VecT<VPT> &v, double *base, int64_t n, int slot, int off) {
  v.p = reinterpret_cast<double2 *>(base + slot * n) + off;
}

// ------------------------------------------------------------------------ RHS (alg1 step 2)
// g = B u^j - [kappa e_j d^0 + sum_{s=1}^{j-1} kappa chat_{j-s} d^s] + f^{j+sigma}
// Returns the local partial ||g||^2; g is left in A[0..npc) (and A[npc..2npc) is zero).
template <int C, int VPT, bool STG>
__device__ __forceinline__ double rhs_phase(const DevParams &P, const Inst &I, int64_t j, const Smem &sm,
                                            uint32_t r, VecT<VPT> &U) {
  const int npc = P.L1p;
  const int64_t n = P.n;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  for_elems<VPT>(npc, [&](int q, int e) {
    sm.A[pidx(e)] = U(q, e);
    sm.A[pidx(e + npc)] = zero2();
  });
  __syncthreads();
  const SpecOp opB = make_op(P, I, j, OP_B, r, sm);
  const double2 *Y = apply<C, false, STG>(sm, P.L1e, geo_embed(P, sm), opB, tw, r);
  const double2 *H = reinterpret_cast<const double2 *>(I.hist) + r * npc;
  const int64_t hstride = n / 2;  // double2 per history row
  double acc = 0.0;
  TSF_PT0();
  for_elems<VPT>(npc, [&](int, int e) {
    double2 g = Y[pidx(e)];
    if (j >= 1) {
      double2 h0 = cscale(H[e], I.hwe[j]);
      double2 h1 = zero2(), h2 = h1, h3 = h1;
      int64_t s = 1;
      for (; s + 3 <= j - 1; s += 4) {
        const double2 d0 = H[s * hstride + e], d1 = H[(s + 1) * hstride + e];
        const double2 d2 = H[(s + 2) * hstride + e], d3 = H[(s + 3) * hstride + e];
        h0 = caxpy(I.hwc[j - s], d0, h0);
        h1 = caxpy(I.hwc[j - s - 1], d1, h1);
        h2 = caxpy(I.hwc[j - s - 2], d2, h2);
        h3 = caxpy(I.hwc[j - s - 3], d3, h3);
      }
      for (; s <= j - 1; ++s) h0 = caxpy(I.hwc[j - s], H[s * hstride + e], h0);
      g = csub(g, cadd(cadd(h0, h1), cadd(h2, h3)));
    }
    if (P.src_kind == TSF_SRC_SEPARABLE) {
      const double2 *Bs = reinterpret_cast<const double2 *>(I.basis) + r * npc;
      for (int k = 0; k < P.K; ++k) g = caxpy(I.scal[j * P.K + k], Bs[k * hstride + e], g);
    } else if (P.src_kind == TSF_SRC_TABLE) {
      const double2 *F = reinterpret_cast<const double2 *>(I.ftab) + r * npc;
      g = cadd(g, F[j * hstride + e]);
    }
    sm.A[pidx(e)] = g;
    sm.A[pidx(e + npc)] = zero2();
    acc += cdot(g, g);
  });
  TSF_PACC(sm, PS_RHS_HIST);
  return acc;
}

// ------------------------------------------------------------------------ one level
// All control flow is uniform over the cluster (every CTA reduces to identical scalars).
template <int C, int METHOD, int VPT, bool STG>
__device__ __forceinline__ void level_solve(const DevParams &P, const Inst &I, int64_t j, const Smem &sm,
                                            uint32_t r, VecT<VPT> &U) {
  const int npc = P.L1p;
  const int64_t n = P.n;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  const bool prec = P.precond != TSF_NOPREC;
  const Geo ge = geo_embed(P, sm), gp = geo_prec(P, sm);
  VecT<VPT> X, R, RH, PV, VV, S, PH, SH;
  if constexpr (VPT == 0) {
    const int off = int(r) * npc;
    bind(X, I.vec, n, V_X, off); bind(R, I.vec, n, V_R, off); bind(RH, I.vec, n, V_RH, off);
    bind(PV, I.vec, n, V_P, off); bind(VV, I.vec, n, V_V, off); bind(S, I.vec, n, V_S, off);
    bind(PH, I.vec, n, V_PH, off); bind(SH, I.vec, n, V_SH, off);
  }
  int par = 0;
#ifdef TSF_PROFILE
  const long long tlev0 = clock64();
#endif

  double g2[1] = {rhs_phase<C, VPT, STG>(P, I, j, sm, r, U)};
  for_elems<VPT>(npc, [&](int q, int e) {
    const double2 g = sm.A[pidx(e)];
    R(q, e) = g;
    if (METHOD == TSF_BICGSTAB) { RH(q, e) = g; PV(q, e) = g; }
    X(q, e) = zero2();
  });
  csum<C, 1>(g2, sm, par);
  const double rr0 = g2[0];
  const double rn0 = sqrt(rr0);
  int hs = 0, status = TSF_LEVEL_OK;
  double relres = 0.0;
  const SpecOp opA = make_op(P, I, j, OP_A, r, sm);
  const SpecOp opP = make_op(P, I, j, OP_PINV, r, sm);
  const double2 *Y = sm.A;      // output buffer of the last operator application

  if (rr0 > 0.0 && METHOD == TSF_BICGSTAB) {
    double rho = rr0, alpha = 0.0, omega = 0.0, beta = 0.0;
    for (int it = 0;; ++it) {
      // Phase A: p = r + beta (p - omega v); phat = P^{-1} p; v = A phat; r^.v
      for_elems<VPT>(npc, [&](int q, int e) {
        double2 pv;
        if (it == 0) pv = R(q, e);
        else {
          pv = caxpy(beta, caxpy(-omega, VV(q, e), PV(q, e)), R(q, e));
          PV(q, e) = pv;
        }
        sm.A[pidx(e)] = pv;
      });
      __syncthreads();
      Y = prec ? apply<C, true, STG>(sm, P.L1e, gp, opP, tw, r) : sm.A;
      for_elems<VPT>(npc, [&](int q, int e) {
        const double2 ph = Y[pidx(e)];
        PH(q, e) = ph;
        sm.A[pidx(e)] = ph;
        sm.A[pidx(e + npc)] = zero2();
      });
      __syncthreads();
      Y = apply<C, false, STG>(sm, P.L1e, ge, opA, tw, r);
      double d[1] = {0.0};
      for_elems<VPT>(npc, [&](int q, int e) {
        const double2 v = Y[pidx(e)];
        VV(q, e) = v;
        d[0] += cdot(RH(q, e), v);
      });
      csum<C, 1>(d, sm, par);
      if (!(fabs(d[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      alpha = rho / d[0];
      // Phase B: s = r - alpha v; half-step exit on ||s||
      double ss[1] = {0.0};
      for_elems<VPT>(npc, [&](int q, int e) {
        const double2 s = caxpy(-alpha, VV(q, e), R(q, e));
        S(q, e) = s;
        sm.A[pidx(e)] = s;
        ss[0] += cdot(s, s);
      });
      csum<C, 1>(ss, sm, par);
      if (sqrt(ss[0]) < P.tol * rn0) {
        for_elems<VPT>(npc, [&](int q, int e) { X(q, e) = caxpy(alpha, PH(q, e), X(q, e)); });
        hs += 1;
        relres = sqrt(ss[0]) / rn0;
        break;
      }
      //          shat = P^{-1} s; t = A shat; t.s, t.t
      Y = prec ? apply<C, true, STG>(sm, P.L1e, gp, opP, tw, r) : sm.A;
      for_elems<VPT>(npc, [&](int q, int e) {
        const double2 sh = Y[pidx(e)];
        SH(q, e) = sh;
        sm.A[pidx(e)] = sh;
        sm.A[pidx(e + npc)] = zero2();
      });
      __syncthreads();
      Y = apply<C, false, STG>(sm, P.L1e, ge, opA, tw, r);
      double tt[2] = {0.0, 0.0};
      for_elems<VPT>(npc, [&](int q, int e) {
        const double2 t = Y[pidx(e)];
        const double2 s = S(q, e);
        tt[0] += cdot(t, s);
        tt[1] += cdot(t, t);
      });
      csum<C, 2>(tt, sm, par);
      if (!(tt[1] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      omega = tt[0] / tt[1];
      // Phase C: x += alpha phat + omega shat; r = s - omega t; r^.r, r.r
      double rr[2] = {0.0, 0.0};
      for_elems<VPT>(npc, [&](int q, int e) {
        X(q, e) = caxpy(omega, SH(q, e), caxpy(alpha, PH(q, e), X(q, e)));
        const double2 rn = caxpy(-omega, Y[pidx(e)], S(q, e));
        R(q, e) = rn;
        rr[0] += cdot(RH(q, e), rn);
        rr[1] += cdot(rn, rn);
      });
      csum<C, 2>(rr, sm, par);
      hs += 2;
      relres = sqrt(rr[1]) / rn0;
      if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
      if (relres < P.tol) break;
      if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
      if (!(fabs(rr[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      beta = (rr[0] / rho) * (alpha / omega);
      rho = rr[0];
    }
  } else if (rr0 > 0.0 && METHOD == TSF_CGNR) {
    // CGLS on K = A P^{-1} (DESIGN.md R-cgnr): y0 = 0, r = b, z = K^T r, p = z.
    const SpecOp opAT = make_op(P, I, j, OP_AT, r, sm);
    const SpecOp opPT = make_op(P, I, j, OP_PTINV, r, sm);
    // z = P^{-T} (A^T r): A^T on the padded input, then P^{-T} on its first npc values
    auto ktrans = [&]() -> const double2 * {
      const double2 *Z = apply<C, false, STG>(sm, P.L1e, ge, opAT, tw, r);
      if (!prec) return Z;
      if (Z != sm.A) {
        for_elems<VPT>(npc, [&](int, int e) { sm.A[pidx(e)] = Z[pidx(e)]; });
        __syncthreads();
      }
      return apply<C, true, STG>(sm, P.L1e, gp, opPT, tw, r);
    };
    // A[0..npc) holds r = g and A[npc..) is zero (rhs_phase)
    __syncthreads();
    Y = ktrans();
    double gz[1] = {0.0};
    for_elems<VPT>(npc, [&](int q, int e) {
      const double2 z = Y[pidx(e)];
      PV(q, e) = z;
      gz[0] += cdot(z, z);
    });
    csum<C, 1>(gz, sm, par);
    double gam = gz[0];
    double beta = 0.0;
    for (int it = 0;; ++it) {
      // Phase A: p = z + beta p; phat = P^{-1} p; q = A phat; ||q||^2
      for_elems<VPT>(npc, [&](int q, int e) {
        double2 pv;
        if (it == 0) pv = PV(q, e);
        else { pv = caxpy(beta, PV(q, e), Y[pidx(e)]); PV(q, e) = pv; }
        sm.A[pidx(e)] = pv;
      });
      __syncthreads();
      Y = prec ? apply<C, true, STG>(sm, P.L1e, gp, opP, tw, r) : sm.A;
      for_elems<VPT>(npc, [&](int q, int e) {
        const double2 ph = Y[pidx(e)];
        PH(q, e) = ph;
        sm.A[pidx(e)] = ph;
        sm.A[pidx(e + npc)] = zero2();
      });
      __syncthreads();
      Y = apply<C, false, STG>(sm, P.L1e, ge, opA, tw, r);
      double qq[1] = {0.0};
      for_elems<VPT>(npc, [&](int, int e) { qq[0] += cdot(Y[pidx(e)], Y[pidx(e)]); });
      csum<C, 1>(qq, sm, par);
      if (!(qq[0] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      const double a = gam / qq[0];
      // Phase B: x += a phat; r -= a q; ||r||; z = P^{-T} A^T r; ||z||^2
      double rl[1] = {0.0};
      for_elems<VPT>(npc, [&](int q, int e) {
        X(q, e) = caxpy(a, PH(q, e), X(q, e));
        const double2 rn = caxpy(-a, Y[pidx(e)], R(q, e));
        R(q, e) = rn;
        sm.A[pidx(e)] = rn;
        sm.A[pidx(e + npc)] = zero2();
        rl[0] += cdot(rn, rn);
      });
      csum<C, 1>(rl, sm, par);
      hs += 2;
      relres = sqrt(rl[0] / rr0);
      if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
      if (relres < P.tol) break;
      if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
      Y = ktrans();
      double zz[1] = {0.0};
      for_elems<VPT>(npc, [&](int, int e) { zz[0] += cdot(Y[pidx(e)], Y[pidx(e)]); });
      csum<C, 1>(zz, sm, par);
      beta = zz[0] / gam;
      gam = zz[0];
    }
  }
  // finalize (alg1 step 3 result): d^j = u^{j+1} - u^j, u^j <- u^{j+1}
  double2 *Hj = reinterpret_cast<double2 *>(I.hist + j * n) + r * npc;
  for_elems<VPT>(npc, [&](int q, int e) {
    const double2 x = X(q, e), u = U(q, e);
    Hj[e] = csub(x, u);
    U(q, e) = x;
  });
  if (r == 0 && threadIdx.x == 0) {
    I.it[j] = hs;
    I.rr[j] = relres;
    I.st[j] = status;
  }
  __syncthreads();
#ifdef TSF_PROFILE
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    sm.prof[PS_LEVEL] += (unsigned long long)(clock64() - tlev0);
    sm.prof[PS_ITERS] += (unsigned long long)hs;
  }
#endif
}

// ------------------------------------------------------------------------ kernels
template <int C, int METHOD, int VPT, bool STG>
__global__ void __launch_bounds__(kThreads, (C == 1 && VPT == 0) ? 2 : 1)
    k_solve(DevParams P, int32_t nlev, int32_t) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.x / C;
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.prof);
  load_constants(P, I.lwe, P.precond != TSF_NOPREC ? I.lwp : nullptr, sm, r);
  const int npc = P.L1p;
  VecT<VPT> U;
  double2 *Ug = reinterpret_cast<double2 *>(I.vec + V_U * P.n) + r * npc;
  if constexpr (VPT > 0) for_elems<VPT>(npc, [&](int q, int e) { U(q, e) = Ug[e]; });
  else U.p = Ug;
  __syncthreads();
  const int64_t j0 = *P.level;
  for (int64_t j = j0; j < j0 + nlev && j < P.M; ++j) level_solve<C, METHOD, VPT, STG>(P, I, j, sm, r, U);
  if constexpr (VPT > 0) for_elems<VPT>(npc, [&](int q, int e) { Ug[e] = U(q, e); });
}

__global__ void k_advance(int64_t *level, int64_t by, int64_t M);

// Debug: one operator application of instance b at level j: in/out are permuted chunks.
template <int C, bool STG>
__global__ void __launch_bounds__(kThreads, 1) k_debug_apply(DevParams P, int32_t, int b, int64_t j,
                                                              int which, const double *in, double *out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.prof);
  load_constants(P, I.lwe, P.precond != TSF_NOPREC ? I.lwp : nullptr, sm, r);
  const int npc = P.L1p;
  const double2 *X = reinterpret_cast<const double2 *>(in) + r * npc;
  double2 *Y = reinterpret_cast<double2 *>(out) + r * npc;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  const bool embed = which <= OP_AT;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    sm.A[pidx(e)] = X[e];
    if (embed) sm.A[pidx(e + npc)] = zero2();
  }
  __syncthreads();
  const SpecOp op = make_op(P, I, j, which, r, sm);
  const double2 *Z = embed ? apply<C, false, STG>(sm, P.L1e, geo_embed(P, sm), op, tw, r)
                           : apply<C, true, STG>(sm, P.L1e, geo_prec(P, sm), op, tw, r);
  for (int e = threadIdx.x; e < npc; e += kThreads) Y[e] = Z[pidx(e)];
}

// Debug: RHS of the current level for every instance into V_R.
template <int C, bool STG>
__global__ void __launch_bounds__(kThreads, 1) k_debug_rhs(DevParams P, int32_t) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.x / C;
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const Smem sm = smem_view(smem_raw, P.L1e, P.L1p, P.staged != 0, P.resident != 0, P.prof);
  load_constants(P, I.lwe, P.precond != TSF_NOPREC ? I.lwp : nullptr, sm, r);
  const int64_t j = *P.level;
  const int npc = P.L1p;
  __syncthreads();
  if (j >= P.M) return;
  VecT<0> U;
  U.p = reinterpret_cast<double2 *>(I.vec + V_U * P.n) + r * npc;
  rhs_phase<C, 0, STG>(P, I, j, sm, r, U);
  double2 *R = reinterpret_cast<double2 *>(I.vec + V_R * P.n) + r * npc;
  for (int e = threadIdx.x; e < npc; e += kThreads) R[e] = sm.A[pidx(e)];
}

// ------------------------------------------------------------------------ launch API
// Implemented per cluster size in tsf_solve_c<C>.cu (parallel compilation).
template <int C>
cudaError_t launch_solve_c(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st);
template <int C>
cudaError_t launch_dbg_apply_c(const Plan &pl, const DevParams &dp, int b, int64_t j, int which,
                               const double *in, double *out, cudaStream_t st);
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

// Staged exchange (STG) exists for C > 1 only; register-resident vectors (VPT > 0) are
// planned only together with the staged exchange or C == 1.
#define TSF_STG_OF(CC, pl) ((CC) > 1 && (pl).staged)
#define TSF_INSTANTIATE_CLUSTER(CC)                                                             \
  template <>                                                                                   \
  cudaError_t launch_solve_c<CC>(const Plan &pl, const DevParams &dp, int32_t nlev, cudaStream_t st) { \
    const int g = pl.B * CC;                                                                    \
    const int32_t z = 0;                                                                        \
    constexpr bool S1 = (CC) > 1;                                                               \
    if (pl.method == TSF_BICGSTAB) {                                                            \
      if (pl.vpt == 1) return launch_cluster(k_solve<CC, TSF_BICGSTAB, 1, S1>, pl, g, st, dp, nlev, z); \
      if (pl.vpt == 2) return launch_cluster(k_solve<CC, TSF_BICGSTAB, 2, S1>, pl, g, st, dp, nlev, z); \
      if (TSF_STG_OF(CC, pl)) return launch_cluster(k_solve<CC, TSF_BICGSTAB, 0, S1>, pl, g, st, dp, nlev, z); \
      return launch_cluster(k_solve<CC, TSF_BICGSTAB, 0, false>, pl, g, st, dp, nlev, z);       \
    }                                                                                           \
    if (pl.vpt == 1) return launch_cluster(k_solve<CC, TSF_CGNR, 1, S1>, pl, g, st, dp, nlev, z); \
    if (pl.vpt == 2) return launch_cluster(k_solve<CC, TSF_CGNR, 2, S1>, pl, g, st, dp, nlev, z); \
    if (TSF_STG_OF(CC, pl)) return launch_cluster(k_solve<CC, TSF_CGNR, 0, S1>, pl, g, st, dp, nlev, z); \
    return launch_cluster(k_solve<CC, TSF_CGNR, 0, false>, pl, g, st, dp, nlev, z);             \
  }                                                                                             \
  template <>                                                                                   \
  cudaError_t launch_dbg_apply_c<CC>(const Plan &pl, const DevParams &dp, int b, int64_t j,     \
                                     int which, const double *in, double *out, cudaStream_t st) { \
    if (TSF_STG_OF(CC, pl))                                                                     \
      return launch_cluster(k_debug_apply<CC, true>, pl, CC, st, dp, int32_t(0), b, j, which, in, out); \
    return launch_cluster(k_debug_apply<CC, false>, pl, CC, st, dp, int32_t(0), b, j, which, in, out); \
  }                                                                                             \
  template <>                                                                                   \
  cudaError_t launch_dbg_rhs_c<CC>(const Plan &pl, const DevParams &dp, cudaStream_t st) {      \
    if (TSF_STG_OF(CC, pl)) return launch_cluster(k_debug_rhs<CC, true>, pl, pl.B * CC, st, dp, int32_t(0)); \
    return launch_cluster(k_debug_rhs<CC, false>, pl, pl.B * CC, st, dp, int32_t(0));           \
  }

}  // namespace tsf
