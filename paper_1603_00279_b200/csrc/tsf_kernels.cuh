// tsf_kernels.cuh -- sm_100a FP64 device code of the per-level Toeplitz Krylov solver.
//
// One thread-block cluster of C CTAs owns one problem instance for a whole level (or for
// the whole run).  Per level (alg1):
//   RHS   g = B u^j - kappa sum_s c_{j-s} d^s + f^{j+sigma}          (eq3.1)
//   Krylov solve A u^{j+1} = g, right-preconditioned BiCGSTAB or CGNR (CGLS on A P^{-1})
//   finalize d^j = u^{j+1} - u^j (history), u^j <- u^{j+1}, per-level stats.
// A, B are applied through the 2n circulant embedding of their Toeplitz generators (P:765-767,
// P:775-776) and the preconditioner is a circulant solve; both are FFT
// -> per-bin spectral op -> inverse FFT fused in shared memory:
//   * the n real unknowns of a CTA are packed as n/(2C) complex values (real-FFT packing);
//   * length-L complex transforms (L = n: embedding, L = n/2: preconditioner) use a
//     four-step split L = C * L1: a local radix-4/2 FFT of length L1 per CTA in SMEM,
//     a length-C DFT across the cluster through distributed shared memory, the per-bin
//     real-split + spectral scaling in registers, and the transposed path back;
//   * the per-level spectra are formed on the fly from one-time base spectra
//     (lambda = eta + mu (c Lambda_Q + p Lambda_W + q conj Lambda_W)).
// Reductions are deterministic (fixed-order warp shuffles, CTA, then cluster).
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

// Deterministic cluster-wide sum of NV scalars: warp butterflies (exactly commutative, so
// every lane holds the same bits) -> 8 warps in order -> C CTAs in rank order.
template <int C, int NV>
__device__ __forceinline__ void csum(double (&v)[NV], double *wred, double *cred, int &par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) wred[warp * 4 + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += wred[w * 4 + k];
      cred[par * 4 + k] = s;
    }
  }
  csync<C>();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < C; ++q) s += remote<C>(cred, q)[par * 4 + k];
    v[k] = s;
  }
  par ^= 1;
}

// ------------------------------------------------------------------------ local FFT (SMEM)
// Plan (DESIGN.md R-fft): DIT stages s = 0..S-1 with radix 4 (s < floor(l/2)) and a final
// radix 2 when l = log2(L1) is odd; m_s = prod_{t<=s} r_t.  The forward transform runs the
// transposed stages (DIF, S-1..0) in place: natural input -> slot order, slot p holding
// X[perm[p]] with perm the gather digit reversal.  The inverse runs the conjugated DIT stages
// 0..S-1 in place: slot order -> natural order (unnormalized).  Twiddles W_m^{kq} come from
// the table tw[e] = exp(-2 pi i e / twN).
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

template <bool INV>
__device__ __forceinline__ void fft_stage(double2 *A, int L1, int lm, int radix,
                                          const double2 *__restrict__ tw, int twN) {
  // lm = log2(m_s); radix 4 or 2; mprev = m_s / radix
  const int lmp = lm - (radix == 4 ? 2 : 1);
  const int mprev = 1 << lmp;
  const int tstep = twN >> lm;                 // W_m^x = tw[x * twN/m]
  const int nb = L1 / radix;
  for (int b = threadIdx.x; b < nb; b += kThreads) {
    const int k = b & (mprev - 1);
    const int base = ((b >> lmp) << lm) + k;
    if (radix == 4) {
      double2 a0 = A[base], a1 = A[base + mprev], a2 = A[base + 2 * mprev], a3 = A[base + 3 * mprev];
      if (k != 0) {
        const double2 w1 = tw[k * tstep], w2 = tw[2 * k * tstep], w3 = tw[3 * k * tstep];
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
      A[base] = a0; A[base + mprev] = a1; A[base + 2 * mprev] = a2; A[base + 3 * mprev] = a3;
    } else {
      double2 a0 = A[base], a1 = A[base + mprev];
      const double2 w = tw[k * tstep];
      if (INV) {
        a1 = cmulc(a1, w);
        A[base] = cadd(a0, a1); A[base + mprev] = csub(a0, a1);
      } else {
        A[base] = cadd(a0, a1); A[base + mprev] = cmul(csub(a0, a1), w);
      }
    }
  }
}

// Requires the input to be visible to all threads (caller synchronizes); ends synchronized.
template <bool INV>
__device__ __noinline__ void local_fft(double2 *A, int L1, const double2 *__restrict__ tw, int twN) {
  const int l = __ffs(L1) - 1;
  const int S4 = l >> 1;
  const bool r2 = l & 1;
  const int S = S4 + (r2 ? 1 : 0);
  if (!INV) {
    for (int s = S - 1; s >= 0; --s) {
      if (r2 && s == S - 1) fft_stage<false>(A, L1, l, 2, tw, twN);
      else fft_stage<false>(A, L1, 2 * (s + 1), 4, tw, twN);
      __syncthreads();
    }
  } else {
    for (int s = 0; s < S; ++s) {
      if (r2 && s == S - 1) fft_stage<true>(A, L1, l, 2, tw, twN);
      else fft_stage<true>(A, L1, 2 * (s + 1), 4, tw, twN);
      __syncthreads();
    }
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
  const double2 *lam;   // task-order base spectrum of this instance
  const double *sq;     // task-order sine table
  double2 nyq;          // base spectrum at the Nyquist bin L
  int np;               // column-pair tasks per CTA
  int rC;               // r * C
  double eta, mu, ppq, pmq, c2, qcorr, scale;
  bool conj;
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
};

// C == 1: the whole transform is local; column pairs are bin pairs (k, L-k).
template <bool DIV>
__device__ __noinline__ void pointwise_local(double2 *A, const Geo &g, const SpecOp &op,
                                                const double2 *__restrict__ tw) {
  for (int i = threadIdx.x; i < g.np; i += kThreads) {
    if (i == 0) {
      const int sa = g.slot[0], sb = g.slot[g.L1 / 2];
      double2 a = A[sa], b = A[sb];
      pair_self<DIV>(a, op.get(0, 0, 0, 0), op.nyquist(g.L), tw[0], op.scale);
      const double2 lm = op.get(0, 1, 0, g.L / 2);
      pair_self<DIV>(b, lm, lm, tw[(g.L / 2) * g.tw2L], op.scale);
      A[sa] = a; A[sb] = b;
    } else {
      const int sa = g.slot[i], sb = g.slot[g.L1 - i];
      double2 a = A[sa], b = A[sb];
      pair_apply<DIV>(a, b, op.get(0, 0, i, i), op.get(0, 1, i, g.L - i), tw[i * g.tw2L], op.scale);
      A[sa] = a; A[sb] = b;
    }
  }
}

// C > 1: gather the C partial transforms of column pair (k1a, k1b) through DSMEM, finish the
// four-step transform with a length-C DFT, apply the spectral op, undo, scatter back.
template <int C, bool DIV>
__device__ __noinline__ void cross_step(double2 *A, const Geo &g, const SpecOp &op,
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
    sa = g.slot[k1a];
    sb = g.slot[k1b];
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
    // za[k2] = Z[k1a + L1 k2], zb[k2] = Z[k1b + L1 k2]
    if (!pseudo) {
#pragma unroll
      for (int k2 = 0; k2 < C; ++k2) {
        const int bin = k1a + g.L1 * k2;
        pair_apply<DIV>(za[k2], zb[C - 1 - k2], op.get(k2, 0, i, bin),
                        op.get(C - 1 - k2, 1, i, g.L - bin), tw[bin * g.tw2L], op.scale);
      }
    } else {
      // column 0: bins L1 k2 paired with L1 (C - k2) (k2 = 0 pairs with the Nyquist bin)
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
      // column L1/2: bins L1/2 + L1 k2 paired with L1/2 + L1 (C-1-k2)
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
  csync<C>();                    // every gather done before any scatter overwrites
  if (act) {
#pragma unroll
    for (int q = 0; q < C; ++q) {
      double2 *Aq = remote<C>(A, uint32_t(q));
      Aq[sa] = za[q];
      Aq[sb] = zb[q];
    }
  }
  csync<C>();                    // scatters landed
}

// y = op(x) for the CTA's local data already in A[0..L1) (natural order, visible).
// On return A[0..L1) holds this CTA's part of the result (natural order, visible).
template <int C, bool DIV>
__device__ __noinline__ void apply(double2 *A, const Geo &g, const SpecOp &op,
                                      const double2 *__restrict__ tw, int twN, uint32_t r) {
  local_fft<false>(A, g.L1, tw, twN);
  if constexpr (C == 1) {
    pointwise_local<DIV>(A, g, op, tw);
    __syncthreads();
  } else {
    csync<C>();                  // every local transform done before remote gathers
    cross_step<C, DIV>(A, g, op, tw, r);
  }
  local_fft<true>(A, g.L1, tw, twN);
}

// ------------------------------------------------------------------------ operator setup
enum Which { OP_A = 0, OP_B = 1, OP_AT = 2, OP_PINV = 3, OP_PTINV = 4 };

__device__ __forceinline__ Geo geo_embed(const DevParams &P) {
  Geo g;
  g.L1 = P.L1e; g.L = int(P.n); g.np = P.npe; g.twL = P.twN / int(P.n); g.tw2L = P.twN / int(2 * P.n);
  g.slot = P.slot_e;
  return g;
}
__device__ __forceinline__ Geo geo_prec(const DevParams &P) {
  Geo g;
  g.L1 = P.L1p; g.L = int(P.n / 2); g.np = P.npp; g.twL = P.twN / int(P.n / 2); g.tw2L = P.twN / int(P.n);
  g.slot = P.slot_p;
  return g;
}

// Level-j operator: which in {A, B, A^T} uses the embedding spectrum, {P^-1, P^-T} the
// preconditioner spectrum.  A = eta I - sigma L_j, B = eta I + (1-sigma) L_j (eq3.3), P the
// circulant of (preku) with s(.) replaced by the chosen circulant approximation.
__device__ __forceinline__ SpecOp make_op(const DevParams &P, const Inst &I, int64_t j, int which,
                                          uint32_t r) {
  const double *lv = I.lev + 4 * j;
  const double eta = lv[0], c = lv[1], p = lv[2], q = lv[3];
  const double sigma = I.par[0];
  SpecOp op;
  op.rC = int(r) * P.C;
  op.eta = eta;
  op.ppq = p + q;
  op.pmq = p - q;
  if (which <= OP_AT) {
    op.lam = I.lwe; op.sq = P.sq_e; op.np = P.npe; op.nyq = I.lwe[P.n];
    op.mu = (which == OP_B) ? (1.0 - sigma) : -sigma;
    op.c2 = 2.0 * c;
    op.qcorr = 0.0;
    op.scale = P.scale_e;
    op.conj = (which == OP_AT);
  } else {
    op.lam = I.lwp; op.sq = P.sq_p; op.np = P.npp; op.nyq = I.lwp[P.n / 2];
    op.mu = -sigma;
    op.c2 = 2.0 * c * P.qscale_p;
    op.qcorr = P.strang ? -q * I.par[2] : 0.0;   // Strang s(W^T) midpoint fix (R-strang)
    op.scale = P.scale_p;
    op.conj = (which == OP_PTINV);
  }
  return op;
}

// ------------------------------------------------------------------------ shared memory
struct Smem {
  double2 *A;
  double *wred, *cred;
};
__device__ __forceinline__ Smem smem_view(unsigned char *raw, int L1e) {
  Smem s;
  s.A = reinterpret_cast<double2 *>(raw);
  s.wred = reinterpret_cast<double *>(s.A + L1e);
  s.cred = s.wred + 32;
  return s;
}

// ------------------------------------------------------------------------ RHS (alg1 step 2)
// g = B u^j - [kappa e_j d^0 + sum_{s=1}^{j-1} kappa chat_{j-s} d^s] + f^{j+sigma}
// writes g to R (and RH, P for BiCGSTAB), zeroes X; returns the local partial ||g||^2.
template <int C>
__device__ __noinline__ double rhs_phase(const DevParams &P, const Inst &I, int64_t j, const Smem &sm, uint32_t r,
                            bool bicg) {
  const int npc = P.L1p;
  const int64_t n = P.n;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  double2 *U = reinterpret_cast<double2 *>(I.vec + V_U * n) + r * npc;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    sm.A[e] = U[e];
    sm.A[e + npc] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const SpecOp opB = make_op(P, I, j, OP_B, r);
  apply<C, false>(sm.A, geo_embed(P), opB, tw, P.twN, r);
  double2 *R = reinterpret_cast<double2 *>(I.vec + V_R * n) + r * npc;
  double2 *RH = reinterpret_cast<double2 *>(I.vec + V_RH * n) + r * npc;
  double2 *PV = reinterpret_cast<double2 *>(I.vec + V_P * n) + r * npc;
  double2 *X = reinterpret_cast<double2 *>(I.vec + V_X * n) + r * npc;
  const double2 *H = reinterpret_cast<const double2 *>(I.hist) + r * npc;
  const int64_t hstride = n / 2;  // double2 per history row
  double acc = 0.0;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    double2 g = sm.A[e];
    if (j >= 1) {
      double2 h0 = cscale(H[e], I.hwe[j]);
      double2 h1 = make_double2(0.0, 0.0), h2 = h1, h3 = h1;
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
    R[e] = g;
    if (bicg) { RH[e] = g; PV[e] = g; }
    X[e] = make_double2(0.0, 0.0);
    acc += cdot(g, g);
  }
  return acc;
}

// ------------------------------------------------------------------------ one level
// Returns through the stats arrays; all control flow is uniform over the cluster.
template <int C, int METHOD>
__device__ void level_solve(const DevParams &P, const Inst &I, int64_t j, const Smem &sm, uint32_t r) {
  const int npc = P.L1p;
  const int64_t n = P.n;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  auto vec = [&](int v) { return reinterpret_cast<double2 *>(I.vec + v * n) + r * npc; };
  double2 *X = vec(V_X), *R = vec(V_R), *RH = vec(V_RH), *PV = vec(V_P), *VV = vec(V_V);
  double2 *S = vec(V_S), *PH = vec(V_PH), *SH = vec(V_SH);
  const bool prec = P.precond != TSF_NOPREC;
  const Geo ge = geo_embed(P), gp = geo_prec(P);
  int par = 0;

  double g2[1] = {rhs_phase<C>(P, I, j, sm, r, METHOD == TSF_BICGSTAB)};
  csum<C, 1>(g2, sm.wred, sm.cred, par);
  const double rr0 = g2[0];
  const double rn0 = sqrt(rr0);
  int hs = 0, status = TSF_LEVEL_OK;
  double relres = 0.0;
  const SpecOp opA = make_op(P, I, j, OP_A, r);
  const SpecOp opP = make_op(P, I, j, OP_PINV, r);

  if (rr0 > 0.0 && METHOD == TSF_BICGSTAB) {
    double rho = rr0, alpha = 0.0, omega = 0.0, beta = 0.0;
    for (int it = 0;; ++it) {
      // Phase A: p = r + beta (p - omega v); phat = P^{-1} p; v = A phat; r^.v
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        double2 pv;
        if (it == 0) pv = R[e];
        else {
          pv = caxpy(beta, caxpy(-omega, VV[e], PV[e]), R[e]);
          PV[e] = pv;
        }
        sm.A[e] = pv;
      }
      __syncthreads();
      if (prec) apply<C, true>(sm.A, gp, opP, tw, P.twN, r);
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        PH[e] = sm.A[e];
        sm.A[e + npc] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      apply<C, false>(sm.A, ge, opA, tw, P.twN, r);
      double d[1] = {0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        const double2 v = sm.A[e];
        VV[e] = v;
        d[0] += cdot(RH[e], v);
      }
      csum<C, 1>(d, sm.wred, sm.cred, par);
      if (!(fabs(d[0]) > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      alpha = rho / d[0];
      // Phase B: s = r - alpha v; half-step exit on ||s||
      double ss[1] = {0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        const double2 s = caxpy(-alpha, sm.A[e], R[e]);
        S[e] = s;
        sm.A[e] = s;
        ss[0] += cdot(s, s);
      }
      csum<C, 1>(ss, sm.wred, sm.cred, par);
      if (sqrt(ss[0]) < P.tol * rn0) {
        for (int e = threadIdx.x; e < npc; e += kThreads) X[e] = caxpy(alpha, PH[e], X[e]);
        hs += 1;
        relres = sqrt(ss[0]) / rn0;
        break;
      }
      //          shat = P^{-1} s; t = A shat; t.s, t.t
      if (prec) apply<C, true>(sm.A, gp, opP, tw, P.twN, r);
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        SH[e] = sm.A[e];
        sm.A[e + npc] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      apply<C, false>(sm.A, ge, opA, tw, P.twN, r);
      double tt[2] = {0.0, 0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        const double2 t = sm.A[e];
        const double2 s = S[e];
        tt[0] += cdot(t, s);
        tt[1] += cdot(t, t);
      }
      csum<C, 2>(tt, sm.wred, sm.cred, par);
      if (!(tt[1] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      omega = tt[0] / tt[1];
      // Phase C: x += alpha phat + omega shat; r = s - omega t; r^.r, r.r
      double rr[2] = {0.0, 0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        X[e] = caxpy(omega, SH[e], caxpy(alpha, PH[e], X[e]));
        const double2 rn = caxpy(-omega, sm.A[e], S[e]);
        R[e] = rn;
        rr[0] += cdot(RH[e], rn);
        rr[1] += cdot(rn, rn);
      }
      csum<C, 2>(rr, sm.wred, sm.cred, par);
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
    const SpecOp opAT = make_op(P, I, j, OP_AT, r);
    const SpecOp opPT = make_op(P, I, j, OP_PTINV, r);
    double2 *Q = VV;
    for (int e = threadIdx.x; e < npc; e += kThreads) {
      sm.A[e] = R[e];
      sm.A[e + npc] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    apply<C, false>(sm.A, ge, opAT, tw, P.twN, r);
    if (prec) apply<C, true>(sm.A, gp, opPT, tw, P.twN, r);
    double gz[1] = {0.0};
    for (int e = threadIdx.x; e < npc; e += kThreads) {
      const double2 z = sm.A[e];
      PV[e] = z;
      gz[0] += cdot(z, z);
    }
    csum<C, 1>(gz, sm.wred, sm.cred, par);
    double gam = gz[0];
    double beta = 0.0;
    for (int it = 0;; ++it) {
      // Phase A: p = z + beta p; phat = P^{-1} p; q = A phat; ||q||^2
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        double2 pv;
        if (it == 0) pv = PV[e];
        else { pv = caxpy(beta, PV[e], sm.A[e]); PV[e] = pv; }
        sm.A[e] = pv;
      }
      __syncthreads();
      if (prec) apply<C, true>(sm.A, gp, opP, tw, P.twN, r);
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        PH[e] = sm.A[e];
        sm.A[e + npc] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      apply<C, false>(sm.A, ge, opA, tw, P.twN, r);
      double qq[1] = {0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        const double2 q = sm.A[e];
        Q[e] = q;
        qq[0] += cdot(q, q);
      }
      csum<C, 1>(qq, sm.wred, sm.cred, par);
      if (!(qq[0] > 1e-300)) { status = TSF_LEVEL_BREAKDOWN; break; }
      const double a = gam / qq[0];
      // Phase B: x += a phat; r -= a q; ||r||; z = P^{-T} A^T r; ||z||^2
      double rl[1] = {0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) {
        X[e] = caxpy(a, PH[e], X[e]);
        const double2 rn = caxpy(-a, sm.A[e], R[e]);
        R[e] = rn;
        sm.A[e] = rn;
        sm.A[e + npc] = make_double2(0.0, 0.0);
        rl[0] += cdot(rn, rn);
      }
      csum<C, 1>(rl, sm.wred, sm.cred, par);
      hs += 2;
      relres = sqrt(rl[0] / rr0);
      if (!isfinite(relres)) { status = TSF_LEVEL_DIVERGED; break; }
      if (relres < P.tol) break;
      if (hs >= 2 * P.maxit) { status = TSF_LEVEL_MAXIT; break; }
      apply<C, false>(sm.A, ge, opAT, tw, P.twN, r);
      if (prec) apply<C, true>(sm.A, gp, opPT, tw, P.twN, r);
      double zz[1] = {0.0};
      for (int e = threadIdx.x; e < npc; e += kThreads) zz[0] += cdot(sm.A[e], sm.A[e]);
      csum<C, 1>(zz, sm.wred, sm.cred, par);
      beta = zz[0] / gam;
      gam = zz[0];
    }
  }
  // finalize (alg1 step 3 result): d^j = u^{j+1} - u^j, u^j <- u^{j+1}
  double2 *U = vec(V_U);
  double2 *Hj = reinterpret_cast<double2 *>(I.hist + j * n) + r * npc;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    const double2 x = X[e], u = U[e];
    Hj[e] = csub(x, u);
    U[e] = x;
  }
  if (r == 0 && threadIdx.x == 0) {
    I.it[j] = hs;
    I.rr[j] = relres;
    I.st[j] = status;
  }
  __syncthreads();
}

// ------------------------------------------------------------------------ kernels
template <int C, int METHOD>
__global__ void __launch_bounds__(kThreads, 1) k_solve(DevParams P, int32_t nlev) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem sm = smem_view(smem_raw, P.L1e);
  const int b = blockIdx.x / C;
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const int64_t j0 = *P.level;
  for (int64_t j = j0; j < j0 + nlev && j < P.M; ++j) level_solve<C, METHOD>(P, I, j, sm, r);
}

__global__ void k_advance(int64_t *level, int64_t by, int64_t M) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t v = *level + by;
    *level = v < M ? v : M;
  }
}

// Debug: one operator application of instance b at level j: in/out are permuted chunks.
template <int C>
__global__ void __launch_bounds__(kThreads, 1) k_debug_apply(DevParams P, int b, int64_t j, int which,
                                                              const double *in, double *out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem sm = smem_view(smem_raw, P.L1e);
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const int npc = P.L1p;
  const double2 *X = reinterpret_cast<const double2 *>(in) + r * npc;
  double2 *Y = reinterpret_cast<double2 *>(out) + r * npc;
  const double2 *__restrict__ tw = reinterpret_cast<const double2 *>(P.tw);
  const bool embed = which <= OP_AT;
  for (int e = threadIdx.x; e < npc; e += kThreads) {
    sm.A[e] = X[e];
    if (embed) sm.A[e + npc] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const SpecOp op = make_op(P, I, j, which, r);
  if (embed) apply<C, false>(sm.A, geo_embed(P), op, tw, P.twN, r);
  else apply<C, true>(sm.A, geo_prec(P), op, tw, P.twN, r);
  for (int e = threadIdx.x; e < npc; e += kThreads) Y[e] = sm.A[e];
}

// Debug: RHS of the current level for every instance into V_R.
template <int C>
__global__ void __launch_bounds__(kThreads, 1) k_debug_rhs(DevParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem sm = smem_view(smem_raw, P.L1e);
  const int b = blockIdx.x / C;
  const uint32_t r = crank<C>();
  const Inst I = inst_view(P, b);
  const int64_t j = *P.level;
  if (j < P.M) rhs_phase<C>(P, I, j, sm, r, false);
}

}  // namespace tsf
