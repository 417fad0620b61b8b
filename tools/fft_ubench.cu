// Microbenchmark of the in-SMEM local FFT (developer tool): cycles per forward+inverse pair
// for the library's local_fft and experimental variants, 1 CTA x 256 threads, direct twiddle
// table in SMEM (the resident mode of the cluster kernels).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I. tools/fft_ubench.cu -o tools/fft_ubench.bin
#include <cstdio>
#include <vector>

#include "../paper_1603_00279_b200/csrc/tsf_kernels.cuh"

using namespace tsf;

// ---- experimental: compile-time radix-4 stages, branch-free twiddles ----------------------
template <bool INV, int LM, int TW>   // stage with m = 2^LM (radix 4); TW 0: 3 table loads, 1: w1 + derive
__device__ __forceinline__ void st4(double2 *A, int L1, const double2 *twd, int L1e) {
  constexpr int lmp = LM - 2, mprev = 1 << lmp;
  const int tstep = L1e >> LM;
  const int nb = L1 >> 2;
  for (int b = threadIdx.x; b < nb; b += kThreads) {
    const int k = b & (mprev - 1);
    const int base = ((b >> lmp) << LM) + k;
    const int p0 = pidx(base), p1 = pidx(base + mprev), p2 = pidx(base + 2 * mprev), p3 = pidx(base + 3 * mprev);
    double2 a0 = A[p0], a1 = A[p1], a2 = A[p2], a3 = A[p3];
    double2 w1, w2, w3;
    if constexpr (TW == 0) { w1 = twd[k * tstep]; w2 = twd[2 * k * tstep]; w3 = twd[3 * k * tstep]; }
    else { w1 = twd[k * tstep]; w2 = cmul(w1, w1); w3 = cmul(w2, w1); }
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

template <bool INV, int L, int TW>
__device__ __forceinline__ void fft_ct(double2 *A, const double2 *twd) {
  constexpr int l = __builtin_ctz(L), S4 = l / 2;
  constexpr bool r2 = l & 1;
  if constexpr (!INV) {
    if constexpr (r2) {
      const int mprev = L / 2;
      for (int b = threadIdx.x; b < L / 2; b += kThreads) {
        const int p0 = pidx(b), p1 = pidx(b + mprev);
        const double2 a0 = A[p0], a1 = A[p1];
        const double2 w = twd[b];
        A[p0] = cadd(a0, a1); A[p1] = cmul(csub(a0, a1), w);
      }
      __syncthreads();
    }
    [&]<int... I>(std::integer_sequence<int, I...>) {
      ((st4<false, 2 * (S4 - I), TW>(A, L, twd, L), __syncthreads()), ...);
    }(std::make_integer_sequence<int, S4>{});
  } else {
    [&]<int... I>(std::integer_sequence<int, I...>) {
      ((st4<true, 2 * (I + 1), TW>(A, L, twd, L), __syncthreads()), ...);
    }(std::make_integer_sequence<int, S4>{});
    if constexpr (r2) {
      const int mprev = L / 2;
      for (int b = threadIdx.x; b < L / 2; b += kThreads) {
        const int p0 = pidx(b), p1 = pidx(b + mprev);
        const double2 a0 = A[p0];
        const double2 a1 = cmulc(A[p1], twd[b]);
        A[p0] = cadd(a0, a1); A[p1] = csub(a0, a1);
      }
      __syncthreads();
    }
  }
}

template <int L, int MODE>
__global__ void k_bench(double2 *buf, const double2 *tw, int reps, long long *cyc) {
  extern __shared__ __align__(16) unsigned char raw[];
  const Smem sm = smem_view(raw, L, L / 2, false, true, false, nullptr, 16 * kThreads);
  for (int i = threadIdx.x; i < L; i += kThreads) { sm.twd[i] = tw[i]; sm.A[pidx(i)] = buf[i]; }
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if constexpr (MODE == 0) {
      local_fft<false>(sm.A, L, sm, L);
      local_fft<true>(sm.A, L, sm, L);
    } else if constexpr (MODE == 3) {
      Smem s2 = sm; s2.fuse_min = 256;
      local_fft<false>(sm.A, L, s2, L);
      local_fft<true>(sm.A, L, s2, L);
    } else {
      fft_ct<false, L, MODE - 1>(sm.A, sm.twd);
      fft_ct<true, L, MODE - 1>(sm.A, sm.twd);
    }
  }
  const long long t1 = clock64();
  for (int i = threadIdx.x; i < L; i += kThreads) buf[i] = sm.A[pidx(i)];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int L>
void run(double2 *dbuf, double2 *dtw, long long *dc) {
  std::vector<double2> h(L), out[4];
  for (int i = 0; i < L; ++i) h[i] = make_double2(std::sin(0.37 * i), std::cos(1.3 * i));
  std::vector<double2> tw(L);
  for (int i = 0; i < L; ++i) { double s, c; sincospi(-2.0 * i / L, &s, &c); tw[i] = make_double2(c, s); }
  cudaMemcpy(dtw, tw.data(), L * 16, cudaMemcpyHostToDevice);
  const size_t dsm = 2 * L * 16 + 8192;
  long long cyc[4];
  void (*ks[4])(double2 *, const double2 *, int, long long *) = {k_bench<L, 0>, k_bench<L, 1>, k_bench<L, 2>, k_bench<L, 3>};
  for (int mode = 0; mode < 4; ++mode) {
    out[mode].resize(L);
    cudaMemcpy(dbuf, h.data(), L * 16, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(ks[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, int(dsm));
    ks[mode]<<<1, kThreads, dsm>>>(dbuf, dtw, 1, dc);
    cudaMemcpy(out[mode].data(), dbuf, L * 16, cudaMemcpyDeviceToHost);
    ks[mode]<<<1, kThreads, dsm>>>(dbuf, dtw, 200, dc);
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc[mode], dc, 8, cudaMemcpyDeviceToHost);
  }
  double md[4] = {0, 0, 0, 0};
  for (int m = 1; m < 4; ++m)
    for (int i = 0; i < L; ++i) md[m] = fmax(md[m], fabs(out[0][i].x - out[m][i].x) + fabs(out[0][i].y - out[m][i].y));
  printf("L=%5d cyc/(fwd+inv): library %6.0f | ct 3-LDS %6.0f | ct w1+derive %6.0f (diff %.1e) | radix-16 %6.0f (diff %.1e)  %s\n",
         L, cyc[0] / 200.0, cyc[1] / 200.0, cyc[2] / 200.0, md[2] / L, cyc[3] / 200.0, md[3] / L,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2 *dbuf, *dtw;
  long long *dc;
  cudaMalloc(&dbuf, 8192 * 16);
  cudaMalloc(&dtw, 8192 * 16);
  cudaMalloc(&dc, 8);
  run<256>(dbuf, dtw, dc);
  run<512>(dbuf, dtw, dc);
  run<1024>(dbuf, dtw, dc);
  run<2048>(dbuf, dtw, dc);
  run<4096>(dbuf, dtw, dc);
  return 0;
}
