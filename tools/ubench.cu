// Microbenchmarks of the B200 features the per-level solver leans on (FP64 pipe, SMEM,
// barriers, DSMEM).  Developer tool: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/ubench.cu -o /tmp/ubench && /tmp/ubench
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_dfma_lat(double *out, long long *cyc, int iters) {
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dadd_lat(double *out, long long *cyc, int iters) {
  double a = out[threadIdx.x], c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = a + c; a = a + c; a = a + c; a = a + c; }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void k_dfma_tput(double *out, long long *cyc, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = out[threadIdx.x] + k;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// SMEM: LDS.128 dependent latency and bandwidth (double2 per lane)
__global__ void k_lds(double *out, long long *cyc, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2((i * 7 + 1) & 2047, 0.5);
  __syncthreads();
  // latency: pointer chase (one warp)
  if (threadIdx.x < 32) {
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) p = int(buf[p].x);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = p; }
  }
  __syncthreads();
  // bandwidth: all threads, 4 independent LDS.128 per iteration
  double2 acc = make_double2(0, 0);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int base = (threadIdx.x + i * 64) & 2047;
#pragma unroll
    for (int k = 0; k < 4; ++k) { double2 v = buf[(base + k * 512) & 2047]; acc.x += v.x; acc.y += v.y; }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  out[1 + threadIdx.x] = acc.x + acc.y;
}
__global__ void k_bar(long long *cyc, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_cbar(long long *cyc, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) cyc[0] = t1 - t0;
}
// barrier.cluster.arrive.relaxed + wait (no fence)
__global__ void k_cbar_relaxed(long long *cyc, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) cyc[0] = t1 - t0;
}
// DSMEM read bandwidth: every CTA reads a 16 KB slab from every other CTA
__global__ void k_dsmem(double *out, long long *cyc, int iters) {
  __shared__ double2 buf[1024];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i, cl.block_rank());
  cl.sync();
  const int C = cl.num_blocks();
  double2 acc = make_double2(0, 0);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int u = threadIdx.x; u < 1024; u += blockDim.x) {
      const int q = u / (1024 / C);
      const double2 *rb = cl.map_shared_rank(buf, q);
      double2 v = rb[(u * 5 + it) & 1023];
      acc.x += v.x; acc.y += v.y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc.x + acc.y;
}

// All-to-all exchange of a 1024-complex (16 KB) chunk per CTA inside a cluster of C CTAs:
// CTA r sends piece q (1024/C values) to CTA q.  mode 0: DSMEM pull (ld remote) after
// cluster.sync; 1: DSMEM push (st remote) then cluster.sync; 2: global st.cg, relaxed arrive
// after fence.acq_rel.cluster, wait, then ld.global.cg; 3: global st.cg + cluster.sync + ld.cg.
__global__ void k_xchg(double2 *gbuf, long long *cyc, int iters, int mode) {
  __shared__ double2 src[1024];
  __shared__ double2 dst[1024];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks();
  const unsigned r = cl.block_rank();
  const int piece = 1024 / C;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) src[i] = make_double2(i, r);
  double2 *G = gbuf + size_t(blockIdx.x / C) * C * 1024;   // [dst q][src r][piece]
  cl.sync();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      cl.sync();
#pragma unroll 4
      for (int u = threadIdx.x; u < 1024; u += blockDim.x) {
        const int q = u / piece, k = u - q * piece;
        dst[u] = cl.map_shared_rank(src, q)[r * piece + k];
      }
      __syncthreads();
    } else if (mode == 1) {
#pragma unroll 4
      for (int u = threadIdx.x; u < 1024; u += blockDim.x) {
        const int q = u / piece, k = u - q * piece;
        cl.map_shared_rank(dst, q)[r * piece + k] = src[u];
      }
      cl.sync();
    } else {
#pragma unroll 4
      for (int u = threadIdx.x; u < 1024; u += blockDim.x) {
        const int q = u / piece, k = u - q * piece;
        __stcg(G + (size_t(q) * C + r) * piece + k, src[u]);
      }
      if (mode == 2) {
        asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
      } else {
        cl.sync();
      }
#pragma unroll 4
      for (int u = threadIdx.x; u < 1024; u += blockDim.x) dst[u] = __ldcg(G + size_t(r) * 1024 + u);
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) cyc[0] = t1 - t0;
  cl.sync();
  if (threadIdx.x == 0) gbuf[size_t(gridDim.x) * 1024 + blockIdx.x].x = dst[5].x + dst[700].y;
}


__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *m, uint32_t bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" :: "r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1; @!p bra W; }"
               :: "r"(smem_u32(m)), "r"(parity) : "memory");
}
// mode 0: cp.async.bulk per destination piece; mode 1: st.async.v2.f64 per element
__global__ void k_xasync(long long *cyc, int iters, int mode) {
  __shared__ __align__(128) double2 src[1024 - 8];
  __shared__ __align__(128) double2 dst[2][1024];
  __shared__ uint64_t mb[2];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks();
  const unsigned r = cl.block_rank();
  const int piece = 1024 / C;
  for (int i = threadIdx.x; i < 1016; i += blockDim.x) src[i] = make_double2(i, r);
  if (threadIdx.x == 0) { mbar_init(&mb[0], 1); mbar_init(&mb[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cl.sync();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    const uint32_t par = (it >> 1) & 1;
    if (threadIdx.x == 0) mbar_expect(&mb[b], 1024 * 16);
    if (mode == 0) {
      if (threadIdx.x < C) {
        const int q = threadIdx.x;
        const uint32_t d = mapa(smem_u32(&dst[b][r * piece]), q);
        const uint32_t m = mapa(smem_u32(&mb[b]), q);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(d), "r"(smem_u32(&src[(q * piece) % 1008])), "r"(piece * 16 > 1008 * 16 ? 1008 * 16 : piece * 16), "r"(m) : "memory");
      }
    } else {
      for (int u = threadIdx.x; u < 1024; u += blockDim.x) {
        const int q = u / piece, k = u - q * piece;
        const uint32_t d = mapa(smem_u32(&dst[b][r * piece + k]), q);
        const uint32_t m = mapa(smem_u32(&mb[b]), q);
        const double2 v = src[u % 1016];
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                     :: "r"(d), "d"(v.x), "d"(v.y), "r"(m) : "memory");
      }
    }
    mbar_wait(&mb[b], par);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) cyc[0] = t1 - t0;
  cl.sync();
  if (threadIdx.x == 0 && dst[0][5].y < -1) cyc[1] = 1;
}

template <class K, class... A>
int launch_cluster(K k, int grid, int block, int C, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(block);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return cudaLaunchKernelEx(&cfg, k, a...) == cudaSuccess ? 0 : 1;
}

int main() {
  double *d; long long *c; long long h[256];
  CK(cudaMalloc(&d, 1 << 20)); CK(cudaMemset(d, 0, 1 << 20));
  CK(cudaMalloc(&c, 4096)); CK(cudaMemset(c, 0, 4096));
  const int it = 4096;
  k_dfma_lat<<<1, 32>>>(d, c, it); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
  printf("DFMA dependent latency: %.2f cyc\n", double(h[0]) / (4.0 * it));
  k_dadd_lat<<<1, 32>>>(d, c, it); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
  printf("DADD dependent latency: %.2f cyc\n", double(h[0]) / (4.0 * it));
  for (int nt : {32, 128, 256, 512, 1024}) {
    k_dfma_tput<<<1, nt>>>(d, c, it); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
    printf("DFMA throughput, 1 CTA x %4d thr: %.2f DFMA/cyc/SM\n", nt, double(nt) * 8.0 * it / double(h[0]));
  }
  k_lds<<<1, 256>>>(d, c, it); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost));
  printf("LDS.64 pointer-chase latency: %.2f cyc; LDS.128 bandwidth (256 thr): %.1f B/cyc/SM\n",
         double(h[0]) / it, 256.0 * 4 * 16 * it / double(h[1]));
  for (int nt : {256, 512, 1024}) {
    k_bar<<<1, nt>>>(c, it); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
    printf("__syncthreads (%4d thr): %.1f cyc\n", nt, double(h[0]) / it);
  }
  for (int C : {2, 4, 8, 16}) {
    if (launch_cluster(k_cbar, C, 256, C, c, 1024)) { printf("cluster launch failed C=%d\n", C); continue; }
    CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
    printf("cluster.sync C=%2d (256 thr): %.1f cyc", C, double(h[0]) / 1024);
    launch_cluster(k_cbar_relaxed, C, 256, C, c, 1024);
    CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
    printf("  relaxed arrive+wait: %.1f cyc", double(h[0]) / 1024);
    launch_cluster(k_dsmem, C, 256, C, d, c, 64);
    CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
    printf("  DSMEM read: %.1f B/cyc/SM\n", 1024.0 * 16 * 64 / double(h[0]));
  }

  double2 *gb; CK(cudaMalloc(&gb, size_t(148) * 1024 * 16 * 2));
  for (int C : {4, 8, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      for (int grid : {C, 8 * C}) {
        if (launch_cluster(k_xchg, grid, 256, C, gb, c, 256, mode)) { printf("launch fail\n"); continue; }
        CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
        printf("xchg C=%2d grid=%3d mode=%d: %.0f cyc per 16 KB exchange\n", C, grid, mode, double(h[0]) / 256);
      }
    }
  }

  for (int C : {2, 4, 8, 16}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int grid : {C, 8 * C}) {
        if (launch_cluster(k_xasync, grid, 256, C, c, 256, mode)) { printf("launch fail\n"); continue; }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("xasync err %s\n", cudaGetErrorString(e)); return 1; }
        CK(cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost));
        printf("xasync C=%2d grid=%3d mode=%d (%s): %.0f cyc per 16 KB exchange\n", C, grid, mode,
               mode ? "st.async" : "bulk", double(h[0]) / 256);
      }
    }
  }
  return 0;
}
