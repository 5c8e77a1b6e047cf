// Microbenchmarks of the latencies the small-problem solver is built from
// (dependent DFMA, LDS, __syncthreads at 256 threads, shuffle, L2 pointer chase,
// grid-wide barrier).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench.cu -o /tmp/ubench
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void k_dfma(double* out, long long* cyc, int n) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// fp64 FMA throughput: 8 independent chains per thread, many warps per SM
__global__ void k_dfma_tput(double* out, int n) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void k_lds(double* out, long long* cyc, int n) {
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i * 97 + 13) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = nxt[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_sync(double* out, long long* cyc, int n) {
  __shared__ double s[1024];
  double a = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    s[threadIdx.x] = a + i;
    __syncthreads();
    a += s[(threadIdx.x + 1) & (blockDim.x - 1)];
    __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl(double* out, long long* cyc, int n) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_up_sync(0xffffffffu, a, 1) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_chase(const long long* nxt, double* out, long long* cyc, int n) {
  long long p = threadIdx.x * 33;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = nxt[p];
  long long t1 = clock64();
  out[threadIdx.x] = (double)p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_grid(double* out, long long* cyc, int n) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}


// flat sense-reversal barrier: one counter, generation word
__device__ __forceinline__ void flat_barrier(unsigned int* cnt, volatile unsigned int* gen, unsigned int nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g0 = *gen;
    __threadfence();
    if (atomicAdd(cnt, 1u) == nb - 1) {
      *cnt = 0;
      __threadfence();
      atomicAdd((unsigned int*)gen, 1u);
    } else {
      unsigned int g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen));
      } while (g == g0);
    }
  }
  __syncthreads();
}
__global__ void k_flat(unsigned int* cnt, unsigned int* gen, long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) flat_barrier(cnt, gen, gridDim.x);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}
// two-level: groups of G blocks arrive on a group counter; the last of a group arrives on the top counter
__device__ __forceinline__ void tree_barrier(unsigned int* cnt, volatile unsigned int* gen, unsigned int nb, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g0 = *gen;
    __threadfence();
    const unsigned int grp = blockIdx.x / G, ngrp = (nb + G - 1) / G;
    const unsigned int gsz = min((unsigned)G, nb - grp * G);
    bool last = false;
    if (atomicAdd(cnt + 1 + grp * 32, 1u) == gsz - 1) {
      cnt[1 + grp * 32] = 0;
      if (atomicAdd(cnt, 1u) == ngrp - 1) last = true;
    }
    if (last) {
      *cnt = 0;
      __threadfence();
      atomicAdd((unsigned int*)gen, 1u);
    } else {
      unsigned int g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen));
      } while (g == g0);
    }
  }
  __syncthreads();
}
__global__ void k_tree(unsigned int* cnt, unsigned int* gen, long long* cyc, int n, int G) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) tree_barrier(cnt, gen, gridDim.x, G);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  long long h;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 64);
  const int n = 4096;
  auto rep = [&](const char* name, int per) {
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %8.1f cycles\n", name, (double)h / (n * per));
  };
  k_dfma<<<1, 32>>>(out, cyc, n);  k_dfma<<<1, 32>>>(out, cyc, n);  rep("dependent DFMA (1 warp)", 1);
  k_dfma<<<1, 256>>>(out, cyc, n); rep("dependent DFMA (8 warps)", 1);
  k_lds<<<1, 32>>>(out, cyc, n);   rep("dependent LDS.32 (1 warp)", 1);
  k_sync<<<1, 256>>>(out, cyc, n); rep("st+sync+ld+sync (8 warps)", 1);
  k_sync<<<1, 512>>>(out, cyc, n); rep("st+sync+ld+sync (16 warps)", 1);
  k_shfl<<<1, 32>>>(out, cyc, n);  rep("dependent shfl+add", 1);
  // L2 pointer chase over 32 MB (L2 resident after a warm pass)
  const long long N = 4 << 20;
  std::vector<long long> hn(N);
  for (long long i = 0; i < N; ++i) hn[i] = (i * 1000003 + 7919) % N;
  long long* dn;
  cudaMalloc(&dn, N * 8);
  cudaMemcpy(dn, hn.data(), N * 8, cudaMemcpyHostToDevice);
  k_chase<<<1, 1>>>(dn, out, cyc, n);
  k_chase<<<1, 1>>>(dn, out, cyc, n); rep("L2 pointer chase (32 MB)", 1);
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int nn = 256;
  void* args[] = {&out, &cyc, &nn};
  for (int b : {1, 2}) {
    cudaLaunchCooperativeKernel((void*)k_grid, dim3(nsm * b), dim3(256), args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync (%d blocks x 256)    %8.1f cycles\n", nsm * b, (double)h / nn);
  }

  {  // fp64 FMA throughput (device-wide, CUDA events)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = nsm * 8, threads = 256;
    k_dfma_tput<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    k_dfma_tput<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("fp64 FMA throughput             %8.2f TFLOP/s (%d SMs)\n", flops / (ms * 1e-3) / 1e12, nsm);
  }

  unsigned int* cnt;
  cudaMalloc(&cnt, 1 << 16);
  cudaMemset(cnt, 0, 1 << 16);
  unsigned int* gen = cnt + 8192;
  {
    void* a2[] = {&cnt, &gen, &cyc, &nn};
    cudaLaunchCooperativeKernel((void*)k_flat, dim3(nsm), dim3(256), a2, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("flat barrier (%d blocks)       %8.1f cycles  (%s)\n", nsm, (double)h / nn, cudaGetErrorString(cudaGetLastError()));
    for (int G : {8, 12, 16}) {
      cudaMemset(cnt, 0, 1 << 16);
      void* a3[] = {&cnt, &gen, &cyc, &nn, &G};
      cudaLaunchCooperativeKernel((void*)k_tree, dim3(nsm), dim3(256), a3, 0, 0);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("tree barrier G=%2d              %8.1f cycles  (%s)\n", G, (double)h / nn, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
