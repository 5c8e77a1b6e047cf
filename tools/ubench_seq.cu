// Microbenchmark of the whole-line sequential sweep (line_seq.cu seq_sweep) and the dependent-DFMA
// latency it rides on.  Build (from the repo root):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/ubench_seq.cu -o tools/ubench_seq.bin
#include <cstdio>
#include <cstring>
#include <vector>

#define GA_SEQ_TRACE 1
#include "../paper_2102_11536_b200/csrc/line_seq.cu"

using namespace ga;

__global__ void k_dfma_lat(double* out, long long* cyc, int n, int chains) {
  double a[4] = {threadIdx.x * 1e-3, 1.0, 2.0, 3.0};
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  if (chains == 1) for (int i = 0; i < n; ++i) a[0] = fma(a[0], b, c);
  else if (chains == 2) for (int i = 0; i < n; ++i) { a[0] = fma(a[0], b, c); a[1] = fma(a[1], b, c); }
  else for (int i = 0; i < n; ++i) { a[0] = fma(a[0], b, c); a[1] = fma(a[1], b, c); a[2] = fma(a[2], b, c); a[3] = fma(a[3], b, c); }
  long long t1 = clock64();
  out[threadIdx.x] = a[0] + a[1] + a[2] + a[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// sweeps only: every CTA fills a tile in shared memory, warp wsel sweeps `lanes` slots
template <int P>
__global__ void __launch_bounds__(128) k_sweep(const double* E, int n, int TS, int lanes, int nwarps, long long* cyc, double* out,
                                               unsigned int* arrival) {
  constexpr int PP = (P + 2) & ~1;
  constexpr int U = P <= 4 ? 8 : 4;
  extern __shared__ __align__(16) double smem[];
  const int SL = 2 * U * max(TS, 4);
  double* tile = smem + SL;
  double* Es = tile + (size_t)n * TS + SL;
  for (int i = threadIdx.x; i < n * TS; i += blockDim.x) tile[i] = 1.0 + 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 2 * n * PP; i += blockDim.x) Es[i] = E[i];
  __syncthreads();
  __shared__ int wsel;
  if (threadIdx.x == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    wsel = arrival ? (int)(atomicAdd(&arrival[smid], 1u) & 3u) : 0;
  }
  __syncthreads();
  int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  w = (w - wsel) & 3;  // nwarps = 1: the sweep warp is warp wsel
  long long t0 = clock64();
  if (w < nwarps && lane < lanes) {
    const int c = (w * lanes + lane) % TS;
    seq_sweep<P, U>(tile, c, TS, n, Es, false);
    seq_sweep<P, U>(tile, c, TS, n, Es + (size_t)n * PP, true);
  }
  long long t1 = clock64();
  if (lane == 0 && w == 0) cyc[blockIdx.x] = t1 - t0;  // the (first) sweep warp
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = tile[5];
}

// variants of the sweep to see what bounds it: NOE: factor rows constant in registers (no LDS.128);
// NOD: data from a register recurrence instead of LDS/STS
template <int P, int U, bool NOE, bool NOD>
__device__ __forceinline__ double sweep_var(double* tile, const int sb, const int ss, const int n, const double* E) {
  constexpr int PP = (P + 2) & ~1;
  double y[P];
#pragma unroll
  for (int u = 0; u < P; ++u) y[u] = 0.0;
  double bA[U], bB[U], eA[U][PP], eB[U][PP];
  int off[U];
#pragma unroll
  for (int u = 0; u < U; ++u) off[u] = u * ss;
  double* dp = tile + sb;
  const double* ep = E;
  auto load = [&](const double* d, const double* er0, double(&b)[U], double(&e)[U][PP]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      b[u] = NOD ? 1.0 + 1e-9 * u : d[off[u]];
      const double2* er = reinterpret_cast<const double2*>(er0 + u * PP);
#pragma unroll
      for (int q = 0; q < PP / 2; ++q) {
        double2 v;
        if (NOE) { v.x = 0.3 + 0.01 * q; v.y = 0.1; } else v = er[q];
        e[u][2 * q] = v.x;
        e[u][2 * q + 1] = v.y;
      }
    }
  };
  auto solve = [&](double(&b)[U], double(&e)[U][PP]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double t = b[u] * e[u][0];
#pragma unroll
      for (int v = P; v >= 2; --v) t = fma(-e[u][v], y[v - 1], t);
      t = fma(-e[u][1], y[0], t);
#pragma unroll
      for (int v = P - 1; v >= 1; --v) y[v] = y[v - 1];
      y[0] = t;
      b[u] = t;
    }
  };
  double acc = 0;
  auto store = [&](double* d, double(&b)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) { if (NOD) acc += b[u]; else d[off[u]] = b[u]; }
  };
  load(dp, ep, bA, eA);
  for (int i0 = 0; i0 < n; i0 += 2 * U) {
    load(dp + U * ss, ep + U * PP, bB, eB);
    solve(bA, eA);
    store(dp, bA);
    load(dp + 2 * U * ss, ep + 2 * U * PP, bA, eA);
    solve(bB, eB);
    store(dp + U * ss, bB);
    dp += 2 * U * ss;
    ep += 2 * U * PP;
  }
  return acc + y[0];
}

template <int P, int U, bool NOE, bool NOD>
__global__ void __launch_bounds__(128) k_var(const double* E, int n, int TS, long long* cyc, double* out) {
  constexpr int PP = (P + 2) & ~1;
  extern __shared__ __align__(16) double smem[];
  double* tile = smem + 512;
  double* Es = tile + (size_t)n * TS + 512;
  for (int i = threadIdx.x; i < n * TS; i += blockDim.x) tile[i] = 1.0 + 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 2 * n * PP; i += blockDim.x) Es[i] = E[i];
  __syncthreads();
  long long t0 = clock64();
  double r = 0;
  if (threadIdx.x < 8) r = sweep_var<P, U, NOE, NOD>(tile, threadIdx.x, TS, n, Es);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (r == 1.2345) out[0] = r;
}

template <int U, bool NOE, bool NOD>
void run_var(const double* dE, int len, size_t sm, long long* cyc, double* out) {
  cudaFuncSetAttribute(k_var<3, U, NOE, NOD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  long long h = 0;
  for (int r = 0; r < 2; ++r) k_var<3, U, NOE, NOD><<<1, 128, sm>>>(dE, len, 8, cyc, out);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("sweep variant U=%2d %s %s: %6.1f cycles/element  %s\n", U, NOE ? "no-E-loads" : "E-loads   ", NOD ? "no-data-LDS/STS" : "data-LDS/STS   ",
         (double)h / len, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1 << 20);
  std::vector<long long> h(4096);
  const int n = 4096;
  for (int ch : {1, 2, 4}) for (int thr : {32, 128, 256}) {
    k_dfma_lat<<<1, thr>>>(out, cyc, n, ch);
    k_dfma_lat<<<1, thr>>>(out, cyc, n, ch);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DFMA: %d chain(s)/thread, %3d threads: %6.1f cycles per step\n", ch, thr, (double)h[0] / n);
  }
  const int P = 3, PP = 4, len = 514;
  std::vector<double> E(2 * len * PP);
  for (int i = 0; i < 2 * len; ++i) { E[i * PP] = 0.9; E[i * PP + 1] = 0.3; E[i * PP + 2] = 0.1; E[i * PP + 3] = 0.01; }
  double* dE; cudaMalloc(&dE, E.size() * 8);
  cudaMemcpy(dE, E.data(), E.size() * 8, cudaMemcpyHostToDevice);
  const int TS = 8;
  const size_t sm = 8 * (2 * 16 * 8 * 2 + (size_t)len * TS + 2 * len * PP + 16 * PP);
  cudaFuncSetAttribute(k_sweep<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  {
    const size_t smv = 8 * (1024 + (size_t)(len + 64) * 8 + 2 * (len + 64) * PP);
    run_var<8, false, false>(dE, len, smv, cyc, out);
    run_var<8, true, false>(dE, len, smv, cyc, out);
    run_var<8, false, true>(dE, len, smv, cyc, out);
    run_var<8, true, true>(dE, len, smv, cyc, out);
    run_var<4, false, false>(dE, len, smv, cyc, out);
    run_var<16, false, false>(dE, len, smv, cyc, out);
    run_var<16, true, true>(dE, len, smv, cyc, out);
  }
  unsigned int* arr; cudaMalloc(&arr, 4096); cudaMemset(arr, 0, 4096);
  for (int spread : {0, 1}) for (int grid : {1, 148, 296, 387, 444}) for (int nw : {1, 2}) for (int lanes : {8}) {
    unsigned int* ap = spread ? arr : nullptr;
    printf("spread %d: ", spread);
    k_sweep<P><<<grid, 128, sm>>>(dE, len, TS, lanes, nw, cyc, out, ap);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_sweep<P><<<grid, 128, sm>>>(dE, len, TS, lanes, nw, cyc, out, ap);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h.data(), cyc, 8 * grid, cudaMemcpyDeviceToHost);
    long long mx = 0, mn = 1LL << 60;
    for (int i = 0; i < grid; ++i) { mx = std::max(mx, h[i]); mn = std::min(mn, h[i]); }
    printf("sweeps n=%d: grid %3d, %d warp(s) x %2d lanes: %7.1f-%7.1f cycles/element (fwd+bwd = 2n elements), kernel %.1f us  %s\n",
           len, grid, nw, lanes, (double)mn / (2 * len), (double)mx / (2 * len), ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  {  // the real kernel on a C5-shaped problem: 3 boxes of 514 x 514, k = 2, both directions
    const int nb = 514, kk = 2, np = 3;
    PrecArgs a;
    memset(&a, 0, sizeof(a));
    a.g.dim = 2; a.nvec = 1; a.kk = kk; a.p = 3; a.npatch = np;
    a.g.nx = 3 * nb; a.g.ny = nb; a.g.nz = 1; a.g.npts = (long long)a.g.nx * a.g.ny; a.g.guard = 2048; a.g.padded = a.g.npts + 2 * a.g.guard;
    { double* v; cudaMalloc(&v, 8 * a.g.padded * kk); cudaMemset(v, 0, 8 * a.g.padded * kk); a.r = v;
      cudaMalloc(&v, 8 * a.g.padded * kk); cudaMemset(v, 0, 8 * a.g.padded * kk); a.z = v;
      cudaMalloc(&v, 8 * 8 * 8192); a.partial = v;
      PcgState* pc; cudaMalloc(&pc, sizeof(PcgState)); cudaMemset(pc, 0, sizeof(PcgState)); a.pcg = pc; a.maxit = 100; }
    DevStatus* st; cudaMalloc(&st, sizeof(DevStatus)); cudaMemset(st, 0, sizeof(DevStatus));
    a.st = st;
    unsigned int* ctr; cudaMalloc(&ctr, 8192); cudaMemset(ctr, 0, 8192);
    a.counter = ctr;
    std::vector<double> EE(2 * nb * PP);
    for (int i = 0; i < 2 * nb; ++i) { EE[i * PP] = 0.9; EE[i * PP + 1] = 0.3; EE[i * PP + 2] = 0.1; EE[i * PP + 3] = 0.01; }
    for (int r = 0; r < np; ++r) {
      a.bd[r][0] = nb; a.bd[r][1] = nb; a.bd[r][2] = 1;
      a.lo[r][0] = r * nb; a.lo[r][1] = 0; a.lo[r][2] = 0;
      { double* sv; cudaMalloc(&sv, 8 * nb * nb); cudaMemset(sv, 0, 8 * nb * nb); a.s[r] = sv; }
      double* t; cudaMalloc(&t, sizeof(double) * nb * nb * kk); cudaMemset(t, 0, sizeof(double) * nb * nb * kk);
      a.t[r] = t;
      for (int d = 0; d < 2; ++d) { double* e; cudaMalloc(&e, EE.size() * 8); cudaMemcpy(e, EE.data(), EE.size() * 8, cudaMemcpyHostToDevice); a.E[r][d] = e; }
    }
    long long* tr; cudaMalloc(&tr, 8 * 8 * 4096); cudaMemset(tr, 0, 8 * 8 * 4096);
    cudaMemcpyToSymbol(g_seq_trace, &tr, sizeof(tr));
    char* flush; cudaMalloc(&flush, 256 << 20);
    for (int fuse = 0; fuse < 1; ++fuse) for (int d = 0; d < 2; ++d) for (int cold = 0; cold < 2; ++cold) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        if (cold) cudaMemset(flush, rep, 256 << 20);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        bool ok = launch_line_seq_multi(a, d, 0);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
        if (!ok) printf("launch_line_seq_multi refused\n");
      }
      std::vector<long long> ht(8 * 4096);
      cudaMemcpy(ht.data(), tr, 8 * 8 * 4096, cudaMemcpyDeviceToHost);
      double ph[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
      int nblk = 0;
      for (int b = 0; b < 4096; ++b) if (ht[b * 8 + 4]) { ++nblk; for (int k2 = 0; k2 < 4; ++k2) { double v = (double)(ht[b * 8 + k2 + 1] - ht[b * 8 + k2]); ph[k2] += v; mx[k2] = std::max(mx[k2], v); } }
      printf("k_line_seq fuse %d dir %d %s: %.1f us; %d CTAs; mean (max) cycles: issue %.0f (%.0f), staged %.0f (%.0f), sweeps %.0f (%.0f), store %.0f (%.0f)  %s\n",
             fuse, d, cold ? "cold" : "warm", best * 1e3, nblk, ph[0] / nblk, mx[0], ph[1] / nblk, mx[1], ph[2] / nblk, mx[2], ph[3] / nblk, mx[3], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
