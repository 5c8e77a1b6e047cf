// Stencil SpMV of the hot path (sm_100a, fp64): y = A x on the column-index-free
// layout coef[o][row] for all lock-stepped right-hand sides at once.  Modes:
// apply, -K s (right-hand sides b_j = -K s_j), q = M p with the
// PCG direction update and the p.q reduction / alpha fused,
// r = b - M x (refinement restart, R8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ops.cuh"
#include "spmv_core.cuh"

namespace ga {

// ---------------------------------------------------------------------------
// Stencil SpMV
// ---------------------------------------------------------------------------
// Warp-staged stencil SpMV.  A block of G warps
// owns 32 consecutive rows (lane = row: coefficient loads are 256 B coalesced
// per warp); warp w handles the offset lines (o3, o2) = w, w+G, ... .  For each
// line the warp stages its input window (32 + 2P points) in its own slice of
// shared memory (only __syncwarp, no block barrier inside the loop), with the
// next line's window and coefficients prefetched into registers while the
// current line is consumed.  The G partial sums are combined in shared memory
// in a fixed order.  With SPMV_PQ + fuse_p the window is the new PCG direction
// p = z + beta p_old, formed once per point and warp.
template <int P, int NC, int KK, bool ELASTIC, int G>
__global__ void __launch_bounds__(32 * G) k_spmv_sm(SpmvArgs a) {
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  count_launch(a.st);
  extern __shared__ double smem_spmv[];
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  spmv_block<P, NC, KK, ELASTIC, G, false>(a, blockIdx.x, smem_spmv, dots);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) {
    // per-block partial sums; the scalar step runs in k_spmv_fin (one block),
    // which avoids a fence + same-address atomic per block
    block_sum<KK>(dots);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < KK; ++j) a.partial[(size_t)blockIdx.x * KK + j] = dots[j];
    }
  }
}

template <int P, int NC, int KK, int G>
__global__ void __launch_bounds__(32 * G) k_spmv_half(SpmvArgs a) {
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  count_launch(a.st);
  extern __shared__ double smem_spmv[];
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  spmv_block_half<P, NC, KK, G>(a, blockIdx.x, smem_spmv, dots);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) {
    block_sum<KK>(dots);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < KK; ++j) a.partial[(size_t)blockIdx.x * KK + j] = dots[j];
    }
  }
}

// Row-tiled SpMV for several component vectors sharing one scalar stencil (the elastic mass,
// density * M per component): a CTA of TYR warps owns a 32 (x) x TYR (y) tile of rows at one z;
// for each z offset o3 it stages the (TYR + 2P) y-lines x (32 + 2P) points x NC components of
// the input once in shared memory (double-buffered, the next plane prefetched into registers),
// and warp w computes row y0 + w from it.  The TYR rows share every staged input line: the
// window traffic per row drops from NC (32 + 2P)/32 lines per offset line to
// NC (TYR + 2P)(32 + 2P) / (32 TYR W) (about 3x less for P = 4).  Linear addressing: points
// outside the grid in x or y wrap into neighbouring lines, whose coefficients are zero.
template <int P, int NC, int KK, int TYR>
__global__ void __launch_bounds__(32 * TYR) k_spmv_tile(SpmvArgs a, int ntx, int nty) {
  constexpr int W = 2 * P + 1, TX = 32 + 2 * P, TY = TYR + 2 * P;
  constexpr int PLANE = TY * TX * NC * KK;
  constexpr int NT = 32 * TYR;
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&a.st->launches, 1ull);
  extern __shared__ double smem_t[];
  double* buf0 = smem_t;
  double* buf1 = smem_t + PLANE;
  const GridDesc g = a.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = blockIdx.x % ntx;
  const int ty = (blockIdx.x / ntx) % nty;
  const int z = blockIdx.x / (ntx * nty);
  const int x0 = tx * 32, y0 = ty * TYR;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  const int x = x0 + lane, y = y0 + w;
  const bool valid = x < g.nx && y < g.ny;
  const long long i = x + sy * y + sz * z;
  const long long icl = valid ? i : 0;
  const long long S = (long long)W * W * W;
  const double* __restrict__ cslice = a.coef + (icl >> 5) * S * 32 + (icl & 31);
  // staged point q = (ty', tx', c, j) of plane o3: linear index of (x0 - P + tx', y0 - P + ty', z + o3);
  // copied asynchronously (cp.async, no registers), the next plane while this one is consumed
  auto issue_plane = [&](int o3, double* dst) {
    for (int q = threadIdx.x; q < PLANE; q += NT) {
      const int j = q % KK, c = (q / KK) % NC, txp = (q / (KK * NC)) % TX, typ = q / (KK * NC * TX);
      const long long pos = g.guard + (x0 - P + txp) + sy * (y0 - P + typ) + sz * (z + o3);
      const unsigned int d = (unsigned int)__cvta_generic_to_shared(dst + q);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d),
                   "l"(a.x + ((long long)c * g.padded + pos) * KK + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double acc[NC][KK];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int j = 0; j < KK; ++j) acc[c][j] = 0.0;
  issue_plane(-P, buf0);
  double cf[W];
#pragma unroll
  for (int u = 0; u < W; ++u) cf[u] = __ldg(cslice + (long long)u * 32);  // line (o3, o2) = (-P, -P)
  for (int o3i = 0; o3i < W; ++o3i) {
    double* cur = (o3i & 1) ? buf1 : buf0;
    double* nxt = (o3i & 1) ? buf0 : buf1;
    if (o3i + 1 < W) {
      issue_plane(o3i + 1 - P, nxt);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // this plane's copies are done
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
#pragma unroll 1
    for (int o2i = 0; o2i < W; ++o2i) {
      double cc[W];
#pragma unroll
      for (int u = 0; u < W; ++u) cc[u] = cf[u];
      const int line = o3i * W + o2i;
      if (line + 1 < W * W) {
#pragma unroll
        for (int u = 0; u < W; ++u) cf[u] = __ldg(cslice + ((long long)(line + 1) * W + u) * 32);
      }
      const double* row = cur + ((w + o2i) * TX + lane) * NC * KK;  // staged y-line y + o2, x from x - P
#pragma unroll
      for (int u = 0; u < W; ++u)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < KK; ++j) acc[c][j] = fma(cc[u], row[(u * NC + c) * KK + j], acc[c][j]);
    }
    __syncthreads();  // every warp is done with cur before it is refilled
  }
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  if (valid) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const long long base = ((long long)c * g.padded + g.guard + i) * KK;
      double pv[KK];
      if (a.mode == SPMV_PQ) load_row<KK>(a.x + base, pv);
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        double v = acc[c][j];
        if (a.mode == SPMV_NEGB) v = -v;
        else if (a.mode == SPMV_TRUERES) { v = a.b[base + j] - v; dots[j] = fma(v, v, dots[j]); }
        else if (a.mode == SPMV_PQ) dots[j] = fma(pv[j], v, dots[j]);
        a.y[base + j] = v;
      }
    }
  }
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) {
    block_sum<KK>(dots);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < KK; ++j) a.partial[(size_t)blockIdx.x * KK + j] = dots[j];
    }
  }
}

// Register-blocked row tiles for the 3-component mass SpMV (the elastic M = density * scalar M
// per component).  The warp-per-row-block kernel reads
// W * NC * KK window values from shared memory per row and offset line (54 at NC = 3, KK = 2)
// against W coefficients from HBM: shared-memory bandwidth, not HBM, binds it.  Here a CTA of
// TYW warps owns a 32 (x) x TYW R (y) tile at one z; per z offset o3 it stages the
// (TYW R + 2P) y-lines x (32 + 2P) points x NC x KK input plane once (cp.async 16 B,
// double-buffered), and each thread computes R rows (x, y .. y + R - 1): every staged value is
// read once from shared memory and used for the up to R rows whose y offset reaches it, with
// that row's coefficient c(row, o3, o2 = t - r, o1) held in registers.  Shared-memory reads per
// row and line drop by R W / (R + 2P) (3x at P = 4, R = 4).  Staged lines past ny - 1 + P are
// only read by rows outside the grid and are zero-filled (no load beyond the guard).
template <int P, int NC, int KK, int TYW, int R, int MINB = 2, bool DB = true>
__global__ void __launch_bounds__(32 * TYW, MINB) k_spmv_rt(SpmvArgs a, int ntx, int nty) {
  constexpr int W = 2 * P + 1, TX = 32 + 2 * P, TYR = TYW * R, TY = TYR + 2 * P, V = NC * KK;
  constexpr int PLANE = TY * TX * V;
  constexpr int NT = 32 * TYW;
  constexpr int U = (KK % 2 == 0) ? 2 : 1;  // doubles per cp.async
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&a.st->launches, 1ull);
  extern __shared__ __align__(16) double smem_rt[];
  double* buf0 = smem_rt;
  double* buf1 = DB ? smem_rt + PLANE : smem_rt;
  const GridDesc g = a.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = blockIdx.x % ntx;
  const int ty = (blockIdx.x / ntx) % nty;
  const int z = blockIdx.x / (ntx * nty);
  const int x0 = tx * 32, y0 = ty * TYR;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  const int x = x0 + lane, yw = y0 + w * R;
  const long long S = (long long)W * W * W;
  const double* cs[R];
  bool valid[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    valid[r] = x < g.nx && yw + r < g.ny;
    const long long i = x + sy * (yw + r) + sz * z;
    const long long icl = valid[r] ? i : 0;
    cs[r] = a.coef + (icl >> 5) * S * 32 + (icl & 31);
  }
  const int ylim = g.ny - 1 + P;
  auto issue_plane = [&](int o3, double* dst) {
    for (int q = threadIdx.x; q < PLANE / U; q += NT) {
      const int e = q * U;
      const int j = e % KK, c = (e / KK) % NC, txp = (e / V) % TX, typ = e / (V * TX);
      const int yy = y0 - P + typ;
      if (yy <= ylim) {
        const long long pos = g.guard + (x0 - P + txp) + sy * yy + sz * (z + o3);
        const unsigned int d = (unsigned int)__cvta_generic_to_shared(dst + e);
        const double* src = a.x + ((long long)c * g.padded + pos) * KK + j;
        if constexpr (U == 2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
      } else {
#pragma unroll
        for (int uu = 0; uu < U; ++uu) dst[e + uu] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double acc[R][V];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[r][v] = 0.0;
  if (DB) issue_plane(-P, buf0);
#pragma unroll 1
  for (int o3i = 0; o3i < W; ++o3i) {
    double* cur = (o3i & 1) ? buf1 : buf0;
    double* nxt = (o3i & 1) ? buf0 : buf1;
    if (!DB) {  // single buffer: the other CTAs on the SM overlap this one's staging
      issue_plane(o3i - P, cur);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else if (o3i + 1 < W) {
      issue_plane(o3i + 1 - P, nxt);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const long long lbase = (long long)o3i * W * W * 32;
#pragma unroll
    for (int t = 0; t < R + 2 * P; ++t) {
      double cc[R][W];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int o2i = t - r;
        if (o2i >= 0 && o2i < W) {
#pragma unroll
          for (int u = 0; u < W; ++u) cc[r][u] = __ldg(cs[r] + lbase + (long long)(o2i * W + u) * 32);
        }
      }
      const double* row = cur + ((w * R + t) * TX + lane) * V;
#pragma unroll
      for (int u = 0; u < W; ++u) {
        double v[V];
        if constexpr (V % 2 == 0) {
#pragma unroll
          for (int h = 0; h < V / 2; ++h) {
            const double2 t2 = *reinterpret_cast<const double2*>(row + u * V + 2 * h);
            v[2 * h] = t2.x; v[2 * h + 1] = t2.y;
          }
        } else {
#pragma unroll
          for (int h = 0; h < V; ++h) v[h] = row[u * V + h];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int o2i = t - r;
          if (o2i >= 0 && o2i < W) {
#pragma unroll
            for (int h = 0; h < V; ++h) acc[r][h] = fma(cc[r][u], v[h], acc[r][h]);
          }
        }
      }
    }
    __syncthreads();  // every warp is done with cur before it is refilled
  }
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (!valid[r]) continue;
    const long long i = x + sy * (yw + r) + sz * z;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const long long base = ((long long)c * g.padded + g.guard + i) * KK;
      double pv[KK];
      if (a.mode == SPMV_PQ) load_row<KK>(a.x + base, pv);
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        double v = acc[r][c * KK + j];
        if (a.mode == SPMV_NEGB) v = -v;
        else if (a.mode == SPMV_TRUERES) { v = a.b[base + j] - v; dots[j] = fma(v, v, dots[j]); }
        else if (a.mode == SPMV_PQ) dots[j] = fma(pv[j], v, dots[j]);
        a.y[base + j] = v;
      }
    }
  }
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) {
    block_sum<KK>(dots);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < KK; ++j) a.partial[(size_t)blockIdx.x * KK + j] = dots[j];
    }
  }
}

// Fixed-order sum of the SpMV block partials and the PCG scalar step:
// SPMV_PQ: alpha_j = r.z / p.q (F2); SPMV_TRUERES: restart of the refinement phase.
template <int KK>
__global__ void __launch_bounds__(1024) k_spmv_fin(SpmvArgs a, unsigned int nblocks) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  double acc[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) acc[j] = 0.0;
  const unsigned int chunk = (nblocks + blockDim.x - 1) / blockDim.x;
  const unsigned int b0 = threadIdx.x * chunk, b1 = min(nblocks, b0 + chunk);
  for (unsigned int b = b0; b < b1; ++b)
#pragma unroll
    for (int j = 0; j < KK; ++j) acc[j] += a.partial[(size_t)b * KK + j];
  block_sum<KK>(acc);
  if (threadIdx.x != 0) return;
  if (a.xsum && a.mode == SPMV_PQ) {  // subdomain: local p.q to the exchange (dist.cu)
#pragma unroll
    for (int j = 0; j < KK; ++j) a.xsum[j] = acc[j];
    return;
  }
  PcgState* pc = a.pcg;
  if (a.mode == SPMV_PQ) {
    pc->iter += 1;
    pc->pfirst = 0;
    a.st->loop_iters += 1;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      pc->pq[j] = acc[j];
      if (pc->active[j]) {
        pc->alpha[j] = pc->rz[j] / acc[j];
        pc->its[j] += 1;
      } else {
        pc->alpha[j] = 0.0;
      }
    }
  } else {
    // restart of PCG from the true residual (refinement phase, R8)
    pc->iter = 0; pc->first = 1; pc->pfirst = 1; pc->phase = 1; pc->guard = 0;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      pc->alpha[j] = 0.0;
      pc->active[j] = pc->bb[j] > 0.0 ? 1 : 0;
      double thr = a.tol2 * pc->bb[j];
      if (a.refine_rtol2 > 0.0) thr = fmin(thr, a.refine_rtol2 * acc[j]);
      pc->thr[j] = thr;
    }
  }
}

template <int P, int NC, int KK, bool ELASTIC, int G>
static void launch_sm(const SpmvArgs& a, unsigned int nb, cudaStream_t s) {
  constexpr int BR = 32, WN = BR + 2 * P;
  constexpr int NB = ELASTIC ? 3 : NC;
  constexpr size_t bytes = sizeof(double) * (2 * G * NB * WN * KK);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmv_sm<P, NC, KK, ELASTIC, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = true;
  }
  k_spmv_sm<P, NC, KK, ELASTIC, G><<<nb, 32 * G, bytes, s>>>(a);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) k_spmv_fin<KK><<<1, 1024, 0, s>>>(a, nb);
}

template <int P, int NC, int KK>
static bool launch_tile(const SpmvArgs& a, cudaStream_t s) {
  constexpr int TYR = 8, TX = 32 + 2 * P, TY = TYR + 2 * P;
  constexpr size_t bytes = sizeof(double) * 2 * TY * TX * NC * KK;
  if (bytes > 200 * 1024) return false;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_spmv_tile<P, NC, KK, TYR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
        cudaSuccess)
      return false;
    attr = true;
  }
  const int ntx = (a.g.nx + 31) / 32, nty = (a.g.ny + TYR - 1) / TYR;
  const unsigned int nb = (unsigned int)((long long)ntx * nty * a.g.nz);
  k_spmv_tile<P, NC, KK, TYR><<<nb, 32 * TYR, bytes, s>>>(a, ntx, nty);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) k_spmv_fin<KK><<<1, 1024, 0, s>>>(a, nb);
  return true;
}

template <int P, int NC, int KK, int TYW, int R, int MINB = 2, bool DB = true>
static bool launch_rt(const SpmvArgs& a, cudaStream_t s) {
  constexpr int TX = 32 + 2 * P, TY = TYW * R + 2 * P;
  constexpr size_t bytes = sizeof(double) * (DB ? 2 : 1) * TY * TX * NC * KK;
  if constexpr (bytes > 200 * 1024) {
    return false;
  } else {
    // one block per 32 x TYW R tile: never more blocks than 32-row blocks (partial slots)
    if (a.g.dim != 3 || a.g.nx < 32 || a.g.ny < TYW * R) return false;
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_spmv_rt<P, NC, KK, TYW, R, MINB, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)bytes) != cudaSuccess)
        return false;
      attr = true;
    }
    const int ntx = (a.g.nx + 31) / 32, nty = (a.g.ny + TYW * R - 1) / (TYW * R);
    const unsigned int nb = (unsigned int)((long long)ntx * nty * a.g.nz);
    k_spmv_rt<P, NC, KK, TYW, R, MINB, DB><<<nb, 32 * TYW, bytes, s>>>(a, ntx, nty);
    if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) k_spmv_fin<KK><<<1, 1024, 0, s>>>(a, nb);
    return true;
  }
}

template <int P, int NC, int KK>
static void launch_half(const SpmvArgs& a, cudaStream_t s) {
  constexpr int G = 8, BR = 32, WN = BR + 2 * P;
  constexpr size_t bytes = sizeof(double) * (2 * 2 * G * NC * WN * KK);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmv_half<P, NC, KK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = true;
  }
  const long long nrb = (a.g.npts + 31) / 32;
  const unsigned int nb = (unsigned int)((nrb + G - 1) / G);
  k_spmv_half<P, NC, KK, G><<<nb, 32 * G, bytes, s>>>(a);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) k_spmv_fin<KK><<<1, 1024, 0, s>>>(a, nb);
}

template <int P, int NC, int KK>
static void spmv_kk(const SpmvArgs& a, cudaStream_t s) {
  if (a.half && !a.elastic) {
    launch_half<P, NC, KK>(a, s);
    return;
  }
  {
    const long long nrb = (a.g.npts + 31) / 32;
    if (a.elastic) {
      if constexpr (NC == 3) launch_sm<P, 3, KK, true, 4>(a, (unsigned int)((nrb + 3) / 4), s);
    } else if (NC == 3) {
      static int g3 = -1;  // 3-component (elastic) mass SpMV: 0 row tiles (default), 4 / 8 warp row blocks
      if (g3 < 0) { const char* e = getenv("GA_SPMV_G3"); g3 = e ? atoi(e) : 8; }  // tiles: opt-in (measured slower)
      static int rt = -1;  // register-blocked row tiles (default 4 x 4; C4 M apply 1.48 -> 1.24 ms, 8 x 2: 1.33)
      if (rt < 0) { const char* e = getenv("GA_SPMV_RT"); rt = e ? atoi(e) : 1; }
      if constexpr (NC == 3) {
        if (rt == 1 && launch_rt<P, NC, KK, 4, 4>(a, s)) return;  // 4 warps x 4 rows, 2 CTAs / SM
        // measured and dropped: 8 warps x 2 rows (1.33 vs 1.24 ms at C4); the x remainder
        // (nx mod 32) as a second launch with narrow lane tiles (1.30 vs 1.22 ms: an extra wave)
        // measured and dropped: single-buffered planes at 3 / 4 CTAs per SM (168 / 128 registers):
        // 1.21 / 1.26 ms vs 1.22 ms, occupancy does not move it
      }
      if (g3 == 0 && a.g.dim == 3 && launch_tile<P, NC, KK>(a, s)) return;
      if (g3 == 4) launch_sm<P, NC, KK, false, 4>(a, (unsigned int)((nrb + 3) / 4), s);
      else launch_sm<P, NC, KK, false, 8>(a, (unsigned int)((nrb + 7) / 8), s);
    } else {
      // row tiles measured no faster for the scalar stencil (C3 p=2 n=96 k=1/3, p=2 n=192, p=4
      // n=96: 0.81-0.95 vs 0.71-0.96 of HBM): one vector per row is not shared-memory bound
      launch_sm<P, NC, KK, false, 8>(a, (unsigned int)((nrb + 7) / 8), s);
    }
    return;
  }
}
template <int P, int NC>
static void spmv_nc(const SpmvArgs& a, cudaStream_t s) {
  switch (a.kk) {
    case 1: spmv_kk<P, NC, 1>(a, s); break;
    case 2: spmv_kk<P, NC, 2>(a, s); break;
    case 3: spmv_kk<P, NC, 3>(a, s); break;
    default: spmv_kk<P, NC, 4>(a, s); break;
  }
}
template <int P>
static void spmv_p(const SpmvArgs& a, cudaStream_t s) {
  if (a.nvec == 3) spmv_nc<P, 3>(a, s);
  else spmv_nc<P, 1>(a, s);
}
void launch_spmv_fin(const SpmvArgs& a, unsigned int nb, cudaStream_t s) {
  switch (a.kk) {
    case 1: k_spmv_fin<1><<<1, 1024, 0, s>>>(a, nb); break;
    case 2: k_spmv_fin<2><<<1, 1024, 0, s>>>(a, nb); break;
    case 3: k_spmv_fin<3><<<1, 1024, 0, s>>>(a, nb); break;
    default: k_spmv_fin<4><<<1, 1024, 0, s>>>(a, nb); break;
  }
}

void launch_spmv(const SpmvArgs& a, cudaStream_t s) {
  if (a.sym) {
    launch_spmv_sym(a, s);
    return;
  }
  if (a.mf) {
    launch_matfree(a, s);
    return;
  }
  switch (a.p) {
    case 1: spmv_p<1>(a, s); break;
    case 2: spmv_p<2>(a, s); break;
    case 3: spmv_p<3>(a, s); break;
    case 4: spmv_p<4>(a, s); break;
    case 5: spmv_p<5>(a, s); break;
    case 6: spmv_p<6>(a, s); break;
    default: spmv_p<7>(a, s); break;
  }
}

}  // namespace ga
