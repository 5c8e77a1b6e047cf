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
      static int g3 = -1;  // warps per block of the 3-component (elastic) mass SpMV
      if (g3 < 0) { const char* e = getenv("GA_SPMV_G3"); g3 = e ? atoi(e) : 8; }
      if (g3 == 4) launch_sm<P, NC, KK, false, 4>(a, (unsigned int)((nrb + 3) / 4), s);
      else launch_sm<P, NC, KK, false, 8>(a, (unsigned int)((nrb + 7) / 8), s);
    } else {
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
