// Stencil SpMV of the hot path (sm_100a, fp64): y = A x on the column-index-free
// layout coef[o][row] for all lock-stepped right-hand sides at once.  Modes:
// apply, -K s (right-hand sides b_j = -K s_j), q = M p with the
// PCG direction update and the p.q reduction / alpha fused,
// r = b - M x (refinement restart, R8).
#include <cuda_runtime.h>

#include <algorithm>

#include "ops.cuh"

namespace ga {

// ---------------------------------------------------------------------------
// Stencil SpMV
// ---------------------------------------------------------------------------
template <int KK>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double (&v)[KK]) {
  if constexpr (KK == 2) {
    double2 t = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = t.x; v[1] = t.y;
  } else if constexpr (KK == 4) {
    double2 t0 = __ldg(reinterpret_cast<const double2*>(p));
    double2 t1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = t0.x; v[1] = t0.y; v[2] = t1.x; v[3] = t1.y;
  } else {
#pragma unroll
    for (int j = 0; j < KK; ++j) v[j] = __ldg(p + j);
  }
}

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
  constexpr int BR = 32;
  constexpr int W = 2 * P + 1, WN = BR + 2 * P;
  constexpr int NA = ELASTIC ? 3 : NC, NB = ELASTIC ? 3 : NC;
  constexpr int NCF = ELASTIC ? 9 : 1;  // coefficient arrays per offset
  constexpr bool PCF = !ELASTIC;         // prefetch the next line's coefficients into registers
  extern __shared__ double smem_spmv[];
  auto win = reinterpret_cast<double (*)[2][NB][WN][KK]>(smem_spmv);                        // [G][2][NB][WN][KK]
  auto red = reinterpret_cast<double (*)[NA * KK][BR]>(smem_spmv + G * 2 * NB * WN * KK);   // [G][NA*KK][BR]
  const GridDesc g = a.g;
  const int r = threadIdx.x & 31, gq = threadIdx.x >> 5;
  const long long i0 = (long long)blockIdx.x * BR;
  const long long i = i0 + r;
  const int W3 = (g.dim == 3) ? W : 1;
  const int P3 = (g.dim == 3) ? P : 0;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  const long long S = (long long)W * W * W3;
  const bool fuse = a.mode == SPMV_PQ && a.fuse_p;
  const double* __restrict__ xin = a.x;
  const double* __restrict__ pold = nullptr;
  double* pnew = nullptr;
  double beta[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) beta[j] = 0.0;
  bool mix = false;
  if (fuse) {
    const int par = a.pcg->iter & 1;
    pold = par ? a.p1 : a.p0;
    pnew = par ? a.p0 : a.p1;
    mix = a.pcg->pfirst == 0;
#pragma unroll
    for (int j = 0; j < KK; ++j) beta[j] = a.pcg->beta[j];
    xin = a.z;
  }
  const bool valid = i < g.npts;
  const long long icl = valid ? i : (g.npts - 1);  // clamp coefficient reads of the tail rows
  auto fetch_win = [&](int line, int q, int c, double (&v)[KK]) {
    const int o3 = line / W - P3, o2 = line % W - P;
    const long long pos = g.guard + i0 - P + q + o3 * sz + o2 * sy;
    const long long e = ((long long)c * g.padded + pos) * KK;
    load_row<KK>(xin + e, v);
    if (mix) {
      double po[KK];
      load_row<KK>(pold + e, po);
#pragma unroll
      for (int j = 0; j < KK; ++j) v[j] = fma(beta[j], po[j], v[j]);
    }
  };
  auto fetch_cf = [&](int line, double (&cf)[PCF ? W : 1][NCF]) {
    if constexpr (!PCF) return;
    // blocked layout: slice (row/32) holds NCF*S offsets x 32 rows contiguously
    const double* cb = a.coef + ((icl >> 5) * NCF * S + (long long)line * W) * 32 + (icl & 31);
#pragma unroll
    for (int o1 = 0; o1 < W; ++o1)
#pragma unroll
      for (int ab = 0; ab < NCF; ++ab) cf[o1][ab] = __ldg(cb + ((long long)ab * S + o1) * 32);
  };
  const int nlines = W3 * W;
  const bool two = r < 2 * P;
  double acc[NA][KK];
#pragma unroll
  for (int c = 0; c < NA; ++c)
#pragma unroll
    for (int j = 0; j < KK; ++j) acc[c][j] = 0.0;
  double pw[2][NB][KK];
  double cf[PCF ? W : 1][NCF];
  int line = gq;
  if (line < nlines) {
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      fetch_win(line, r, c, pw[0][c]);
      if (two) fetch_win(line, BR + r, c, pw[1][c]);
    }
    fetch_cf(line, cf);
  }
  int buf = 0;
  for (; line < nlines; line += G) {
    // publish the prefetched window of `line`
#pragma unroll
    for (int c = 0; c < NB; ++c)
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        win[gq][buf][c][r][j] = pw[0][c][j];
        if (two) win[gq][buf][c][BR + r][j] = pw[1][c][j];
      }
    double ccur[PCF ? W : 1][NCF];
    if constexpr (PCF) {
#pragma unroll
      for (int o1 = 0; o1 < W; ++o1) ccur[o1][0] = cf[o1][0];
    }
    const double* cbl = a.coef + ((icl >> 5) * NCF * S + (long long)line * W) * 32 + (icl & 31);
    __syncwarp();
    // prefetch the next line of this warp
    const int nl = line + G;
    if (nl < nlines) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        fetch_win(nl, r, c, pw[0][c]);
        if (two) fetch_win(nl, BR + r, c, pw[1][c]);
      }
      fetch_cf(nl, cf);
    }
#pragma unroll
    for (int o1 = 0; o1 < W; ++o1) {
      if constexpr (!ELASTIC) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < KK; ++j) acc[c][j] = fma(ccur[o1][0], win[gq][buf][c][r + o1][j], acc[c][j]);
      } else {
#pragma unroll
        for (int aa = 0; aa < 3; ++aa)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            const double c9 = __ldg(cbl + ((long long)(aa * 3 + bb) * S + o1) * 32);
#pragma unroll
            for (int j = 0; j < KK; ++j) acc[aa][j] = fma(c9, win[gq][buf][bb][r + o1][j], acc[aa][j]);
          }
      }
    }
    buf ^= 1;
  }
  // combine the G warps (fixed order) and run the epilogue in warp 0
#pragma unroll
  for (int c = 0; c < NA; ++c)
#pragma unroll
    for (int j = 0; j < KK; ++j) red[gq][c * KK + j][r] = acc[c][j];
  __syncthreads();
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  if (gq == 0 && valid) {
#pragma unroll
    for (int c = 0; c < NA; ++c) {
      const long long base = ((long long)c * g.padded + g.guard + i) * KK;
      double pv[KK];
      if (a.mode == SPMV_PQ) {
        if (fuse) {
          load_row<KK>(a.z + base, pv);
          if (mix) {
            double po[KK];
            load_row<KK>(pold + base, po);
#pragma unroll
            for (int j = 0; j < KK; ++j) pv[j] = fma(beta[j], po[j], pv[j]);
          }
#pragma unroll
          for (int j = 0; j < KK; ++j) pnew[base + j] = pv[j];
        } else {
          load_row<KK>(a.x + base, pv);
        }
      }
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        double v = 0.0;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) v += red[gg][c * KK + j][r];
        if (a.mode == SPMV_NEGB) v = -v;
        else if (a.mode == SPMV_TRUERES) { v = a.b[base + j] - v; dots[j] = fma(v, v, dots[j]); }
        else if (a.mode == SPMV_PQ) dots[j] = fma(pv[j], v, dots[j]);
        a.y[base + j] = v;
      }
    }
  }
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
  constexpr int BR = 32, W = 2 * P + 1, WN = BR + 2 * P;
  constexpr int NA = ELASTIC ? 3 : NC, NB = ELASTIC ? 3 : NC;
  constexpr size_t bytes = sizeof(double) * (2 * G * NB * WN * KK + G * NA * KK * BR);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmv_sm<P, NC, KK, ELASTIC, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = true;
  }
  k_spmv_sm<P, NC, KK, ELASTIC, G><<<nb, 32 * G, bytes, s>>>(a);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) k_spmv_fin<KK><<<1, 1024, 0, s>>>(a, nb);
}

template <int P, int NC, int KK>
static void spmv_kk(const SpmvArgs& a, cudaStream_t s) {
  {
    const unsigned int nb = (unsigned int)((a.g.npts + 31) / 32);
    if (a.elastic) {
      if constexpr (NC == 3) launch_sm<P, 3, KK, true, 4>(a, nb, s);
    } else {
      launch_sm<P, NC, KK, false, 8>(a, nb, s);
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
void launch_spmv(const SpmvArgs& a, cudaStream_t s) {
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
