// Stencil SpMV of the hot path (sm_100a, fp64): y = A x on the column-index-free
// layout coef[o][row] for all lock-stepped right-hand sides at once.  Modes:
// apply, -K s (right-hand sides b_j = -K s_j), q = M p with the
// PCG direction update and the p.q reduction / alpha fused,
// r = b - M x (refinement restart, R8).
#include <cuda_runtime.h>

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

// Shared-memory staged stencil SpMV.  A block of
// BR x G threads owns BR consecutive rows; thread (r, g) handles row r for the
// offset lines (o3, o2) = g, g+G, ... .  Each chunk of G offset lines has its
// input windows (BR + 2P points each) staged in shared memory by the group
// that uses them (double buffered: the next chunk is prefetched into
// registers while the current one is consumed), so every input value is read
// from L2 once per block and line, coefficient loads are coalesced (thread =
// row), and small grids still keep 16 warps per block in flight.  The G
// partial sums are combined in shared memory in a fixed order.  With SPMV_PQ +
// fuse_p the window is the new PCG direction p = z + beta p_old.
template <int P, int NC, int KK, bool ELASTIC, int G>
__global__ void __launch_bounds__(64 * G) k_spmv_sm(SpmvArgs a) {
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  count_launch(a.st);
  constexpr int BR = 64;
  constexpr int W = 2 * P + 1, WN = BR + 2 * P;
  constexpr int NA = ELASTIC ? 3 : NC, NB = ELASTIC ? 3 : NC;
  extern __shared__ double smem_spmv[];
  auto win = reinterpret_cast<double (*)[G][NB][WN][KK]>(smem_spmv);                        // [2][G][NB][WN][KK]
  auto red = reinterpret_cast<double (*)[NA * KK][BR]>(smem_spmv + 2 * G * NB * WN * KK);   // [G][NA*KK][BR]
  const GridDesc g = a.g;
  const int r = threadIdx.x % BR, gq = threadIdx.x / BR;
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
  auto fetch = [&](int line, int q, int c, double (&v)[KK]) {
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
  const int nlines = W3 * W;
  const int nch = (nlines + G - 1) / G;
  const bool two = r < 2 * P;
  double pre[2][NB][KK];
  {
    const int line = gq;
    if (line < nlines) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        fetch(line, r, c, pre[0][c]);
        if (two) fetch(line, BR + r, c, pre[1][c]);
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          win[0][gq][c][r][j] = pre[0][c][j];
          if (two) win[0][gq][c][BR + r][j] = pre[1][c][j];
        }
      }
    }
  }
  __syncthreads();
  double acc[NA][KK];
#pragma unroll
  for (int c = 0; c < NA; ++c)
#pragma unroll
    for (int j = 0; j < KK; ++j) acc[c][j] = 0.0;
  const bool valid = i < g.npts;
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = ch & 1;
    const int line = ch * G + gq;
    const int nline = line + G;
    const bool more = ch + 1 < nch && nline < nlines;
    if (more) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        fetch(nline, r, c, pre[0][c]);
        if (two) fetch(nline, BR + r, c, pre[1][c]);
      }
    }
    if (valid && line < nlines) {
      const double* cb = a.coef + (long long)line * W * g.cs + i;
      if constexpr (!ELASTIC) {
        double cf[W];
#pragma unroll
        for (int o1 = 0; o1 < W; ++o1) cf[o1] = __ldg(cb + (long long)o1 * g.cs);
#pragma unroll
        for (int o1 = 0; o1 < W; ++o1)
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int j = 0; j < KK; ++j) acc[c][j] = fma(cf[o1], win[buf][gq][c][r + o1][j], acc[c][j]);
      } else {
#pragma unroll
        for (int o1 = 0; o1 < W; ++o1)
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
              const double cf = __ldg(cb + ((long long)(aa * 3 + bb) * S + o1) * g.cs);
#pragma unroll
              for (int j = 0; j < KK; ++j) acc[aa][j] = fma(cf, win[buf][gq][bb][r + o1][j], acc[aa][j]);
            }
      }
    }
    if (more) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          win[buf ^ 1][gq][c][r][j] = pre[0][c][j];
          if (two) win[buf ^ 1][gq][c][BR + r][j] = pre[1][c][j];
        }
    }
    __syncthreads();
  }
  // combine the G groups (fixed order) and run the epilogue in group 0
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
  if (a.mode == SPMV_PQ) {
    double tot[KK];
    if (reduce_last_block<KK>(dots, a.partial, a.counter, tot)) {
      PcgState* pc = a.pcg;
      pc->iter += 1;
      pc->pfirst = 0;
      a.st->loop_iters += 1;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        pc->pq[j] = tot[j];
        if (pc->active[j]) {
          pc->alpha[j] = pc->rz[j] / tot[j];
          pc->its[j] += 1;
        } else {
          pc->alpha[j] = 0.0;
        }
      }
    }
  } else if (a.mode == SPMV_TRUERES) {
    double tot[KK];
    if (reduce_last_block<KK>(dots, a.partial, a.counter, tot)) {
      PcgState* pc = a.pcg;
      pc->iter = 0; pc->first = 1; pc->pfirst = 1; pc->phase = 1;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        pc->alpha[j] = 0.0;
        pc->active[j] = pc->bb[j] > 0.0 ? 1 : 0;
        double thr = a.tol2 * pc->bb[j];
        if (a.refine_rtol2 > 0.0) thr = fmin(thr, a.refine_rtol2 * tot[j]);
        pc->thr[j] = thr;
      }
    }
  }
}

template <int P, int NC, int KK, bool ELASTIC, int G>
static void launch_sm(const SpmvArgs& a, unsigned int nb, cudaStream_t s) {
  constexpr int BR = 64, W = 2 * P + 1, WN = BR + 2 * P;
  constexpr int NA = ELASTIC ? 3 : NC, NB = ELASTIC ? 3 : NC;
  constexpr size_t bytes = sizeof(double) * (2 * G * NB * WN * KK + G * NA * KK * BR);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmv_sm<P, NC, KK, ELASTIC, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    attr = true;
  }
  k_spmv_sm<P, NC, KK, ELASTIC, G><<<nb, 64 * G, bytes, s>>>(a);
}

template <int P, int NC, int KK>
static void spmv_kk(const SpmvArgs& a, cudaStream_t s) {
  {
    const unsigned int nb = (unsigned int)((a.g.npts + 63) / 64);
    if (a.elastic) {
      if constexpr (NC == 3) launch_sm<P, 3, KK, true, 4>(a, nb, s);
    } else if constexpr (NC == 3) {
      launch_sm<P, NC, KK, false, 4>(a, nb, s);
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
