// Device core of the warp-staged stencil SpMV (included by spmv.cu and the
// persistent solver in ops.cu).
#pragma once
#include "ops.cuh"

namespace ga {

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

// Warp-owned row block: warp w of the block owns
// the 32 consecutive rows rb = rbg*G + w (lane = row: 256-byte coalesced
// coefficient loads from the 32-row slice) and walks all offset lines
// (o3, o2); per line it stages its (32 + 2P)-point input window in its own
// shared-memory slice (__syncwarp only) while the next line's window and
// coefficients are prefetched into registers.  Warps are independent: no
// block barrier, so many row blocks are in flight per SM.
// FUSE: the fused PCG direction update (a.fuse_p) is compiled in (persistent solver only);
// the standalone kernel never uses it, which saves the p_old prefetch registers.
template <int P, int NC, int KK, bool ELASTIC, int G, bool FUSE = true>
__device__ __forceinline__ void spmv_block(const SpmvArgs& a, long long rbg, double* smem_spmv, double (&dots)[KK]) {
  constexpr int BR = 32;
  constexpr int W = 2 * P + 1, WN = BR + 2 * P;
  constexpr int NA = ELASTIC ? 3 : NC, NB = ELASTIC ? 3 : NC;
  constexpr int NCF = ELASTIC ? 9 : 1;  // coefficient arrays per offset
  auto win = reinterpret_cast<double (*)[2][NB][WN][KK]>(smem_spmv);  // [G][2][NB][WN][KK]
  const GridDesc g = a.g;
  const int r = threadIdx.x & 31, gq = threadIdx.x >> 5;
  const long long rb = rbg * G + gq;
  const long long i0 = rb * BR;
  if (i0 >= g.npts) return;  // whole warp
  if (a.skip && a.skip[rb]) return;  // no free row in this block (masked grid)
  const long long i = i0 + r;
  const bool valid = i < g.npts;
  const long long icl = valid ? i : (g.npts - 1);  // clamp coefficient reads of the tail rows
  const int W3 = (g.dim == 3) ? W : 1;
  const int P3 = (g.dim == 3) ? P : 0;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  const long long S = (long long)W * W * W3;
  const double* xin = a.x;
  const double* __restrict__ cslice = a.coef + (icl >> 5) * NCF * S * 32 + (icl & 31);
  // fused PCG direction: the input window is p_new = z + beta p_old (z on the first iteration)
  const bool fuse = FUSE && a.mode == SPMV_PQ && a.fuse_p;
  const bool mix = fuse && !a.fpfirst;
  if (fuse) xin = a.z;
  // raw window loads (the p_old part is combined when the window is staged,
  // one line later, so the prefetch really overlaps the current line)
  auto fetch_win = [&](int line, int q, int c, double (&v)[KK], double (&vo)[KK]) {
    const int o3 = line / W - P3, o2 = line % W - P;
    const long long pos = g.guard + i0 - P + q + o3 * sz + o2 * sy;
    const long long e = ((long long)c * g.padded + pos) * KK;
    load_row<KK>(xin + e, v);
    if (mix) load_row<KK>(a.p0 + e, vo);
  };
  auto staged = [&](const double (&v)[KK], const double (&vo)[KK], int j) {
    return mix ? fma(a.fbeta[j], vo[j], v[j]) : v[j];
  };
  const int nlines = W3 * W;
  const bool two = r < 2 * P;
  double acc[NA][KK];
#pragma unroll
  for (int c = 0; c < NA; ++c)
#pragma unroll
    for (int j = 0; j < KK; ++j) acc[c][j] = 0.0;
  double pw[2][NB][KK], po[2][NB][KK];
  double cf[ELASTIC ? 1 : W];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    fetch_win(0, r, c, pw[0][c], po[0][c]);
    if (two) fetch_win(0, BR + r, c, pw[1][c], po[1][c]);
  }
  if constexpr (!ELASTIC) {
#pragma unroll
    for (int o1 = 0; o1 < W; ++o1) cf[o1] = __ldg(cslice + (long long)o1 * 32);
  }
  int buf = 0;
  for (int line = 0; line < nlines; ++line) {
#pragma unroll
    for (int c = 0; c < NB; ++c)
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        win[gq][buf][c][r][j] = staged(pw[0][c], po[0][c], j);
        if (two) win[gq][buf][c][BR + r][j] = staged(pw[1][c], po[1][c], j);
      }
    double ccur[ELASTIC ? 1 : W];
    if constexpr (!ELASTIC) {
#pragma unroll
      for (int o1 = 0; o1 < W; ++o1) ccur[o1] = cf[o1];
    }
    __syncwarp();
    if (line + 1 < nlines) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        fetch_win(line + 1, r, c, pw[0][c], po[0][c]);
        if (two) fetch_win(line + 1, BR + r, c, pw[1][c], po[1][c]);
      }
      if constexpr (!ELASTIC) {
#pragma unroll
        for (int o1 = 0; o1 < W; ++o1) cf[o1] = __ldg(cslice + ((long long)(line + 1) * W + o1) * 32);
      }
    }
#pragma unroll
    for (int o1 = 0; o1 < W; ++o1) {
      if constexpr (!ELASTIC) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < KK; ++j) acc[c][j] = fma(ccur[o1], win[gq][buf][c][r + o1][j], acc[c][j]);
      } else {
#pragma unroll
        for (int aa = 0; aa < 3; ++aa)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            const double c9 = __ldg(cslice + ((long long)(aa * 3 + bb) * S + (long long)line * W + o1) * 32);
#pragma unroll
            for (int j = 0; j < KK; ++j) acc[aa][j] = fma(c9, win[gq][buf][bb][r + o1][j], acc[aa][j]);
          }
      }
    }
    buf ^= 1;
  }
  if (!valid) return;
#pragma unroll
  for (int c = 0; c < NA; ++c) {
    const long long base = ((long long)c * g.padded + g.guard + i) * KK;
    double pv[KK];
    if (a.mode == SPMV_PQ) {
      if (fuse) {
        load_row<KK>(a.z + base, pv);
        if (mix) {
          double po[KK];
          load_row<KK>(a.p0 + base, po);
          if (a.fx) {  // deferred x += alpha_prev p_old
            double xv[KK];
#pragma unroll
            for (int j = 0; j < KK; ++j) xv[j] = a.fx[base + j];
#pragma unroll
            for (int j = 0; j < KK; ++j) a.fx[base + j] = fma(a.falpha[j], po[j], xv[j]);
          }
#pragma unroll
          for (int j = 0; j < KK; ++j) pv[j] = fma(a.fbeta[j], po[j], pv[j]);
        }
#pragma unroll
        for (int j = 0; j < KK; ++j) a.p1[base + j] = pv[j];
      } else {
        load_row<KK>(a.x + base, pv);
      }
    }
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


// Half-symmetric stencil (SURVEY §8a a1 option): only the
// offsets o >= 0 (lexicographic) are stored, coef_h[(row + G)/32][o - S/2][(row + G)%32] with a
// zero guard of G rows before row 0; the other half follows from symmetry,
//   c(i, -o) = c(i - s(o), o),  s(o) = o1 + o2 sy + o3 sz  (M, K symmetric).
// The warp walks the (W3 W + 1)/2 offset lines (o3, o2) >= (0, 0); per line it stages the input
// window at +line (own terms, coefficients of its own rows) and at -line (mirror terms,
// coefficients of the rows i - s(o): one shifted, still contiguous 32-row slice per o1).
template <int P, int NC, int KK, int G>
__device__ __forceinline__ void spmv_block_half(const SpmvArgs& a, long long rbg, double* smem_spmv,
                                                double (&dots)[KK]) {
  constexpr int BR = 32;
  constexpr int W = 2 * P + 1, WN = BR + 2 * P;
  auto win = reinterpret_cast<double (*)[2][2][NC][WN][KK]>(smem_spmv);  // [G][buf][own/mirror][NC][WN][KK]
  const GridDesc g = a.g;
  const int r = threadIdx.x & 31, gq = threadIdx.x >> 5;
  const long long rb = rbg * G + gq;
  const long long i0 = rb * BR;
  if (i0 >= g.npts) return;
  if (a.skip && a.skip[rb]) return;  // no free row in this block (masked grid)
  const long long i = i0 + r;
  const bool valid = i < g.npts;
  const long long icl = valid ? i : (g.npts - 1);
  const int W3 = (g.dim == 3) ? W : 1;
  const int P3 = (g.dim == 3) ? P : 0;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  const long long Sh = ((long long)W * W * W3 + 1) / 2;
  const long long hg = a.hguard;
  const int nlh = (W3 * W + 1) / 2;
  const int c2 = P + W * P3;  // lin2 of the centre line
  auto rowc = [&](long long row, long long hidx) -> double {  // coef_h of a (guard-shifted) row
    const long long rr = row + hg;
    return __ldg(a.coef + ((rr >> 5) * Sh + hidx) * 32 + (rr & 31));
  };
  auto fetch_win = [&](int t, int sign, int q, int c, double (&v)[KK]) {
    const int lin2 = c2 + t, o3 = lin2 / W - P3, o2 = lin2 % W - P;
    const long long pos = g.guard + i0 - P + q + sign * (o3 * sz + o2 * sy);
    load_row<KK>(a.x + ((long long)c * g.padded + pos) * KK, v);
  };
  auto fetch_coef = [&](int t, double (&co)[W], double (&cm)[W]) {
    const int lin2 = c2 + t, o3 = lin2 / W - P3, o2 = lin2 % W - P;
    const long long sline = o3 * sz + o2 * sy;
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int o1 = u - P;
      const long long hidx = o1 + (long long)W * t;
      co[u] = (t > 0 || o1 >= 0) ? rowc(icl, hidx) : 0.0;
      cm[u] = (t > 0 || o1 > 0) ? rowc(icl - (o1 + sline), hidx) : 0.0;
    }
  };
  const bool two = r < 2 * P;
  double acc[NC][KK];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int j = 0; j < KK; ++j) acc[c][j] = 0.0;
  double pw[2][2][NC][KK];  // [own/mirror][first/second part of the window]
  double cf[W], cm[W];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int sgn = 0; sgn < 2; ++sgn) {
      fetch_win(0, sgn ? -1 : 1, r, c, pw[sgn][0][c]);
      if (two) fetch_win(0, sgn ? -1 : 1, BR + r, c, pw[sgn][1][c]);
    }
  fetch_coef(0, cf, cm);
  int buf = 0;
  for (int t = 0; t < nlh; ++t) {
#pragma unroll
    for (int sgn = 0; sgn < 2; ++sgn)
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          win[gq][buf][sgn][c][r][j] = pw[sgn][0][c][j];
          if (two) win[gq][buf][sgn][c][BR + r][j] = pw[sgn][1][c][j];
        }
    double co[W], cmc[W];
#pragma unroll
    for (int u = 0; u < W; ++u) { co[u] = cf[u]; cmc[u] = cm[u]; }
    __syncwarp();
    if (t + 1 < nlh) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int sgn = 0; sgn < 2; ++sgn) {
          fetch_win(t + 1, sgn ? -1 : 1, r, c, pw[sgn][0][c]);
          if (two) fetch_win(t + 1, sgn ? -1 : 1, BR + r, c, pw[sgn][1][c]);
        }
      fetch_coef(t + 1, cf, cm);
    }
#pragma unroll
    for (int u = 0; u < W; ++u) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          acc[c][j] = fma(co[u], win[gq][buf][0][c][r + u][j], acc[c][j]);           // x[i + o]
          acc[c][j] = fma(cmc[u], win[gq][buf][1][c][r + 2 * P - u][j], acc[c][j]);  // x[i - o]
        }
    }
    buf ^= 1;
  }
  if (!valid) return;
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



}  // namespace ga
