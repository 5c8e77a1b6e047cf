// Single-read symmetric stencil SpMV for the 3D half-symmetric operators (sm_100a, fp64;
// DESIGN.md "Symmetric SpMV").  M and K are symmetric (M_ij = sum_q w|J| B_i B_j, the
// stiffness the same with gradients), so only the offsets o >= 0 (lexicographic, z major) of a row
// are stored, and every stored coefficient c(i, o) serves two products:
//   own    y[i]        += c(i, o) x[i + s(o)]      (o >= 0)
//   mirror y[i + s(o)] += c(i, o) x[i]             (o >  0)          s(o) = o1 + o2 nx + o3 nx ny.
// The two-pass kernel (spmv_core.cuh spmv_block_half) fetched each coefficient a second time for
// the mirror term, from a row s(o) away: an L2 miss in 3D, so it moved twice the compulsory bytes.
// Here each coefficient is read exactly once.
//
// Walk.  A CTA owns one x-segment (XS <= 32 points) of TY consecutive y-lines and a chunk of
// source z-planes [Z0, Z1); warp w = y-line y0 + w, lane = x.  It walks the TARGET planes
// Z = Z0 .. Z1 + P - 1: at step Z it reads, for every o3 = 0..P, the coefficients c(i, o) of its
// source rows i in plane Z - o3 with that o3 (one contiguous 169-offset slice per row block in
// the layout below).  Every product of the step then lands in plane Z:
//   own:    row i (plane Z - o3) gathers x at (x + o1, y + o2, Z)       -> own[o3] in registers
//   mirror: target (x + o1, y + o2, Z) receives c x[i], x[i] of plane Z - o3 in registers
// so only ONE plane of the input (the window of plane Z, staged in shared memory by cp.async)
// and ONE plane of mirror accumulators are live.  For fixed (o1, o2) the mirror products of all
// o3 share the target, so they are summed in registers first; the sum moves to the target lane
// x + o1 by a warp shuffle (values wrapping around the 32 lanes belong to the neighbouring
// segments: a per-lane spill accumulator), and after all o1 one read-modify-write per o2 goes to
// the warp's private (2P+1)-line accumulator slab (no inter-warp conflicts, no atomics).
// After the step the CTA sums the TY slabs in a fixed order and adds the plane to y with fp64
// reductions in L2 (red.global.add.f64): y's own rows plus the halo rows other CTAs also reach.
// A row's own sum is complete after step z + P (registers ring-shifted per step) and is added
// the same way.  y is cleared (or set to b) by k_sym_init first; the PCG dot products of
// SPMV_PQ / SPMV_TRUERES follow in k_sym_dots + k_spmv_fin.
//
// Layout (genalpha.cu sym_layout, written by the assembly): rows are grouped in blocks of one
// x-segment of XS points (nx split into nseg equal segments, XS a multiple of 4 so a warp load is
// XS*8 bytes of whole 32-byte sectors), block b = seg + nseg (y + ny z); coefficient h = o - S/2
// (0 <= h < Sh = (S+1)/2) of lane l at coef[(b Sh + h) 32 + l] (lanes XS..31 unused, never read).
// Offsets of one o3 are contiguous.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ops.cuh"

namespace ga {

template <int KK>
__device__ __forceinline__ void red_add(double* p, double v) {
  // fp64 reduction in L2 (no return value: RED, not ATOM)
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// D: coefficient rows (one o1 of one o2 stage: the P+1 values c(i, (o1, o2, o3)), o3 = 0..P) a
// warp keeps in flight in registers, D <= 2P + 1 (the prefetch runs at most one stage ahead)
template <int P, int KK, int TY, int D>
struct SymShape {
  static constexpr int W = 2 * P + 1;
  static constexpr int XW = 32 + 2 * P;  // staged x positions: x0 - P .. x0 + 31 + P
  static constexpr int YW = TY + 2 * P;  // staged y lines:     y0 - P .. y0 + TY - 1 + P
  static constexpr int WIN = YW * XW * KK;
  static constexpr int SLAB = W * XW * KK;  // one warp's mirror accumulators: lines y + o2
  static constexpr size_t bytes = sizeof(double) * (2 * WIN + TY * SLAB);
};

template <int P, int KK, int TY, int D>
__global__ void __launch_bounds__(32 * TY, (TY >= 8 ? 1 : 2)) k_spmv_sym(SpmvArgs a, int nty, int zlen) {
  using SS = SymShape<P, KK, TY, D>;
  constexpr int W = SS::W, XW = SS::XW, YW = SS::YW, WIN = SS::WIN, SLAB = SS::SLAB;
  constexpr int NT = 32 * TY;
  constexpr int U = (KK % 2 == 0) ? 2 : 1;  // doubles per cp.async of the window
  constexpr int R = W % D;                  // rotation of the prefetch registers per stage
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  count_launch(a.st);
  extern __shared__ __align__(16) double smem_sym[];
  double* win0 = smem_sym;
  double* win1 = smem_sym + WIN;
  double* slab = smem_sym + 2 * WIN;
  const GridDesc g = a.g;
  const int nseg = a.snseg;
  const long long Sh = ((long long)W * W * W + 1) / 2;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int seg = blockIdx.x % nseg;
  const int ty = (blockIdx.x / nseg) % nty;
  const int chunk = blockIdx.x / (nseg * nty);
  const int x0 = seg * SYM_STRIDE, y0 = ty * TY;
  const int Z0 = chunk * zlen, Z1 = min(g.nz, Z0 + zlen);
  const int Zend = min(g.nz, Z1 + P);
  const int x = x0 + lane, y = y0 + w;
  const bool lrow = x < g.nx && y < g.ny;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  const double sign = (a.mode == SPMV_NEGB || a.mode == SPMV_TRUERES) ? -1.0 : 1.0;
  // stage the input window of plane Z (cp.async, no registers); lines past ny - 1 + P are read
  // only by rows outside the grid: zero-filled, so no load leaves the vector's guard
  const int ylim = g.ny - 1 + P;
  auto issue_win = [&](int Z, double* dst) {
    for (int q = threadIdx.x; q < WIN / U; q += NT) {
      const int e = q * U;
      const int j = e % KK, pos = (e / KK) % XW, l = e / (KK * XW);
      const int yy = y0 - P + l;
      if (yy <= ylim) {
        const long long gi = g.guard + (x0 - P + pos) + sy * yy + sz * Z;
        const unsigned int d = (unsigned int)__cvta_generic_to_shared(dst + e);
        const double* src = a.x + gi * KK + j;
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
  // ---- coefficient prefetch, D rows ahead of the consumer, across stage and step ends.
  // Row (Z, o2, o1) = the P+1 coefficients c(i, (o1, o2, o3)) of this lane's row i in the source
  // planes Z - o3: P+1 coalesced 8-byte loads (lane = x) into registers.  Rows that are not
  // stored (o3 = 0, (o2, o1) < 0), planes outside the chunk and lanes outside the grid read the
  // zero block a.symzero (L2-resident) instead: every load is unconditional, with a
  // compile-time offset.  Stage = one (Z, o2), 2P+1 rows; A = the consumer's stage, B = the next
  // one (the consumer's u + D < 2P+1 decides at compile time which a prefetch belongs to).
  const double* zb = a.symzero + lane;  // zero block (Sh x 32 doubles), this lane's column
  auto block = [&](int z) -> const double* {  // row block of plane z, or the zero block
    if (!lrow || z < Z0 || z >= Z1) return zb;
    return a.coef + ((long long)(seg + (long long)nseg * (y + (long long)g.ny * z)) * Sh) * SYM_STRIDE + lane;
  };
  const double* icb[P + 1];  // block of source plane iZ - o3 (iZ = step of stage B)
#pragma unroll
  for (int o3 = 0; o3 <= P; ++o3) icb[o3] = zb;
  icb[0] = block(Z0);
  int iZ = Z0;
  const double* pA[P + 1];  // stage A rows at o1 = -P
  const double* pB[P + 1];
#pragma unroll
  for (int o3 = 0; o3 <= P; ++o3) {
    pA[o3] = icb[o3] + (W * W * o3 - W * P - P) * SYM_STRIDE;
    pB[o3] = pA[o3] + W * SYM_STRIDE;
  }
  int o2A = -P, o2B = 1 - P;
  auto load_row = [&](const double* const (&pp)[P + 1], int o2, int u, double (&c)[P + 1]) {
    const int o1 = u - P;
    const bool z0own = o1 >= 0 ? o2 >= 0 : o2 > 0;  // o3 = 0 stores only (o2, o1) >= 0
    const double* p0 = z0own ? pp[0] + u * SYM_STRIDE : zb;
    c[0] = __ldg(p0);
#pragma unroll
    for (int o3 = 1; o3 <= P; ++o3) c[o3] = __ldg(pp[o3] + u * SYM_STRIDE);
  };
  // the consumer moves to the next stage: B becomes A, B advances (into the next step after o2 = P)
  auto advance_stage = [&]() {
#pragma unroll
    for (int o3 = 0; o3 <= P; ++o3) pA[o3] = pB[o3];
    o2A = o2B;
    if (o2B == P) {
      ++iZ;
#pragma unroll
      for (int o3 = P; o3 > 0; --o3) icb[o3] = icb[o3 - 1];
      icb[0] = block(iZ);
      o2B = -P;
#pragma unroll
      for (int o3 = 0; o3 <= P; ++o3) pB[o3] = icb[o3] + (W * W * o3 - W * P - P) * SYM_STRIDE;
    } else {
      ++o2B;
#pragma unroll
      for (int o3 = 0; o3 <= P; ++o3) pB[o3] += W * SYM_STRIDE;
    }
  };
  // ---- consumer rings over the source planes Z - o3, o3 = 0..P (index = o3; shifted per step)
  double own[P + 1][KK], xsrc[P + 1][KK];
  bool vpl[P + 1];
#pragma unroll
  for (int o3 = 0; o3 <= P; ++o3) {
    vpl[o3] = false;
#pragma unroll
    for (int j = 0; j < KK; ++j) own[o3][j] = xsrc[o3][j] = 0.0;
  }
  for (int q = threadIdx.x; q < TY * SLAB; q += NT) slab[q] = 0.0;
  issue_win(Z0, win0);
  double cq[D][P + 1];  // prefetched rows; row u of a stage sits in cq[u % D]
#pragma unroll
  for (int u = 0; u < D; ++u) load_row(pA, o2A, u, cq[u]);
  double* mslab = slab + w * SLAB;
#pragma unroll 1
  for (int Z = Z0; Z < Zend; ++Z) {
    double* cur = ((Z - Z0) & 1) ? win1 : win0;
    double* nxt = ((Z - Z0) & 1) ? win0 : win1;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // this step's window (issued a step ago)
    __syncthreads();  // window of plane Z staged; last step's slabs combined and cleared
    if (Z + 1 < Zend) issue_win(Z + 1, nxt);
    // shift the rings: slot o3 now holds source plane Z - o3
#pragma unroll
    for (int o3 = P; o3 > 0; --o3) {
      vpl[o3] = vpl[o3 - 1];
#pragma unroll
      for (int j = 0; j < KK; ++j) { own[o3][j] = own[o3 - 1][j]; xsrc[o3][j] = xsrc[o3 - 1][j]; }
    }
    vpl[0] = Z < Z1;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      own[0][j] = 0.0;
      xsrc[0][j] = (lrow && Z < Z1) ? cur[((w + P) * XW + lane + P) * KK + j] : 0.0;
    }
    bool vp[P + 1];
#pragma unroll
    for (int o3 = 0; o3 <= P; ++o3) vp[o3] = vpl[o3] && lrow;
#pragma unroll 1
    for (int o2i = 0; o2i < W; ++o2i) {
      const int o2 = o2i - P;
      const double* xr = cur + ((w + o2i) * XW + lane) * KK;  // window line y + o2, position x + o1 + P
      double tm[KK], ts[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) tm[j] = ts[j] = 0.0;
#pragma unroll
      for (int u = 0; u < W; ++u) {
        const int o1 = u - P;
        double c[P + 1];
#pragma unroll
        for (int o3 = 0; o3 <= P; ++o3) c[o3] = cq[u % D][o3];
        // refill this register slot with the row D ahead (this stage or the next)
        if (u + D < W) load_row(pA, o2A, u + D, cq[u % D]);
        else load_row(pB, o2B, u + D - W, cq[u % D]);
        double xv[KK];
#pragma unroll
        for (int j = 0; j < KK; ++j) xv[j] = xr[u * KK + j];
        const bool z0mir = o2 > 0 || (o2 == 0 && o1 > 0);  // o3 = 0: no mirror term at o = 0
        double m[KK];
#pragma unroll
        for (int j = 0; j < KK; ++j) m[j] = 0.0;
#pragma unroll
        for (int o3 = 0; o3 <= P; ++o3) {
          const double cm = (o3 > 0 || z0mir) ? c[o3] : 0.0;
#pragma unroll
          for (int j = 0; j < KK; ++j) {
            own[o3][j] = fma(c[o3], xv[j], own[o3][j]);
            m[j] = fma(cm, xsrc[o3][j], m[j]);
          }
        }
        // mirror products of source lane l go to target lane l + o1
        const int src = (lane - o1) & 31;
        const bool main = (lane - o1 >= 0) && (lane - o1 < 32);
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          const double v = __shfl_sync(0xffffffffu, m[j], src);
          if (main) tm[j] += v; else ts[j] += v;
        }
      }
      // the next stage's row u sits in cq[(u + W) % D]: rotate so it is in cq[u % D]
      if constexpr (R != 0) {
        double t[D][P + 1];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int o3 = 0; o3 <= P; ++o3) t[i][o3] = cq[(i + R) % D][o3];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int o3 = 0; o3 <= P; ++o3) cq[i][o3] = t[i][o3];
      }
      advance_stage();
      // one read-modify-write per o2 into this warp's slab line y + o2 (private: no conflicts)
      double* sl = mslab + o2i * XW * KK;
#pragma unroll
      for (int j = 0; j < KK; ++j) sl[(lane + P) * KK + j] += tm[j];
      if (lane < P) {
#pragma unroll
        for (int j = 0; j < KK; ++j) sl[(lane + 32 + P) * KK + j] += ts[j];
      } else if (lane >= 32 - P) {
#pragma unroll
        for (int j = 0; j < KK; ++j) sl[(lane - 32 + P) * KK + j] += ts[j];
      }
    }
    // own sums complete after step z + P (or at the last plane of the grid)
#pragma unroll
    for (int o3 = 0; o3 <= P; ++o3) {
      if (vp[o3] && (o3 == P || Z == g.nz - 1)) {
        double* yp = a.y + (g.guard + x + sy * y + sz * (Z - o3)) * KK;
#pragma unroll
        for (int j = 0; j < KK; ++j) red_add<KK>(yp + j, sign * own[o3][j]);
      }
    }
    __syncthreads();  // every warp's slab of plane Z is complete
    // fixed-order sum of the TY slabs -> plane Z of y (rows of this CTA and the halo other CTAs
    // also reach); each slab entry is read once and cleared for the next step
    for (int q = threadIdx.x; q < YW * XW; q += NT) {
      const int l = q / XW, pos = q % XW;
      double sum[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) sum[j] = 0.0;
      const int wlo = max(0, l - 2 * P), whi = min(TY - 1, l);
      for (int ww = wlo; ww <= whi; ++ww) {
        double* e = slab + ww * SLAB + ((l - ww) * XW + pos) * KK;
#pragma unroll
        for (int j = 0; j < KK; ++j) { sum[j] += e[j]; e[j] = 0.0; }
      }
      const int gx = x0 - P + pos, gy = y0 - P + l;
      if (gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny) {
        double* yp = a.y + (g.guard + gx + sy * gy + sz * Z) * KK;
#pragma unroll
        for (int j = 0; j < KK; ++j)
          if (sum[j] != 0.0) red_add<KK>(yp + j, sign * sum[j]);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // nothing lands in shared memory after exit
}

// y = 0 (apply, -K s, q = M p) or y = b (r = b - M x) on the grid points, before k_spmv_sym
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_sym_init(SpmvArgs a) {
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  const long long tot = g.npts * KK;
  const long long base = g.guard * KK;
  for (long long e = (long long)gtid(); e < tot; e += (long long)gridDim.x * blockDim.x)
    a.y[base + e] = (a.mode == SPMV_TRUERES) ? a.b[base + e] : 0.0;
}

// per-block partial dot products after k_spmv_sym: p.q (SPMV_PQ) or r.r (SPMV_TRUERES)
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_sym_dots(SpmvArgs a) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  const double* u = a.mode == SPMV_PQ ? a.x : a.y;
  for (long long i = (long long)gtid(); i < g.npts; i += (long long)gridDim.x * blockDim.x) {
    const long long o = (g.guard + i) * KK;
#pragma unroll
    for (int j = 0; j < KK; ++j) dots[j] = fma(u[o + j], a.y[o + j], dots[j]);
  }
  block_sum<KK>(dots);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < KK; ++j) a.partial[(size_t)blockIdx.x * KK + j] = dots[j];
  }
}

// plan only (eff_out != nullptr): the modelled efficiency of this TY with its best chunk count,
// no launch
template <int P, int KK, int TY, int D>
static bool launch_sym_ty(const SpmvArgs& a, cudaStream_t s, double* eff_out = nullptr) {
  using SS = SymShape<P, KK, TY, D>;
  if constexpr (SS::bytes > 225 * 1024) {
    return false;
  } else {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_spmv_sym<P, KK, TY, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)SS::bytes) != cudaSuccess)
        return false;
      attr = true;
    }
    const GridDesc& g = a.g;
    const int nty = (g.ny + TY - 1) / TY;
    const long long nxy = (long long)a.snseg * nty;
    // z-chunks: each coefficient is still read once (a chunk owns its source planes); a chunk
    // adds P partial steps (window / flush overhead, predicated work).  Pick the chunk count that
    // fills the resident CTA slots best: efficiency = work / (whole waves x slots), weighted by
    // the partial-step overhead zlen / (zlen + P)
    static int slots = 0;
    if (!slots) {
      int per_sm = 0, nsm = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_sym<P, KK, TY, D>, 32 * TY, SS::bytes);
      slots = std::max(1, per_sm) * std::max(1, nsm);
    }
    static int force_nch = -1;
    if (force_nch < 0) { const char* e = getenv("GA_SYM_NCH"); force_nch = e ? std::max(1, atoi(e)) : 0; }
    long long nch = 1;
    double best = -1.0;
    for (long long c = 1; c <= std::min<long long>(g.nz, 64); ++c) {
      const long long zl = (g.nz + c - 1) / c, cc = (g.nz + zl - 1) / zl;
      const double ctas = (double)(nxy * cc), waves = std::ceil(ctas / slots);
      const double eff = ctas / (waves * slots) * (double)zl / (zl + 0.5 * P);
      if (eff > best + 1e-9) { best = eff; nch = cc; }
    }
    if (eff_out) { *eff_out = best * (double)g.ny / ((double)nty * TY); return true; }
    if (force_nch > 0) nch = std::min<long long>(force_nch, g.nz);
    const int zlen = (int)((g.nz + nch - 1) / nch);
    nch = (g.nz + zlen - 1) / zlen;
    const unsigned int nb = (unsigned int)(nxy * nch);
    const unsigned int ib = 148 * 4;
    k_sym_init<KK><<<ib, NTHREADS, 0, s>>>(a);
    k_spmv_sym<P, KK, TY, D><<<nb, 32 * TY, SS::bytes, s>>>(a, nty, zlen);
    if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) {
      k_sym_dots<KK><<<ib, NTHREADS, 0, s>>>(a);
      launch_spmv_fin(a, ib, s);
    }
    return true;
  }
}

// warps (y-lines) per CTA: TY = 4 (two CTAs per SM) unless 2-warp CTAs fill the resident slots
// clearly better in whole waves (modelled efficiency of launch_sym_ty; measured: C3 p=4 n=96
// 747 -> 616 us per M apply with TY = 2, equal at p=4 n=192, TY = 4 3 % faster at p=2 n=192);
// GA_SYM_TY = 2 / 4 / 8 overrides (measurement)
template <int P, int KK>
static void launch_sym_kk(const SpmvArgs& a, cudaStream_t s) {
  static int ty = -1;
  if (ty < 0) {
    const char* e = getenv("GA_SYM_TY");
    ty = e ? atoi(e) : 0;
  }
  constexpr int D = (2 * P + 1) < 4 ? (2 * P + 1) : 4;  // prefetched rows (at most one stage ahead)
  if (ty == 0) {
    double e4 = 0.0, e2 = 0.0;
    const bool ok4 = launch_sym_ty<P, KK, 4, D>(a, s, &e4);
    const bool ok2 = launch_sym_ty<P, KK, 2, D>(a, s, &e2);
    if (ok4 && !(ok2 && e2 > 1.08 * e4)) { launch_sym_ty<P, KK, 4, D>(a, s); return; }
    launch_sym_ty<P, KK, 2, D>(a, s);
    return;
  }
  if (ty >= 8 && launch_sym_ty<P, KK, 8, D>(a, s)) return;
  if (ty >= 4 && launch_sym_ty<P, KK, 4, D>(a, s)) return;
  launch_sym_ty<P, KK, 2, D>(a, s);
}

template <int P>
static void launch_sym_p(const SpmvArgs& a, cudaStream_t s) {
  switch (a.kk) {
    case 1: launch_sym_kk<P, 1>(a, s); break;
    case 2: launch_sym_kk<P, 2>(a, s); break;
    case 3: launch_sym_kk<P, 3>(a, s); break;
    default: launch_sym_kk<P, 4>(a, s); break;
  }
}

void launch_spmv_sym(const SpmvArgs& a, cudaStream_t s) {
  switch (a.p) {
    case 1: launch_sym_p<1>(a, s); break;
    case 2: launch_sym_p<2>(a, s); break;
    case 3: launch_sym_p<3>(a, s); break;
    case 4: launch_sym_p<4>(a, s); break;
    case 5: launch_sym_p<5>(a, s); break;
    case 6: launch_sym_p<6>(a, s); break;
    default: launch_sym_p<7>(a, s); break;
  }
}

}  // namespace ga
