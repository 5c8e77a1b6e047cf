// Hot-path kernels of the explicit order-2k generalized-alpha step (sm_100a, fp64).
//
//  * k_spmv      stencil SpMV y = A x on the column-index-free layout coef[o][row]
//                for all lock-stepped right-hand sides at once (coefficients are
//                read once per k RHS).  Modes: apply, -A x (right-hand sides
//                b_j = -K s_j), q = M p with the p.q reduction and the
//                alpha update fused (PCG), r = b - M x (refinement R8).
//  * k_line      banded Cholesky forward/backward substitution along grid lines:
//                the Kronecker factor Mh_d^{-1} of calM^{-1}.
//  * k_prec_*    diagonal scaling s = sqrt(Dh/D) and additive Schwarz
//                gather / sum, with the r.z and r.r reductions fused.
//  * k_stage     the 3k-variable update of P:408-431 (reading R1) for all blocks
//                at once, per DoF, fused with the next step's predictors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ops.cuh"

namespace ga {

// grid of a reducing grid-stride kernel: one completion atomic per block on a
// single counter, so keep the block count bounded (148 SMs x 8 blocks)
static unsigned int red_grid(long long n) {
  const long long b = (n + NTHREADS - 1) / NTHREADS;
  return (unsigned int)(b < 1184 ? (b > 0 ? b : 1) : 1184);
}

#define CUDA_LAUNCH_CHECK()

// ---------------------------------------------------------------------------
// Preconditioner: scaling, line solves, Schwarz sum
// ---------------------------------------------------------------------------
// x += alpha p, r -= alpha q (when a PCG iteration precedes), then the scaled
// input t = s o r of the (single) patch into z, or of every patch into its box.
// the KK right-hand-side values of one grid point (contiguous, 8 KK-byte aligned): 16-byte
// accesses for even KK
template <int KK>
__device__ __forceinline__ void ld_k(const double* __restrict__ p, double (&v)[KK]) {
  if constexpr (KK % 2 == 0) {
#pragma unroll
    for (int h = 0; h < KK / 2; ++h) {
      const double2 t = reinterpret_cast<const double2*>(p)[h];
      v[2 * h] = t.x;
      v[2 * h + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < KK; ++j) v[j] = p[j];
  }
}
template <int KK>
__device__ __forceinline__ void st_k(double* __restrict__ p, const double (&v)[KK]) {
  if constexpr (KK % 2 == 0) {
#pragma unroll
    for (int h = 0; h < KK / 2; ++h) reinterpret_cast<double2*>(p)[h] = make_double2(v[2 * h], v[2 * h + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < KK; ++j) p[j] = v[j];
  }
}

template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_xr_prec_in(PrecArgs a) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  const long long tot = (long long)a.nvec * g.npts;  // one thread per (component, grid point)
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const long long i = e % g.npts;
  const int c = (int)(e / g.npts);
  const long long base = ((long long)c * g.padded + g.guard + i) * KK;
  double r[KK];
  ld_k<KK>(a.r + base, r);
  if (a.update && !a.pcg->first) {
    const double* pp = (a.pcg->iter & 1) ? a.p1 : a.p0;
    double al[KK];
    bool any = false;
#pragma unroll
    for (int j = 0; j < KK; ++j) { al[j] = a.pcg->alpha[j]; any |= al[j] != 0.0; }
    if (any) {
      double x[KK], p[KK], q[KK];
      ld_k<KK>(a.x + base, x);
      ld_k<KK>(pp + base, p);
      ld_k<KK>(a.q + base, q);
#pragma unroll
      for (int j = 0; j < KK; ++j) {  // alpha_j = 0 (converged block): x, r unchanged bit for bit
        if (al[j] != 0.0) { x[j] = fma(al[j], p[j], x[j]); r[j] = fma(-al[j], q[j], r[j]); }
      }
      st_k<KK>(a.x + base, x);
      st_k<KK>(a.r + base, r);
    }
  }
  if (a.npatch == 1 && a.t[0] == nullptr) {
    const double sv = a.s[0][i];
#pragma unroll
    for (int j = 0; j < KK; ++j) r[j] *= sv;
    st_k<KK>(a.z + base, r);
  }
}
static void launch_xr_prec_in(const PrecArgs& a, cudaStream_t s) {
  const long long tot = (long long)a.nvec * a.g.npts;
  const unsigned int nb = (unsigned int)((tot + NTHREADS - 1) / NTHREADS);
  switch (a.kk) {
    case 1: k_xr_prec_in<1><<<nb, NTHREADS, 0, s>>>(a); break;
    case 2: k_xr_prec_in<2><<<nb, NTHREADS, 0, s>>>(a); break;
    case 3: k_xr_prec_in<3><<<nb, NTHREADS, 0, s>>>(a); break;
    default: k_xr_prec_in<4><<<nb, NTHREADS, 0, s>>>(a); break;
  }
}

// multi-patch prologue fused with the gather (additive Schwarz): one thread per (grid
// point, rhs) applies x += alpha p, r -= alpha q once, then writes s_r o r into the box of every
// patch that contains the point (interface points belong to 2-4 boxes); 32-bit index math
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_xr_gather(PrecArgs a) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  const int npts = (int)g.npts;
  const int tot = a.nvec * npts;  // one thread per (component, grid point): 16-byte accesses for even KK
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const int c = e / npts, i = e - c * npts;
  const long long base = ((long long)c * g.padded + g.guard + i) * KK;
  const bool free_pt = a.mask == nullptr || a.mask[i];  // not free: r = 0, only the boxes get their zeros
  double r[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) r[j] = 0.0;
  if (free_pt) ld_k<KK>(a.r + base, r);
  if (free_pt && a.update && !a.pcg->first) {
    const double* pp = (a.pcg->iter & 1) ? a.p1 : a.p0;
    double al[KK];
    bool any = false;
#pragma unroll
    for (int j = 0; j < KK; ++j) { al[j] = a.pcg->alpha[j]; any |= al[j] != 0.0; }
    if (any) {
      double x[KK], p[KK], q[KK];
      ld_k<KK>(a.x + base, x);
      ld_k<KK>(pp + base, p);
      ld_k<KK>(a.q + base, q);
#pragma unroll
      for (int j = 0; j < KK; ++j)
        if (al[j] != 0.0) { x[j] = fma(al[j], p[j], x[j]); r[j] = fma(-al[j], q[j], r[j]); }
      st_k<KK>(a.x + base, x);
      st_k<KK>(a.r + base, r);
    }
  }
  const int ix = i % g.nx, iyz = i / g.nx;
  const int iy = iyz % g.ny, iz = iyz / g.ny;
  for (int pr = 0; pr < a.npatch; ++pr) {
    const int lx = ix - a.lo[pr][0], ly = iy - a.lo[pr][1], lz = iz - a.lo[pr][2];
    const int bx = a.bd[pr][0], by = a.bd[pr][1], bz = a.bd[pr][2];
    if (lx < 0 || ly < 0 || lz < 0 || lx >= bx || ly >= by || lz >= bz) continue;
    const int bi = lx + bx * (ly + by * lz);
    const long long nbox = (long long)bx * by * bz;
    const double sv = a.s[pr][bi];
    double t[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) t[j] = sv * r[j];
    st_k<KK>(a.t[pr] + ((long long)c * nbox + bi) * KK, t);
  }
}

// multi-patch gather: t_r = s_r o R_r r on the box of patch r
// all patches in one launch: element ranges of the patches are consecutive
__global__ void __launch_bounds__(NTHREADS) k_prec_gather_all(PrecArgs a) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  long long e = (long long)gtid();
  int pr = 0;
  for (; pr < a.npatch; ++pr) {
    const long long n = (long long)a.nvec * a.bd[pr][0] * a.bd[pr][1] * a.bd[pr][2] * a.kk;
    if (e < n) break;
    e -= n;
  }
  if (pr >= a.npatch) return;
  const int bx = a.bd[pr][0], by = a.bd[pr][1], bz = a.bd[pr][2];
  const long long nbox = (long long)bx * by * bz;
  const int j = (int)(e % a.kk);
  const long long ci = e / a.kk;
  const long long bi = ci % nbox;
  const int c = (int)(ci / nbox);
  const int ix = (int)(bi % bx), iy = (int)((bi / bx) % by), iz = (int)(bi / ((long long)bx * by));
  const long long gi = (a.lo[pr][0] + ix) + (long long)g.nx * ((a.lo[pr][1] + iy) + (long long)g.ny * (a.lo[pr][2] + iz));
  const double sv = a.s[pr][bi];
  const double r = a.r[((long long)c * g.padded + g.guard + gi) * a.kk + j];
  a.t[pr][((long long)c * nbox + bi) * a.kk + j] = sv * r;
}

__global__ void __launch_bounds__(NTHREADS) k_prec_gather(PrecArgs a, int pr) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  const int bx = a.bd[pr][0], by = a.bd[pr][1], bz = a.bd[pr][2];
  const long long nbox = (long long)bx * by * bz;
  const long long tot = (long long)a.nvec * nbox * a.kk;
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const int j = (int)(e % a.kk);
  const long long ci = e / a.kk;
  const long long bi = ci % nbox;
  const int c = (int)(ci / nbox);
  const int ix = (int)(bi % bx), iy = (int)((bi / bx) % by), iz = (int)(bi / ((long long)bx * by));
  const long long gi = (a.lo[pr][0] + ix) + (long long)g.nx * ((a.lo[pr][1] + iy) + (long long)g.ny * (a.lo[pr][2] + iz));
  const double sv = a.s[pr][bi];
  const double r = a.r[((long long)c * g.padded + g.guard + gi) * a.kk + j];
  a.t[pr][((long long)c * nbox + bi) * a.kk + j] = sv * r;
}

// Forward then backward substitution with the banded Cholesky factor along
// lines of length len (element stride es); one thread per (comp, line, rhs),
// consecutive threads = consecutive (x, rhs) so y/z lines are coalesced.
// Streaming version for many lines (3D): the loads of the next D elements are
// issued before the D recurrence steps of the current block (software
// pipelining, D independent loads in flight per thread).
template <int P>
__global__ void __launch_bounds__(NTHREADS) k_line(double* __restrict__ t, const double* __restrict__ L, int len,
                                                   long long es, int na, long long sa, int nb, long long sb, int kk,
                                                   int nvec, long long sc, DevStatus* st) {
  constexpr int D = 8;
  if (st->status != 0) return;
  count_launch(st);
  const long long nl = (long long)nvec * nb * na * kk;
  const long long l = (long long)gtid();
  if (l >= nl) return;
  const int j = (int)(l % kk);
  long long rem = l / kk;
  const int ia = (int)(rem % na);
  rem /= na;
  const int ib = (int)(rem % nb);
  const int c = (int)(rem / nb);
  double* base = t + c * sc + ib * sb + ia * sa + j;
  double y[P];
#pragma unroll
  for (int u = 0; u < P; ++u) y[u] = 0.0;
  double nxt[D];
#pragma unroll
  for (int d = 0; d < D; ++d) nxt[d] = d < len ? base[(long long)d * es] : 0.0;
  // forward: y_i = (t_i - sum_{u=1..P} L_{i,i-u} y_{i-u}) / L_ii
  for (int i0 = 0; i0 < len; i0 += D) {
    double cur[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cur[d] = nxt[d];
#pragma unroll
    for (int d = 0; d < D; ++d) nxt[d] = (i0 + D + d < len) ? base[(long long)(i0 + D + d) * es] : 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int i = i0 + d;
      if (i < len) {
        double v = cur[d];
        const double* Li = L + (long long)i * (P + 1);
#pragma unroll
        for (int u = P; u >= 1; --u) v = fma(-__ldg(Li + u), y[u - 1], v);
        v *= __ldg(Li);
#pragma unroll
        for (int u = P - 1; u >= 1; --u) y[u] = y[u - 1];
        y[0] = v;
        base[(long long)i * es] = v;
      }
    }
  }
  // backward: z_i = (y_i - sum_{u=1..P} L_{i+u,i} z_{i+u}) / L_ii   (L padded with P zero rows)
#pragma unroll
  for (int u = 0; u < P; ++u) y[u] = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) nxt[d] = (len - 1 - d >= 0) ? base[(long long)(len - 1 - d) * es] : 0.0;
  for (int i0 = len - 1; i0 >= 0; i0 -= D) {
    double cur[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cur[d] = nxt[d];
#pragma unroll
    for (int d = 0; d < D; ++d) nxt[d] = (i0 - D - d >= 0) ? base[(long long)(i0 - D - d) * es] : 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int i = i0 - d;
      if (i >= 0) {
        double v = cur[d];
#pragma unroll
        for (int u = P; u >= 1; --u) v = fma(-__ldg(L + (long long)(i + u) * (P + 1) + u), y[u - 1], v);
        v *= __ldg(L + (long long)i * (P + 1));
#pragma unroll
        for (int u = P - 1; u >= 1; --u) y[u] = y[u - 1];
        y[0] = v;
        base[(long long)i * es] = v;
      }
    }
  }
}

template <int P>
static void line_launch(double* t, const double* L, int len, long long es, int na, long long sa, int nb,
                        long long sb, int kk, int nvec, long long sc, DevStatus* st, cudaStream_t s) {
  const long long nl = (long long)nvec * nb * na * kk;
  const unsigned int blocks = (unsigned int)((nl + NTHREADS - 1) / NTHREADS);
  k_line<P><<<blocks, NTHREADS, 0, s>>>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st);
}
static void line_dispatch(int p, double* t, const double* L, int len, long long es, int na, long long sa, int nb,
                          long long sb, int kk, int nvec, long long sc, DevStatus* st, cudaStream_t s) {
  switch (p) {
    case 1: line_launch<1>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
    case 2: line_launch<2>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
    case 3: line_launch<3>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
    case 4: line_launch<4>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
    case 5: line_launch<5>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
    case 6: line_launch<6>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
    default: line_launch<7>(t, L, len, es, na, sa, nb, sb, kk, nvec, sc, st, s); break;
  }
}

}  // namespace ga

#include "tile_core.cuh"

namespace ga {

// ---------------------------------------------------------------------------
// Streaming line solver with fused PCG prologue/epilogue (single patch, many
// lines: 3D).  One thread per (comp, line, rhs); consecutive threads are
// consecutive (x, rhs) slots so y/z lines are coalesced.  The loads of the
// next D elements are issued before the D recurrence steps of the current
// block (software pipelining).  PRO: input = s o (r - alpha q) with
// x += alpha p, r updated in place.  EPI: output z = s o (L^T)^{-1} y, with
// the r.z / r.r partial sums and the PCG scalar step F1 in the last block.
// ---------------------------------------------------------------------------
struct LineArgs {
  double* t;
  const double* L;
  int len;
  long long es;
  int na, nb, kk, nvec;
  long long sa, sb, sc;
  const double* s;
  double *x, *r;
  const double *p, *q;
  PcgState* pcg;
  DevStatus* st;
  double* partial;
  unsigned int* counter;
  int maxit, update;
  unsigned long long cond;
};

template <int P, bool PRO, bool EPI>
__global__ void __launch_bounds__(NTHREADS) k_line_sf(LineArgs a) {
  constexpr int D = (PRO || EPI) ? 8 : 16;
  if (a.st->status != 0) return;  // uniform
  count_launch(a.st);
  const long long nl = (long long)a.nvec * a.nb * a.na * a.kk;
  const long long l = (long long)gtid();
  double acc[2 * KMAX];
#pragma unroll
  for (int q = 0; q < 2 * KMAX; ++q) acc[q] = 0.0;
  if (l < nl) {
    const int j = (int)(l % a.kk);
    long long rem = l / a.kk;
    const int ia = (int)(rem % a.na);
    rem /= a.na;
    const int ib = (int)(rem % a.nb);
    const int c = (int)(rem / a.nb);
    const long long pos = ib * a.sb + ia * a.sa;   // component-free offset of element 0
    const long long o0 = c * a.sc + pos + j;         // offset of element 0 (relative to t, x, r, p, q)
    const long long gp0 = pos / a.kk, ges = a.es / a.kk;
    const int len = a.len;
    const double* L = a.L;
    double* t = a.t;
    double al = 0.0;
    bool upd = false;
    if (PRO && a.update && !a.pcg->first) {
      al = a.pcg->alpha[j];
      upd = al != 0.0;
    }
    auto fetch_in = [&](int i) -> double {
      const long long o = o0 + (long long)i * a.es;
      if (PRO) {
        double rv = a.r[o];
        if (upd) {
          const double xv = a.x[o], pv = a.p[o], qv = a.q[o];
          a.x[o] = fma(al, pv, xv);
          rv = fma(-al, qv, rv);
          a.r[o] = rv;
        }
        return rv * a.s[gp0 + (long long)i * ges];
      }
      return t[o];
    };
    double y[P];
#pragma unroll
    for (int u = 0; u < P; ++u) y[u] = 0.0;
    double nxt[D];
#pragma unroll
    for (int d = 0; d < D; ++d) nxt[d] = d < len ? fetch_in(d) : 0.0;
    // forward: y_i = (t_i - sum_u L_{i,i-u} y_{i-u}) / L_ii
    for (int i0 = 0; i0 < len; i0 += D) {
      double cur[D];
#pragma unroll
      for (int d = 0; d < D; ++d) cur[d] = nxt[d];
#pragma unroll
      for (int d = 0; d < D; ++d) nxt[d] = (i0 + D + d < len) ? fetch_in(i0 + D + d) : 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int i = i0 + d;
        if (i < len) {
          double v = cur[d];
          const double* Li = L + (long long)i * (P + 1);
#pragma unroll
          for (int u = P; u >= 1; --u) v = fma(-__ldg(Li + u), y[u - 1], v);
          v *= __ldg(Li);
#pragma unroll
          for (int u = P - 1; u >= 1; --u) y[u] = y[u - 1];
          y[0] = v;
          t[o0 + (long long)i * a.es] = v;
        }
      }
    }
    // backward: z_i = (y_i - sum_u L_{i+u,i} z_{i+u}) / L_ii   (L padded with P zero rows)
#pragma unroll
    for (int u = 0; u < P; ++u) y[u] = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) nxt[d] = (len - 1 - d >= 0) ? t[o0 + (long long)(len - 1 - d) * a.es] : 0.0;
    for (int i0 = len - 1; i0 >= 0; i0 -= D) {
      double cur[D], sv[D], rv[D];
#pragma unroll
      for (int d = 0; d < D; ++d) cur[d] = nxt[d];
      if (EPI) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int i = i0 - d;
          const long long ii = i >= 0 ? i : 0;
          sv[d] = a.s[gp0 + ii * ges];
          rv[d] = a.r[o0 + ii * a.es];
        }
      }
#pragma unroll
      for (int d = 0; d < D; ++d) nxt[d] = (i0 - D - d >= 0) ? t[o0 + (long long)(i0 - D - d) * a.es] : 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int i = i0 - d;
        if (i >= 0) {
          double v = cur[d];
#pragma unroll
          for (int u = P; u >= 1; --u) v = fma(-__ldg(L + (long long)(i + u) * (P + 1) + u), y[u - 1], v);
          v *= __ldg(L + (long long)i * (P + 1));
#pragma unroll
          for (int u = P - 1; u >= 1; --u) y[u] = y[u - 1];
          y[0] = v;
          if (EPI) {
            const double z = v * sv[d];
#pragma unroll
            for (int q = 0; q < KMAX; ++q)
              {  // branch-free (keeps acc in registers)
                const double m = (q == j) ? rv[d] : 0.0;
                acc[q] = fma(m, z, acc[q]);
                acc[KMAX + q] = fma(m, rv[d], acc[KMAX + q]);
              }
            t[o0 + (long long)i * a.es] = z;
          } else {
            t[o0 + (long long)i * a.es] = v;
          }
        }
      }
    }
  }
  if (EPI) {
    double out[2 * KMAX];
    if (reduce_last_block<2 * KMAX>(acc, a.partial, a.counter, out))
      pcg_finalize(a.pcg, a.st, a.kk, a.maxit, a.cond, out, out + KMAX);
  }
}

template <int P>
static void line_sf_launch(const LineArgs& a, bool pro, bool epi, cudaStream_t s) {
  const long long nl = (long long)a.nvec * a.nb * a.na * a.kk;
  const unsigned int blocks = (unsigned int)((nl + NTHREADS - 1) / NTHREADS);
  if (pro) k_line_sf<P, true, false><<<blocks, NTHREADS, 0, s>>>(a);
  else if (epi) k_line_sf<P, false, true><<<blocks, NTHREADS, 0, s>>>(a);
  else k_line_sf<P, false, false><<<blocks, NTHREADS, 0, s>>>(a);
}
static void line_sf_dispatch(int p, const LineArgs& a, bool pro, bool epi, cudaStream_t s) {
  switch (p) {
    case 1: line_sf_launch<1>(a, pro, epi, s); break;
    case 2: line_sf_launch<2>(a, pro, epi, s); break;
    case 3: line_sf_launch<3>(a, pro, epi, s); break;
    case 4: line_sf_launch<4>(a, pro, epi, s); break;
    case 5: line_sf_launch<5>(a, pro, epi, s); break;
    case 6: line_sf_launch<6>(a, pro, epi, s); break;
    default: line_sf_launch<7>(a, pro, epi, s); break;
  }
}

template <int P>
__global__ void __launch_bounds__(512) k_line_tile(TileLine a) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  extern __shared__ double smem[];
  const int n = a.n, ST = a.ST, LD = ST + 1;
  double* Fs = smem + (size_t)n * LD + (size_t)a.C * P * ST;
  const int nthr = blockDim.x, tid = threadIdx.x;
  // factors -> shared memory
  for (int idx = tid; idx < 2 * a.flen; idx += nthr) Fs[idx] = idx < a.flen ? a.Ff[idx] : a.Fb[idx - a.flen];
  // PCG scalars of the fused update (read once)
  bool upd = false;
  double al[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) al[j] = 0.0;
  const double* pp = a.p0;
  if (a.pro && a.update && !a.pcg->first) {
    upd = true;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) al[j] = j < a.kk ? a.pcg->alpha[j] : 0.0;
    pp = (a.pcg->iter & 1) ? a.p1 : a.p0;
  }
  double acc[2 * KMAX];
#pragma unroll
  for (int j = 0; j < 2 * KMAX; ++j) acc[j] = 0.0;
  __syncthreads();
  tile_solve<P>(a, blockIdx.x, smem, Fs, upd, al, pp, acc);
  if (a.epi) {
    double out[2 * KMAX];
    if (reduce_last_block<2 * KMAX>(acc, a.partial, a.counter, out))
      pcg_finalize(a.pcg, a.st, a.kk, a.maxit, a.cond, out, out + KMAX);
  }
}

// Line tiles of several boxes (the patches of an additive Schwarz
// preconditioner) in one launch: block b -> (patch, tile) by the prefix
// table; every patch has its own factors and geometry, launch-wide ST.
struct TileMulti {
  TileLine tl[MAXPATCH];
  int tstart[MAXPATCH + 1];
  int np;
};

template <int P>
__global__ void __launch_bounds__(512) k_line_tile_multi(TileMulti mt) {
  int pr = 0;
  while (pr + 1 < mt.np && (int)blockIdx.x >= mt.tstart[pr + 1]) ++pr;
  const TileLine& a = mt.tl[pr];
  if (a.st->status != 0) return;
  if (blockIdx.x == 0) count_launch(a.st);
  extern __shared__ double smem[];
  const int n = a.n, ST = a.ST, LD = ST + 1;
  double* Fs = smem + (size_t)n * LD + (size_t)a.C * P * ST;
  for (int idx = threadIdx.x; idx < 2 * a.flen; idx += blockDim.x) Fs[idx] = idx < a.flen ? a.Ff[idx] : a.Fb[idx - a.flen];
  double al[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) al[j] = 0.0;
  double acc[2 * KMAX];
#pragma unroll
  for (int j = 0; j < 2 * KMAX; ++j) acc[j] = 0.0;
  __syncthreads();
  tile_solve<P>(a, (int)blockIdx.x - mt.tstart[pr], smem, Fs, false, al, a.p0, acc);
}

static size_t tile_smem(int n, int C, int p, int ST, int flen) {
  return sizeof(double) * ((size_t)n * (ST + 1) + (size_t)C * p * ST + 2 * (size_t)flen);
}

template <int P>
static bool tile_launch(TileLine a, cudaStream_t s) {
  if (a.C > 64) return false;
  const int nsl_total = a.mode == 0 ? -1 : a.nlines * a.kk;
  auto ntiles_for = [&](int st) -> long long {
    return a.mode == 0 ? (long long)a.nrows * ((a.rowlen + st - 1) / st) : ((long long)nsl_total + st - 1) / st;
  };
  int ST = 32;
  if (ntiles_for(32) < 296) ST = (ntiles_for(16) >= 148) ? 16 : 8;
  // at most 16 warps per block (launch bounds 512 -> 128 registers, no spills)
  while (ST > 8 && (a.C + 32 / ST - 1) / (32 / ST) > 16) ST >>= 1;
  a.ST = ST;
  const size_t sm = tile_smem(a.n, a.C, P, ST, a.flen);
  static size_t attr_max = 0, static_sm = (size_t)-1;
  if (static_sm == (size_t)-1) {
    cudaFuncAttributes fa;
    static_sm = cudaFuncGetAttributes(&fa, k_line_tile<P>) == cudaSuccess ? fa.sharedSizeBytes : 16384;
  }
  if (sm + static_sm > 227 * 1024) return false;
  if (sm > attr_max) {
    if (cudaFuncSetAttribute(k_line_tile<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
      return false;
    attr_max = sm;
  }
  const int cpw = 32 / ST;
  const int nwarps = (a.C + cpw - 1) / cpw;
  k_line_tile<P><<<(unsigned int)ntiles_for(ST), 32 * nwarps, sm, s>>>(a);
  return true;
}
static bool tile_dispatch(int p, const TileLine& a, cudaStream_t s) {
  switch (p) {
    case 1: return tile_launch<1>(a, s);
    case 2: return tile_launch<2>(a, s);
    case 3: return tile_launch<3>(a, s);
    case 4: return tile_launch<4>(a, s);
    case 5: return tile_launch<5>(a, s);
    case 6: return tile_launch<6>(a, s);
    default: return tile_launch<7>(a, s);
  }
}

template <int P>
static bool tile_multi_launch(TileMulti m, cudaStream_t s) {
  // common slots per tile: the smallest any patch would use, <= 16 warps per block
  int ST = 32, C = 1, nmax = 1, flen = 1;
  long long tot32 = 0;
  for (int r = 0; r < m.np; ++r) {
    C = std::max(C, m.tl[r].C);
    nmax = std::max(nmax, m.tl[r].n);
    flen = std::max(flen, m.tl[r].flen);
    if (m.tl[r].C > 64) return false;
  }
  auto ntiles_for = [&](const TileLine& t, int st) -> long long {
    return t.mode == 0 ? (long long)t.nrows * ((t.rowlen + st - 1) / st) : ((long long)t.nlines * t.kk + st - 1) / st;
  };
  for (int r = 0; r < m.np; ++r) tot32 += ntiles_for(m.tl[r], 32);
  if (tot32 < 296) {
    long long tot16 = 0;
    for (int r = 0; r < m.np; ++r) tot16 += ntiles_for(m.tl[r], 16);
    ST = tot16 >= 148 ? 16 : 8;
  }
  static int min_st = -1;  // GA_TILE_MINST: smallest slots per tile (8: up to 16 warps per CTA)
  if (min_st < 0) {  // clamped to 1..8: larger minimums would exceed 16 warps (512 threads) per CTA
    const char* e = getenv("GA_TILE_MINST");
    min_st = std::min(8, std::max(1, e ? atoi(e) : 8));
  }
  while (ST > min_st && (C + 32 / ST - 1) / (32 / ST) > 16) ST >>= 1;
  if (min_st < 8) while (ST > min_st && (C + 32 / ST - 1) / (32 / ST) > 8) ST >>= 1;
  int t0 = 0;
  for (int r = 0; r < m.np; ++r) {
    m.tl[r].ST = ST;
    m.tstart[r] = t0;
    t0 += (int)ntiles_for(m.tl[r], ST);
  }
  m.tstart[m.np] = t0;
  const size_t sm = tile_smem(nmax, C, P, ST, flen);
  static size_t attr_max = 0;
  if (sm + 4096 > 227 * 1024) return false;
  if (sm > attr_max) {
    if (cudaFuncSetAttribute(k_line_tile_multi<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
      return false;
    attr_max = sm;
  }
  const int cpw = 32 / ST;
  const int nwarps = (C + cpw - 1) / cpw;
  k_line_tile_multi<P><<<(unsigned int)t0, 32 * nwarps, sm, s>>>(m);
  return true;
}
static bool tile_multi_dispatch(int p, const TileMulti& m, cudaStream_t s) {
  switch (p) {
    case 1: return tile_multi_launch<1>(m, s);
    case 2: return tile_multi_launch<2>(m, s);
    case 3: return tile_multi_launch<3>(m, s);
    case 4: return tile_multi_launch<4>(m, s);
    case 5: return tile_multi_launch<5>(m, s);
    case 6: return tile_multi_launch<6>(m, s);
    default: return tile_multi_launch<7>(m, s);
  }
}

// z = sum_r s_r o t_r (single patch: z *= s in place), then r.z and r.r.
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_prec_out(PrecArgs a) {
  const bool dead = a.st->status != 0;
  if (!dead) count_launch(a.st);
  const GridDesc g = a.g;
  const long long tot = (long long)a.nvec * g.npts;
  const long long estride = (long long)gridDim.x * blockDim.x;
  double v[2 * KK];
#pragma unroll
  for (int j = 0; j < 2 * KK; ++j) v[j] = 0.0;
  const int npts = (int)g.npts;  // < 2^31 grid points (checked by the launcher)
  if (!dead) for (long long e = (long long)gtid(); e < tot; e += estride) {
    const int c = (int)(e / npts);
    const int i = (int)e - c * npts;
    const long long base = ((long long)c * g.padded + g.guard + i) * KK;
    double z[KK];
    if (a.npatch == 1 && a.t[0] == nullptr) {
      const double sv = a.s[0][i];
      ld_k<KK>(a.z + base, z);
#pragma unroll
      for (int j = 0; j < KK; ++j) z[j] *= sv;
    } else {
#pragma unroll
      for (int j = 0; j < KK; ++j) z[j] = 0.0;
      const int iyz = i / g.nx, ix = i - iyz * g.nx;
      const int iz = iyz / g.ny, iy = iyz - iz * g.ny;
      if (a.mask != nullptr && !a.mask[i]) continue;  // not free: z and r stay zero there
      for (int pr = 0; pr < a.npatch; ++pr) {
        const int lx = ix - a.lo[pr][0], ly = iy - a.lo[pr][1], lz = iz - a.lo[pr][2];
        if (lx < 0 || ly < 0 || lz < 0 || lx >= a.bd[pr][0] || ly >= a.bd[pr][1] || lz >= a.bd[pr][2]) continue;
        const long long nbox = (long long)a.bd[pr][0] * a.bd[pr][1] * a.bd[pr][2];
        const int bi = lx + a.bd[pr][0] * (ly + a.bd[pr][1] * lz);
        const double sv = a.s[pr][bi];
        double tv[KK];
        ld_k<KK>(a.t[pr] + ((long long)c * nbox + bi) * KK, tv);
#pragma unroll
        for (int j = 0; j < KK; ++j) z[j] = fma(sv, tv[j], z[j]);
      }
    }
    // subdomain (a.xsum): r.z over every local DoF (z_r unassembled: r.z = sum_r r_r . z_r),
    // r.r over the owned DoFs only (each global DoF once)
    const double wr = (a.xsum && a.mask && a.mask[i] != 1) ? 0.0 : 1.0;
    double rv[KK];
    ld_k<KK>(a.r + base, rv);
    st_k<KK>(a.z + base, z);
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      v[j] = fma(rv[j], z[j], v[j]);
      v[KK + j] = fma(wr * rv[j], rv[j], v[KK + j]);
    }
  }
  if (dead) return;
  double out[2 * KK];
  if (reduce_last_block<2 * KK>(v, a.partial, a.counter, out)) {
    if (a.xsum) {
      for (int j = 0; j < 2 * KK; ++j) a.xsum[j] = out[j];
      return;
    }
    double rz[KMAX], rr[KMAX];
    for (int j = 0; j < KK; ++j) { rz[j] = out[j]; rr[j] = out[KK + j]; }
    pcg_finalize(a.pcg, a.st, KK, a.maxit, a.cond, rz, rr);
  }
}

void launch_precond(const PrecArgs& a, cudaStream_t s) {
  const GridDesc& g = a.g;
  const bool single = (a.npatch == 1 && a.t[0] == nullptr);
  // line mode: tiles (chunked, shared memory; few lines, small grids), whole-line sweeps from
  // shared memory (many lines; line_seq.cu) or streaming thread-per-line sweeps (fallback for
  // lines too long for shared memory).  GA_LINE_MODE overrides.
  static int line_mode = -1;  // 0 auto, 1 tile, 2 stream, 4 whole-line
  if (line_mode < 0) {
    const char* e = getenv("GA_LINE_MODE");
    line_mode = (e && e[0] == 't') ? 1 : ((e && e[0] == 's') ? 2 : ((e && e[0] == 'q') ? 4 : 0));
  }
  long long minslots = 1LL << 62;
  for (int pr = 0; pr < a.npatch; ++pr)
    for (int d = 0; d < g.dim; ++d) {
      long long sl = (long long)a.nvec * a.kk;
      for (int e2 = 0; e2 < g.dim; ++e2)
        if (e2 != d) sl *= a.bd[pr][e2];
      minslots = std::min(minslots, sl);
    }
  const bool stream = line_mode >= 2 || (line_mode == 0 && minslots >= 148LL * 128);
  // single patch: whole-line sweeps from shared memory (line_seq.cu): prologue pass, one launch per
  // direction (forward + backward on-chip, every direction coalesced), epilogue pass with the dot
  // products.  Auto: every 3D grid (measured against the fused chunked tiles, step times: n_f = 27
  // 4.39 vs 4.74 ms, 34: 2.11 vs 2.04, 49: 1.49 vs 1.93, 66: 5.07 vs 6.09, 81: 3.77 vs 4.45 ms) and
  // 2D grids with lines longer than 768 points (2D p=3 n=512: 1.28 vs 1.19 ms for the tiles;
  // n=1024: 2.8 vs 16.7 ms, n=2048: 18.5 vs 38.5 ms - the tiles' 64-chunk limit)
  bool want_seq = line_mode == 4;
  if (line_mode == 0 && single) {
    const int lmax = std::max(a.bd[0][0], std::max(a.bd[0][1], a.bd[0][2]));
    want_seq = g.dim == 3 || lmax > 768 || stream;
  }
  if (single && want_seq && a.nvec * g.npts * a.kk < (1LL << 31)) {
    bool ok = true;
    for (int d = 0; d < g.dim && ok; ++d) ok = launch_line_seq_multi(a, d, s, true);
    if (ok) {
      launch_xr_prec_in(a, s);
      for (int d = 0; d < g.dim; ++d) launch_line_seq_multi(a, d, s);
      const unsigned int nb = red_grid((long long)a.nvec * g.npts);
      switch (a.kk) {
        case 1: k_prec_out<1><<<nb, NTHREADS, 0, s>>>(a); break;
        case 2: k_prec_out<2><<<nb, NTHREADS, 0, s>>>(a); break;
        case 3: k_prec_out<3><<<nb, NTHREADS, 0, s>>>(a); break;
        default: k_prec_out<4><<<nb, NTHREADS, 0, s>>>(a); break;
      }
      return;
    }
  }
  if (single && stream) {
    // streaming fused path (3D): first direction y (PRO, coalesced), then x, then z (EPI)
    const int bd[3] = {a.bd[0][0], a.bd[0][1], a.bd[0][2]};
    const long long str[3] = {a.kk, (long long)g.nx * a.kk, (long long)g.nx * g.ny * a.kk};
    const long long off = g.guard * a.kk;
    int order[3] = {1, 0, 2};
    if (g.dim == 2) { order[0] = 1; order[1] = 0; }
    for (int k = 0; k < g.dim; ++k) {
      const int d = order[k];
      LineArgs la;
      memset(&la, 0, sizeof(la));
      la.t = a.z + off; la.L = a.L[0][d]; la.len = bd[d]; la.es = str[d]; la.kk = a.kk; la.nvec = a.nvec;
      la.sc = g.padded * a.kk;
      const int o1 = (d == 0) ? 1 : 0, o2 = (d == 2) ? 1 : 2;
      la.na = bd[o1]; la.sa = str[o1];
      la.nb = (g.dim == 3) ? bd[o2] : 1; la.sb = (g.dim == 3) ? str[o2] : 0;
      la.s = a.s[0];
      la.x = a.x + off; la.r = a.r + off; la.p = a.p0 + off; la.q = a.q + off;
      la.pcg = a.pcg; la.st = a.st; la.partial = a.partial; la.counter = a.counter;
      la.maxit = a.maxit; la.update = a.update; la.cond = a.cond;
      line_sf_dispatch(a.p, la, k == 0, k == g.dim - 1, s);
    }
    return;
  }
  // fused path: single patch, tile solver available for every direction
  bool fused = single && !stream;
  for (int d = 0; d < g.dim && fused; ++d) fused = a.Ff[0][d] != nullptr && a.nchunk[0][d] <= 64;
  if (fused) {
    const int bd[3] = {a.bd[0][0], a.bd[0][1], a.bd[0][2]};
    const long long str[3] = {a.kk, (long long)g.nx * a.kk, (long long)g.nx * g.ny * a.kk};
    const long long sc = g.padded * a.kk;
    bool ok = true;
    for (int d = 0; d < g.dim && ok; ++d) {
      TileLine tl;
      memset(&tl, 0, sizeof(tl));
      tl.t = a.z + g.guard * a.kk; tl.n = bd[d]; tl.kk = a.kk; tl.st = a.st;
      tl.Ff = a.Ff[0][d]; tl.Fb = a.Fb[0][d]; tl.flen = a.flen[0][d];
      tl.clen = a.clen[0][d]; tl.C = a.nchunk[0][d]; tl.L = a.nlev[0][d];
      if (d == 0) {
        tl.mode = 1; tl.nlines = a.nvec * bd[1] * bd[2]; tl.nl2 = bd[1] * bd[2]; tl.sA = sc; tl.sB = str[1];
      } else {
        tl.mode = 0; tl.es = str[d]; tl.rowlen = bd[0] * a.kk;
        const int other = (d == 1) ? 2 : 1;
        const int nother = (g.dim == 3) ? bd[other] : 1;
        tl.nrows = a.nvec * nother; tl.nr2 = nother; tl.sA = sc; tl.sB = (g.dim == 3) ? str[other] : 0;
      }
      // fusion: offsets into z (= t) are offsets into x, r, p, q (same MV layout)
      const long long off = g.guard * a.kk;
      tl.padkk = g.padded * a.kk;
      tl.s = a.s[0];  // s index = (offset mod padkk)/kk = grid point
      tl.x = a.x + off; tl.r = a.r + off; tl.p0 = a.p0 + off; tl.p1 = a.p1 + off; tl.q = a.q + off;
      tl.pcg = a.pcg; tl.partial = a.partial; tl.counter = a.counter;
      tl.tol2 = a.tol2; tl.maxit = a.maxit; tl.cond = a.cond; tl.update = a.update;
      tl.pro = (d == 0);
      tl.epi = (d == g.dim - 1);
      ok = tile_dispatch(a.p, tl, s);
    }
    if (ok) return;
  }
  // general path (multi-patch / very long lines)
  // boxes of a multi-patch problem: every patch in one launch per direction (chunked tiles for few
  // lines; the whole-line solver also for many lines, 3D boxes)
  bool seq_multi = !single && stream && (line_mode == 0 || line_mode == 4);
  for (int d = 0; d < g.dim && seq_multi; ++d) seq_multi = launch_line_seq_multi(a, d, s, true);
  const bool batched = !single && (!stream || seq_multi);
  if (batched && a.nvec * g.npts * a.kk < (1LL << 31)) {
    // batched Schwarz: prologue + gather in one pass, then one tile launch per direction
    const unsigned int nbg = (unsigned int)((a.nvec * g.npts + NTHREADS - 1) / NTHREADS);
    switch (a.kk) {
      case 1: k_xr_gather<1><<<nbg, NTHREADS, 0, s>>>(a); break;
      case 2: k_xr_gather<2><<<nbg, NTHREADS, 0, s>>>(a); break;
      case 3: k_xr_gather<3><<<nbg, NTHREADS, 0, s>>>(a); break;
      default: k_xr_gather<4><<<nbg, NTHREADS, 0, s>>>(a); break;
    }
  } else {
    launch_xr_prec_in(a, s);
    if (batched) {
      long long tb = 0;
      for (int pr = 0; pr < a.npatch; ++pr) tb += (long long)a.nvec * a.bd[pr][0] * a.bd[pr][1] * a.bd[pr][2] * a.kk;
      k_prec_gather_all<<<(unsigned int)((tb + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(a);
    }
  }
  if (batched) {
    bool ok = true;
    for (int d = 0; d < g.dim && ok; ++d) {
      TileMulti m;
      memset(&m, 0, sizeof(m));
      m.np = a.npatch;
      for (int pr = 0; pr < a.npatch; ++pr) {
        const int bd[3] = {a.bd[pr][0], a.bd[pr][1], a.bd[pr][2]};
        const long long nbox = (long long)bd[0] * bd[1] * bd[2];
        const long long str[3] = {a.kk, (long long)bd[0] * a.kk, (long long)bd[0] * bd[1] * a.kk};
        const long long sc = nbox * a.kk;
        TileLine& tl = m.tl[pr];
        tl.t = a.t[pr]; tl.n = bd[d]; tl.kk = a.kk; tl.st = a.st;
        tl.Ff = a.Ff[pr][d]; tl.Fb = a.Fb[pr][d]; tl.flen = a.flen[pr][d];
        tl.clen = a.clen[pr][d]; tl.C = a.nchunk[pr][d]; tl.L = a.nlev[pr][d];
        if (!tl.Ff) ok = false;
        if (d == 0) {
          tl.mode = 1; tl.nlines = a.nvec * bd[1] * bd[2]; tl.nl2 = bd[1] * bd[2]; tl.sA = sc; tl.sB = str[1];
        } else {
          tl.mode = 0; tl.es = str[d]; tl.rowlen = bd[0] * a.kk;
          const int other = (d == 1) ? 2 : 1;
          const int nother = (g.dim == 3) ? bd[other] : 1;
          tl.nrows = a.nvec * nother; tl.nr2 = nother; tl.sA = sc; tl.sB = (g.dim == 3) ? str[other] : 0;
        }
      }
      if (ok && launch_line_seq_multi(a, d, s)) continue;
      if (ok) ok = tile_multi_dispatch(a.p, m, s);
    }
    if (ok) {
      const long long tot2 = (long long)a.nvec * g.npts;
      const unsigned int nb = red_grid(tot2);
      switch (a.kk) {
        case 1: k_prec_out<1><<<nb, NTHREADS, 0, s>>>(a); break;
        case 2: k_prec_out<2><<<nb, NTHREADS, 0, s>>>(a); break;
        case 3: k_prec_out<3><<<nb, NTHREADS, 0, s>>>(a); break;
        default: k_prec_out<4><<<nb, NTHREADS, 0, s>>>(a); break;
      }
      return;
    }
    // (fall through: per-patch path; the gather above is repeated harmlessly)
  }
  for (int pr = 0; pr < a.npatch; ++pr) {
    double* t;
    long long str[3];
    long long sc;
    int bd[3] = {a.bd[pr][0], a.bd[pr][1], a.bd[pr][2]};
    if (single) {
      t = a.z + g.guard * a.kk;
      str[0] = a.kk; str[1] = (long long)g.nx * a.kk; str[2] = (long long)g.nx * g.ny * a.kk;
      sc = g.padded * a.kk;
    } else {
      const long long nbox = (long long)bd[0] * bd[1] * bd[2];
      k_prec_gather<<<(unsigned int)((a.nvec * nbox * a.kk + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(a, pr);
      t = a.t[pr];
      str[0] = a.kk; str[1] = (long long)bd[0] * a.kk; str[2] = (long long)bd[0] * bd[1] * a.kk;
      sc = nbox * a.kk;
    }
    for (int d = 0; d < g.dim; ++d) {
      bool done = false;
      if (a.Ff[pr][d] && !stream) {
        TileLine tl;
        memset(&tl, 0, sizeof(tl));
        tl.t = t; tl.n = bd[d]; tl.kk = a.kk; tl.st = a.st;
        tl.Ff = a.Ff[pr][d]; tl.Fb = a.Fb[pr][d]; tl.flen = a.flen[pr][d];
        tl.clen = a.clen[pr][d]; tl.C = a.nchunk[pr][d]; tl.L = a.nlev[pr][d];
        if (d == 0) {
          tl.mode = 1; tl.nlines = a.nvec * bd[1] * bd[2]; tl.nl2 = bd[1] * bd[2]; tl.sA = sc; tl.sB = str[1];
        } else {
          tl.mode = 0; tl.es = str[d]; tl.rowlen = bd[0] * a.kk;
          const int other = (d == 1) ? 2 : 1;
          const int nother = (g.dim == 3) ? bd[other] : 1;
          tl.nrows = a.nvec * nother; tl.nr2 = nother; tl.sA = sc; tl.sB = (g.dim == 3) ? str[other] : 0;
        }
        done = tile_dispatch(a.p, tl, s);
      }
      if (!done) {
        int o1 = (d == 0) ? 1 : 0;
        int o2 = (d == 2) ? 1 : 2;
        int na = bd[o1], nb = (g.dim == 3) ? bd[o2] : 1;
        long long sa = str[o1], sb = (g.dim == 3) ? str[o2] : 0;
        line_dispatch(a.p, t, a.L[pr][d], bd[d], str[d], na, sa, nb, sb, a.kk, a.nvec, sc, a.st, s);
      }
    }
  }
  const long long tot = (long long)a.nvec * g.npts;
  const unsigned int nb = red_grid(tot);
  switch (a.kk) {
    case 1: k_prec_out<1><<<nb, NTHREADS, 0, s>>>(a); break;
    case 2: k_prec_out<2><<<nb, NTHREADS, 0, s>>>(a); break;
    case 3: k_prec_out<3><<<nb, NTHREADS, 0, s>>>(a); break;
    default: k_prec_out<4><<<nb, NTHREADS, 0, s>>>(a); break;
  }
}

// ---------------------------------------------------------------------------
// PCG vector kernels
// ---------------------------------------------------------------------------
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_init_from_b(VecArgs a) {
  const bool dead = a.st->status != 0;
  if (!dead) count_launch(a.st);
  const GridDesc g = a.g;
  const long long tot = (long long)a.nvec * g.npts;
  const long long estride = (long long)gridDim.x * blockDim.x;
  double v[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) v[j] = 0.0;
  const int npts = (int)g.npts;  // < 2^31 grid points (checked by the launcher)
  if (!dead) for (long long e = (long long)gtid(); e < tot; e += estride) {
    const int c = (int)(e / npts);
    const int i = (int)e - c * npts;
    const long long base = ((long long)c * g.padded + g.guard + i) * KK;
    const double wb = (a.own && a.own[i] != 1) ? 0.0 : 1.0;  // subdomain: owned DoFs only
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      const double b = a.b[base + j];
      a.r[base + j] = b;
      a.x[base + j] = 0.0;
      v[j] = fma(wb * b, b, v[j]);
    }
  }
  if (dead) return;
  double out[KK];
  if (reduce_last_block<KK>(v, a.partial, a.counter, out)) {
    if (a.xsum) {
      for (int j = 0; j < KK; ++j) a.xsum[j] = out[j];
      return;
    }
    PcgState* pc = a.pcg;
    pc->iter = 0; pc->first = 1; pc->pfirst = 1; pc->nrhs = KK; pc->phase = 0; pc->guard = 0;
    for (int j = 0; j < KK; ++j) {
      pc->bb[j] = out[j];
      pc->thr[j] = a.tol2 * out[j];
      pc->active[j] = out[j] > 0.0 ? 1 : 0;
      pc->its[j] = 0;
      pc->alpha[j] = 0.0;
      pc->beta[j] = 0.0;
    }
  }
}
void launch_init_from_b(const VecArgs& a, cudaStream_t s) {
  const long long tot = (long long)a.nvec * a.g.npts;
  const unsigned int nb = red_grid(tot);
  switch (a.kk) {
    case 1: k_init_from_b<1><<<nb, NTHREADS, 0, s>>>(a); break;
    case 2: k_init_from_b<2><<<nb, NTHREADS, 0, s>>>(a); break;
    case 3: k_init_from_b<3><<<nb, NTHREADS, 0, s>>>(a); break;
    default: k_init_from_b<4><<<nb, NTHREADS, 0, s>>>(a); break;
  }
}

// p = z (first iteration of a phase) or p = z + beta p, for active blocks.
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_p_update(VecArgs a) {
  if (a.st->status != 0) return;
  count_launch(a.st);
  const GridDesc g = a.g;
  const long long tot = (long long)a.nvec * g.npts;  // one thread per (component, grid point)
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const long long i = e % g.npts;
  const int c = (int)(e / g.npts);
  if (a.mask && !a.mask[i]) return;  // not a free point: every vector is zero there
  const long long base = ((long long)c * g.padded + g.guard + i) * KK;
  bool any = false;
#pragma unroll
  for (int j = 0; j < KK; ++j) any |= a.pcg->active[j] != 0;
  if (!any) return;
  double z[KK], p[KK];
  ld_k<KK>(a.z + base, z);
  ld_k<KK>(a.p + base, p);
  const bool pfirst = a.pcg->pfirst != 0;
#pragma unroll
  for (int j = 0; j < KK; ++j)
    if (a.pcg->active[j]) p[j] = pfirst ? z[j] : fma(a.pcg->beta[j], p[j], z[j]);  // inactive: unchanged
  st_k<KK>(a.p + base, p);
}
void launch_p_update(const VecArgs& a, cudaStream_t s) {
  const long long tot = (long long)a.nvec * a.g.npts;
  const unsigned int nb = (unsigned int)((tot + NTHREADS - 1) / NTHREADS);
  switch (a.kk) {
    case 1: k_p_update<1><<<nb, NTHREADS, 0, s>>>(a); break;
    case 2: k_p_update<2><<<nb, NTHREADS, 0, s>>>(a); break;
    case 3: k_p_update<3><<<nb, NTHREADS, 0, s>>>(a); break;
    default: k_p_update<4><<<nb, NTHREADS, 0, s>>>(a); break;
  }
}

__global__ void k_solve_end(PcgState* pc, DevStatus* st) {
  count_launch(st);
  if (threadIdx.x != 0) return;
  long long ns = 0;
  for (int j = 0; j < pc->nrhs; ++j) {
    if (pc->bb[j] > 0.0) {
      ++ns;
      st->pcg_iters[j] += pc->its[j];
      st->last_iters[j] = pc->its[j];
      if (pc->its[j] > st->max_iters) st->max_iters = pc->its[j];
      double rel = sqrt(pc->rr[j] / pc->bb[j]);
      if (rel > st->max_relres) st->max_relres = rel;
    } else {
      st->last_iters[j] = 0;
    }
  }
  st->solves += ns;
}
void launch_solve_end(PcgState* pcg, DevStatus* st, cudaStream_t s) { k_solve_end<<<1, 32, 0, s>>>(pcg, st); }

// ---------------------------------------------------------------------------
// Stage update (reading R1): one thread per (component, DoF)
// ---------------------------------------------------------------------------
// T_m(c) = sum_{i=0}^{3k-1-m} tau^i / i! c_{m+i}, compile-time k: all registers
template <int K>
__device__ __forceinline__ double taylor_k(const double (&c)[3 * K], int m, const double* f) {
  double s = 0.0;
#pragma unroll
  for (int i = 3 * K - 1; i >= 0; --i)
    if (i <= 3 * K - 1 - m) s = fma(f[i], c[m + i], s);
  return s;
}

template <bool STEP, int K>
__global__ void __launch_bounds__(NTHREADS) k_stage(StageArgs a) {
  constexpr int N3 = 3 * K;
  const bool dead = a.st->status != 0;
  if (!dead) count_launch(a.st);
  const GridDesc g = a.g;
  const long long npts = g.npts;
  const long long vstride = (long long)a.nvec * g.padded;
  const long long estride = (long long)gridDim.x * blockDim.x;
  double f[N3];
#pragma unroll
  for (int i = 0; i < N3; ++i) f[i] = a.f[i];
  double u2[1] = {0.0};
  if (!dead)
    for (int c = 0; c < a.nvec; ++c) {
      const long long cb = (long long)c * g.padded + g.guard;
      for (long long i = (long long)gtid(); i < npts; i += estride) {
        const long long off = cb + i;
        double cc[N3], nw[N3];
#pragma unroll
        for (int m = 0; m < N3; ++m) cc[m] = a.chain[m * vstride + off];
        if (STEP) {
          double y[K];
#pragma unroll
          for (int j = 0; j < K; ++j) y[j] = a.ysol[off * K + j];
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const int d = 3 * j, v = 3 * j + 1, ac = 3 * j + 2;
            const double Td = taylor_k<K>(cc, d, f), Tv = taylor_k<K>(cc, v, f), Ta = taylor_k<K>(cc, ac, f);
            // Rayleigh damping (reading R16): y_j - a0 w_j, w_j = T_vel (j < k), c_vel (j = k)
            const double wj = (j < K - 1) ? Tv : cc[v];
            const double P = (fma(-a.damp_a0, wj, y[j]) - Ta) / a.alpha[j];
            nw[d] = fma(a.beta[j] * a.tau * a.tau, P, Td);
            nw[v] = fma(a.gamma[j] * a.tau, P, Tv);
            nw[ac] = Ta + P;
          }
#pragma unroll
          for (int m = 0; m < N3; ++m) a.chain[m * vstride + off] = nw[m];
        } else {
#pragma unroll
          for (int m = 0; m < N3; ++m) nw[m] = cc[m];
        }
        // predictors of the next step: s_j = T_disp(c) (j < k), s_k = c_{3k-3}
#pragma unroll
        for (int j = 0; j < K; ++j) {
          // K acts on s_j + a1 w_j (Rayleigh damping folded into the -K s SpMV; a1 = 0: s_j exactly)
          const double sj = (j < K - 1) ? taylor_k<K>(nw, 3 * j, f) : nw[3 * j];
          const double wj = (j < K - 1) ? taylor_k<K>(nw, 3 * j + 1, f) : nw[3 * j + 1];
          a.pred[off * K + j] = fma(a.damp_a1, wj, sj);
        }
        u2[0] = fma(nw[0], nw[0], u2[0]);
      }
    }
  if (dead || !STEP) return;
  double out[1];
  if (reduce_last_block<1>(u2, a.partial, a.counter, out)) {
    DevStatus* st = a.st;
    st->steps += 1;
    st->tstep += 1;
    // reference of the instability detector: set at ga_set_state from U0 and dt V0; a run that
    // starts from rest (U0 = V0 = 0: forcing or lifting) adopts its first non-zero ||U_n||^2
    if (st->u0norm2 == 0.0) st->u0norm2 = out[0];
    else if (a.unstable2 > 0.0 && !(out[0] <= a.unstable2 * st->u0norm2)) {
      st->status = -6;  // GA_ERR_UNSTABLE
      st->fail_step = st->steps;
      st->fail_block = -1;
    }
  }
}

template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_add_forcing(ForceArgs a) {
  if (a.st->status != 0) return;
  count_launch(const_cast<DevStatus*>(a.st));
  const GridDesc g = a.g;
  // h_r^{(m)}(t) per pair and slot, identical in every thread (a few terms, computed redundantly)
  double hj[FMAXPAIRS][KK];
  const double tn = a.t0 + (double)a.st->tstep * a.dt;
#pragma unroll
  for (int r = 0; r < FMAXPAIRS; ++r)
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      double h = 0.0;
      if (r < a.npairs && a.slots->active[j]) {
        const int m = a.slots->order[j];
        const double t = tn + a.slots->toff[j];
        for (int i = 0; i < a.nterms[r]; ++i)
          h += a.amp[r][i] * pow(a.omega[r][i], (double)m) * cos(a.omega[r][i] * t + a.phase[r][i] + m * 1.5707963267948966);
      }
      hj[r][j] = h;
    }
  const long long tot = (long long)a.nvec * g.npts;
  for (long long e = (long long)gtid(); e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / g.npts, i = e - c * g.npts;
    const long long gi = c * g.padded + g.guard + i;
    double add[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) add[j] = 0.0;
#pragma unroll
    for (int r = 0; r < FMAXPAIRS; ++r) {
      if (r >= a.npairs || !a.G[r]) continue;
      const double G = a.G[r][gi];
#pragma unroll
      for (int j = 0; j < KK; ++j) add[j] = fma(hj[r][j], G, add[j]);
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) a.b[gi * KK + j] += add[j];
  }
}

void launch_add_forcing(const ForceArgs& a, cudaStream_t s) {
  const unsigned int nb = red_grid((long long)a.nvec * a.g.npts);
  switch (a.kk) {
    case 1: k_add_forcing<1><<<nb, NTHREADS, 0, s>>>(a); break;
    case 2: k_add_forcing<2><<<nb, NTHREADS, 0, s>>>(a); break;
    case 3: k_add_forcing<3><<<nb, NTHREADS, 0, s>>>(a); break;
    default: k_add_forcing<4><<<nb, NTHREADS, 0, s>>>(a); break;
  }
}

template <bool STEP>
static void stage_go(const StageArgs& a, cudaStream_t s) {
  const unsigned int nb = red_grid(a.g.npts);
  switch (a.k) {
    case 1: k_stage<STEP, 1><<<nb, NTHREADS, 0, s>>>(a); break;
    case 2: k_stage<STEP, 2><<<nb, NTHREADS, 0, s>>>(a); break;
    case 3: k_stage<STEP, 3><<<nb, NTHREADS, 0, s>>>(a); break;
    default: k_stage<STEP, 4><<<nb, NTHREADS, 0, s>>>(a); break;
  }
}
void launch_stage(const StageArgs& a, cudaStream_t s) { stage_go<true>(a, s); }
void launch_predict(const StageArgs& a, cudaStream_t s) { stage_go<false>(a, s); }

// ---------------------------------------------------------------------------
// Packing / copies / small reductions
// ---------------------------------------------------------------------------
struct Idx4 { int v[KMAX]; };

// mv slot j = chain[src_j] + a1 chain[src2_j]  (src2 < 0: no damping term)
__global__ void k_pack(GridDesc g, int nvec, int kk, const double* chain, Idx4 src, Idx4 src2, double a1, double* mv,
                       DevStatus* st) {
  count_launch(st);
  const long long tot = (long long)nvec * g.npts * kk;
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const int j = (int)(e % kk);
  const long long ci = e / kk;
  const long long i = ci % g.npts;
  const int c = (int)(ci / g.npts);
  const long long vstride = (long long)nvec * g.padded;
  double v = src.v[j] >= 0 ? chain[src.v[j] * vstride + (long long)c * g.padded + g.guard + i] : 0.0;
  if (src2.v[j] >= 0) v = fma(a1, chain[src2.v[j] * vstride + (long long)c * g.padded + g.guard + i], v);
  mv[((long long)c * g.padded + g.guard + i) * kk + j] = v;
}
// chain[dst_j] = mv slot j - a0 chain[src2_j]  (src2 < 0: no damping term)
__global__ void k_unpack(GridDesc g, int nvec, int kk, const double* mv, Idx4 dst, Idx4 src2, double a0, double* chain,
                         DevStatus* st) {
  count_launch(st);
  const long long tot = (long long)nvec * g.npts * kk;
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const int j = (int)(e % kk);
  if (dst.v[j] < 0) return;
  const long long ci = e / kk;
  const long long i = ci % g.npts;
  const int c = (int)(ci / g.npts);
  const long long vstride = (long long)nvec * g.padded;
  double v = mv[((long long)c * g.padded + g.guard + i) * kk + j];
  if (src2.v[j] >= 0) v = fma(-a0, chain[src2.v[j] * vstride + (long long)c * g.padded + g.guard + i], v);
  chain[dst.v[j] * vstride + (long long)c * g.padded + g.guard + i] = v;
}
void launch_pack(const GridDesc& g, int nvec, int kk, const double* chain, const int* src, double* mv,
                 DevStatus* st, cudaStream_t s, const int* src2, double a1) {
  Idx4 ix, ix2;
  for (int j = 0; j < KMAX; ++j) { ix.v[j] = j < kk ? src[j] : -1; ix2.v[j] = (src2 && j < kk) ? src2[j] : -1; }
  const long long tot = (long long)nvec * g.npts * kk;
  k_pack<<<(unsigned int)((tot + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(g, nvec, kk, chain, ix, ix2, a1, mv, st);
}
void launch_unpack(const GridDesc& g, int nvec, int kk, const double* mv, const int* dst, double* chain,
                   DevStatus* st, cudaStream_t s, const int* src2, double a0) {
  Idx4 ix, ix2;
  for (int j = 0; j < KMAX; ++j) { ix.v[j] = j < kk ? dst[j] : -1; ix2.v[j] = (src2 && j < kk) ? src2[j] : -1; }
  const long long tot = (long long)nvec * g.npts * kk;
  k_unpack<<<(unsigned int)((tot + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(g, nvec, kk, mv, ix, ix2, a0, chain, st);
}

// api[c*nfree + f] <-> grid[((c*padded + guard + map[f]) * kk + slot)]
__global__ void k_api_to_grid(GridDesc g, int nvec, long long nfree, const long long* map, const double* api,
                              double* gv, int kk, int slot, DevStatus* st) {
  count_launch(st);
  const long long tot = (long long)nvec * nfree;
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const long long f = e % nfree;
  const int c = (int)(e / nfree);
  const long long gi = map ? map[f] : f;
  gv[((long long)c * g.padded + g.guard + gi) * kk + slot] = api[e];
}
__global__ void k_grid_to_api(GridDesc g, int nvec, long long nfree, const long long* map, const double* gv, int kk,
                              int slot, double* api, DevStatus* st) {
  count_launch(st);
  const long long tot = (long long)nvec * nfree;
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const long long f = e % nfree;
  const int c = (int)(e / nfree);
  const long long gi = map ? map[f] : f;
  api[e] = gv[((long long)c * g.padded + g.guard + gi) * kk + slot];
}
void launch_api_to_grid(const GridDesc& g, int nvec, long long nfree, const long long* map, const double* api,
                        double* gridv, int kk, int slot, DevStatus* st, cudaStream_t s) {
  const long long tot = (long long)nvec * nfree;
  if (tot == 0) return;
  k_api_to_grid<<<(unsigned int)((tot + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(g, nvec, nfree, map, api, gridv,
                                                                                   kk, slot, st);
}
void launch_grid_to_api(const GridDesc& g, int nvec, long long nfree, const long long* map, const double* gridv,
                        int kk, int slot, double* api, DevStatus* st, cudaStream_t s) {
  const long long tot = (long long)nvec * nfree;
  if (tot == 0) return;
  k_grid_to_api<<<(unsigned int)((tot + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(g, nvec, nfree, map, gridv, kk,
                                                                                   slot, api, st);
}

__global__ void __launch_bounds__(NTHREADS) k_dot(GridDesc g, int nvec, int kk, const double* a, const double* b,
                                                  double* outp, double* partial, unsigned int* counter) {
  const long long tot = (long long)nvec * g.npts;
  const long long estride = (long long)gridDim.x * blockDim.x;
  double v[1] = {0.0};
  for (long long e = (long long)gtid(); e < tot; e += estride) {
    const long long i = e % g.npts;
    const int c = (int)(e / g.npts);
    const long long idx = ((long long)c * g.padded + g.guard + i) * kk;
    v[0] = fma(a[idx], b[idx], v[0]);
  }
  double out[1];
  if (reduce_last_block<1>(v, partial, counter, out)) *outp = out[0];
}
// reference norm of the instability detector: ||c0||^2 + tau^2 ||c1||^2 (slot 0 of the chain)
__global__ void __launch_bounds__(NTHREADS) k_ref_norm(GridDesc g, int nvec, const double* c0, const double* c1,
                                                       double tau, DevStatus* st, double* partial,
                                                       unsigned int* counter) {
  const long long tot = (long long)nvec * g.npts;
  const long long estride = (long long)gridDim.x * blockDim.x;
  double v[1] = {0.0};
  for (long long e = (long long)gtid(); e < tot; e += estride) {
    const long long i = e % g.npts;
    const int c = (int)(e / g.npts);
    const long long idx = (long long)c * g.padded + g.guard + i;
    const double w = tau * c1[idx];
    v[0] = fma(c0[idx], c0[idx], fma(w, w, v[0]));
  }
  double out[1];
  if (reduce_last_block<1>(v, partial, counter, out)) st->u0norm2 = out[0];
}
void launch_ref_norm(const GridDesc& g, int nvec, const double* c0, const double* c1, double tau, DevStatus* st,
                     double* partial, unsigned int* counter, cudaStream_t s) {
  const long long tot = (long long)nvec * g.npts;
  k_ref_norm<<<red_grid(tot), NTHREADS, 0, s>>>(g, nvec, c0, c1, tau, st, partial, counter);
}
void launch_dot(const GridDesc& g, int nvec, int kk, const double* a, const double* b, double* out, double* partial,
                unsigned int* counter, cudaStream_t s) {
  const long long tot = (long long)nvec * g.npts;
  k_dot<<<red_grid(tot), NTHREADS, 0, s>>>(g, nvec, kk, a, b, out, partial, counter);
}
__global__ void k_scale(GridDesc g, int nvec, int kk, double* a, const double* num, int inv_sqrt) {
  const long long tot = (long long)nvec * g.npts;
  const long long e = (long long)gtid();
  if (e >= tot) return;
  const long long i = e % g.npts;
  const int c = (int)(e / g.npts);
  const long long idx = ((long long)c * g.padded + g.guard + i) * kk;
  const double sc = inv_sqrt ? 1.0 / sqrt(*num) : *num;
  a[idx] *= sc;
}
void launch_scale(const GridDesc& g, int nvec, int kk, double* a, const double* num, int inv_sqrt, cudaStream_t s) {
  const long long tot = (long long)nvec * g.npts;
  k_scale<<<(unsigned int)((tot + NTHREADS - 1) / NTHREADS), NTHREADS, 0, s>>>(g, nvec, kk, a, num, inv_sqrt);
}

}  // namespace ga

