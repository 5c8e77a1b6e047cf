// Slab line solver of the Kronecker preconditioner for many-line (3D) grids
// (DESIGN.md "Line solves").
//
// One warp owns a slab of 32 line-slots (a slot = one line x one right-hand
// side) and the whole line length: the slab is staged in shared memory with
// coalesced 256-byte rows (y and z lines: 32 consecutive doubles of the
// multi-vector per line position; x lines: each line's contiguous run read in
// 32-double chunks and transposed through a padded slab, row stride 32 + kk,
// conflict-free both ways), then each lane runs the banded forward and
// backward substitution of its slot on-chip, and the slab is written back.
// Each sweep therefore moves 16 B per DoF and right-hand side (read + write),
// against 32 B for a streamed sweep that round-trips the forward result.
// PRO (first direction): input = s o (r - alpha q) with x += alpha p, r updated
// in place.  EPI (last direction): output z = s o y with the r.z / r.r partial
// sums and the PCG scalar step F1 in the last block.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tile_core.cuh"

namespace ga {

// 8-byte asynchronous global -> shared copy (Ampere-style LDGSTS, sm_80+): the whole
// slab of a warp is in flight at once without staging through registers
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned int d = (unsigned int)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

struct SlabArgs {
  double* t;            // z multi-vector (guard-offset): input/output of the sweep
  const double* L;      // banded Cholesky rows of the direction, (len + P + 1) x (P + 1)
  int len;              // line length
  long long es;         // element stride along the line (doubles)
  int dirx;             // 1: lines along x (contiguous runs of len * kk doubles)
  int kk, nvec;
  long long nrow;       // dirx: lines per component; else rows (the remaining coordinate)
  long long rowlen;     // !dirx: doubles per row (nx * kk)
  long long srow;       // !dirx: stride between rows; dirx: stride between lines (nx * kk)
  long long sc;         // component stride (padded * kk)
  const double* s;      // scaling per grid point
  double *x, *r;
  const double *p, *q;
  PcgState* pcg;
  DevStatus* st;
  double* partial;
  unsigned int* counter;
  int maxit, update;
  unsigned long long cond;
};

template <int P, bool DIRX, bool PRO, bool EPI, int NW>
__global__ void __launch_bounds__(32 * NW) k_line_slab(SlabArgs a) {
  if (a.st->status != 0) return;  // uniform
  count_launch(a.st);
  extern __shared__ double sm_slab[];
  const int len = a.len, kk = a.kk, LD = 32 + kk;
  double* Ls = sm_slab;                                   // (len + P + 1) x (P + 1)
  const int nL = (len + P + 1) * (P + 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* slab = sm_slab + ((nL + 1) & ~1) + (size_t)w * len * LD;
  for (int i = threadIdx.x; i < nL; i += 32 * NW) Ls[i] = __ldg(a.L + i);
  double al[KMAX];
  bool upd = false;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) al[j] = 0.0;
  if (PRO && a.update && !a.pcg->first) {
    upd = true;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) al[j] = j < kk ? a.pcg->alpha[j] : 0.0;
  }
  __syncthreads();
  // ---- this warp's slab
  const long long sid = (long long)blockIdx.x * NW + w;
  long long nslab, base;
  int ncol;            // valid columns (slots)
  int lps = 32 / kk;   // dirx: lines per slab
  if (DIRX) {
    const long long nl = (long long)a.nvec * a.nrow;
    nslab = (nl + lps - 1) / lps;
    const long long l0 = sid * lps;
    ncol = (int)(nl - l0 < lps ? nl - l0 : lps) * kk;
    const long long c = l0 / a.nrow;  // component of the first line (lines of one slab may span two)
    base = l0;                        // line index; offsets computed per line below
    (void)c;
  } else {
    const long long per = (a.rowlen + 31) / 32;
    nslab = (long long)a.nvec * a.nrow * per;
    const long long c = sid / (a.nrow * per), rem = sid % (a.nrow * per);
    const long long row = rem / per, ch = rem % per;
    ncol = (int)(a.rowlen - ch * 32 < 32 ? a.rowlen - ch * 32 : 32);
    base = c * a.sc + row * a.srow + ch * 32;
  }
  const bool live = sid < nslab;
  auto line_off = [&](long long line) -> long long {  // dirx: offset of element 0 of a line
    const long long c = line / a.nrow, l = line % a.nrow;
    return c * a.sc + l * a.srow;
  };
  auto sel_alpha = [&](long long j) -> double {
    double aj = al[0];
#pragma unroll
    for (int jj = 1; jj < KMAX; ++jj) aj = (jj == j) ? al[jj] : aj;
    return aj;
  };
  auto fetch = [&](long long o) -> double {
    if (PRO) {
      double rv = a.r[o];
      if (upd) {
        const int j = (int)(o % kk);
        const double xv = a.x[o], pv = a.p[o], qv = a.q[o];
        double aj = al[0];
#pragma unroll
        for (int jj = 1; jj < KMAX; ++jj) aj = (jj == j) ? al[jj] : aj;
        a.x[o] = fma(aj, pv, xv);
        rv = fma(-aj, qv, rv);
        a.r[o] = rv;
      }
      return rv * __ldg(a.s + (o % a.sc) / kk);
    }
    return a.t[o];
  };
  double acc[2 * KMAX];
#pragma unroll
  for (int j = 0; j < 2 * KMAX; ++j) acc[j] = 0.0;
  auto emit = [&](long long o, double v) {
    if (EPI) {
      const double z = v * __ldg(a.s + (o % a.sc) / kk);
      const double rv = a.r[o];
      const int j = (int)(o % kk);
#pragma unroll
      for (int jj = 0; jj < KMAX; ++jj) {  // branch-free selects keep acc in registers
        const double m = (jj == j) ? rv : 0.0;
        acc[jj] = fma(m, z, acc[jj]);
        acc[KMAX + jj] = fma(m, rv, acc[KMAX + jj]);
      }
      a.t[o] = z;
    } else {
      a.t[o] = v;
    }
  };
  if (live) {
    // ---- load
    if (!PRO) {
      // plain input: asynchronous copies, all rows of the slab in flight
      if (DIRX) {
        const int nl = ncol / kk;
        const int run = len * kk;
        for (int l = 0; l < nl; ++l) {
          const double* src = a.t + line_off(base + l);
          for (int e = lane; e < run; e += 32) cp_async8(slab + (e / kk) * LD + l * kk + e % kk, src + e);
        }
      } else if (lane < ncol) {
        const double* src = a.t + base + lane;
        for (int i = 0; i < len; ++i) cp_async8(slab + i * LD + lane, src + (long long)i * a.es);
      }
      cp_async_wait_all();
    } else if (DIRX) {
      const int nl = ncol / kk;
      const int run = len * kk;
      for (int l = 0; l < nl; ++l) {
        const long long lo = line_off(base + l);
        for (int e0 = 0; e0 < run; e0 += 32 * 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * 32 + lane;
            v[u] = e < run ? fetch(lo + e) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * 32 + lane;
            if (e < run) slab[(e / kk) * LD + l * kk + e % kk] = v[u];
          }
        }
      }
    } else {
      // prologue rows in batches: every load of the batch is issued before any store
      // (the x / r stores could alias later loads, which would serialise the rows)
      constexpr int B = 8;
      const double aj = sel_alpha((base + lane) % kk);
      for (int i0 = 0; i0 < len; i0 += B) {
        double rv[B], xv[B], pv[B], qv[B], sv[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const bool ok = i0 + u < len && lane < ncol;
          const long long o = base + lane + (long long)(i0 + u) * a.es;
          rv[u] = ok ? a.r[o] : 0.0;
          sv[u] = ok ? __ldg(a.s + (o % a.sc) / kk) : 0.0;
          if (upd) {
            xv[u] = ok ? a.x[o] : 0.0;
            pv[u] = ok ? a.p[o] : 0.0;
            qv[u] = ok ? a.q[o] : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const bool ok = i0 + u < len && lane < ncol;
          const long long o = base + lane + (long long)(i0 + u) * a.es;
          if (upd && ok) {
            a.x[o] = fma(aj, pv[u], xv[u]);
            rv[u] = fma(-aj, qv[u], rv[u]);
            a.r[o] = rv[u];
          }
          if (i0 + u < len) slab[(i0 + u) * LD + lane] = rv[u] * sv[u];
        }
      }
    }
    __syncwarp();
    // ---- forward L y = t and backward L^T z = y, lane = slot
    if (lane < ncol) {
      double* col = slab + lane;
      double ym[P];
#pragma unroll
      for (int u = 0; u < P; ++u) ym[u] = 0.0;
#pragma unroll 4
      for (int i = 0; i < len; ++i) {
        const double* Li = Ls + i * (P + 1);
        double v = col[i * LD];
#pragma unroll
        for (int u = P; u >= 1; --u) v = fma(-Li[u], ym[u - 1], v);
        v *= Li[0];
#pragma unroll
        for (int u = P - 1; u >= 1; --u) ym[u] = ym[u - 1];
        ym[0] = v;
        col[i * LD] = v;
      }
#pragma unroll
      for (int u = 0; u < P; ++u) ym[u] = 0.0;
#pragma unroll 4
      for (int i = len - 1; i >= 0; --i) {
        double v = col[i * LD];
#pragma unroll
        for (int u = P; u >= 1; --u) v = fma(-Ls[(i + u) * (P + 1) + u], ym[u - 1], v);
        v *= Ls[i * (P + 1)];
#pragma unroll
        for (int u = P - 1; u >= 1; --u) ym[u] = ym[u - 1];
        ym[0] = v;
        col[i * LD] = v;
      }
    }
    __syncwarp();
    // ---- store
    if (DIRX) {
      const int nl = ncol / kk;
      const int run = len * kk;
      for (int l = 0; l < nl; ++l) {
        const long long lo = line_off(base + l);
#pragma unroll 4
        for (int e = lane; e < run; e += 32) emit(lo + e, slab[(e / kk) * LD + l * kk + e % kk]);
      }
    } else if (lane < ncol) {
      if (!EPI) {
        for (int i = 0; i < len; ++i) a.t[base + lane + (long long)i * a.es] = slab[i * LD + lane];
      } else {
        constexpr int B = 8;
        const int j = (int)((base + lane) % kk);
        double rz = 0.0, rr = 0.0;
        for (int i0 = 0; i0 < len; i0 += B) {
          double rv[B], sv[B];
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const long long o = base + lane + (long long)(i0 + u) * a.es;
            const bool ok = i0 + u < len;
            rv[u] = ok ? a.r[o] : 0.0;
            sv[u] = ok ? __ldg(a.s + (o % a.sc) / kk) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < B; ++u) {
            if (i0 + u < len) {
              const double z = slab[(i0 + u) * LD + lane] * sv[u];
              rz = fma(rv[u], z, rz);
              rr = fma(rv[u], rv[u], rr);
              a.t[base + lane + (long long)(i0 + u) * a.es] = z;
            }
          }
        }
#pragma unroll
        for (int jj = 0; jj < KMAX; ++jj) {
          acc[jj] += (jj == j) ? rz : 0.0;
          acc[KMAX + jj] += (jj == j) ? rr : 0.0;
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

static size_t slab_smem(int len, int p, int kk, int nw) {
  const size_t nL = (size_t)(len + p + 1) * (p + 1);
  return sizeof(double) * (((nL + 1) & ~(size_t)1) + (size_t)nw * len * (32 + kk));
}

template <int P, bool DIRX, bool PRO, bool EPI>
static bool slab_go(const SlabArgs& a, cudaStream_t s) {
  constexpr int NW = 2;
  const size_t sm = slab_smem(a.len, P, a.kk, NW);
  if (sm > 227 * 1024) return false;
  static size_t attr = 0;
  if (sm > attr) {
    if (cudaFuncSetAttribute(k_line_slab<P, DIRX, PRO, EPI, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm) != cudaSuccess)
      return false;
    attr = sm;
  }
  long long nslab;
  if (DIRX) {
    const int lps = 32 / a.kk;
    nslab = ((long long)a.nvec * a.nrow + lps - 1) / lps;
  } else {
    nslab = (long long)a.nvec * a.nrow * ((a.rowlen + 31) / 32);
  }
  const unsigned int blocks = (unsigned int)((nslab + NW - 1) / NW);
  k_line_slab<P, DIRX, PRO, EPI, NW><<<blocks, 32 * NW, sm, s>>>(a);
  return true;
}

template <int P>
static bool slab_p(const SlabArgs& a, bool pro, bool epi, cudaStream_t s) {
  if (a.dirx) {
    if (pro) return slab_go<P, true, true, false>(a, s);
    if (epi) return slab_go<P, true, false, true>(a, s);
    return slab_go<P, true, false, false>(a, s);
  }
  if (pro) return slab_go<P, false, true, false>(a, s);
  if (epi) return slab_go<P, false, false, true>(a, s);
  return slab_go<P, false, false, false>(a, s);
}

// Fits the slab of one line set in shared memory?
bool slab_supported(int len, int p, int kk) { return slab_smem(len, p, kk, 2) <= 227 * 1024; }

bool launch_line_slab(int p, const SlabArgs& a, bool pro, bool epi, cudaStream_t s) {
  switch (p) {
    case 1: return slab_p<1>(a, pro, epi, s);
    case 2: return slab_p<2>(a, pro, epi, s);
    case 3: return slab_p<3>(a, pro, epi, s);
    case 4: return slab_p<4>(a, pro, epi, s);
    case 5: return slab_p<5>(a, pro, epi, s);
    case 6: return slab_p<6>(a, pro, epi, s);
    default: return slab_p<7>(a, pro, epi, s);
  }
}

// Plane-fused y and x sweeps (3D, single patch, a whole xy-plane of the k right-hand sides in
// shared memory): one CTA per (component, z-plane) loads the plane with the PCG prologue fused
// (x += alpha p, r -= alpha q, t = s o r), runs the y-line solves (thread per (x, rhs) column)
// and the x-line solves (thread per (y, rhs) row) on-chip, and writes the plane once; the z
// sweep with the epilogue follows as a streamed kernel.  Row stride LDR = nx*kk + 1 (odd):
// column walks and row walks are both conflict-free per half warp.
template <int P>
__global__ void __launch_bounds__(512) k_prec_plane(SlabArgs ay, SlabArgs ax, int nx, int ny, int nz) {
  if (ay.st->status != 0) return;
  count_launch(ay.st);
  extern __shared__ double sm_pl[];
  const int kk = ay.kk, rl = nx * kk, LDR = rl + 1;
  double* Ly = sm_pl;                              // (ny + P + 1) x (P + 1)
  double* Lx = Ly + (ny + P + 1) * (P + 1);        // (nx + P + 1) x (P + 1)
  double* pl = Lx + (nx + P + 1) * (P + 1);        // [ny][LDR]
  for (int i = threadIdx.x; i < (ny + P + 1) * (P + 1); i += blockDim.x) Ly[i] = __ldg(ay.L + i);
  for (int i = threadIdx.x; i < (nx + P + 1) * (P + 1); i += blockDim.x) Lx[i] = __ldg(ax.L + i);
  const int c = blockIdx.x / nz, z = blockIdx.x % nz;
  const long long base = c * ay.sc + (long long)z * ny * rl;  // offset of (c, z, 0, 0, 0)
  double al[KMAX];
  bool upd = false;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) al[j] = 0.0;
  if (ay.update && !ay.pcg->first) {
    upd = true;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) al[j] = j < kk ? ay.pcg->alpha[j] : 0.0;
  }
  // ---- load with the prologue: rows of the plane are contiguous runs of rl doubles
  for (int i = threadIdx.x; i < ny * rl; i += blockDim.x) {
    const int y = i / rl, q = i - y * rl;
    const long long o = base + i;
    const int j = q % kk;
    double aj = al[0];
#pragma unroll
    for (int jj = 1; jj < KMAX; ++jj) aj = (jj == j) ? al[jj] : aj;
    double rv = ay.r[o];
    if (upd) {
      const double xv = ay.x[o], pv = ay.p[o], qv = ay.q[o];
      ay.x[o] = fma(aj, pv, xv);
      rv = fma(-aj, qv, rv);
      ay.r[o] = rv;
    }
    pl[y * LDR + q] = rv * __ldg(ay.s + (o % ay.sc) / kk);
  }
  __syncthreads();
  // ---- y lines: thread per column q = x*kk + j
  for (int q = threadIdx.x; q < rl; q += blockDim.x) {
    double* col = pl + q;
    double ym[P];
#pragma unroll
    for (int u = 0; u < P; ++u) ym[u] = 0.0;
    for (int i = 0; i < ny; ++i) {
      const double* Li = Ly + i * (P + 1);
      double v = col[i * LDR];
#pragma unroll
      for (int u = P; u >= 1; --u) v = fma(-Li[u], ym[u - 1], v);
      v *= Li[0];
#pragma unroll
      for (int u = P - 1; u >= 1; --u) ym[u] = ym[u - 1];
      ym[0] = v;
      col[i * LDR] = v;
    }
#pragma unroll
    for (int u = 0; u < P; ++u) ym[u] = 0.0;
    for (int i = ny - 1; i >= 0; --i) {
      double v = col[i * LDR];
#pragma unroll
      for (int u = P; u >= 1; --u) v = fma(-Ly[(i + u) * (P + 1) + u], ym[u - 1], v);
      v *= Ly[i * (P + 1)];
#pragma unroll
      for (int u = P - 1; u >= 1; --u) ym[u] = ym[u - 1];
      ym[0] = v;
      col[i * LDR] = v;
    }
  }
  __syncthreads();
  // ---- x lines: thread per (y, j)
  for (int t = threadIdx.x; t < ny * kk; t += blockDim.x) {
    const int y = t / kk, j = t - y * kk;
    double* row = pl + y * LDR + j;
    double ym[P];
#pragma unroll
    for (int u = 0; u < P; ++u) ym[u] = 0.0;
    for (int i = 0; i < nx; ++i) {
      const double* Li = Lx + i * (P + 1);
      double v = row[i * kk];
#pragma unroll
      for (int u = P; u >= 1; --u) v = fma(-Li[u], ym[u - 1], v);
      v *= Li[0];
#pragma unroll
      for (int u = P - 1; u >= 1; --u) ym[u] = ym[u - 1];
      ym[0] = v;
      row[i * kk] = v;
    }
#pragma unroll
    for (int u = 0; u < P; ++u) ym[u] = 0.0;
    for (int i = nx - 1; i >= 0; --i) {
      double v = row[i * kk];
#pragma unroll
      for (int u = P; u >= 1; --u) v = fma(-Lx[(i + u) * (P + 1) + u], ym[u - 1], v);
      v *= Lx[i * (P + 1)];
#pragma unroll
      for (int u = P - 1; u >= 1; --u) ym[u] = ym[u - 1];
      ym[0] = v;
      row[i * kk] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ny * rl; i += blockDim.x) {
    const int y = i / rl, q = i - y * rl;
    ay.t[base + i] = pl[y * LDR + q];
  }
}

static size_t plane_smem(int nx, int ny, int p, int kk) {
  return sizeof(double) * ((size_t)(ny + p + 1) * (p + 1) + (size_t)(nx + p + 1) * (p + 1) + (size_t)ny * (nx * kk + 1));
}

template <int P>
static bool plane_go(const SlabArgs& ay, const SlabArgs& ax, int nx, int ny, int nz, int nvec, cudaStream_t s) {
  const size_t sm = plane_smem(nx, ny, P, ay.kk);
  if (sm > 227 * 1024) return false;
  static size_t attr = 0;
  if (sm > attr) {
    if (cudaFuncSetAttribute(k_prec_plane<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
      return false;
    attr = sm;
  }
  const int work = std::max(nx * ay.kk, ny * ay.kk);
  const int threads = std::min(512, (work + 31) / 32 * 32);
  k_prec_plane<P><<<(unsigned int)(nvec * nz), threads, sm, s>>>(ay, ax, nx, ny, nz);
  return true;
}

bool launch_line_sf_epi_z(const PrecArgs& a, cudaStream_t s);  // ops.cu: streamed z sweep with the epilogue

static bool launch_precond_plane(const PrecArgs& a, cudaStream_t s) {
  const GridDesc& g = a.g;
  const int bd[3] = {a.bd[0][0], a.bd[0][1], a.bd[0][2]};
  const long long kk = a.kk, off = g.guard * kk;
  SlabArgs ay, ax;
  memset(&ay, 0, sizeof(ay));
  ay.t = a.z + off; ay.L = a.L[0][1]; ay.len = bd[1]; ay.kk = a.kk; ay.nvec = a.nvec; ay.sc = g.padded * kk;
  ay.s = a.s[0]; ay.x = a.x + off; ay.r = a.r + off; ay.p = a.p0 + off; ay.q = a.q + off;
  ay.pcg = a.pcg; ay.st = a.st; ay.update = a.update;
  ax = ay;
  ax.L = a.L[0][0]; ax.len = bd[0];
  bool ok = false;
  switch (a.p) {
    case 1: ok = plane_go<1>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
    case 2: ok = plane_go<2>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
    case 3: ok = plane_go<3>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
    case 4: ok = plane_go<4>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
    case 5: ok = plane_go<5>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
    case 6: ok = plane_go<6>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
    default: ok = plane_go<7>(ay, ax, bd[0], bd[1], bd[2], a.nvec, s); break;
  }
  if (!ok) return false;
  return launch_line_sf_epi_z(a, s);
}

// The x sweep alone as a slab (no prologue / epilogue), between streamed y and z sweeps.
bool launch_xslab(const PrecArgs& a, cudaStream_t s) {
  const GridDesc& g = a.g;
  if (!slab_supported(a.bd[0][0], a.p, a.kk)) return false;
  const long long kk = a.kk, off = g.guard * kk;
  SlabArgs sa;
  memset(&sa, 0, sizeof(sa));
  sa.t = a.z + off; sa.L = a.L[0][0]; sa.len = a.bd[0][0]; sa.kk = a.kk; sa.nvec = a.nvec;
  sa.sc = g.padded * kk; sa.s = a.s[0];
  sa.pcg = a.pcg; sa.st = a.st; sa.partial = a.partial; sa.counter = a.counter;
  sa.dirx = 1; sa.es = kk; sa.nrow = (long long)g.ny * g.nz; sa.srow = (long long)g.nx * kk;
  return launch_line_slab(a.p, sa, false, false, s);
}

// Host helper: one preconditioner application on a single-patch grid by slab
// sweeps, directions y (PRO), x, z (EPI) as in the streamed path.
bool launch_precond_slab(const PrecArgs& a, cudaStream_t s) {
  const GridDesc& g = a.g;
  if (g.dim != 3) return false;
  const int bd[3] = {a.bd[0][0], a.bd[0][1], a.bd[0][2]};
  // plane-fused y/x sweeps: opt-in (GA_PLANE=1).  Measured: 117 vs 136 us per
  // application warm at C3 p=4 n=96 but equal cold and a slower step (one wave of n_f CTAs
  // with one plane each is latency-bound), so the default keeps slabs / streamed sweeps
  static int plane_mode = -1;
  if (plane_mode < 0) { const char* e = getenv("GA_PLANE"); plane_mode = (e && *e == '1') ? 1 : 0; }
  if (plane_mode && plane_smem(bd[0], bd[1], a.p, a.kk) <= 227 * 1024 && launch_precond_plane(a, s)) return true;
  // measured: the slab wins for short lines of one component (C3 p=4 n=96:
  // 137 vs 167 us per application); longer lines leave only ~4 warps per SM (one line set
  // per warp in shared memory) and the streamed sweeps are faster (n=128: 251 vs 309 us)
  if (a.nvec != 1 || std::max(bd[0], std::max(bd[1], bd[2])) > 100) return false;
  for (int d = 0; d < 3; ++d)
    if (!slab_supported(bd[d], a.p, a.kk)) return false;
  const long long kk = a.kk;
  const long long off = g.guard * kk;
  const int order[3] = {1, 0, 2};
  for (int k = 0; k < 3; ++k) {
    const int d = order[k];
    SlabArgs sa;
    memset(&sa, 0, sizeof(sa));
    sa.t = a.z + off; sa.L = a.L[0][d]; sa.len = bd[d]; sa.kk = a.kk; sa.nvec = a.nvec;
    sa.sc = g.padded * kk;
    sa.s = a.s[0];
    sa.x = a.x + off; sa.r = a.r + off; sa.p = a.p0 + off; sa.q = a.q + off;
    sa.pcg = a.pcg; sa.st = a.st; sa.partial = a.partial; sa.counter = a.counter;
    sa.maxit = a.maxit; sa.update = a.update; sa.cond = a.cond;
    if (d == 0) {
      sa.dirx = 1; sa.es = kk; sa.nrow = (long long)g.ny * g.nz; sa.srow = (long long)g.nx * kk;
    } else if (d == 1) {
      sa.es = (long long)g.nx * kk; sa.rowlen = (long long)g.nx * kk; sa.nrow = g.nz;
      sa.srow = (long long)g.nx * g.ny * kk;
    } else {
      sa.es = (long long)g.nx * g.ny * kk; sa.rowlen = (long long)g.nx * kk; sa.nrow = g.ny;
      sa.srow = (long long)g.nx * kk;
    }
    if (!launch_line_slab(a.p, sa, k == 0, k == 2, s)) return false;
  }
  return true;
}

}  // namespace ga
