// Device core of the chunked shared-memory line solver (included by ops.cu
// and the persistent solver persist.cu).
#pragma once
#include <cuda_runtime.h>

#include "ops.cuh"

namespace ga {

// ---------------------------------------------------------------------------
// Tile line solver: a CTA stages ST line-slots x the
// full line length in shared memory (coalesced), plus the sweep factors, then
// solves them with the chunked recurrence: lane -> (slot, chunk), local
// substitution from a zero state, Kogge-Stone scan of the chunk states,
// correction with the precomputed homogeneous responses.  Forward (L) and
// backward (L^T, as a forward sweep of the reversed line) back to back.
// Single patch: the first direction fuses the PCG update x += alpha p,
// r -= alpha q and the input scaling s o r; the last direction fuses the
// output scaling, the r.z / r.r reductions and the PCG scalar step (F1).
// ---------------------------------------------------------------------------
struct TileLine {
  long long* trace;    // debug timestamps (GA_TRACE)
  double* t;
  int mode;            // 0: slots contiguous at fixed element (y/z lines); 1: lines contiguous (x lines)
  int n;               // line length
  long long es;        // mode 0: element stride
  int nrows, nr2, rowlen;
  long long sA, sB;    // mode 0 row offset (r/nr2)*sA + (r%nr2)*sB; mode 1 line base likewise
  int nlines, nl2, kk;
  int ST;              // slots per tile (8, 16 or 32)
  const double* Ff;
  const double* Fb;
  int flen;            // doubles per factor buffer
  int clen, C, L;
  // fusion (single patch; t is the z vector, offsets into x/r/p/q/s are the same)
  int pro, epi, update;
  const double* s;     // scaling per grid point
  long long padkk;     // padded * kk (component stride of an MV)
  double *x, *r;
  const double *p0, *p1, *q;
  PcgState* pcg;
  double* partial;
  unsigned int* counter;
  double tol2;
  int maxit;
  unsigned long long cond;
  DevStatus* st;
};

// F1: convergence test, beta, loop condition (thread 0 of the last block).
static __device__ void pcg_finalize(PcgState* pc, DevStatus* st, int kk, int maxit, unsigned long long condh,
                             const double* rz, const double* rr) {
  int any = 0;
  for (int j = 0; j < kk; ++j) {
    pc->rz[j] = rz[j];
    pc->rr[j] = rr[j];
    if (pc->active[j] && rr[j] <= pc->thr[j]) pc->active[j] = 0;
    if (pc->first) {
      pc->beta[j] = 0.0;
    } else {
      pc->beta[j] = pc->rzold[j] != 0.0 ? rz[j] / pc->rzold[j] : 0.0;
    }
    pc->rzold[j] = rz[j];
    any |= pc->active[j];
  }
  if (pc->first) pc->pfirst = 1;
  pc->first = 0;
  int cond = any;
  // safety: the iteration counter lives in F2; never loop more than maxit + 2 F1 calls
  pc->guard += 1;
  if ((long long)pc->guard > (long long)maxit + 2 && st->status == 0) {
    st->status = -7;  // GA_ERR_CUDA: inconsistent device state
    st->fail_step = st->steps;
  }
  if (any && pc->iter >= maxit) {
    if (st->status == 0 && pc->phase == 0) {  // the refinement phase may stop at maxit
      st->status = -5;  // GA_ERR_NOCONV
      st->fail_step = st->steps;
      for (int j = 0; j < kk; ++j)
        if (pc->active[j]) { st->fail_block = j; break; }
    }
    cond = 0;
  }
  if (st->status != 0) cond = 0;
  if (condh) cudaGraphSetConditional((cudaGraphConditionalHandle)condh, cond ? 1u : 0u);
}

template <int P>
__device__ __forceinline__ void tile_sweep(double* __restrict__ tile, int LD, double* __restrict__ bsc,
                                           const double* __restrict__ F, const TileLine& a, bool rev) {
  const int n = a.n, ST = a.ST, cpw = 32 / ST;
  const int lane = threadIdx.x & 31;
  const int sl = lane % ST;
  const int ch = (threadIdx.x >> 5) * cpw + lane / ST;  // chunk of this thread
  const double* dinv = F;
  const double* coef = F + n;
  const double* H = F + (size_t)n * (1 + P);
  const double* A = F + (size_t)n * (1 + 2 * P);
  const int lo = ch * a.clen, hi = min(n, lo + a.clen);
  double y[P];
#pragma unroll
  for (int u = 0; u < P; ++u) y[u] = 0.0;
  // phase A: local substitution of chunk ch from a zero incoming state
  for (int i = lo; i < hi; ++i) {
    const int pi = rev ? n - 1 - i : i;
    double v = tile[pi * LD + sl];
#pragma unroll
    for (int u = P; u >= 1; --u) v = fma(-coef[i * P + u - 1], y[u - 1], v);
    v *= dinv[i];
#pragma unroll
    for (int u = P - 1; u >= 1; --u) y[u] = y[u - 1];
    y[0] = v;
    tile[pi * LD + sl] = v;
  }
  // phase B: sigma_{w+1} = T_w sigma_w + tau_w, w = 0..C-2, Kogge-Stone over chunks
  const int E = a.C - 1;
  double b[P];
#pragma unroll
  for (int u = 0; u < P; ++u) b[u] = y[u];  // tau_w[u] = y_{hi-1-u}
  for (int l = 0; l < a.L; ++l) {
    const int d = 1 << l;
    if (ch < E) {
#pragma unroll
      for (int u = 0; u < P; ++u) bsc[(ch * P + u) * ST + sl] = b[u];
    }
    __syncthreads();
    if (ch < E && ch >= d) {
      const double* Aw = A + ((size_t)l * a.C + ch) * P * P;
      double bp[P];
#pragma unroll
      for (int u = 0; u < P; ++u) bp[u] = bsc[((ch - d) * P + u) * ST + sl];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        double s2 = b[r];
#pragma unroll
        for (int c = 0; c < P; ++c) s2 = fma(Aw[r * P + c], bp[c], s2);
        b[r] = s2;
      }
    }
    __syncthreads();
  }
  if (ch < E) {
#pragma unroll
    for (int u = 0; u < P; ++u) bsc[(ch * P + u) * ST + sl] = b[u];
  }
  __syncthreads();
  // phase C: y_i += sum_u H_{i,u} sigma_ch[u]
  if (ch >= 1 && ch < a.C) {
    double sg[P];
#pragma unroll
    for (int u = 0; u < P; ++u) sg[u] = bsc[((ch - 1) * P + u) * ST + sl];
    for (int i = lo; i < hi; ++i) {
      const int pi = rev ? n - 1 - i : i;
      double v = tile[pi * LD + sl];
#pragma unroll
      for (int u = 0; u < P; ++u) v = fma(H[i * P + u], sg[u], v);
      tile[pi * LD + sl] = v;
    }
  }
  __syncthreads();
}

// element e of this tile -> (tile column, global offset); returns false if outside
struct TileMap {
  int mode, n, ST, nsl, kk;
  long long base;  // mode 0
  long long es;
  int l0, sig0, per, nl2;
  long long sA, sB;
};

__device__ __forceinline__ int div_kk(int e, int kk) {
  return kk == 2 ? (e >> 1) : (kk == 1 ? e : (kk == 4 ? (e >> 2) : e / 3));
}

// One element of the tile: global offset g (relative to a.t), grid point gp
// (index of the scaling s), rhs j, tile position (i, col).
template <int P, bool LOAD>
__device__ __forceinline__ void tile_elem(const TileLine& a, double* tile, int LD, long long g, long long gp, int j,
                                          int i, int col, bool upd, const double* al, const double* pp,
                                          double* acc) {
  if (LOAD) {
    double v;
    if (a.pro) {
      v = a.r[g];
      const double sv = a.s[gp];
      if (upd) {
        double alj = al[0];
#pragma unroll
        for (int jj = 1; jj < KMAX; ++jj) alj = (j == jj) ? al[jj] : alj;
        if (alj != 0.0) {
          a.x[g] = fma(alj, pp[g], a.x[g]);
          v = fma(-alj, a.q[g], v);
          a.r[g] = v;
        }
      }
      v *= sv;
    } else {
      v = a.t[g];
    }
    tile[i * LD + col] = v;
  } else {
    double v = tile[i * LD + col];
    if (a.epi) {
      v *= a.s[gp];
      const double rv = a.r[g];
#pragma unroll
      for (int jj = 0; jj < KMAX; ++jj)
        if (jj == j) { acc[jj] = fma(rv, v, acc[jj]); acc[KMAX + jj] = fma(rv, rv, acc[KMAX + jj]); }
    }
    a.t[g] = v;
  }
}

template <int P, bool LOAD>
__device__ __forceinline__ void tile_io(const TileLine& a, int tileid, double* tile, int LD, bool upd, const double* al,
                                        const double* pp, double* acc) {
  const int n = a.n, ST = a.ST, nthr = blockDim.x, tid = threadIdx.x;
  const int lgST = ST == 32 ? 5 : (ST == 16 ? 4 : 3);
  if (a.mode == 0) {
    // y/z lines: ST slots f0..f0+nsl-1 of one row, contiguous at every element i
    const int tpr = (a.rowlen + ST - 1) / ST;
    const int r = tileid / tpr;
    const int f0 = (tileid - r * tpr) * ST;
    const long long roff = (long long)(r % a.nr2) * a.sB;
    const long long base = (long long)(r / a.nr2) * a.sA + roff + f0;
    const long long gp0 = roff / a.kk;      // grid point of slot 0 at element 0 (component-free)
    const long long ges = a.es / a.kk;
    const int nsl = min(ST, a.rowlen - f0);
#pragma unroll 4
    for (int idx = tid; idx < (n << lgST); idx += nthr) {
      const int i = idx >> lgST, col = idx & (ST - 1);
      if (col >= nsl) continue;
      const int f = f0 + col;
      const int xo = div_kk(f, a.kk);
      tile_elem<P, LOAD>(a, tile, LD, base + col + (long long)i * a.es, gp0 + xo + (long long)i * ges, f - xo * a.kk,
                         i, col, upd, al, pp, acc);
    }
  } else {
    // x lines: contiguous n*kk elements per line; slots (line, rhs) sig0..sig0+nsl-1
    const int sig0 = tileid * ST;
    const int nsl = min(ST, a.nlines * a.kk - sig0);
    const int l0 = div_kk(sig0, a.kk), l1 = div_kk(sig0 + nsl - 1, a.kk);
    const int per = n * a.kk;
    for (int ll = l0; ll <= l1; ++ll) {
      const int lq = ll / a.nl2;
      const long long lr = (long long)(ll - lq * a.nl2) * a.sB;
      const long long lbase = (long long)lq * a.sA + lr;
      const long long lgp = lr / a.kk;
      const int c0 = ll * a.kk - sig0;
#pragma unroll 4
      for (int e = tid; e < per; e += nthr) {
        const int i = div_kk(e, a.kk);
        const int j = e - i * a.kk;
        const int col = c0 + j;
        if (col < 0 || col >= nsl) continue;
        tile_elem<P, LOAD>(a, tile, LD, lbase + e, lgp + i, j, i, col, upd, al, pp, acc);
      }
    }
  }
}

// One tile (ST slots x the whole line) through shared memory: load (with the
// optional fused PCG update / input scaling), forward and backward chunked
// sweeps, store (with the optional output scaling and r.z / r.r partials in
// acc).  All threads of the block call it; factors already in Fs.
template <int P>
__device__ __forceinline__ void tile_solve(const TileLine& a, int tileid, double* smem, const double* Fs, bool upd,
                                           const double* al, const double* pp, double* acc) {
  const int LD = a.ST + 1;
  double* tile = smem;
  double* bsc = tile + (size_t)a.n * LD;
  auto tt = [&](int k) {
    if (a.trace && tileid == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[4000 + (a.epi ? 5 : 0) + k] = (long long)t;
    }
  };
  tt(0);
  tile_io<P, true>(a, tileid, tile, LD, upd, al, pp, acc);
  __syncthreads();
  tt(1);
  tile_sweep<P>(tile, LD, bsc, Fs, a, false);
  tt(2);
  tile_sweep<P>(tile, LD, bsc, Fs + a.flen, a, true);
  tt(3);
  tile_io<P, false>(a, tileid, tile, LD, upd, al, pp, acc);
  __syncthreads();
  tt(4);
}


}  // namespace ga
