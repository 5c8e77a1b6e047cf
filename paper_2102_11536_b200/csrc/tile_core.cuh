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
  int xdefer;          // pro + update: skip x += alpha p (done by the next SpMV, persistent solver)
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

// Phase B of the chunked sweep: sigma_{w+1} = T_w sigma_w + tau_w over the
// chunks w = 0..C-2 of every slot, Kogge-Stone in L levels through bsc
// ([C][P][ST]); on return bsc[w] holds sigma_{w+1}.  ch is this thread's chunk
// (>= C-1: no chunk state to contribute).  All threads of the block call it.
template <int P>
__device__ __forceinline__ void chunk_scan(double (&b)[P], double* __restrict__ bsc, const double* __restrict__ A,
                                           int C, int L, int ST, int sl, int ch) {
  const int E = C - 1;
  for (int l = 0; l < L; ++l) {
    const int d = 1 << l;
    if (ch < E) {
#pragma unroll
      for (int u = 0; u < P; ++u) bsc[(ch * P + u) * ST + sl] = b[u];
    }
    __syncthreads();
    if (ch < E && ch >= d) {
      const double* Aw = A + ((size_t)l * C + ch) * P * P;
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
  // chunk bounds: forward from index 0 (short remainder last); backward = the
  // mirror partition on the reversed line (short chunk first), host_math.cpp
  const int rem = n - (a.C - 1) * a.clen;
  const int lo = !rev ? ch * a.clen : (ch == 0 ? 0 : rem + (ch - 1) * a.clen);
  const int hi = !rev ? min(n, lo + a.clen) : (ch == 0 ? rem : min(n, lo + a.clen));
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
  double b[P];
#pragma unroll
  for (int u = 0; u < P; ++u) b[u] = y[u];  // tau_w[u] = y_{hi-1-u}
  chunk_scan<P>(b, bsc, A, a.C, a.L, ST, sl, ch);
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
// Tile load/store.  Each thread handles the elements idx = tid + u*nthr in
// batches of TB: the addresses of a batch are computed first, then all its
// global loads are issued before any is consumed (one memory round trip per
// batch instead of one per element).
template <int P, bool LOAD>
__device__ __forceinline__ void tile_io(const TileLine& a, int tileid, double* tile, int LD, bool upd, const double* al,
                                        const double* pp, double* acc) {
  constexpr int TB = 4;
  const int n = a.n, ST = a.ST, nthr = blockDim.x, tid = threadIdx.x;
  const int lgST = 31 - __clz(ST);  // ST is a power of two (1..32)
  // tile geometry
  long long base = 0, gp0 = 0, ges = 0;
  int f0 = 0, nsl, sig0 = 0, l0 = 0, per = 1, tot;
  if (a.mode == 0) {
    const int tpr = (a.rowlen + ST - 1) / ST;
    const int r = tileid / tpr;
    f0 = (tileid - r * tpr) * ST;
    const long long roff = (long long)(r % a.nr2) * a.sB;
    base = (long long)(r / a.nr2) * a.sA + roff + f0;
    gp0 = roff / a.kk;
    ges = a.es / a.kk;
    nsl = min(ST, a.rowlen - f0);
    tot = n << lgST;
  } else {
    sig0 = tileid * ST;
    nsl = min(ST, a.nlines * a.kk - sig0);
    l0 = div_kk(sig0, a.kk);
    const int l1 = div_kk(sig0 + nsl - 1, a.kk);
    per = n * a.kk;
    tot = (l1 - l0 + 1) * per;
  }
  for (int b0 = tid; b0 < tot; b0 += TB * nthr) {
    long long g[TB], gp[TB];
    int jj[TB], ii[TB], col[TB];
    bool ok[TB];
#pragma unroll
    for (int u = 0; u < TB; ++u) {
      const int idx = b0 + u * nthr;
      ok[u] = idx < tot;
      if (a.mode == 0) {
        const int i = idx >> lgST, c = idx & (ST - 1);
        ok[u] = ok[u] && c < nsl;
        const int f = f0 + c;
        const int xo = div_kk(f, a.kk);
        jj[u] = f - xo * a.kk;
        ii[u] = i;
        col[u] = c;
        g[u] = base + c + (long long)i * a.es;
        gp[u] = gp0 + xo + (long long)i * ges;
      } else {
        const int lrel = idx / per;
        const int e = idx - lrel * per;
        const int ll = l0 + lrel;
        const int i = div_kk(e, a.kk);
        const int j = e - i * a.kk;
        const int c = ll * a.kk + j - sig0;
        ok[u] = ok[u] && c >= 0 && c < nsl;
        const int lq = ll / a.nl2;
        const long long lr = (long long)(ll - lq * a.nl2) * a.sB;
        jj[u] = j;
        ii[u] = i;
        col[u] = c;
        g[u] = (long long)lq * a.sA + lr + e;
        gp[u] = lr / a.kk + i;
      }
    }
    if (LOAD) {
      double v[TB], sv[TB], xv[TB], pv[TB], qv[TB];
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const long long gg = ok[u] ? g[u] : 0, gpp = ok[u] ? gp[u] : 0;
        if (a.pro) {
          v[u] = a.r[gg];
          sv[u] = a.s[gpp];
          if (upd) {
            qv[u] = a.q[gg];
            if (!a.xdefer) { xv[u] = a.x[gg]; pv[u] = pp[gg]; }
          }
        } else {
          v[u] = a.t[gg];
        }
      }
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        if (!ok[u]) continue;
        double w = v[u];
        if (a.pro) {
          if (upd) {
            double alj = al[0];
#pragma unroll
            for (int q = 1; q < KMAX; ++q) alj = (jj[u] == q) ? al[q] : alj;
            if (alj != 0.0) {
              if (!a.xdefer) a.x[g[u]] = fma(alj, pv[u], xv[u]);
              w = fma(-alj, qv[u], w);
              a.r[g[u]] = w;
            }
          }
          w *= sv[u];
        }
        tile[ii[u] * LD + col[u]] = w;
      }
    } else {
      double sv[TB], rv[TB];
      if (a.epi) {
#pragma unroll
        for (int u = 0; u < TB; ++u) {
          const long long gg = ok[u] ? g[u] : 0, gpp = ok[u] ? gp[u] : 0;
          sv[u] = a.s[gpp];
          rv[u] = a.r[gg];
        }
      }
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        if (!ok[u]) continue;
        double w = tile[ii[u] * LD + col[u]];
        if (a.epi) {
          w *= sv[u];
#pragma unroll
          for (int q = 0; q < KMAX; ++q)
            {  // branch-free (a data-dependent branch here turns acc into local memory)
              const double m = (q == jj[u]) ? rv[u] : 0.0;
              acc[q] = fma(m, w, acc[q]);
              acc[KMAX + q] = fma(m, rv[u], acc[KMAX + q]);
            }
        }
        a.t[g[u]] = w;
      }
    }
  }
}

// Register-resident variant of tile_solve (chunk length <= CL): each thread
// loads the elements of its chunk straight from global memory into the CL
// register slots v[0..CL) (element lo+q in slot q; slots q >= cnt are dead)
// and runs phases A and C of both sweeps there; only the P-wide chunk states
// go through shared memory (chunk_scan).  A thread that owns forward chunk w
// owns backward chunk C-1-w, the same elements (mirror partition,
// host_math.cpp make_sweep).  Every register index is a compile-time constant
// (the recurrence reads v[q-u] / v[q+u] directly, no shifted state array), so
// v stays in registers; the sweeps are branch-free and read the factors at
// fixed offsets from per-thread base pointers.  Dead slots compute finite
// garbage in the forward sweep (after the live ones), are zeroed before the
// backward sweep (which meets them first) and are never stored.  Factor
// reads of dead slots may run up to CL elements past either end of a factor
// buffer: they stay inside the adjacent [Ff | Fb] pair (finite values), which
// every caller lays out contiguously.  Same arithmetic, in the same order, as
// tile_sweep (the skipped terms multiply the zero incoming state).
template <int P, int CL>
__device__ __forceinline__ void tile_solve_reg(const TileLine& a, int tileid, double* smem, const double* Ff,
                                               const double* Fb, bool upd, const double* al, const double* pp,
                                               double* acc, unsigned long long* tprev) {
  const int n = a.n, ST = a.ST, cpw = 32 / ST, C = a.C;
  const int lane = threadIdx.x & 31;
  const int sl = lane & (ST - 1);
  const int ch = (threadIdx.x >> 5) * cpw + lane / ST;
  double* bsc = smem;
  // this thread's slot: element i at t[gb + i*gst], grid point gpb + i*gpst
  long long gb, gpb;
  int gst, gpst, j;
  bool valid;
  if (a.mode == 0) {
    const int tpr = (a.rowlen + ST - 1) / ST;
    const int r = tileid / tpr;
    const int f = (tileid - r * tpr) * ST + sl;
    valid = f < a.rowlen;
    const long long roff = (long long)(r % a.nr2) * a.sB;
    gb = (long long)(r / a.nr2) * a.sA + roff + f;
    const int xo = div_kk(f, a.kk);
    j = f - xo * a.kk;
    gpb = roff / a.kk + xo;
    gst = (int)a.es;
    gpst = (int)(a.es / a.kk);
  } else {
    const int sig = tileid * ST + sl;
    valid = sig < a.nlines * a.kk;
    const int ll = div_kk(sig, a.kk);
    j = sig - ll * a.kk;
    const int lq = ll / a.nl2;
    const long long lr = (long long)(ll - lq * a.nl2) * a.sB;
    gb = (long long)lq * a.sA + lr + j;
    gpb = lr / a.kk;
    gst = a.kk;
    gpst = 1;
  }
  const bool live = valid && ch < C;
  const int lo = live ? ch * a.clen : 0;
  const int cnt = live ? min(n, lo + a.clen) - lo : 0;
  double* __restrict__ tp = a.t + gb + (long long)lo * gst;
  double* __restrict__ rp = a.r + gb + (long long)lo * gst;
  const double* __restrict__ sp = a.s + gpb + (long long)lo * gpst;
  double alj = 0.0;
  if (upd) {
    alj = al[0];
#pragma unroll
    for (int q = 1; q < KMAX; ++q) alj = (j == q) ? al[q] : alj;
  }
  auto tt = [&](int k) {
    if (a.trace && threadIdx.x == 0) {
      unsigned long long t;
      t = (unsigned long long)clock64();  // SM cycles
      long long* slot = a.trace + 4096 + blockIdx.x * 12 + (a.epi ? 6 : 0);
      if (k > 0) slot[k - 1] += (long long)(t - *tprev);
      else slot[5] += 1;
      *tprev = t;
    }
  };
  tt(0);
  double v[CL];
  // ---- load (+ fused PCG update x += alpha p, r -= alpha q, input scaling)
  if (a.pro) {
    const bool ur = upd && alj != 0.0;
    const bool ux = ur && !a.xdefer;
    double* __restrict__ xp = a.x + gb + (long long)lo * gst;
    const double* __restrict__ qp = a.q + gb + (long long)lo * gst;
    const double* __restrict__ ppp = pp + gb + (long long)lo * gst;
    // every load of the chunk first (one memory round trip), then the stores
    double sv[CL], qv[CL];
#pragma unroll
    for (int q = 0; q < CL; ++q) {
      const bool ok = q < cnt;
      v[q] = ok ? rp[q * gst] : 0.0;
      sv[q] = ok ? sp[q * gpst] : 0.0;
      qv[q] = (ok && ur) ? qp[q * gst] : 0.0;
    }
    if (ux) {
#pragma unroll
      for (int q0 = 0; q0 < CL; q0 += 4) {
        double xv[4], pv[4];
#pragma unroll
        for (int u = 0; u < 4 && q0 + u < CL; ++u) {
          const bool ok = q0 + u < cnt;
          xv[u] = ok ? xp[(q0 + u) * gst] : 0.0;
          pv[u] = ok ? ppp[(q0 + u) * gst] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4 && q0 + u < CL; ++u)
          if (q0 + u < cnt) xp[(q0 + u) * gst] = fma(alj, pv[u], xv[u]);
      }
    }
#pragma unroll
    for (int q = 0; q < CL; ++q) {
      if (ur) {
        v[q] = fma(-alj, qv[q], v[q]);
        if (q < cnt) rp[q * gst] = v[q];
      }
      v[q] *= sv[q];
    }
  } else {
#pragma unroll
    for (int q = 0; q < CL; ++q) v[q] = q < cnt ? tp[q * gst] : 0.0;
  }
  tt(1);
  // ---- forward sweep L y = b: element lo+q in slot q
  {
    const double* fd = Ff + lo;                                    // dinv[lo+q]      = fd[q]
    const double* fc = Ff + n + (size_t)lo * P;                    // coef[lo+q][u-1] = fc[q*P+u-1]
    const double* fh = Ff + (size_t)n * (1 + P) + (size_t)lo * P;  // H[lo+q][u]      = fh[q*P+u]
    const double* A = Ff + (size_t)n * (1 + 2 * P);
#pragma unroll
    for (int q = 0; q < CL; ++q) {
      double w = v[q];
#pragma unroll
      for (int u = P; u >= 1; --u)
        if (q - u >= 0) w = fma(-fc[q * P + u - 1], v[q - u], w);
      v[q] = w * fd[q];
    }
    // outgoing state tau[u] = y_{hi-1-u} (zero before the chunk start)
    double y[P];
#pragma unroll
    for (int u = 0; u < P; ++u) y[u] = 0.0;
#pragma unroll
    for (int q = 0; q < CL; ++q)
#pragma unroll
      for (int u = 0; u < P; ++u) y[u] = (q == cnt - 1 - u) ? v[q] : y[u];
    chunk_scan<P>(y, bsc, A, C, a.L, ST, sl, ch);
    if (ch >= 1 && ch < C) {
      double sg[P];
#pragma unroll
      for (int u = 0; u < P; ++u) sg[u] = bsc[((ch - 1) * P + u) * ST + sl];
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        double w = v[q];
#pragma unroll
        for (int u = 0; u < P; ++u) w = fma(fh[q * P + u], sg[u], w);
        v[q] = w;
      }
    }
#pragma unroll
    for (int q = 0; q < CL; ++q) v[q] = q < cnt ? v[q] : 0.0;  // dead slots: zero for the backward sweep
    __syncthreads();  // bsc is reused by the backward scan
  }
  tt(2);
  // ---- backward sweep L^T z = y: forward sweep of the reversed line, i' = n-1-(lo+q), chunk C-1-ch
  {
    const int ib = n - 1 - lo;
    const double* fd = Fb + ib;                                    // dinv'[i']      = fd[-q]
    const double* fc = Fb + n + (ptrdiff_t)ib * P;                 // coef'[i'][u-1] = fc[-q*P+u-1]
    const double* fh = Fb + (size_t)n * (1 + P) + (ptrdiff_t)ib * P;  // H'[i'][u]   = fh[-q*P+u]
    const double* A = Fb + (size_t)n * (1 + 2 * P);
    const int w = ch < C ? C - 1 - ch : C;
#pragma unroll
    for (int q = CL - 1; q >= 0; --q) {
      double x = v[q];
#pragma unroll
      for (int u = P; u >= 1; --u)
        if (q + u <= CL - 1) x = fma(-fc[-q * P + u - 1], v[q + u], x);
      v[q] = x * fd[-q];
    }
    // outgoing state: the last P live elements in reversed order are slots 0..P-1
    double y[P];
#pragma unroll
    for (int u = 0; u < P; ++u) y[u] = (u < cnt) ? v[u] : 0.0;
    chunk_scan<P>(y, bsc, A, C, a.L, ST, sl, w);
    if (w >= 1 && w < C) {
      double sg[P];
#pragma unroll
      for (int u = 0; u < P; ++u) sg[u] = bsc[((w - 1) * P + u) * ST + sl];
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        double x = v[q];
#pragma unroll
        for (int u = 0; u < P; ++u) x = fma(fh[-q * P + u], sg[u], x);
        v[q] = x;
      }
    }
    __syncthreads();  // bsc is free for the next tile
  }
  tt(3);
  // ---- store (+ output scaling and the r.z / r.r partials); loads first
  if (a.epi) {
    double rz = 0.0, rr = 0.0;
    double rv[CL], sv[CL];
#pragma unroll
    for (int q = 0; q < CL; ++q) {
      const bool ok = q < cnt;
      rv[q] = ok ? rp[q * gst] : 0.0;
      sv[q] = ok ? sp[q * gpst] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < CL; ++q) {
      if (q < cnt) {
        const double z = v[q] * sv[q];
        rz = fma(rv[q], z, rz);
        rr = fma(rv[q], rv[q], rr);
        tp[q * gst] = z;
      }
    }
#pragma unroll
    for (int q = 0; q < KMAX; ++q) {  // branch-free select (keeps acc in registers)
      acc[q] += (q == j) ? rz : 0.0;
      acc[KMAX + q] += (q == j) ? rr : 0.0;
    }
  } else {
#pragma unroll
    for (int q = 0; q < CL; ++q)
      if (q < cnt) tp[q * gst] = v[q];
  }
  tt(4);
}

// One tile (ST slots x the whole line) through shared memory: load (with the
// optional fused PCG update / input scaling), forward and backward chunked
// sweeps, store (with the optional output scaling and r.z / r.r partials in
// acc).  All threads of the block call it; factors already in Fs.
template <int P, int CLMAX = 12>
__device__ __forceinline__ void tile_solve(const TileLine& a, int tileid, double* smem, const double* Fs, bool upd,
                                           const double* al, const double* pp, double* acc) {
  // GA_TRACE: per-block accumulated phase durations (SM cycles) at trace[4096 + block*12 + (epi ? 6 : 0) + k]
  unsigned long long tprev = 0;
  if (a.clen <= 4) { tile_solve_reg<P, 4>(a, tileid, smem, Fs, Fs + a.flen, upd, al, pp, acc, &tprev); return; }
  if (a.clen <= 8) { tile_solve_reg<P, 8>(a, tileid, smem, Fs, Fs + a.flen, upd, al, pp, acc, &tprev); return; }
  if constexpr (CLMAX >= 12) {
    if (a.clen <= 12) { tile_solve_reg<P, 12>(a, tileid, smem, Fs, Fs + a.flen, upd, al, pp, acc, &tprev); return; }
  }
  const int LD = a.ST + 1;
  double* tile = smem;
  double* bsc = tile + (size_t)a.n * LD;
  auto tt = [&](int k) {
    if (a.trace && threadIdx.x == 0) {
      unsigned long long t;
      t = (unsigned long long)clock64();  // SM cycles
      long long* slot = a.trace + 4096 + blockIdx.x * 12 + (a.epi ? 6 : 0);
      if (k > 0) slot[k - 1] += (long long)(t - tprev);
      else slot[5] += 1;
      tprev = t;
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
