// Whole-line sequential Kronecker line solves from shared memory (DESIGN.md §6 "Whole-line
// solver"): the factor Mh_d^{-1} of calM^{-1}.  Used for the boxes of a
// multi-patch problem (additive Schwarz, C5: 514 lines x 2 right-hand sides per patch and
// direction, where a thread-per-line recurrence is latency-bound and the chunked tiles of
// tile_core.cuh pay a scan of ~50 chunk states per sweep), for every 3D single-patch grid outside
// the persistent solver and for 2D grids with lines longer than 768 points.
//
// A CTA of 4 warps stages TS line-slots (a line x one right-hand side) over the WHOLE line length
// in shared memory, together with the two sweeps' factor rows; then ONE warp (warp 0), one lane per
// slot, runs the banded forward and backward substitutions straight through the line - the sweep
// is bound by the instruction stream per warp and by the recurrence, not by lanes, so fewer,
// fuller warps win.  The divisions are folded into the band on the host (host_math.cpp make_seq):
// y_i = t_i d_i - sum_u e_{i,u} y_{i-u}, and the term of y_{i-1} is taken last, so ONE fp64 FMA per
// element is on the recurrence's critical path; data and factor rows of the next batch of elements
// are loaded into registers while the current batch is computed (the loads do not depend on the
// recurrence).  TS is the smallest power of two in 4..32 with all tiles of the launch resident at
// once and at most 4 sweep warps per SM (C5: 387 CTAs of 8 slots, 2-3 per SM - measured, three
// sweep warps interleave on an SM at no cost), else 32 (3D: staging and store of one CTA overlap
// the sweeps of the others).
//
// Staging: y/z lines (slots contiguous at a fixed element) by 16-byte cp.async; x lines (each line
// contiguous) by one bulk copy per line (cp.async.bulk + mbarrier, TMA unit), line-major in shared
// memory with a padded pitch, and bulk stores back.  Unaligned shapes fall back to 8-byte cp.async.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ops.cuh"

namespace ga {

struct SeqLine {
  double* t;         // box array [c][box][kk] (multi-patch) or the z vector (single patch)
  const double* E;   // make_seq rows: forward [n][PP], backward (reversed line) [n][PP]
  int mode;          // 0: slots contiguous at a fixed element (y/z lines); 1: lines contiguous (x lines)
  int n, kk;
  long long es;      // mode 0: element stride
  int nrows, nr2, rowlen;
  long long sA, sB;  // mode 0: row r at (r / nr2) sA + (r % nr2) sB; mode 1: line l likewise (nl2)
  int nlines, nl2;
  int pitch;         // mode 1: shared-memory pitch of a line (doubles)
  int bulk;          // mode 1: lines are 16-byte multiples at 16-byte addresses (bulk copies)
};

struct SeqMulti {
  SeqLine tl[MAXPATCH];
  int tstart[MAXPATCH + 1];
  int np, TS;
  DevStatus* st;
};

__device__ __forceinline__ unsigned int smem_u32(const void* p) { return (unsigned int)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// mbarrier + bulk copy (TMA unit, 1D): global -> shared with transaction-count completion, and
// shared -> global in a bulk group
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned int parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned int bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned int bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One triangular sweep of one slot: element i of the sweep order is tile[sb + (rev ? n-1-i : i) ss].
// Batches of U elements ping-pong between two register sets: the next batch (data + factor rows) is
// loaded before the current one is computed and stored.  Loads are unconditional (the tile has
// 2 U ss doubles of slack on both sides, the factor rows 2 U rows at the end); elements past the
// line end are computed from whatever the slack holds and never stored.
template <int P, int U>
__device__ __forceinline__ void seq_sweep(double* tile, const int sb, const int ss, const int n, const double* E,
                                          const bool rev) {
  constexpr int PP = (P + 2) & ~1;
  double y[P];
#pragma unroll
  for (int u = 0; u < P; ++u) y[u] = 0.0;
  double bA[U], bB[U], eA[U][PP], eB[U][PP];
  const int step = rev ? -ss : ss;
  int off[U];
#pragma unroll
  for (int u = 0; u < U; ++u) off[u] = u * step;
  double* dp = tile + sb + (rev ? (n - 1) * ss : 0);
  const double* ep = E;
  auto load = [&](const double* d, const double* er0, double(&b)[U], double(&e)[U][PP]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      b[u] = d[off[u]];
      const double2* er = reinterpret_cast<const double2*>(er0 + u * PP);
#pragma unroll
      for (int q = 0; q < PP / 2; ++q) {
        const double2 v = er[q];
        e[u][2 * q] = v.x;
        e[u][2 * q + 1] = v.y;
      }
    }
  };
  auto solve = [&](double(&b)[U], double(&e)[U][PP]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double t = b[u] * e[u][0];
#pragma unroll
      for (int v = P; v >= 2; --v) t = fma(-e[u][v], y[v - 1], t);
      t = fma(-e[u][1], y[0], t);  // critical path: y_{i-1} -> y_i
#pragma unroll
      for (int v = P - 1; v >= 1; --v) y[v] = y[v - 1];
      y[0] = t;
      b[u] = t;
    }
  };
  auto store = [&](double* d, int cnt, double(&b)[U]) {
    if (cnt >= U) {
#pragma unroll
      for (int u = 0; u < U; ++u) d[off[u]] = b[u];
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < cnt) d[off[u]] = b[u];
    }
  };
  load(dp, ep, bA, eA);
  for (int i0 = 0; i0 < n; i0 += 2 * U) {
    load(dp + U * step, ep + U * PP, bB, eB);
    solve(bA, eA);
    store(dp, n - i0, bA);
    if (i0 + U >= n) break;
    load(dp + 2 * U * step, ep + 2 * U * PP, bA, eA);
    solve(bB, eB);
    store(dp + U * step, n - i0 - U, bB);
    dp += 2 * U * step;
    ep += 2 * U * PP;
  }
}


#ifdef GA_SEQ_TRACE  // tools/ubench_seq.cu: per-CTA phase clocks
__device__ long long* g_seq_trace;
#define SEQ_T(k)                                                                          \
  do {                                                                                    \
    if (threadIdx.x == 0 && g_seq_trace) g_seq_trace[blockIdx.x * 8 + (k)] = clock64();  \
  } while (0)
#else
#define SEQ_T(k)
#endif

template <int P>
__global__ void __launch_bounds__(128) k_line_seq(SeqMulti mt) {
  int pr = 0;
  while (pr + 1 < mt.np && (int)blockIdx.x >= mt.tstart[pr + 1]) ++pr;
  const SeqLine a = mt.tl[pr];  // by value: no indexed parameter loads inside the sweeps
  if (mt.st->status != 0) return;
  count_launch(mt.st);
  constexpr int PP = (P + 2) & ~1;
  constexpr int U = P <= 4 ? 8 : 4;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int n = a.n, TS = mt.TS, kk = a.kk;
  const int tileid = (int)blockIdx.x - mt.tstart[pr];
  const int SL = 2 * U * max(TS, 4);  // slack (doubles) on both sides of the tile
  double* tile = smem + SL;
  const size_t tdoubles = a.mode == 0 ? (size_t)n * TS : (size_t)max(1, TS / kk) * a.pitch;
  double* Es = tile + ((tdoubles + SL + 1) & ~(size_t)1);
  // ---- tile geometry
  long long base = 0;  // mode 0: first slot of element 0
  int nsl;             // live slots
  int l0 = 0, nl = 0;  // mode 1: first line, lines
  if (a.mode == 0) {
    const int tpr = (a.rowlen + TS - 1) / TS;
    const int r = tileid / tpr;
    const int f0 = (tileid - r * tpr) * TS;
    base = (long long)(r / a.nr2) * a.sA + (long long)(r % a.nr2) * a.sB + f0;
    nsl = min(TS, a.rowlen - f0);
  } else {
    const int LT = max(1, TS / kk);
    l0 = tileid * LT;
    nl = min(LT, a.nlines - l0);
    nsl = nl * kk;
  }
  auto line_base = [&](int l) { return (long long)(l / a.nl2) * a.sA + (long long)(l % a.nl2) * a.sB; };
  const bool bulk = a.mode == 1 && a.bulk;
  const bool v16 = a.mode == 0 && ((base | a.es) & 1) == 0 && (nsl & 1) == 0 && (TS & 1) == 0 &&
                   ((reinterpret_cast<unsigned long long>(a.t) & 15) == 0);
  // ---- stage the factor rows (16-byte cp.async) and the tile
  SEQ_T(0);
  if (tid == 0) {
    if (bulk) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      fence_proxy_async();
    }
  }
  {
    const int nu = n * PP;  // 16-byte units of both tables
    const double2* src = reinterpret_cast<const double2*>(a.E);
    for (int u = tid; u < nu; u += nthr) cp_async16(Es + 2 * u, src + u);
  }
  if (a.mode == 0) {
    if (v16 && nsl == TS && (nthr % (TS >> 1)) == 0) {
      // full tile: thread -> (column pair, first row); rows advance by nthr / h, pointers by adds
      const int h = TS >> 1, rstep = nthr / h;
      const int c = (tid % h) * 2, i0 = tid / h;
      double* dst = tile + (size_t)i0 * TS + c;
      const double* src = a.t + base + c + (long long)i0 * a.es;
      const long long sstep = (long long)rstep * a.es;
      const int dstep = rstep * TS;
      for (int i = i0; i < n; i += rstep, dst += dstep, src += sstep) cp_async16(dst, src);
    } else if (v16) {
      const int h = nsl >> 1, tot = n * h;
      for (int idx = tid; idx < tot; idx += nthr) {
        const int i = idx / h, c = (idx - i * h) * 2;
        cp_async16(tile + (size_t)i * TS + c, a.t + base + c + (long long)i * a.es);
      }
    } else {
      const int tot = n * nsl;
      for (int idx = tid; idx < tot; idx += nthr) {
        const int i = idx / nsl, c = idx - i * nsl;
        cp_async8(tile + (size_t)i * TS + c, a.t + base + c + (long long)i * a.es);
      }
    }
  } else if (bulk) {
    __syncthreads();  // barrier initialised
    if (tid == 0) {
      const unsigned int bytes = (unsigned int)(n * kk * 8);
      mbar_expect_tx(&bar, bytes * nl);
      for (int l = 0; l < nl; ++l) bulk_g2s(tile + (size_t)l * a.pitch, a.t + line_base(l0 + l), bytes, &bar);
    }
  } else {
    const int len = n * kk;
    for (int l = 0; l < nl; ++l) {
      const double* src = a.t + line_base(l0 + l);
      double* dst = tile + (size_t)l * a.pitch;
      for (int e = tid; e < len; e += nthr) cp_async8(dst + e, src + e);
    }
  }
  SEQ_T(1);
  cp_async_wait_all();
  __syncthreads();
  SEQ_T(2);
  // ---- sweeps: one warp (lane = slot); the other warps wait at the barrier
  if (tid < 32) {
    if (bulk) mbar_wait(&bar, 0);
    const int c = tid & 31;
    if (c < nsl) {
      int sb, ss;
      if (a.mode == 0) { sb = c; ss = TS; }
      else { sb = (c / kk) * a.pitch + (c % kk); ss = kk; }
      seq_sweep<P, U>(tile, sb, ss, n, Es, false);
      seq_sweep<P, U>(tile, sb, ss, n, Es + (size_t)n * PP, true);
    }
    if (bulk) fence_proxy_async();  // generic-proxy writes of the sweeps -> visible to the bulk stores
  }
  __syncthreads();
  SEQ_T(3);
  // ---- store
  if (bulk) {
    if (tid == 0) {
      const unsigned int bytes = (unsigned int)(n * kk * 8);
      for (int l = 0; l < nl; ++l) bulk_s2g(a.t + line_base(l0 + l), tile + (size_t)l * a.pitch, bytes);
      bulk_commit_wait();
    }
    SEQ_T(4);
    return;
  }
  if (a.mode == 0) {
    if (v16 && nsl == TS && (nthr % (TS >> 1)) == 0) {
      const int h = TS >> 1, rstep = nthr / h;
      const int c = (tid % h) * 2, i0 = tid / h;
      const double* src = tile + (size_t)i0 * TS + c;
      double* dst = a.t + base + c + (long long)i0 * a.es;
      const long long dstep = (long long)rstep * a.es;
      const int sstep = rstep * TS;
      for (int i = i0; i < n; i += rstep, dst += dstep, src += sstep)
        *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(src);
    } else if (v16) {
      const int h = nsl >> 1, tot = n * h;
      for (int idx = tid; idx < tot; idx += nthr) {
        const int i = idx / h, c = (idx - i * h) * 2;
        *reinterpret_cast<double2*>(a.t + base + c + (long long)i * a.es) =
            *reinterpret_cast<const double2*>(tile + (size_t)i * TS + c);
      }
    } else {
      const int tot = n * nsl;
      for (int idx = tid; idx < tot; idx += nthr) {
        const int i = idx / nsl, c = idx - i * nsl;
        a.t[base + c + (long long)i * a.es] = tile[(size_t)i * TS + c];
      }
    }
  } else {
    const int len = n * kk;
    for (int l = 0; l < nl; ++l) {
      double* dst = a.t + line_base(l0 + l);
      const double* src = tile + (size_t)l * a.pitch;
      for (int e = tid; e < len; e += nthr) dst[e] = src[e];
    }
  }
  SEQ_T(4);
}

// shared-memory pitch of a contiguous line of len doubles: 16-byte aligned when the bulk path is
// possible, and lines of one warp on distinct banks (pitch = kk' mod 16 doubles, kk' = kk rounded
// up to even: line l starts 4 l banks on for kk = 2)
static int seq_pitch(int len, int kk, bool aligned) {
  if (!aligned) return len | 1;
  const int want = (kk + 1) & ~1;
  int p = len;
  while ((p & 15) != (want & 15)) ++p;
  return p;
}

// once per degree (ga_create calls it outside any stream capture): the kernel may use all of the
// shared memory of an SM
template <int P>
static size_t seq_prepare() {  // returns the dynamic shared memory the kernel may use (0: failed)
  static int state = 0;  // 0 not tried, 1 ok, -1 failed
  static size_t dyn_max = 0;
  if (state == 0) {
    cudaFuncAttributes fa;
    state = -1;
    if (cudaFuncGetAttributes(&fa, k_line_seq<P>) == cudaSuccess) {
      dyn_max = (size_t)227 * 1024 - fa.sharedSizeBytes;  // static: mbarrier + reduction scratch
      if (cudaFuncSetAttribute(k_line_seq<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max) == cudaSuccess)
        state = 1;
    }
    if (state < 0) { cudaGetLastError(); dyn_max = 0; }
  }
  return state > 0 ? dyn_max : 0;
}
bool line_seq_prepare(int p) {
  switch (p) {
    case 1: return seq_prepare<1>() > 0;
    case 2: return seq_prepare<2>() > 0;
    case 3: return seq_prepare<3>() > 0;
    case 4: return seq_prepare<4>() > 0;
    case 5: return seq_prepare<5>() > 0;
    case 6: return seq_prepare<6>() > 0;
    default: return seq_prepare<7>() > 0;
  }
}

template <int P>
static bool seq_launch(SeqMulti m, cudaStream_t s, bool dry) {
  constexpr int PP = (P + 2) & ~1;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  auto tiles = [&](const SeqLine& t, int TS) -> long long {
    if (t.mode == 0) return (long long)t.nrows * ((t.rowlen + TS - 1) / TS);
    const int LT = std::max(1, TS / t.kk);
    return (t.nlines + LT - 1) / LT;
  };
  constexpr int U = P <= 4 ? 8 : 4;  // as in the kernel
  auto smem_for = [&](int TS) -> size_t {
    size_t mx = 0;
    const size_t SL = (size_t)2 * U * std::max(TS, 4);
    for (int r = 0; r < m.np; ++r) {
      const SeqLine& t = m.tl[r];
      const size_t td = t.mode == 0 ? (size_t)t.n * TS : (size_t)std::max(1, TS / t.kk) * t.pitch;
      mx = std::max(mx, sizeof(double) * (SL + ((td + SL + 1) & ~(size_t)1) + (size_t)2 * t.n * PP + (size_t)2 * U * PP));
    }
    return mx;
  };
  // the smallest tile whose CTAs are all resident at once (one wave over every SM); else the
  // largest that fits in shared memory
  const size_t dyn_max = seq_prepare<P>();
  if (!dyn_max) return false;
  int TS = 0;
  const int minTS = 4;
  for (int cand = minTS; cand <= 32; cand <<= 1) {
    const size_t sm = smem_for(cand);
    if (sm > dyn_max) break;
    long long ct = 0;
    for (int r = 0; r < m.np; ++r) ct += tiles(m.tl[r], cand);
    const long long per_sm = std::min<long long>(16, (long long)(227 * 1024) / (long long)(sm + 1024 + (227 * 1024 - dyn_max)));
    TS = cand;
    if (ct <= std::min<long long>(per_sm, 4) * nsm) break;  // <= 4 sweep warps per SM (measured: 3 are free)
  }
  if (!TS) return false;
  for (int r = 0; r < m.np; ++r)
    if (m.tl[r].mode == 1 && m.tl[r].kk > TS) return false;
  m.TS = TS;
  int t0 = 0;
  for (int r = 0; r < m.np; ++r) {
    m.tstart[r] = t0;
    t0 += (int)tiles(m.tl[r], TS);
  }
  m.tstart[m.np] = t0;
  const size_t sm = smem_for(TS);
  if (dry) return true;
  k_line_seq<P><<<(unsigned int)t0, 128, sm, s>>>(m);
  return true;
}

// Direction d of the Kronecker solve on the boxes of every patch, one launch (the batched additive
// Schwarz path of launch_precond).  False: not applicable (no factor rows, or a line set does not
// fit in shared memory) - the caller uses the chunked tiles.
// GA_LINE_SEQ=0: the chunked tiles instead (A/B measurements)
int line_seq_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("GA_LINE_SEQ");
    mode = (e && *e == '0') ? 0 : 1;
  }
  return mode;
}

// Single patch (a.t[0] == nullptr): the lines of the z vector itself (the box is the whole grid).
// dry: only report whether the launch is possible.
bool launch_line_seq_multi(const PrecArgs& a, int d, cudaStream_t s, bool dry) {
  if (!line_seq_mode()) return false;
  const GridDesc& g = a.g;
  const bool single = a.npatch == 1 && a.t[0] == nullptr;
  SeqMulti m;
  memset(&m, 0, sizeof(m));
  m.np = a.npatch;
  m.st = a.st;
  for (int pr = 0; pr < a.npatch; ++pr) {
    if (!a.E[pr][d] || (!a.t[pr] && !single)) return false;
    const int bd[3] = {a.bd[pr][0], a.bd[pr][1], a.bd[pr][2]};
    const long long nbox = (long long)bd[0] * bd[1] * bd[2];
    long long str[3] = {a.kk, (long long)bd[0] * a.kk, (long long)bd[0] * bd[1] * a.kk};
    long long sc = nbox * a.kk;
    SeqLine& tl = m.tl[pr];
    tl.t = a.t[pr]; tl.E = a.E[pr][d]; tl.n = bd[d]; tl.kk = a.kk;
    if (single) {
      tl.t = a.z + g.guard * a.kk;
      str[1] = (long long)g.nx * a.kk; str[2] = (long long)g.nx * g.ny * a.kk;
      sc = g.padded * a.kk;
    }
    if (d == 0) {
      tl.mode = 1; tl.nlines = a.nvec * bd[1] * bd[2]; tl.nl2 = bd[1] * bd[2]; tl.sA = sc; tl.sB = str[1];
      const bool al = ((bd[0] * a.kk) & 1) == 0 && (sc & 1) == 0 &&
                      (reinterpret_cast<unsigned long long>(tl.t) & 15) == 0;
      tl.bulk = al ? 1 : 0;
      tl.pitch = seq_pitch(bd[0] * a.kk, a.kk, al);
    } else {
      tl.mode = 0; tl.es = str[d]; tl.rowlen = bd[0] * a.kk;
      const int other = (d == 1) ? 2 : 1;
      const int nother = (g.dim == 3) ? bd[other] : 1;
      tl.nrows = a.nvec * nother; tl.nr2 = nother; tl.sA = sc; tl.sB = (g.dim == 3) ? str[other] : 0;
    }
  }
  switch (a.p) {
    case 1: return seq_launch<1>(m, s, dry);
    case 2: return seq_launch<2>(m, s, dry);
    case 3: return seq_launch<3>(m, s, dry);
    case 4: return seq_launch<4>(m, s, dry);
    case 5: return seq_launch<5>(m, s, dry);
    case 6: return seq_launch<6>(m, s, dry);
    default: return seq_launch<7>(m, s, dry);
  }
}

}  // namespace ga
