// Persistent cooperative PCG solve for small single-patch scalar problems (core).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "ops.cuh"
#include "spmv_core.cuh"
#include "tile_core.cuh"

// ===========================================================================
// Persistent cooperative PCG solve
// ===========================================================================

namespace ga {

namespace cg = cooperative_groups;

constexpr int PBLK = 256;  // threads per block of the persistent kernel

struct PersistDev {
  GridDesc g;
  int nvec, kk, dim, refine, maxit;
  double tol2, refine_rtol2;
  SpmvArgs spq, str;
  TileLine tl[3];
  int ntiles[3];
  int fofs[3];          // offsets of the direction factors in shared memory
  int scratch_ofs;
  double* gpart;        // [2][gridDim][2*KMAX]
  double *b, *x, *r, *z, *p, *p1;   // p, p1: the two direction buffers (fused update)
  PcgState* pcg;
  DevStatus* st;
  long long* trace;     // optional phase timestamps (GA_TRACE): [iter][5] globaltimer ns
};

// GA_TRACE: per-block accumulated durations (SM cycles) at trace[6000 + block*4 + k]
__device__ __forceinline__ void btrace(const PersistDev& A, int k, unsigned long long& tprev) {
  if (A.trace && threadIdx.x == 0) {
    unsigned long long t;
    t = (unsigned long long)clock64();  // SM cycles
    if (k >= 0) A.trace[6000 + blockIdx.x * 4 + k] += (long long)(t - tprev);
    tprev = t;
  }
}

__device__ __forceinline__ void ptrace(const PersistDev& A, long long slot) {
  if (A.trace && blockIdx.x == 0 && threadIdx.x == 0 && slot < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.trace[slot] = (long long)t;
  }
}

// grid-wide sum of NV values (every thread of every block gets the totals);
// double-buffered partials so one grid barrier per reduction suffices
template <int NV>
__device__ __forceinline__ void gsum(double (&v)[NV], double* gpart, int& buf, cg::grid_group& grid) {
  __shared__ double tot_sh[NV > 0 ? NV : 1];
  block_sum<NV>(v);
  double* part = gpart + (size_t)buf * gridDim.x * 2 * KMAX;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) part[(size_t)blockIdx.x * NV + j] = v[j];
  }
  grid.sync();
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] += part[(size_t)b * NV + j];
  block_sum<NV>(acc);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) tot_sh[j] = acc[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = tot_sh[j];
  __syncthreads();
  buf ^= 1;
}

template <int P, int KK>
__device__ __forceinline__ void persist_precond(const PersistDev& A, double* smem, bool upd, const double* al,
                                                const double* pnew_off, double (&rz)[KK], double (&rr)[KK], int& gbuf,
                                                cg::grid_group& grid, long long tslot = -1) {
  double acc[2 * KMAX];
#pragma unroll
  for (int j = 0; j < 2 * KMAX; ++j) acc[j] = 0.0;
  for (int d = 0; d < A.dim; ++d) {
    const TileLine& tl = A.tl[d];
    for (int t = blockIdx.x; t < A.ntiles[d]; t += gridDim.x)
      tile_solve<P, 8>(tl, t, smem + A.scratch_ofs, smem + A.fofs[d], upd && d == 0, al, pnew_off, acc);
    if (d < A.dim - 1) grid.sync();
    if (d == 0 && tslot >= 0) ptrace(A, tslot);
  }
  double v[2 * KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) { v[j] = acc[j]; v[KK + j] = acc[KMAX + j]; }
  gsum<2 * KK>(v, A.gpart, gbuf, grid);
#pragma unroll
  for (int j = 0; j < KK; ++j) { rz[j] = v[j]; rr[j] = v[KK + j]; }
}

template <int P, int KK>
__global__ void __launch_bounds__(PBLK) k_pcg_persist(PersistDev A) {
  cg::grid_group grid = cg::this_grid();
  if (A.st->status != 0) return;  // uniform: read before any barrier
  count_launch(A.st);
  extern __shared__ double smem[];
  // sweep factors of every direction stay resident in shared memory
  for (int d = 0; d < A.dim; ++d) {
    const TileLine& tl = A.tl[d];
    for (int idx = threadIdx.x; idx < 2 * tl.flen; idx += blockDim.x)
      smem[A.fofs[d] + idx] = idx < tl.flen ? tl.Ff[idx] : tl.Fb[idx - tl.flen];
  }
  __syncthreads();
  const GridDesc g = A.g;
  const long long nel = (long long)A.nvec * g.npts;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  int gbuf = 0;
  // ---- r = b, x = 0, ||b||^2
  double bb[KK];
  {
    double v[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) v[j] = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nel; e += gstride) {
      const long long i = e % g.npts;
      const int c = (int)(e / g.npts);
      const long long base = ((long long)c * g.padded + g.guard + i) * KK;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        const double b = A.b[base + j];
        A.r[base + j] = b;
        A.x[base + j] = 0.0;
        v[j] = fma(b, b, v[j]);
      }
    }
    gsum<KK>(v, A.gpart, gbuf, grid);
#pragma unroll
    for (int j = 0; j < KK; ++j) bb[j] = v[j];
  }
  double thr[KK], rz[KK], rr[KK], rzold[KK], alpha[KMAX], beta[KK];
  int active[KK], its[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) { its[j] = 0; alpha[j] = 0.0; beta[j] = 0.0; rzold[j] = 0.0; }
#pragma unroll
  for (int j = KK; j < KMAX; ++j) alpha[j] = 0.0;
  long long loops = 0;
  int status = 0, fail_block = -1;
  // the two direction buffers, selected without an indexed array (keeps them out of local memory)
  auto pbuf = [&](int w) { return w ? A.p1 : A.p; };
  int par = 0;
  for (int phase = 0; phase < (A.refine ? 2 : 1); ++phase) {
    if (phase == 0) {
#pragma unroll
      for (int j = 0; j < KK; ++j) { thr[j] = A.tol2 * bb[j]; active[j] = bb[j] > 0.0; }
    } else {
      // refinement restart from the true residual r = b - M x (R8)
      double v[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) v[j] = 0.0;
      const long long nrg = ((g.npts + 31) / 32 + 7) / 8;
      for (long long rb = blockIdx.x; rb < nrg; rb += gridDim.x) spmv_block<P, 1, KK, false, 8>(A.str, rb, smem + A.scratch_ofs, v);
      gsum<KK>(v, A.gpart, gbuf, grid);
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        active[j] = bb[j] > 0.0;
        double t = A.tol2 * bb[j];
        if (A.refine_rtol2 > 0.0) t = fmin(t, A.refine_rtol2 * v[j]);
        thr[j] = t;
      }
    }
    bool first = true, pfirst = true;
    int iter = 0;
    persist_precond<P, KK>(A, smem, false, alpha, pbuf(par) + g.guard * KK, rz, rr, gbuf, grid);
    for (;;) {
      // F1: convergence, beta
      int any = 0;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        if (active[j] && rr[j] <= thr[j]) active[j] = 0;
        beta[j] = first ? 0.0 : (rzold[j] != 0.0 ? rz[j] / rzold[j] : 0.0);
        rzold[j] = rz[j];
        any |= active[j];
      }
      if (first) pfirst = true;
      first = false;
      if (!any) break;
      if (iter >= A.maxit) {
        if (phase == 0) {
          status = -5;
#pragma unroll
          for (int j = KK - 1; j >= 0; --j)
            if (active[j]) fail_block = j;
        }
        break;
      }
      ptrace(A, loops * 5 + 0);
      ptrace(A, loops * 5 + 1);
      // q = M p with p = z + beta p_old formed on the SpMV input window (fused
      // direction update, double-buffered p), p.q
      SpmvArgs sq = A.spq;
      sq.fuse_p = 1;
      sq.z = A.z;
      sq.p0 = pbuf(par);
      sq.p1 = pbuf(par ^ 1);
      sq.fpfirst = pfirst ? 1 : 0;
      sq.fx = A.x;  // x += alpha_prev p_old on the own rows (deferred from the last preconditioner)
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        sq.fbeta[j] = j < KK ? (active[j] ? beta[j] : 0.0) : 0.0;
        sq.falpha[j] = j < KK ? alpha[j] : 0.0;
      }
      double pq[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) pq[j] = 0.0;
      const long long nrg = ((g.npts + 31) / 32 + 7) / 8;
      unsigned long long tb = 0;
      btrace(A, -1, tb);
      for (long long rb = blockIdx.x; rb < nrg; rb += gridDim.x) spmv_block<P, 1, KK, false, 8>(sq, rb, smem + A.scratch_ofs, pq);
      btrace(A, 0, tb);
      __syncthreads();
      btrace(A, 1, tb);
      par ^= 1;
      gsum<KK>(pq, A.gpart, gbuf, grid);
      btrace(A, 2, tb);
      if (A.trace && threadIdx.x == 0) A.trace[6000 + blockIdx.x * 4 + 3] += 1950;  // count (x 1950: the script divides by cycles/us)
      ptrace(A, loops * 5 + 2);
      ++iter;
      ++loops;
      pfirst = false;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        alpha[j] = active[j] ? rz[j] / pq[j] : 0.0;
        if (active[j]) its[j] += 1;
      }
      // x += alpha p, r -= alpha q, z = calM^{-1} r, r.z, r.r
      persist_precond<P, KK>(A, smem, true, alpha, pbuf(par) + g.guard * KK, rz, rr, gbuf, grid, (loops - 1) * 5 + 3);
      ptrace(A, (loops - 1) * 5 + 4);
    }
    if (iter > 0) {
      // the last iteration's deferred x += alpha p (p = pbuf(par), the newest direction)
      const double* pc = pbuf(par);
      for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < g.npts * KK; e += gstride) {
        const long long idx = g.guard * KK + e;
        const int jj = (int)(e % KK);
        double al = alpha[0];
#pragma unroll
        for (int q = 1; q < KK; ++q) al = (jj == q) ? alpha[q] : al;
        if (al != 0.0) A.x[idx] = fma(al, pc[idx], A.x[idx]);
      }
      if (phase == 0 && A.refine && status == 0) grid.sync();  // the true residual reads x
    }
    if (status != 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    PcgState* pc = A.pcg;
    pc->nrhs = KK;
    for (int j = 0; j < KK; ++j) {
      pc->bb[j] = bb[j]; pc->rr[j] = rr[j]; pc->rz[j] = rz[j]; pc->its[j] = its[j]; pc->active[j] = active[j];
    }
    A.st->loop_iters += loops;
    if (status != 0 && A.st->status == 0) {
      A.st->status = status;
      A.st->fail_step = A.st->steps;
      A.st->fail_block = fail_block;
    }
  }
}

static inline TileLine fused_tile(const PrecArgs& a, int d, int ST) {
  const GridDesc& g = a.g;
  const int bd[3] = {a.bd[0][0], a.bd[0][1], a.bd[0][2]};
  const long long str[3] = {a.kk, (long long)g.nx * a.kk, (long long)g.nx * g.ny * a.kk};
  const long long sc = g.padded * a.kk;
  TileLine tl;
  memset(&tl, 0, sizeof(tl));
  tl.t = a.z + g.guard * a.kk; tl.n = bd[d]; tl.kk = a.kk; tl.st = a.st;
  tl.Ff = a.Ff[0][d]; tl.Fb = a.Fb[0][d]; tl.flen = a.flen[0][d];
  tl.clen = a.clen[0][d]; tl.C = a.nchunk[0][d]; tl.L = a.nlev[0][d];
  tl.ST = ST;
  if (d == 0) {
    tl.mode = 1; tl.nlines = a.nvec * bd[1] * bd[2]; tl.nl2 = bd[1] * bd[2]; tl.sA = sc; tl.sB = str[1];
  } else {
    tl.mode = 0; tl.es = str[d]; tl.rowlen = bd[0] * a.kk;
    const int other = (d == 1) ? 2 : 1;
    const int nother = (g.dim == 3) ? bd[other] : 1;
    tl.nrows = a.nvec * nother; tl.nr2 = nother; tl.sA = sc; tl.sB = (g.dim == 3) ? str[other] : 0;
  }
  const long long off = g.guard * a.kk;
  tl.padkk = g.padded * a.kk;
  tl.s = a.s[0];
  tl.x = a.x + off; tl.r = a.r + off; tl.p0 = a.p0 + off; tl.p1 = a.p0 + off; tl.q = a.q + off;
  tl.pcg = a.pcg; tl.maxit = a.maxit; tl.update = 1;
  tl.xdefer = 1;  // x += alpha p rides on the next SpMV (and the exit pass)
  tl.pro = (d == 0);
  tl.epi = (d == g.dim - 1);
  return tl;
}

static inline void persist_layout(const PersistArgs& Aa, PersistDev& D, size_t& smem_bytes) {
  const PrecArgs& a = Aa.pa;
  size_t ofs = 0;
  size_t scratch = 0;
  for (int d = 0; d < a.g.dim; ++d) {
    // slots per tile so that 8 warps cover the chunks: 8 * (32/ST) >= C (C <= 64)
    const int C = a.nchunk[0][d];
    int ST = 32;
    while (ST > 4 && 8 * (32 / ST) < C) ST >>= 1;
    D.tl[d] = fused_tile(a, d, ST);
    D.fofs[d] = (int)ofs;
    ofs += 2 * (size_t)a.flen[0][d];
    // register-resident tiles (clen <= 8) need only the chunk-state scratch
    const size_t tsz = (a.clen[0][d] <= 8 ? 0 : (size_t)D.tl[d].n * (ST + 1)) + (size_t)C * a.p * ST;
    scratch = std::max(scratch, tsz);
    D.ntiles[d] = D.tl[d].mode == 0 ? D.tl[d].nrows * ((D.tl[d].rowlen + ST - 1) / ST)
                                    : (D.tl[d].nlines * D.tl[d].kk + ST - 1) / ST;
  }
  const int W = 2 * a.p + 1;
  const size_t sp = 2 * 8 * (size_t)(32 + 2 * a.p) * a.kk + 8 * (size_t)a.kk * 32;
  (void)W;
  scratch = std::max(scratch, sp);
  D.scratch_ofs = (int)ofs;
  smem_bytes = sizeof(double) * (ofs + scratch);
}

inline bool persist_supported_impl(const PersistArgs& A) {
  const PrecArgs& a = A.pa;
  if (a.npatch != 1 || a.t[0] != nullptr || a.nvec != 1) return false;
  for (int d = 0; d < a.g.dim; ++d)
    if (!a.Ff[0][d] || a.nchunk[0][d] > 64) return false;
  PersistDev D;
  size_t bytes = 0;
  persist_layout(A, D, bytes);
  return bytes + 8192 <= 220 * 1024;
}

template <int P, int KK>
static bool persist_launch_t(const PersistArgs& A, cudaStream_t s) {
  PersistDev D;
  memset(&D, 0, sizeof(D));
  size_t bytes = 0;
  persist_layout(A, D, bytes);
  const PrecArgs& a = A.pa;
  D.g = a.g; D.nvec = a.nvec; D.kk = a.kk; D.dim = a.g.dim; D.refine = A.refine; D.maxit = a.maxit;
  D.tol2 = a.tol2; D.refine_rtol2 = A.refine_rtol2;
  D.spq = A.spq; D.str = A.str;
  D.gpart = a.partial;
  D.b = A.va.b; D.x = a.x; D.r = a.r; D.z = a.z; D.p = const_cast<double*>(a.p0); D.p1 = A.p1;
  D.pcg = a.pcg; D.st = a.st; D.trace = A.trace;
  for (int d = 0; d < 3; ++d) D.tl[d].trace = A.trace;
  static int max_blocks = -1;
  static size_t attr_bytes = 0;
  if (bytes > attr_bytes) {
    if (cudaFuncSetAttribute(k_pcg_persist<P, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      return false;
    attr_bytes = bytes;
    max_blocks = -1;
  }
  if (max_blocks < 0) {
    int per_sm = 0, dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_persist<P, KK>, PBLK, bytes) != cudaSuccess ||
        per_sm < 1)
      return false;
    max_blocks = nsm * std::min(per_sm, 2);
  }
  void* args[] = {&D};
  return cudaLaunchCooperativeKernel((const void*)k_pcg_persist<P, KK>, dim3(max_blocks), dim3(PBLK), args, bytes, s) ==
         cudaSuccess;
}

}  // namespace ga
