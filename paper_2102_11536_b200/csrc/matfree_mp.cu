// Multi-pass matrix-free mass apply in 3D (SURVEY §8a a5 alternative; DESIGN.md
// "Matrix-free operator"): the non-redundant global sum factorisation
//   y = B^T (W o (B x)),  B = B_z (x) B_y (x) B_x  (Gauss rule R12)
// as five bandwidth-bound passes through HBM intermediates, each output computed by one
// thread in a fixed order (deterministic):
//   A  z-forward   T1[qz][y][x]   = sum_a N_z(qz,a) X[e(qz)+a][y][x]
//   B  y-forward   T2[qz][qy][x]  = sum_a N_y(qy,a) T1[qz][e(qy)+a][x]
//   C  x rows      T3[qz][qy][x]  = sum_{qx in supp x} N_x(qx,.) W[qz][qy][qx] sum_a N_x(qx,a) T2[qz][qy][e(qx)+a]
//                  (one warp per chunk of 32 elements of a row; the element contributions to
//                   the p+1 bases they touch are combined by warp shuffles)
//   D  y-back      T1[qz][y][x]   = sum_{qy in supp y} N_y(qy,.) T3[qz][qy][x]   (chunked walks)
//   E  z-back      Y[z][y][x]     = sum_{qz in supp z} N_z(qz,.) T1[qz][y][x], + the PCG epilogue
// Per DoF and right-hand side the passes move about (2 + 2(p+1) + 2(p+1)^2) doubles plus the
// (p+1)^3 Gauss-point weights shared by the k right-hand sides, against (2p+1)^3 coefficients
// for the stencil SpMV.  Free basis b (full index b+1 in 1..m-2) of a direction is touched by
// elements e = b+1-p .. b+1.
#include <cuda_runtime.h>

#include <algorithm>

#include "ops.cuh"

namespace ga {

namespace {

struct MpDims {
  int n, nf, nvec;
  int nq;
};

constexpr int MPT = 256;  // threads per CTA (flat grid-stride mappings, x * k innermost)

// T1 [c][qz][y][x][j], T2 / T3 [c][qz][qy][x][j]; row = all (x, j) of one (c, a, b)
__device__ __forceinline__ long long mp_row(long long c, long long a, long long b, int nb, int na, int nf, int kk) {
  return (((c * na + a) * nb + b) * nf) * kk;
}

// A: thread per (c, ez, y, x*k + j); writes the P1 Gauss planes of element ez
template <int P, int KK>
__global__ void __launch_bounds__(MPT) k_mp_zfwd(const double* __restrict__ X, GridDesc g, const double* __restrict__ tv,
                                                 double* __restrict__ T1, MpDims d) {
  constexpr int P1 = P + 1;
  const int rowlen = d.nf * KK;
  const long long tot = (long long)d.nvec * d.n * d.nf * rowlen;
  for (long long t = (long long)blockIdx.x * MPT + threadIdx.x; t < tot; t += (long long)gridDim.x * MPT) {
    const int q = (int)(t % rowlen);
    const long long row = t / rowlen;  // (c, ez, y)
    const int y = (int)(row % d.nf);
    const int ez = (int)((row / d.nf) % d.n);
    const int c = (int)(row / ((long long)d.nf * d.n));
    double in[P1];
#pragma unroll
    for (int a = 0; a < P1; ++a) {
      const int z = ez + a - 1;
      in[a] = (z >= 0 && z < d.nf)
                  ? __ldg(X + ((long long)c * g.padded + g.guard + ((long long)z * d.nf + y) * d.nf) * KK + q)
                  : 0.0;
    }
#pragma unroll
    for (int qq = 0; qq < P1; ++qq) {
      const double* nr = tv + ((long long)ez * P1 + qq) * P1;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < P1; ++a) s = fma(__ldg(nr + a), in[a], s);
      T1[mp_row(c, (long long)ez * P1 + qq, y, d.nf, d.nq, d.nf, KK) + q] = s;
    }
  }
}

// B: thread per (c, qz, ey, x*k + j); writes the P1 Gauss rows of element ey
template <int P, int KK>
__global__ void __launch_bounds__(MPT) k_mp_yfwd(const double* __restrict__ T1, const double* __restrict__ tv,
                                                 double* __restrict__ T2, MpDims d) {
  constexpr int P1 = P + 1;
  const int rowlen = d.nf * KK;
  const long long tot = (long long)d.nvec * d.nq * d.n * rowlen;
  for (long long t = (long long)blockIdx.x * MPT + threadIdx.x; t < tot; t += (long long)gridDim.x * MPT) {
    const int q = (int)(t % rowlen);
    const long long row = t / rowlen;  // (c*nq + qz, ey)
    const int ey = (int)(row % d.n);
    const long long cq = row / d.n;
    const double* src = T1 + cq * d.nf * rowlen + q;
    double in[P1];
#pragma unroll
    for (int a = 0; a < P1; ++a) {
      const int y = ey + a - 1;
      in[a] = (y >= 0 && y < d.nf) ? __ldg(src + (long long)y * rowlen) : 0.0;
    }
    double* dst = T2 + (cq * d.nq + (long long)ey * P1) * rowlen + q;
#pragma unroll
    for (int qq = 0; qq < P1; ++qq) {
      const double* nr = tv + ((long long)ey * P1 + qq) * P1;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < P1; ++a) s = fma(__ldg(nr + a), in[a], s);
      dst[(long long)qq * rowlen] = s;
    }
  }
}

// C: one warp per (c, qz, qy, chunk of 32 - p elements): lane L owns element e = e0 + L; it
// x-forwards its P1 Gauss points, multiplies by W and x-back-contracts to its P1 local
// contributions ca[a] (basis e + a); basis e0 + L then gathers ca[a] of lane L - a by shuffles.
// (Measured alternatives: a CTA per rows with the Gauss values in shared memory,
// tables staged in shared memory with W through a per-warp slice, two rows per warp — all
// slower on B200 than this register version.)
template <int P, int KK>
__global__ void __launch_bounds__(MPT) k_mp_xrow(const double* __restrict__ T2, const double* __restrict__ W,
                                                 const double* __restrict__ tv, double* __restrict__ T3, MpDims d,
                                                 int nchunk) {
  constexpr int P1 = P + 1;
  const int lane = threadIdx.x & 31;
  const long long nwarp = (long long)d.nvec * d.nq * d.nq * nchunk;
  const long long nqq = (long long)d.nq * d.nq;
  const int rowlen = d.nf * KK;
  for (long long w = (long long)blockIdx.x * (MPT / 32) + (threadIdx.x >> 5); w < nwarp;
       w += (long long)gridDim.x * (MPT / 32)) {
    const int ch = (int)(w % nchunk);
    const long long row = w / nchunk;  // (c * nq + qz) * nq + qy
    const int e0 = ch * (32 - P);
    const int e = e0 + lane;
    const bool ev = e < d.n;
    const double* in = T2 + row * rowlen;
    const double* wr = W + (row % nqq) * d.nq + (long long)e * P1;
    double xin[P1][KK];
#pragma unroll
    for (int a = 0; a < P1; ++a) {
      const int x = e + a - 1;
      const bool ok = ev && x >= 0 && x < d.nf;
#pragma unroll
      for (int j = 0; j < KK; ++j) xin[a][j] = ok ? __ldg(in + x * KK + j) : 0.0;
    }
    double ca[P1][KK];
#pragma unroll
    for (int a = 0; a < P1; ++a)
#pragma unroll
      for (int j = 0; j < KK; ++j) ca[a][j] = 0.0;
#pragma unroll
    for (int qq = 0; qq < P1; ++qq) {
      double nt[P1];
      const double* nr = tv + ((long long)e * P1 + qq) * P1;
#pragma unroll
      for (int a = 0; a < P1; ++a) nt[a] = ev ? __ldg(nr + a) : 0.0;
      const double wq = ev ? __ldg(wr + qq) : 0.0;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < P1; ++a) s = fma(nt[a], xin[a][j], s);
        s *= wq;
#pragma unroll
        for (int a = 0; a < P1; ++a) ca[a][j] = fma(nt[a], s, ca[a][j]);
      }
    }
    const int xo = e0 + lane - 1;  // free index of basis e0 + lane
    const bool own = (ch == 0 ? lane >= 1 : lane >= P) && xo >= 0 && xo < d.nf;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
      double out = ca[0][j];
#pragma unroll
      for (int a = 1; a < P1; ++a) {
        const double v = __shfl_up_sync(0xffffffffu, ca[a][j], a);
        out += lane >= a ? v : 0.0;
      }
      if (own) T3[row * rowlen + xo * KK + j] = out;
    }
  }
}

// Sliding-window back contraction along a strided direction: a thread owns one (x, j) slot of
// a row and a chunk [b0, b1) of full basis indices; it walks the elements touching the chunk
// (owner computes: the p elements before the chunk are re-evaluated), reads every Gauss value
// once and emits each basis when its last element has been added.
template <int P, typename Emit>
__device__ __forceinline__ void mp_walk(const double* __restrict__ src, long long qstride, const double* __restrict__ tv,
                                        int n, int nf, int b0, int b1, Emit emit) {
  constexpr int P1 = P + 1;
  const int e0 = max(0, b0 - P), e1 = min(n - 1, b1 - 1);
  double acc[P1];
#pragma unroll
  for (int u = 0; u < P1; ++u) acc[u] = 0.0;
  for (int e = e0; e <= e1; ++e) {
    double v[P1];
#pragma unroll
    for (int qq = 0; qq < P1; ++qq) v[qq] = __ldg(src + ((long long)e * P1 + qq) * qstride);
#pragma unroll
    for (int qq = 0; qq < P1; ++qq) {
      const double* nr = tv + ((long long)e * P1 + qq) * P1;
#pragma unroll
      for (int u = 0; u < P1; ++u) acc[u] = fma(__ldg(nr + u), v[qq], acc[u]);
    }
    if (e >= b0 && e < b1 && e >= 1) emit(e - 1, acc[0]);
#pragma unroll
    for (int u = 0; u < P; ++u) acc[u] = acc[u + 1];
    acc[P] = 0.0;
  }
#pragma unroll
  for (int u = 0; u < P; ++u) {
    const int b = e1 + 1 + u;
    if (b >= b0 && b < b1 && b <= nf) emit(b - 1, acc[u]);
  }
}

// D: thread per (c, qz, y-chunk, x*k + j): T1[c][qz][y][:] = sum_{qy in supp y} N_y T3[c][qz][qy][:]
template <int P, int KK>
__global__ void __launch_bounds__(MPT) k_mp_yback(const double* __restrict__ T3, const double* __restrict__ tv,
                                                  double* __restrict__ T1, MpDims d, int YC, int nyc) {
  const int rowlen = d.nf * KK;
  const long long tot = (long long)d.nvec * d.nq * nyc * rowlen;
  for (long long t = (long long)blockIdx.x * MPT + threadIdx.x; t < tot; t += (long long)gridDim.x * MPT) {
    const int q = (int)(t % rowlen);
    const long long row = t / rowlen;  // (c*nq + qz, yc)
    const int yc = (int)(row % nyc);
    const long long cq = row / nyc;
    const int b0 = 1 + yc * YC, b1 = min(b0 + YC, d.nf + 1);
    double* dst = T1 + cq * d.nf * rowlen + q;
    mp_walk<P>(T3 + cq * d.nq * rowlen + q, rowlen, tv, d.n, d.nf, b0, b1,
               [&](int y, double v) { dst[(long long)y * rowlen] = v; });
  }
}

// E: thread per (c, z-chunk, y, x*k + j): Y = sum_{qz in supp z} N_z T1[c][qz][y][:], + the SpMV epilogue
template <int P, int KK>
__global__ void __launch_bounds__(MPT) k_mp_zback(const double* __restrict__ T1, const double* __restrict__ tv, SpmvArgs a,
                                                  MpDims d, int ZC, int nzc) {
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&a.st->launches, 1ull);
  const GridDesc g = a.g;
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  const int rowlen = d.nf * KK;
  const long long tot = (long long)d.nvec * nzc * d.nf * rowlen;
  for (long long t = (long long)blockIdx.x * MPT + threadIdx.x; t < tot; t += (long long)gridDim.x * MPT) {
    const int q = (int)(t % rowlen);
    const int j = q % KK;
    const long long row = t / rowlen;  // (c, zc, y)
    const int y = (int)(row % d.nf);
    const int zc = (int)((row / d.nf) % nzc);
    const long long c = row / ((long long)d.nf * nzc);
    const int b0 = 1 + zc * ZC, b1 = min(b0 + ZC, d.nf + 1);
    const double* src = T1 + ((c * d.nq) * d.nf + y) * rowlen + q;
    mp_walk<P>(src, (long long)d.nf * rowlen, tv, d.n, d.nf, b0, b1, [&](int z, double sv) {
      const long long e = (c * g.padded + g.guard + ((long long)z * d.nf + y) * d.nf) * KK + q;
      double v = sv, dd = 0.0;
      if (a.mode == SPMV_NEGB) v = -v;
      else if (a.mode == SPMV_TRUERES) { v = a.b[e] - v; dd = v * v; }
      else if (a.mode == SPMV_PQ) dd = a.x[e] * v;
      a.y[e] = v;
#pragma unroll
      for (int jj = 0; jj < KK; ++jj) dots[jj] += (jj == j) ? dd : 0.0;
    });
  }
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) {
    block_sum<KK>(dots);
    if (threadIdx.x == 0)
      for (int q = 0; q < KK; ++q) a.partial[(size_t)blockIdx.x * KK + q] = dots[q];
  }
}

unsigned int mp_blocks(long long rows) { return (unsigned int)std::max(1LL, std::min<long long>(rows, 148LL * 16)); }

template <int P, int KK>
void mp_launch_kk(const SpmvArgs& a, cudaStream_t s) {
  MpDims d;
  d.n = a.mfn; d.nf = a.g.nx; d.nvec = a.nvec; d.nq = a.mfn * (P + 1);
  const long long nf = d.nf, nq = d.nq, rl = nf * KK;
  auto blocks = [](long long threads) { return mp_blocks((threads + MPT - 1) / MPT); };
  k_mp_zfwd<P, KK><<<blocks((long long)d.nvec * d.n * nf * rl), MPT, 0, s>>>(a.x, a.g, a.mfv, a.mpT1, d);
  k_mp_yfwd<P, KK><<<blocks((long long)d.nvec * nq * d.n * rl), MPT, 0, s>>>(a.mpT1, a.mfv, a.mpT2, d);
  const int nchunk = (d.n + P + 31 - P - 1) / (32 - P) + 1;  // covers full bases 1 .. n + p - 2
  k_mp_xrow<P, KK><<<blocks((long long)d.nvec * nq * nq * nchunk * 32), MPT, 0, s>>>(a.mpT2, a.mfW, a.mfv, a.mpT3, d,
                                                                                     nchunk);
  const int YC = 16, nyc = (d.nf + YC - 1) / YC;
  k_mp_yback<P, KK><<<blocks((long long)d.nvec * nq * nyc * rl), MPT, 0, s>>>(a.mpT3, a.mfv, a.mpT1, d, YC, nyc);
  const int ZC = 16, nzc = (d.nf + ZC - 1) / ZC;
  const unsigned int nb = blocks((long long)d.nvec * nzc * nf * rl);
  k_mp_zback<P, KK><<<nb, MPT, 0, s>>>(a.mpT1, a.mfv, a, d, ZC, nzc);
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) launch_spmv_fin(a, nb, s);
}

template <int P>
void mp_launch(const SpmvArgs& a, cudaStream_t s) {
  switch (a.kk) {
    case 1: mp_launch_kk<P, 1>(a, s); break;
    case 2: mp_launch_kk<P, 2>(a, s); break;
    case 3: mp_launch_kk<P, 3>(a, s); break;
    default: mp_launch_kk<P, 4>(a, s); break;
  }
}

}  // namespace

void launch_matfree_mp(const SpmvArgs& a, cudaStream_t s) {
  switch (a.p) {
    case 1: mp_launch<1>(a, s); break;
    case 2: mp_launch<2>(a, s); break;
    case 3: mp_launch<3>(a, s); break;
    case 4: mp_launch<4>(a, s); break;
    case 5: mp_launch<5>(a, s); break;
    case 6: mp_launch<6>(a, s); break;
    default: mp_launch<7>(a, s); break;
  }
}

}  // namespace ga
