// Matrix-free sum-factorised operator apply (SURVEY §8a row a5 "matrix-free
// alternative").  The operators are the
// Gauss-quadrature Galerkin forms of P:695-697 / the weak form of P:57,
//   M_ij = sum_q W(q) B_i(q) B_j(q),          W = w|J| (x density, elastic mass)
//   K_ij = sum_q grad^ B_i(q)^T Wk(q) grad^ B_j(q),   Wk = omega^2 w|J| J^-1 J^-T,
// with B_i = N_{i_x}(x) N_{i_y}(y) N_{i_z}(z) the tensor-product B-splines, so
// y = A x factorises direction by direction (B = B_z (x) B_y (x) B_x):
//   forward  z, x, y contractions to the Gauss points, pointwise W,
//   backward y, x, z contractions to the basis functions.
//
// Tiling (3D): a CTA owns a DX x DY column of basis functions (owner computes:
// it also evaluates the p-wide halo of elements around the column, so no two
// CTAs write the same output) and a chunk of ZL basis layers along z.  It
// streams the element layers e_z of its chunk: a ring of p+1 input planes
// (bases e_z..e_z+p) lives in shared memory; for each of the p+1 Gauss points
// q_z of the layer the plane is z-contracted, x-contracted, and then one
// thread per (x Gauss point, rhs) walks the y elements with sliding register
// windows doing the y contraction, the W product and the y back-contraction;
// the x back-contraction and the z back-contraction accumulate into a ring of
// p+1 output planes, one of which completes per layer and is written out with
// the PCG epilogue of the stencil SpMV (apply, -K s, q = M p with p.q, b - M x).
// 2D: the same with y as the streamed direction and no middle direction.
// All accumulation orders are fixed (deterministic results).
#pragma once
#include "ops.cuh"

namespace ga {

template <int P, int KK, bool STIFF, int DX, int DY>
struct Mf3Shape {
  static constexpr int P1 = P + 1, IX = DX + 2 * P, IY = DY + 2 * P, EX = DX + P, EY = DY + P, QX = EX * P1;
  static constexpr int NZF = STIFF ? 2 : 1, NF = STIFF ? 3 : 1;
  static constexpr int PLANE = IY * IX * KK;
  static constexpr int RING = P1 * PLANE;
  static constexpr int TZ = NZF * PLANE;
  static constexpr int TXS = IY * QX * KK;
  static constexpr int TX = NF * TXS;
  static constexpr int VS = DY * QX * KK;
  static constexpr int V = NF * VS;
  static constexpr int ACCS = DY * DX * KK;
  static constexpr int ACC = P1 * ACCS;
  static constexpr int TABX = EX * P1 * P1, TABY = EY * P1 * P1;  // per-tile 1D tables (val; der)
  static constexpr int TAB = (STIFF ? 2 : 1) * (TABX + TABY);
  static constexpr int TOTAL = RING + TZ + TX + V + ACC + TAB;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

template <int P, int KK, bool STIFF, int DX>
struct Mf2Shape {
  static constexpr int P1 = P + 1, IX = DX + 2 * P, EX = DX + P, QX = EX * P1;
  static constexpr int NYF = STIFF ? 2 : 1, NF = STIFF ? 2 : 1;
  static constexpr int LINE = IX * KK;
  static constexpr int RING = P1 * LINE;
  static constexpr int TY = NYF * LINE;
  static constexpr int US = QX * KK;
  static constexpr int U = NF * US;
  static constexpr int ACCS = DX * KK;
  static constexpr int ACC = P1 * ACCS;
  static constexpr int TOTAL = RING + TY + U + ACC;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

__device__ __forceinline__ void mf_count_launch(DevStatus* st) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) atomicAdd(&st->launches, 1ull);
}

// Output epilogue shared by both kernels (the modes of the stencil SpMV).
template <int KK>
__device__ __forceinline__ void mf_emit(const SpmvArgs& a, long long e, int j, double v, double pval,
                                        double (&dots)[KK]) {
  double d = 0.0;
  if (a.mode == SPMV_NEGB) v = -v;
  else if (a.mode == SPMV_TRUERES) { v = a.b[e] - v; d = v * v; }
  else if (a.mode == SPMV_PQ) d = pval * v;
  a.y[e] = v;
#pragma unroll
  for (int jj = 0; jj < KK; ++jj) dots[jj] += (jj == j) ? d : 0.0;  // branch-free select
}

template <int KK, int NT>
__device__ __forceinline__ void mf_finish(const SpmvArgs& a, double (&dots)[KK]) {
  if (a.mode != SPMV_PQ && a.mode != SPMV_TRUERES) return;
  block_sum<KK>(dots);
  if (threadIdx.x == 0) {
    const long long blin = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
#pragma unroll
    for (int j = 0; j < KK; ++j) a.partial[blin * a.kk + a.mfj0 + j] = dots[j];
  }
}

// ---------------------------------------------------------------------------
// 3D
// ---------------------------------------------------------------------------
template <int P, int KK, bool STIFF, int DX, int DY, int NT>
__global__ void __launch_bounds__(NT, (STIFF || P <= 4) ? 1 : 2) k_mf3(SpmvArgs a, int ZL, int nzc) {
  using L = Mf3Shape<P, KK, STIFF, DX, DY>;
  constexpr int P1 = L::P1, IX = L::IX, IY = L::IY, EY = L::EY, QX = L::QX, PLANE = L::PLANE;
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  mf_count_launch(a.st);
  extern __shared__ double smem_mf[];
  double* ring = smem_mf;      // [P1][IY][IX][KK]   input bases e_z..e_z+p (slot = basis % P1)
  double* tz = ring + L::RING; // [NZF][IY][IX][KK]  z-contracted plane (N_z; D_z)
  double* tx = tz + L::TZ;     // [NF][IY][QX][KK]   + x-contracted (N_x N_z; D_x N_z; N_x D_z)
  double* vv = tx + L::TX;     // [NF][DY][QX][KK]   after y forward, W, y back (owned y bases)
  double* acc = vv + L::V;     // [P1][DY][DX][KK]   output ring (slot = basis % P1)
  double* snx = acc + L::ACC;  // [EX][P1][P1] N_x of the tile's elements (0 outside the patch)
  double* sny = snx + L::TABX; // [EY][P1][P1]
  double* sdx = sny + L::TABY; // derivatives (stiffness only)
  double* sdy = sdx + L::TABX;
  const GridDesc g = a.g;
  const int n = a.mfn, m = n + P;
  const long long nq = (long long)n * P1;
  const int tid = threadIdx.x;
  const int comp = blockIdx.z / nzc, zc = blockIdx.z % nzc;
  const int bx0 = 1 + blockIdx.x * DX, by0 = 1 + blockIdx.y * DY;  // first owned basis (full index)
  const int bz0 = 1 + zc * ZL, bz1 = min(bz0 + ZL, m - 1);
  const int exb = bx0 - P, eyb = by0 - P;  // global index of local element / local input basis 0
  const int ez0 = max(0, bz0 - P), ez1 = min(n - 1, bz1 - 1);
  const double* __restrict__ tv = a.mfv;
  const double* __restrict__ td = a.mfd;
  const long long ks = a.kk;
  const int j0 = a.mfj0;
  const long long cbase = (long long)comp * g.padded + g.guard;
  const long long sy = g.nx, sz = (long long)g.nx * g.ny;
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  for (int i = tid; i < L::ACC; i += NT) acc[i] = 0.0;
  for (int i = tid; i < L::TABX; i += NT) {
    const int ex = exb + i / (P1 * P1);
    const bool ok = ex >= 0 && ex < n;
    snx[i] = ok ? __ldg(tv + (long long)exb * P1 * P1 + i) : 0.0;
    if (STIFF) sdx[i] = ok ? __ldg(td + (long long)exb * P1 * P1 + i) : 0.0;
  }
  for (int i = tid; i < L::TABY; i += NT) {
    const int ey = eyb + i / (P1 * P1);
    const bool ok = ey >= 0 && ey < n;
    sny[i] = ok ? __ldg(tv + (long long)eyb * P1 * P1 + i) : 0.0;
    if (STIFF) sdy[i] = ok ? __ldg(td + (long long)eyb * P1 * P1 + i) : 0.0;
  }

  constexpr int LPT = (PLANE + NT - 1) / NT;
  auto load_plane = [&](int bz, double (&pf)[LPT]) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int idx = tid + u * NT;
      double v = 0.0;
      if (idx < PLANE) {
        const int j = idx % KK, xl = (idx / KK) % IX, yl = idx / (KK * IX);
        const int bx = exb + xl, by = eyb + yl;
        if (bz >= 1 && bz <= m - 2 && bx >= 1 && bx <= m - 2 && by >= 1 && by <= m - 2)
          v = __ldg(a.x + (cbase + (bx - 1) + sy * (by - 1) + sz * (bz - 1)) * ks + j0 + j);
      }
      pf[u] = v;
    }
  };
  auto store_plane = [&](int bz, const double (&pf)[LPT]) {
    double* dst = ring + (bz % P1) * PLANE;
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int idx = tid + u * NT;
      if (idx < PLANE) dst[idx] = pf[u];
    }
  };
  // write the completed output plane of basis bz (owned layers only) and clear its slot
  auto flush = [&](int bz) {
    const bool owned = bz >= bz0 && bz < bz1;  // block-uniform; halo layers are only cleared
    for (int i = tid; i < L::ACCS; i += NT) {
      const int j = i % KK, bxl = (i / KK) % DX, byl = i / (KK * DX);
      double* slot = acc + (bz % P1) * L::ACCS + i;
      const double v = *slot;
      *slot = 0.0;
      const int bx = bx0 + bxl, by = by0 + byl;
      if (owned && bx <= m - 2 && by <= m - 2) {
        const double pval = ring[(bz % P1) * PLANE + ((byl + P) * IX + bxl + P) * KK + j];
        const long long e = (cbase + (bx - 1) + sy * (by - 1) + sz * (bz - 1)) * ks + j0 + j;
        mf_emit<KK>(a, e, j, v, pval, dots);
      }
    }
  };

  double pf[LPT];
  for (int bz = ez0; bz < ez0 + P; ++bz) {
    load_plane(bz, pf);
    store_plane(bz, pf);
  }
  load_plane(ez0 + P, pf);
  for (int ez = ez0; ez <= ez1; ++ez) {
    __syncthreads();  // the previous flush has read the slot replaced here
    store_plane(ez + P, pf);
    __syncthreads();
    if (ez < ez1) load_plane(ez + 1 + P, pf);  // in flight during this layer
    for (int qz = 0; qz < P1; ++qz) {
      const long long qzg = (long long)ez * P1 + qz;
      double cz[P1], dz[P1];
#pragma unroll
      for (int u = 0; u < P1; ++u) {
        cz[u] = __ldg(tv + qzg * P1 + u);
        dz[u] = STIFF ? __ldg(td + qzg * P1 + u) : 0.0;
      }
      // (a) z contraction of the ring
      for (int i = tid; i < PLANE; i += NT) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int u = 0; u < P1; ++u) {
          const double r = ring[((ez + u) % P1) * PLANE + i];
          s0 = fma(cz[u], r, s0);
          if (STIFF) s1 = fma(dz[u], r, s1);
        }
        tz[i] = s0;
        if (STIFF) tz[PLANE + i] = s1;
      }
      __syncthreads();
      // (b) x contraction to the x Gauss points of the tile's elements
      for (int i = tid; i < L::TXS; i += NT) {
        const int j = i % KK, qxl = (i / KK) % QX, yl = i / (KK * QX);
        const int exl = qxl / P1;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        {
          const double* nr = snx + qxl * P1;  // zero rows outside the patch
          const double* dr = sdx + qxl * P1;
          const double* t0 = tz + (yl * IX + exl) * KK + j;
#pragma unroll
          for (int u = 0; u < P1; ++u) {
            const double nxu = nr[u];
            s0 = fma(nxu, t0[u * KK], s0);
            if (STIFF) {
              s1 = fma(dr[u], t0[u * KK], s1);
              s2 = fma(nxu, t0[PLANE + u * KK], s2);
            }
          }
        }
        tx[i] = s0;
        if (STIFF) { tx[L::TXS + i] = s1; tx[2 * L::TXS + i] = s2; }
      }
      __syncthreads();
      // (c) per (x Gauss point, rhs): walk the y elements; the quadrature data of the
      //     next element is loaded one step ahead (software pipeline)
      for (int t = tid; t < QX * KK; t += NT) {
        const int j = t % KK, qxl = t / KK;
        const int ex = exb + qxl / P1;
        const bool xv = ex >= 0 && ex < n;
        const double* wbase = a.mfW + (qzg * nq) * nq + ((long long)exb * P1 + qxl);  // + qyg * nq
        constexpr int NW = STIFF ? 6 * P1 : P1;
        double in0[P1], in1[P1], in2[P1], ac0[P1], ac1[P1], ac2[P1], wn[NW];
        auto load_w = [&](int eyl) {
          const int ey = eyb + eyl;
          const bool ok = xv && ey >= 0 && ey < n;
          const double* wr = wbase + (long long)ey * P1 * nq;
#pragma unroll
          for (int qy = 0; qy < P1; ++qy) {
            if (!STIFF) {
              wn[qy] = ok ? __ldg(wr + qy * nq) : 0.0;
            } else {
#pragma unroll
              for (int c = 0; c < 6; ++c) wn[c * P1 + qy] = ok ? __ldg(wr + qy * nq + c * a.mfws) : 0.0;
            }
          }
        };
#pragma unroll
        for (int u = 0; u < P; ++u) {
          in0[u] = tx[(u * QX + qxl) * KK + j];
          if (STIFF) {
            in1[u] = tx[L::TXS + (u * QX + qxl) * KK + j];
            in2[u] = tx[2 * L::TXS + (u * QX + qxl) * KK + j];
          }
        }
#pragma unroll
        for (int u = 0; u < P1; ++u) { ac0[u] = 0.0; ac1[u] = 0.0; ac2[u] = 0.0; }
        if (!STIFF) load_w(0);
        for (int eyl = 0; eyl < EY; ++eyl) {
          in0[P] = tx[((eyl + P) * QX + qxl) * KK + j];
          if (STIFF) {
            in1[P] = tx[L::TXS + ((eyl + P) * QX + qxl) * KK + j];
            in2[P] = tx[2 * L::TXS + ((eyl + P) * QX + qxl) * KK + j];
          }
          double w[NW];
          if constexpr (STIFF) load_w(eyl);  // 6 (p+1) values: no room to pipeline in registers
#pragma unroll
          for (int c = 0; c < NW; ++c) w[c] = wn[c];
          if (!STIFF && eyl + 1 < EY) load_w(eyl + 1);
#pragma unroll
          for (int qy = 0; qy < P1; ++qy) {
            const double* nr = sny + (eyl * P1 + qy) * P1;  // zero outside the patch
            double ny[P1];
#pragma unroll
            for (int u = 0; u < P1; ++u) ny[u] = nr[u];
            if (!STIFF) {
              double s = 0.0;
#pragma unroll
              for (int u = 0; u < P1; ++u) s = fma(ny[u], in0[u], s);
              s *= w[qy];
#pragma unroll
              for (int u = 0; u < P1; ++u) ac0[u] = fma(ny[u], s, ac0[u]);
            } else {
              const double* dr = sdy + (eyl * P1 + qy) * P1;
              double dy[P1];
#pragma unroll
              for (int u = 0; u < P1; ++u) dy[u] = dr[u];
              double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
              for (int u = 0; u < P1; ++u) {
                gx = fma(ny[u], in1[u], gx);  // D_x N_y N_z
                gy = fma(dy[u], in0[u], gy);  // N_x D_y N_z
                gz = fma(ny[u], in2[u], gz);  // N_x N_y D_z
              }
              const double w00 = w[qy], w01 = w[P1 + qy], w02 = w[2 * P1 + qy];
              const double w11 = w[3 * P1 + qy], w12 = w[4 * P1 + qy], w22 = w[5 * P1 + qy];
              const double fx = w00 * gx + w01 * gy + w02 * gz;
              const double fy = w01 * gx + w11 * gy + w12 * gz;
              const double fz = w02 * gx + w12 * gy + w22 * gz;
#pragma unroll
              for (int u = 0; u < P1; ++u) {
                ac0[u] = fma(ny[u], fx, ac0[u]);
                ac1[u] = fma(dy[u], fy, ac1[u]);
                ac2[u] = fma(ny[u], fz, ac2[u]);
              }
            }
          }
          // local y basis eyl is complete; owned bases are eyl in [P, P + DY)
          if (eyl >= P) {
            vv[((eyl - P) * QX + qxl) * KK + j] = ac0[0];
            if (STIFF) {
              vv[L::VS + ((eyl - P) * QX + qxl) * KK + j] = ac1[0];
              vv[2 * L::VS + ((eyl - P) * QX + qxl) * KK + j] = ac2[0];
            }
          }
#pragma unroll
          for (int u = 0; u < P; ++u) {
            ac0[u] = ac0[u + 1]; in0[u] = in0[u + 1];
            if (STIFF) { ac1[u] = ac1[u + 1]; ac2[u] = ac2[u + 1]; in1[u] = in1[u + 1]; in2[u] = in2[u + 1]; }
          }
          ac0[P] = 0.0; ac1[P] = 0.0; ac2[P] = 0.0;
        }
      }
      __syncthreads();
      // (d) x back-contraction to the owned x bases, then z back-contraction into the
      //     output ring (each thread owns fixed acc entries: no barrier needed)
      for (int i = tid; i < L::ACCS; i += NT) {
        const int j = i % KK, bxl = (i / KK) % DX, byl = i / (KK * DX);
        double r0 = 0.0, r1 = 0.0;
        constexpr int XB_UNROLL = P <= 4 ? P + 1 : 1;  // full unroll costs ~80 registers at high p
#pragma unroll XB_UNROLL
        for (int e2 = 0; e2 <= P; ++e2) {
          const int exl = bxl + e2;
          const int u = P - e2;  // local index of basis bx within element exl (zero rows outside)
          const double* vr = vv + (byl * QX + exl * P1) * KK + j;
#pragma unroll
          for (int qx = 0; qx < P1; ++qx) {
            const int row = (exl * P1 + qx) * P1 + u;
            const double nxv = snx[row];
            if (!STIFF) {
              r0 = fma(nxv, vr[qx * KK], r0);
            } else {
              r0 = fma(sdx[row], vr[qx * KK], r0);
              r0 = fma(nxv, vr[L::VS + qx * KK], r0);
              r1 = fma(nxv, vr[2 * L::VS + qx * KK], r1);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < P1; ++u) {
          double* ap = acc + ((ez + u) % P1) * L::ACCS + i;
          double v = fma(cz[u], r0, *ap);
          if (STIFF) v = fma(dz[u], r1, v);
          *ap = v;
        }
      }
    }
    flush(ez);
  }
  for (int bz = ez1 + 1; bz <= ez1 + P; ++bz) flush(bz);
  mf_finish<KK, NT>(a, dots);
}

// ---------------------------------------------------------------------------
// 2D: tiles of DX bases along x, streamed along y
// ---------------------------------------------------------------------------
template <int P, int KK, bool STIFF, int DX, int NT>
__global__ void __launch_bounds__(NT) k_mf2(SpmvArgs a, int YL, int nyc) {
  using L = Mf2Shape<P, KK, STIFF, DX>;
  constexpr int P1 = L::P1, IX = L::IX, QX = L::QX, LINE = L::LINE;
  if (a.st->status != 0 && a.mode != SPMV_APPLY) return;
  mf_count_launch(a.st);
  extern __shared__ double smem_mf[];
  double* ring = smem_mf;       // [P1][IX][KK]
  double* ty = ring + L::RING;  // [NYF][IX][KK]
  double* uu = ty + L::TY;      // [NF][QX][KK]
  double* acc = uu + L::U;      // [P1][DX][KK]
  const GridDesc g = a.g;
  const int n = a.mfn, m = n + P;
  const long long nq = (long long)n * P1;
  const int tid = threadIdx.x;
  const int comp = blockIdx.y / nyc, yc = blockIdx.y % nyc;
  const int bx0 = 1 + blockIdx.x * DX;
  const int by0 = 1 + yc * YL, by1 = min(by0 + YL, m - 1);
  const int exb = bx0 - P;
  const int ey0 = max(0, by0 - P), ey1 = min(n - 1, by1 - 1);
  const double* __restrict__ tv = a.mfv;
  const double* __restrict__ td = a.mfd;
  const long long ks = a.kk;
  const int j0 = a.mfj0;
  const long long cbase = (long long)comp * g.padded + g.guard;
  const long long sy = g.nx;
  double dots[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) dots[j] = 0.0;
  for (int i = tid; i < L::ACC; i += NT) acc[i] = 0.0;
  constexpr int LPT = (LINE + NT - 1) / NT;
  auto load_line = [&](int by, double (&pf)[LPT]) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int idx = tid + u * NT;
      double v = 0.0;
      if (idx < LINE) {
        const int j = idx % KK, xl = idx / KK;
        const int bx = exb + xl;
        if (by >= 1 && by <= m - 2 && bx >= 1 && bx <= m - 2)
          v = __ldg(a.x + (cbase + (bx - 1) + sy * (by - 1)) * ks + j0 + j);
      }
      pf[u] = v;
    }
  };
  auto store_line = [&](int by, const double (&pf)[LPT]) {
    double* dst = ring + (by % P1) * LINE;
#pragma unroll
    for (int u = 0; u < LPT; ++u) {
      const int idx = tid + u * NT;
      if (idx < LINE) dst[idx] = pf[u];
    }
  };
  auto flush = [&](int by) {
    const bool owned = by >= by0 && by < by1;
    for (int i = tid; i < L::ACCS; i += NT) {
      const int j = i % KK, bxl = i / KK;
      double* slot = acc + (by % P1) * L::ACCS + i;
      const double v = *slot;
      *slot = 0.0;
      const int bx = bx0 + bxl;
      if (owned && bx <= m - 2) {
        const double pval = ring[(by % P1) * LINE + (bxl + P) * KK + j];
        const long long e = (cbase + (bx - 1) + sy * (by - 1)) * ks + j0 + j;
        mf_emit<KK>(a, e, j, v, pval, dots);
      }
    }
  };
  double pf[LPT];
  for (int by = ey0; by < ey0 + P; ++by) {
    load_line(by, pf);
    store_line(by, pf);
  }
  load_line(ey0 + P, pf);
  for (int ey = ey0; ey <= ey1; ++ey) {
    __syncthreads();
    store_line(ey + P, pf);
    __syncthreads();
    if (ey < ey1) load_line(ey + 1 + P, pf);
    for (int qy = 0; qy < P1; ++qy) {
      const long long qyg = (long long)ey * P1 + qy;
      double cy[P1], dy[P1];
#pragma unroll
      for (int u = 0; u < P1; ++u) {
        cy[u] = __ldg(tv + qyg * P1 + u);
        dy[u] = STIFF ? __ldg(td + qyg * P1 + u) : 0.0;
      }
      for (int i = tid; i < LINE; i += NT) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int u = 0; u < P1; ++u) {
          const double r = ring[((ey + u) % P1) * LINE + i];
          s0 = fma(cy[u], r, s0);
          if (STIFF) s1 = fma(dy[u], r, s1);
        }
        ty[i] = s0;
        if (STIFF) ty[LINE + i] = s1;
      }
      __syncthreads();
      for (int i = tid; i < L::US; i += NT) {
        const int j = i % KK, qxl = i / KK;
        const int exl = qxl / P1, qx = qxl - exl * P1, ex = exb + exl;
        double f0 = 0.0, f1 = 0.0;
        if (ex >= 0 && ex < n) {
          const double* nr = tv + ((long long)ex * P1 + qx) * P1;
          const double* t0 = ty + exl * KK + j;
          const long long wi = qyg * nq + (long long)ex * P1 + qx;
          if (!STIFF) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < P1; ++u) s = fma(__ldg(nr + u), t0[u * KK], s);
            f0 = s * __ldg(a.mfW + wi);
          } else {
            const double* dr = td + ((long long)ex * P1 + qx) * P1;
            double gx = 0.0, gy = 0.0;
#pragma unroll
            for (int u = 0; u < P1; ++u) {
              gx = fma(__ldg(dr + u), t0[u * KK], gx);         // D_x N_y
              gy = fma(__ldg(nr + u), t0[LINE + u * KK], gy);  // N_x D_y
            }
            const double w00 = __ldg(a.mfW + wi), w01 = __ldg(a.mfW + a.mfws + wi), w11 = __ldg(a.mfW + 2 * a.mfws + wi);
            f0 = w00 * gx + w01 * gy;
            f1 = w01 * gx + w11 * gy;
          }
        }
        uu[i] = f0;
        if (STIFF) uu[L::US + i] = f1;
      }
      __syncthreads();
      for (int i = tid; i < L::ACCS; i += NT) {
        const int j = i % KK, bxl = i / KK;
        double r0 = 0.0, r1 = 0.0;
        constexpr int XB_UNROLL = P <= 4 ? P + 1 : 1;  // full unroll costs ~80 registers at high p
#pragma unroll XB_UNROLL
        for (int e2 = 0; e2 <= P; ++e2) {
          const int exl = bxl + e2, ex = exb + exl;
          if (ex < 0 || ex >= n) continue;
          const int u = P - e2;
          const double* ur = uu + (exl * P1) * KK + j;
#pragma unroll
          for (int qx = 0; qx < P1; ++qx) {
            const long long row = ((long long)ex * P1 + qx) * P1 + u;
            if (!STIFF) {
              r0 = fma(__ldg(tv + row), ur[qx * KK], r0);
            } else {
              r0 = fma(__ldg(td + row), ur[qx * KK], r0);
              r1 = fma(__ldg(tv + row), ur[L::US + qx * KK], r1);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < P1; ++u) {
          double* ap = acc + ((ey + u) % P1) * L::ACCS + i;
          double v = fma(cy[u], r0, *ap);
          if (STIFF) v = fma(dy[u], r1, v);
          *ap = v;
        }
      }
    }
    flush(ey);
  }
  for (int by = ey1 + 1; by <= ey1 + P; ++by) flush(by);
  mf_finish<KK, NT>(a, dots);
}

// Host launcher of one (P) instantiation; defined in matfree_p<P>.cu.
template <int P>
void mf_launch_p(const SpmvArgs& a, cudaStream_t s);

}  // namespace ga
