// Host-side launch of the matrix-free operator for one degree P (included by
// matfree_p<P>.cu): tile shape, z (or y) chunking, right-hand-side sub-batches
// of <= 2 (so the shared-memory footprint stays inside one SM), and the
// fixed-order partial-sum finish for the PCG modes.
#pragma once
#include <algorithm>

#include "matfree_core.cuh"

namespace ga {

constexpr size_t MF_SMEM_MAX = 227 * 1024;
constexpr size_t MF_SMEM_SM = 228 * 1024;

template <int P, int KK, bool STIFF>
static unsigned int mf3_go(const SpmvArgs& a, cudaStream_t s, bool launch) {
  constexpr int DX = 8, DY = 8;
  using L = Mf3Shape<P, KK, STIFF, DX, DY>;
  // one thread per (x Gauss point, rhs) of the y walk (phase c), rounded to warps, >= 128
  constexpr int NTW = ((L::QX * KK + 31) / 32) * 32;
  constexpr int NT = NTW < 128 ? 128 : NTW;
  if constexpr (L::BYTES > MF_SMEM_MAX) {
    return 0;
  } else {
    const GridDesc g = a.g;
    const int tx = (g.nx + DX - 1) / DX, ty = (g.ny + DY - 1) / DY;
    const long long tiles = (long long)tx * ty * a.nvec;
    // chunking from the 1-rhs footprint: every sub-batch must use the same blocks (partial sums)
    const int occ = std::max(1, std::min(2048 / 128, (int)(MF_SMEM_SM / (Mf3Shape<P, 1, STIFF, DX, DY>::BYTES + 1024))));
    const long long target = 2LL * 148 * occ;
    int nzc = (int)std::min<long long>((target + tiles - 1) / tiles, std::max(1, g.nz / (2 * P)));
    nzc = std::max(1, nzc);
    const int ZL = (g.nz + nzc - 1) / nzc;
    nzc = (g.nz + ZL - 1) / ZL;
    if (launch) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_mf3<P, KK, STIFF, DX, DY, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)L::BYTES);
        attr = true;
      }
      dim3 grid(tx, ty, nzc * a.nvec);
      k_mf3<P, KK, STIFF, DX, DY, NT><<<grid, NT, L::BYTES, s>>>(a, ZL, nzc);
    }
    return (unsigned int)(tiles * nzc);
  }
}

template <int P, int KK, bool STIFF>
static unsigned int mf2_go(const SpmvArgs& a, cudaStream_t s, bool launch) {
  constexpr int DX = 128, NT = 256;
  using L = Mf2Shape<P, KK, STIFF, DX>;
  const GridDesc g = a.g;
  const int tx = (g.nx + DX - 1) / DX;
  const long long tiles = (long long)tx * a.nvec;
  const int occ = std::max(1, std::min(2048 / NT, (int)(MF_SMEM_SM / (Mf2Shape<P, 1, STIFF, DX>::BYTES + 1024))));
  const long long target = 2LL * 148 * occ;
  int nyc = (int)std::min<long long>((target + tiles - 1) / tiles, std::max(1, g.ny / (2 * P)));
  nyc = std::max(1, nyc);
  const int YL = (g.ny + nyc - 1) / nyc;
  nyc = (g.ny + YL - 1) / YL;
  if (launch) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_mf2<P, KK, STIFF, DX, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
      attr = true;
    }
    dim3 grid(tx, nyc * a.nvec);
    k_mf2<P, KK, STIFF, DX, NT><<<grid, NT, L::BYTES, s>>>(a, YL, nyc);
  }
  return (unsigned int)(tiles * nyc);
}

template <int P, int KK>
static unsigned int mf_go(const SpmvArgs& a, cudaStream_t s, bool launch) {
  if (a.g.dim == 3) return a.mfstiff ? mf3_go<P, KK, true>(a, s, launch) : mf3_go<P, KK, false>(a, s, launch);
  return a.mfstiff ? mf2_go<P, KK, true>(a, s, launch) : mf2_go<P, KK, false>(a, s, launch);
}

template <int P>
void mf_launch_p(const SpmvArgs& a, cudaStream_t s) {
  // right-hand sides in sub-batches of 2 (1 where two do not fit in shared memory)
  const bool two_fit = mf_go<P, 2>(a, s, false) > 0;
  SpmvArgs b = a;
  unsigned int nb = 0;
  for (int j0 = 0; j0 < a.kk;) {
    b.mfj0 = j0;
    if (two_fit && a.kk - j0 >= 2) {
      nb = mf_go<P, 2>(b, s, true);
      j0 += 2;
    } else {
      nb = mf_go<P, 1>(b, s, true);
      j0 += 1;
    }
  }
  if (a.mode == SPMV_PQ || a.mode == SPMV_TRUERES) launch_spmv_fin(a, nb, s);
}

}  // namespace ga
