// Dispatcher of the matrix-free operator (per-degree instantiations in
// matfree_p<P>.cu) and diag(M) for the preconditioner scaling.
#include <cuda_runtime.h>

#include "matfree_core.cuh"

namespace ga {

extern template void mf_launch_p<1>(const SpmvArgs&, cudaStream_t);
extern template void mf_launch_p<2>(const SpmvArgs&, cudaStream_t);
extern template void mf_launch_p<3>(const SpmvArgs&, cudaStream_t);
extern template void mf_launch_p<4>(const SpmvArgs&, cudaStream_t);
extern template void mf_launch_p<5>(const SpmvArgs&, cudaStream_t);
extern template void mf_launch_p<6>(const SpmvArgs&, cudaStream_t);
extern template void mf_launch_p<7>(const SpmvArgs&, cudaStream_t);

void launch_matfree(const SpmvArgs& a, cudaStream_t s) {
  if (a.g.dim == 3 && !a.mfstiff && a.mpT1) {  // non-redundant multi-pass mass apply
    launch_matfree_mp(a, s);
    return;
  }
  switch (a.p) {
    case 1: mf_launch_p<1>(a, s); break;
    case 2: mf_launch_p<2>(a, s); break;
    case 3: mf_launch_p<3>(a, s); break;
    case 4: mf_launch_p<4>(a, s); break;
    case 5: mf_launch_p<5>(a, s); break;
    case 6: mf_launch_p<6>(a, s); break;
    default: mf_launch_p<7>(a, s); break;
  }
}

// diag(M)_i = sum_q W(q) prod_d N_{i_d}(q_d)^2, one thread per grid point (setup only).
template <int DIM>
__global__ void k_mf_diag(GridDesc g, int p, int n, const double* __restrict__ W, const double* __restrict__ tv,
                          double* __restrict__ diag) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.npts) return;
  const int pp1 = p + 1;
  const long long nq = (long long)n * pp1;
  int b[3];
  b[0] = (int)(i % g.nx) + 1;
  b[1] = (int)((i / g.nx) % g.ny) + 1;
  b[2] = DIM == 3 ? (int)(i / ((long long)g.nx * g.ny)) + 1 : 0;
  double sum = 0.0;
  const int ezlo = DIM == 3 ? max(0, b[2] - p) : 0, ezhi = DIM == 3 ? min(n - 1, b[2]) : 0;
  for (int ez = ezlo; ez <= ezhi; ++ez)
    for (int qz = 0; qz < (DIM == 3 ? pp1 : 1); ++qz) {
      const long long qzg = (long long)ez * pp1 + qz;
      const double nz = DIM == 3 ? tv[qzg * pp1 + (b[2] - ez)] : 1.0;
      double sy = 0.0;
      for (int ey = max(0, b[1] - p); ey <= min(n - 1, b[1]); ++ey)
        for (int qy = 0; qy < pp1; ++qy) {
          const long long qyg = (long long)ey * pp1 + qy;
          const double ny = tv[qyg * pp1 + (b[1] - ey)];
          double sx = 0.0;
          for (int ex = max(0, b[0] - p); ex <= min(n - 1, b[0]); ++ex)
            for (int qx = 0; qx < pp1; ++qx) {
              const long long qxg = (long long)ex * pp1 + qx;
              const double nx = tv[qxg * pp1 + (b[0] - ex)];
              sx = fma(nx * nx, W[((DIM == 3 ? qzg * nq : 0) + qyg) * nq + qxg], sx);
            }
          sy = fma(ny * ny, sx, sy);
        }
      sum = fma(nz * nz, sy, sum);
    }
  diag[i] = sum;
}

void launch_mf_diag(const GridDesc& g, int p, int n, const double* W, const double* tv, double* diag,
                    cudaStream_t s) {
  const unsigned int nb = (unsigned int)((g.npts + 127) / 128);
  if (g.dim == 3) k_mf_diag<3><<<nb, 128, 0, s>>>(g, p, n, W, tv, diag);
  else k_mf_diag<2><<<nb, 128, 0, s>>>(g, p, n, W, tv, diag);
}

}  // namespace ga
