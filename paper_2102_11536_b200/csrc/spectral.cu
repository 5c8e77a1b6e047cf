// Batched spectral radius of the amplification matrix G(Theta) (PAPER.md
// §3.2, §4.1, P:281 Theta = tau^2 lambda): one thread per Theta.  For one mode (M = 1, K = Theta,
// tau = 1) block j's new variables depend only on chain entries m >= 3j-3, so G is block upper
// triangular with the 3x3 diagonal blocks Lambda_j; the block of j is obtained by
// stepping its three unit vectors through the step of P:408-431 (reading R1: s_j = T_{3j-3} for
// j < k, c_{3k-3} for j = k), and rho(G) = max_j of the largest root modulus of det(mu - Lambda_j),
// a cubic solved in closed form (Cardano / trigonometric).
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/genalpha.h"
#include "host_math.h"

namespace ga {

struct ScanArgs {
  int k;
  double alpha[4], beta[4], gamma[4];
  const double* theta;
  double* rho;
  int n;
};

__device__ double cubic_max_modulus(double a, double b, double c) {
  // roots of mu^3 + a mu^2 + b mu + c, max |mu|
  const double a3 = a / 3.0;
  const double p = b - a * a3;                         // depressed t^3 + p t + q, mu = t - a/3
  const double q = 2.0 * a3 * a3 * a3 - a3 * b + c;
  const double disc = 0.25 * q * q + p * p * p / 27.0;
  if (disc > 0.0) {
    const double sd = sqrt(disc);
    const double u = cbrt(-0.5 * q + sd), v = cbrt(-0.5 * q - sd);
    const double r1 = u + v - a3;                     // real root
    const double re = -0.5 * (u + v) - a3, im = 0.5 * sqrt(3.0) * (u - v);
    return fmax(fabs(r1), sqrt(re * re + im * im));
  }
  // three real roots (p <= 0)
  const double m = 2.0 * sqrt(fmax(-p / 3.0, 0.0));
  double arg = (m > 0.0) ? (3.0 * q / (p * m)) : 0.0;  // cos(3 phi)
  arg = fmin(1.0, fmax(-1.0, arg));
  const double phi = acos(arg) / 3.0;
  double best = 0.0;
  for (int i = 0; i < 3; ++i) {
    const double r = m * cos(phi - 2.0943951023931953 * i) - a3;
    best = fmax(best, fabs(r));
  }
  return best;
}

__global__ void k_spectral_scan(ScanArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double th = a.theta[i];
  double rho = 0.0;
  for (int j = 0; j < a.k; ++j) {
    double B[3][3];
    for (int col = 0; col < 3; ++col) {
      const double cd = col == 0, cv = col == 1, ca = col == 2;  // unit vector in block j
      const double Td = cd + cv + 0.5 * ca, Tv = cv + ca, Ta = ca;  // Taylor with tau = 1
      const double s = (j < a.k - 1) ? Td : cd;
      const double y = -th * s;
      const double P = (y - Ta) / a.alpha[j];
      B[0][col] = Td + a.beta[j] * P;
      B[1][col] = Tv + a.gamma[j] * P;
      B[2][col] = Ta + P;
    }
    const double tr = B[0][0] + B[1][1] + B[2][2];
    const double m2 = B[0][0] * B[1][1] - B[0][1] * B[1][0] + B[0][0] * B[2][2] - B[0][2] * B[2][0] +
                      B[1][1] * B[2][2] - B[1][2] * B[2][1];
    const double det = B[0][0] * (B[1][1] * B[2][2] - B[1][2] * B[2][1]) -
                       B[0][1] * (B[1][0] * B[2][2] - B[1][2] * B[2][0]) +
                       B[0][2] * (B[1][0] * B[2][1] - B[1][1] * B[2][0]);
    rho = fmax(rho, cubic_max_modulus(-tr, m2, -det));
  }
  a.rho[i] = rho;
}

}  // namespace ga

extern "C" ga_status ga_spectral_scan(int k, double rho_b, double rho_s, int param_set, const double* d_theta, int n,
                                      double* d_rho, void* stream) {
  using namespace ga;
  if (k < 1 || k > 4 || n < 0 || (n > 0 && (!d_theta || !d_rho))) return GA_ERR_ARG;
  if (param_set != 0 && param_set != 1) return GA_ERR_ARG;
  ScanArgs a;
  double af[4], th;
  if (scheme_params(k, rho_b, rho_s, param_set, a.alpha, a.beta, a.gamma, af, &th) != 0) return GA_ERR_PARAM;
  a.k = k; a.theta = d_theta; a.rho = d_rho; a.n = n;
  if (n == 0) return GA_OK;
  k_spectral_scan<<<(unsigned int)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? GA_OK : GA_ERR_CUDA;
}
