// Host-side (CPU) setup arithmetic of the CUDA path: knot vector, Gauss rule,
// B-spline tables, 1D parametric mass matrices and their banded Cholesky
// factors, generalized-alpha parameters.  Independent of oracle/ (no shared
// code); cited to PAPER.md (P:line).
#pragma once
#include <vector>

namespace ga {

// Open uniform knot vector, n elements, degree p (maximal regularity P:811).
std::vector<double> open_knots(int p, int n);

// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on P_q (q points).
void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w);

// Values (der=0) or first derivatives (der=1) of the p+1 B-splines that are
// non-zero on element e (global indices e..e+p) at parameter x, by the
// Cox-de Boor recursion with 0/0 = 0.
void local_basis(const std::vector<double>& knots, int p, int e, double x, double* val, double* der);

// 1D tables at the n(p+1) Gauss points (element-major):
//   val[q*(p+1)+a], der[...] for local function a (global e+a), wq[q] weight*jacobian.
struct Tables1D {
  int p = 0, n = 0, nq = 0, m = 0;
  std::vector<double> pts, wq, val, der;
};
Tables1D make_tables(int p, int n);

// Dense-band 1D parametric mass matrix Mh[i][i+t], t = 0..p over all m functions.
std::vector<double> param_mass_band(const Tables1D& T);  // size m*(p+1)

// Banded Cholesky of the restriction of Mh to indices [lo, hi] (inclusive).
// Output per row i (local): L[i*(p+1)+0] = 1/L_ii, L[i*(p+1)+t] = L_{i,i-t}.
// Also returns diag of the restricted Mh.
bool band_cholesky(const std::vector<double>& band, int p, int lo, int hi,
                   std::vector<double>& L, std::vector<double>& diag);

// Generalized-alpha parameters (R2).
int scheme_params(int k, double rb, double rs, int param_set,
                  double* alpha, double* beta, double* gamma, double* alpha_f, double* theta_max);

}  // namespace ga

namespace ga {

// Chunked form of one triangular sweep y_i = (t_i - sum_{u=1..p} c_{i,u} y_{i-u}) * dinv_i
// over a line of length n: the line is cut into C
// chunks of length clen >= p; chunk w is solved locally from a zero incoming
// state and corrected with the precomputed homogeneous responses H of its p
// incoming values; the incoming states follow from an affine recurrence
// sigma_{w+1} = T_w sigma_w + tau_w solved by a Kogge-Stone scan whose
// (data-independent) matrix products A^(l)_w are precomputed here.
// Device buffer layout (doubles): dinv[n] | coef[n][p] | H[n][p] | A[L][C][p][p]
struct SweepFactor {
  int n = 0, p = 0, clen = 0, C = 0, L = 0;
  std::vector<double> buf;
};
// From the band Cholesky rows (L[i*(p+1)+0] = 1/L_ii, L[i*(p+1)+u] = L_{i,i-u}):
// backward = false: forward sweep L y = t; true: backward sweep L^T z = y
// written as a forward sweep on the reversed line.
SweepFactor make_sweep(const std::vector<double>& Lrows, int n, int p, bool backward, int chunks_target = 32);

// Sequential form of both sweeps for the whole-line shared-memory solver (line_seq.cu): the
// divisions are folded into the band, y_i = t_i d_i - sum_{u=1..p} e_{i,u} y_{i-u} with
// e_{i,u} = c_{i,u} d_i, so one FMA per element is on the recurrence's critical path.
// Layout (doubles): forward rows [n][PP] = {d_i, e_{i,1..p}, 0 pad}, then the backward rows of the
// reversed line [n][PP]; PP = seq_row(p) (p + 1 rounded up to even: 16-byte rows).
inline int seq_row(int p) { return (p + 2) & ~1; }
std::vector<double> make_seq(const std::vector<double>& Lrows, int n, int p);

}  // namespace ga
