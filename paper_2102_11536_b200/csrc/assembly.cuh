// GPU assembly (sum-factorised Gauss quadrature) — launcher declarations.
#pragma once
#include <cuda_runtime.h>

namespace ga {

struct AsmPatch {
  int p, n, m, nq;         // degree, elements, functions (n+p), Gauss points n(p+1) per direction
  const double* ctrl;      // device, m^dim points x dim
  const double* val;       // device, [nq][p+1] basis values of the p+1 local functions
  const double* der;       // device, [nq][p+1] derivatives
  const double* wq;        // device, [nq] Gauss weight x element length
};

// One quadrature term W(q): kind 0 = scale*w|J| (mass), 1 = scale*w|J| (J^-1 J^-T)_{ce}
// (scalar stiffness), 2 = elastic block (a,b), derivative pair (c,e).
struct TermSpec {
  int kind, a, b, c, e;
  double scale, lam, mu;
};

struct ContractDesc {
  long long nouter, nmid, ninner;
  long long in_s_outer, in_s_q, in_s_mid, in_s_inner;
  long long out_s_outer, out_s_o, out_s_mid, out_s_i, out_s_inner;
  int W1, m, p, n, qoff;
};

struct FinalDesc {
  int W1, m, p, n, qoff, r0, r1;
  int cell[3];
  int org[3];                  // grid coordinate = cell (m - 1) + local index - org (1: Dirichlet ring)
  int G[3];
  long long npts;
  long long S;                 // offsets per coefficient array
  int ncf, ab;                 // coefficient arrays per row slice (1 or 9) and the target block
  const unsigned char* mask;
  int half;                    // half-symmetric layout: offsets o >= 0 only, rows shifted by hguard
  long long hguard;
  int sym, sxs, snseg;         // 3D scalar half layout: segment-blocked (common.cuh sym_index)
  // boundary apply (Dirichlet lifting): instead of storing coefficients, accumulate
  // bout[row] += A(row, col) bg[col] over the boundary columns col (patch-local full index)
  const double* bg;
  double* bout;
};

void launch_geometry(const AsmPatch& P, int dim, int qa, int nqs, double* geo, long long gstride, double* minmax,
                     cudaStream_t s);
void launch_wterm(const double* geo, long long gstride, long long npts, int dim, const TermSpec& T, double* W,
                  cudaStream_t s);
void launch_contract(const double* in, double* out, const double* A, const ContractDesc& c, cudaStream_t s);
void launch_contract_final(int dim, const double* in, const double* A, const FinalDesc& f, double* coef,
                           cudaStream_t s);

}  // namespace ga
