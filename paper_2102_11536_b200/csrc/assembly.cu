// GPU assembly of M and K into the column-index-free stencil layout
// coef[row/32][ab][o][row%32] (o in [-p,p]^d, lexicographic, x fastest; row = global grid
// point), by global sum factorisation over the tensor Gauss grid.
//
// Definitions (weak form of P:57; elasticity DESIGN.md "Elasticity"):
//   M_ij   = sum_q w|J| B_i B_j
//   K_ij   = sum_q w|J| omega^2 sum_f (J^-T grad B_i)_f (J^-T grad B_j)_f
//   K^{ab}_ij = sum_q w|J| [lam d_aB_i d_bB_j + mu d_bB_i d_aB_j + mu delta_ab grad B_i.grad B_j]
// Each is a sum of "terms" sum_q W(q) prod_d A_d(i_d, o_d, q_d), with
// A_d(i, o, q) = phi^{(s_d)}_i(q) phi^{(t_d)}_{i+o}(q) the 1D product of basis
// values (s,t = 0) or derivatives (s,t = 1).  The d-fold sum over q is done as
// d banded contractions (one per direction), slab by slab along the outermost
// direction so that the scratch fits any given budget.
#include <cuda_runtime.h>

#include "assembly.cuh"
#include "common.cuh"

namespace ga {

// geo[0] = w|J|, geo[1 + c*dim + a] = (J^{-1})_{ca};  one thread per Gauss point of the slab
template <int DIM>
__global__ void k_geometry(AsmPatch P, int qa, int nqs, double* __restrict__ geo, long long gstride,
                           double* __restrict__ minmax) {
  const int p = P.p, pp1 = p + 1, nq = P.nq, m = P.m;
  const long long npts = (long long)nq * (DIM == 3 ? (long long)nq * nqs : nqs);
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double det = 1e300;
  if (e < npts) {
    int q[3];
    q[0] = (int)(e % nq);
    if (DIM == 3) {
      q[1] = (int)((e / nq) % nq);
      q[2] = qa + (int)(e / ((long long)nq * nq));
    } else {
      q[1] = qa + (int)(e / nq);
      q[2] = 0;
    }
    double J[DIM][DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) J[a][b] = 0.0;
    int el[3];
    for (int d = 0; d < DIM; ++d) el[d] = q[d] / pp1;
    const double* v0 = P.val + (long long)q[0] * pp1;
    const double* d0 = P.der + (long long)q[0] * pp1;
    const double* v1 = P.val + (long long)q[1] * pp1;
    const double* d1 = P.der + (long long)q[1] * pp1;
    const double* v2 = P.val + (long long)q[2] * pp1;
    const double* d2 = P.der + (long long)q[2] * pp1;
    const int a3max = DIM == 3 ? p : 0;
    for (int a3 = 0; a3 <= a3max; ++a3) {
      for (int a2 = 0; a2 <= p; ++a2) {
        for (int a1 = 0; a1 <= p; ++a1) {
          long long idx = (el[0] + a1) + (long long)m * ((el[1] + a2) + (DIM == 3 ? (long long)m * (el[2] + a3) : 0));
          double g[DIM];
          if (DIM == 3) {
            g[0] = d0[a1] * v1[a2] * v2[a3];
            g[1] = v0[a1] * d1[a2] * v2[a3];
            g[2] = v0[a1] * v1[a2] * d2[a3];
          } else {
            g[0] = d0[a1] * v1[a2];
            g[1] = v0[a1] * d1[a2];
          }
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            const double C = P.ctrl[idx * DIM + a];
#pragma unroll
            for (int b = 0; b < DIM; ++b) J[a][b] = fma(C, g[b], J[a][b]);
          }
        }
      }
    }
    double inv[DIM][DIM];
    if (DIM == 3) {
      inv[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      inv[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
      inv[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
      inv[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      inv[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
      inv[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
      inv[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      inv[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
      inv[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      det = J[0][0] * inv[0][0] + J[0][1] * inv[1][0] + J[0][2] * inv[2][0];
    } else {
      inv[0][0] = J[1][1];
      inv[0][1] = -J[0][1];
      inv[1][0] = -J[1][0];
      inv[1][1] = J[0][0];
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    }
    double w = P.wq[q[0]] * P.wq[q[1]] * (DIM == 3 ? P.wq[q[2]] : 1.0);
    geo[e] = w * det;
    const double id = 1.0 / det;
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int a = 0; a < DIM; ++a) geo[(1 + c * DIM + a) * gstride + e] = inv[c][a] * id;
  }
  // block min of |J| (for GA_ERR_GEOMETRY)
  __shared__ double sm[32];
  for (int o = 16; o > 0; o >>= 1) det = fmin(det, __shfl_xor_sync(0xffffffffu, det, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = det;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mn = sm[0];
    for (int w = 1; w < (int)(blockDim.x + 31) / 32; ++w) mn = fmin(mn, sm[w]);
    // atomic min on a double via CAS
    unsigned long long* addr = (unsigned long long*)minmax;
    unsigned long long old = *addr, assumed;
    do {
      assumed = old;
      if (__longlong_as_double(assumed) <= mn) break;
      old = atomicCAS(addr, assumed, __double_as_longlong(mn));
    } while (assumed != old);
  }
}

// W(q) of one term from the geometry buffer.
__global__ void k_wterm(const double* __restrict__ geo, long long gstride, long long npts, int dim, TermSpec T,
                        double* __restrict__ W) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= npts) return;
  const double wd = geo[e];
  auto Ji = [&](int c, int a) { return geo[(1 + c * dim + a) * gstride + e]; };
  double v;
  if (T.kind == 0) {
    v = T.scale * wd;
  } else if (T.kind == 1) {
    double s = 0.0;
    for (int f = 0; f < dim; ++f) s = fma(Ji(T.c, f), Ji(T.e, f), s);
    v = T.scale * wd * s;
  } else {
    double s = 0.0;
    if (T.a == T.b)
      for (int f = 0; f < dim; ++f) s = fma(Ji(T.c, f), Ji(T.e, f), s);
    v = wd * (T.lam * Ji(T.c, T.a) * Ji(T.e, T.b) + T.mu * Ji(T.c, T.b) * Ji(T.e, T.a) + T.mu * s);
  }
  W[e] = v;
}

// Banded contraction of one direction (intermediate stages):
//   out[outer][o][mid][i][inner] = sum_{q in supp(i)} A[i][o][q - qs(i)] in[outer][q - qoff][mid][inner]
__global__ void k_contract(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ A,
                           ContractDesc c) {
  const long long tot = (long long)c.nouter * c.W1 * c.nmid * c.m * c.ninner;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  long long r = e;
  const long long inner = r % c.ninner; r /= c.ninner;
  const int i = (int)(r % c.m); r /= c.m;
  const long long mid = r % c.nmid; r /= c.nmid;
  const int o = (int)(r % c.W1); r /= c.W1;
  const long long outer = r;
  const int pp1 = c.p + 1;
  const int qs = max(0, i - c.p) * pp1, qe = (min(c.n - 1, i) + 1) * pp1;
  const double* Ai = A + ((long long)i * c.W1 + o) * pp1 * pp1;
  const double* src = in + outer * c.in_s_outer + mid * c.in_s_mid + inner * c.in_s_inner;
  double s = 0.0;
  for (int q = qs; q < qe; ++q) s = fma(__ldg(Ai + (q - qs)), __ldg(src + (long long)(q - c.qoff) * c.in_s_q), s);
  out[outer * c.out_s_outer + o * c.out_s_o + mid * c.out_s_mid + (long long)i * c.out_s_i + inner * c.out_s_inner] = s;
}

// Last direction: contract the outer quadrature index for rows i_out in
// [r0, r1) and add the result into the global stencil arrays at (o, grid row)
// when both the row and the column i+o are free points of the global grid.
//   in: X[qs][o_lower...][i_lower...] with lower = the other d-1 directions
template <int DIM>
__global__ void k_contract_final(const double* __restrict__ in, const double* __restrict__ A, FinalDesc f,
                                 double* __restrict__ coef) {
  const int W1 = f.W1, m = f.m, pp1 = f.p + 1;
  const long long nlow_i = (DIM == 3) ? (long long)m * m : m;
  const long long nlow_o = (DIM == 3) ? (long long)W1 * W1 : W1;
  const int nrows = f.r1 - f.r0;
  const long long tot = (long long)nrows * W1 * nlow_o * nlow_i;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  long long r = e;
  const long long il = r % nlow_i; r /= nlow_i;
  const long long ol = r % nlow_o; r /= nlow_o;
  const int o_out = (int)(r % W1); r /= W1;
  const int i_out = f.r0 + (int)r;
  int ii[3], oo[3];
  ii[0] = (int)(il % m);
  oo[0] = (int)(ol % W1) - f.p;
  if (DIM == 3) {
    ii[1] = (int)(il / m);
    oo[1] = (int)(ol / W1) - f.p;
    ii[2] = i_out;
    oo[2] = o_out - f.p;
  } else {
    ii[1] = i_out;
    oo[1] = o_out - f.p;
    ii[2] = 0; oo[2] = 0;
  }
  // global grid coordinates (interior coords: Dirichlet ring removed)
  long long grow = 0, gcol_ok = 1, rmul = 1;
  int gr[3], gc[3];
  for (int d = 0; d < DIM; ++d) {
    gr[d] = f.cell[d] * (m - 1) + ii[d] - f.org[d];
    gc[d] = gr[d] + oo[d];
    if (gr[d] < 0 || gr[d] >= f.G[d]) return;
    if (gc[d] < 0 || gc[d] >= f.G[d]) gcol_ok = 0;
  }
  if (f.bout) {
    // boundary apply: only columns outside the free grid but inside the patch (boundary bases)
    if (gcol_ok) return;
    long long cl = 0, mul = 1;
    for (int d = 0; d < DIM; ++d) {
      const int cf = ii[d] + oo[d];  // patch-local full index of the column
      if (cf < 0 || cf > m - 1) return;
      cl += cf * mul;
      mul *= m;
    }
    grow = gr[0] + (long long)f.G[0] * (gr[1] + (DIM == 3 ? (long long)f.G[1] * gr[2] : 0));
    const int qs = max(0, i_out - f.p) * pp1, qe = (min(f.n - 1, i_out) + 1) * pp1;
    const double* Ai = A + ((long long)i_out * W1 + o_out) * pp1 * pp1;
    const double* src = in + ol * nlow_i + il;
    const long long sq = nlow_o * nlow_i;
    double sb = 0.0;
    for (int q = qs; q < qe; ++q) sb = fma(__ldg(Ai + (q - qs)), __ldg(src + (long long)(q - f.qoff) * sq), sb);
    atomicAdd(f.bout + grow, sb * f.bg[cl]);
    return;
  }
  if (!gcol_ok) return;
  grow = gr[0] + (long long)f.G[0] * (gr[1] + (DIM == 3 ? (long long)f.G[1] * gr[2] : 0));
  const long long gcol = gc[0] + (long long)f.G[0] * (gc[1] + (DIM == 3 ? (long long)f.G[1] * gc[2] : 0));
  if (f.mask && (!f.mask[grow] || !f.mask[gcol])) return;
  (void)rmul;
  // sum over the outer quadrature index
  const int qs = max(0, i_out - f.p) * pp1, qe = (min(f.n - 1, i_out) + 1) * pp1;
  const double* Ai = A + ((long long)i_out * W1 + o_out) * pp1 * pp1;
  const double* src = in + ol * nlow_i + il;
  const long long sq = nlow_o * nlow_i;
  double s = 0.0;
  for (int q = qs; q < qe; ++q) s = fma(__ldg(Ai + (q - qs)), __ldg(src + (long long)(q - f.qoff) * sq), s);
  // stencil offset index, lexicographic with x fastest
  long long olin = (oo[0] + f.p) + (long long)W1 * ((oo[1] + f.p) + (DIM == 3 ? (long long)W1 * (oo[2] + f.p) : 0));
  if (f.half) {  // o >= 0 only (index o - S/2), rows shifted by the zero guard
    const long long Sh = (f.S + 1) / 2, hl = olin - f.S / 2;
    if (hl < 0) return;
    if (f.sym) {
      coef[sym_index(gr[0], gr[1], DIM == 3 ? gr[2] : 0, hl, f.sxs, f.snseg, f.G[1], Sh)] += s;
      return;
    }
    const long long rr = grow + f.hguard;
    coef[((rr >> 5) * Sh + hl) * 32 + (rr & 31)] += s;
    return;
  }
  // blocked layout: 32-row slices, all NCF*S offsets of a slice contiguous
  coef[((grow >> 5) * f.ncf * f.S + (long long)f.ab * f.S + olin) * 32 + (grow & 31)] += s;
}

static inline unsigned int nblk(long long n) { return (unsigned int)((n + 255) / 256); }

void launch_geometry(const AsmPatch& P, int dim, int qa, int nqs, double* geo, long long gstride, double* minmax,
                     cudaStream_t s) {
  const long long npts = (long long)P.nq * (dim == 3 ? (long long)P.nq * nqs : nqs);
  if (dim == 3) k_geometry<3><<<nblk(npts), 256, 0, s>>>(P, qa, nqs, geo, gstride, minmax);
  else k_geometry<2><<<nblk(npts), 256, 0, s>>>(P, qa, nqs, geo, gstride, minmax);
}
void launch_wterm(const double* geo, long long gstride, long long npts, int dim, const TermSpec& T, double* W,
                  cudaStream_t s) {
  k_wterm<<<nblk(npts), 256, 0, s>>>(geo, gstride, npts, dim, T, W);
}
void launch_contract(const double* in, double* out, const double* A, const ContractDesc& c, cudaStream_t s) {
  const long long tot = (long long)c.nouter * c.W1 * c.nmid * c.m * c.ninner;
  k_contract<<<nblk(tot), 256, 0, s>>>(in, out, A, c);
}
void launch_contract_final(int dim, const double* in, const double* A, const FinalDesc& f, double* coef,
                           cudaStream_t s) {
  const long long nlow = (dim == 3) ? (long long)f.W1 * f.W1 * f.m * f.m : (long long)f.W1 * f.m;
  const long long tot = (long long)(f.r1 - f.r0) * f.W1 * nlow;
  if (tot <= 0) return;
  if (dim == 3) k_contract_final<3><<<nblk(tot), 256, 0, s>>>(in, A, f, coef);
  else k_contract_final<2><<<nblk(tot), 256, 0, s>>>(in, A, f, coef);
}

}  // namespace ga
