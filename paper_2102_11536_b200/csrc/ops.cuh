// Hot-path kernels (stencil SpMV, Kronecker line solves, PCG vector ops,
// stage update) — declarations of the host-side launchers.
#pragma once
#include "common.cuh"

namespace ga {

enum SpmvMode { SPMV_APPLY = 0, SPMV_NEGB = 1, SPMV_PQ = 2, SPMV_TRUERES = 3 };

// Multi-vector (MV) layout: element (comp c, grid point i, rhs j) at
//   ((c * padded + guard + i) * kk + j)
struct SpmvArgs {
  const double* coef;  // scalar: [S][npts]; elastic: [9][S][npts]
  const double* x;
  double* y;
  const double* b;     // SPMV_TRUERES
  GridDesc g;
  int nvec;            // component vectors per MV (1 or 3)
  int kk;              // rhs per MV
  int p;
  int elastic;         // 1: 3x3 block stencil
  int mode;
  int fuse_p;          // SPMV_PQ: form p = z + beta p_old on the fly (x is ignored)
  const double* z;
  double *p0, *p1;     // fuse_p: p_old (read) and p_new (written) direction buffers
  double fbeta[KMAX];  // fuse_p: beta of this iteration
  int fpfirst;         // fuse_p: first iteration of the phase (p = z)
  double* fx;          // fuse_p and not first: also x += falpha p_old (the x update deferred from
  double falpha[KMAX]; //   the previous iteration's preconditioner), null: off
  double tol2, refine_rtol2;  // SPMV_TRUERES: thresholds of the refinement phase
  PcgState* pcg;
  DevStatus* st;
  double* partial;
  unsigned int* counter;
  // matrix-free sum-factorised operator (mf = 1; coef unused), single patch, scalar M / K
  // or the elastic mass (density * scalar M per component), DESIGN.md "Matrix-free operator"
  int mf;              // 1: apply by sum factorisation from the quadrature data
  int mfstiff;         // 0: mass  sum_q W B_i B_j ;  1: stiffness sum_q grad^T B_i W grad B_j
  int mfn;             // elements per direction
  int mfj0;            // first right-hand side of this launch (sub-batches of <= 2 rhs)
  const double* mfW;   // mass: W[nq^d]; stiffness: d(d+1)/2 symmetric entries, SoA with stride mfws
  long long mfws;      // nq^d, nq = n (p+1) (global tensor Gauss grid, x fastest)
  const double* mfv;   // 1D basis values  [nq][p+1]  (local function a of element q/(p+1))
  const double* mfd;   // 1D derivatives   [nq][p+1]
  // half-symmetric stencil (half = 1): offsets o >= 0 only, rows shifted by a zero guard of
  // hguard rows (spmv_core.cuh spmv_block_half); not for the elastic (3x3-block) K
  int half;
  long long hguard;
  // 3D scalar half-symmetric operators in the segment-blocked layout of the single-read SpMV
  // (sym = 1, spmv_sym.cu): XS points per x-segment, nseg segments per x-line
  int sym, sxs, snseg;
  const double* symzero;  // zero block of Sh x 32 doubles (loads of unstored / outside rows)
  // 3D matrix-free mass by the multi-pass non-redundant sum factorisation (matfree_mp.cu):
  // intermediates T1 [c][n_q][nf][nf][k], T2 / T3 [c][n_q][n_q][nf][k]
  double *mpT1, *mpT2, *mpT3;
  // subdomain group (dist.cu): SPMV_PQ writes its local p.q sums here (k_spmv_fin) instead of
  // taking the PCG scalar step, which runs after the exchange (null: ordinary context)
  double* xsum;
  // masked grids (multi-patch): skip[rb] = 1 if none of the 32 rows of row block rb is free (its
  // rows and columns are zero, and every vector is zero there): the warp of that block does
  // nothing.  C5: the [1,2]^2 quadrant of the L-shape's bounding grid, 25 % of the row blocks.
  const unsigned char* skip;
};
void launch_spmv(const SpmvArgs& a, cudaStream_t s);
void launch_spmv_sym(const SpmvArgs& a, cudaStream_t s);  // a.sym = 1 (spmv_sym.cu)
// matrix-free variants (matfree.cu): the same contract as launch_spmv for a.mf = 1
void launch_matfree(const SpmvArgs& a, cudaStream_t s);
void launch_matfree_mp(const SpmvArgs& a, cudaStream_t s);  // 3D mass, multi-pass (a.mpT1 != null)
// fixed-order sum of nb block partials + the PCG scalar step (SPMV_PQ / SPMV_TRUERES)
void launch_spmv_fin(const SpmvArgs& a, unsigned int nb, cudaStream_t s);
// diag(M) of the matrix-free mass operator on the single-patch grid, diag[npts]
void launch_mf_diag(const GridDesc& g, int p, int n, const double* W, const double* tv, double* diag,
                    cudaStream_t s);

struct PrecArgs {
  GridDesc g;
  int nvec, kk, p;
  int npatch;
  // per patch box in grid coordinates
  int lo[MAXPATCH][3];
  int bd[MAXPATCH][3];
  const double* s[MAXPATCH];      // scaling sqrt(Dh/D) on the box (0 on masked points)
  double* t[MAXPATCH];            // box work arrays [c][box][kk] (single patch: nullptr, uses z)
  const double* L[MAXPATCH][3];   // banded Cholesky factors per direction, (len+p) rows of p+1
  const double* Ff[MAXPATCH][3];  // chunked sweep factors (host_math.h SweepFactor), forward
  const double* Fb[MAXPATCH][3];  // and backward (reversed line)
  int clen[MAXPATCH][3], nchunk[MAXPATCH][3], nlev[MAXPATCH][3], flen[MAXPATCH][3];
  const double* E[MAXPATCH][3];   // sequential sweep rows (host_math.h make_seq), whole-line solver
  const unsigned char* mask;      // grid mask (nullptr: all free)
  // PCG vectors (MV)
  double *x, *r, *z;
  const double *p0, *p1, *q;  // p_new = (pcg->iter & 1) ? p1 : p0
  PcgState* pcg;
  DevStatus* st;
  double* partial;
  unsigned int* counter;          // 1 site
  double tol2;
  int maxit;
  unsigned long long cond;        // graph conditional handle (0: none)
  int update;                     // apply x += alpha p, r -= alpha q first (if !pcg->first)
  // subdomain group (dist.cu): k_prec_out writes its local sums [r.z (kk) | owned r.r (kk)] here
  // and skips the scalar step (run after the exchange); null: ordinary context
  double* xsum;
};
void launch_precond(const PrecArgs& a, cudaStream_t s);
// direction d of every patch box by the whole-line shared-memory solver (line_seq.cu); false if
// not applicable (caller uses the chunked tiles)
bool launch_line_seq_multi(const PrecArgs& a, int d, cudaStream_t s, bool dry = false);
int line_seq_mode();  // GA_LINE_SEQ=0: off (the chunked tiles instead)
bool line_seq_prepare(int p);  // function attributes of degree p's kernel, outside stream capture

struct VecArgs {
  GridDesc g;
  int nvec, kk;
  double tol2;
  double *x, *r, *z, *p, *b;
  PcgState* pcg;
  DevStatus* st;
  double* partial;
  unsigned int* counter;
  // subdomain group (dist.cu): k_init_from_b writes the owned ||b||^2 (mask value 1) here and
  // leaves the PcgState set-up to the step after the exchange; null: ordinary context
  const unsigned char* own;
  double* xsum;
  const unsigned char* mask;  // grid mask (masked grids: points that are not free are skipped), or null
};
void launch_init_from_b(const VecArgs& a, cudaStream_t s);
void launch_p_update(const VecArgs& a, cudaStream_t s);
void launch_solve_end(PcgState* pcg, DevStatus* st, cudaStream_t s);

struct StageArgs {
  GridDesc g;
  int nvec, k;
  double* chain;        // [3k][nvec][padded]
  const double* ysol;   // MV (x of the solve), kk = k
  double* pred;         // MV, kk = k
  double alpha[KMAX], beta[KMAX], gamma[KMAX];
  double f[3 * KMAX];   // tau^i / i!
  double tau;
  double unstable2;     // threshold on ||U||^2 / ||U0||^2 (0: off)
  double damp_a0, damp_a1;  // Rayleigh damping C = a0 M + a1 K (reading R16)
  DevStatus* st;
  double* partial;
  unsigned int* counter;
};
void launch_stage(const StageArgs& a, cudaStream_t s);

// Forcing F(x, t) = G(x) h(t), h(t) = sum_i amp_i cos(omega_i t + phase_i) (eq:ho1):
// b_j += h^{(order_j)}(t0 + steps dt + toff_j) G for the active right-hand-side slots j.  The slot
// table lives on the device (written before each solve set: the initial chain uses orders m-2 at
// t0, the step orders 3j at t_n + alpha_fj dt), so the captured graphs need no rebuild.
constexpr int FMAXTERMS = 8;
constexpr int FMAXPAIRS = 3;  // pair 0: ga_set_forcing; pairs 1, 2: Dirichlet lifting (ga_set_dirichlet)
struct ForceSlots {
  int active[KMAX];
  int order[KMAX];
  double toff[KMAX];
};
struct ForceArgs {
  GridDesc g;
  int nvec, kk, npairs;
  int nterms[FMAXPAIRS];
  double amp[FMAXPAIRS][FMAXTERMS], omega[FMAXPAIRS][FMAXTERMS], phase[FMAXPAIRS][FMAXTERMS];
  double t0, dt;
  const double* G[FMAXPAIRS];  // grid vectors [c][guard | npts | guard] (b += sum_pairs h^{(m)} G)
  double* b;                 // MV [c][guard | npts | guard][kk]
  const ForceSlots* slots;   // device
  const DevStatus* st;       // st->steps: completed steps since ga_set_state
};
void launch_add_forcing(const ForceArgs& a, cudaStream_t s);

// Predictors from the chain (after set_state / set_chain), same rule as the stage kernel.
void launch_predict(const StageArgs& a, cudaStream_t s);

// chain <-> MV slot packing for the initial chain (src/dst < 0: zero / skip).
// with damping: pack slot = chain[src] + a1 chain[src2], unpack chain[dst] = slot - a0 chain[src2]
void launch_pack(const GridDesc& g, int nvec, int kk, const double* chain, const int* src, double* mv,
                 DevStatus* st, cudaStream_t s, const int* src2 = nullptr, double a1 = 0.0);
void launch_unpack(const GridDesc& g, int nvec, int kk, const double* mv, const int* dst, double* chain,
                   DevStatus* st, cudaStream_t s, const int* src2 = nullptr, double a0 = 0.0);

// free-DoF (API) vector <-> grid vector (stride kk, slot j) with optional map
void launch_api_to_grid(const GridDesc& g, int nvec, long long nfree, const long long* map, const double* api,
                        double* gridv, int kk, int slot, DevStatus* st, cudaStream_t s);
void launch_grid_to_api(const GridDesc& g, int nvec, long long nfree, const long long* map, const double* gridv,
                        int kk, int slot, double* api, DevStatus* st, cudaStream_t s);

// dot products of MV slot 0 of two grid vectors (stride kk) into out[0] (device), via partials.
void launch_ref_norm(const GridDesc& g, int nvec, const double* c0, const double* c1, double tau, DevStatus* st,
                     double* partial, unsigned int* counter, cudaStream_t s);
void launch_dot(const GridDesc& g, int nvec, int kk, const double* a, const double* b, double* out,
                double* partial, unsigned int* counter, cudaStream_t s);
void launch_scale(const GridDesc& g, int nvec, int kk, double* a, const double* num, int inv_sqrt,
                  cudaStream_t s);

}  // namespace ga

namespace ga {

// Persistent cooperative PCG solve (small single-patch scalar problems, where
// every kernel is latency-bound): the whole lock-stepped solve of the k
// right-hand sides in b -- main phase and refinement restart -- in ONE
// cooperative launch, phases separated by grid-wide barriers, scalars
// reduced redundantly (same order) by every block.  Returns false if the
// configuration is not supported (caller uses the graph path).
struct PersistArgs {
  PrecArgs pa;        // preconditioner (single patch, fused tile path)
  SpmvArgs spq;       // M p -> q (SPMV_PQ, unfused)
  SpmvArgs str;       // b - M x -> r (SPMV_TRUERES)
  VecArgs va;
  int refine;
  double refine_rtol2;
  long long* trace;
  double* p1;         // second direction buffer (fused direction update)
};
bool persist_supported(const PersistArgs& A);
bool launch_pcg_persist(const PersistArgs& A, cudaStream_t s);

}  // namespace ga
