// Internal: the context structure of the C ABI (include/genalpha.h) and the argument builders
// shared by genalpha.cu (single contexts) and dist.cu (groups of subdomain contexts).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/genalpha.h"
#include "common.cuh"
#include "host_math.h"
#include "ops.cuh"

namespace gaint {

using namespace ga;

struct PatchHost {
  int cell[3];
  std::vector<double> ctrl;
};

struct PrecPatch {
  int lo[3], bd[3];     // box in grid coordinates
  int llo[3];           // first local basis index per direction
  double* s = nullptr;  // device, box points
  double* t = nullptr;  // device, nvec*box*k (multi-patch only)
  double* L[3] = {nullptr, nullptr, nullptr};
  double* Ff[3] = {nullptr, nullptr, nullptr};
  double* Fb[3] = {nullptr, nullptr, nullptr};
  double* E[3] = {nullptr, nullptr, nullptr};   // make_seq rows (device)
  int clen[3] = {0, 0, 0}, nchunk[3] = {0, 0, 0}, nlev[3] = {0, 0, 0};
  std::vector<double> hL[3], hdiag[3], hE[3];
  SweepFactor sf[3], sb[3];
};

}  // namespace gaint

using namespace ga;  // internal header: the device types of common.cuh / ops.cuh

struct ga_ctx {
  ga_desc d{};
  std::vector<gaint::PatchHost> patches;
  int dim = 2, nvec = 1, p = 1, n = 1, m = 2, k = 1, W1 = 3;
  long long S = 0;
  GridDesc g{};
  long long nfree = 0;  // scalar free DoFs
  std::vector<long long> hmap;           // api -> grid (multi-patch)
  std::vector<unsigned char> hmask;      // grid mask (multi-patch)
  std::vector<long long> hlocal;         // api -> patch*m^dim + local
  double alpha[KMAX], beta[KMAX], gamma[KMAX], alpha_f[KMAX], theta_max = 0;
  // device views into the workspace
  char* ws = nullptr;
  size_t ws_bytes = 0;
  double *coefM = nullptr, *coefK = nullptr, *chain = nullptr;
  double *pred = nullptr, *b = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *pv = nullptr, *q = nullptr, *pv1 = nullptr;
  unsigned char* mask = nullptr;
  unsigned char* blkskip = nullptr;  // per 32-row block: 1 = no free row (masked grids), SpmvArgs::skip
  long long* map = nullptr;
  PcgState* pcg = nullptr;
  DevStatus* st = nullptr;
  double* partial = nullptr;
  unsigned int* counter = nullptr;
  double* dscal = nullptr;  // small device scalars
  std::vector<gaint::PrecPatch> prec;
  // graphs
  cudaStream_t aux = nullptr, cap = nullptr;  // private capture streams
  cudaGraphExec_t g_step = nullptr, g_solveK = nullptr, g_solveB = nullptr;
  cudaGraph_t gr_step = nullptr, gr_solveK = nullptr, gr_solveB = nullptr;
  std::string err;
  bool nograph = false;  // GA_NO_GRAPH=1: direct launches, host-driven PCG loop (profiling/debug)
  bool persist = false;  // small single-patch scalar problems: one cooperative kernel per solve
  bool mf = false;       // matrix-free M (and scalar K): sum factorisation from Gauss-point data
  bool half = false;     // half-symmetric stencils (offsets o >= 0, zero guard of g.guard rows)
  bool sym = false;      // 3D scalar half stencils in the segment-blocked layout (spmv_sym.cu)
  double* symzero = nullptr;  // zero block read by the single-read SpMV for unstored rows
  SymLayout sl = {0, 0};
  double *mfWM = nullptr, *mfWK = nullptr, *mftv = nullptr, *mftd = nullptr, *diagM = nullptr;
  double *mpT1 = nullptr, *mpT2 = nullptr, *mpT3 = nullptr;  // 3D multi-pass mass intermediates
  // forcing F = G h(t) (ga_set_forcing): grid vector, device slot table, host parameters
  double* forceG = nullptr;
  ForceSlots* fslots = nullptr;
  bool forcing = false;       // any pair active (pair 0 ga_set_forcing, 1-2 ga_set_dirichlet)
  double *lzv = nullptr, *lzab = nullptr;  // Lanczos vectors and alpha/beta (ga_lambda_max)
  int fnterms[FMAXPAIRS] = {0, 0, 0};
  double famp[FMAXPAIRS][FMAXTERMS], fomega[FMAXPAIRS][FMAXTERMS], fphase[FMAXPAIRS][FMAXTERMS], ft0 = 0.0;
  long long mfws = 0;    // Gauss points (n(p+1))^dim
  long long* trace = nullptr;  // GA_TRACE=1: persistent-solver phase timestamps (debug)
  // subdomain of a partitioned problem (ga_desc.sub, dist.cu): the grid is the bounding box of
  // the patch's free control points (grid coordinate = local index - org), mask 1 = free and
  // owned, 2 = free copy owned by another subdomain; interface exchange lists and buffers
  bool sub = false;
  int org[3] = {1, 1, 1};      // local control-point index of grid coordinate 0 (1: Dirichlet ring)
  long long n_iface = 0;       // interface DoFs of the whole partitioned problem
  long long nxl = 0;           // interface DoFs held by this subdomain
  int* xgi = nullptr;          // device [nxl]: grid index of each held interface DoF
  int* xslot = nullptr;        // device [nxl]: its global interface slot
  int* xinv = nullptr;         // device [n_iface]: grid index of a slot in this subdomain, or -1
  double* xbuf = nullptr;      // device exchange buffer [nvec][n_iface][k] + XSCAL scalars
  double* xrecv = nullptr;     // device, same size: the summed buffer
  long long xcount = 0;        // doubles of xbuf
  ga_group* grp = nullptr;     // the group this context belongs to (one at a time)
};


namespace gaint {

void seterr(ga_ctx* ctx, const std::string& s);
PrecArgs prec_args(ga_ctx* c, unsigned long long cond, int update);
SpmvArgs spmv_args(ga_ctx* c, int which, const double* x, double* y, int mode);
VecArgs vec_args(ga_ctx* c);
StageArgs stage_args(ga_ctx* c);
ForceArgs force_args(ga_ctx* c);
ga_status set_step_slots(ga_ctx* ctx, cudaStream_t s);
ga_status set_predictors_and_norm(ga_ctx* ctx, cudaStream_t s);
void reset_status(ga_ctx* ctx, cudaStream_t s, int keep_time = 0);
// preconditioner scalings s = sqrt(Dh / D) of every patch box from diag(M) (ctx->diagM if set,
// else the stencil centre); SYNCHRONIZES s
ga_status compute_scaling(ga_ctx* ctx, cudaStream_t s);

}  // namespace gaint
