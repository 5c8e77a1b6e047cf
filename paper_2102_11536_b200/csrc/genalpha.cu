// C ABI (include/genalpha.h) of the B200 explicit order-2k generalized-alpha
// integrator: descriptor validation, workspace layout, GPU assembly driver,
// preconditioner setup, CUDA-graph construction (PCG loops as conditional
// WHILE nodes, no host synchronisation inside a step) and the entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/genalpha.h"
#include "assembly.cuh"
#include "common.cuh"
#include "host_math.h"
#include "ops.cuh"

using namespace ga;

#include "ctx.cuh"

#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

namespace {
// GA_BACKTRACE=1: print the native stack on SIGSEGV (debug aid; offsets resolve with addr2line)
void ga_segv_handler(int sig) {
  void* fr[64];
  const int n = backtrace(fr, 64);
  backtrace_symbols_fd(fr, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct GaSegvInit {
  GaSegvInit() {
    const char* e = getenv("GA_BACKTRACE");
    if (e && *e == '1') {
      static char alt[1 << 16];
      stack_t ss;
      ss.ss_sp = alt; ss.ss_size = sizeof(alt); ss.ss_flags = 0;
      sigaltstack(&ss, nullptr);
      struct sigaction sa;
      memset(&sa, 0, sizeof(sa));
      sa.sa_handler = ga_segv_handler;
      sa.sa_flags = SA_ONSTACK;
      sigaction(SIGSEGV, &sa, nullptr);
    }
  }
} ga_segv_init;
}  // namespace

namespace {
thread_local std::string g_thread_err;
}  // namespace

namespace gaint {

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      seterr(ctx, std::string(#call) + ": " + cudaGetErrorString(e_));              \
      return GA_ERR_CUDA;                                                           \
    }                                                                               \
  } while (0)

void seterr(ga_ctx* ctx, const std::string& s) {
  if (ctx) ctx->err = s;
  g_thread_err = s;
}

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

struct Layout {
  size_t off_coefM, off_coefK, off_symzero, off_chain, off_mv[8], off_mask, off_skip, off_map, off_pcg, off_st, off_partial, off_counter,
      off_dscal, off_mfWM, off_mfWK, off_mftab, off_diag, off_mpT1, off_mpT2, off_mpT3, off_forceG, off_fslots,
      off_lz, off_lzab, off_xgi, off_xslot, off_xinv, off_xbuf, off_xrecv;
  std::vector<size_t> off_s, off_t, off_L[3], off_F[3], off_E[3];
  size_t total;
};

// Derived sizes that do not need the GPU.
struct Shape {
  int dim, nvec, p, n, m, k, W1;
  long long S;
  GridDesc g;
  std::vector<PrecPatch> prec;  // boxes only
  long long nfree;
  std::vector<unsigned char> mask;
  std::vector<long long> map;
  std::vector<long long> local;
  int pmin[3], pmax[3];
  bool mf = false;     // matrix-free operators (op_mode 2, or auto)
  bool half = false;   // half-symmetric stencils (op_mode 3, or auto)
  bool sym = false;    // ... in the segment-blocked layout of the single-read 3D SpMV (scalar, 3D)
  SymLayout sl = {0, 0};
  int org[3] = {1, 1, 1};  // local control-point index of grid coordinate 0
  bool sub = false;        // subdomain of a partitioned problem (make_shape_sub)
  long long n_iface = 0;
  std::vector<int> xgi, xslot;  // held interface DoFs: grid index, global slot
};

int op_auto(const ga_desc* d);

ga_status validate(const ga_desc* d, ga_ctx* ctx) {
  if (!d) { seterr(ctx, "desc is NULL"); return GA_ERR_ARG; }
  if (d->dim != 2 && d->dim != 3) { seterr(ctx, "dim must be 2 or 3"); return GA_ERR_ARG; }
  if (d->ncomp != 1 && !(d->ncomp == 3 && d->dim == 3)) { seterr(ctx, "ncomp must be 1 or 3 (dim 3)"); return GA_ERR_ARG; }
  if (d->p < 1 || d->p > 7) { seterr(ctx, "p must be in 1..7"); return GA_ERR_ARG; }
  if (d->n < 1) { seterr(ctx, "n must be >= 1"); return GA_ERR_ARG; }
  if (d->n + d->p < 3) { seterr(ctx, "n + p must be >= 3 (at least one free DoF)"); return GA_ERR_ARG; }
  if (d->npatch < 1 || d->npatch > MAXPATCH || !d->patches) { seterr(ctx, "npatch must be 1..16"); return GA_ERR_ARG; }
  if (d->k < 1 || d->k > KMAX) { seterr(ctx, "k must be 1..4"); return GA_ERR_ARG; }
  if (!(d->dt > 0.0) || !std::isfinite(d->dt)) { seterr(ctx, "dt must be > 0"); return GA_ERR_ARG; }
  if (!(d->pcg_refine_rtol >= 0.0) || d->pcg_refine_rtol >= 1.0) { seterr(ctx, "pcg_refine_rtol must be in [0,1)"); return GA_ERR_ARG; }
  if (!(d->pcg_rtol > 0.0) || d->pcg_maxit < 1) { seterr(ctx, "pcg_rtol > 0 and pcg_maxit >= 1 required"); return GA_ERR_ARG; }
  if (d->param_set != 0 && d->param_set != 1) { seterr(ctx, "param_set must be 0 or 1"); return GA_ERR_ARG; }
  if (d->op_mode < 0 || d->op_mode > 3) { seterr(ctx, "op_mode must be 0, 1, 2 or 3"); return GA_ERR_ARG; }
  if (!std::isfinite(d->damp_a0) || !std::isfinite(d->damp_a1) || d->damp_a0 < 0.0 || d->damp_a1 < 0.0) {
    seterr(ctx, "damping coefficients must be finite and >= 0");
    return GA_ERR_ARG;
  }
  if (d->op_mode == 2 && d->npatch != 1) { seterr(ctx, "op_mode 2 (matrix-free) supports a single patch"); return GA_ERR_ARG; }
  if (d->sub) {
    if (d->npatch != 1 || !d->sub->free_mask || !d->sub->owned || !d->sub->iface || d->sub->n_iface < 0) {
      seterr(ctx, "subdomain: npatch 1 and free_mask, owned, iface arrays required");
      return GA_ERR_ARG;
    }
    if (d->op_mode == 2) { seterr(ctx, "subdomain: op_mode 2 (matrix-free) is not available"); return GA_ERR_ARG; }
  }
  double a[KMAX], b[KMAX], g[KMAX], f[KMAX], th;
  int rc = scheme_params(d->k, d->rho_b, d->rho_s, d->param_set, a, b, g, f, &th);
  if (rc != 0) { seterr(ctx, "invalid rho_b/rho_s (need 0 <= rho_s <= rho_b <= 1; param_set 1 needs rho < 1)"); return GA_ERR_PARAM; }
  for (int i = 0; i < d->npatch; ++i) {
    if (!d->patches[i].ctrl) { seterr(ctx, "patch ctrl is NULL"); return GA_ERR_ARG; }
    for (int c = 0; c < 3; ++c)
      if (d->patches[i].cell[c] < 0 || d->patches[i].cell[c] > 64 || (c >= d->dim && d->patches[i].cell[c] != 0)) {
        seterr(ctx, "patch cell out of range");
        return GA_ERR_ARG;
      }
    for (int j = 0; j < i; ++j)
      if (!memcmp(d->patches[i].cell, d->patches[j].cell, sizeof(int) * 3)) { seterr(ctx, "two patches share a cell"); return GA_ERR_ARG; }
  }
  return GA_OK;
}

// Subdomain grid (ga_desc.sub): the bounding box [lo, hi] of the patch's free control points;
// grid coordinate = local index - lo (org = lo); mask 1 = free and owned, 2 = free copy owned by
// another subdomain, 0 = Dirichlet point inside the box (e.g. the re-entrant corner of an
// L-shape patch); one preconditioner box = the grid, local basis range [lo, hi] (reading R6:
// zero extension of the non-tensor free set to its bounding box).
ga_status make_shape_sub(const ga_desc* d, Shape& sh, ga_ctx* ctx) {
  const int m = sh.m, dim = sh.dim;
  const long long mpow = dim == 3 ? (long long)m * m * m : (long long)m * m;
  const ga_subdomain* sd = d->sub;
  sh.sym = false;  // the single-read 3D SpMV assumes a full box; masked grids use the two-pass half kernel
  int lo[3] = {m, m, m}, hi[3] = {-1, -1, -1};
  for (long long i = 0; i < mpow; ++i) {
    if (!sd->free_mask[i]) continue;
    const int li[3] = {(int)(i % m), (int)((i / m) % m), dim == 3 ? (int)(i / ((long long)m * m)) : 0};
    for (int c = 0; c < dim; ++c) { lo[c] = std::min(lo[c], li[c]); hi[c] = std::max(hi[c], li[c]); }
  }
  if (hi[0] < 0) { seterr(ctx, "subdomain has no free DoF"); return GA_ERR_ARG; }
  int G[3] = {1, 1, 1};
  for (int c = 0; c < dim; ++c) { G[c] = hi[c] - lo[c] + 1; sh.org[c] = lo[c]; }
  sh.g.dim = dim; sh.g.nx = G[0]; sh.g.ny = G[1]; sh.g.nz = dim == 3 ? G[2] : 1;
  sh.g.npts = (long long)sh.g.nx * sh.g.ny * sh.g.nz;
  long long guard = (long long)sh.p * (1 + sh.g.nx + (dim == 3 ? (long long)sh.g.nx * sh.g.ny : 0));
  guard = (guard + 32 + 31) / 32 * 32;
  sh.g.guard = guard;
  sh.g.padded = sh.g.npts + 2 * guard;
  sh.g.cs = (sh.g.npts + 31) / 32 * 32;
  sh.sl = sym_layout(sh.g.nx);
  sh.mask.assign(sh.g.npts, 0);
  sh.map.clear();
  sh.local.clear();
  sh.xgi.clear();
  sh.xslot.clear();
  for (long long gi = 0; gi < sh.g.npts; ++gi) {
    const int gc[3] = {(int)(gi % sh.g.nx), (int)((gi / sh.g.nx) % sh.g.ny), (int)(gi / ((long long)sh.g.nx * sh.g.ny))};
    long long loc = 0, mul = 1;
    for (int c = 0; c < dim; ++c) { loc += (long long)(gc[c] + lo[c]) * mul; mul *= m; }
    if (!sd->free_mask[loc]) continue;
    sh.mask[gi] = sd->owned[loc] ? 1 : 2;
    sh.map.push_back(gi);
    sh.local.push_back(loc);
    if (sd->iface[loc] >= 0) {
      if (sd->iface[loc] >= sd->n_iface) { seterr(ctx, "subdomain: interface slot out of range"); return GA_ERR_ARG; }
      sh.xgi.push_back((int)gi);
      sh.xslot.push_back((int)sd->iface[loc]);
    }
  }
  sh.nfree = (long long)sh.map.size();
  sh.prec.clear();
  PrecPatch pp;
  for (int c = 0; c < 3; ++c) {
    if (c >= dim) { pp.lo[c] = 0; pp.bd[c] = 1; pp.llo[c] = 0; continue; }
    pp.lo[c] = 0; pp.bd[c] = G[c]; pp.llo[c] = lo[c];
  }
  sh.prec.push_back(pp);
  sh.sub = true;
  sh.n_iface = sd->n_iface;
  return GA_OK;
}

// Global masked grid, boxes, maps.
ga_status make_shape(const ga_desc* d, Shape& sh, ga_ctx* ctx, bool check_conformity) {
  sh.dim = d->dim; sh.nvec = d->ncomp; sh.p = d->p; sh.n = d->n; sh.m = d->n + d->p; sh.k = d->k; sh.W1 = 2 * d->p + 1;
  {
    const int pick = d->op_mode == 0 ? op_auto(d) : d->op_mode;
    sh.mf = pick == 2;
    sh.half = pick == 3;
  }
  sh.sym = sh.half && d->dim == 3 && d->ncomp == 1;
  sh.S = (long long)sh.W1 * sh.W1 * (sh.dim == 3 ? sh.W1 : 1);
  const int m = sh.m, dim = sh.dim;
  for (int c = 0; c < 3; ++c) sh.org[c] = 1;
  if (d->sub) return make_shape_sub(d, sh, ctx);
  int cmax[3] = {0, 0, 0};
  for (int i = 0; i < d->npatch; ++i)
    for (int c = 0; c < dim; ++c) cmax[c] = std::max(cmax[c], d->patches[i].cell[c]);
  // full global point counts (incl. boundary): (cmax+1)(m-1)+1 per direction
  int Gfull[3] = {1, 1, 1}, G[3] = {1, 1, 1};
  for (int c = 0; c < dim; ++c) { Gfull[c] = (cmax[c] + 1) * (m - 1) + 1; G[c] = Gfull[c] - 2; }
  sh.g.dim = dim; sh.g.nx = G[0]; sh.g.ny = G[1]; sh.g.nz = dim == 3 ? G[2] : 1;
  sh.g.npts = (long long)sh.g.nx * sh.g.ny * sh.g.nz;
  long long guard = (long long)sh.p * (1 + sh.g.nx + (dim == 3 ? (long long)sh.g.nx * sh.g.ny : 0));
  guard = (guard + 32 + 31) / 32 * 32;  // + register-blocked SpMV window overhang
  sh.g.guard = guard;
  sh.g.padded = sh.g.npts + 2 * guard;
  sh.g.cs = (sh.g.npts + 31) / 32 * 32;
  sh.sl = sym_layout(sh.g.nx);
  // occupancy of coarse cells
  std::map<long long, int> cellid;
  auto ckey = [&](int x, int y, int z) { return ((long long)z * 1000 + y) * 1000 + x; };
  for (int i = 0; i < d->npatch; ++i) cellid[ckey(d->patches[i].cell[0], d->patches[i].cell[1], d->patches[i].cell[2])] = i;
  const bool multi = d->npatch > 1;
  // a grid point (interior coords) is free iff every coarse cell whose closure contains it is a patch
  if (multi) {
    sh.mask.assign(sh.g.npts, 0);
    for (long long gi = 0; gi < sh.g.npts; ++gi) {
      int gc[3] = {(int)(gi % sh.g.nx), (int)((gi / sh.g.nx) % sh.g.ny), (int)(gi / ((long long)sh.g.nx * sh.g.ny))};
      int lo[3], hi[3];
      for (int c = 0; c < 3; ++c) {
        if (c >= dim) { lo[c] = hi[c] = 0; continue; }
        int I = gc[c] + 1;  // full coordinate
        int cc = I / (m - 1);
        if (I % (m - 1) == 0) { lo[c] = cc - 1; hi[c] = cc; } else { lo[c] = hi[c] = cc; }
      }
      bool ok = true;
      for (int z = lo[2]; z <= hi[2] && ok; ++z)
        for (int y = lo[1]; y <= hi[1] && ok; ++y)
          for (int x = lo[0]; x <= hi[0] && ok; ++x) {
            if (x < 0 || y < 0 || z < 0 || !cellid.count(ckey(x, y, z))) ok = false;
          }
      sh.mask[gi] = ok ? 1 : 0;
    }
    sh.map.clear();
    for (long long gi = 0; gi < sh.g.npts; ++gi)
      if (sh.mask[gi]) sh.map.push_back(gi);
    sh.nfree = (long long)sh.map.size();
  } else {
    sh.nfree = sh.g.npts;
  }
  // (patch, local) of each free DoF: first patch in order whose closed cell contains it
  const long long mpow = dim == 3 ? (long long)m * m * m : (long long)m * m;
  sh.local.assign(sh.nfree, -1);
  for (long long f = 0; f < sh.nfree; ++f) {
    long long gi = multi ? sh.map[f] : f;
    int gc[3] = {(int)(gi % sh.g.nx), (int)((gi / sh.g.nx) % sh.g.ny), (int)(gi / ((long long)sh.g.nx * sh.g.ny))};
    for (int r = 0; r < d->npatch; ++r) {
      long long loc = 0, mul = 1;
      bool in = true;
      for (int c = 0; c < dim; ++c) {
        int li = gc[c] + 1 - d->patches[r].cell[c] * (m - 1);
        if (li < 0 || li > m - 1) { in = false; break; }
        loc += li * mul;
        mul *= m;
      }
      if (in) { sh.local[f] = r * mpow + loc; break; }
    }
  }
  // preconditioner boxes: free local indices of patch r (tensor superset, reading R6)
  sh.prec.clear();
  for (int r = 0; r < d->npatch; ++r) {
    PrecPatch pp;
    for (int c = 0; c < 3; ++c) {
      if (c >= dim) { pp.lo[c] = 0; pp.bd[c] = 1; pp.llo[c] = 0; continue; }
      int cell = d->patches[r].cell[c];
      // local index range [1, m-2] plus the interface ends if the neighbour cell exists
      int llo = 1, lhi = m - 2;
      int nb[3] = {d->patches[r].cell[0], d->patches[r].cell[1], d->patches[r].cell[2]};
      nb[c] = cell - 1;
      if (cell > 0 && cellid.count(ckey(nb[0], nb[1], nb[2]))) llo = 0;
      nb[c] = cell + 1;
      if (cellid.count(ckey(nb[0], nb[1], nb[2]))) lhi = m - 1;
      pp.llo[c] = llo;
      pp.lo[c] = cell * (m - 1) + llo - 1;
      pp.bd[c] = lhi - llo + 1;
    }
    sh.prec.push_back(pp);
  }
  if (multi && check_conformity) {
    // coincident global points must have bitwise identical control points
    std::map<long long, std::vector<double>> seen;
    long long Gx = Gfull[0], Gy = Gfull[1];
    for (int r = 0; r < d->npatch; ++r) {
      for (long long loc = 0; loc < mpow; ++loc) {
        int li[3] = {(int)(loc % m), (int)((loc / m) % m), dim == 3 ? (int)(loc / ((long long)m * m)) : 0};
        bool onface = false;
        for (int c = 0; c < dim; ++c) onface |= (li[c] == 0 || li[c] == m - 1);
        if (!onface) continue;
        long long key = 0;
        int I[3];
        for (int c = 0; c < dim; ++c) I[c] = d->patches[r].cell[c] * (m - 1) + li[c];
        key = I[0] + Gx * (I[1] + (dim == 3 ? Gy * (long long)I[2] : 0));
        std::vector<double> pt(d->patches[r].ctrl + loc * dim, d->patches[r].ctrl + loc * dim + dim);
        auto it = seen.find(key);
        if (it == seen.end()) seen[key] = pt;
        else if (memcmp(it->second.data(), pt.data(), sizeof(double) * dim) != 0) {
          seterr(ctx, "patch interfaces are not conforming (control points differ)");
          return GA_ERR_CONFORMITY;
        }
      }
    }
  }
  return GA_OK;
}

// op_mode 0 (R14, §6 "Stencil vs matrix-free", "Symmetric SpMV"): measured per apply.
// The full stencil SpMV streams its (2p+1)^d coefficients at 0.8-1.0 of HBM bandwidth; the
// single-read symmetric SpMV (3D scalar, spmv_sym.cu) streams half of them at 0.75-0.88, so it
// wins wherever its 32-point x-segments are well used (C3 n = 192: p = 2 1.20 -> 0.89 ms,
// p = 4 6.6 -> 4.2 ms per M apply; n = 96: p = 2, 4, 5 faster) and loses where the last segment
// is nearly empty at low p (p = 3, n = 96: nx = 97 = 3 x 32 + 1, 0.40 vs 0.44 ms).  So: 3D scalar
// -> half-symmetric if p >= 4 or the segments are >= 90 % used, else full stencils if they fit
// in ~150 GB, else half-symmetric, else matrix-free (multi-patch grids: stencils).
int op_auto(const ga_desc* d) {
  const double W1 = 2.0 * d->p + 1.0, S = d->dim == 3 ? W1 * W1 * W1 : W1 * W1;
  if (d->sub) {  // subdomain: full stencils unless they do not fit (the masked-grid rule below)
    const double nsub = std::pow((double)(d->n + d->p), d->dim);
    return 8.0 * S * nsub * (d->ncomp == 3 ? 10.0 : 2.0) <= 150e9 ? 1 : 3;
  }
  const double npts = std::pow((double)((d->n + d->p - 1) * 2), d->dim);  // generous (multi-patch box)
  const double nsp = d->npatch == 1 ? std::pow((double)(d->n + d->p - 2), d->dim) : npts;
  const double full = 8.0 * S * nsp * (d->ncomp == 3 ? 10.0 : 2.0);
  const double half = 8.0 * nsp * (d->ncomp == 3 ? (S + 1) / 2 + 9 * S : S + 1);
  if (d->dim == 3 && d->ncomp == 1 && d->npatch == 1) {
    const int nx = d->n + d->p - 2, nseg = (nx + 31) / 32;
    const double sym = 2.0 * 8.0 * ((S + 1) / 2) * 32.0 * nseg * (double)nx * nx;  // M + K, segment layout
    // small grids stay on full stencils: the persistent cooperative solver (latency-bound regime,
    // the rule of ga_create) is faster there than any graph of separate kernels
    const bool small = nsp * d->k <= 600000.0 && S * nsp * 8.0 <= 64e6;
    // measured (tools/kbench.py, step time, sym vs full): p=3 n=96/128/160/192 6.99/12.6/22.6/38.3 vs
    // 7.52/14.5/28.8/49.4 ms; p=2 n=100 (78 % of the x-segments used) 3.45 vs 3.31 ms
    // p=3 n=64 (68 % used): 3.18 vs 2.82 ms; p >= 4: symmetric at every measured size (n = 48..192)
    const double need = d->p >= 4 ? 0.0 : (d->p == 3 ? 0.72 : 0.9);
    if (!small && sym <= 165e9 && nx >= need * 32 * nseg) return 3;
    if (full <= 150e9) return 1;
    if (sym <= 165e9) return 3;
    return 2;
  }
  if (full <= 150e9) return 1;
  if (half <= 150e9) return 3;
  return d->npatch == 1 ? 2 : 3;
}

constexpr int LZMAX = 512;  // Lanczos steps of ga_lambda_max

// bytes of one scalar stencil operator (M, or the scalar K) in the layout of the shape
size_t coef_bytes(const Shape& sh) {
  const long long Sh = (sh.S + 1) / 2;
  if (sh.sym)
    return sizeof(double) * Sh * SYM_STRIDE * (long long)sh.sl.nseg * sh.g.ny * sh.g.nz;
  if (sh.half) return sizeof(double) * Sh * ((sh.g.npts + sh.g.guard + 31) / 32 * 32);
  return sizeof(double) * sh.S * sh.g.cs;
}

size_t sweep_bytes(int n, int p) {
  // dinv + coef + H + A (L <= 6 levels, C <= 64 chunks)
  return align256(sizeof(double) * ((size_t)n * (1 + 2 * p) + (size_t)6 * 64 * p * p));
}

Layout make_layout(const Shape& sh) {
  Layout L;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes); return r; };
  const long long npts = sh.g.npts;
  const bool mfK = sh.mf && sh.nvec == 1;  // the elastic K stays a full stencil
  const size_t mbytes = coef_bytes(sh);
  L.off_coefM = take(sh.mf ? 0 : mbytes);
  L.off_coefK = take(mfK ? 0 : (sh.nvec == 3 ? sizeof(double) * sh.S * sh.g.cs * 9 : mbytes));
  L.off_symzero = take(sh.sym ? sizeof(double) * ((sh.S + 1) / 2) * SYM_STRIDE : 0);
  {
    const long long nq = (long long)sh.n * (sh.p + 1);
    const long long nqd = sh.dim == 3 ? nq * nq * nq : nq * nq;
    L.off_mfWM = take(sh.mf ? sizeof(double) * nqd : 0);
    L.off_mfWK = take(mfK ? sizeof(double) * nqd * (sh.dim == 3 ? 6 : 3) : 0);
    L.off_mftab = take(sh.mf ? sizeof(double) * 2 * nq * (sh.p + 1) : 0);
    L.off_diag = take((sh.mf || sh.sub) ? sizeof(double) * npts : 0);
    // multi-pass 3D mass intermediates (matfree_mp.cu)
    const bool mp = sh.mf && sh.dim == 3;
    const long long nfd = sh.g.nx;
    L.off_mpT1 = take(mp ? sizeof(double) * sh.nvec * nq * nfd * nfd * sh.k : 0);
    L.off_mpT2 = take(mp ? sizeof(double) * sh.nvec * nq * nq * nfd * sh.k : 0);
    L.off_mpT3 = take(mp ? sizeof(double) * sh.nvec * nq * nq * nfd * sh.k : 0);
  }
  L.off_chain = take(sizeof(double) * 3 * sh.k * sh.nvec * sh.g.padded);
  for (int i = 0; i < 8; ++i) L.off_mv[i] = take(sizeof(double) * sh.nvec * sh.g.padded * sh.k);
  const bool multi = sh.prec.size() > 1 || sh.sub;
  L.off_mask = take(multi ? npts : 0);
  L.off_skip = take(multi ? (npts + 31) / 32 : 0);
  L.off_map = take(multi ? sizeof(long long) * sh.nfree : 0);
  L.off_pcg = take(sizeof(PcgState));
  L.off_st = take(sizeof(DevStatus));
  // reduction partials: one slot per block of any reducing kernel; the line
  // tile kernels can launch more blocks than the grid kernels on small grids
  // grid kernels, SpMV (32 rows/block), persistent solver (2 x 1184 blocks, double-buffered)
  long long maxblocks = std::max(std::max((sh.nvec * npts + NTHREADS - 1) / NTHREADS, (npts + 31) / 32), 2LL * 1184) + 1;
  long long sumt[3] = {0, 0, 0};
  for (const PrecPatch& pp : sh.prec) {
    const long long nb0 = pp.bd[0], nb1 = pp.bd[1], nb2 = pp.bd[2];
    // >= 4 slots per tile (line_seq.cu; the chunked tiles use >= 8)
    const long long xt = (sh.nvec * nb1 * nb2 * sh.k + 3) / 4;            // x lines
    const long long yt = sh.nvec * nb2 * ((nb0 * sh.k + 3) / 4);           // y lines
    const long long zt = sh.nvec * nb1 * ((nb0 * sh.k + 3) / 4);           // z lines
    maxblocks = std::max(maxblocks, std::max(xt, std::max(yt, zt)) + 1);
    sumt[0] += xt; sumt[1] += yt; sumt[2] += zt;
  }
  // the tiles of all patches in one launch (additive Schwarz, fused epilogue of line_seq.cu)
  maxblocks = std::max(maxblocks, std::max(sumt[0], std::max(sumt[1], sumt[2])) + 1);
  L.off_partial = take(sizeof(double) * 2 * KMAX * maxblocks);
  L.off_counter = take(sizeof(unsigned int) * 16);
  L.off_dscal = take(sizeof(double) * 16);
  L.off_forceG = take(sizeof(double) * FMAXPAIRS * sh.nvec * sh.g.padded);
  L.off_fslots = take(sizeof(ForceSlots));
  L.off_lz = take(sizeof(double) * 2 * sh.nvec * sh.g.padded * sh.k);  // Lanczos v_{j-1}, v_j (MV layout)
  L.off_lzab = take(sizeof(double) * 2 * (LZMAX + 2));
  // subdomain exchange: held interface lists, slot -> grid index, send and receive buffers
  const long long xcount = sh.sub ? (long long)sh.nvec * sh.n_iface * sh.k + XSCAL : 0;
  L.off_xgi = take(sizeof(int) * sh.xgi.size());
  L.off_xslot = take(sizeof(int) * sh.xslot.size());
  L.off_xinv = take(sh.sub ? sizeof(int) * sh.n_iface : 0);
  L.off_xbuf = take(sizeof(double) * xcount);
  L.off_xrecv = take(sizeof(double) * xcount);
  for (size_t r = 0; r < sh.prec.size(); ++r) {
    const PrecPatch& pp = sh.prec[r];
    long long nbox = (long long)pp.bd[0] * pp.bd[1] * pp.bd[2];
    L.off_s.push_back(take(sizeof(double) * nbox));
    L.off_t.push_back(take(multi ? sizeof(double) * sh.nvec * nbox * sh.k : 0));
    for (int c = 0; c < 3; ++c) L.off_L[c].push_back(take(sizeof(double) * (pp.bd[c] + sh.p + 1) * (sh.p + 1)));
    for (int c = 0; c < 3; ++c) L.off_F[c].push_back(take(2 * sweep_bytes(pp.bd[c], sh.p)));
    for (int c = 0; c < 3; ++c) L.off_E[c].push_back(take(sizeof(double) * 2 * pp.bd[c] * seq_row(sh.p)));
  }
  L.total = o;
  return L;
}

// Assembly scratch per "outer plane" of quadrature points.
size_t plane_bytes(const Shape& sh) {
  const long long nq = (long long)sh.n * (sh.p + 1);
  const long long m = sh.m, W1 = sh.W1;
  if (sh.dim == 3) return sizeof(double) * (11 * nq * nq + nq * W1 * m + W1 * W1 * m * m);
  return sizeof(double) * (6 * nq + W1 * m);
}
size_t asm_fixed_bytes(const Shape& sh) {
  const long long nq = (long long)sh.n * (sh.p + 1);
  const long long mp = sh.dim == 3 ? (long long)sh.m * sh.m * sh.m : (long long)sh.m * sh.m;
  size_t b = align256(sizeof(double) * nq * (sh.p + 1)) * 2 + align256(sizeof(double) * nq) +
             align256(sizeof(double) * 4 * sh.m * sh.W1 * (sh.p + 1) * (sh.p + 1)) +
             align256(sizeof(double) * mp * sh.dim) + 256 * 4;
  return b;
}

__global__ void k_scaling(double* s, int bx, int by, int bz, int lox, int loy, int loz, const double* d0,
                          const double* d1, const double* d2, const double* coefM, const double* diagM, long long S,
                          int nx, int ny, const unsigned char* mask, long long hguard, SymLayout sl) {
  const long long nbox = (long long)bx * by * bz;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nbox) return;
  const int ix = (int)(e % bx), iy = (int)((e / bx) % by), iz = (int)(e / ((long long)bx * by));
  const long long gi = (lox + ix) + (long long)nx * ((loy + iy) + (long long)ny * (loz + iz));
  double v = 0.0;
  if (!mask || mask[gi]) {
    const double dh = d0[ix] * d1[iy] * (d2 ? d2[iz] : 1.0);
    // diag(M): matrix-free array, or the centre offset of the blocked stencil layout
    const long long hr = gi + hguard;  // half-symmetric layout: centre offset = index 0
    const double D = diagM ? diagM[gi]
                           : (sl.xs > 0 ? coefM[sym_index(lox + ix, loy + iy, loz + iz, 0, sl.xs, sl.nseg, ny, (S + 1) / 2)]
                              : hguard >= 0 ? coefM[((hr >> 5) * ((S + 1) / 2)) * 32 + (hr & 31)]
                                            : coefM[((gi >> 5) * S + S / 2) * 32 + (gi & 31)]);
    v = sqrt(dh / D);  // s = sqrt(Dh / D): calM^{-1} = S Mh^{-1} S
  }
  s[e] = v;
}

__global__ void k_altsign(GridDesc g, int nvec, int kk, double* v, const unsigned char* mask) {
  const long long tot = (long long)nvec * g.npts;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const long long i = e % g.npts;
  const int c = (int)(e / g.npts);
  const int ix = (int)(i % g.nx), iy = (int)((i / g.nx) % g.ny), iz = (int)(i / ((long long)g.nx * g.ny));
  double val = ((ix + iy + iz + c) & 1) ? -1.0 : 1.0;
  if (mask && !mask[i]) val = 0.0;
  v[((long long)c * g.padded + g.guard + i) * kk] = val;
}

PrecArgs prec_args(ga_ctx* c, unsigned long long cond, int update) {
  PrecArgs a;
  memset(&a, 0, sizeof(a));
  a.g = c->g; a.nvec = c->nvec; a.kk = c->k; a.p = c->p;
  a.npatch = (int)c->prec.size();
  for (int r = 0; r < a.npatch; ++r) {
    for (int d = 0; d < 3; ++d) {
      a.lo[r][d] = c->prec[r].lo[d]; a.bd[r][d] = c->prec[r].bd[d]; a.L[r][d] = c->prec[r].L[d];
      a.Ff[r][d] = (d < c->dim) ? c->prec[r].Ff[d] : nullptr;
      a.Fb[r][d] = (d < c->dim) ? c->prec[r].Fb[d] : nullptr;
      a.E[r][d] = (d < c->dim) ? c->prec[r].E[d] : nullptr;
      a.clen[r][d] = c->prec[r].clen[d]; a.nchunk[r][d] = c->prec[r].nchunk[d]; a.nlev[r][d] = c->prec[r].nlev[d];
      a.flen[r][d] = (int)c->prec[r].sf[d].buf.size();
    }
    a.s[r] = c->prec[r].s;
    a.t[r] = c->prec[r].t;
  }
  a.mask = c->mask;
  a.x = c->x; a.r = c->r; a.z = c->z; a.q = c->q;
  a.p0 = c->pv; a.p1 = c->pv;  // unfused direction update: p lives in pv (pv1 only for fuse_p)
  a.pcg = c->pcg; a.st = c->st; a.partial = c->partial; a.counter = c->counter;
  a.tol2 = c->d.pcg_rtol * c->d.pcg_rtol;
  a.maxit = c->d.pcg_maxit;
  a.cond = cond;
  a.update = update;
  return a;
}

SpmvArgs spmv_args(ga_ctx* c, int which, const double* x, double* y, int mode) {
  SpmvArgs a;
  memset(&a, 0, sizeof(a));
  a.coef = which == 0 ? c->coefM : c->coefK;
  a.x = x; a.y = y; a.b = c->b;
  a.g = c->g; a.nvec = c->nvec; a.kk = c->k; a.p = c->p;
  a.elastic = (which == 1 && c->nvec == 3) ? 1 : 0;
  a.skip = c->blkskip;
  if (c->half && !a.elastic) { a.half = 1; a.hguard = c->g.guard; }
  if (c->sym && !a.elastic) { a.sym = 1; a.sxs = c->sl.xs; a.snseg = c->sl.nseg; a.symzero = c->symzero; }
  if (c->mf && !a.elastic) {
    a.mf = 1; a.mfstiff = which; a.mfn = c->n; a.mfj0 = 0;
    a.mfW = which == 0 ? c->mfWM : c->mfWK; a.mfws = c->mfws;
    a.mfv = c->mftv; a.mfd = c->mftd;
    if (which == 0) { a.mpT1 = c->mpT1; a.mpT2 = c->mpT2; a.mpT3 = c->mpT3; }
  }
  a.mode = mode;
  // p = z + beta p as a separate elementwise pass (measured faster than forming
  // it on the SpMV input window, which doubles the vector loads)
  a.fuse_p = 0;
  a.z = c->z; a.p0 = c->pv; a.p1 = c->pv1;
  a.tol2 = c->d.pcg_rtol * c->d.pcg_rtol;
  a.refine_rtol2 = c->d.pcg_refine_rtol > 0 ? c->d.pcg_refine_rtol * c->d.pcg_refine_rtol : 0.0;
  a.pcg = c->pcg; a.st = c->st; a.partial = c->partial; a.counter = c->counter;
  return a;
}

VecArgs vec_args(ga_ctx* c) {
  VecArgs a;
  a.g = c->g; a.nvec = c->nvec; a.kk = c->k;
  a.tol2 = c->d.pcg_rtol * c->d.pcg_rtol;
  a.x = c->x; a.r = c->r; a.z = c->z; a.p = c->pv; a.b = c->b;
  a.pcg = c->pcg; a.st = c->st; a.partial = c->partial; a.counter = c->counter;
  a.own = nullptr; a.xsum = nullptr;
  a.mask = c->mask;
  return a;
}

StageArgs stage_args(ga_ctx* c) {
  StageArgs a;
  memset(&a, 0, sizeof(a));
  a.g = c->g; a.nvec = c->nvec; a.k = c->k;
  a.chain = c->chain; a.ysol = c->x; a.pred = c->pred;
  for (int j = 0; j < KMAX; ++j) { a.alpha[j] = c->alpha[j]; a.beta[j] = c->beta[j]; a.gamma[j] = c->gamma[j]; }
  double fact = 1.0, tp = 1.0;
  for (int i = 0; i < 3 * KMAX; ++i) {
    if (i > 0) { fact *= i; tp *= c->d.dt; }
    a.f[i] = tp / fact;
  }
  a.tau = c->d.dt;
  a.unstable2 = c->d.unstable_factor > 0 ? c->d.unstable_factor * c->d.unstable_factor : 0.0;
  a.damp_a0 = c->d.damp_a0; a.damp_a1 = c->d.damp_a1;
  a.st = c->st; a.partial = c->partial; a.counter = c->counter;
  return a;
}

ForceArgs force_args(ga_ctx* c) {
  ForceArgs a;
  memset(&a, 0, sizeof(a));
  a.g = c->g; a.nvec = c->nvec; a.kk = c->k; a.npairs = FMAXPAIRS;
  for (int r = 0; r < FMAXPAIRS; ++r) {
    a.nterms[r] = c->fnterms[r];
    a.G[r] = c->fnterms[r] > 0 ? c->forceG + (size_t)r * c->nvec * c->g.padded : nullptr;
    for (int i = 0; i < c->fnterms[r]; ++i) {
      a.amp[r][i] = c->famp[r][i]; a.omega[r][i] = c->fomega[r][i]; a.phase[r][i] = c->fphase[r][i];
    }
  }
  a.t0 = c->ft0; a.dt = c->d.dt;
  a.b = c->b; a.slots = c->fslots; a.st = c->st;
  return a;
}

PersistArgs persist_args(ga_ctx* ctx) {
  PersistArgs A;
  memset(&A, 0, sizeof(A));
  A.pa = prec_args(ctx, 0ull, 1);
  A.spq = spmv_args(ctx, 0, ctx->pv, ctx->q, SPMV_PQ);
  A.str = spmv_args(ctx, 0, ctx->x, ctx->r, SPMV_TRUERES);
  A.va = vec_args(ctx);
  A.refine = ctx->d.pcg_refine;
  A.refine_rtol2 = ctx->d.pcg_refine_rtol > 0 ? ctx->d.pcg_refine_rtol * ctx->d.pcg_refine_rtol : 0.0;
  A.trace = ctx->trace;
  A.p1 = ctx->pv1;
  return A;
}

// One PCG phase loop: pre-loop preconditioner (sets the loop condition) and a
// conditional WHILE node whose body is one PCG iteration.  `s` is capturing.
ga_status capture_pcg_loop(ga_ctx* ctx, cudaStream_t s) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &graph, &deps, &nd));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));  // 0 unless F1 runs
  launch_precond(prec_args(ctx, (unsigned long long)h, 1), s);
  CK(cudaGetLastError());
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &graph, &deps, &nd));
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, graph, deps, nd, &cp));
  CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(ctx->aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  launch_p_update(vec_args(ctx), ctx->aux);
  launch_spmv(spmv_args(ctx, 0, ctx->pv, ctx->q, SPMV_PQ), ctx->aux);
  launch_precond(prec_args(ctx, (unsigned long long)h, 1), ctx->aux);
  cudaGraph_t outg;
  CK(cudaStreamEndCapture(ctx->aux, &outg));
  return GA_OK;
}

// b is in place: PCG (+ refinement restart) solve of M x = b for all k slots.
ga_status capture_solve(ga_ctx* ctx, cudaStream_t s) {
  if (ctx->persist) {
    if (!launch_pcg_persist(persist_args(ctx), s)) {
      seterr(ctx, "persistent PCG launch failed");
      return GA_ERR_CUDA;
    }
    launch_solve_end(ctx->pcg, ctx->st, s);
    return GA_OK;
  }
  launch_init_from_b(vec_args(ctx), s);
  ga_status rc = capture_pcg_loop(ctx, s);
  if (rc != GA_OK) return rc;
  if (ctx->d.pcg_refine) {
    launch_spmv(spmv_args(ctx, 0, ctx->x, ctx->r, SPMV_TRUERES), s);
    rc = capture_pcg_loop(ctx, s);
    if (rc != GA_OK) return rc;
  }
  launch_solve_end(ctx->pcg, ctx->st, s);
  return GA_OK;
}

enum GraphKind { GK_STEP = 0, GK_SOLVEK = 1, GK_SOLVEB = 2 };

ga_status build_graph(ga_ctx* ctx, cudaStream_t s, GraphKind kind, cudaGraph_t* gout, cudaGraphExec_t* eout) {
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
  if (kind != GK_SOLVEB) launch_spmv(spmv_args(ctx, 1, ctx->pred, ctx->b, SPMV_NEGB), s);
  if (kind != GK_SOLVEB && ctx->forcing) launch_add_forcing(force_args(ctx), s);
  ga_status rc = capture_solve(ctx, s);
  if (rc == GA_OK && kind == GK_STEP) launch_stage(stage_args(ctx), s);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &g);
  if (rc != GA_OK) return rc;
  if (e != cudaSuccess) { seterr(ctx, std::string("capture: ") + cudaGetErrorString(e)); return GA_ERR_CUDA; }
  CK(cudaGraphInstantiate(eout, g, 0));
  *gout = g;
  return GA_OK;
}

// GPU assembly of M and K (sum factorisation, slab by slab).
// bg/boutM/boutK != null: boundary apply (Dirichlet lifting, ga_set_dirichlet): accumulate
// M_fb bg and K_fb bg (free rows, boundary columns) into boutM/boutK instead of assembling.
ga_status assemble(ga_ctx* ctx, const Shape& sh, char* scratch, size_t scratch_bytes, cudaStream_t s,
                   const double* bg = nullptr, double* boutM = nullptr, double* boutK = nullptr) {
  const bool bapply = boutM != nullptr;
  const int dim = sh.dim, p = sh.p, n = sh.n, m = sh.m, W1 = sh.W1, pp1 = p + 1;
  const long long nq = (long long)n * pp1;
  Tables1D T = make_tables(p, n);
  // A tables: A[st][i][o][qq] = phi^(s)_i(q) phi^(t)_{i+o}(q), q = qs(i)+qq
  const size_t asz = (size_t)m * W1 * pp1 * pp1;
  std::vector<double> hA(4 * asz, 0.0);
  for (int st = 0; st < 4; ++st) {
    const int sdr = st >> 1, tdr = st & 1;
    for (int i = 0; i < m; ++i) {
      const int qs = std::max(0, i - p) * pp1, qe = (std::min(n - 1, i) + 1) * pp1;
      for (int o = -p; o <= p; ++o) {
        const int j = i + o;
        if (j < 0 || j >= m) continue;
        for (int q = qs; q < qe; ++q) {
          const int e = q / pp1;
          const int a = i - e, b = j - e;
          if (a < 0 || a > p || b < 0 || b > p) continue;
          const double fi = (sdr ? T.der : T.val)[(size_t)q * pp1 + a];
          const double fj = (tdr ? T.der : T.val)[(size_t)q * pp1 + b];
          hA[st * asz + ((size_t)i * W1 + (o + p)) * pp1 * pp1 + (q - qs)] = fi * fj;
        }
      }
    }
  }
  // carve scratch: fixed tables first
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = scratch + off; off += align256(bytes); return (double*)r; };
  double* dval = take(sizeof(double) * nq * pp1);
  double* dder = take(sizeof(double) * nq * pp1);
  double* dwq = take(sizeof(double) * nq);
  double* dA = take(sizeof(double) * 4 * asz);
  const long long mpow = dim == 3 ? (long long)m * m * m : (long long)m * m;
  double* dctrl = take(sizeof(double) * mpow * dim);
  double* dmin = take(sizeof(double) * 4);
  if (off > scratch_bytes) { seterr(ctx, "scratch too small"); return GA_ERR_OOM; }
  CK(cudaMemcpyAsync(dval, T.val.data(), sizeof(double) * nq * pp1, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dder, T.der.data(), sizeof(double) * nq * pp1, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dwq, T.wq.data(), sizeof(double) * nq, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dA, hA.data(), sizeof(double) * 4 * asz, cudaMemcpyHostToDevice, s));
  double big = 1e300;
  CK(cudaMemcpyAsync(dmin, &big, sizeof(double), cudaMemcpyHostToDevice, s));
  // slab size from the remaining scratch
  const size_t pb = plane_bytes(sh);
  const size_t avail = scratch_bytes - off;
  long long planes = (long long)(avail / (pb + 1024));
  int Z = (int)(planes / pp1) - p;  // rows per slab along the outer direction
  if (Z < 1) { seterr(ctx, "scratch too small for one assembly slab"); return GA_ERR_OOM; }
  Z = std::min(Z, m);
  const long long maxq = (long long)(Z + p) * pp1;
  const long long lowpts = dim == 3 ? nq * nq : nq;
  double* geo = take(sizeof(double) * (dim == 3 ? 10 : 5) * lowpts * maxq);
  double* W = take(sizeof(double) * lowpts * maxq);
  double* X1 = take(sizeof(double) * (dim == 3 ? nq * W1 * m : W1 * m) * maxq);
  double* X2 = dim == 3 ? take(sizeof(double) * W1 * W1 * m * m * maxq) : nullptr;
  if (off > scratch_bytes) { seterr(ctx, "scratch too small (slab)"); return GA_ERR_OOM; }

  const bool mfK = sh.mf && sh.nvec == 1;
  const size_t mbytes = coef_bytes(sh);
  if (!sh.mf && !bapply) CK(cudaMemsetAsync(ctx->coefM, 0, mbytes, s));
  if (!mfK && !bapply) CK(cudaMemsetAsync(ctx->coefK, 0, sh.nvec == 3 ? sizeof(double) * sh.S * sh.g.cs * 9 : mbytes, s));
  // term list: (target block pointer, spec, derivative flags per direction)
  struct Term { double* coef; TermSpec ts; int sflag[3], tflag[3]; int ab; };
  std::vector<Term> terms;
  if (!sh.mf || bapply) {
    Term t;
    memset(&t, 0, sizeof(t));
    t.coef = ctx->coefM;
    t.ts.kind = 0;
    t.ts.scale = sh.nvec == 3 ? ctx->d.density : 1.0;
    terms.push_back(t);
  }
  if (sh.nvec == 1 && (!mfK || bapply)) {
    for (int c = 0; c < dim; ++c)
      for (int e = 0; e < dim; ++e) {
        Term t;
        memset(&t, 0, sizeof(t));
        t.coef = ctx->coefK;
        t.ts.kind = 1; t.ts.c = c; t.ts.e = e; t.ts.scale = ctx->d.omega * ctx->d.omega;
        for (int d = 0; d < 3; ++d) { t.sflag[d] = (d == c); t.tflag[d] = (d == e); }
        terms.push_back(t);
      }
  } else if (sh.nvec == 3) {
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        for (int c = 0; c < 3; ++c)
          for (int e = 0; e < 3; ++e) {
            Term t;
            memset(&t, 0, sizeof(t));
            t.coef = ctx->coefK;
            t.ab = a * 3 + b;
            t.ts.kind = 2; t.ts.a = a; t.ts.b = b; t.ts.c = c; t.ts.e = e;
            t.ts.lam = ctx->d.lame_lambda; t.ts.mu = ctx->d.lame_mu;
            for (int d = 0; d < 3; ++d) { t.sflag[d] = (d == c); t.tflag[d] = (d == e); }
            terms.push_back(t);
          }
  }
  for (size_t r = 0; r < ctx->patches.size(); ++r) {
    CK(cudaMemcpyAsync(dctrl, ctx->patches[r].ctrl.data(), sizeof(double) * mpow * dim, cudaMemcpyHostToDevice, s));
    AsmPatch P;
    P.p = p; P.n = n; P.m = m; P.nq = (int)nq; P.ctrl = dctrl; P.val = dval; P.der = dder; P.wq = dwq;
    for (int r0 = 0; r0 < m; r0 += Z) {
      const int r1 = std::min(m, r0 + Z);
      const int ea = std::max(0, r0 - p), eb = std::min(n, r1);  // elements feeding rows [r0, r1)
      const int qa = ea * pp1, nqs = (eb - ea) * pp1;
      const long long npts_s = lowpts * nqs;
      launch_geometry(P, dim, qa, nqs, geo, npts_s, dmin, s);
      if (sh.mf && !bapply) {
        // Gauss-point data of the matrix-free operators for quadrature planes [qa, qa + nqs)
        // (overlapping slabs rewrite identical values): W_M = density w|J|, and for the scalar
        // K the symmetric omega^2 w|J| (J^-1 J^-T)_{ce}, c <= e (SoA, stride mfws)
        TermSpec tm;
        memset(&tm, 0, sizeof(tm));
        tm.kind = 0;
        tm.scale = sh.nvec == 3 ? ctx->d.density : 1.0;
        launch_wterm(geo, npts_s, npts_s, dim, tm, ctx->mfWM + (long long)qa * lowpts, s);
        if (mfK) {
          int idx = 0;
          for (int c = 0; c < dim; ++c)
            for (int e = c; e < dim; ++e, ++idx) {
              TermSpec tk;
              memset(&tk, 0, sizeof(tk));
              tk.kind = 1; tk.c = c; tk.e = e; tk.scale = ctx->d.omega * ctx->d.omega;
              launch_wterm(geo, npts_s, npts_s, dim, tk, ctx->mfWK + idx * ctx->mfws + (long long)qa * lowpts, s);
            }
        }
      }
      for (const Term& t : terms) {
        launch_wterm(geo, npts_s, npts_s, dim, t.ts, W, s);
        const double* A0 = dA + (size_t)(t.sflag[0] * 2 + t.tflag[0]) * asz;
        const double* A1 = dA + (size_t)(t.sflag[1] * 2 + t.tflag[1]) * asz;
        const double* A2 = dA + (size_t)(t.sflag[2] * 2 + t.tflag[2]) * asz;
        ContractDesc c1;
        memset(&c1, 0, sizeof(c1));
        c1.W1 = W1; c1.m = m; c1.p = p; c1.n = n; c1.qoff = 0;
        c1.nouter = (dim == 3 ? nq : 1) * nqs; c1.nmid = 1; c1.ninner = 1;
        c1.in_s_outer = nq; c1.in_s_q = 1; c1.in_s_mid = 0; c1.in_s_inner = 0;
        c1.out_s_outer = (long long)W1 * m; c1.out_s_o = m; c1.out_s_mid = 0; c1.out_s_i = 1; c1.out_s_inner = 0;
        launch_contract(W, X1, A0, c1, s);
        FinalDesc f;
        memset(&f, 0, sizeof(f));
        f.W1 = W1; f.m = m; f.p = p; f.n = n; f.qoff = qa; f.r0 = r0; f.r1 = r1;
        for (int d = 0; d < 3; ++d) { f.cell[d] = ctx->sub ? 0 : ctx->patches[r].cell[d]; f.org[d] = ctx->org[d]; }
        f.G[0] = sh.g.nx; f.G[1] = sh.g.ny; f.G[2] = sh.g.nz;
        f.npts = sh.g.cs;
        f.S = sh.S;
        f.ncf = (t.coef == ctx->coefK && sh.nvec == 3) ? 9 : 1;
        f.ab = t.ab;
        f.mask = ctx->mask;
        f.half = (sh.half && f.ncf == 1) ? 1 : 0;  // the elastic K stays full
        f.hguard = sh.g.guard;
        f.sym = sh.sym ? 1 : 0; f.sxs = sh.sl.xs; f.snseg = sh.sl.nseg;
        if (bapply) { f.bg = bg; f.bout = (t.coef == ctx->coefM) ? boutM : boutK; }
        if (dim == 3) {
          ContractDesc c2;
          memset(&c2, 0, sizeof(c2));
          c2.W1 = W1; c2.m = m; c2.p = p; c2.n = n; c2.qoff = 0;
          c2.nouter = nqs; c2.nmid = W1; c2.ninner = m;
          c2.in_s_outer = nq * W1 * m; c2.in_s_q = (long long)W1 * m; c2.in_s_mid = m; c2.in_s_inner = 1;
          c2.out_s_outer = (long long)W1 * W1 * m * m; c2.out_s_o = (long long)W1 * m * m; c2.out_s_mid = (long long)m * m;
          c2.out_s_i = m; c2.out_s_inner = 1;
          launch_contract(X1, X2, A1, c2, s);
          launch_contract_final(3, X2, A2, f, t.coef, s);
        } else {
          launch_contract_final(2, X1, A1, f, t.coef, s);
        }
        CK(cudaGetLastError());
      }
    }
  }
  double hmin = 0;
  CK(cudaMemcpyAsync(&hmin, dmin, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!(hmin > 0.0)) {
    char buf[128];
    snprintf(buf, sizeof buf, "non-positive Jacobian determinant (min |J| = %.3e)", hmin);
    seterr(ctx, buf);
    return GA_ERR_GEOMETRY;
  }
  return GA_OK;
}

// Direct execution of a graph kind (GA_NO_GRAPH): same kernels, PCG loop
// condition evaluated on the host after a synchronisation per iteration.
static void dbg(ga_ctx* ctx, cudaStream_t s, const char* what) {
  static int on = -1;
  if (on < 0) { const char* e = getenv("GA_DEBUG"); on = e && *e && *e != '0'; }
  if (!on) return;
  unsigned int cnt = 0;
  PcgState h;
  cudaMemcpyAsync(&cnt, ctx->counter, sizeof(cnt), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&h, ctx->pcg, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  fprintf(stderr, "[ga dbg] %-10s err=%d counter=%u iter=%d first=%d bb=%.3e,%.3e rr=%.3e,%.3e act=%d,%d its=%d,%d alpha=%.3e\n", what, (int)e,
          cnt, h.iter, h.first, h.bb[0], h.bb[1], h.rr[0], h.rr[1], h.active[0], h.active[1], h.its[0], h.its[1], h.alpha[0]);
}

ga_status run_pcg_loop_direct(ga_ctx* ctx, cudaStream_t s) {
  launch_precond(prec_args(ctx, 0ull, 1), s);
  dbg(ctx, s, "precond0");
  for (int guard_it = 0; guard_it < 100000; ++guard_it) {
    PcgState h;
    DevStatus hs;
    CK(cudaMemcpyAsync(&h, ctx->pcg, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs, ctx->st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int any = 0;
    for (int j = 0; j < ctx->k; ++j) any |= h.active[j];
    if (!any || hs.status != 0 || h.iter >= ctx->d.pcg_maxit) break;
    launch_p_update(vec_args(ctx), s);
    launch_spmv(spmv_args(ctx, 0, ctx->pv, ctx->q, SPMV_PQ), s);
    dbg(ctx, s, "spmv_pq");
    launch_precond(prec_args(ctx, 0ull, 1), s);
    dbg(ctx, s, "precond");
  }
  return GA_OK;
}

ga_status run_direct(ga_ctx* ctx, GraphKind kind, cudaStream_t s) {
  if (kind != GK_SOLVEB) launch_spmv(spmv_args(ctx, 1, ctx->pred, ctx->b, SPMV_NEGB), s);
  if (kind != GK_SOLVEB && ctx->forcing) launch_add_forcing(force_args(ctx), s);
  dbg(ctx, s, "negb");
  if (ctx->persist) {
    if (!launch_pcg_persist(persist_args(ctx), s)) {
      seterr(ctx, "persistent PCG launch failed");
      return GA_ERR_CUDA;
    }
    launch_solve_end(ctx->pcg, ctx->st, s);
    if (kind == GK_STEP) launch_stage(stage_args(ctx), s);
    CK(cudaGetLastError());
    return GA_OK;
  }
  launch_init_from_b(vec_args(ctx), s);
  dbg(ctx, s, "init_b");
  ga_status rc = run_pcg_loop_direct(ctx, s);
  if (rc != GA_OK) return rc;
  if (ctx->d.pcg_refine) {
    launch_spmv(spmv_args(ctx, 0, ctx->x, ctx->r, SPMV_TRUERES), s);
    rc = run_pcg_loop_direct(ctx, s);
    if (rc != GA_OK) return rc;
  }
  launch_solve_end(ctx->pcg, ctx->st, s);
  if (kind == GK_STEP) launch_stage(stage_args(ctx), s);
  CK(cudaGetLastError());
  return GA_OK;
}

ga_status run_kind(ga_ctx* ctx, GraphKind kind, cudaStream_t s) {
  if (ctx->nograph) return run_direct(ctx, kind, s);
  cudaGraphExec_t e = kind == GK_STEP ? ctx->g_step : (kind == GK_SOLVEK ? ctx->g_solveK : ctx->g_solveB);
  CK(cudaGraphLaunch(e, s));
  return GA_OK;
}

}  // namespace gaint

using namespace gaint;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

ga_status ga_params(int k, double rho_b, double rho_s, int param_set, double* alpha, double* beta, double* gamma,
                    double* alpha_f, double* theta_max) {
  if (param_set != 0 && param_set != 1) return GA_ERR_ARG;
  int rc = scheme_params(k, rho_b, rho_s, param_set, alpha, beta, gamma, alpha_f, theta_max);
  if (rc == -1) return GA_ERR_ARG;
  if (rc != 0) return GA_ERR_PARAM;
  return GA_OK;
}

ga_status ga_query(const ga_desc* desc, size_t* n_free, size_t* workspace_bytes, size_t* scratch_bytes,
                   size_t* scratch_min) {
  ga_status rc = validate(desc, nullptr);
  if (rc != GA_OK) return rc;
  Shape sh;
  rc = make_shape(desc, sh, nullptr, false);
  if (rc != GA_OK) return rc;
  Layout L = make_layout(sh);
  if (n_free) *n_free = (size_t)(sh.nfree * sh.nvec);
  if (workspace_bytes) *workspace_bytes = L.total;
  const size_t fixed = asm_fixed_bytes(sh), pb = plane_bytes(sh) + 1024;
  const size_t smin = fixed + pb * (size_t)(sh.p + 2) * (sh.p + 1) + (1 << 20);
  const size_t sall = fixed + pb * (size_t)(sh.m + sh.p + 1) * (sh.p + 1) + (1 << 20);
  const size_t cap = (size_t)8 << 30;
  if (scratch_min) *scratch_min = smin;
  if (scratch_bytes) *scratch_bytes = std::max(smin, std::min(sall, cap));
  return GA_OK;
}

}  // extern "C"

// diag(M) of the local operator from the stencil centre (subdomain contexts)
__global__ void k_centre(double* diag, long long npts, const double* coefM, long long S, long long hguard) {
  const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= npts) return;
  const long long hr = gi + hguard;
  diag[gi] = hguard >= 0 ? coefM[((hr >> 5) * ((S + 1) / 2)) * 32 + (hr & 31)]
                         : coefM[((gi >> 5) * S + S / 2) * 32 + (gi & 31)];
}

namespace gaint {
ga_status compute_scaling(ga_ctx* ctx, cudaStream_t s) {
  for (size_t r = 0; r < ctx->prec.size(); ++r) {
    PrecPatch& pp = ctx->prec[r];
    const long long nbox = (long long)pp.bd[0] * pp.bd[1] * pp.bd[2];
    // 1D diagonals of the parametric mass go to the q vector temporarily
    double* tmp = ctx->q;
    const double* dd[3] = {nullptr, nullptr, nullptr};
    size_t o = 0;
    for (int d = 0; d < ctx->dim; ++d) {
      CK(cudaMemcpyAsync(tmp + o, pp.hdiag[d].data(), sizeof(double) * pp.bd[d], cudaMemcpyHostToDevice, s));
      dd[d] = tmp + o;
      o += pp.bd[d];
    }
    k_scaling<<<(unsigned int)((nbox + 255) / 256), 256, 0, s>>>(pp.s, pp.bd[0], pp.bd[1], pp.bd[2], pp.lo[0], pp.lo[1],
                                                                 pp.lo[2], dd[0], dd[1], ctx->dim == 3 ? dd[2] : nullptr,
                                                                 ctx->coefM, ctx->diagM, ctx->S, ctx->g.nx, ctx->g.ny,
                                                                 ctx->mask, ctx->half ? ctx->g.guard : -1,
                                                                 ctx->sym ? ctx->sl : SymLayout{0, 0});
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));  // tmp reused by the next patch
  }
  CK(cudaMemsetAsync(ctx->q, 0, sizeof(double) * ctx->nvec * ctx->g.padded * ctx->k, s));
  return GA_OK;
}
}  // namespace gaint

extern "C" {

ga_status ga_create(const ga_desc* desc, void* d_workspace, size_t workspace_bytes, void* d_scratch,
                    size_t scratch_bytes, void* stream, ga_ctx** out) {
  if (out) *out = nullptr;
  if (!out) return GA_ERR_ARG;
  ga_ctx* ctx = new ga_ctx();
  ga_status rc = validate(desc, ctx);
  if (rc != GA_OK) { delete ctx; return rc; }
  ctx->d = *desc;
  ctx->d.patches = nullptr;
  Shape sh;
  rc = make_shape(desc, sh, ctx, true);
  if (rc != GA_OK) { delete ctx; return rc; }
  Layout L = make_layout(sh);
  if (!d_workspace || workspace_bytes < L.total || ((size_t)d_workspace & 255)) {
    seterr(ctx, "workspace too small or misaligned");
    delete ctx;
    return GA_ERR_OOM;
  }
  if (!d_scratch) { seterr(ctx, "scratch is NULL"); delete ctx; return GA_ERR_OOM; }
  cudaStream_t s = (cudaStream_t)stream;
  ctx->dim = sh.dim; ctx->nvec = sh.nvec; ctx->p = sh.p; ctx->n = sh.n; ctx->m = sh.m; ctx->k = sh.k; ctx->W1 = sh.W1;
  ctx->S = sh.S; ctx->g = sh.g; ctx->nfree = sh.nfree;
  ctx->hmap = sh.map; ctx->hmask = sh.mask; ctx->hlocal = sh.local;
  scheme_params(desc->k, desc->rho_b, desc->rho_s, desc->param_set, ctx->alpha, ctx->beta, ctx->gamma,
                ctx->alpha_f, &ctx->theta_max);
  const long long mpow = sh.dim == 3 ? (long long)sh.m * sh.m * sh.m : (long long)sh.m * sh.m;
  for (int r = 0; r < desc->npatch; ++r) {
    PatchHost ph;
    memcpy(ph.cell, desc->patches[r].cell, sizeof(ph.cell));
    ph.ctrl.assign(desc->patches[r].ctrl, desc->patches[r].ctrl + mpow * sh.dim);
    for (double v : ph.ctrl)
      if (!std::isfinite(v)) { seterr(ctx, "non-finite control point"); delete ctx; return GA_ERR_ARG; }
    ctx->patches.push_back(ph);
  }
  char* ws = (char*)d_workspace;
  ctx->ws = ws; ctx->ws_bytes = workspace_bytes;
  ctx->coefM = (double*)(ws + L.off_coefM);
  ctx->coefK = (double*)(ws + L.off_coefK);
  ctx->mf = sh.mf;
  ctx->half = sh.half;
  ctx->sym = sh.sym;
  ctx->sl = sh.sl;
  ctx->symzero = (double*)(ws + L.off_symzero);
  if (sh.mf) {
    const long long nq = (long long)sh.n * (sh.p + 1);
    ctx->mfws = sh.dim == 3 ? nq * nq * nq : nq * nq;
    ctx->mfWM = (double*)(ws + L.off_mfWM);
    ctx->mfWK = sh.nvec == 1 ? (double*)(ws + L.off_mfWK) : nullptr;
    ctx->mftv = (double*)(ws + L.off_mftab);
    ctx->mftd = ctx->mftv + nq * (sh.p + 1);
    ctx->diagM = (double*)(ws + L.off_diag);
    if (sh.dim == 3) {
      ctx->mpT1 = (double*)(ws + L.off_mpT1);
      ctx->mpT2 = (double*)(ws + L.off_mpT2);
      ctx->mpT3 = (double*)(ws + L.off_mpT3);
    }
  }
  ctx->chain = (double*)(ws + L.off_chain);
  double** mv[8] = {&ctx->pred, &ctx->b, &ctx->x, &ctx->r, &ctx->z, &ctx->pv, &ctx->q, &ctx->pv1};
  for (int i = 0; i < 8; ++i) *mv[i] = (double*)(ws + L.off_mv[i]);
  const bool multi = desc->npatch > 1 || sh.sub;
  ctx->sub = sh.sub;
  for (int c = 0; c < 3; ++c) ctx->org[c] = sh.org[c];
  if (sh.sub) {
    ctx->n_iface = sh.n_iface;
    ctx->nxl = (long long)sh.xgi.size();
    ctx->xgi = (int*)(ws + L.off_xgi);
    ctx->xslot = (int*)(ws + L.off_xslot);
    ctx->xinv = (int*)(ws + L.off_xinv);
    ctx->xcount = (long long)sh.nvec * sh.n_iface * sh.k + XSCAL;
    ctx->xbuf = (double*)(ws + L.off_xbuf);
    ctx->xrecv = (double*)(ws + L.off_xrecv);
    ctx->diagM = (double*)(ws + L.off_diag);
  }
  ctx->mask = multi ? (unsigned char*)(ws + L.off_mask) : nullptr;
  ctx->blkskip = multi ? (unsigned char*)(ws + L.off_skip) : nullptr;
  ctx->map = multi ? (long long*)(ws + L.off_map) : nullptr;
  ctx->pcg = (PcgState*)(ws + L.off_pcg);
  ctx->st = (DevStatus*)(ws + L.off_st);
  ctx->partial = (double*)(ws + L.off_partial);
  ctx->counter = (unsigned int*)(ws + L.off_counter);
  ctx->dscal = (double*)(ws + L.off_dscal);
  ctx->forceG = (double*)(ws + L.off_forceG);
  ctx->fslots = (ForceSlots*)(ws + L.off_fslots);
  ctx->lzv = (double*)(ws + L.off_lz);
  ctx->lzab = (double*)(ws + L.off_lzab);
#define CKD(call)                           \
  do {                                      \
    cudaError_t e_ = (call);                \
    if (e_ != cudaSuccess) {                \
      seterr(ctx, std::string(#call) + ": " + cudaGetErrorString(e_)); \
      ga_destroy(ctx);                      \
      return GA_ERR_CUDA;                   \
    }                                       \
  } while (0)
  CKD(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
  CKD(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
  // zero everything small + vectors (guards must be zero/finite)
  CKD(cudaMemsetAsync(ws + L.off_chain, 0, L.off_mask - L.off_chain, s));
  CKD(cudaMemsetAsync(ws + L.off_pcg, 0, L.off_dscal + 256 - L.off_pcg, s));
  if (sh.sym) CKD(cudaMemsetAsync(ws + L.off_symzero, 0, sizeof(double) * ((sh.S + 1) / 2) * SYM_STRIDE, s));
  if (multi) {
    CKD(cudaMemcpyAsync(ctx->mask, sh.mask.data(), sh.g.npts, cudaMemcpyHostToDevice, s));
    {
      const long long nrb = (sh.g.npts + 31) / 32;
      std::vector<unsigned char> skip((size_t)nrb, 1);
      for (long long gi = 0; gi < sh.g.npts; ++gi)
        if (sh.mask[gi]) skip[(size_t)(gi >> 5)] = 0;
      CKD(cudaMemcpy(ctx->blkskip, skip.data(), (size_t)nrb, cudaMemcpyHostToDevice));
    }
    CKD(cudaMemcpyAsync(ctx->map, sh.map.data(), sizeof(long long) * sh.nfree, cudaMemcpyHostToDevice, s));
  }
  std::vector<int> hxinv;
  if (sh.sub) {
    hxinv.assign((size_t)sh.n_iface, -1);
    for (size_t i = 0; i < sh.xgi.size(); ++i) hxinv[(size_t)sh.xslot[i]] = sh.xgi[i];
    if (!sh.xgi.empty()) {
      CKD(cudaMemcpyAsync(ctx->xgi, sh.xgi.data(), sizeof(int) * sh.xgi.size(), cudaMemcpyHostToDevice, s));
      CKD(cudaMemcpyAsync(ctx->xslot, sh.xslot.data(), sizeof(int) * sh.xslot.size(), cudaMemcpyHostToDevice, s));
    }
    if (!hxinv.empty()) CKD(cudaMemcpyAsync(ctx->xinv, hxinv.data(), sizeof(int) * hxinv.size(), cudaMemcpyHostToDevice, s));
    CKD(cudaMemsetAsync(ctx->xbuf, 0, sizeof(double) * 2 * ctx->xcount, s));
    CKD(cudaStreamSynchronize(s));  // hxinv is a stack vector
  }
  if (sh.mf) {  // 1D basis tables of the matrix-free apply (host_math.cpp)
    Tables1D T0 = make_tables(sh.p, sh.n);
    CKD(cudaMemcpyAsync(ctx->mftv, T0.val.data(), sizeof(double) * T0.val.size(), cudaMemcpyHostToDevice, s));
    CKD(cudaMemcpyAsync(ctx->mftd, T0.der.data(), sizeof(double) * T0.der.size(), cudaMemcpyHostToDevice, s));
  }
  // assembly
  rc = assemble(ctx, sh, (char*)d_scratch, scratch_bytes, s);
  if (rc != GA_OK) { ga_destroy(ctx); return rc; }
  if (sh.mf) {
    launch_mf_diag(sh.g, sh.p, sh.n, ctx->mfWM, ctx->mftv, ctx->diagM, s);
    CKD(cudaGetLastError());
  }
  // preconditioner: per patch 1D factors (host) and scaling s (device)
  Tables1D T = make_tables(sh.p, sh.n);
  std::vector<double> band = param_mass_band(T);
  ctx->prec = sh.prec;
  for (size_t r = 0; r < ctx->prec.size(); ++r) {
    PrecPatch& pp = ctx->prec[r];
    pp.s = (double*)(ws + L.off_s[r]);
    pp.t = multi ? (double*)(ws + L.off_t[r]) : nullptr;
    for (int d = 0; d < 3; ++d) {
      pp.L[d] = (double*)(ws + L.off_L[d][r]);
      if (d >= sh.dim) continue;
      std::vector<double> Lf, diag;
      if (!band_cholesky(band, sh.p, pp.llo[d], pp.llo[d] + pp.bd[d] - 1, Lf, diag)) {
        seterr(ctx, "parametric mass matrix not SPD");
        ga_destroy(ctx);
        return GA_ERR_ARG;
      }
      Lf.resize((size_t)(pp.bd[d] + sh.p + 1) * (sh.p + 1), 0.0);  // P zero rows for the backward sweep
      pp.hL[d] = Lf;
      pp.hdiag[d] = diag;
      // chunks per line: enough threads (slots x chunks) to fill the GPU, <= 64; the
      // slots of all patches run in one launch (additive Schwarz)
      long long slots = 0;
      for (const PrecPatch& q : ctx->prec) {
        long long sl = (long long)sh.nvec * sh.k;
        for (int e = 0; e < sh.dim; ++e)
          if (e != d) sl *= q.bd[e];
        slots += sl;
      }
      static long long thr_target = -1;
      if (thr_target < 0) {
        const char* e = getenv("GA_CHUNK_THREADS");
        thr_target = e ? atoll(e) : 150000;
      }
      const long long tt = thr_target;  // measured on C5: more chunks (shorter serial chains) is faster
      const int ctarget = (int)std::max(2LL, std::min(64LL, (tt + slots - 1) / slots));
      pp.sf[d] = make_sweep(Lf, pp.bd[d], sh.p, false, ctarget);
      pp.sb[d] = make_sweep(Lf, pp.bd[d], sh.p, true, ctarget);
      pp.Ff[d] = (double*)(ws + L.off_F[d][r]);
      pp.Fb[d] = (double*)(ws + L.off_F[d][r] + sweep_bytes(pp.bd[d], sh.p));
      pp.clen[d] = pp.sf[d].clen; pp.nchunk[d] = pp.sf[d].C; pp.nlev[d] = pp.sf[d].L;
      CKD(cudaMemcpyAsync(pp.Ff[d], pp.sf[d].buf.data(), sizeof(double) * pp.sf[d].buf.size(), cudaMemcpyHostToDevice, s));
      CKD(cudaMemcpyAsync(pp.Fb[d], pp.sb[d].buf.data(), sizeof(double) * pp.sb[d].buf.size(), cudaMemcpyHostToDevice, s));
      CKD(cudaMemcpyAsync(pp.L[d], pp.hL[d].data(), sizeof(double) * Lf.size(), cudaMemcpyHostToDevice, s));
      pp.hE[d] = make_seq(Lf, pp.bd[d], sh.p);
      pp.E[d] = (double*)(ws + L.off_E[d][r]);
      CKD(cudaMemcpyAsync(pp.E[d], pp.hE[d].data(), sizeof(double) * pp.hE[d].size(), cudaMemcpyHostToDevice, s));
    }
  }
  if (sh.sub) {  // local diag(M) (the group sums the interface copies and recomputes the scalings)
    k_centre<<<(unsigned int)((sh.g.npts + 255) / 256), 256, 0, s>>>(ctx->diagM, sh.g.npts, ctx->coefM, ctx->S,
                                                                    sh.half ? sh.g.guard : -1);
    CKD(cudaGetLastError());
  }
  rc = compute_scaling(ctx, s);
  if (rc != GA_OK) { ga_destroy(ctx); return rc; }
  line_seq_prepare(sh.p);
  CKD(cudaMemsetAsync(ctx->q, 0, sizeof(double) * sh.nvec * sh.g.padded * sh.k, s));
  // graphs
  // graphs are captured on a private stream (the caller's may be the legacy stream)
  {
    const char* e = getenv("GA_NO_GRAPH");
    ctx->nograph = e && *e && *e != '0';
    const char* pe = getenv("GA_PERSIST");  // 0: never, 1: always when supported, unset: auto (small grids)
    // latency-bound regime: little data per PCG phase (C2-like); bandwidth-bound grids keep the graph path
    const bool small = (long long)sh.g.npts * sh.k <= 600000 && (double)sh.S * sh.g.npts * 8.0 <= 64e6;
    const bool want = pe ? (*pe != '0') : small;
    ctx->persist = want && !ctx->mf && !ctx->half && !ctx->sub && persist_supported(persist_args(ctx));
    if (ctx->sub) ctx->nograph = true;  // subdomains are stepped by their ga_group (dist.cu)
    const char* te = getenv("GA_TRACE");
    if (te && *te && *te != '0') {
      cudaMalloc(&ctx->trace, 8192 * sizeof(long long));  // debug only
      cudaMemset(ctx->trace, 0, 8192 * sizeof(long long));
    }
  }
  if (!ctx->nograph && !ctx->sub) {
    rc = build_graph(ctx, ctx->cap, GK_STEP, &ctx->gr_step, &ctx->g_step);
    if (rc == GA_OK) rc = build_graph(ctx, ctx->cap, GK_SOLVEK, &ctx->gr_solveK, &ctx->g_solveK);
    if (rc == GA_OK) rc = build_graph(ctx, ctx->cap, GK_SOLVEB, &ctx->gr_solveB, &ctx->g_solveB);
  }
  if (rc != GA_OK) { ga_destroy(ctx); return rc; }
  CKD(cudaStreamSynchronize(s));
  *out = ctx;
  return GA_OK;
}

// Lanczos for M^{-1} K in the M inner product (slot 0 of MV-layout vectors, stride kk):
// w = A v_j - alpha_j v_j - beta_{j-1} v_{j-1} with A v_j = -x (x = M^{-1}(-K v_j)),
// alpha_j = v_j.K v_j = -(v_j . b) (b = -K v_j); written into vn (= v_{j-1}'s buffer)
__global__ void k_lz_update(GridDesc g, int nvec, int kk, const double* x, const double* v, double* vn,
                            const double* dal, const double* dbe, const unsigned char* mask) {
  const long long tot = (long long)nvec * g.npts;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const long long c = e / g.npts, i = e - c * g.npts;
  const long long o = (c * g.padded + g.guard + i) * kk;
  const double al = -dal[0], be = dbe[0];
  double w = -x[o] - al * v[o] - be * vn[o];
  if (mask && !mask[i]) w = 0.0;
  vn[o] = w;
}
// v *= 1 / sqrt(d[0]) and record beta = sqrt(d[0]) in rec (device)
__global__ void k_lz_norm(GridDesc g, int nvec, int kk, double* v, const double* d, double* rec) {
  const double b = sqrt(fmax(d[0], 0.0));
  if (blockIdx.x == 0 && threadIdx.x == 0) rec[0] = b;
  const long long tot = (long long)nvec * g.npts;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot || b == 0.0) return;
  const long long c = e / g.npts, i = e - c * g.npts;
  v[(c * g.padded + g.guard + i) * kk] *= 1.0 / b;
}
__global__ void k_lz_copy_alpha(const double* src, double* dst) { dst[0] = -src[0]; }

__global__ void k_reset_status(DevStatus* st, PcgState* pc, int keep_time) {
  const long long tstep = keep_time ? st->tstep : 0;
  memset(st, 0, sizeof(DevStatus));
  st->tstep = tstep;
  st->fail_step = -1;
  st->fail_block = -1;
  memset(pc, 0, sizeof(PcgState));
}

}  // extern "C"

namespace gaint {
// keep_time: the simulation step index (forcing clock) survives, e.g. ga_set_chain on a resume
void reset_status(ga_ctx* ctx, cudaStream_t s, int keep_time) {
  k_reset_status<<<1, 1, 0, s>>>(ctx->st, ctx->pcg, keep_time);
}

}  // namespace gaint

extern "C" {

static ga_status check_ctx(ga_ctx* ctx) {
  if (!ctx) { seterr(nullptr, "ctx is NULL"); return GA_ERR_ARG; }
  return GA_OK;
}

// entry points that step or solve need the whole problem: a subdomain goes through its ga_group
static ga_status check_whole(ga_ctx* ctx) {
  if (!ctx) { seterr(nullptr, "ctx is NULL"); return GA_ERR_ARG; }
  if (ctx->sub) { seterr(ctx, "subdomain context: step and solve through its ga_group"); return GA_ERR_ARG; }
  return GA_OK;
}

}  // extern "C"

namespace gaint {
// step slot table: block j (slot j-1) takes F^{(3j-3)} at t_n + alpha_fj dt (eq:ho1)
ga_status set_step_slots(ga_ctx* ctx, cudaStream_t s) {
  if (!ctx->forcing) return GA_OK;
  ForceSlots fs;
  memset(&fs, 0, sizeof(fs));
  for (int j = 0; j < ctx->k; ++j) { fs.active[j] = 1; fs.order[j] = 3 * j; fs.toff[j] = ctx->alpha_f[j] * ctx->d.dt; }
  CK(cudaMemcpyAsync(ctx->fslots, &fs, sizeof(fs), cudaMemcpyHostToDevice, s));
  return GA_OK;
}

ga_status set_predictors_and_norm(ga_ctx* ctx, cudaStream_t s) {
  {
    ga_status rc = set_step_slots(ctx, s);
    if (rc != GA_OK) return rc;
  }
  launch_predict(stage_args(ctx), s);
  // reference of the instability detector: ||U0||^2 + dt^2 ||V0||^2 (0 from rest: the first
  // non-zero ||U_n||^2 is adopted by the stage kernel)
  const long long vstride = (long long)ctx->nvec * ctx->g.padded;
  launch_ref_norm(ctx->g, ctx->nvec, ctx->chain, ctx->chain + vstride, ctx->d.dt, ctx->st, ctx->partial,
                  ctx->counter, s);
  CK(cudaGetLastError());
  return GA_OK;
}

}  // namespace gaint

extern "C" {

ga_status ga_set_state(ga_ctx* ctx, const double* d_u0, const double* d_v0, void* stream) {
  ga_status rc = check_whole(ctx);
  if (rc != GA_OK) return rc;
  if (!d_u0) { seterr(ctx, "u0 is NULL"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const int k = ctx->k, nvec = ctx->nvec;
  const long long vstride = (long long)nvec * ctx->g.padded;
  reset_status(ctx, s);
  CK(cudaMemsetAsync(ctx->chain, 0, sizeof(double) * 3 * k * vstride, s));
  launch_api_to_grid(ctx->g, nvec, ctx->nfree, ctx->map, d_u0, ctx->chain, 1, 0, ctx->st, s);
  if (d_v0) launch_api_to_grid(ctx->g, nvec, ctx->nfree, ctx->map, d_v0, ctx->chain + vstride, 1, 0, ctx->st, s);
  CK(cudaGetLastError());
  // c_m = M^{-1}(-K c_{m-2}), m = 2..3k-1, two at a time when k >= 2
  // damping couples c_m to c_{m-1}: the chain entries are then solved one at a time
  const bool damped = ctx->d.damp_a0 != 0.0 || ctx->d.damp_a1 != 0.0;
  const int batch = damped ? 1 : std::min(2, k);
  for (int m0 = 2; m0 <= 3 * k - 1; m0 += batch) {
    int src[KMAX] = {-1, -1, -1, -1}, dst[KMAX] = {-1, -1, -1, -1}, src2[KMAX] = {-1, -1, -1, -1};
    for (int j = 0; j < batch; ++j)
      if (m0 + j <= 3 * k - 1) { src[j] = m0 + j - 2; dst[j] = m0 + j; if (damped) src2[j] = m0 + j - 1; }
    if (ctx->forcing) {  // c_m = M^{-1}(F^{(m-2)}(t0) - K c_{m-2}) (eq:ho1 differentiated)
      ForceSlots fs;
      memset(&fs, 0, sizeof(fs));
      for (int j = 0; j < batch; ++j)
        if (dst[j] >= 0) { fs.active[j] = 1; fs.order[j] = dst[j] - 2; fs.toff[j] = 0.0; }
      CK(cudaMemcpyAsync(ctx->fslots, &fs, sizeof(fs), cudaMemcpyHostToDevice, s));
    }
    // c_m = M^{-1}(F^{(m-2)} - K (c_{m-2} + a1 c_{m-1})) - a0 c_{m-1}  (Rayleigh C = a0 M + a1 K)
    launch_pack(ctx->g, nvec, k, ctx->chain, src, ctx->pred, ctx->st, s, src2, ctx->d.damp_a1);
    rc = run_kind(ctx, GK_SOLVEK, s);
    if (rc != GA_OK) return rc;
    launch_unpack(ctx->g, nvec, k, ctx->x, dst, ctx->chain, ctx->st, s, src2, ctx->d.damp_a0);
    CK(cudaGetLastError());
  }
  return set_predictors_and_norm(ctx, s);
}

// (re)capture the graphs after a change of the forcing pairs and refresh the step slots
static ga_status rebuild_forcing_graphs(ga_ctx* ctx, cudaStream_t s) {
  ga_status rc = GA_OK;
  ctx->forcing = false;
  for (int r = 0; r < FMAXPAIRS; ++r) ctx->forcing |= ctx->fnterms[r] > 0;
  CK(cudaStreamSynchronize(s));
  if (!ctx->nograph) {
    cudaGraphExec_t* ex[3] = {&ctx->g_step, &ctx->g_solveK, &ctx->g_solveB};
    cudaGraph_t* gr[3] = {&ctx->gr_step, &ctx->gr_solveK, &ctx->gr_solveB};
    for (int i = 0; i < 3; ++i) {
      if (*ex[i]) cudaGraphExecDestroy(*ex[i]);
      if (*gr[i]) cudaGraphDestroy(*gr[i]);
      *ex[i] = nullptr; *gr[i] = nullptr;
    }
    rc = build_graph(ctx, ctx->cap, GK_STEP, &ctx->gr_step, &ctx->g_step);
    if (rc == GA_OK) rc = build_graph(ctx, ctx->cap, GK_SOLVEK, &ctx->gr_solveK, &ctx->g_solveK);
    if (rc == GA_OK) rc = build_graph(ctx, ctx->cap, GK_SOLVEB, &ctx->gr_solveB, &ctx->g_solveB);
    if (rc != GA_OK) return rc;
  }
  return set_step_slots(ctx, s);
}

ga_status ga_set_forcing(ga_ctx* ctx, const double* d_G, int nterms, const double* amp, const double* omega,
                         const double* phase, double t0, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const bool on = d_G != nullptr && nterms > 0;
  if (on && (nterms > FMAXTERMS || !amp || !omega || !phase)) {
    seterr(ctx, "forcing: 1..8 terms with amp, omega and phase arrays required");
    return GA_ERR_ARG;
  }
  for (int i = 0; on && i < nterms; ++i)
    if (!std::isfinite(amp[i]) || !std::isfinite(omega[i]) || !std::isfinite(phase[i])) {
      seterr(ctx, "forcing: non-finite term");
      return GA_ERR_ARG;
    }
  ctx->fnterms[0] = on ? nterms : 0;
  ctx->ft0 = t0;
  for (int i = 0; i < ctx->fnterms[0]; ++i) { ctx->famp[0][i] = amp[i]; ctx->fomega[0][i] = omega[i]; ctx->fphase[0][i] = phase[i]; }
  if (on) {
    CK(cudaMemsetAsync(ctx->forceG, 0, sizeof(double) * ctx->nvec * ctx->g.padded, s));
    launch_api_to_grid(ctx->g, ctx->nvec, ctx->nfree, ctx->map, d_G, ctx->forceG, 1, 0, ctx->st, s);
    CK(cudaGetLastError());
  }
  return rebuild_forcing_graphs(ctx, s);
}

ga_status ga_set_dirichlet(ga_ctx* ctx, const double* h_g, int nterms, const double* amp, const double* omega,
                           const double* phase, void* d_scratch, size_t scratch_bytes, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const bool on = h_g != nullptr && nterms > 0;
  if (on && (ctx->patches.size() != 1 || ctx->nvec != 1 || ctx->sub)) {
    seterr(ctx, "Dirichlet lifting: single patch, scalar wave only");
    return GA_ERR_ARG;
  }
  if (on && (2 * nterms > FMAXTERMS || !amp || !omega || !phase || !d_scratch)) {
    seterr(ctx, "Dirichlet lifting: 1..4 terms, amp/omega/phase and scratch required");
    return GA_ERR_ARG;
  }
  for (int i = 0; on && i < nterms; ++i)
    if (!std::isfinite(amp[i]) || !std::isfinite(omega[i]) || !std::isfinite(phase[i])) {
      seterr(ctx, "Dirichlet lifting: non-finite term");
      return GA_ERR_ARG;
    }
  ctx->fnterms[1] = ctx->fnterms[2] = 0;
  if (on) {
    // boundary apply: M_fb g and K_fb g by the assembly's last contraction (free rows, boundary
    // columns) into the pair-1/2 load vectors; the pairs carry the signs:
    //   pair 1: -(M_fb g) (h'' + a0 h'),  pair 2: -(K_fb g) (h + a1 h')   (R16)
    const long long mpow = ctx->dim == 3 ? (long long)ctx->m * ctx->m * ctx->m : (long long)ctx->m * ctx->m;
    const size_t gbytes = (sizeof(double) * mpow + 255) & ~(size_t)255;
    if (scratch_bytes < gbytes) { seterr(ctx, "scratch too small"); return GA_ERR_OOM; }
    double* dg = (double*)d_scratch;
    CK(cudaMemcpyAsync(dg, h_g, sizeof(double) * mpow, cudaMemcpyHostToDevice, s));
    const size_t vb = sizeof(double) * ctx->nvec * ctx->g.padded;
    double* GM = ctx->forceG + ctx->nvec * ctx->g.padded;
    double* GK = GM + ctx->nvec * ctx->g.padded;
    CK(cudaMemsetAsync(GM, 0, 2 * vb, s));
    Shape sh;
    sh.dim = ctx->dim; sh.nvec = ctx->nvec; sh.p = ctx->p; sh.n = ctx->n; sh.m = ctx->m; sh.k = ctx->k;
    sh.W1 = ctx->W1; sh.S = ctx->S; sh.g = ctx->g; sh.nfree = ctx->nfree; sh.mf = ctx->mf; sh.half = ctx->half;
    rc = assemble(ctx, sh, (char*)d_scratch + gbytes, scratch_bytes - gbytes, s, dg, GM + ctx->g.guard,
                  GK + ctx->g.guard);
    if (rc != GA_OK) return rc;
    const double a0 = ctx->d.damp_a0, a1 = ctx->d.damp_a1;
    int n1 = 0, n2 = 0;
    for (int i = 0; i < nterms; ++i) {
      const double a = amp[i], w = omega[i], ph = phase[i];
      ctx->famp[1][n1] = -a * w * w; ctx->fomega[1][n1] = w; ctx->fphase[1][n1++] = ph + 3.141592653589793;
      ctx->famp[1][n1] = -a0 * a * w; ctx->fomega[1][n1] = w; ctx->fphase[1][n1++] = ph + 1.5707963267948966;
      ctx->famp[2][n2] = -a; ctx->fomega[2][n2] = w; ctx->fphase[2][n2++] = ph;
      ctx->famp[2][n2] = -a1 * a * w; ctx->fomega[2][n2] = w; ctx->fphase[2][n2++] = ph + 1.5707963267948966;
    }
    ctx->fnterms[1] = n1; ctx->fnterms[2] = n2;
  }
  return rebuild_forcing_graphs(ctx, s);
}

ga_status ga_advance(ga_ctx* ctx, int nsteps, void* stream) {
  ga_status rc = check_whole(ctx);
  if (rc != GA_OK) return rc;
  if (nsteps < 0) { seterr(ctx, "nsteps < 0"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  for (int i = 0; i < nsteps; ++i) {
    rc = run_kind(ctx, GK_STEP, s);
    if (rc != GA_OK) return rc;
  }
  return GA_OK;
}

ga_status ga_get_chain(ga_ctx* ctx, int m, double* d_out, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  if (m < 0 || m >= 3 * ctx->k || !d_out) { seterr(ctx, "bad chain index or NULL"); return GA_ERR_ARG; }
  const long long vstride = (long long)ctx->nvec * ctx->g.padded;
  launch_grid_to_api(ctx->g, ctx->nvec, ctx->nfree, ctx->map, ctx->chain + m * vstride, 1, 0, d_out, ctx->st,
                     (cudaStream_t)stream);
  CK(cudaGetLastError());
  return GA_OK;
}

ga_status ga_set_chain(ga_ctx* ctx, int m, const double* d_in, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  if (m < 0 || m >= 3 * ctx->k || !d_in) { seterr(ctx, "bad chain index or NULL"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const long long vstride = (long long)ctx->nvec * ctx->g.padded;
  if (m == 0) reset_status(ctx, s, /*keep_time=*/1);  // the forcing clock is not the statistics
  launch_api_to_grid(ctx->g, ctx->nvec, ctx->nfree, ctx->map, d_in, ctx->chain + m * vstride, 1, 0, ctx->st, s);
  CK(cudaGetLastError());
  // predictors and ||U0|| follow the chain; cheap to refresh after every entry
  return set_predictors_and_norm(ctx, s);
}

__global__ void k_set_tstep(DevStatus* st, long long n) { st->tstep = n; }

ga_status ga_set_time(ga_ctx* ctx, long long step_index, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  if (step_index < 0) { seterr(ctx, "step_index < 0"); return GA_ERR_ARG; }
  k_set_tstep<<<1, 1, 0, (cudaStream_t)stream>>>(ctx->st, step_index);
  CK(cudaGetLastError());
  return GA_OK;
}

ga_status ga_get_state(ga_ctx* ctx, double* d_u, double* d_v, double* d_a, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  double* outs[3] = {d_u, d_v, d_a};
  for (int m = 0; m < 3; ++m)
    if (outs[m]) {
      rc = ga_get_chain(ctx, m, outs[m], stream);
      if (rc != GA_OK) return rc;
    }
  return GA_OK;
}

ga_status ga_get_stats(ga_ctx* ctx, ga_stats* out, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  if (!out) return GA_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  DevStatus h;
  CK(cudaMemcpyAsync(&h, ctx->st, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  memset(out, 0, sizeof(*out));
  out->steps = h.steps;
  out->solves = h.solves;
  for (int j = 0; j < KMAX; ++j) { out->pcg_iters[j] = h.pcg_iters[j]; out->last_iters[j] = h.last_iters[j]; }
  out->max_iters = h.max_iters;
  out->max_rel_residual = h.max_relres;
  out->status = h.status;
  out->fail_step = h.fail_step;
  out->fail_block = h.fail_block;
  out->kernel_launches = (long long)h.launches;
  out->loop_iters = h.loop_iters;
  out->step_index = h.tstep;
  return GA_OK;
}

ga_status ga_profile_op(ga_ctx* ctx, int op, int reps, void* stream) {
  ga_status rc = check_whole(ctx);
  if (rc != GA_OK) return rc;
  if (op < 0 || op > 6 || reps < 0) { seterr(ctx, "bad op"); return GA_ERR_ARG; }
  if (op == 6) {
    cudaStream_t s = (cudaStream_t)stream;
    // one complete mass solve on the current b (persistent kernel or graph), e.g. to time it
    for (int i = 0; i < reps; ++i) {
      rc = run_kind(ctx, GK_SOLVEB, s);
      if (rc != GA_OK) return rc;
    }
    return GA_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (op == 2 || op == 5) {
    // a profiling PcgState in which every block is active, past its first iteration and with
    // beta != 0, so the direction update and the preconditioner do their full work (the state
    // left by the last solve has every block converged: those kernels would return at once)
    PcgState h;
    memset(&h, 0, sizeof(h));
    for (int j = 0; j < KMAX; ++j) {
      h.active[j] = j < ctx->k ? 1 : 0;
      h.alpha[j] = 0.5; h.beta[j] = 0.25; h.rz[j] = h.rzold[j] = h.bb[j] = 1.0;
    }
    h.nrhs = ctx->k; h.iter = 1; h.pfirst = 0; h.first = 0;
    CK(cudaMemcpyAsync(ctx->pcg, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  }
  for (int i = 0; i < reps; ++i) {
    switch (op) {
      case 0: launch_spmv(spmv_args(ctx, 0, ctx->pv, ctx->q, SPMV_PQ), s); break;
      case 1: launch_spmv(spmv_args(ctx, 1, ctx->pred, ctx->b, SPMV_NEGB), s); break;
      case 2: {
        PrecArgs a = prec_args(ctx, 0ull, 0);
        a.maxit = 0x7fffffff;
        launch_precond(a, s);
        break;
      }
      case 3: launch_predict(stage_args(ctx), s); break;
      case 4: launch_spmv(spmv_args(ctx, 0, ctx->pv, ctx->q, SPMV_APPLY), s); break;
      default: launch_p_update(vec_args(ctx), s); break;
    }
  }
  if (op == 2 || op == 5) CK(cudaMemsetAsync(ctx->pcg, 0, sizeof(PcgState), s));
  CK(cudaGetLastError());
  return GA_OK;
}

ga_status ga_apply(ga_ctx* ctx, int which, const double* d_x, double* d_y, void* stream) {
  ga_status rc = check_ctx(ctx);
  if (rc != GA_OK) return rc;
  if (which < 0 || which > 2 || !d_x || !d_y) { seterr(ctx, "bad operator or NULL"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t mvbytes = sizeof(double) * ctx->nvec * ctx->g.padded * ctx->k;
  if (which < 2) {
    CK(cudaMemsetAsync(ctx->pv, 0, mvbytes, s));
    launch_api_to_grid(ctx->g, ctx->nvec, ctx->nfree, ctx->map, d_x, ctx->pv, ctx->k, 0, ctx->st, s);
    launch_spmv(spmv_args(ctx, which, ctx->pv, ctx->q, SPMV_APPLY), s);
    launch_grid_to_api(ctx->g, ctx->nvec, ctx->nfree, ctx->map, ctx->q, ctx->k, 0, d_y, ctx->st, s);
  } else {
    CK(cudaMemsetAsync(ctx->r, 0, mvbytes, s));
    CK(cudaMemsetAsync(ctx->pcg, 0, sizeof(PcgState), s));
    launch_api_to_grid(ctx->g, ctx->nvec, ctx->nfree, ctx->map, d_x, ctx->r, ctx->k, 0, ctx->st, s);
    PrecArgs a = prec_args(ctx, 0ull, 0);
    a.maxit = 0x7fffffff;
    launch_precond(a, s);
    launch_grid_to_api(ctx->g, ctx->nvec, ctx->nfree, ctx->map, ctx->z, ctx->k, 0, d_y, ctx->st, s);
  }
  CK(cudaGetLastError());
  return GA_OK;
}

ga_status ga_solve_mass(ga_ctx* ctx, const double* d_b, double* d_x, int* iters, void* stream) {
  ga_status rc = check_whole(ctx);
  if (rc != GA_OK) return rc;
  if (!d_b || !d_x) { seterr(ctx, "NULL vector"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t mvbytes = sizeof(double) * ctx->nvec * ctx->g.padded * ctx->k;
  CK(cudaMemsetAsync(ctx->b, 0, mvbytes, s));
  launch_api_to_grid(ctx->g, ctx->nvec, ctx->nfree, ctx->map, d_b, ctx->b, ctx->k, 0, ctx->st, s);
  rc = run_kind(ctx, GK_SOLVEB, s);
  if (rc != GA_OK) return rc;
  launch_grid_to_api(ctx->g, ctx->nvec, ctx->nfree, ctx->map, ctx->x, ctx->k, 0, d_x, ctx->st, s);
  CK(cudaGetLastError());
  if (iters) {
    PcgState h;
    DevStatus hs;
    CK(cudaMemcpyAsync(&h, ctx->pcg, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs, ctx->st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *iters = h.its[0];
    if (hs.status != 0) return (ga_status)hs.status;
  }
  return GA_OK;
}

ga_status ga_lambda_max(ga_ctx* ctx, int iters, double* lam, void* stream) {
  // lambda_max(M^{-1} K) by Lanczos in the M inner product: each step
  // one K apply + one PCG mass solve (the K-solve graph) + one M apply; the alpha/beta stay on
  // the device, the largest eigenvalue of the tridiagonal matrix is found on the host
  ga_status rc = check_whole(ctx);
  if (rc != GA_OK) return rc;
  if (iters < 1 || !lam) { seterr(ctx, "iters >= 1 and lam required"); return GA_ERR_ARG; }
  iters = std::min(iters, LZMAX);
  cudaStream_t s = (cudaStream_t)stream;
  const GridDesc& g = ctx->g;
  const int nvec = ctx->nvec, k = ctx->k;
  const size_t mvbytes = sizeof(double) * nvec * g.padded * k;
  const long long tot = (long long)nvec * g.npts;
  const unsigned int nb = (unsigned int)((tot + 255) / 256);
  // the predictor MV is state: keep a host copy and restore it at the end
  std::vector<double> hsave(mvbytes / sizeof(double));
  CK(cudaMemcpyAsync(hsave.data(), ctx->pred, mvbytes, cudaMemcpyDeviceToHost, s));
  // the statistics and the failure status are state too: the Lanczos solves must not count as
  // step solves, and a NOCONV inside Lanczos is returned, not latched (restored on every exit)
  DevStatus stsave;
  CK(cudaMemcpyAsync(&stsave, ctx->st, sizeof(stsave), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  auto restore = [&](ga_status rc0) -> ga_status {
    cudaError_t e1 = cudaMemcpyAsync(ctx->pred, hsave.data(), mvbytes, cudaMemcpyHostToDevice, s);
    cudaError_t e2 = cudaMemcpyAsync(ctx->st, &stsave, sizeof(stsave), cudaMemcpyHostToDevice, s);
    cudaError_t e3 = cudaStreamSynchronize(s);
    ga_status rs = set_step_slots(ctx, s);
    if (rc0 != GA_OK) return rc0;
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      seterr(ctx, "ga_lambda_max: restoring the state failed");
      return GA_ERR_CUDA;
    }
    return rs;
  };
  if (ctx->forcing) {  // the K-solve graph would add F: switch the slots off meanwhile
    ForceSlots fs;
    memset(&fs, 0, sizeof(fs));
    if ((cudaMemcpyAsync(ctx->fslots, &fs, sizeof(fs), cudaMemcpyHostToDevice, s)) != cudaSuccess) return restore(GA_ERR_CUDA);
  }
  if ((cudaStreamSynchronize(s)) != cudaSuccess) return restore(GA_ERR_CUDA);
  double* vp = ctx->lzv;                                   // v_{j-1} (then w)
  double* vc = ctx->lzv + (size_t)nvec * g.padded * k;     // v_j
  double* al = ctx->lzab;                                  // alpha_j, j < iters
  double* be = ctx->lzab + LZMAX + 2;                      // beta_j (be[0] = norm of the start vector)
  double* dn = ctx->dscal;
  if ((cudaMemsetAsync(ctx->lzv, 0, 2 * mvbytes, s)) != cudaSuccess) return restore(GA_ERR_CUDA);
  if ((cudaMemsetAsync(ctx->lzab, 0, sizeof(double) * 2 * (LZMAX + 2), s)) != cudaSuccess) return restore(GA_ERR_CUDA);
  k_altsign<<<nb, 256, 0, s>>>(g, nvec, k, vc, ctx->mask);
  // v_1 = v / ||v||_M
  launch_spmv(spmv_args(ctx, 0, vc, ctx->q, SPMV_APPLY), s);
  launch_dot(g, nvec, k, vc, ctx->q, dn, ctx->partial, ctx->counter, s);
  k_lz_norm<<<nb, 256, 0, s>>>(g, nvec, k, vc, dn, be);
  int done = iters;
  for (int j = 0; j < iters; ++j) {
    if ((cudaMemsetAsync(ctx->pred, 0, mvbytes, s)) != cudaSuccess) return restore(GA_ERR_CUDA);
    if ((cudaMemcpy2DAsync(ctx->pred, sizeof(double) * k, vc, sizeof(double) * k, sizeof(double),
                         (size_t)nvec * g.padded, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return restore(GA_ERR_CUDA);
    rc = run_kind(ctx, GK_SOLVEK, s);  // b = -K v_j, x = M^{-1} b
    if (rc != GA_OK) return restore(rc);
    launch_dot(g, nvec, k, vc, ctx->b, dn, ctx->partial, ctx->counter, s);  // -alpha_j
    k_lz_copy_alpha<<<1, 1, 0, s>>>(dn, al + j);
    // w = A v_j - alpha_j v_j - beta_{j-1} v_{j-1}, into vp
    k_lz_update<<<nb, 256, 0, s>>>(g, nvec, k, ctx->x, vc, vp, dn, be + j, ctx->mask);
    launch_spmv(spmv_args(ctx, 0, vp, ctx->q, SPMV_APPLY), s);
    launch_dot(g, nvec, k, vp, ctx->q, dn + 1, ctx->partial, ctx->counter, s);
    k_lz_norm<<<nb, 256, 0, s>>>(g, nvec, k, vp, dn + 1, be + j + 1);
    std::swap(vp, vc);  // v_{j+1} = w / beta_j becomes current, v_j previous
    if (cudaGetLastError() != cudaSuccess) return restore(GA_ERR_CUDA);
  }
  std::vector<double> ha(done), hb(done + 1);
  DevStatus hs;
  if (cudaMemcpyAsync(ha.data(), al, sizeof(double) * done, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(hb.data(), be, sizeof(double) * (done + 1), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(&hs, ctx->st, sizeof(hs), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return restore(GA_ERR_CUDA);
  rc = restore(hs.status != 0 ? (ga_status)hs.status : GA_OK);
  if (rc != GA_OK) return rc;
  // stop at a (numerically) invariant subspace: beta_j ~ 0
  int m = done;
  for (int j = 1; j < done; ++j)
    if (!(hb[j] > 1e-14 * std::fabs(ha[0]))) { m = j; break; }
  // largest eigenvalue of the symmetric tridiagonal T (diag ha, off-diag hb[1..m-1]) by bisection
  double lo = 1e300, hi = -1e300;
  for (int j = 0; j < m; ++j) {
    const double r = (j > 0 ? std::fabs(hb[j]) : 0.0) + (j + 1 < m ? std::fabs(hb[j + 1]) : 0.0);
    lo = std::min(lo, ha[j] - r);
    hi = std::max(hi, ha[j] + r);
  }
  auto count_below = [&](double x) {  // Sturm count of eigenvalues < x
    int c = 0;
    double d = 1.0;
    for (int j = 0; j < m; ++j) {
      const double off = j > 0 ? hb[j] * hb[j] : 0.0;
      d = (ha[j] - x) - (j > 0 ? off / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0.0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(1.0, std::fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) < m) lo = mid; else hi = mid;
  }
  *lam = 0.5 * (lo + hi);
  return GA_OK;
}

int ga_uses_persistent_solver(const ga_ctx* ctx) { return ctx && ctx->persist ? 1 : 0; }
int ga_uses_matrix_free(const ga_ctx* ctx) { return ctx && ctx->mf ? 1 : 0; }
int ga_operator_mode(const ga_ctx* ctx) { return !ctx ? 0 : (ctx->mf ? 2 : (ctx->half ? 3 : 1)); }

// debug: copy the persistent-solver trace (GA_TRACE=1) to the host; returns slots copied
int ga_debug_trace(ga_ctx* ctx, long long* host, int n) {
  if (!ctx || !ctx->trace || !host) return 0;
  if (n > 8192) n = 8192;
  if (cudaMemcpy(host, ctx->trace, sizeof(long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

ga_status ga_free_dof_map(const ga_ctx* ctx, long long* host_map) {
  if (!ctx || !host_map) return GA_ERR_ARG;
  memcpy(host_map, ctx->hlocal.data(), sizeof(long long) * ctx->hlocal.size());
  return GA_OK;
}

void ga_destroy(ga_ctx* ctx) {
  if (!ctx) return;
  if (ctx->g_step) cudaGraphExecDestroy(ctx->g_step);
  if (ctx->g_solveK) cudaGraphExecDestroy(ctx->g_solveK);
  if (ctx->g_solveB) cudaGraphExecDestroy(ctx->g_solveB);
  if (ctx->gr_step) cudaGraphDestroy(ctx->gr_step);
  if (ctx->gr_solveK) cudaGraphDestroy(ctx->gr_solveK);
  if (ctx->gr_solveB) cudaGraphDestroy(ctx->gr_solveB);
  if (ctx->trace) cudaFree(ctx->trace);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->cap) cudaStreamDestroy(ctx->cap);
  delete ctx;
}

const char* ga_last_error(const ga_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  return g_thread_err.c_str();
}

}  // extern "C"
