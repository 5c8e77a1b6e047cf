// Partitioned multi-patch (patch-per-GPU) stepping: ga_group (include/genalpha.h; SURVEY §8e,
// §8f NEXT-4).  Each subdomain context holds one patch with its LOCAL operators M^(r), K^(r)
// on the bounding box of its free control points (make_shape_sub, genalpha.cu).
// Global vectors are kept CONSISTENT: every copy of an interface DoF holds the same value.
//
//   q = M p       : q_r = M^(r) p_r locally, then the copies of each interface DoF are summed
//   z = calM^-1 r : z_r = R_r^T calM^(r)-1 R_r r locally (one additive-Schwarz term),
//                   then the copies are summed (the sum over r of eq. def:asp)
//   p.q, r.z      : sums of the unassembled local products (p^T M p = sum_r p_r^T M^(r) p_r,
//                   r^T z = sum_r r_r^T z_r), ||r||^2, ||b||^2 over the owned DoFs (mask 1)
//
// One exchange = each context writes [its interface values | its partial sums] to its send
// buffer (interface values by slot, zero where the context holds no copy), the buffers of the
// process are summed in a fixed order, NCCL all-reduces the sum across processes (multi-GPU),
// and every context takes back the interface sums and runs the scalar step of the site (alpha,
// beta / convergence, PCG set-up) from the same summed scalars -- so all subdomains take the
// same decisions.  Two exchanges per PCG iteration (after the SpMV and after the
// preconditioner), one after -K s (the right-hand side), one for ||b||^2.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "tile_core.cuh"

using namespace ga;
using namespace gaint;

namespace {

constexpr int GMAX = 32;  // subdomain contexts per process in one group

// ----------------------------------------------------------------------------------- NCCL
typedef int nccl_res;
struct nccl_uid { char internal[128]; };
typedef void* nccl_comm;
constexpr int NCCL_FLOAT64 = 8, NCCL_SUM = 0;
struct Nccl {
  bool tried = false, ok = false;
  nccl_res (*get_unique_id)(nccl_uid*) = nullptr;
  nccl_res (*comm_init_rank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  nccl_res (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_res (*comm_destroy)(nccl_comm) = nullptr;
  const char* (*error_string)(nccl_res) = nullptr;
  std::string err;
};
Nccl g_nccl;

bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  const char* path = getenv("GA_NCCL_LIB");
  void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { g_nccl.err = std::string("dlopen libnccl.so.2: ") + dlerror(); return false; }
  g_nccl.get_unique_id = (nccl_res(*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
  g_nccl.comm_init_rank = (nccl_res(*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
  g_nccl.all_reduce = (nccl_res(*)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
  g_nccl.comm_destroy = (nccl_res(*)(nccl_comm))dlsym(h, "ncclCommDestroy");
  g_nccl.error_string = (const char* (*)(nccl_res))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.all_reduce && g_nccl.comm_destroy;
  if (!g_nccl.ok) g_nccl.err = "libnccl.so.2 lacks the NCCL symbols";
  return g_nccl.ok;
}

// ------------------------------------------------------------------------------- kernels
enum Site { X_NONE = 0, X_BB = 1, X_Q = 2, X_Z = 3, X_RR = 4 };

// send buffer: buf[(c n_iface + slot) kk + j] = v at the slot's grid point, 0 where this
// subdomain holds no copy (every slot written: no clearing pass)
__global__ void k_x_pack(GridDesc g, int nvec, int kk, long long n_iface, const int* __restrict__ xinv,
                         const double* __restrict__ v, double* __restrict__ buf, DevStatus* st) {
  count_launch(st);
  const long long tot = (long long)nvec * n_iface * kk;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const int j = (int)(e % kk);
  const long long cs = e / kk;
  const long long slot = cs % n_iface;
  const int c = (int)(cs / n_iface);
  const int gi = xinv[slot];
  buf[e] = gi >= 0 ? v[((long long)c * g.padded + g.guard + gi) * kk + j] : 0.0;
}

struct XComb {
  const double* in[GMAX];
  int nin;
  double* out;
  long long cnt;
};
// sum of the process's send buffers in context order (deterministic)
__global__ void k_x_combine(XComb a) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.cnt) return;
  double s = a.in[0][e];
  for (int r = 1; r < a.nin; ++r) s += a.in[r][e];
  a.out[e] = s;
}

struct XUnpack {
  GridDesc g;
  int nvec, kk;
  long long n_iface, nxl;
  const int* xgi;
  const int* xslot;
  const double* recv;   // summed buffer (values at [0, nvec n_iface kk), scalars after)
  double* v;            // vector to overwrite at the held interface DoFs (null: none)
  int site;
  PcgState* pcg;
  DevStatus* st;
  double tol2, refine_rtol2;
  int maxit;
  unsigned long long cond;  // graph conditional handle (X_Z of the context that owns the loop)
};

// the interface sums back into v, and the scalar step of the site from the summed scalars
// (thread 0 of block 0): the same code paths as the single-context finishers
template <int KK>
__global__ void k_x_unpack(XUnpack a) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.v) {
    const long long tot = (long long)a.nvec * a.nxl * KK;
    if (e < tot) {
      const int j = (int)(e % KK);
      const long long ci = e / KK;
      const long long i = ci % a.nxl;
      const int c = (int)(ci / a.nxl);
      a.v[((long long)c * a.g.padded + a.g.guard + a.xgi[i]) * KK + j] =
          a.recv[((long long)c * a.n_iface + a.xslot[i]) * KK + j];
    }
  }
  if (e != 0) return;
  count_launch(a.st);
  const double* sc = a.recv + (long long)a.nvec * a.n_iface * KK;
  PcgState* pc = a.pcg;
  if (a.site == X_BB) {  // k_init_from_b's set-up with the global ||b||^2
    if (a.st->status != 0) return;
    pc->iter = 0; pc->first = 1; pc->pfirst = 1; pc->nrhs = KK; pc->phase = 0; pc->guard = 0;
    for (int j = 0; j < KK; ++j) {
      pc->bb[j] = sc[j];
      pc->thr[j] = a.tol2 * sc[j];
      pc->active[j] = sc[j] > 0.0 ? 1 : 0;
      pc->its[j] = 0;
      pc->alpha[j] = 0.0;
      pc->beta[j] = 0.0;
    }
  } else if (a.site == X_Q) {  // k_spmv_fin (SPMV_PQ) with the global p.q
    if (a.st->status != 0) return;
    pc->iter += 1;
    pc->pfirst = 0;
    a.st->loop_iters += 1;
    for (int j = 0; j < KK; ++j) {
      pc->pq[j] = sc[j];
      if (pc->active[j]) {
        pc->alpha[j] = pc->rz[j] / sc[j];
        pc->its[j] += 1;
      } else {
        pc->alpha[j] = 0.0;
      }
    }
  } else if (a.site == X_Z) {  // k_prec_out's F1 with the global r.z, r.r
    if (a.st->status != 0) {
      if (a.cond) cudaGraphSetConditional((cudaGraphConditionalHandle)a.cond, 0u);
      return;
    }
    double rz[KMAX], rr[KMAX];
    for (int j = 0; j < KK; ++j) { rz[j] = sc[j]; rr[j] = sc[KK + j]; }
    pcg_finalize(pc, a.st, KK, a.maxit, a.cond, rz, rr);
  } else if (a.site == X_RR) {  // k_spmv_fin (SPMV_TRUERES): restart from b - M x
    if (a.st->status != 0) return;
    pc->iter = 0; pc->first = 1; pc->pfirst = 1; pc->phase = 1; pc->guard = 0;
    for (int j = 0; j < KK; ++j) {
      pc->alpha[j] = 0.0;
      pc->active[j] = pc->bb[j] > 0.0 ? 1 : 0;
      double thr = a.tol2 * pc->bb[j];
      if (a.refine_rtol2 > 0.0) thr = fmin(thr, a.refine_rtol2 * sc[j]);
      pc->thr[j] = thr;
    }
  }
}

// r = b - r (r holds the assembled M x), zero on masked points; owned ||r||^2 to xsum
template <int KK>
__global__ void __launch_bounds__(NTHREADS) k_x_trueres(GridDesc g, int nvec, const unsigned char* __restrict__ mask,
                                                        const double* __restrict__ b, double* __restrict__ r,
                                                        double* partial, unsigned int* counter, double* xsum,
                                                        DevStatus* st) {
  const bool dead = st->status != 0;
  if (!dead) count_launch(st);
  const long long tot = (long long)nvec * g.npts;
  const long long estride = (long long)gridDim.x * blockDim.x;
  double v[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) v[j] = 0.0;
  if (!dead)
    for (long long e = (long long)gtid(); e < tot; e += estride) {
      const long long c = e / g.npts, i = e - c * g.npts;
      const long long base = (c * g.padded + g.guard + i) * KK;
      const unsigned char mk = mask[i];
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        const double rv = mk ? b[base + j] - r[base + j] : 0.0;
        r[base + j] = rv;
        if (mk == 1) v[j] = fma(rv, rv, v[j]);
      }
    }
  if (dead) return;
  double out[KK];
  if (reduce_last_block<KK>(v, partial, counter, out))
    for (int j = 0; j < KK; ++j) xsum[j] = out[j];
}

// forcing of a subdomain: the load vector is local, so it is added before the exchange (the
// ordinary k_add_forcing), nothing special here.

unsigned int nblk(long long n) { return (unsigned int)std::max(1LL, (n + 255) / 256); }
unsigned int red_blocks(long long n) {
  const long long b = (n + NTHREADS - 1) / NTHREADS;
  return (unsigned int)(b < 1184 ? (b > 0 ? b : 1) : 1184);
}

}  // namespace

// --------------------------------------------------------------------------------- group
struct ga_group {
  std::vector<ga_ctx*> c;
  nccl_comm comm = nullptr;
  int k = 1, nvec = 1;
  long long n_iface = 0, xcount = 0, vcount = 0;
  double* recv = nullptr;
  std::vector<cudaStream_t> st;  // one stream per context (fork/join inside a step)
  cudaStream_t cap = nullptr, aux = nullptr;
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_join;
  // a second fork/join set for the capture of the WHILE body (stream aux): the streams of the
  // first set are still part of the outer capture (stream cap) while the body is captured, and a
  // stream cannot join two captures
  std::vector<cudaStream_t> st2;
  cudaEvent_t ev_fork2 = nullptr;
  std::vector<cudaEvent_t> ev_join2;
  cudaGraphExec_t g_step = nullptr, g_solveK = nullptr, g_solveB = nullptr;
  cudaGraph_t gr_step = nullptr, gr_solveK = nullptr, gr_solveB = nullptr;
  bool host_loop = false;  // NCCL: the PCG loop is driven by the host (flags polled)
  std::string err;
};

namespace {

thread_local std::string g_group_err;

void gseterr(ga_group* G, const std::string& s) {
  if (G) G->err = s;
  g_group_err = s;
}

#define GCK(call)                                                                  \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      gseterr(G, std::string(#call) + ": " + cudaGetErrorString(e_));              \
      return GA_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

// run f(ctx, stream) for every context on its own stream, forked from and joined into s
template <class F>
ga_status par(ga_group* G, cudaStream_t s, F f) {
  const int R = (int)G->c.size();
  if (R == 1) { f(G->c[0], s); return GA_OK; }
  const bool body = (s == G->aux);
  const std::vector<cudaStream_t>& st = body ? G->st2 : G->st;
  const std::vector<cudaEvent_t>& ej = body ? G->ev_join2 : G->ev_join;
  cudaEvent_t ef = body ? G->ev_fork2 : G->ev_fork;
  GCK(cudaEventRecord(ef, s));
  for (int r = 0; r < R; ++r) {
    GCK(cudaStreamWaitEvent(st[r], ef, 0));
    f(G->c[r], st[r]);
    GCK(cudaEventRecord(ej[r], st[r]));
  }
  for (int r = 0; r < R; ++r) GCK(cudaStreamWaitEvent(s, ej[r], 0));
  return GA_OK;
}

// vector selector of an exchange
enum Vec { V_NONE = 0, V_B, V_Q, V_Z, V_R };
double* vec_of(ga_ctx* c, Vec v) {
  switch (v) {
    case V_B: return c->b;
    case V_Q: return c->q;
    case V_Z: return c->z;
    case V_R: return c->r;
    default: return nullptr;
  }
}

// one exchange (see the file comment); cond: conditional handle for the X_Z step of context 0
ga_status xchg(ga_group* G, cudaStream_t s, Site site, Vec vec, unsigned long long cond = 0ull) {
  const int R = (int)G->c.size();
  const bool withv = vec != V_NONE && G->n_iface > 0;
  if (withv) {
    ga_status rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
      k_x_pack<<<nblk(G->vcount), 256, 0, ss>>>(c->g, c->nvec, c->k, c->n_iface, c->xinv, vec_of(c, vec), c->xbuf, c->st);
    });
    if (rc != GA_OK) return rc;
  }
  const long long off = withv ? 0 : G->vcount, cnt = withv ? G->xcount : G->xcount - G->vcount;
  const bool direct = R == 1 && G->comm;  // one local buffer: NCCL reads it directly
  if (!direct) {
    XComb a;
    memset(&a, 0, sizeof(a));
    for (int r = 0; r < R; ++r) a.in[r] = G->c[r]->xbuf + off;
    a.nin = R;
    a.out = G->recv + off;
    a.cnt = cnt;
    k_x_combine<<<nblk(cnt), 256, 0, s>>>(a);
    GCK(cudaGetLastError());
  }
  if (G->comm) {
    const double* src = direct ? G->c[0]->xbuf + off : G->recv + off;
    nccl_res e = g_nccl.all_reduce(src, G->recv + off, (size_t)cnt, NCCL_FLOAT64, NCCL_SUM, G->comm, s);
    if (e != 0) {
      gseterr(G, std::string("ncclAllReduce: ") + (g_nccl.error_string ? g_nccl.error_string(e) : "error"));
      return GA_ERR_CUDA;
    }
  }
  return par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
    XUnpack u;
    memset(&u, 0, sizeof(u));
    u.g = c->g; u.nvec = c->nvec; u.kk = c->k; u.n_iface = c->n_iface; u.nxl = c->nxl;
    u.xgi = c->xgi; u.xslot = c->xslot; u.recv = G->recv;
    u.v = withv ? vec_of(c, vec) : nullptr;
    u.site = site; u.pcg = c->pcg; u.st = c->st;
    u.tol2 = c->d.pcg_rtol * c->d.pcg_rtol;
    u.refine_rtol2 = c->d.pcg_refine_rtol > 0 ? c->d.pcg_refine_rtol * c->d.pcg_refine_rtol : 0.0;
    u.maxit = c->d.pcg_maxit;
    u.cond = (c == G->c[0]) ? cond : 0ull;
    const long long tot = withv ? (long long)c->nvec * c->nxl * c->k : 1;
    switch (c->k) {
      case 1: k_x_unpack<1><<<nblk(tot), 256, 0, ss>>>(u); break;
      case 2: k_x_unpack<2><<<nblk(tot), 256, 0, ss>>>(u); break;
      case 3: k_x_unpack<3><<<nblk(tot), 256, 0, ss>>>(u); break;
      default: k_x_unpack<4><<<nblk(tot), 256, 0, ss>>>(u); break;
    }
  });
}

double* xsum_of(ga_ctx* c) { return c->xbuf + (long long)c->nvec * c->n_iface * c->k; }

// ---- PCG phases (every context, then the exchange)
ga_status enqueue_precond(ga_group* G, cudaStream_t s, unsigned long long cond) {
  ga_status rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
    PrecArgs a = prec_args(c, 0ull, 1);
    a.xsum = xsum_of(c);
    launch_precond(a, ss);
  });
  if (rc != GA_OK) return rc;
  return xchg(G, s, X_Z, V_Z, cond);
}

ga_status enqueue_iteration(ga_group* G, cudaStream_t s, unsigned long long cond) {
  ga_status rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
    launch_p_update(vec_args(c), ss);
    SpmvArgs a = spmv_args(c, 0, c->pv, c->q, SPMV_PQ);
    a.xsum = xsum_of(c);
    launch_spmv(a, ss);
  });
  if (rc != GA_OK) return rc;
  rc = xchg(G, s, X_Q, V_Q);
  if (rc != GA_OK) return rc;
  return enqueue_precond(G, s, cond);
}

// PCG loop: pre-loop preconditioner + WHILE(iteration) (graph), or host-driven (NCCL)
ga_status pcg_loop(ga_group* G, cudaStream_t s, bool capturing) {
  if (!capturing) {
    ga_status rc = enqueue_precond(G, s, 0ull);
    if (rc != GA_OK) return rc;
    ga_ctx* c0 = G->c[0];
    for (int it = 0; it < 100000; ++it) {
      PcgState h;
      DevStatus hs;
      GCK(cudaMemcpyAsync(&h, c0->pcg, sizeof(h), cudaMemcpyDeviceToHost, s));
      GCK(cudaMemcpyAsync(&hs, c0->st, sizeof(hs), cudaMemcpyDeviceToHost, s));
      GCK(cudaStreamSynchronize(s));
      int any = 0;
      for (int j = 0; j < G->k; ++j) any |= h.active[j];
      if (!any || hs.status != 0 || h.iter >= c0->d.pcg_maxit) break;
      rc = enqueue_iteration(G, s, 0ull);
      if (rc != GA_OK) return rc;
    }
    return GA_OK;
  }
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  GCK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &graph, &deps, &nd));
  cudaGraphConditionalHandle h;
  GCK(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
  ga_status rc = enqueue_precond(G, s, (unsigned long long)h);
  if (rc != GA_OK) return rc;
  GCK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &graph, &deps, &nd));
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  GCK(cudaGraphAddNode(&node, graph, deps, nd, &cp));
  GCK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  GCK(cudaStreamBeginCaptureToGraph(G->aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  rc = enqueue_iteration(G, G->aux, (unsigned long long)h);
  cudaGraph_t outg;
  cudaError_t e = cudaStreamEndCapture(G->aux, &outg);
  if (rc != GA_OK) return rc;
  GCK(e);
  return GA_OK;
}

// b in place (consistent): lock-stepped PCG (+ refinement restart) of M x = b
ga_status enqueue_solve(ga_group* G, cudaStream_t s, bool capturing) {
  ga_status rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
    VecArgs v = vec_args(c);
    v.own = c->mask;
    v.xsum = xsum_of(c);
    launch_init_from_b(v, ss);
  });
  if (rc != GA_OK) return rc;
  rc = xchg(G, s, X_BB, V_NONE);
  if (rc != GA_OK) return rc;
  rc = pcg_loop(G, s, capturing);
  if (rc != GA_OK) return rc;
  if (G->c[0]->d.pcg_refine) {
    rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) { launch_spmv(spmv_args(c, 0, c->x, c->r, SPMV_APPLY), ss); });
    if (rc != GA_OK) return rc;
    rc = xchg(G, s, X_NONE, V_R);  // r = M x, assembled
    if (rc != GA_OK) return rc;
    rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
      const unsigned int nb = red_blocks((long long)c->nvec * c->g.npts);
      switch (c->k) {
        case 1: k_x_trueres<1><<<nb, NTHREADS, 0, ss>>>(c->g, c->nvec, c->mask, c->b, c->r, c->partial, c->counter, xsum_of(c), c->st); break;
        case 2: k_x_trueres<2><<<nb, NTHREADS, 0, ss>>>(c->g, c->nvec, c->mask, c->b, c->r, c->partial, c->counter, xsum_of(c), c->st); break;
        case 3: k_x_trueres<3><<<nb, NTHREADS, 0, ss>>>(c->g, c->nvec, c->mask, c->b, c->r, c->partial, c->counter, xsum_of(c), c->st); break;
        default: k_x_trueres<4><<<nb, NTHREADS, 0, ss>>>(c->g, c->nvec, c->mask, c->b, c->r, c->partial, c->counter, xsum_of(c), c->st); break;
      }
    });
    if (rc != GA_OK) return rc;
    rc = xchg(G, s, X_RR, V_NONE);
    if (rc != GA_OK) return rc;
    rc = pcg_loop(G, s, capturing);
    if (rc != GA_OK) return rc;
  }
  return par(G, s, [&](ga_ctx* c, cudaStream_t ss) { launch_solve_end(c->pcg, c->st, ss); });
}

enum Kind { K_STEP = 0, K_SOLVEK = 1, K_SOLVEB = 2 };

ga_status enqueue_kind(ga_group* G, cudaStream_t s, Kind kind, bool capturing) {
  ga_status rc = GA_OK;
  if (kind != K_SOLVEB) {
    rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) {
      launch_spmv(spmv_args(c, 1, c->pred, c->b, SPMV_NEGB), ss);  // b_r = -K^(r) s (local)
      if (c->forcing) launch_add_forcing(force_args(c), ss);       // + local load integrals
    });
    if (rc != GA_OK) return rc;
    rc = xchg(G, s, X_NONE, V_B);
    if (rc != GA_OK) return rc;
  }
  rc = enqueue_solve(G, s, capturing);
  if (rc != GA_OK) return rc;
  if (kind == K_STEP) rc = par(G, s, [&](ga_ctx* c, cudaStream_t ss) { launch_stage(stage_args(c), ss); });
  if (rc == GA_OK) GCK(cudaGetLastError());
  return rc;
}

void destroy_graphs(ga_group* G) {
  cudaGraphExec_t* ex[3] = {&G->g_step, &G->g_solveK, &G->g_solveB};
  cudaGraph_t* gr[3] = {&G->gr_step, &G->gr_solveK, &G->gr_solveB};
  for (int i = 0; i < 3; ++i) {
    if (*ex[i]) cudaGraphExecDestroy(*ex[i]);
    if (*gr[i]) cudaGraphDestroy(*gr[i]);
    *ex[i] = nullptr; *gr[i] = nullptr;
  }
}

ga_status build_graphs(ga_group* G) {
  destroy_graphs(G);
  if (G->host_loop) return GA_OK;
  cudaGraphExec_t* ex[3] = {&G->g_step, &G->g_solveK, &G->g_solveB};
  cudaGraph_t* gr[3] = {&G->gr_step, &G->gr_solveK, &G->gr_solveB};
  for (int i = 0; i < 3; ++i) {
    GCK(cudaStreamBeginCapture(G->cap, cudaStreamCaptureModeRelaxed));
    ga_status rc = enqueue_kind(G, G->cap, (Kind)i, true);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(G->cap, &g);
    if (rc != GA_OK) return rc;
    GCK(e);
    GCK(cudaGraphInstantiate(ex[i], g, 0));
    *gr[i] = g;
  }
  return GA_OK;
}

ga_status run(ga_group* G, Kind kind, cudaStream_t s) {
  if (G->host_loop) return enqueue_kind(G, s, kind, false);
  cudaGraphExec_t e = kind == K_STEP ? G->g_step : (kind == K_SOLVEK ? G->g_solveK : G->g_solveB);
  GCK(cudaGraphLaunch(e, s));
  return GA_OK;
}

ga_status check_group(ga_group* G) {
  if (!G) { gseterr(nullptr, "group is NULL"); return GA_ERR_ARG; }
  return GA_OK;
}

}  // namespace

extern "C" {

ga_status ga_nccl_unique_id(void* id128) {
  if (!id128) return GA_ERR_ARG;
  if (!nccl_load()) { gseterr(nullptr, g_nccl.err); return GA_ERR_ARG; }
  nccl_uid u;
  if (g_nccl.get_unique_id(&u) != 0) { gseterr(nullptr, "ncclGetUniqueId failed"); return GA_ERR_ARG; }
  memcpy(id128, &u, sizeof(u));
  return GA_OK;
}

ga_status ga_nccl_comm_init(int nranks, const void* id128, int rank, void** comm) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return GA_ERR_ARG;
  *comm = nullptr;
  if (!nccl_load()) { gseterr(nullptr, g_nccl.err); return GA_ERR_ARG; }
  nccl_uid u;
  memcpy(&u, id128, sizeof(u));
  nccl_comm c = nullptr;
  nccl_res e = g_nccl.comm_init_rank(&c, nranks, u, rank);
  if (e != 0) {
    gseterr(nullptr, std::string("ncclCommInitRank: ") + (g_nccl.error_string ? g_nccl.error_string(e) : "error"));
    return GA_ERR_ARG;
  }
  *comm = c;
  return GA_OK;
}

void ga_nccl_comm_destroy(void* comm) {
  if (comm && nccl_load()) g_nccl.comm_destroy((nccl_comm)comm);
}

ga_status ga_group_create(ga_ctx* const* ctxs, int nctx, void* nccl_comm_p, void* stream, ga_group** out) {
  if (out) *out = nullptr;
  if (!out || !ctxs || nctx < 1 || nctx > GMAX) { gseterr(nullptr, "group: 1..32 contexts and out required"); return GA_ERR_ARG; }
  ga_group* G = new ga_group();
  for (int r = 0; r < nctx; ++r) {
    ga_ctx* c = ctxs[r];
    if (!c || !c->sub) { gseterr(G, "group: every context must be a subdomain (ga_desc.sub)"); delete G; return GA_ERR_ARG; }
    if (c->grp) { gseterr(G, "group: a context already belongs to a group"); delete G; return GA_ERR_ARG; }
    const ga_ctx* c0 = ctxs[0];
    if (c->k != c0->k || c->nvec != c0->nvec || c->n_iface != c0->n_iface || c->d.dt != c0->d.dt ||
        c->d.pcg_rtol != c0->d.pcg_rtol || c->d.pcg_maxit != c0->d.pcg_maxit || c->d.pcg_refine != c0->d.pcg_refine ||
        c->d.pcg_refine_rtol != c0->d.pcg_refine_rtol || c->d.rho_b != c0->d.rho_b || c->d.rho_s != c0->d.rho_s) {
      gseterr(G, "group: contexts differ in k, ncomp, interface count, dt, rho or PCG settings");
      delete G;
      return GA_ERR_ARG;
    }
    for (int q = 0; q < r; ++q)
      if (ctxs[q] == c) { gseterr(G, "group: a context is listed twice"); delete G; return GA_ERR_ARG; }
    G->c.push_back(c);
  }
  if (nccl_comm_p && !nccl_load()) { gseterr(G, g_nccl.err); delete G; return GA_ERR_ARG; }
  G->comm = (nccl_comm)nccl_comm_p;
  G->host_loop = G->comm != nullptr && !getenv("GA_GROUP_NCCL_GRAPH");
  G->k = ctxs[0]->k; G->nvec = ctxs[0]->nvec; G->n_iface = ctxs[0]->n_iface;
  G->vcount = (long long)G->nvec * G->n_iface * G->k;
  G->xcount = G->vcount + XSCAL;
  G->recv = ctxs[0]->xrecv;
  cudaStream_t s = (cudaStream_t)stream;
  auto fail = [&](ga_status rc) { ga_group_destroy(G); return rc; };
#define GCKF(call)                                                     \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) {                                           \
      gseterr(G, std::string(#call) + ": " + cudaGetErrorString(e_));  \
      return fail(GA_ERR_CUDA);                                        \
    }                                                                  \
  } while (0)
  G->st.resize(nctx, nullptr);
  G->ev_join.resize(nctx, nullptr);
  G->st2.resize(nctx, nullptr);
  G->ev_join2.resize(nctx, nullptr);
  for (int r = 0; r < nctx; ++r) {
    GCKF(cudaStreamCreateWithFlags(&G->st[r], cudaStreamNonBlocking));
    GCKF(cudaEventCreateWithFlags(&G->ev_join[r], cudaEventDisableTiming));
    GCKF(cudaStreamCreateWithFlags(&G->st2[r], cudaStreamNonBlocking));
    GCKF(cudaEventCreateWithFlags(&G->ev_join2[r], cudaEventDisableTiming));
  }
  GCKF(cudaEventCreateWithFlags(&G->ev_fork, cudaEventDisableTiming));
  GCKF(cudaEventCreateWithFlags(&G->ev_fork2, cudaEventDisableTiming));
  GCKF(cudaStreamCreateWithFlags(&G->cap, cudaStreamNonBlocking));
  GCKF(cudaStreamCreateWithFlags(&G->aux, cudaStreamNonBlocking));
  for (ga_ctx* c : G->c) c->grp = G;
  // global diag(M): sum the copies of the local diagonals, then the scalings (reading R6)
  GCKF(cudaStreamSynchronize(s));
  for (ga_ctx* c : G->c) {
    // the diagonal into slot 0 of the b vector, the exchange brings the sums back
    GCKF(cudaMemsetAsync(c->b, 0, sizeof(double) * c->nvec * c->g.padded * c->k, s));
    GCKF(cudaMemcpy2DAsync(c->b + c->g.guard * c->k, sizeof(double) * c->k, c->diagM, sizeof(double), sizeof(double),
                           (size_t)c->g.npts, cudaMemcpyDeviceToDevice, s));
  }
  ga_status rc = xchg(G, s, X_NONE, V_B);
  if (rc != GA_OK) return fail(rc);
  for (ga_ctx* c : G->c) {
    GCKF(cudaMemcpy2DAsync(c->diagM, sizeof(double), c->b + c->g.guard * c->k, sizeof(double) * c->k, sizeof(double),
                           (size_t)c->g.npts, cudaMemcpyDeviceToDevice, s));
    GCKF(cudaMemsetAsync(c->b, 0, sizeof(double) * c->nvec * c->g.padded * c->k, s));
    rc = compute_scaling(c, s);
    if (rc != GA_OK) { gseterr(G, c->err); return fail(rc); }
  }
  GCKF(cudaStreamSynchronize(s));
  rc = build_graphs(G);
  if (rc != GA_OK) return fail(rc);
  *out = G;
  return GA_OK;
#undef GCKF
}

ga_status ga_group_set_forcing(ga_group* G, int i, const double* d_G, int nterms, const double* amp,
                               const double* omega, const double* phase, double t0, void* stream) {
  ga_status rc = check_group(G);
  if (rc != GA_OK) return rc;
  if (i < 0 || i >= (int)G->c.size()) { gseterr(G, "group: context index out of range"); return GA_ERR_ARG; }
  rc = ga_set_forcing(G->c[i], d_G, nterms, amp, omega, phase, t0, stream);
  if (rc != GA_OK) { gseterr(G, G->c[i]->err); return rc; }
  GCK(cudaStreamSynchronize((cudaStream_t)stream));
  return build_graphs(G);  // the step graphs add the forcing kernels of the forced contexts
}

ga_status ga_group_set_state(ga_group* G, const double* const* d_u0, const double* const* d_v0, void* stream) {
  ga_status rc = check_group(G);
  if (rc != GA_OK) return rc;
  if (!d_u0) { gseterr(G, "u0 is NULL"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const int k = G->k;
  for (size_t r = 0; r < G->c.size(); ++r) {
    ga_ctx* c = G->c[r];
    if (!d_u0[r]) { gseterr(G, "u0 entry is NULL"); return GA_ERR_ARG; }
    const long long vstride = (long long)c->nvec * c->g.padded;
    reset_status(c, s, 0);
    GCK(cudaMemsetAsync(c->chain, 0, sizeof(double) * 3 * k * vstride, s));
    launch_api_to_grid(c->g, c->nvec, c->nfree, c->map, d_u0[r], c->chain, 1, 0, c->st, s);
    if (d_v0 && d_v0[r]) launch_api_to_grid(c->g, c->nvec, c->nfree, c->map, d_v0[r], c->chain + vstride, 1, 0, c->st, s);
    GCK(cudaGetLastError());
  }
  // initial chain c_m = M^{-1}(F^{(m-2)} - K c_{m-2} [- C c_{m-1}]) as in ga_set_state (reading R3)
  const ga_ctx* c0 = G->c[0];
  const bool damped = c0->d.damp_a0 != 0.0 || c0->d.damp_a1 != 0.0;
  const int batch = damped ? 1 : std::min(2, k);
  for (int m0 = 2; m0 <= 3 * k - 1; m0 += batch) {
    int src[KMAX] = {-1, -1, -1, -1}, dst[KMAX] = {-1, -1, -1, -1}, src2[KMAX] = {-1, -1, -1, -1};
    for (int j = 0; j < batch; ++j)
      if (m0 + j <= 3 * k - 1) { src[j] = m0 + j - 2; dst[j] = m0 + j; if (damped) src2[j] = m0 + j - 1; }
    for (ga_ctx* c : G->c) {
      if (c->forcing) {
        ForceSlots fs;
        memset(&fs, 0, sizeof(fs));
        for (int j = 0; j < batch; ++j)
          if (dst[j] >= 0) { fs.active[j] = 1; fs.order[j] = dst[j] - 2; fs.toff[j] = 0.0; }
        GCK(cudaMemcpyAsync(c->fslots, &fs, sizeof(fs), cudaMemcpyHostToDevice, s));
      }
      launch_pack(c->g, c->nvec, k, c->chain, src, c->pred, c->st, s, src2, c->d.damp_a1);
    }
    GCK(cudaStreamSynchronize(s));  // fs lives on the host stack
    rc = run(G, K_SOLVEK, s);
    if (rc != GA_OK) return rc;
    for (ga_ctx* c : G->c) launch_unpack(c->g, c->nvec, k, c->x, dst, c->chain, c->st, s, src2, c->d.damp_a0);
    GCK(cudaGetLastError());
  }
  for (ga_ctx* c : G->c) {
    rc = set_predictors_and_norm(c, s);
    if (rc != GA_OK) { gseterr(G, c->err); return rc; }
  }
  GCK(cudaStreamSynchronize(s));
  return GA_OK;
}

ga_status ga_group_advance(ga_group* G, int nsteps, void* stream) {
  ga_status rc = check_group(G);
  if (rc != GA_OK) return rc;
  if (nsteps < 0) { gseterr(G, "nsteps < 0"); return GA_ERR_ARG; }
  for (int i = 0; i < nsteps; ++i) {
    rc = run(G, K_STEP, (cudaStream_t)stream);
    if (rc != GA_OK) return rc;
  }
  return GA_OK;
}

ga_status ga_group_apply(ga_group* G, int which, const double* const* d_x, double* const* d_y, void* stream) {
  ga_status rc = check_group(G);
  if (rc != GA_OK) return rc;
  if (which < 0 || which > 2 || !d_x || !d_y) { gseterr(G, "bad operator or NULL"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  for (size_t r = 0; r < G->c.size(); ++r) {
    ga_ctx* c = G->c[r];
    if (!d_x[r] || !d_y[r]) { gseterr(G, "NULL vector"); return GA_ERR_ARG; }
    const size_t mvbytes = sizeof(double) * c->nvec * c->g.padded * c->k;
    if (which < 2) {
      GCK(cudaMemsetAsync(c->pv, 0, mvbytes, s));
      launch_api_to_grid(c->g, c->nvec, c->nfree, c->map, d_x[r], c->pv, c->k, 0, c->st, s);
      launch_spmv(spmv_args(c, which, c->pv, c->q, SPMV_APPLY), s);
    } else {
      GCK(cudaMemsetAsync(c->r, 0, mvbytes, s));
      GCK(cudaMemsetAsync(c->pcg, 0, sizeof(PcgState), s));
      launch_api_to_grid(c->g, c->nvec, c->nfree, c->map, d_x[r], c->r, c->k, 0, c->st, s);
      PrecArgs a = prec_args(c, 0ull, 0);
      a.maxit = 0x7fffffff;
      a.xsum = xsum_of(c);  // no scalar step
      launch_precond(a, s);
    }
  }
  rc = xchg(G, s, X_NONE, which < 2 ? V_Q : V_Z);
  if (rc != GA_OK) return rc;
  for (size_t r = 0; r < G->c.size(); ++r) {
    ga_ctx* c = G->c[r];
    launch_grid_to_api(c->g, c->nvec, c->nfree, c->map, which < 2 ? c->q : c->z, c->k, 0, d_y[r], c->st, s);
  }
  GCK(cudaGetLastError());
  return GA_OK;
}

ga_status ga_group_solve_mass(ga_group* G, const double* const* d_b, double* const* d_x, int* iters, void* stream) {
  ga_status rc = check_group(G);
  if (rc != GA_OK) return rc;
  if (!d_b || !d_x) { gseterr(G, "NULL vector"); return GA_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  for (size_t r = 0; r < G->c.size(); ++r) {
    ga_ctx* c = G->c[r];
    if (!d_b[r] || !d_x[r]) { gseterr(G, "NULL vector"); return GA_ERR_ARG; }
    GCK(cudaMemsetAsync(c->b, 0, sizeof(double) * c->nvec * c->g.padded * c->k, s));
    launch_api_to_grid(c->g, c->nvec, c->nfree, c->map, d_b[r], c->b, c->k, 0, c->st, s);
  }
  rc = run(G, K_SOLVEB, s);
  if (rc != GA_OK) return rc;
  for (size_t r = 0; r < G->c.size(); ++r) {
    ga_ctx* c = G->c[r];
    launch_grid_to_api(c->g, c->nvec, c->nfree, c->map, c->x, c->k, 0, d_x[r], c->st, s);
  }
  GCK(cudaGetLastError());
  if (iters) {
    PcgState h;
    DevStatus hs;
    GCK(cudaMemcpyAsync(&h, G->c[0]->pcg, sizeof(h), cudaMemcpyDeviceToHost, s));
    GCK(cudaMemcpyAsync(&hs, G->c[0]->st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    GCK(cudaStreamSynchronize(s));
    *iters = h.its[0];
    if (hs.status != 0) return (ga_status)hs.status;
  }
  return GA_OK;
}

const char* ga_group_last_error(const ga_group* G) {
  if (G) return G->err.c_str();
  return g_group_err.c_str();
}

void ga_group_destroy(ga_group* G) {
  if (!G) return;
  destroy_graphs(G);
  for (ga_ctx* c : G->c)
    if (c && c->grp == G) c->grp = nullptr;
  for (cudaStream_t t : G->st)
    if (t) cudaStreamDestroy(t);
  for (cudaEvent_t e : G->ev_join)
    if (e) cudaEventDestroy(e);
  if (G->ev_fork) cudaEventDestroy(G->ev_fork);
  for (cudaStream_t t : G->st2)
    if (t) cudaStreamDestroy(t);
  for (cudaEvent_t e : G->ev_join2)
    if (e) cudaEventDestroy(e);
  if (G->ev_fork2) cudaEventDestroy(G->ev_fork2);
  if (G->cap) cudaStreamDestroy(G->cap);
  if (G->aux) cudaStreamDestroy(G->aux);
  delete G;
}

}  // extern "C"
