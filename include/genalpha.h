/*
 * genalpha.h — C ABI of the B200-native explicit order-2k generalized-alpha
 * integrator for isogeometric (B-spline) discretizations of the scalar wave
 * equation and linear elastodynamics (arXiv 2102.11536, "PAPER.md").
 *
 * Citations are PAPER.md line numbers (P:line) and DESIGN.md readings (Rn).
 *
 * Problem:  M U'' + C U' + K U = F, U(0) = U0, U'(0) = V0, with M, K
 * the Galerkin mass and stiffness matrices of a maximal-regularity B-spline
 * space of degree p on one patch or on a block-structured conforming
 * multi-patch domain, Dirichlet data on the whole boundary:
 * homogeneous by default, non-homogeneous by lifting (ga_set_dirichlet).
 * C = 0 and F = 0 unless set: Rayleigh damping C = damp_a0 M + damp_a1 K
 * (ga_desc, reading R16) and forcing F = G h(t) (ga_set_forcing, reading
 * R15).  Time stepping is the explicit order-2k
 * scheme of P:398-431 (k mass solves + updates of the other 2k variables per
 * step), with the K-term reading R1 and parameter set R2 of DESIGN.md.  Each
 * mass solve is PCG with the diagonal-scaled Kronecker preconditioner
 * (P:703-713), additive Schwarz across patches.
 *
 * Conventions (apply to every entry point)
 *  - Ownership: the CALLER owns all device memory.  The library never calls
 *    cudaMalloc: it carves its arrays out of the workspace passed to
 *    ga_create.  Host arrays passed in are copied before the call returns.
 *  - Streams: device work is enqueued on the given stream, asynchronously,
 *    unless the entry point says it synchronizes.  A context must be used by
 *    one stream at a time (the caller orders calls on different streams).
 *  - Vectors ("free-DoF vectors") are fp64 device arrays of length n_free
 *    (from ga_query).  Order: component-major (all DoFs of component 0, then
 *    1, ...); within a component the free DoFs in co-lexicographic order
 *    (x fastest) of the global masked grid;
 *    ga_free_dof_map gives (patch, control point) of each entry.
 *  - Errors are status codes; nothing throws across the ABI.  After a device
 *    side failure (PCG not converged, instability) the context refuses
 *    further stepping until ga_set_state / ga_set_chain.
 *  - Numbers: everything is IEEE fp64.
 */
#ifndef GENALPHA_H
#define GENALPHA_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GA_OK = 0,
  GA_ERR_ARG = -1,         /* invalid argument / unsupported layout                      */
  GA_ERR_PARAM = -2,       /* rho outside [0,1], rho_s > rho_b, or undefined parameters   */
  GA_ERR_GEOMETRY = -3,    /* |J| <= 0 at a Gauss point (assumption P:699-701)           */
  GA_ERR_CONFORMITY = -4,  /* patch interfaces do not match (assumption P:645-652)       */
  GA_ERR_NOCONV = -5,      /* a PCG solve reached pcg_maxit                              */
  GA_ERR_UNSTABLE = -6,    /* ||U||_2 exceeded unstable_factor * ||U_0||_2               */
  GA_ERR_CUDA = -7,        /* a CUDA runtime call failed (see ga_last_error)             */
  GA_ERR_OOM = -8          /* workspace or scratch smaller than ga_query asked for       */
} ga_status;

typedef struct ga_ctx ga_ctx; /* opaque; holds host metadata and views into the workspace */

/* One patch.  All patches share p and n ("same degree p", uniform
 * refinement).  cell = position of the patch in the coarse patch grid of a
 * block-structured multi-patch layout (identity orientation); the patch
 * occupies [cell_d, cell_d + 1] in parametric "patch-grid" coordinates.
 * ctrl: HOST array of (n+p)^dim control points, co-lexicographic (x fastest),
 * dim doubles per point.  Copied by ga_query/ga_create. */
typedef struct {
  int cell[3];
  const double* ctrl;
} ga_patch;

/* Subdomain of a partitioned multi-patch problem (patch-per-GPU mode): the
 * context holds ONE patch of a conforming multi-patch domain of any layout (arbitrary patch
 * orientations, any number of patches at a vertex, e.g. a fan) and its operators are the patch's
 * LOCAL contributions M^(r), K^(r) (M = sum_r P_r^T M^(r) P_r).  Interface DoFs are
 * free DoFs of every patch that holds a copy; a ga_group (below) sums the partial values of the
 * copies after every operator and preconditioner application, so the vectors of all subdomains
 * stay consistent (equal values on every copy).  Produce the arrays with ga_partition_plan.
 * All arrays are HOST, (n+p)^dim entries in the patch's co-lexicographic control-point order,
 * copied by ga_create. */
typedef struct {
  const unsigned char* free_mask; /* 1: free DoF of the global problem (not Dirichlet)      */
  const unsigned char* owned;     /* 1: this subdomain counts the DoF in global norms (one owner   */
                                  /*    per free DoF across all subdomains)                       */
  const long long* iface;         /* global interface slot (0..n_iface-1) of a DoF with copies in  */
                                  /* >= 2 patches, -1 otherwise                                   */
  long long n_iface;              /* number of interface DoFs of the whole domain (same for all)  */
} ga_subdomain;

typedef struct {
  int dim;              /* 2 or 3                                                     */
  int ncomp;            /* 1: scalar wave u'' = div(omega^2 grad u);            */
                        /* dim: linear elasticity (lame_lambda, lame_mu, density)      */
  int p;                /* spline degree, 1..7, maximal regularity C^{p-1}    */
  int n;                /* elements per direction per patch, >= 1                     */
  int npatch;           /* 1..16.  Layouts are block-structured (each patch one cell   */
                        /* of a coarse patch grid, identity orientation), so there is  */
                        /* no interface list and no preconditioner choice in the       */
                        /* descriptor: interfaces follow from the cells, and the       */
                        /* preconditioner is always the banded Kronecker one (K4; the  */
                        /* fast-diagonalisation variant K4' is not built)              */
  const ga_patch* patches;
  double omega;         /* wave speed (scalar wave)                                   */
  double lame_lambda, lame_mu, density; /* elasticity only                            */
  int k;                /* accuracy order 2k, 1 <= k <= 4                 */
  double rho_b, rho_s;  /* spectral radius parameters, 0 <= rho_s <= rho_b <= 1*/
  int param_set;        /* 0: isospectral j<k set (R2, default);            */
                        /* 1: j<k set as printed in P:494-496 (requires rho_b < 1)     */
  double dt;            /* time step tau > 0                                          */
  double pcg_rtol;      /* stop when ||r||_2 <= pcg_rtol ||b||_2 (BASELINE: 1e-13)      */
  int pcg_maxit;        /* per solve (main + refinement), e.g. 500                    */
  int pcg_refine;       /* 1: after convergence restart once from the true residual  */
                        /*    b - M x (R8); 0: plain PCG                     */
  double pcg_refine_rtol; /* refinement stop: 0 -> ||r|| <= pcg_rtol ||b||; > 0 ->      */
                        /*    ||r|| <= min(pcg_rtol ||b||, pcg_refine_rtol ||b - M x0||)*/
                        /*    (x0 = main-phase result; reaching pcg_maxit here is not   */
                        /*    an error).  1e-3 recommended for p >= 5 (kappa(M) ~1e8)   */
  double unstable_factor; /* GA_ERR_UNSTABLE threshold on ||U|| / sqrt(ref); ref =      */
                        /* ||U0||^2 + dt^2 ||V0||^2, or the first non-zero ||U_n||^2  */
                        /* of a run that starts from rest; 0 disables                 */
  int op_mode;          /* operator representation: */
                        /* 1: assembled column-index-free stencils (2p+1)^dim per row;  */
                        /* 2: matrix-free sum factorisation from the Gauss-point data   */
                        /*    (single patch only; the elastic K stays a stencil);       */
                        /* 3: half-symmetric stencils, offsets o >= 0 only: half the    */
                        /*    memory; 3D scalar grids read each stored coefficient once */
                        /*    (single-read symmetric SpMV, half the bytes per apply),   */
                        /*    2D and the elastic mass twice; the elastic K stays full;  */
                        /* 0: auto, the measured-faster one (R14): 3D scalar  */
                        /*    grids beyond the persistent solver's size take 3 when     */
                        /*    p >= 4, or the 32-point x-segments are well used; else    */
                        /*    full stencils if they fit in ~150 GB, else half-          */
                        /*    symmetric, else matrix-free                               */
  double damp_a0, damp_a1; /* Rayleigh damping C = damp_a0 M + damp_a1 K, >= 0 (SURVEY    */
                        /* NEXT-2; reading R16: block j subtracts C w_j, w_j the Taylor */
                        /* predictor of its velocity-level entry for j < k); 0 0: none  */
  const ga_subdomain* sub; /* NULL: the context is the whole problem.  Non-NULL: npatch must */
                        /* be 1 and the context is one subdomain of a partitioned problem */
                        /* (cell ignored); it is stepped only through a ga_group, op_mode */
                        /* 2 (matrix-free) and Dirichlet lifting are not available       */
} ga_desc;

typedef struct {
  long long steps;          /* steps completed since the last ga_set_state/ga_set_chain */
                            /* (statistics counter)                                     */
  long long solves;         /* mass solves completed                                    */
  long long pcg_iters[4];   /* total PCG iterations per block (incl. refinement)        */
  int last_iters[4];        /* iterations of the most recent solve, per block          */
  int max_iters;            /* max iterations of any single solve                       */
  double max_rel_residual;  /* max final ||r||/||b|| (recursive) over solves            */
  int status;               /* ga_status of the device-side run                         */
  long long fail_step;      /* step at which status became non-zero (-1 if none)        */
  int fail_block;           /* block (0-based) that failed (-1 if none)                 */
  long long kernel_launches;/* kernels of this library executed on the device since    */
                            /* the last ga_set_state (counted on the device)            */
  long long loop_iters;     /* lock-stepped PCG iterations executed (all solves)        */
  long long step_index;     /* simulation step n of the state (t_n = t0 + n dt for the   */
                            /* forcing): 0 after ga_set_state, +1 per step, NOT reset by */
                            /* ga_set_chain, set by ga_set_time                         */
} ga_stats;

/* Generalized-alpha parameters of the k blocks (host only, no GPU).
 * alpha/beta/gamma/alpha_f: arrays of length k (block j = index j-1):
 * blocks j < k: alpha_f = 1 and (param_set 0) the isospectral closed forms of
 * DESIGN.md R2, or (1) P:494-496; block k: P:497-499, alpha_f = 0;
 * gamma = 1/2 - alpha_f + alpha.  theta_max (may be NULL) receives the
 * stability limit Theta_max = tau^2 lambda_max of block k (R2/G3),
 * equal for every block under param_set 0.  Returns GA_ERR_PARAM on bad rho. */
ga_status ga_params(int k, double rho_b, double rho_s, int param_set,
                    double* alpha, double* beta, double* gamma, double* alpha_f,
                    double* theta_max);

/* Spectral radius rho(G(Theta)) of the amplification matrix for n values Theta = tau^2 lambda
 * (Figs. 1-2): d_theta, d_rho device arrays of n doubles; G is
 * block upper triangular with the 3x3 blocks Lambda_j of the same parameters as
 * ga_params, so rho(G) = max_j of the largest root of det(mu - Lambda_j) (closed-form cubic).
 * Asynchronous on stream, no context needed.  GA_ERR_PARAM on bad rho. */
ga_status ga_spectral_scan(int k, double rho_b, double rho_s, int param_set, const double* d_theta, int n,
                           double* d_rho, void* stream);

/* Sizes for a descriptor (host only, no GPU).  n_free: length of a free-DoF
 * vector (= ncomp * scalar free DoFs).  workspace_bytes: device memory the
 * context keeps for its lifetime.  scratch_bytes: device memory needed only
 * during ga_create (operator assembly); any size >= scratch_min works
 * (smaller means more assembly passes).  Pointers may be NULL. */
ga_status ga_query(const ga_desc* desc, size_t* n_free, size_t* workspace_bytes,
                   size_t* scratch_bytes, size_t* scratch_min);

/* Create a context: validates desc, uploads geometry, assembles M and K on
 * the GPU into the stencil layout, builds the preconditioner and the step
 * graphs.  d_workspace: >= workspace_bytes, 256-byte aligned, owned by the
 * caller and kept alive until ga_destroy.  d_scratch: >= scratch_min bytes,
 * may be released after return.  SYNCHRONIZES stream once (reads back the
 * minimum |J| for GA_ERR_GEOMETRY).  *out is NULL on failure. */
ga_status ga_create(const ga_desc* desc, void* d_workspace, size_t workspace_bytes,
                    void* d_scratch, size_t scratch_bytes, void* stream, ga_ctx** out);

/* Initial chain (R3): c0 = U0, c1 = V0,
 * c_m = M^{-1}(-K c_{m-2}), m = 2..3k-1 (3k-2 PCG solves; zero right-hand
 * sides are skipped).  d_v0 may be NULL (V0 = 0).  Resets stats. */
ga_status ga_set_state(ga_ctx* ctx, const double* d_u0, const double* d_v0, void* stream);

/* Forcing F(x, t) = G(x) h(t) with h(t) = sum_{i<nterms} amp_i cos(omega_i t + phase_i)
 * (eq:ho1 P:398-404): block j's right-hand side becomes
 * F^{(3j-3)}(t_n + alpha_fj dt) - K s_j, and the initial chain of ga_set_state
 * c_m = M^{-1}(F^{(m-2)}(t0) - K c_{m-2}); t_n = t0 + n dt with n the steps since
 * ga_set_state.  d_G: device free-DoF vector of the load integrals int g B_i (layout as
 * ga_set_state's u0), copied; NULL (or nterms = 0) removes the forcing.  1 <= nterms <= 8,
 * amp/omega/phase: host arrays, copied.  Call before ga_set_state for a forced initial
 * chain.  SYNCHRONIZES stream (the step graphs are re-captured).  GA_ERR_ARG on bad terms. */
ga_status ga_set_forcing(ga_ctx* ctx, const double* d_G, int nterms, const double* amp, const double* omega,
                         const double* phase, double t0, void* stream);

/* Set the simulation step index n (t_n = t0 + n dt of the forcing and lifting time functions),
 * e.g. after restoring a checkpoint into a fresh context with ga_set_chain.  Asynchronous.
 * GA_ERR_ARG if step_index < 0. */
ga_status ga_set_time(ga_ctx* ctx, long long step_index, void* stream);

/* Non-homogeneous Dirichlet data by lifting, single patch,
 * scalar wave: the boundary control coefficients are U_b(t) = g_b h_D(t), h_D(t) = sum_{i<nterms}
 * amp_i cos(omega_i t + phase_i), 1 <= nterms <= 4.  h_g: HOST array of all (n+p)^dim control
 * values of the patch (co-lexicographic); only the boundary entries are used.  The free
 * equations receive -M_fb g_b (h_D'' + a0 h_D') - K_fb g_b (h_D + a1 h_D') (C = a0 M + a1 K,
 * ga_desc.damp_a0/a1) as two forcing pairs on top of ga_set_forcing's, with the same time origin
 * t0 (set by ga_set_forcing, default 0); M_fb g_b and K_fb g_b are computed once on the GPU by
 * the assembly (boundary columns).  The returned u, v, a are the free DoFs; the boundary values
 * are g_b h_D(t).  d_scratch: >= ga_query's scratch_min bytes, released by the caller after the
 * call.  h_g = NULL removes the lifting.  SYNCHRONIZES stream.  GA_ERR_ARG: multi-patch or
 * elasticity, bad terms. */
ga_status ga_set_dirichlet(ga_ctx* ctx, const double* h_g, int nterms, const double* amp, const double* omega,
                           const double* phase, void* d_scratch, size_t scratch_bytes, void* stream);

/* Advance nsteps explicit steps.  Asynchronous; a device-side
 * failure stops further steps and is reported by ga_get_stats. */
ga_status ga_advance(ga_ctx* ctx, int nsteps, void* stream);

/* Copy U, V, A (c0, c1, c2) to caller vectors; any pointer may be NULL. */
ga_status ga_get_state(ga_ctx* ctx, double* d_u, double* d_v, double* d_a, void* stream);

/* Checkpoint / resume of the whole chain c_m, m = 0..3k-1 (free-DoF vectors).  ga_set_chain
 * with m = 0 resets the statistics and the failure status but keeps the simulation step index
 * (ga_stats.step_index; set it with ga_set_time when resuming in a new context). */
ga_status ga_get_chain(ga_ctx* ctx, int m, double* d_out, void* stream);
ga_status ga_set_chain(ga_ctx* ctx, int m, const double* d_in, void* stream);

/* SYNCHRONIZES stream; fills *out. */
ga_status ga_get_stats(ga_ctx* ctx, ga_stats* out, void* stream);

/* Test / tooling hooks.  which: 0 = M, 1 = K, 2 = preconditioner inverse
 * calM^{-1} (P:703-713 / P:766).  y = op(x), free-DoF vectors. */
ga_status ga_apply(ga_ctx* ctx, int which, const double* d_x, double* d_y, void* stream);

/* x = M^{-1} b by the same PCG the step uses (zero initial guess).
 * *iters (may be NULL) receives the iteration count; if non-NULL the call
 * SYNCHRONIZES stream. */
ga_status ga_solve_mass(ga_ctx* ctx, const double* d_b, double* d_x, int* iters, void* stream);

/* lambda_max(M^{-1} K) by `iters` (<= 512) Lanczos steps in the M inner product (each one K
 * apply, one PCG mass solve and one M apply; no reorthogonalisation: the extremal Ritz value
 * converges first), for the CFL time step dt = c sqrt(theta_max / lambda_max).  The time-
 * stepping state (chain, predictors, forcing slots) and the statistics / status are restored
 * on every return path, so a Lanczos solve never counts as a step solve and a Lanczos NOCONV
 * is returned, not latched.  SYNCHRONIZES stream. */
ga_status ga_lambda_max(ga_ctx* ctx, int iters, double* lam, void* stream);

/* host_map[f] = patch * (n+p)^dim + local control-point index (co-lex) of
 * free scalar DoF f, f < n_free / ncomp.  Host only. */
ga_status ga_free_dof_map(const ga_ctx* ctx, long long* host_map);

/* Tooling: enqueue `reps` launches of one hot-path kernel with the launch
 * configuration the step uses, on the context's scratch PCG vectors (the
 * time-stepping state is not modified), so a caller can time it with events.
 * op: 0 = M stencil SpMV + p.q reduction on the k lock-stepped vectors,
 *     1 = K stencil SpMV (b = -K s), 2 = one preconditioner application
 *     (scaling + all line sweeps + r.z/r.r reductions), 3 = predictor pass of
 *     the stage kernel (reads the 3k chain, writes the k predictors),
 *     4 = M stencil SpMV without reduction, 5 = PCG direction update p = z + beta p,
 *     (ops 2 and 5 run on a profiling PcgState with every block active and beta != 0, so
 *     they do their full work; the PcgState is zeroed afterwards),
 *     6 = one complete lock-stepped mass solve of the current right-hand sides
 *     (the persistent solver kernel on small grids; its step graph otherwise). */
/* Persistent-solver mode: 1 if ga_create chose the single-kernel cooperative PCG
 * solve (small single-patch scalar problems; env GA_PERSIST=0/1 overrides). */
int ga_uses_persistent_solver(const ga_ctx* ctx);
/* 1 if the context applies M (and the scalar K) matrix-free (op_mode 2, or op_mode 0's pick). */
int ga_uses_matrix_free(const ga_ctx* ctx);
/* Operator representation in use: 1 full stencils, 2 matrix-free, 3 half-symmetric stencils. */
int ga_operator_mode(const ga_ctx* ctx);
ga_status ga_profile_op(ga_ctx* ctx, int op, int reps, void* stream);

void ga_destroy(ga_ctx* ctx);

/* ===========================================================================================
 * Partitioned multi-patch (patch-per-GPU; additive Schwarz P:763-783)
 * =========================================================================================== */

/* Partition plan of a conforming multi-patch domain (host only, no GPU).  ctrl[r]: HOST array of
 * (n+p)^dim control points of patch r (co-lex, dim doubles each).  Gluing: two local
 * control points are copies of one global function iff their control points are bitwise equal
 * (conformity); a patch face is an interface iff its control-point set equals a face
 * of another patch; a global function is Dirichlet iff a copy lies on a face that is not an
 * interface.  Outputs (caller-allocated, npatch * (n+p)^dim entries, patch-major), the
 * ga_subdomain arrays of every patch: free_mask, owned (the first copy in (patch, local index)
 * order owns a free DoF), iface (slots numbered in first-copy order).  *n_iface and
 * *n_free_global (either may be NULL) receive the interface and free DoF counts.
 * GA_ERR_ARG: bad sizes / NULL; GA_ERR_CONFORMITY: a face shares some but not all of its points
 * with another patch's face (non-conforming interface). */
ga_status ga_partition_plan(int dim, int p, int n, int npatch, const double* const* ctrl,
                            unsigned char* free_mask, unsigned char* owned, long long* iface,
                            long long* n_iface, long long* n_free_global);

/* A group steps the subdomain contexts of one partitioned problem together.  The contexts of
 * this process are passed in ctxs (any number >= 1, all created with a ga_subdomain of the same
 * plan, the same k, ncomp, dt, rho, PCG settings, all on the current device); the others live in
 * other processes, one NCCL communicator connecting the processes (nccl_comm from
 * ga_nccl_comm_init, NULL for a single process).  Per PCG iteration of the lock-stepped solve the
 * group makes two exchanges (after q = M p and after z = calM^{-1} r): each context writes the
 * partial values of its interface DoFs and its partial dot products into its exchange buffer,
 * the buffers of the process are summed in a fixed order, then NCCL all-reduces the sum across
 * processes (ncclSum, fp64), and every context takes back the sums: q, z stay consistent and all
 * contexts compute the same alpha, beta and convergence decisions.  p.q and r.z are sums of the
 * unassembled local products (p^T M p = sum_r p_r^T M^(r) p_r), ||r||^2 and ||b||^2 count every
 * DoF once (owned mask).  The step is one CUDA graph (PCG loops as conditional WHILE nodes) for
 * a single process; with NCCL the iteration is a captured graph relaunched by the host, which
 * polls the convergence flags one iteration behind.
 * ga_group_create SYNCHRONIZES stream: it sums diag(M) over the copies (D^(r) of P:779 is the
 * global diagonal, reading R6), sets the preconditioner scalings and builds the graphs. */
typedef struct ga_group ga_group;
ga_status ga_group_create(ga_ctx* const* ctxs, int nctx, void* nccl_comm, void* stream, ga_group** out);
/* ga_set_state of every local context (d_u0[i], d_v0[i] for ctxs[i]; d_v0 or entries may be
 * NULL): consistent free-DoF vectors of each subdomain (equal values on interface copies). */
ga_status ga_group_set_state(ga_group* g, const double* const* d_u0, const double* const* d_v0, void* stream);
ga_status ga_group_advance(ga_group* g, int nsteps, void* stream);
/* which: 0 = M, 1 = K, 2 = calM_ad^{-1}: y_i = (op x)_i restricted to subdomain i, with
 * the operators of the whole (glued) problem; x consistent.  For tests / tooling. */
ga_status ga_group_apply(ga_group* g, int which, const double* const* d_x, double* const* d_y, void* stream);
/* x = M^{-1} b by the group PCG (zero initial guess); *iters (may be NULL) SYNCHRONIZES. */
ga_status ga_group_solve_mass(ga_group* g, const double* const* d_b, double* const* d_x, int* iters, void* stream);
/* Forcing of a subdomain context: as ga_set_forcing, but d_G holds this subdomain's LOCAL load
 * integrals int_{Omega_r} g B_i (the group sums the copies).  Call before ga_group_set_state. */
ga_status ga_group_set_forcing(ga_group* g, int i, const double* d_G, int nterms, const double* amp,
                               const double* omega, const double* phase, double t0, void* stream);
void ga_group_destroy(ga_group* g);
/* Last error message of a group call (or of the calling thread's last group call if g is NULL). */
const char* ga_group_last_error(const ga_group* g);

/* NCCL plumbing for multi-process groups (libnccl.so.2 is loaded at run time: env GA_NCCL_LIB or
 * the default search path).  ga_nccl_unique_id: rank 0 writes 128 bytes that every rank passes
 * to ga_nccl_comm_init (the caller moves them, e.g. with torch.distributed.broadcast).
 * GA_ERR_ARG if NCCL cannot be loaded or fails. */
ga_status ga_nccl_unique_id(void* id128);
ga_status ga_nccl_comm_init(int nranks, const void* id128, int rank, void** comm);
void ga_nccl_comm_destroy(void* comm);

/* Last error message of ctx (or of the calling thread if ctx is NULL). */
const char* ga_last_error(const ga_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GENALPHA_H */
