// Shared device-side definitions of the CUDA path (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ga {

constexpr int KMAX = 4;           // max blocks k (right-hand sides per lock-stepped solve)
constexpr int NTHREADS = 256;     // default block size for grid kernels
constexpr int MAXPATCH = 16;
constexpr int XSCAL = 4 * KMAX;  // scalars of a subdomain exchange (dist.cu): up to 2 KMAX sums + spare

// Device-resident PCG scalars of one lock-stepped solve set.
struct PcgState {
  double bb[KMAX];      // ||b_j||^2
  double rz[KMAX];      // r.z of the current iteration
  double rzold[KMAX];   // r.z of the previous iteration
  double rr[KMAX];      // ||r_j||^2
  double pq[KMAX];      // p.q
  double alpha[KMAX];
  double beta[KMAX];
  double thr[KMAX];     // convergence threshold on ||r_j||^2 of the current phase
  int active[KMAX];     // 1 while block j has not converged
  int its[KMAX];        // iterations of block j in this solve (both phases)
  int iter;             // iterations of the current phase
  int pfirst;           // next p update is p = z
  int first;            // F1 has not run yet in this phase
  int nrhs;             // right-hand sides in use (<= KMAX)
  int phase;            // 0 main solve, 1 refinement restart
  int guard;            // F1 calls in this phase (safety stop if F2 never ran)
};

// Device-resident run status and statistics.
struct DevStatus {
  int status;                 // ga_status of the device-side run
  int fail_block;
  long long fail_step;
  long long steps;
  long long solves;
  long long pcg_iters[KMAX];
  int last_iters[KMAX];
  int max_iters;
  double max_relres;
  double u0norm2;             // instability reference: ||U_0||^2 + dt^2 ||V_0||^2, or the first
                              // non-zero ||U_n||^2 when the run starts from rest (0 = not yet set)
  long long tstep;            // simulation step index n (t_n = t0 + n dt of the forcing); reset by
                              // ga_set_state / ga_set_time only, never by ga_set_chain
  unsigned long long launches;
  long long loop_iters;       // lock-stepped PCG iterations executed
};

// Reduction scratch: partial sums per block + a completion counter per site.
struct RedScratch {
  double* partial;            // [maxblocks][2*KMAX]
  unsigned int* counter;      // one per reduction site
};

// Description of the global grid of free points (interior coordinates).
struct GridDesc {
  int dim;
  int nx, ny, nz;             // nz = 1 in 2D
  long long npts;             // nx*ny*nz
  long long guard;            // guard elements before/after each vector
  long long padded;           // npts + 2*guard
  long long cs;               // row stride of the stencil coefficient arrays (npts rounded up to 32)
};

// Segment-blocked layout of the 3D half-symmetric stencils (spmv_sym.cu): each x-line of nx
// points is split into nseg = ceil(nx / 32) segments of XS = 32 points (the last one partial).
// Row block b = seg + nseg (y + ny z); coefficient h (0 <= h < Sh) of point x = 32 seg + l at
// ((b Sh + h) 32 + l): one offset of a block is 256 contiguous bytes, so a warp load is whole
// 64-byte DRAM granules and every offset of the kernel's loads is an immediate.
constexpr int SYM_STRIDE = 32;
struct SymLayout {
  int xs, nseg;
};
inline SymLayout sym_layout(int nx) {
  SymLayout L;
  L.nseg = (nx + 31) / 32;
  L.xs = SYM_STRIDE;
  return L;
}
__host__ __device__ __forceinline__ long long sym_index(int x, int y, int z, long long h, int xs, int nseg, int ny,
                                                        long long Sh) {
  const int seg = x / xs;
  const long long b = seg + (long long)nseg * (y + (long long)ny * z);
  return (b * Sh + h) * SYM_STRIDE + (x - seg * xs);
}

__device__ __forceinline__ unsigned long long gtid() {
  return (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV values per thread; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double sh[32][NV > 0 ? NV : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) sh[wid][j] = v[j];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double t = lane < nw ? sh[lane][j] : 0.0;
      v[j] = warp_sum(t);
    }
  }
  __syncthreads();
}

// Write this block's NV partial sums; returns true in thread 0 of the LAST
// block to finish, after which `out` holds the totals summed in block order
// (deterministic: independent of which block finishes last).
template <int NV>
__device__ __forceinline__ bool reduce_last_block(double (&v)[NV], double* partial,
                                                  unsigned int* counter, double (&out)[NV]) {
  block_sum<NV>(v);
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) partial[(size_t)blockIdx.x * NV + j] = v[j];
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // the last block sums the partials: thread t takes a contiguous chunk of
  // blocks, then a fixed-shape block reduction combines the chunks; the
  // result depends only on gridDim/blockDim, not on which block finished last
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  const unsigned int nb = gridDim.x;
  const unsigned int chunk = (nb + blockDim.x - 1) / blockDim.x;
  unsigned int b0 = threadIdx.x * chunk, b1 = min(nb, b0 + chunk);
  for (unsigned int b = b0; b < b1; ++b)
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] += ((volatile double*)partial)[(size_t)b * NV + j];
  block_sum<NV>(acc);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) out[j] = acc[j];
    *counter = 0u;  // ready for the next launch
  }
  return threadIdx.x == 0;
}

__device__ __forceinline__ void count_launch(DevStatus* st) {
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&st->launches, 1ull);
}

}  // namespace ga
