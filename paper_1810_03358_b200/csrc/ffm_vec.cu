// ffm_vec.cu -- optimiser vector algebra kept resident in HBM.
//
// The reference drivers do their vector algebra in NumPy on the host
// (ffmin/optimizers/*.py); here x, g, s, y and the search directions never
// leave the device.  All reductions use a fixed grid and a fixed combination
// order, so every dot product -- and therefore every optimiser trace -- is
// bit-identical run to run.
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "../../include/ffmin_b200.h"
#include "ffm_kernels.h"
#include "ffm_two_loop.cuh"

namespace cg = cooperative_groups;

namespace ffm {

constexpr int kVecBlocks = 296;  // 2 per SM on 148 SMs
constexpr int kVecThreads = 256;

int vec_reduce_blocks() { return kVecBlocks; }

__device__ __forceinline__ double block_sum256(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kVecThreads / 32; ++w) s += sh[w];
  __syncthreads();
  return s;  // thread 0
}

__global__ void __launch_bounds__(kVecThreads)
dot_partial_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                   double* __restrict__ part) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[kVecThreads / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < n;
       i += (int64_t)kVecBlocks * kVecThreads)
    acc = fma(x[i], y[i], acc);
  const double s = block_sum256(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kVecThreads)
dot_final_kernel(const double* __restrict__ part, double* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[kVecThreads / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < kVecBlocks; i += kVecThreads) acc += part[i];
  const double s = block_sum256(acc, sh);
  if (threadIdx.x == 0) *out = s;
}

cudaError_t launch_dot(int64_t n, const double* x, const double* y, double* part,
                       double* out, cudaStream_t st) {
  count_launch(); launch_k(dot_partial_kernel, kVecBlocks, kVecThreads, 0, st, n, x, y, part);
  count_launch(); launch_k(dot_final_kernel, 1, kVecThreads, 0, st, part, out);
  return cudaGetLastError();
}

// up to kMaxDots dot products in one pass (the optimisers need 3-5 per step)
constexpr int kMaxDots = 8;
struct DotArgs {
  int k;
  const double* x[kMaxDots];
  const double* y[kMaxDots];
};

__global__ void __launch_bounds__(kVecThreads)
dots_partial_kernel(int64_t n, DotArgs A, double* __restrict__ part) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[kVecThreads / 32];
  for (int q = 0; q < A.k; ++q) {
    double acc = 0.0;
    const double* __restrict__ x = A.x[q];
    const double* __restrict__ y = A.y[q];
    for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < n;
         i += (int64_t)kVecBlocks * kVecThreads)
      acc = fma(x[i], y[i], acc);
    const double s = block_sum256(acc, sh);
    if (threadIdx.x == 0) part[q * kVecBlocks + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kVecThreads)
dots_final_kernel(int k, const double* __restrict__ part, double* __restrict__ out) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[kVecThreads / 32];
  for (int q = 0; q < k; ++q) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < kVecBlocks; i += kVecThreads) acc += part[q * kVecBlocks + i];
    const double s = block_sum256(acc, sh);
    if (threadIdx.x == 0) out[q] = s;
  }
}

// vectors this short are reduced by one block in one launch (the small
// systems' minimiser graphs run ~3 of these per iteration: one node instead
// of two, no partial round trip)
constexpr int64_t kSmallVecN = 6144;

__global__ void __launch_bounds__(kVecThreads)
dots_small_kernel(int64_t n, DotArgs A, double* __restrict__ out) {
  pdl_wait();
  FFM_MSTAMP(22);
  pdl_launch_dependents();
  __shared__ double sh[kVecThreads / 32];
  for (int q = 0; q < A.k; ++q) {
    double acc = 0.0;
    const double* __restrict__ x = A.x[q];
    const double* __restrict__ y = A.y[q];
    for (int64_t i = threadIdx.x; i < n; i += kVecThreads) acc = fma(x[i], y[i], acc);
    const double s = block_sum256(acc, sh);
    if (threadIdx.x == 0) out[q] = s;
  }
}

cudaError_t launch_dots(int64_t n, int k, const double* const* x, const double* const* y,
                        double* part, double* out, cudaStream_t st) {
  if (k < 1 || k > kMaxDots) return cudaErrorInvalidValue;
  DotArgs A;
  A.k = k;
  for (int q = 0; q < k; ++q) {
    A.x[q] = x[q];
    A.y[q] = y[q];
  }
  if (n <= kSmallVecN) {
    count_launch();
    launch_k(dots_small_kernel, 1, kVecThreads, 0, st, n, A, out);
    return cudaGetLastError();
  }
  count_launch();
  launch_k(dots_partial_kernel, kVecBlocks, kVecThreads, 0, st, n, A, part);
  count_launch();
  launch_k(dots_final_kernel, 1, kVecThreads, 0, st, k, part, out);
  return cudaGetLastError();
}

// z = sa * (a * x + b * y); a, b from device pointers when given.  y may be
// null (then b is ignored).
__global__ void axpby_kernel(int64_t n, const double* __restrict__ a_dev, double a_host,
                             double sa, const double* __restrict__ x,
                             const double* __restrict__ b_dev, double b_host,
                             const double* __restrict__ y, double* __restrict__ z) {
  pdl_wait();
  pdl_launch_dependents();
  const double a = a_dev ? *a_dev : a_host;
  const double b = b_dev ? *b_dev : b_host;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = a * x[i];
    if (y) v = fma(b, y[i], v);
    z[i] = sa * v;
  }
}

cudaError_t launch_axpby(int64_t n, const double* a_dev, double a_host, double sa,
                         const double* x, const double* b_dev, double b_host,
                         const double* y, double* z, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * kVecBlocks) blocks = 4 * kVecBlocks;
  if (blocks < 1) blocks = 1;
  count_launch(); launch_k(axpby_kernel, (int)blocks, 256, 0, st, n, a_dev, a_host, sa, x, b_dev, b_host, y, z);
  return cudaGetLastError();
}

// --------------------------------------------------- L-BFGS two-loop
// ffmin/optimizers/lbfgs.py:53-75 (Algorithm 3): one cooperative kernel with
// 2 m + 1 grid-wide phases and no host round trip.  S and Y are ring buffers
// [m][n]; the host passes the ring order (newest first) and rho_i.  Partial
// sums rotate through three scratch rows so a row is never rewritten while a
// slower block may still be reading it.
struct TwoLoopArgs {
  int64_t n;
  int count;
  int idx[kMaxLbfgsPairs];     // ring slots, newest first
  double rho[kMaxLbfgsPairs];  // 1 / <s_i, y_i>, same order
  const double* S;
  const double* Y;
  const double* g;
  double* q;     // output: the raw quasi-Newton direction -H g
  double* part;  // scratch [5][kVecBlocks]
};

__device__ __forceinline__ double grid_sum(const double* part) {
  double s = 0.0;  // every block sums every partial in the same order
  for (int b = 0; b < (int)gridDim.x; ++b) s += part[b];
  return s;
}

// one-block grids (short vectors, two_loop_grid) are launched as plain
// kernels and need only the block barrier; the global memory they exchange
// through is then written and read by the same block
__device__ __forceinline__ void grid_barrier(cg::grid_group& grid) {
  if (gridDim.x == 1) __syncthreads();
  else grid.sync();
}

__device__ __forceinline__ void two_loop_body(const TwoLoopArgs& A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kVecThreads / 32];
  __shared__ double bc;
  const int64_t n = A.n;
  const int64_t stride = (int64_t)gridDim.x * kVecThreads;
  const int64_t i0 = (int64_t)blockIdx.x * kVecThreads + threadIdx.x;
  const int G = gridDim.x;
  double* rot = A.part;  // rows 0..2 rotate
  double* psy = A.part + 3 * kVecBlocks;
  double* pyy = A.part + 4 * kVecBlocks;
  double alpha[kMaxLbfgsPairs];
  int p = 0;

  double a = 0.0, b = 0.0, c = 0.0;
  {  // phase 0: q = g;  <s_0, g>, <s_0, y_0>, <y_0, y_0>  (index 0 = newest)
    const double* s0 = A.S + (int64_t)A.idx[0] * n;
    const double* y0 = A.Y + (int64_t)A.idx[0] * n;
    for (int64_t i = i0; i < n; i += stride) {
      const double v = A.g[i];
      A.q[i] = v;
      a = fma(s0[i], v, a);
      b = fma(s0[i], y0[i], b);
      c = fma(y0[i], y0[i], c);
    }
    a = block_sum256(a, sh);
    b = block_sum256(b, sh);
    c = block_sum256(c, sh);
    if (threadIdx.x == 0 && gridDim.x > 1) {
      rot[blockIdx.x] = a;
      psy[blockIdx.x] = b;
      pyy[blockIdx.x] = c;
    }
  }
  grid_barrier(grid);
  // one-block grids: thread 0 already holds the block sums (grid_sum of one
  // partial is 0 + it, the same bits), no global round trip per phase
  const bool one = G == 1;
  double prev_sum = a;  // thread 0: the block sum the next phase reads
  if (threadIdx.x == 0) bc = one ? (0.0 + b) / (0.0 + c) : grid_sum(psy) / grid_sum(pyy);
  __syncthreads();
  const double gamma = bc;  // <s,y>/<y,y> of the newest pair (H0 scaling)

  // first loop, newest -> oldest: alpha_k = rho_k <s_k, q>;  q -= alpha_k y_k
  for (int k = 0; k < A.count; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) bc = A.rho[k] * (one ? 0.0 + prev_sum : grid_sum(rot + (p % 3) * kVecBlocks));
    __syncthreads();
    alpha[k] = bc;
    const bool last = k + 1 == A.count;
    const double* y = A.Y + (int64_t)A.idx[k] * n;
    // next dot: <s_{k+1}, q>, or after scaling by gamma <y_oldest, q>
    const double* w = last ? A.Y + (int64_t)A.idx[A.count - 1] * n
                           : A.S + (int64_t)A.idx[k + 1] * n;
    double acc = 0.0;
    for (int64_t i = i0; i < n; i += stride) {
      double v = fma(-alpha[k], y[i], A.q[i]);
      if (last) v *= gamma;
      A.q[i] = v;
      acc = fma(w[i], v, acc);
    }
    acc = block_sum256(acc, sh);
    ++p;
    prev_sum = acc;
    if (threadIdx.x == 0 && !one) rot[(p % 3) * kVecBlocks + blockIdx.x] = acc;
    grid_barrier(grid);
  }
  // second loop, oldest -> newest: beta = rho_k <y_k, q>;  q += (alpha_k - beta) s_k
  for (int k = A.count - 1; k >= 0; --k) {
    __syncthreads();
    if (threadIdx.x == 0) bc = A.rho[k] * (one ? 0.0 + prev_sum : grid_sum(rot + (p % 3) * kVecBlocks));
    __syncthreads();
    const double coef = alpha[k] - bc;
    const double* s = A.S + (int64_t)A.idx[k] * n;
    if (k == 0) {
      for (int64_t i = i0; i < n; i += stride) A.q[i] = -fma(coef, s[i], A.q[i]);
      break;
    }
    const double* y2 = A.Y + (int64_t)A.idx[k - 1] * n;
    double acc = 0.0;
    for (int64_t i = i0; i < n; i += stride) {
      const double v = fma(coef, s[i], A.q[i]);
      A.q[i] = v;
      acc = fma(y2[i], v, acc);
    }
    acc = block_sum256(acc, sh);
    ++p;
    prev_sum = acc;
    if (threadIdx.x == 0 && !one) rot[(p % 3) * kVecBlocks + blockIdx.x] = acc;
    grid_barrier(grid);
  }
}

__global__ void __launch_bounds__(kVecThreads) two_loop_kernel(TwoLoopArgs A) {
  pdl_wait();  // (one-block grids are plain launches with programmatic serialization)
  two_loop_body(A);
}

// Device-driven variant for the graph-resident L-BFGS (ffm_min.cuh): the
// pair count, ring slots (newest first) and rho come from device memory
// (TwoLoopDevArgs, ffm_two_loop.cuh).  count = 0 gives the normalised
// antigradient of lbfgs_direction (ffmin/optimizers/lbfgs.py:53-58):
// d = (1 / |g|) (-g), or -g when |g| = 0.
__global__ void __launch_bounds__(kVecThreads) two_loop_dev_kernel(TwoLoopDevArgs D) {
  pdl_wait();
  FFM_MSTAMP(20);
  const int count = *D.count;
  if (count == 0) {
    const double gn = *D.gn;
    const double inv = 1.0 / gn;
    for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < D.n;
         i += (int64_t)gridDim.x * kVecThreads) {
      const double v = -D.g[i];
      D.q[i] = gn == 0.0 ? v : inv * v;
    }
    return;
  }
  TwoLoopArgs A;
  A.n = D.n;
  A.count = count;
  for (int k = 0; k < count; ++k) {
    A.idx[k] = D.idx[k];
    A.rho[k] = D.rho[k];
  }
  A.S = D.S;
  A.Y = D.Y;
  A.g = D.g;
  A.q = D.q;
  A.part = D.part;
  two_loop_body(A);
  FFM_MSTAMP(21);
}

size_t two_loop_scratch_doubles() { return (size_t)kMaxDots * kVecBlocks; }

// co-resident grid of the two-loop kernels: both variants use the same size
// so their reductions combine partials in the same order
static int two_loop_grid(int64_t n) {
  int dev = 0, sms = 0, per_sm = 0, per_sm2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, two_loop_kernel, kVecThreads, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, two_loop_dev_kernel, kVecThreads, 0);
  if (per_sm2 < per_sm) per_sm = per_sm2;
  int blocks = sms * (per_sm < 2 ? per_sm : 2);
  if (n <= kSmallVecN) return 1;  // one block: plain launch, block barriers only
  const int64_t need = (n + kVecThreads - 1) / kVecThreads;
  if (blocks > need) blocks = (int)need;
  if (blocks > kVecBlocks) blocks = kVecBlocks;
  // at most 64 blocks: the 2 m + 1 grid-wide phases are latency-bound (grid
  // barrier, every block summing every partial), not bandwidth-bound
  // (tools/lbfgs_launches.py, FP64 L-BFGS per iteration, blocks 118 -> 64:
  // 10k atoms 0.924 -> 0.905 ms, 30k 5.10 -> 5.01 ms; 100k unchanged)
  int cap = 64;
  if (const char* f = getenv("FFM_TWOLOOP_BLOCKS"))  // tuning aid
    if (atoi(f) > 0) cap = atoi(f);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return blocks;
}

cudaError_t launch_lbfgs_two_loop(int64_t n, int count, const int* idx, const double* rho,
                                  const double* S, const double* Y, const double* g,
                                  double* q, double* scratch, cudaStream_t st) {
  if (count < 1 || count > kMaxLbfgsPairs) return cudaErrorInvalidValue;
  TwoLoopArgs a;
  a.n = n;
  a.count = count;
  for (int k = 0; k < count; ++k) {
    a.idx[k] = idx[k];
    a.rho[k] = rho[k];
  }
  a.S = S;
  a.Y = Y;
  a.g = g;
  a.q = q;
  a.part = scratch;
  void* args[] = {&a};
  count_launch();
  const int grid = two_loop_grid(n);
  if (grid == 1) {
    launch_k(two_loop_kernel, 1, kVecThreads, 0, st, a);
    return cudaGetLastError();
  }
  return cudaLaunchCooperativeKernel((void*)two_loop_kernel, grid, kVecThreads, args, 0, st);
}

// Short vectors (one-block grids): the recursion with the ring pairs staged
// in shared memory and q in registers (ffm_two_loop.cuh; 500 atoms: 19 ->
// 9 us per direction, tools/lbfgs_timeline.py).
constexpr size_t kTwoLoopSmallSmem = 200 * 1024;

__global__ void __launch_bounds__(kVecThreads) two_loop_dev_small_kernel(TwoLoopDevArgs D) {
  pdl_wait();
  FFM_MSTAMP(20);
  extern __shared__ double ring[];
  double q[kTwoLoopSmallE];
  two_loop_small_body(D, ring, q);
  FFM_MSTAMP(21);
}

// opt the staged kernel in to its shared memory (outside any graph capture)
cudaError_t two_loop_small_prepare() {
  return cudaFuncSetAttribute(two_loop_dev_small_kernel,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)kTwoLoopSmallSmem);
}

cudaError_t launch_lbfgs_two_loop_dev(int64_t n, int m, const int* count, const int* idx,
                                      const double* rho, const double* gn, const double* S,
                                      const double* Y, const double* g, double* q,
                                      double* scratch, cudaStream_t st) {
  TwoLoopDevArgs d{n, count, idx, rho, gn, S, Y, g, q, scratch};
  void* args[] = {&d};
  count_launch();
  const size_t ring = (size_t)2 * m * n * sizeof(double);
  if (n <= (int64_t)kTwoLoopSmallE * kVecThreads && m <= kMaxLbfgsPairs &&
      ring <= kTwoLoopSmallSmem) {
    launch_k(two_loop_dev_small_kernel, 1, kVecThreads, ring, st, d);
    return cudaGetLastError();
  }
  const int grid = two_loop_grid(n);
  if (grid == 1) {
    launch_k(two_loop_dev_kernel, 1, kVecThreads, 0, st, d);
    return cudaGetLastError();
  }
  return cudaLaunchCooperativeKernel((void*)two_loop_dev_kernel, grid, kVecThreads, args, 0,
                                     st);
}

}  // namespace ffm


namespace ffm {

// ---- device-side completion of a sharded evaluation (ffm_system_set_comm)
// buf = [gradient (3n) | energies (5) | error (key + 1) x 4 | reporting x 4];
// a rank reporting an error adds (key + 1, 1), and all reporting ranks
// report the same key (parallel.py), so key = sum / count - 1 exactly.
__global__ void combine_encode_kernel(int64_t n3, int64_t natoms, const double* __restrict__ grad,
                                      const double* __restrict__ energies,
                                      const int64_t* __restrict__ status, double* __restrict__ buf) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (grad)
    for (int64_t i = i0; i < n3; i += (int64_t)gridDim.x * blockDim.x) buf[i] = grad[i];
  if (i0 == 0) {
    double* t = buf + n3;
    for (int q = 0; q < FFM_NTERMS; ++q) t[q] = energies[q];
    const int64_t keys[4] = {status[FFM_ST_NB_BAD_I] >= 0
                                 ? status[FFM_ST_NB_BAD_I] * natoms + status[FFM_ST_NB_BAD_J]
                                 : -1,
                             status[FFM_ST_BOND], status[FFM_ST_ANGLE], status[FFM_ST_DIHEDRAL]};
    for (int q = 0; q < 4; ++q) {
      t[FFM_NTERMS + q] = keys[q] >= 0 ? (double)(keys[q] + 1) : 0.0;
      t[FFM_NTERMS + 4 + q] = keys[q] >= 0 ? 1.0 : 0.0;
    }
  }
}

__global__ void combine_decode_kernel(int64_t n3, int64_t natoms, const double* __restrict__ buf,
                                      double* __restrict__ grad, double* __restrict__ energies,
                                      int64_t* __restrict__ status) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (grad)
    for (int64_t i = i0; i < n3; i += (int64_t)gridDim.x * blockDim.x) grad[i] = buf[i];
  if (i0 == 0) {
    const double* t = buf + n3;
    for (int q = 0; q < FFM_NTERMS; ++q) energies[q] = t[q];
    int64_t key[4];
    for (int q = 0; q < 4; ++q) {
      const double c = t[FFM_NTERMS + 4 + q];
      key[q] = c > 0.0 ? (int64_t)llround(t[FFM_NTERMS + q] / c) - 1 : -1;
    }
    status[FFM_ST_NB_BAD_I] = key[0] >= 0 ? key[0] / natoms : -1;
    status[FFM_ST_NB_BAD_J] = key[0] >= 0 ? key[0] % natoms : -1;
    status[FFM_ST_BOND] = key[1];
    status[FFM_ST_ANGLE] = key[2];
    status[FFM_ST_DIHEDRAL] = key[3];
  }
}

static int comb_blocks(int64_t n3) {
  int64_t b = (n3 + 255) / 256;
  if (b > 1184) b = 1184;
  return b < 1 ? 1 : (int)b;
}

cudaError_t launch_combine_encode(int64_t natoms, const double* grad, const double* energies,
                                  const int64_t* status, double* buf, cudaStream_t st) {
  count_launch();
  launch_k(combine_encode_kernel, grad ? comb_blocks(3 * natoms) : 1, 256, 0, st, 
      3 * natoms, natoms, grad, energies, status, buf);
  return cudaGetLastError();
}

cudaError_t launch_combine_decode(int64_t natoms, const double* buf, double* grad,
                                  double* energies, int64_t* status, cudaStream_t st) {
  count_launch();
  launch_k(combine_decode_kernel, grad ? comb_blocks(3 * natoms) : 1, 256, 0, st, 
      3 * natoms, natoms, buf, grad, energies, status);
  return cudaGetLastError();
}

}  // namespace ffm

#ifdef FFM_MIN_STAMPS
extern "C" int ffm_debug_min_clock_vec(void* clock_d) {
  return (int)cudaMemcpyToSymbol(ffm::g_mclk, &clock_d, sizeof(void*));
}
#endif
