// ffm_common.cuh -- shared definitions for the B200 force-field kernels.
//
// Packed-arithmetic layer: the O(N^2) pair kernel is issue-slot bound on the
// FP32 pipe, so its inner loop is written on Blackwell's packed f32x2
// instructions (FADD2/FMUL2/FFMA2: two FP32 lanes per issue slot, same
// 128 FMA/clk/SM pipe rate, see profiles/r01_pipes_microbench.txt).  The
// same kernel templates instantiate on double with a plain two-lane struct,
// so FP32 and FP64 modes share one tiling/reduction structure.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffm {

// Programmatic dependent launch (PDL, launch_k in ffm_kernels.h): a kernel
// may be scheduled while its stream predecessor is still finishing; every
// kernel calls pdl_wait() before touching memory (griddepcontrol.wait: the
// predecessor grid has completed and its writes are visible -- a no-op for
// kernels launched without PDL), then lets its own dependents launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ffmin/constants.py:10, 13, 16
constexpr double kCoulomb = 1389.38757;
constexpr double kRmin = 1e-12;
constexpr double kDegenerateEps = 1e-12;

// The i-side LJ records (ilj) carry a factor 6: the pair kernel then forms
// 6A/r^6 and 6B directly, so the gradient needs no separate scaling multiply
// (12 A/r^12 - 6 B/r^6 = (6A/r^6 + 6(A/r^6 - B))/r^6), and the vdW energy
// sum is divided by 6 once per super-unit.  (FP64 took it in round 2 with the
// 4-warp CTAs: 100k energy+gradient 11.43 -> 11.25 ms; round 1's 8-warp FP64
// kernel had measured the explicit multiply faster.)
#ifndef FFM_F64SCALE
#define FFM_F64SCALE 1  // FP64 i-side LJ scaled by 6 as well (w = fma(pw, r^-6, ecp))
#endif
template <typename T> struct LjIScale { static constexpr double value = 6.0; };
template <> struct LjIScale<double> { static constexpr double value = FFM_F64SCALE ? 6.0 : 1.0; };

// Pair-kernel tiling:
//   a warp tile is 128 i-atoms (4 per lane, two packed pairs) x 32 j-atoms;
//   a CTA is 8 warps and owns one super-unit of S x S atoms.
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kIB = 128;  // i-sub-block
constexpr int kJB = 32;   // j-block

// ------------------------------------------------------------ packed math
template <typename T> struct Pk;

template <> struct Pk<float> {
  using V = uint64_t;  // two fp32 lanes in one 64-bit register pair
  static __device__ __forceinline__ V make(float a, float b) {
    V r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
  }
  static __device__ __forceinline__ V bc(float a) { return make(a, a); }
  static __device__ __forceinline__ float lo(V v) {
    return __uint_as_float((unsigned)(v & 0xffffffffull));
  }
  static __device__ __forceinline__ float hi(V v) { return __uint_as_float((unsigned)(v >> 32)); }
  static __device__ __forceinline__ V add(V a, V b) {
    V d;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
  }
  static __device__ __forceinline__ V mul(V a, V b) {
    V d;
    asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
  }
  static __device__ __forceinline__ V fma(V a, V b, V c) {
    V d;
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
  }
  // two FFMA2 sharing the multiplicands, emitted back to back so the
  // second can take g and d from the operand reuse cache (register-file
  // read bandwidth, not the FMA pipe, limits 3-source FFMA2)
  static __device__ __forceinline__ void fma_pair(V g, V d, V& a, V& b) {
    asm("fma.rn.ftz.f32x2 %0, %2, %3, %0;\n\t"
        "fma.rn.ftz.f32x2 %1, %2, %3, %1;"
        : "+l"(a), "+l"(b) : "l"(g), "l"(d));
  }
  // MUFU.RSQ on each lane (no packed form exists)
  static __device__ __forceinline__ V rsqrt(V v) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    float ra, rb;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(a));
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(b));
    return make(ra, rb);
  }
  static __device__ __forceinline__ V rsqrt_e(V v) { return rsqrt(v); }
  // r^-2: MUFU.RCP per lane (the XU pipe has slack; the FMA pipe is the bound)
  static __device__ __forceinline__ V rcp_or_sq(V r2, V /*ri*/) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r2));
    float ra, rb;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(a));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(b));
    return make(ra, rb);
  }
  static __device__ __forceinline__ V zero() { return 0ull; }
};

// Tuning aid (variant builds with -DFFM_MIN_STAMPS only): a timeline of
// globaltimer stamps from the minimiser's controller kernels and the fused
// small-system evaluation, [0] = count, then (tag, ns) pairs
// (tools/lbfgs_timeline.py); each translation unit has its own pointer.
#ifdef FFM_MIN_STAMPS
static __device__ unsigned long long* g_mclk = nullptr;
__device__ __forceinline__ void mstamp(int tag, bool last_block = false) {
  if (g_mclk && threadIdx.x == 0 && blockIdx.x == (last_block ? gridDim.x - 1 : 0)) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    const unsigned long long k = atomicAdd(g_mclk, 1ull);
    if (k < 200000) {
      g_mclk[1 + 2 * k] = (unsigned long long)tag;
      g_mclk[2 + 2 * k] = t;
    }
  }
}
#define FFM_MSTAMP(t) ::ffm::mstamp(t)
#define FFM_MSTAMP_LAST(t) ::ffm::mstamp(t, true)
#else
#define FFM_MSTAMP_LAST(t) \
  do {                     \
  } while (0)
#define FFM_MSTAMP(t) \
  do {                \
  } while (0)
#endif

#ifndef FFM_F64HALF
#define FFM_F64HALF 1  // FP64 energy-only rsqrt Newton step: y / 2 by an exponent decrement
#endif

struct D2 {
  double x, y;
};

template <> struct Pk<double> {
  // explicitly rounded operations: no contraction under any -fmad setting,
  // so every translation unit evaluates a pair to the same bits
  using V = D2;
  static __device__ __forceinline__ V make(double a, double b) { return {a, b}; }
  static __device__ __forceinline__ V bc(double a) { return {a, a}; }
  static __device__ __forceinline__ double lo(V v) { return v.x; }
  static __device__ __forceinline__ double hi(V v) { return v.y; }
  static __device__ __forceinline__ V add(V a, V b) {
    return {__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)};
  }
  static __device__ __forceinline__ V mul(V a, V b) {
    return {__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)};
  }
  static __device__ __forceinline__ V fma(V a, V b, V c) {
    return {__fma_rn(a.x, b.x, c.x), __fma_rn(a.y, b.y, c.y)};
  }
  // MUFU.RSQ64H seed + one Newton step: relative error ~1e-14.  HALFI: the
  // step's y / 2 is taken on the integer pipe (exponent - 1: the same bits
  // as the FP64 multiply for every normal y; y is 1/r of a finite r > 0, or
  // inf / NaN for r = 0, where the step yields NaN either way), leaving three
  // FP64 operations (energy-only tiles: 100k FP64 5.64 -> 5.51 ms; the
  // register-bound gradient tile measured 0.4% slower with it)
  template <bool HALFI>
  static __device__ __forceinline__ double rsqrt1(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = __dmul_rn(x, y);
    const double e = __fma_rn(-h, y, 1.0);
    const double yh = HALFI && FFM_F64HALF
                          ? __hiloint2double(__double2hiint(y) - (1 << 20), __double2loint(y))
                          : __dmul_rn(0.5, y);
    return __fma_rn(yh, e, y);
  }
  static __device__ __forceinline__ V rsqrt(V v) { return {rsqrt1<false>(v.x), rsqrt1<false>(v.y)}; }
  static __device__ __forceinline__ V rsqrt_e(V v) { return {rsqrt1<true>(v.x), rsqrt1<true>(v.y)}; }
  // FP64 keeps r^-2 = (r^-1)^2 (no full-precision MUFU reciprocal)
  static __device__ __forceinline__ V rcp_or_sq(V /*r2*/, V ri) { return mul(ri, ri); }
  static __device__ __forceinline__ void fma_pair(V g, V d, V& a, V& b) {
    a = fma(g, d, a);
    b = fma(g, d, b);
  }
  static __device__ __forceinline__ V zero() { return {0.0, 0.0}; }
};

// Atom records in HBM (padded to the super-unit size):
//   pos[a] = (x, y, z, q~)   with q~ = q * sqrt(C) so q~_i q~_j = C q_i q_j
//   lj[a]  = (a_i, b_i)      with a_i = 2 sqrt(eps_i) sigma_i^6,
//                                 b_i = 2 sqrt(eps_i) sigma_i^3
// so the geometric-mean LJ of ffmin/kernels.py:340-344 factorises:
//   4 eps_ij (sig_ij/r)^12 = a_i a_j / r^12,  4 eps_ij (sig_ij/r)^6 = b_i b_j / r^6.
template <typename T> struct Vec4T;
template <> struct Vec4T<float> { using type = float4; };
template <> struct Vec4T<double> { using type = double4; };
template <typename T> struct Vec2T;
template <> struct Vec2T<float> { using type = float2; };
template <> struct Vec2T<double> { using type = double2; };

// Coordinates of an evaluation: x itself, or a line-search trial point
// x + h r formed on the fly with the same fma as the trial buffer's
// (ffm_small.cu P0), so every reader sees the same doubles.
struct CoordSrc {
  const double* x;
  const double* r;  // null: plain coordinates
  double h;
  __device__ __forceinline__ double at(int64_t q) const { return r ? fma(h, r[q], x[q]) : x[q]; }
};

// Status words written by the kernels (device int64[kStatusWords]).
enum StatusSlot : int {
  kStNbBadI = 0,      // first coincident nonbonded pair (i, j), -1 clean
  kStNbBadJ = 1,
  kStBond = 2,        // first degenerate bond term, -1 clean
  kStAngle = 3,
  kStDihedral = 4,
  kStNbSuspect = 5,   // set when the pair sweep saw a possible coincidence
  kStNbKey = 6,       // scratch: min (i * n + j) over coincident pairs
  kStCount = 7,       // scratch, 0 between evaluations: the finder's finished-block counter
  kStWords = 8
};

}  // namespace ffm
