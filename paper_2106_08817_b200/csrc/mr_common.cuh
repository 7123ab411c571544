// mr_common.cuh -- shared device helpers for the sm_100a geodesic-shooting kernels.
//
// Semantics follow the reference package morphreg (/root/reference/pkg/src/morphreg);
// every helper cites the line it restates.  See DESIGN.md for layouts and rooflines.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>

#include "../../include/morphreg_sm100.h"

namespace mr {

constexpr int kMaxR = MR_MAX_RADIUS;
constexpr int kThreads = 256;

// Gaussian taps passed BY VALUE as a kernel parameter: they live in the
// constant bank, so with a compile-time radius every tap is an FFMA
// constant-bank operand (no LDS/LDC per tap).
//   w[t] : forward taps, t = 0..2R (symmetrised on the host)    kernel.py:24-31
//   e[m] : cumulative sums W[m] = sum_{k<=m} w_k, m = 0..R, for the edge rows of
//          the exact transpose (kernel.py:48-68)
template <typename T>
struct Taps {
  T w[2 * kMaxR + 1];
  T e[kMaxR + 1];
};

struct Grid2 {
  int B, H, W;
  long long N;  // H*W
};

// One-time cudaFuncSetAttribute(MaxDynamicSharedMemorySize) per (kernel, device):
// the attribute is per device, so a process that drives several GPUs sets it on
// each; a failed call is not cached (the next launch retries).
constexpr int kMaxDevices = 64;
template <auto Kernel>
inline cudaError_t ensure_smem(size_t bytes) {
  static std::atomic<int> done[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool cached = dev >= 0 && dev < kMaxDevices;
  if (cached && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && cached) done[dev].store(1, std::memory_order_release);
  return e;
}

// ---- finite differences (fields.py:144-158) ------------------------------------

// np.gradient along one axis at index j of a length-n line, values at j-1, j, j+1
// supplied by the caller (fm = f[j-1], f0 = f[j], fp = f[j+1]; unused ones ignored).
template <typename T>
__device__ __forceinline__ T grad1(T fm, T f0, T fp, int j, int n) {
  if (j == 0) return fp - f0;
  if (j == n - 1) return f0 - fm;
  return (fp - fm) / T(2);
}

// Gather form of axis_diff_adjoint (fields.py:148-158) at index j:
// gm = g[j-1], gp = g[j+1], g0 = g[0], gl = g[n-1] (caller passes what exists).
// Term order follows the reference: edge updates first, then +0.5 g[j-1], -0.5 g[j+1].
template <typename T>
__device__ __forceinline__ T diff_adj1(T gm, T gp, T gfirst, T glast, int j, int n) {
  T out = T(0);
  if (j == 1) out += gfirst;
  if (j == 0) out -= gfirst;
  if (j == n - 1) out += glast;
  if (j == n - 2) out -= glast;
  if (j - 1 >= 1 && j - 1 <= n - 2) out += T(0.5) * gm;
  if (j + 1 >= 1 && j + 1 <= n - 2) out -= T(0.5) * gp;
  return out;
}

// ---- bilinear plan (fields.py:207-224) -------------------------------------------

template <typename T>
struct AxisPlan {
  int i0;
  T f;
  bool inside;
};

// Foot coordinate pos - dt*vel on an axis of n samples, clamped to [0, n-1],
// i0 = min(floor, n-2), strict inside mask (0 < y < n-1).
// float: integer base + fractional displacement (SURVEY §7 hard part 2) so the
// fraction keeps full fp32 precision far from the origin.
// double: the reference's absolute-coordinate formula, rounding-identical.
template <typename T>
__device__ __forceinline__ AxisPlan<T> plan_axis(int pos, T vel, T dt, int n);

template <>
__device__ __forceinline__ AxisPlan<float> plan_axis<float>(int pos, float vel, float dt, int n) {
  AxisPlan<float> p;
  const float d = -(dt * vel);
  // floor as a saturating int conversion; bounded so pos + fl cannot overflow
  // (huge displacements only occur after the guard fired)
  const int fl = min(max(__float2int_rd(d), -(1 << 24)), 1 << 24);
  const float fr = d - (float)fl;
  const int ii = pos + fl;
  if ((unsigned)(ii - 1) < (unsigned)(n - 2)) {  // 1 <= ii <= n - 2: the common case, no clamp
    p.i0 = ii;
    p.f = fr;
    p.inside = true;
    return p;
  }
  const bool lo = ii < 0 || (ii == 0 && fr == 0.0f);
  const bool hi = ii >= n - 1;
  p.i0 = lo ? 0 : (hi ? n - 2 : ii);
  p.f = lo ? 0.0f : (hi ? 1.0f : fr);
  p.inside = !(lo || hi);
  return p;
}

template <>
__device__ __forceinline__ AxisPlan<double> plan_axis<double>(int pos, double vel, double dt, int n) {
  AxisPlan<double> p;
  double y = (double)pos + (-(dt * vel));
  double yc = fmin(fmax(y, 0.0), (double)(n - 1));
  if (!(yc == yc)) yc = 0.0;  // NaN: guard reports it; keep indices in range
  int i0 = min((int)floor(yc), n - 2);
  p.i0 = i0;
  p.f = yc - (double)i0;
  p.inside = (y > 0.0) && (y < (double)(n - 1));
  return p;
}

// fields.py:235-240, same term order (bitwise-exact at nodes).
template <typename T>
__device__ __forceinline__ T bilerp(T a, T b, T c, T d, T fy, T fx) {
  T wy = T(1) - fy, wx = T(1) - fx;
  return wy * wx * a + fy * wx * b + wy * fx * c + fy * fx * d;
}

// ---- guard (integrator.py:113-118) -----------------------------------------------

template <typename T>
__device__ __forceinline__ unsigned guard_bits(T x, unsigned nonfinite_bit) {
  if (!isfinite(x)) return nonfinite_bit;
  if (fabs(x) > T(1e6)) return nonfinite_bit << 1;
  return 0u;
}

__device__ __forceinline__ void flush_flags(unsigned flags, int32_t* dst) {
  unsigned all = __reduce_or_sync(0xffffffffu, flags);
  if (all && (threadIdx.x & 31) == 0 && dst) atomicOr(reinterpret_cast<int*>(dst), (int)all);
}

// ---- deterministic (order-independent) accumulation ----------------------------
// With MR_OPT_DETERMINISTIC the adjoint's scatter targets accumulate in 64-bit
// two's-complement fixed point (red.global.add.u64): integer addition is
// associative, so the result does not depend on the order in which warps add and
// every run gives the same bits (the reference's replay promise,
// optimizer.py:5-7).  Per pair the contributions are scaled by 2^S with
// S = kFixBits - ilogb(max |input|): 2^-kFixBits relative resolution (finer than
// an fp32 ulp), and 2^(63 - kFixBits) of headroom for the fan-in of a cell.  A
// contribution outside the range (or non-finite) raises the overflow flag
// instead of wrapping silently.
constexpr int kFixBits = 48;

__device__ __forceinline__ double fix_factor(const unsigned long long* mbits, long long b) {
  const double m = __longlong_as_double((long long)mbits[b]);
  if (!(m > 0.0) || !isfinite(m)) return 1.0;
  return ldexp(1.0, kFixBits - ilogb(m));
}

__device__ __forceinline__ long long to_fix(double x, double f, unsigned& ovf) {
  const double y = x * f;
  if (!(fabs(y) < 7.2e16)) {  // 2^56: 2^7 contributions of that size still fit
    ovf = 1u;
    return 0;
  }
  return __double2ll_rn(y);
}

__device__ __forceinline__ void fix_add(unsigned long long* p, long long v) {
  atomicAdd(p, (unsigned long long)v);
}

// Warp-merged bilinear-transpose scatter (scatter4_merged) in fixed point: every
// contribution is converted before any merge, so merged and unmerged sums agree.
__device__ __forceinline__ void scatter4_merged_fix(unsigned long long* __restrict__ out,
                                                    long long cell, bool valid, long long W,
                                                    double f, double ca, double cb, double cc,
                                                    double cd, unsigned& ovf) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  long long qa = valid ? to_fix(ca, f, ovf) : 0, qb = valid ? to_fix(cb, f, ovf) : 0;
  const long long qc = valid ? to_fix(cc, f, ovf) : 0, qd = valid ? to_fix(cd, f, ovf) : 0;
  const long long key = valid ? cell : -4;
  const long long prev_key = __shfl_up_sync(full, key, 1);
  const long long next_key = __shfl_down_sync(full, key, 1);
  const long long pc = __shfl_up_sync(full, qc, 1);
  const long long pd = __shfl_up_sync(full, qd, 1);
  if (!valid) return;
  const bool merge_left = lane > 0 && prev_key >= 0 && prev_key + 1 == key;
  const bool merged_by_next = lane < 31 && next_key >= 0 && key + 1 == next_key;
  if (merge_left) {
    qa += pc;
    qb += pd;
  }
  fix_add(out + cell, qa);
  fix_add(out + cell + W, qb);
  if (!merged_by_next) {
    fix_add(out + cell + 1, qc);
    fix_add(out + cell + W + 1, qd);
  }
}

// Per-pair max |a|, |b| over [B][N] (grid: x blocks per pair, y = pair) as double
// bits: non-negative doubles order like their bit patterns, so atomicMax is exact.
template <typename T>
__global__ void k_absmax_pair(const T* __restrict__ a, const T* __restrict__ b, long long N,
                              unsigned long long* mbits) {
  const long long pb = blockIdx.y;
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    m = fmax(m, fabs((double)a[pb * N + i]));
    if (b) m = fmax(m, fabs((double)b[pb * N + i]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(mbits + pb, (unsigned long long)__double_as_longlong(m));
}

// Fixed-point cells -> T (q * 2^-S of the pair); resets the cells for the next step.
template <typename T>
__global__ void k_fix_to_float(unsigned long long* __restrict__ q, T* __restrict__ out,
                               long long N, const unsigned long long* mbits) {
  const long long pb = blockIdx.y;
  const double inv = 1.0 / fix_factor(mbits, pb);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    out[pb * N + i] = (T)((double)(long long)q[pb * N + i] * inv);
    q[pb * N + i] = 0ull;
  }
}

// ---- cp.async (LDGSTS) staging: many loads in flight, no register round trip ----

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem),
               "n"((int)sizeof(T)));
}

// zero-fills the destination when !valid (src-size 0; gmem must still be a valid address)
template <typename T>
__device__ __forceinline__ void cp_async_elem_zfill(T* smem, const T* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? (int)sizeof(T) : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem),
               "n"((int)sizeof(T)), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- packed FP32x2 FMA (FFMA2, sm_100a): two FMAs per issue slot ----------------
__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %4};\n"
      "mov.b64 rc, {%5, %6};\nfma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(w), "f"(c.x), "f"(c.y));
  return d;
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier ---------------------------------------

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 3D tiled TMA load of box (x, y, z) into smem; completion counted on `bar`.
// Out-of-bounds elements (negative or beyond the extents) are zero-filled.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// CTAs ahead of the running one whose inputs get an L2 prefetch (MR_PF_AHEAD, default: the
// number of SMs; 0 disables).  Used by k_vel_a: cfg2 12.17 -> 12.0 ms per grad on B200.
inline int prefetch_ahead() {
  static const int v = [] {
    if (const char* e = getenv("MR_PF_AHEAD")) return atoi(e);
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    return n_sm;
  }();
  return v;
}

}  // namespace mr

#define MR_RADIUS_LIST(X)                                                       \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14)   \
  X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26)      \
  X(27) X(28) X(29) X(30) X(31) X(32)
