// mr_fir_axis0.cuh -- 1D FIR along axis 0 of a stack of volumes [V][D][HW]: the
// whole-column pass of the split 2D velocity / velocity adjoint and the axis-0
// pass of the 3D smoothing.  Only mr_fir_axis0_<precision>.cu includes this
// header; everything else calls launch_fir_axis0 (mr_launch.cuh).
#pragma once

#include "mr_launch.cuh"
#include "mr_tma.h"

namespace mr {

// ------------------------------------------------------------------------------
// 1D FIR along axis 0 of a stack of volumes [V][D][HW] (V = B*3):
//  forward: replicate borders (conv1d_replicate, kernel.py:36-45)
//  transpose: exact transpose (kernel.py:48-68): zero padding + edge rows.
// Tile: 64 consecutive HW elements x OD outputs along D, halo R, register
// blocking kRB outputs per thread.  EPI = 1: out = -acc with the velocity
// guard (per pair b = volume / 3).
// ------------------------------------------------------------------------------
constexpr int kAx0X = 64, kAx0D = 32;

template <typename T, int R>
struct Ax0Smem {
  static constexpr int RD = kAx0D + 2 * R;
  static constexpr size_t bytes = sizeof(T) * (size_t)RD * kAx0X;
};

template <typename T, int R, bool TRANSPOSE, int EPI>
__global__ void __launch_bounds__(kThreads)
    k_fir_axis0(const T* __restrict__ in, T* out, int D, long long HW, int32_t* guard,
                int guard_stride, int ncomp, Taps<T> tp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* rg = reinterpret_cast<T*>(smem_raw);
  constexpr int RD = kAx0D + 2 * R;
  const long long x0 = (long long)blockIdx.x * kAx0X;
  const int d_org = blockIdx.y * kAx0D;
  const int vol = blockIdx.z;
  const T* __restrict__ src = in + (long long)vol * D * HW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < RD; j += kNW) {
    int gd = d_org - R + j;
    bool rin = true;
    if (TRANSPOSE) {
      rin = gd >= 0 && gd < D;
      gd = rin ? gd : 0;
    } else {
      gd = min(max(gd, 0), D - 1);
    }
    const T* row = src + (long long)gd * HW;
    for (int i = lane; i < kAx0X; i += 32) {
      const long long gx = x0 + i;
      const bool in_ = rin && gx < HW;
      cp_async_elem_zfill(rg + j * kAx0X + i, row + (in_ ? gx : 0), in_);
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  constexpr int NB = kAx0D / kRB;
  unsigned flags = 0;
  for (int cb = warp; cb < NB; cb += kNW)
    for (int i = lane; i < kAx0X; i += 32) {
      const T* s = rg + cb * kRB * kAx0X + i;
      T acc[kRB];
#pragma unroll
      for (int o = 0; o < kRB; ++o) acc[o] = T(0);
#pragma unroll
      for (int t = 0; t < kRB + 2 * R; ++t) {
        const T xv = s[t * kAx0X];
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
          const int tap = t - o;
          if (tap >= 0 && tap <= 2 * R) acc[o] = fma(tp.w[tap], xv, acc[o]);
        }
      }
      const int gd0 = d_org + cb * kRB;
      if (TRANSPOSE) {
        if (gd0 <= 0 && gd0 + kRB > 0) {
          const int o = -gd0;
          T a = T(0);
#pragma unroll
          for (int dd = 0; dd <= R; ++dd) a = fma(tp.e[R - dd], s[(o + R + dd) * kAx0X], a);
#pragma unroll
          for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = a;
        }
        if (gd0 <= D - 1 && gd0 + kRB > D - 1) {
          const int o = D - 1 - gd0;
          T a = T(0);
#pragma unroll
          for (int dd = -R; dd <= 0; ++dd) a = fma(tp.e[R + dd], s[(o + R + dd) * kAx0X], a);
#pragma unroll
          for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = a;
        }
      }
      const long long gx = x0 + i;
      if (gx >= HW) continue;
      T* dst = out + (long long)vol * D * HW + gx;
#pragma unroll
      for (int o = 0; o < kRB; ++o) {
        const int gd = gd0 + o;
        if (gd < D) {
          T val = acc[o];
          if (EPI == 1) {
            val = -val;
            flags |= guard_bits(val, MR_GUARD_VELOCITY_NONFINITE);
          }
          dst[(long long)gd * HW] = val;
        }
      }
    }
  if (EPI == 1 && guard && flags)
    atomicOr(reinterpret_cast<int*>(guard + (long long)(vol / ncomp) * guard_stride), (int)flags);
}

// 16-byte cp.async with zero fill (src-size 0 when !valid; gmem must stay a valid address)
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

// ------------------------------------------------------------------------------
// fp32 axis-0 FIR (same contract as k_fir_axis0): tile of 64 columns x kA0D outputs
// along D plus the R halo, staged with 16-B cp.async (row index clamped for the
// forward, zero rows outside [0, D) for the transpose); one warp per block of
// kA0RB output rows, lanes <-> column pairs, packed FFMA2.  FIR work is exactly
// 2R+1 FFMA per output (the halo costs loads, not FLOPs).
// ------------------------------------------------------------------------------
constexpr int kA0RB = 16;  // outputs per thread along axis 0 (register block)
constexpr int kA0X = 64, kA0D = kNW * kA0RB;

template <int R>
struct Ax0F32Smem {
  static constexpr int RD = kA0D + 2 * R;
  static constexpr size_t bytes = sizeof(float) * (size_t)RD * kA0X;
};

template <int R, bool TRANSPOSE, int EPI>
__global__ void __launch_bounds__(kThreads)
    k_fir_axis0_f32(const float* __restrict__ in, float* out, int D, long long HW,
                    int32_t* guard, int guard_stride, int ncomp, Taps<float> tp) {
  static_assert(kA0D == kNW * kA0RB && kA0X == 64, "one row block per warp, a column pair per lane");
  extern __shared__ __align__(128) float rgf[];  // [RD][kA0X]
  constexpr int RD = Ax0F32Smem<R>::RD;
  const long long x0 = (long long)blockIdx.x * kA0X;
  const int d_org = blockIdx.y * kA0D;
  const int vol = blockIdx.z;
  const float* __restrict__ src = in + (long long)vol * D * HW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = ((HW & 3) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
  {
    // 16 lanes per row (one 16-B chunk each), 16 rows per pass of the CTA
    const int c4 = threadIdx.x & 15;
    const long long gx = x0 + 4 * c4;
    const bool full = vec && gx + 3 < HW;
    float* dst = rgf + 4 * c4;
    for (int j = threadIdx.x >> 4; j < RD; j += kThreads / 16) {
      int gd = d_org - R + j;
      bool rin = true;
      if (TRANSPOSE) {
        rin = gd >= 0 && gd < D;
        gd = rin ? gd : 0;
      } else {
        gd = min(max(gd, 0), D - 1);
      }
      const float* row = src + (long long)gd * HW + gx;
      if (full) {
        cp_async16_zfill(dst + j * kA0X, row, rin);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = rin && gx + e < HW;
          cp_async_elem_zfill(dst + j * kA0X + e, ok ? row + e : src, ok);
        }
      }
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  const int i = 2 * lane;
  const float2* s2 = reinterpret_cast<const float2*>(rgf + warp * kA0RB * kA0X + i);
  float2 acc[kA0RB];
#pragma unroll
  for (int o = 0; o < kA0RB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < kA0RB + 2 * R; ++t) {
    const float2 xv = s2[t * (kA0X / 2)];
#pragma unroll
    for (int o = 0; o < kA0RB; ++o) {
      const int tap = t - o;
      if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(xv, (float)tp.w[tap], acc[o]);
    }
  }
  const int gd0 = d_org + warp * kA0RB;
  const long long gx = x0 + i;
  unsigned flags = 0;
  if (gx < HW) {
    float* p = out + (long long)vol * D * HW + (long long)gd0 * HW + gx;
    const bool pair = gx + 1 < HW && ((HW & 1) == 0) && ((reinterpret_cast<uintptr_t>(out) & 7) == 0);
#pragma unroll
    for (int o = 0; o < kA0RB; ++o, p += HW) {
      const int gd = gd0 + o;
      if (gd < D) {
        float2 val = acc[o];
        if (EPI == 1) {
          val = make_float2(-val.x, -val.y);
          if (!(fabsf(val.x) <= 1e6f && fabsf(val.y) <= 1e6f)) {
            flags |= guard_bits(val.x, MR_GUARD_VELOCITY_NONFINITE);
            if (gx + 1 < HW) flags |= guard_bits(val.y, MR_GUARD_VELOCITY_NONFINITE);
          }
        }
        if (pair) {
          *reinterpret_cast<float2*>(p) = val;
        } else {
          p[0] = val.x;
          if (gx + 1 < HW) p[1] = val.y;
        }
      }
    }
  }
  if (EPI == 1 && guard && flags)
    atomicOr(reinterpret_cast<int*>(guard + (long long)(vol / ncomp) * guard_stride), (int)flags);
  if (TRANSPOSE && gx < HW) {
    // edge rows 0 and n-1 of the transpose (cumulative-weight taps)
    // overwrite what the interior formula stored there, after the accumulators
    // are dead (keeps the main loop at the forward kernel's register count)
    float* p = out + (long long)vol * D * HW + gx;
    const bool pair = gx + 1 < HW && ((HW & 1) == 0) && ((reinterpret_cast<uintptr_t>(out) & 7) == 0);
    auto put = [&](int gd, float2 val) {
      float* r = p + (long long)gd * HW;
      if (pair) {
        *reinterpret_cast<float2*>(r) = val;
      } else {
        r[0] = val.x;
        if (gx + 1 < HW) r[1] = val.y;
      }
    };
    if (gd0 <= 0 && gd0 + kA0RB > 0) {  // output row 0: sum_{d=0..R} W[R-d] g[d]
      const int o = -gd0;
      float2 a2 = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int dd = 0; dd <= R; ++dd) a2 = ffma2(s2[(o + R + dd) * (kA0X / 2)], (float)tp.e[R - dd], a2);
      put(0, a2);
    }
    if (gd0 <= D - 1 && gd0 + kA0RB > D - 1) {  // row n-1: sum_{d=-R..0} W[R+d] g[n-1+d]
      const int o = D - 1 - gd0;
      float2 a2 = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int dd = -R; dd <= 0; ++dd) a2 = ffma2(s2[(o + R + dd) * (kA0X / 2)], (float)tp.e[R + dd], a2);
      put(D - 1, a2);
    }
  }
}

template <typename T, int R, bool TR, int EPI>
int fir_axis0_r(const Taps<T>& tp, const T* in, T* out, int V, int D, long long HW,
                int32_t* guard, int guard_stride, int ncomp, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {  // fp32: FFMA2 engine, 64-column x kA0D-row tiles
    constexpr size_t bytes = Ax0F32Smem<R>::bytes;
    const cudaError_t attr = ensure_smem<k_fir_axis0_f32<R, TR, EPI>>(bytes);
    if (attr != cudaSuccess) return cuda_status(attr);
    dim3 grid((unsigned)((HW + kA0X - 1) / kA0X), (unsigned)((D + kA0D - 1) / kA0D), (unsigned)V);
    k_fir_axis0_f32<R, TR, EPI><<<grid, kThreads, bytes, s>>>(in, out, D, HW, guard, guard_stride,
                                                               ncomp, tp);
    return cuda_status(cudaGetLastError());
  } else {
  constexpr size_t bytes = Ax0Smem<T, R>::bytes;
  const cudaError_t attr = ensure_smem<k_fir_axis0<T, R, TR, EPI>>(bytes);
  if (attr != cudaSuccess) return cuda_status(attr);
  dim3 grid((unsigned)((HW + kAx0X - 1) / kAx0X), (unsigned)((D + kAx0D - 1) / kAx0D),
            (unsigned)V);
  k_fir_axis0<T, R, TR, EPI><<<grid, kThreads, bytes, s>>>(in, out, D, HW, guard, guard_stride,
                                                            ncomp, tp);
  return cuda_status(cudaGetLastError());
  }
}

template <typename T>
int launch_fir_axis0(int R, const Taps<T>& tp, const T* in, T* out, int V, int D, long long HW,
                     bool transpose, int epi, int32_t* guard, int guard_stride, int ncomp,
                     cudaStream_t s) {
  switch (R) {
#define MR_CASE(RR)                                                                          \
  case RR:                                                                                   \
    if (transpose)                                                                           \
      return fir_axis0_r<T, RR, true, 0>(tp, in, out, V, D, HW, guard, guard_stride, ncomp, s);     \
    if (epi) return fir_axis0_r<T, RR, false, 1>(tp, in, out, V, D, HW, guard, guard_stride, ncomp, s); \
    return fir_axis0_r<T, RR, false, 0>(tp, in, out, V, D, HW, guard, guard_stride, ncomp, s);
    MR_RADIUS_LIST(MR_CASE)
#undef MR_CASE
    default: return MR_EINVAL;
  }
}

}  // namespace mr

#define MR_INSTANTIATE_AXIS0(T)                                                                 \
  namespace mr {                                                                                \
  template int launch_fir_axis0<T>(int, const Taps<T>&, const T*, T*, int, int, long long, bool, \
                                   int, int32_t*, int, int, cudaStream_t);                      \
  }

// Radius groups (r % 4 == k) of the per-radius kernels, instantiated in
// mr_fir_axis0_<prec>_g<k>.cu so the unrolled FIR kernels compile in parallel;
// the dispatching translation unit sees them as extern templates.
#define MR_AX0_R_DECL(PFX, T, RR)                                                                \
  PFX template int fir_axis0_r<T, RR, true, 0>(const Taps<T>&, const T*, T*, int, int, long long, \
                                               int32_t*, int, int, cudaStream_t);                \
  PFX template int fir_axis0_r<T, RR, false, 1>(const Taps<T>&, const T*, T*, int, int,          \
                                                long long, int32_t*, int, int, cudaStream_t);    \
  PFX template int fir_axis0_r<T, RR, false, 0>(const Taps<T>&, const T*, T*, int, int,          \
                                                long long, int32_t*, int, int, cudaStream_t);
#define MR_AX0_EXTERN_F32(RR) MR_AX0_R_DECL(extern, float, RR)
#define MR_AX0_EXTERN_F64(RR) MR_AX0_R_DECL(extern, double, RR)
#define MR_AX0_INST_F32(RR) MR_AX0_R_DECL(, float, RR)
#define MR_AX0_INST_F64(RR) MR_AX0_R_DECL(, double, RR)
#define MR_AX0_GROUP0(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32)
#define MR_AX0_GROUP1(X) X(1) X(5) X(9) X(13) X(17) X(21) X(25) X(29)
#define MR_AX0_GROUP2(X) X(2) X(6) X(10) X(14) X(18) X(22) X(26) X(30)
#define MR_AX0_GROUP3(X) X(3) X(7) X(11) X(15) X(19) X(23) X(27) X(31)
