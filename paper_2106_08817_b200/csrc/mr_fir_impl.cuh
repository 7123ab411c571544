// mr_fir_impl.cuh -- radius-dispatching launchers of the FIR-engine kernels.
#pragma once

#include "mr_launch.cuh"

namespace mr {

inline dim3 fir_grid(int W, int H, int B, int tx, int ty) {
  return dim3((unsigned)((W + tx - 1) / tx), (unsigned)((H + ty - 1) / ty), (unsigned)B);
}

template <typename T, int R>
int velocity_r(const Grid2& g, const Taps<T>& tp, const VelArgs<T>& a, cudaStream_t s) {
  using S = FirSmem<T, R, 2>;
  constexpr size_t bytes = VelSmem<T, R>::bytes;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_velocity2d<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (attr != cudaSuccess) return MR_ECUDA;
  k_velocity2d<T, R><<<fir_grid(g.W, g.H, g.B, S::OX, S::OY), kThreads, bytes, s>>>(a, tp);
  return cuda_status(cudaGetLastError());
}

template <typename T, int R, bool TR>
int smooth_r(const Grid2& g, const Taps<T>& tp, const SmoothArgs<T>& a, cudaStream_t s) {
  using S = FirSmem<T, R, 1>;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_smooth2d<T, R, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
  if (attr != cudaSuccess) return MR_ECUDA;
  k_smooth2d<T, R, TR><<<fir_grid(g.W, g.H, g.B, S::OX, S::OY), kThreads, S::bytes, s>>>(a, tp);
  return cuda_status(cudaGetLastError());
}

template <typename T, int R, bool REG>
int veladj_r(const Grid2& g, const Taps<T>& tp, const VelAdjArgs<T>& a, cudaStream_t s) {
  using S = FirSmem<T, R, 2>;
  constexpr size_t bytes = VelAdjSmem<T, R>::bytes;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_velocity_adj2d<T, R, REG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (attr != cudaSuccess) return MR_ECUDA;
  k_velocity_adj2d<T, R, REG>
      <<<fir_grid(g.W, g.H, g.B, S::OX - 2, S::OY - 2), kThreads, bytes, s>>>(a, tp);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_velocity2d(const Grid2& g, int R, const Taps<T>& tp, const T* I, const T* z, T* v,
                      int32_t* guard, int guard_stride, cudaStream_t s) {
  VelArgs<T> a{I, z, v, guard, guard_stride, g};
  switch (R) {
#define MR_CASE(RR) \
  case RR: return velocity_r<T, RR>(g, tp, a, s);
    MR_RADIUS_LIST(MR_CASE)
#undef MR_CASE
    default: return MR_EINVAL;
  }
}

template <typename T>
int launch_smooth2d(const Grid2& g, int R, const Taps<T>& tp, const T* src, T* out, bool transpose,
                    cudaStream_t s) {
  SmoothArgs<T> a{src, out, g};
  switch (R) {
#define MR_CASE(RR)                                                          \
  case RR:                                                                   \
    return transpose ? smooth_r<T, RR, true>(g, tp, a, s) : smooth_r<T, RR, false>(g, tp, a, s);
    MR_RADIUS_LIST(MR_CASE)
#undef MR_CASE
    default: return MR_EINVAL;
  }
}

template <typename T>
int launch_velocity_adj2d(const Grid2& g, int R, const Taps<T>& tp, const VelAdjArgs<T>& a,
                          bool reg, cudaStream_t s) {
  switch (R) {
#define MR_CASE(RR)                                                          \
  case RR:                                                                   \
    return reg ? veladj_r<T, RR, true>(g, tp, a, s) : veladj_r<T, RR, false>(g, tp, a, s);
    MR_RADIUS_LIST(MR_CASE)
#undef MR_CASE
    default: return MR_EINVAL;
  }
}

}  // namespace mr

#define MR_INSTANTIATE_FIR(T)                                                                   \
  namespace mr {                                                                                \
  template int launch_velocity2d<T>(const Grid2&, int, const Taps<T>&, const T*, const T*, T*,  \
                                    int32_t*, int, cudaStream_t);                               \
  template int launch_smooth2d<T>(const Grid2&, int, const Taps<T>&, const T*, T*, bool,        \
                                  cudaStream_t);                                                \
  template int launch_velocity_adj2d<T>(const Grid2&, int, const Taps<T>&,                      \
                                        const VelAdjArgs<T>&, bool, cudaStream_t);              \
  }
