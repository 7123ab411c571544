// mr_launch.cuh -- host-side launchers (templated on precision) shared by the
// translation units.  The FIR-engine launchers (radius dispatch 1..MR_MAX_RADIUS)
// are defined in mr_fir_impl.cuh and explicitly instantiated per precision in
// mr_fir_<launcher>_<precision>.cu so the heavy unrolled kernels compile in parallel.
#pragma once

#include "mr_kernels2d.cuh"
#include "mr_kernels3d.cuh"

#include <climits>
#include <cstdlib>

namespace mr {

// last CUDA error seen by a launcher on this thread (reported by mr_last_error)
inline thread_local cudaError_t g_last_cuda = cudaSuccess;

inline int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return MR_OK;
  g_last_cuda = e;
  return MR_ECUDA;
}

template <typename T>
int launch_velocity2d(const Grid2& g, int R, const Taps<T>& tp, const T* I, const T* z, T* v,
                      int32_t* guard, int guard_stride, cudaStream_t s, T* vtmp = nullptr);
template <typename T>
int launch_smooth2d(const Grid2& g, int R, const Taps<T>& tp, const T* a, T* out, bool transpose,
                    cudaStream_t s);
template <typename T>
int launch_velocity_adj2d(const Grid2& g, int R, const Taps<T>& tp, const VelAdjArgs<T>& args,
                          bool reg, cudaStream_t s);

// 1D FIR along axis 0 of V volumes [V][D][HW] (3D velocity / its adjoint);
// epi = 1: negate + velocity guard (guard word of pair vol/ncomp).
template <typename T>
int launch_fir_axis0(int R, const Taps<T>& tp, const T* in, T* out, int V, int D, long long HW,
                     bool transpose, int epi, int32_t* guard, int guard_stride, int ncomp,
                     cudaStream_t s);

}  // namespace mr
