// mr_fir_impl.cuh -- radius-dispatching launchers of the FIR-engine kernels.
#pragma once

#include "mr_launch.cuh"
#include "mr_tma.h"

#include <cstdlib>

namespace mr {

inline dim3 fir_grid(int W, int H, int B, int tx, int ty) {
  return dim3((unsigned)((W + tx - 1) / tx), (unsigned)((H + ty - 1) / ty), (unsigned)B);
}


// Register-window fp32 velocity around a transposed intermediate (mr_vel2d.cuh,
// instantiated in mr_fir_vel2_g*.cu); returns 1 when not applicable.
template <int R>
int launch_vel2d_fast(const Grid2& g, const Taps<float>& tp, const float* I, const float* z,
                      float* v, int32_t* guard, int guard_stride, float* ws, cudaStream_t s);

// Split velocity (fp32, scratch given): product +
// axis-1 FIR per tile (k_velocity2d_h) into a.vtmp, then the axis-0 FIR over whole
// columns with negate + velocity guard (k_fir_axis0_f32<R, false, 1>).
template <typename T, int R>
int velocity_split_r(const Grid2& g, const Taps<T>& tp, VelArgs<T> a, cudaStream_t s) {
  if constexpr (sizeof(T) != 4) {
    return 1;
  } else {
    using S = FirSmem<T, R, 2>;
    using V = VelHSmem<R>;
    if (!a.vtmp) return 1;
    static const bool classic = getenv("MR_VEL_CLASSIC") != nullptr;  // A/B switch
    if (!classic) {
      int rc = launch_vel2d_fast<R>(g, tp, a.I, a.z, a.v, a.guard, a.guard_stride, a.vtmp, s);
      if (rc != 1) return rc;
    }
    CUtensorMap mI, mZ;
    if (!make_map3<T>(&mI, a.I, g.W, g.H, g.B, V::PXI, S::OY + 2) ||
        !make_map3<T>(&mZ, a.z, g.W, g.H, g.B, V::PXZ, S::OY))
      return 1;
    const cudaError_t attr = ensure_smem<k_velocity2d_h<R>>(V::bytes);
    if (attr != cudaSuccess) return cuda_status(attr);
    k_velocity2d_h<R><<<fir_grid(g.W, g.H, g.B, S::OX, S::OY), kThreads, V::bytes, s>>>(
        a, tp, mI, mZ, a.vtmp);
    int rc = cuda_status(cudaGetLastError());
    if (rc) return rc;
    return launch_fir_axis0<T>(R, tp, a.vtmp, a.v, 2 * g.B, g.H, (long long)g.W, false, 1,
                               a.guard, a.guard_stride, 2, s);
  }
}

template <typename T, int R>
int velocity_r(const Grid2& g, const Taps<T>& tp, VelArgs<T> a, cudaStream_t s) {
  {
    int rc = velocity_split_r<T, R>(g, tp, a, s);
    if (rc != 1) return rc;
  }
  using S = FirSmem<T, R, 2>;
  using V = VelSmem<T, R>;
  constexpr size_t bytes = V::bytes;
  const cudaError_t attr = ensure_smem<k_velocity2d<T, R>>(bytes);
  if (attr != cudaSuccess) return cuda_status(attr);
  CUtensorMap mI, mZ;
  a.use_tma = make_map3<T>(&mI, a.I, g.W, g.H, g.B, V::PXI, S::RY + 2) &&
              make_map3<T>(&mZ, a.z, g.W, g.H, g.B, S::PX, S::RY);
  k_velocity2d<T, R>
      <<<fir_grid(g.W, g.H, g.B, S::OX, S::OY), kThreads, bytes, s>>>(a, tp, mI, mZ);
  return cuda_status(cudaGetLastError());
}

template <typename T, int R, bool TR>
int smooth_r(const Grid2& g, const Taps<T>& tp, const SmoothArgs<T>& a, cudaStream_t s) {
  using S = FirSmem<T, R, 1>;
  if constexpr (sizeof(T) == 4) {  // TMA-staged region when the layout is describable
    CUtensorMap m;
    if (g.N < (1LL << 31) && make_map3<T>(&m, a.a, g.W, g.H, g.B, S::PX, S::RY)) {
      constexpr size_t bytes = SmoothTmaSmem<R>::bytes;
      const cudaError_t attr = ensure_smem<k_smooth2d_tma<R, TR>>(bytes);
      if (attr != cudaSuccess) return cuda_status(attr);
      k_smooth2d_tma<R, TR><<<fir_grid(g.W, g.H, g.B, S::OX, S::OY), kThreads, bytes, s>>>(a, tp, m);
      return cuda_status(cudaGetLastError());
    }
  }
  const cudaError_t attr = ensure_smem<k_smooth2d<T, R, TR>>(S::bytes);
  if (attr != cudaSuccess) return cuda_status(attr);
  k_smooth2d<T, R, TR><<<fir_grid(g.W, g.H, g.B, S::OX, S::OY), kThreads, S::bytes, s>>>(a, tp);
  return cuda_status(cudaGetLastError());
}


// Split velocity adjoint (fp32, scratch given): whole-column axis-0 transposed FIR
// into a.vtmp (k_fir_axis0_f32), then the axis-1 pass + epilogue
// (k_velocity_adj2d_h).  FIR work 2*(2R+1) FFMA per output plus the 1-px owner
// overlap, against (2 + 2R/OX)*(2R+1) in the single-kernel tile engine.
template <typename T, int R, bool REG>
int veladj_split_r(const Grid2& g, const Taps<T>& tp, VelAdjArgs<T> a, cudaStream_t s) {
  if constexpr (sizeof(T) != 4) {
    return 1;
  } else {
    if (!a.vtmp) return 1;
    using S = FirSmem<T, R, 2>;
    using V = VelAdjHSmem<R>;
    VelAdjMaps m;
    const long long B2 = 2LL * g.B;
    const bool ok = make_map3<T>(&m.vbar, a.vtmp, g.W, g.H, B2, S::PX, S::OY) &&
                    make_map3<T>(&m.I, a.I, g.W, g.H, g.B, V::OXP, S::OY) &&
                    make_map3<T>(&m.z, a.z, g.W, g.H, g.B, V::OXP, S::OY);
    if (!ok) return 1;
    int rc = launch_fir_axis0<T>(R, tp, a.vbar, a.vtmp, (int)B2, g.H, (long long)g.W, true, 0,
                                 nullptr, 0, 2, s);
    if (rc) return rc;
    constexpr size_t bytes = V::bytes;
    const cudaError_t attr = ensure_smem<k_velocity_adj2d_h<R, REG>>(bytes);
    if (attr != cudaSuccess) return cuda_status(attr);
    a.vbar = a.vtmp;
    k_velocity_adj2d_h<R, REG>
        <<<fir_grid(g.W, g.H, g.B, S::OX - 2, S::OY - 2), kThreads, bytes, s>>>(a, tp, m);
    return cuda_status(cudaGetLastError());
  }
}

template <typename T, int R, bool REG>
int veladj_r(const Grid2& g, const Taps<T>& tp, VelAdjArgs<T> a, cudaStream_t s) {
  {
    int rc = veladj_split_r<T, R, REG>(g, tp, a, s);
    if (rc != 1) return rc;
  }
  using S = FirSmem<T, R, 2>;
  using V = VelAdjSmem<T, R>;
  constexpr size_t bytes = VelAdjSmem<T, R>::bytes;
  const cudaError_t attr = ensure_smem<k_velocity_adj2d<T, R, REG>>(bytes);
  if (attr != cudaSuccess) return cuda_status(attr);
  VelAdjMaps m;
  const long long B2 = 2LL * g.B;
  a.use_tma = make_map3<T>(&m.vbar, a.vbar, g.W, g.H, B2, S::PX, S::RY) &&
              make_map3<T>(&m.I, a.I, g.W, g.H, g.B, V::OXP, S::OY) &&
              make_map3<T>(&m.z, a.z, g.W, g.H, g.B, V::OXP, S::OY) &&
              (REG ? make_map3<T>(&m.op2, a.v0, g.W, g.H, B2, V::OXP, S::OY)
                   : make_map3<T>(&m.op2, a.ib, g.W, g.H, g.B, V::OXP, S::OY)) &&
              make_map3<T>(&m.zb, a.zb, g.W, g.H, g.B, V::OXP, S::OY);
  k_velocity_adj2d<T, R, REG>
      <<<fir_grid(g.W, g.H, g.B, S::OX - 2, S::OY - 2), kThreads, bytes, s>>>(a, tp, m);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_velocity2d(const Grid2& g, int R, const Taps<T>& tp, const T* I, const T* z, T* v,
                      int32_t* guard, int guard_stride, cudaStream_t s, T* vtmp) {
  VelArgs<T> a{I, z, v, guard, guard_stride, 0, g, vtmp};
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

// One launcher per translation unit (mr_fir_<launcher>_<precision>.cu) so the
// heavily unrolled radius instantiations compile in parallel.
#define MR_INSTANTIATE_VELOCITY(T)                                                              \
  namespace mr {                                                                                \
  template int launch_velocity2d<T>(const Grid2&, int, const Taps<T>&, const T*, const T*, T*,  \
                                    int32_t*, int, cudaStream_t, T*);                           \
  }
#define MR_INSTANTIATE_SMOOTH(T)                                                                \
  namespace mr {                                                                                \
  template int launch_smooth2d<T>(const Grid2&, int, const Taps<T>&, const T*, T*, bool,        \
                                  cudaStream_t);                                                \
  }
#define MR_INSTANTIATE_VELADJ(T)                                                                \
  namespace mr {                                                                                \
  template int launch_velocity_adj2d<T>(const Grid2&, int, const Taps<T>&,                      \
                                        const VelAdjArgs<T>&, bool, cudaStream_t);              \
  }
// Radius groups: the per-radius kernels of the two heavy launchers (velocity,
// velocity adjoint) are instantiated in mr_fir_<launcher>_<prec>_g<k>.cu (radius
// r with r % 4 == k) so they compile in parallel; the dispatching translation unit
// sees them as extern templates.
#define MR_RADIUS_GROUP0(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32)
#define MR_RADIUS_GROUP1(X) X(1) X(5) X(9) X(13) X(17) X(21) X(25) X(29)
#define MR_RADIUS_GROUP2(X) X(2) X(6) X(10) X(14) X(18) X(22) X(26) X(30)
#define MR_RADIUS_GROUP3(X) X(3) X(7) X(11) X(15) X(19) X(23) X(27) X(31)
#define MR_VELOCITY_R_DECL(PFX, T, RR) \
  PFX template int velocity_r<T, RR>(const Grid2&, const Taps<T>&, VelArgs<T>, cudaStream_t);
#define MR_VELADJ_R_DECL(PFX, T, RR)                                                           \
  PFX template int veladj_r<T, RR, true>(const Grid2&, const Taps<T>&, VelAdjArgs<T>,           \
                                         cudaStream_t);                                         \
  PFX template int veladj_r<T, RR, false>(const Grid2&, const Taps<T>&, VelAdjArgs<T>,          \
                                          cudaStream_t);
#define MR_VEL2_DECL(PFX, RR)                                                                  \
  PFX template int launch_vel2d_fast<RR>(const Grid2&, const Taps<float>&, const float*,         \
                                         const float*, float*, int32_t*, int, float*,            \
                                         cudaStream_t);
#define MR_VEL2_EXTERN(RR) MR_VEL2_DECL(extern, RR)
#define MR_VEL2_INST(RR) MR_VEL2_DECL(, RR)
#define MR_VEL_EXTERN_F32(RR) MR_VELOCITY_R_DECL(extern, float, RR)
#define MR_VEL_EXTERN_F64(RR) MR_VELOCITY_R_DECL(extern, double, RR)
#define MR_VEL_INST_F32(RR) MR_VELOCITY_R_DECL(, float, RR)
#define MR_VEL_INST_F64(RR) MR_VELOCITY_R_DECL(, double, RR)
#define MR_VADJ_EXTERN_F32(RR) MR_VELADJ_R_DECL(extern, float, RR)
#define MR_VADJ_EXTERN_F64(RR) MR_VELADJ_R_DECL(extern, double, RR)
#define MR_VADJ_INST_F32(RR) MR_VELADJ_R_DECL(, float, RR)
#define MR_VADJ_INST_F64(RR) MR_VELADJ_R_DECL(, double, RR)
