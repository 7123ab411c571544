// mr_vel2d.cuh -- 2D fp32 velocity v = -K*(z grad I), column pass first
// (integrator.py:93-94: gradient_arr fields.py:161-162 + smooth_vec_arr
// kernel.py:82-85).
//
// The separable replicate-border Gaussian is the tensor product K0 (x) K1 of the
// two clamped 1D convolutions, so the two passes commute exactly; running the
// axis-0 (column) pass first lets the momentum product be formed straight into
// the column-pass tile, where every product sample is read by 2R+1 outputs of
// one thread's register window:
//
//   k_vel_col   TMA-stage I (+1 halo) and z for a 32-column x (TY + 2R)-row
//               region; m = z grad I at the clamped row (replicate border along
//               axis 0, kernel.py:43-44) into smem as (m0, m1) float2; each thread
//               filters one column over 16 rows (register window, packed FFMA2 with
//               the two components as the pair) -> h, interleaved [B][H][W][2].
//   k_vel_row   stage 32 rows x (64 + 2R) columns of h with 8-byte cp.async from
//               the CLAMPED column (replicate border along axis 1), odd float2
//               pitch (lanes <-> rows, conflict-free); each thread filters 8
//               outputs of its row; negate, velocity guard (integrator.py:113-118),
//               store v [B][2][H][W].
//
// Shared-memory traffic per pixel ~80 B (col) / ~70 B (row), below the FFMA2
// issue time of the 2(2R+1) FMAs per pixel: both kernels are FMA-bound.
#pragma once

#include "mr_kernels2d.cuh"
#include "mr_tma.h"

namespace mr {

constexpr int kVcTX = 32, kVcRB = 16, kVcTY = kNW * kVcRB;  // 32 x 128 output tile
constexpr int kVcIX = 40;                                     // I box: columns x0-4 .. x0+35

template <int R>
struct VelColSmem {
  static constexpr int RY = kVcTY + 2 * R;  // m rows
  static constexpr int IY = RY + 2;         // I rows
  static constexpr size_t offI = 128;
  static constexpr size_t offZ = offI + sizeof(float) * (size_t)IY * kVcIX;
  static constexpr size_t offM = (offZ + sizeof(float) * (size_t)RY * kVcTX + 127) / 128 * 128;
  static constexpr size_t bytes = offM + sizeof(float2) * (size_t)RY * kVcTX;
};

template <int R>
__global__ void __launch_bounds__(kThreads)
    k_vel_col(const __grid_constant__ CUtensorMap mI, const __grid_constant__ CUtensorMap mZ,
              float2* __restrict__ h, int H, int W, Taps<float> tp) {
  using S = VelColSmem<R>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  float* sI = reinterpret_cast<float*>(smem_raw + S::offI);
  float* sZ = reinterpret_cast<float*>(smem_raw + S::offZ);
  float2* sM = reinterpret_cast<float2*>(smem_raw + S::offM);
  const int x0 = blockIdx.x * kVcTX, y0 = blockIdx.y * kVcTY, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(float) * (S::IY * kVcIX + S::RY * kVcTX)));
    tma_load_3d(sI, &mI, x0 - 4, y0 - R - 1, b, bar);
    tma_load_3d(sZ, &mZ, x0, y0 - R, b, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // m = z grad I at row clamp(gy) (the column pass clamps its input rows)
  const int gx = x0 + lane;
  const bool colok = gx < W;
  const bool xin = gx > 0 && gx < W - 1;
  for (int j = warp; j < S::RY; j += kNW) {
    const int cy = min(max(y0 - R + j, 0), H - 1);
    const float* pI = sI + (cy - (y0 - R - 1)) * kVcIX + lane + 4;
    const float c = pI[0];
    float g0, g1;
    if (cy > 0 && cy < H - 1) g0 = (pI[kVcIX] - pI[-kVcIX]) * 0.5f;
    else g0 = cy == 0 ? pI[kVcIX] - c : c - pI[-kVcIX];
    if (xin) g1 = (pI[1] - pI[-1]) * 0.5f;
    else g1 = gx == 0 ? pI[1] - c : c - pI[-1];
    const float zz = sZ[(cy - (y0 - R)) * kVcTX + lane];
    sM[j * kVcTX + lane] = colok ? make_float2(zz * g0, zz * g1) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const float2* src = sM + warp * kVcRB * kVcTX + lane;
  float2 acc[kVcRB];
#pragma unroll
  for (int o = 0; o < kVcRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < kVcRB + 2 * R; ++t) {
    const float2 xv = src[t * kVcTX];
#pragma unroll
    for (int o = 0; o < kVcRB; ++o) {
      const int tap = t - o;
      if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(xv, (float)tp.w[tap], acc[o]);
    }
  }
  if (!colok) return;
  const int gy0 = y0 + warp * kVcRB;
  float2* dst = h + ((long long)b * H + gy0) * W + gx;
#pragma unroll
  for (int o = 0; o < kVcRB; ++o)
    if (gy0 + o < H) dst[(long long)o * W] = acc[o];
}

constexpr int kVrTX = 64, kVrTY = 32, kVrRB = 8;  // row pass: 64 x 32 tile, 8 outputs / thread

template <int R>
struct VelRowSmem {
  static constexpr int RX = kVrTX + 2 * R;
  static constexpr int P = RX | 1;  // odd float2 pitch: lanes <-> rows conflict-free
  static constexpr size_t bytes = sizeof(float2) * (size_t)kVrTY * P;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

template <int R>
__global__ void __launch_bounds__(kThreads)
    k_vel_row(const float2* __restrict__ h, float* __restrict__ v, int H, int W,
              int32_t* guard, int guard_stride, Taps<float> tp) {
  using S = VelRowSmem<R>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* sH = reinterpret_cast<float2*>(smem_raw);
  const int x0 = blockIdx.x * kVrTX, y0 = blockIdx.y * kVrTY, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // stage rows y0..y0+31, columns clamp(x0-R .. x0+64+R-1) (replicate border)
  for (int e = tid; e < kVrTY * S::RX; e += kThreads) {
    const int r = e / S::RX, i = e - r * S::RX;
    const int gy = min(y0 + r, H - 1);
    const int gx = min(max(x0 - R + i, 0), W - 1);
    cp_async8(sH + r * S::P + i, h + ((long long)b * H + gy) * W + gx);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // lanes <-> rows; warp w filters output columns [8w, 8w + 8)
  const float2* src = sH + lane * S::P + warp * kVrRB;
  float2 acc[kVrRB];
#pragma unroll
  for (int o = 0; o < kVrRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < kVrRB + 2 * R; ++t) {
    const float2 xv = src[t];
#pragma unroll
    for (int o = 0; o < kVrRB; ++o) {
      const int tap = t - o;
      if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(xv, (float)tp.w[tap], acc[o]);
    }
  }
  const int gy = y0 + lane, gx0 = x0 + warp * kVrRB;
  unsigned flags = 0;
  if (gy < H && gx0 < W) {
    const long long N = (long long)H * W;
    float* d0 = v + (long long)b * 2 * N + (long long)gy * W + gx0;
    float* d1 = d0 + N;
    float o0[kVrRB], o1[kVrRB];
#pragma unroll
    for (int o = 0; o < kVrRB; ++o) {
      o0[o] = -acc[o].x;
      o1[o] = -acc[o].y;
      if (!(fabsf(o0[o]) <= 1e6f && fabsf(o1[o]) <= 1e6f) && gx0 + o < W) {
        flags |= guard_bits(o0[o], MR_GUARD_VELOCITY_NONFINITE);
        flags |= guard_bits(o1[o], MR_GUARD_VELOCITY_NONFINITE);
      }
    }
    if (gx0 + kVrRB <= W) {
#pragma unroll
      for (int o = 0; o < kVrRB; o += 4) {
        *reinterpret_cast<float4*>(d0 + o) = make_float4(o0[o], o0[o + 1], o0[o + 2], o0[o + 3]);
        *reinterpret_cast<float4*>(d1 + o) = make_float4(o1[o], o1[o + 1], o1[o + 2], o1[o + 3]);
      }
    } else {
#pragma unroll
      for (int o = 0; o < kVrRB; ++o)
        if (gx0 + o < W) {
          d0[o] = o0[o];
          d1[o] = o1[o];
        }
    }
  }
  if (guard) flush_flags(flags, guard + (long long)b * guard_stride);
}

// Launch both passes; returns 1 (not applicable) when the layout is not
// TMA-describable / 16-byte aligned, so the caller keeps its other paths.
template <int R>
int launch_vel2d_colfirst(const Grid2& g, const Taps<float>& tp, const float* I, const float* z,
                          float* v, int32_t* guard, int guard_stride, float* ws, cudaStream_t s) {
  using C = VelColSmem<R>;
  using Rw = VelRowSmem<R>;
  if (!ws || (g.W & 3) || (reinterpret_cast<uintptr_t>(v) & 15) ||
      (reinterpret_cast<uintptr_t>(ws) & 15) || C::IY > 256)
    return 1;
  CUtensorMap mI, mZ;
  if (!make_map3<float>(&mI, I, g.W, g.H, g.B, kVcIX, C::IY) ||
      !make_map3<float>(&mZ, z, g.W, g.H, g.B, kVcTX, C::RY))
    return 1;
  cudaError_t e = ensure_smem<k_vel_col<R>>(C::bytes);
  if (e != cudaSuccess) return cuda_status(e);
  e = ensure_smem<k_vel_row<R>>(Rw::bytes);
  if (e != cudaSuccess) return cuda_status(e);
  float2* h = reinterpret_cast<float2*>(ws);
  k_vel_col<R><<<dim3((g.W + kVcTX - 1) / kVcTX, (g.H + kVcTY - 1) / kVcTY, g.B), kThreads,
                 C::bytes, s>>>(mI, mZ, h, g.H, g.W, tp);
  int rc = cuda_status(cudaGetLastError());
  if (rc) return rc;
  k_vel_row<R><<<dim3((g.W + kVrTX - 1) / kVrTX, (g.H + kVrTY - 1) / kVrTY, g.B), kThreads,
                 Rw::bytes, s>>>(h, v, g.H, g.W, guard, guard_stride, tp);
  return cuda_status(cudaGetLastError());
}

}  // namespace mr
