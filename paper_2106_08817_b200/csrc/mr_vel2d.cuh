// mr_vel2d.cuh -- fp32 2D velocity v = -K*(z grad I) (integrator.py:93-94:
// gradient_arr fields.py:161-162 + smooth_vec_arr kernel.py:82-85) as two
// register-window FIR kernels around a transposed intermediate.
//
// The separable replicate-border Gaussian is the tensor product K0 (x) K1 of two
// clamped 1D convolutions, so the two passes commute exactly.  Both passes have the
// same shape: a thread owns ONE line along the filter axis and produces kFRB = 16
// consecutive outputs from a sliding window of 16 + 2R samples, the 32 lanes of a warp
// sitting on 32 neighbouring lines (conflict-free LDS.64, one load per 12 packed FFMA2
// at R = 24; the two vector components are the two halves of the FFMA2).  The first
// pass writes a TRANSPOSED intermediate hT [B][W][H][2], which makes the second pass
// (along x) the same kind of kernel with lanes along y.  Output tiles go through smem
// so that every store instruction of a warp writes 512 contiguous bytes.
//
//   k_vel_a   m = z grad I at the clamped row (replicate border) into smem, straight
//             from global memory (float4 loads, rows rolling in registers); y pass -> hT.
//   k_vel_b   TMA-stage (128 + 2R) x 32 of hT, clamp the x border in smem; x pass;
//             negate, velocity guard (integrator.py:113-118); v [B][2][H][W].
//
// Measured at 32 x 512^2, R = 24 (profiles/r02/fir2d.md): 54 + 38 us against 60 + 43 us
// for k_velocity2d_h + k_fir_axis0_f32.  The same structure for the velocity ADJOINT
// (transposed passes + epilogue) measured 47 + 71 us against 43 + 74 us for the
// k_fir_axis0_f32 / k_velocity_adj2d_h pair and was not kept: its epilogue moves
// 268 MB per launch and is memory-bound either way.
#pragma once

#include "mr_kernels2d.cuh"
#include "mr_tma.h"

namespace mr {

constexpr int kFX = 32;              // lines per tile (one per lane)
constexpr int kFRB = 16;             // outputs per thread along the filter axis
constexpr int kFY = kNW * kFRB;      // 128 outputs along the filter axis per CTA

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// window FIR: acc[o] = sum_t w[t - o] * src[t * P], t - o in [0, 2R]
template <int R, int P>
__device__ __forceinline__ void fir_window_p(const float2* __restrict__ src, const Taps<float>& tp,
                                             float2 (&acc)[kFRB]) {
#pragma unroll
  for (int o = 0; o < kFRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < kFRB + 2 * R; ++t) {
    const float2 xv = src[t * P];
#pragma unroll
    for (int o = 0; o < kFRB; ++o) {
      const int tap = t - o;
      if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(xv, tp.w[tap], acc[o]);
    }
  }
}
template <int R>
__device__ __forceinline__ void fir_window(const float2* __restrict__ src, const Taps<float>& tp,
                                           float2 (&acc)[kFRB]) {
  fir_window_p<R, kFX>(src, tp, acc);
}

// Coalesced stores of a CTA tile of hT through smem: every thread holds a run of 16
// float2 along the filter axis of line `col`; the runs go to sT[col][y] (pitch kTP:
// conflict-free STS.128 across lanes), then each warp instruction writes 512
// contiguous bytes of one hT line.
constexpr int kTP = kFY + 2;  // float2 pitch of sT: 1040 B = 16 (mod 128)
__device__ __forceinline__ void store_tile_hT(float2* sT, const float2 (&acc)[kFRB], int col, int warp,
                                              float2* __restrict__ hT, int b, int x0, int y0, int H,
                                              int W) {
  float2* d = sT + col * kTP + warp * kFRB;
#pragma unroll
  for (int o = 0; o < kFRB; o += 2)
    *reinterpret_cast<float4*>(d + o) = make_float4(acc[o].x, acc[o].y, acc[o + 1].x, acc[o + 1].y);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < (kFX * kFY / 2) / kThreads; ++i) {
    const int idx = threadIdx.x + i * kThreads;  // float4 index: column idx / 64, row pair idx % 64
    const int c = idx >> 6, yp = (idx & 63) * 2;
    const int gx = x0 + c, gy = y0 + yp;
    if (gx < W && gy < H)  // H even: a row pair is inside or outside as a whole
      *reinterpret_cast<float4*>(hT + ((long long)b * W + gx) * H + gy) =
          *reinterpret_cast<const float4*>(sT + c * kTP + yp);
  }
}

// ------------------------------------------------------------------------------
// k_vel_a: product + y pass.  grid (ceil(W/32), ceil(H/128), B)
// ------------------------------------------------------------------------------
template <int R>
struct VelASmem {
  static constexpr int RY = kFY + 2 * R;
  static constexpr size_t bytes = sizeof(float2) * (size_t)RY * kFX;
};

template <int R>
__global__ void __launch_bounds__(kThreads, 4)
    k_vel_a(const float* __restrict__ I, const float* __restrict__ z, float2* __restrict__ hT,
            int H, int W, Taps<float> tp, int pf_ahead) {
  constexpr int RY = VelASmem<R>::RY, RPW = (RY + kNW - 1) / kNW;
  if (pf_ahead > 0) {
    // L2 prefetch of the I / z rows of the CTA that will run `pf_ahead` CTAs later
    const long long lin = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z) + pf_ahead;
    const int px = (int)(lin % gridDim.x), py = (int)((lin / gridDim.x) % gridDim.y);
    const long long pb = lin / ((long long)gridDim.x * gridDim.y);
    if (pb < gridDim.z) {
      const int r = py * kFY - R + (int)threadIdx.x;  // one row per thread (RY <= 256)
      if ((int)threadIdx.x < RY && r >= 0 && r < H && px * kFX < W) {
        const long long off = (pb * H + r) * W + px * kFX;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(I + off));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(z + off));
      }
    }
  }
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* sM = reinterpret_cast<float2*>(smem_raw);
  const int x0 = blockIdx.x * kFX, y0 = blockIdx.y * kFY, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long base = (long long)b * H * W;
  const float* __restrict__ Ib = I + base;
  const float* __restrict__ zb = z + base;
  // m = z grad I for the sample rows inside the image: 8 threads per row (4 columns
  // each, float4 loads), 32 row slots of RPT consecutive rows (rows rolling in registers)
  {
    constexpr int RPT = (RY + 31) / 32;
    const int cg = threadIdx.x & 7, rs = threadIdx.x >> 3;
    const int jlo = rs * RPT, jhi = min(jlo + RPT, RY);
    const int ra = max(y0 - R + jlo, 0), rb = min(y0 - R + jhi, H);
    if (ra < rb) {
      const int xg = min(x0 + 4 * cg, W - 4);  // W % 4 == 0: a group is inside or outside as a whole
      const int xl = max(xg - 1, 0), xr = min(xg + 4, W - 1);
      const float c0 = xg == 0 ? 1.f : 0.5f, c3 = xg + 4 == W ? 1.f : 0.5f;
      float4 Iu = ldg4(Ib + max(ra - 1, 0) * W + xg), Ic = ldg4(Ib + ra * W + xg);
      float* dst = reinterpret_cast<float*>(sM + (ra - (y0 - R)) * kFX + 4 * cg);
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = ra + i;
        if (r >= rb) break;
        const float4 Id = ldg4(Ib + min(r + 1, H - 1) * W + xg);
        const float4 zz = ldg4(zb + r * W + xg);
        const float lf = __ldg(Ib + r * W + xl), rt = __ldg(Ib + r * W + xr);
        const float cgy = (r == 0 || r == H - 1) ? 1.f : 0.5f;  // one-sided rows: Iu / Id == Ic there
        const float g0x = (Id.x - Iu.x) * cgy, g0y = (Id.y - Iu.y) * cgy;
        const float g0z = (Id.z - Iu.z) * cgy, g0w = (Id.w - Iu.w) * cgy;
        const float g1x = (Ic.y - lf) * c0, g1y = (Ic.z - Ic.x) * 0.5f;
        const float g1z = (Ic.w - Ic.y) * 0.5f, g1w = (rt - Ic.z) * c3;
        *reinterpret_cast<float4*>(dst) = make_float4(zz.x * g0x, zz.x * g1x, zz.y * g0y, zz.y * g1y);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(zz.z * g0z, zz.z * g1z, zz.w * g0w, zz.w * g1w);
        dst += 2 * kFX;
        Iu = Ic;
        Ic = Id;
      }
    }
  }
  __syncthreads();
  // replicate border along y: sample rows outside [0, H) take row 0 / H - 1
  const bool top = y0 - R < 0, bot = y0 + kFY + R > H;
  if (top || bot) {
    const int j0 = R - y0, j1 = H - 1 - (y0 - R);  // sample index of rows 0 and H - 1
    for (int j = warp; j < RY; j += kNW) {
      const int r = y0 - R + j;
      if (r < 0) sM[j * kFX + lane] = sM[j0 * kFX + lane];
      else if (r >= H) sM[j * kFX + lane] = sM[j1 * kFX + lane];
    }
    __syncthreads();
  }
  float2 acc[kFRB];
  fir_window<R>(sM + warp * kFRB * kFX + lane, tp, acc);
  __syncthreads();  // every warp is done with sM: reuse it for the output tile
  store_tile_hT(sM, acc, lane, warp, hT, b, x0, y0, H, W);
}

// ------------------------------------------------------------------------------
// k_vel_b: x pass on hT + negate / guard / store.  grid (ceil(H/32), ceil(W/128), B)
// ------------------------------------------------------------------------------
constexpr int kVP = 132;  // pitch of the v output tile rows: 4 (mod 32) -> conflict-free STS.128
template <int R>
struct VelBSmem {
  static constexpr int RX = kFY + 2 * R;
  static constexpr size_t stage = sizeof(float2) * (size_t)RX * kFX;
  static constexpr size_t out = sizeof(float) * 2 * kFX * kVP;
  static constexpr size_t bytes = 128 + (stage > out ? stage : out);
};

template <int R>
__global__ void __launch_bounds__(kThreads, 4)
    k_vel_b(const __grid_constant__ CUtensorMap mH, float* __restrict__ v, int H, int W,
            int32_t* guard, int guard_stride, Taps<float> tp) {
  constexpr int RX = VelBSmem<R>::RX;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  float2* sH = reinterpret_cast<float2*>(smem_raw + 128);
  float* sT = reinterpret_cast<float*>(smem_raw + 128);  // [2][32][kVP], after the FIR
  const int y0 = blockIdx.x * kFX, x0 = blockIdx.y * kFY, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(float2) * RX * kFX));
    tma_load_3d(sH, &mH, 2 * y0, x0 - R, b, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // replicate border along x: sample columns outside [0, W) take column 0 / W - 1
  const bool lft = x0 - R < 0, rgt = x0 + kFY + R > W;
  if (lft || rgt) {
    const int j0 = R - x0, j1 = W - 1 - (x0 - R);
    for (int j = warp; j < RX; j += kNW) {
      const int x = x0 - R + j;
      if (x < 0) sH[j * kFX + lane] = sH[j0 * kFX + lane];
      else if (x >= W) sH[j * kFX + lane] = sH[j1 * kFX + lane];
    }
    __syncthreads();
  }
  float2 acc[kFRB];
  fir_window<R>(sH + warp * kFRB * kFX + lane, tp, acc);
  __syncthreads();  // every warp is done with the staged tile: reuse it for the output
  {
    float* d0 = sT + lane * kVP + warp * kFRB;
    float* d1 = d0 + kFX * kVP;
#pragma unroll
    for (int o = 0; o < kFRB; o += 4) {
      *reinterpret_cast<float4*>(d0 + o) = make_float4(-acc[o].x, -acc[o + 1].x, -acc[o + 2].x, -acc[o + 3].x);
      *reinterpret_cast<float4*>(d1 + o) = make_float4(-acc[o].y, -acc[o + 1].y, -acc[o + 2].y, -acc[o + 3].y);
    }
  }
  __syncthreads();
  // coalesced stores: a warp instruction writes one 512-byte row segment; velocity guard
  unsigned flags = 0;
  const long long N = (long long)H * W;
  const int gx = x0 + 4 * lane;
#pragma unroll
  for (int i = 0; i < 2 * kFX / kNW; ++i) {
    const int rc = warp + i * kNW;  // component * 32 + row
    const int c = rc >> 5, r = rc & 31, gy = y0 + r;
    if (gy < H && gx < W) {  // W % 4 == 0: a chunk is inside or outside as a whole
      const float4 o4 = *reinterpret_cast<const float4*>(sT + rc * kVP + 4 * lane);
      if (!(fabsf(o4.x) <= 1e6f && fabsf(o4.y) <= 1e6f && fabsf(o4.z) <= 1e6f && fabsf(o4.w) <= 1e6f))
        flags |= guard_bits(o4.x, MR_GUARD_VELOCITY_NONFINITE) | guard_bits(o4.y, MR_GUARD_VELOCITY_NONFINITE) |
                 guard_bits(o4.z, MR_GUARD_VELOCITY_NONFINITE) | guard_bits(o4.w, MR_GUARD_VELOCITY_NONFINITE);
      *reinterpret_cast<float4*>(v + ((long long)b * 2 + c) * N + (long long)gy * W + gx) = o4;
    }
  }
  if (guard) flush_flags(flags, guard + (long long)b * guard_stride);
}

// ------------------------------------------------------------------------------
// launchers; return 1 (not applicable) when the layout is not TMA-describable /
// 16-byte aligned, so the caller keeps its other paths
// ------------------------------------------------------------------------------
inline bool fast2d_ok(const Grid2& g, const void* p0, const void* p1, const void* p2,
                      const void* p3 = nullptr, const void* p4 = nullptr) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return (g.W & 3) == 0 && (g.H & 1) == 0 && g.N < (1LL << 30) && g.B <= 65535 && al(p0) && al(p1) && al(p2) &&
         al(p3) && al(p4);
}

template <int R>
int launch_vel2d_fast(const Grid2& g, const Taps<float>& tp, const float* I, const float* z,
                      float* v, int32_t* guard, int guard_stride, float* ws, cudaStream_t s) {
  using A = VelASmem<R>;
  using Bs = VelBSmem<R>;
  if (!ws || !fast2d_ok(g, I, z, v, ws)) return 1;
  CUtensorMap mH;  // hT [B][W][H][2] as floats: (2H, W, B)
  if (!make_map3<float>(&mH, ws, 2 * g.H, g.W, g.B, 2 * kFX, Bs::RX)) return 1;
  cudaError_t e = ensure_smem<k_vel_a<R>>(A::bytes);
  if (e != cudaSuccess) return cuda_status(e);
  e = ensure_smem<k_vel_b<R>>(Bs::bytes);
  if (e != cudaSuccess) return cuda_status(e);
  float2* hT = reinterpret_cast<float2*>(ws);
  const int pf = prefetch_ahead();
  k_vel_a<R><<<dim3((g.W + kFX - 1) / kFX, (g.H + kFY - 1) / kFY, g.B), kThreads, A::bytes, s>>>(
      I, z, hT, g.H, g.W, tp, pf);
  int rc = cuda_status(cudaGetLastError());
  if (rc) return rc;
  k_vel_b<R><<<dim3((g.H + kFX - 1) / kFX, (g.W + kFY - 1) / kFY, g.B), kThreads, Bs::bytes, s>>>(
      mH, v, g.H, g.W, guard, guard_stride, tp);
  return cuda_status(cudaGetLastError());
}

}  // namespace mr
