// mr_kernels2d.cuh -- 2D sm_100a kernels of the semi-Lagrangian shooting path.
//
// K1 k_velocity2d      v = -K*(z grad I)                 integrator.py:93-94
// K2 k_sl_step2d       fused bilinear transport step       integrator.py:101-110,193-205
// K3 k_sl_adjoint2d    transport adjoint (scatter + gathers) objective.py:118-147
// K4 k_velocity_adj2d  -K^T, z-bar / i-bar stencil adjoint  objective.py:157-169
// K5 k_cost_terms2d    SSD, <m0,K m0>, |z0|^2 (fp64 accum)  objective.py:64-88
// plus k_smooth2d (smooth_arr / smooth_adjoint_arr, kernel.py:71-79).
//
// The separable Gaussian runs in a shared-memory tile engine (fir2d_tile): the
// tile plus an R-pixel halo is staged in smem once, then a vertical and a
// horizontal pass run with register blocking (RB outputs per thread, sliding
// over RB+2R inputs) and the radius R as a template parameter so every tap is
// an FFMA with a constant-bank weight.  Layout: SoA [B][c][H][W].
#pragma once

#include "mr_common.cuh"

namespace mr {

constexpr int kRB = 8;  // outputs per thread in each FIR pass
constexpr int kNW = kThreads / 32;

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// shift of a box starting at column x0 relative to the aligned column below it
__device__ __forceinline__ int align_shift(int x0, int A) { return ((x0 % A) + A) % A; }

// Output tile (OX x OY) of the FIR engine per precision.
template <typename T> struct Tile2;
template <> struct Tile2<float> { static constexpr int OX = 64, OY = 32; };
template <> struct Tile2<double> { static constexpr int OX = 32, OY = 32; };

template <typename T, int R, int C>
struct FirSmem {
  static constexpr int OX = Tile2<T>::OX, OY = Tile2<T>::OY;
  static constexpr int RX = OX + 2 * R;  // region width
  static constexpr int RY = OY + 2 * R;
  // TMA boxes must start at a 16-byte aligned column: a box starts at the
  // aligned column at or below the wanted one and the smem view is shifted by
  // the remainder (0 .. A-1 elements), so the pitch leaves room for it.
  static constexpr int A = 16 / (int)sizeof(T);
  static constexpr int PX = round_up(RX + A - 1, A);  // region pitch = TMA box width
  static constexpr int VP = RX + 1;      // pass-1 output pitch (odd: conflict-free rows)
  static constexpr int OP = OX + 1;      // result pitch
  static constexpr int CS = round_up(RY * PX, 32);  // component stride (128-B aligned TMA dst)
  static constexpr int region = round_up(C * CS + A, 32);
  static constexpr int vt = round_up(C * OY * VP, 32);
  static constexpr size_t bytes = sizeof(T) * (size_t)(region + vt);
  static_assert(C * OY * OP <= region, "result must fit in the region buffer");
};

// Pass 2 of the FIR engine: along axis 1 over the pass-1 output vt [C][OY][VP]
// (odd pitch, lanes <-> rows) into res [C][OY][OP]; transpose edge columns at
// image columns 0 and n-1.
template <typename T, int R, int C, bool TRANSPOSE>
__device__ __forceinline__ void fir2d_pass2(const T* vt, T* res, const Taps<T>& tp, int x_org,
                                            int W) {
  using S = FirSmem<T, R, C>;
  constexpr int OX = S::OX, OY = S::OY, VP = S::VP, OP = S::OP;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NB2 = OX / kRB;
  static_assert(OY == 32, "pass 2 maps lanes to the 32 rows of a tile");
  if constexpr (sizeof(T) == 4) {
    // fp32: rows (j, j+16) packed per thread (FFMA2); half-warps take two column blocks
    static_assert(NB2 % 2 == 0, "column blocks come in pairs");
    for (int cb = warp; cb < C * NB2 / 2; cb += kNW) {
      const int j = lane & 15;
      // half-warps take column blocks 16 columns apart: with the odd pitch the two
      // halves' 16 rows then fall in complementary bank sets (conflict-free)
      static_assert(NB2 == 8, "column-block pairing assumes 8 blocks");
      const int pb = cb % (NB2 / 2);
      const int ib = (pb & 1) + 4 * (pb >> 1) + 2 * (lane >> 4);
      const int c = cb / (NB2 / 2);
      const T* s0 = vt + (c * OY + j) * VP + ib * kRB;
      const T* s1 = s0 + 16 * VP;
      float2 acc[kRB];
#pragma unroll
      for (int o = 0; o < kRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < kRB + 2 * R; ++t) {
        const float2 x = make_float2(s0[t], s1[t]);
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
          const int tap = t - o;
          if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(x, (float)tp.w[tap], acc[o]);
        }
      }
      if (TRANSPOSE) {
        const int gx0 = x_org + ib * kRB;
        if (gx0 <= 0 && gx0 + kRB > 0) {
          const int o = -gx0;
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int d = 0; d <= R; ++d)
            s2 = ffma2(make_float2(s0[o + R + d], s1[o + R + d]), (float)tp.e[R - d], s2);
#pragma unroll
          for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
        }
        if (gx0 <= W - 1 && gx0 + kRB > W - 1) {
          const int o = W - 1 - gx0;
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int d = -R; d <= 0; ++d)
            s2 = ffma2(make_float2(s0[o + R + d], s1[o + R + d]), (float)tp.e[R + d], s2);
#pragma unroll
          for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
        }
      }
      T* d0 = res + (c * OY + j) * OP + ib * kRB;
      T* d1 = d0 + 16 * OP;
#pragma unroll
      for (int o = 0; o < kRB; ++o) {
        d0[o] = acc[o].x;
        d1[o] = acc[o].y;
      }
    }
  } else {
  for (int cb = warp; cb < C * NB2; cb += kNW) {
    const int j = lane;
    const int ib = cb % NB2;
    const int c = cb / NB2;
    const T* src = vt + (c * OY + j) * VP + ib * kRB;
    T acc[kRB];
#pragma unroll
    for (int o = 0; o < kRB; ++o) acc[o] = T(0);
#pragma unroll
    for (int t = 0; t < kRB + 2 * R; ++t) {
      T x = src[t];
#pragma unroll
      for (int o = 0; o < kRB; ++o) {
        const int tap = t - o;
        if (tap >= 0 && tap <= 2 * R) acc[o] = fma(tp.w[tap], x, acc[o]);
      }
    }
    if (TRANSPOSE) {
      const int gx0 = x_org + ib * kRB;
      if (gx0 <= 0 && gx0 + kRB > 0) {
        const int o = -gx0;
        T s = T(0);
#pragma unroll
        for (int d = 0; d <= R; ++d) s = fma(tp.e[R - d], src[o + R + d], s);
#pragma unroll
        for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s;
      }
      if (gx0 <= W - 1 && gx0 + kRB > W - 1) {
        const int o = W - 1 - gx0;
        T s = T(0);
#pragma unroll
        for (int d = -R; d <= 0; ++d) s = fma(tp.e[R + d], src[o + R + d], s);
#pragma unroll
        for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s;
      }
    }
    T* dst = res + (c * OY + j) * OP + ib * kRB;
#pragma unroll
    for (int o = 0; o < kRB; ++o) dst[o] = acc[o];
  }
  }
}

// Separable FIR passes over one staged tile.  rg holds the region
// [c][RY][PX] covering output rows [y_org, y_org+OY) x cols [x_org, x_org+OX)
// plus an R halo:
//  - forward (TRANSPOSE=false): replicate borders (conv1d_replicate,
//    kernel.py:36-45) -- the region holds clamped-index samples, so the in-tile
//    FIR is exact.
//  - transpose (TRANSPOSE=true): exact transpose conv1d_replicate_adjoint
//    (kernel.py:48-68) = zero-padded correlation plus cumulative-weight edge
//    rows/columns at index 0 and n-1; the region holds
//    zeros outside the image.
// Pass 1 runs along axis 0 for every region column (register blocking kRB
// outputs per thread, sliding over kRB+2R inputs), pass 2 along axis 1 with
// lanes mapped to rows (odd pitch: conflict-free).  The result
// res[c*OY*OP + j*OP + i] aliases the FIRST C*OY*OP elements of rg; the rest
// of rg is free from the start of pass 2 (`mid` runs between the passes, e.g.
// to issue prefetches of epilogue operands into rg's tail).
// Caller must __syncthreads() before reading res.
template <typename T, int R, int C, bool TRANSPOSE, class Mid>
__device__ __forceinline__ const T* fir2d_passes(T* rg, T* vt, const Taps<T>& tp, int x_org,
                                                 int y_org, int H, int W, Mid mid) {
  using S = FirSmem<T, R, C>;
  constexpr int OX = S::OX, OY = S::OY, RX = S::RX, PX = S::PX, VP = S::VP, OP = S::OP,
                CS = S::CS;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  // ---- pass 1: along axis 0 (rows), for every region column ----
  constexpr int NB1 = OY / kRB;
  if constexpr (sizeof(T) == 4) {
    // fp32: two adjacent columns per thread, packed FFMA2 on (col i, col i+1) with
    // 8-byte aligned smem pairs (the pair grid follows the smem address parity)
    const int par = (int)((reinterpret_cast<uintptr_t>(rg) >> 2) & 1);
    const int npairs = (RX + par + 1) / 2;
    for (int cb = warp; cb < C * NB1; cb += kNW)
    for (int pp = lane; pp < npairs; pp += 32) {
      const int jb = cb % NB1;
      const int c = cb / NB1;
      const int i0 = 2 * pp - par;
      const float2* src = reinterpret_cast<const float2*>(rg + c * CS + jb * kRB * PX + i0);
      float2 acc[kRB];
#pragma unroll
      for (int o = 0; o < kRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < kRB + 2 * R; ++t) {
        const float2 x = src[t * (PX / 2)];
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
          const int tap = t - o;
          if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(x, (float)tp.w[tap], acc[o]);
        }
      }
      if (TRANSPOSE) {
        const int gy0 = y_org + jb * kRB;
        const float* fsrc = reinterpret_cast<const float*>(src);
        if (gy0 <= 0 && gy0 + kRB > 0) {
          const int o = -gy0;
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int d = 0; d <= R; ++d)
            s2 = ffma2(make_float2(fsrc[(o + R + d) * PX], fsrc[(o + R + d) * PX + 1]),
                       (float)tp.e[R - d], s2);
#pragma unroll
          for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
        }
        if (gy0 <= H - 1 && gy0 + kRB > H - 1) {
          const int o = H - 1 - gy0;
          float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int d = -R; d <= 0; ++d)
            s2 = ffma2(make_float2(fsrc[(o + R + d) * PX], fsrc[(o + R + d) * PX + 1]),
                       (float)tp.e[R + d], s2);
#pragma unroll
          for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
        }
      }
      T* dst = vt + (c * OY + jb * kRB) * VP + i0;
      if (i0 >= 0 && i0 < RX) {
#pragma unroll
        for (int o = 0; o < kRB; ++o) dst[o * VP] = acc[o].x;
      }
      if (i0 + 1 < RX) {
#pragma unroll
        for (int o = 0; o < kRB; ++o) dst[o * VP + 1] = acc[o].y;
      }
    }
  } else {
  for (int cb = warp; cb < C * NB1; cb += kNW)
  for (int i = lane; i < RX; i += 32) {
    const int jb = cb % NB1;
    const int c = cb / NB1;
    const T* src = rg + c * CS + jb * kRB * PX + i;
    T acc[kRB];
#pragma unroll
    for (int o = 0; o < kRB; ++o) acc[o] = T(0);
#pragma unroll
    for (int t = 0; t < kRB + 2 * R; ++t) {
      T x = src[t * PX];
#pragma unroll
      for (int o = 0; o < kRB; ++o) {
        const int tap = t - o;
        if (tap >= 0 && tap <= 2 * R) acc[o] = fma(tp.w[tap], x, acc[o]);
      }
    }
    if (TRANSPOSE) {
      const int gy0 = y_org + jb * kRB;
      if (gy0 <= 0 && gy0 + kRB > 0) {  // output row 0: sum_{d=0..R} W[R-d] g[d]
        const int o = -gy0;
        T s = T(0);
#pragma unroll
        for (int d = 0; d <= R; ++d) s = fma(tp.e[R - d], src[(o + R + d) * PX], s);
#pragma unroll
        for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s;
      }
      if (gy0 <= H - 1 && gy0 + kRB > H - 1) {  // row n-1: sum_{d=-R..0} W[R+d] g[n-1+d]
        const int o = H - 1 - gy0;
        T s = T(0);
#pragma unroll
        for (int d = -R; d <= 0; ++d) s = fma(tp.e[R + d], src[(o + R + d) * PX], s);
#pragma unroll
        for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s;
      }
    }
    T* dst = vt + (c * OY + jb * kRB) * VP + i;
#pragma unroll
    for (int o = 0; o < kRB; ++o) dst[o * VP] = acc[o];
  }
  }
  __syncthreads();
  mid();

  T* res = rg;
  fir2d_pass2<T, R, C, TRANSPOSE>(vt, res, tp, x_org, W);
  return res;
}

struct NoMid {
  __device__ void operator()() const {}
};

// Generic tile: staging through `ld(gy, gx, out[C])` (clamped / zero-padded as
// above), then the passes.  Used by the smoothing entry points; the hot
// kernels stage with TMA (or cp.async) instead.
template <typename T, int R, int C, bool TRANSPOSE, class Loader>
__device__ __forceinline__ const T* fir2d_tile(T* sm, const Taps<T>& tp, int x_org, int y_org,
                                               int H, int W, Loader ld) {
  using S = FirSmem<T, R, C>;
  constexpr int RX = S::RX, RY = S::RY, PX = S::PX, CS = S::CS;
  T* rg = sm;
  T* vt = sm + S::region;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < RY; j += kNW)
    for (int i = lane; i < RX; i += 32) {
      int gy = y_org - R + j, gx = x_org - R + i;
      T vals[C];
      if (TRANSPOSE) {
        if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
          ld(gy, gx, vals);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) vals[c] = T(0);
        }
      } else {
        gy = min(max(gy, 0), H - 1);
        gx = min(max(gx, 0), W - 1);
        ld(gy, gx, vals);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) rg[c * CS + j * PX + i] = vals[c];
    }
  __syncthreads();
  const T* res = fir2d_passes<T, R, C, TRANSPOSE>(rg, vt, tp, x_org, y_org, H, W, NoMid{});
  __syncthreads();
  return res;
}

// np.gradient of I at (y, x) along both axes (fields.py:144-145, 161-162).
template <typename T>
__device__ __forceinline__ void grad2(const T* __restrict__ I, int y, int x, int H, int W, T& g0,
                                     T& g1) {
  const long long row = (long long)y * W;
  T c = I[row + x];
  T up = (y > 0) ? I[row - W + x] : c;
  T dn = (y < H - 1) ? I[row + W + x] : c;
  T lf = (x > 0) ? I[row + x - 1] : c;
  T rt = (x < W - 1) ? I[row + x + 1] : c;
  g0 = grad1(up, c, dn, y, H);
  g1 = grad1(lf, c, rt, x, W);
}

// ------------------------------------------------------------------------------
// K1: v = -K*(z grad I) (+ guard on I, z, v)
// ------------------------------------------------------------------------------
template <typename T>
struct VelArgs {
  const T* I;
  const T* z;
  T* v;
  int32_t* guard;     // nullable, guard[b * guard_stride]
  int guard_stride;
  int use_tma;        // tensor maps valid (else cp.async staging)
  Grid2 g;
  T* vtmp;            // nullable [B][2][N] scratch: enables the split (two-kernel) path
};

// smem of K1: mbarrier | region m[2][RY][PX] (z staged into m[1]) |
//             union{ I stage [(RY+2)][PXI], pass-1 output }
template <typename T, int R>
struct VelSmem {
  using S = FirSmem<T, R, 2>;
  static constexpr int PXI = round_up(S::RX + 2 + S::A - 1, S::A);  // I stage pitch / box width
  static constexpr int istage = round_up((S::RY + 2) * PXI + S::A, 32);
  static constexpr int aux = istage > S::vt ? istage : S::vt;
  static constexpr size_t head = 128;  // mbarriers
  static constexpr size_t bytes = head + sizeof(T) * (size_t)(S::region + aux);
};

template <typename T, int R>
__global__ void __launch_bounds__(kThreads)
    k_velocity2d(VelArgs<T> a, Taps<T> tp, const __grid_constant__ CUtensorMap mapI,
                 const __grid_constant__ CUtensorMap mapZ) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using S = FirSmem<T, R, 2>;
  using V = VelSmem<T, R>;
  constexpr int RX = S::RX, RY = S::RY, PX = S::PX, PXI = V::PXI;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* rg0 = reinterpret_cast<T*>(smem_raw + V::head);
  T* ist0 = rg0 + S::region;  // I stage; later the pass-1 output
  const int H = a.g.H, W = a.g.W;
  const int b = blockIdx.z;
  const int x_org = blockIdx.x * S::OX, y_org = blockIdx.y * S::OY;
  unsigned flags = 0;
  const int offZ = align_shift(x_org - R, S::A), offI = align_shift(x_org - R - 1, S::A);
  T* rg = rg0 + offZ;  // region element (j, i) at rg[j*PX + i]
  T* m0 = rg;
  T* m1 = rg + S::CS;
  T* ist = ist0 + offI;  // I stage element (j, i) at ist[j*PXI + i]
  const T* __restrict__ I = a.I + b * a.g.N;
  const T* __restrict__ z = a.z + b * a.g.N;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- stage I (region + 1) and z (region) ----
  if (a.use_tma) {
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_barrier_init();
      mbar_expect_tx(bar, (unsigned)(sizeof(T) * (PXI * (RY + 2) + PX * RY)));
      tma_load_3d(ist0, &mapI, x_org - R - 1 - offI, y_org - R - 1, b, bar);
      tma_load_3d(rg0 + S::CS, &mapZ, x_org - R - offZ, y_org - R, b, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
  } else {
    for (int j = warp; j < RY + 2; j += kNW) {
      const T* row = I + (long long)min(max(y_org - R - 1 + j, 0), H - 1) * W;
      for (int i = lane; i < RX + 2; i += 32)
        cp_async_elem(ist + j * PXI + i, row + min(max(x_org - R - 1 + i, 0), W - 1));
    }
    for (int j = warp; j < RY; j += kNW) {
      const T* row = z + (long long)min(max(y_org - R + j, 0), H - 1) * W;
      for (int i = lane; i < RX; i += 32)
        cp_async_elem(m1 + j * PX + i, row + min(max(x_org - R + i, 0), W - 1));
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }

  // ---- m = z grad I at in-image region samples (integrator.py:94) ----
  // (the guard on I and z runs in the transport kernel that produces them)
  const int i_lo = max(0, R - x_org), i_hi = min(RX, W - x_org + R);  // in-image columns
  const int j_lo = max(0, R - y_org), j_hi = min(RY, H - y_org + R);  // in-image rows
  // interior tile: every in-image sample has both neighbours on both axes
  const bool interior = (y_org - R >= 1) && (y_org - R + RY <= H - 1) && (x_org - R >= 1) &&
                        (x_org - R + RX <= W - 1);
  for (int j = j_lo + warp; j < j_hi; j += kNW) {
    const int uy = y_org - R + j;
    const T* crow = ist + (j + 1) * PXI + 1;
    for (int i = i_lo + lane; i < i_hi; i += 32) {
      const T* c = crow + i;
      const T f0 = c[0];
      T g0, g1;
      if (interior) {
        g0 = (c[PXI] - c[-PXI]) / T(2);
        g1 = (c[1] - c[-1]) / T(2);
      } else {
        const int ux = x_org - R + i;
        g0 = grad1(c[-PXI], f0, c[PXI], uy, H);
        g1 = grad1(c[-1], f0, c[1], ux, W);
      }
      const int p = j * PX + i;
      const T zz = m1[p];
      m0[p] = zz * g0;
      m1[p] = zz * g1;
    }
  }
  __syncthreads();
  // border tiles: replicate the border samples into the clamped halo
  // (columns of in-image rows first, then whole rows)
  if (i_lo > 0 || i_hi < RX) {
    const int nl = i_lo, nr = RX - i_hi;
    for (int j = j_lo + warp; j < j_hi; j += kNW)
      for (int t = lane; t < nl + nr; t += 32) {
        const int i = t < nl ? t : i_hi + (t - nl);
        const int ir = t < nl ? i_lo : i_hi - 1;
        m0[j * PX + i] = m0[j * PX + ir];
        m1[j * PX + i] = m1[j * PX + ir];
      }
    __syncthreads();
  }
  if (j_lo > 0 || j_hi < RY) {
    const int nt = j_lo, nb = RY - j_hi;
    for (int t = warp; t < nt + nb; t += kNW) {
      const int j = t < nt ? t : j_hi + (t - nt);
      const int jr = t < nt ? j_lo : j_hi - 1;
      for (int i = lane; i < RX; i += 32) {
        m0[j * PX + i] = m0[jr * PX + i];
        m1[j * PX + i] = m1[jr * PX + i];
      }
    }
    __syncthreads();
  }

  const T* res = fir2d_passes<T, R, 2, false>(rg, ist0, tp, x_org, y_org, H, W, NoMid{});
  __syncthreads();

  T* v0 = a.v + (long long)b * 2 * a.g.N;
  T* v1 = v0 + a.g.N;
  for (int j = warp; j < S::OY; j += kNW) {
    const int gy = y_org + j;
    if (gy >= H) break;
    for (int i = lane; i < S::OX; i += 32) {
      const int gx = x_org + i;
      if (gx >= W) break;
      const long long q = (long long)gy * W + gx;
      const T a0 = -res[j * S::OP + i];
      const T a1 = -res[(S::OY + j) * S::OP + i];
      v0[q] = a0;
      v1[q] = a1;
      flags |= guard_bits(a0, MR_GUARD_VELOCITY_NONFINITE);
      flags |= guard_bits(a1, MR_GUARD_VELOCITY_NONFINITE);
    }
  }
  if (a.guard) flush_flags(flags, a.guard + (long long)b * a.guard_stride);
}

// ------------------------------------------------------------------------------
// smooth_arr / smooth_adjoint_arr on a scalar batch (kernel.py:71-79)
// ------------------------------------------------------------------------------
template <typename T>
struct SmoothArgs {
  const T* a;
  T* out;
  Grid2 g;
};

template <typename T, int R, bool TRANSPOSE>
__global__ void __launch_bounds__(kThreads) k_smooth2d(SmoothArgs<T> a, Taps<T> tp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  using S = FirSmem<T, R, 1>;
  const int H = a.g.H, W = a.g.W;
  const int b = blockIdx.z;
  const int x_org = blockIdx.x * S::OX, y_org = blockIdx.y * S::OY;
  const T* __restrict__ src = a.a + b * a.g.N;
  auto ld = [&](int gy, int gx, T* out) { out[0] = src[(long long)gy * W + gx]; };
  const T* res = fir2d_tile<T, R, 1, TRANSPOSE>(sm, tp, x_org, y_org, H, W, ld);
  T* dst = a.out + b * a.g.N;
  for (int p = threadIdx.x; p < S::OX * S::OY; p += kThreads) {
    int j = p / S::OX, i = p - j * S::OX;
    int gy = y_org + j, gx = x_org + i;
    if (gy < H && gx < W) dst[(long long)gy * W + gx] = res[j * S::OP + i];
  }
}

// TMA-staged variant (fp32): the whole region (tile + R halo) arrives as one box;
// the box's zero fill outside the image is the transpose's zero padding, and for
// the forward FIR border tiles copy each out-of-image element from its clamped
// (in-image, in-region) source = replicate borders.  Then the same FIR passes.
template <int R>
struct SmoothTmaSmem {
  using S = FirSmem<float, R, 1>;
  static constexpr size_t head = 128;
  static constexpr size_t bytes = head + S::bytes;
};

template <int R, bool TRANSPOSE>
__global__ void __launch_bounds__(kThreads)
    k_smooth2d_tma(SmoothArgs<float> a, Taps<float> tp, const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using S = FirSmem<float, R, 1>;
  constexpr int RX = S::RX, RY = S::RY, PX = S::PX;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  float* rg0 = reinterpret_cast<float*>(smem_raw + SmoothTmaSmem<R>::head);
  float* vt = rg0 + S::region;
  const int H = a.g.H, W = a.g.W;
  const int b = blockIdx.z;
  const int x_org = blockIdx.x * S::OX, y_org = blockIdx.y * S::OY;
  const int xs = x_org - R, ys = y_org - R;
  const int offV = align_shift(xs, S::A);
  float* rg = rg0 + offV;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(float) * PX * RY));
    tma_load_3d(rg0, &map, xs - offV, ys, b, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  if (!TRANSPOSE && (xs < 0 || ys < 0 || xs + RX > W || ys + RY > H)) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int jlo = max(0, -ys), jhi = min(RY, H - ys);  // in-image rows [jlo, jhi)
    const int ilo = max(0, -xs), ihi = min(RX, W - xs);  // in-image columns [ilo, ihi)
    if (ilo > 0 || ihi < RX) {  // 1) out-of-image columns of in-image rows
      const int nl = ilo, nr = RX - ihi;
      for (int j = jlo + warp; j < jhi; j += kNW)
        for (int t = lane; t < nl + nr; t += 32) {
          const int i = t < nl ? t : ihi + (t - nl);
          rg[j * PX + i] = rg[j * PX + (t < nl ? ilo : ihi - 1)];
        }
      __syncthreads();
    }
    // 2) out-of-image rows copy their clamped row (whole width, columns already fixed)
    for (int j = warp; j < RY; j += kNW) {
      if (j >= jlo && j < jhi) continue;
      const int src = j < jlo ? jlo : jhi - 1;
      for (int i = lane; i < RX; i += 32) rg[j * PX + i] = rg[src * PX + i];
    }
    __syncthreads();
  }
  const float* res = fir2d_passes<float, R, 1, TRANSPOSE>(rg, vt, tp, x_org, y_org, H, W, NoMid{});
  __syncthreads();
  float* dst = a.out + b * a.g.N;
  for (int p = threadIdx.x; p < S::OX * S::OY; p += kThreads) {
    const int j = p / S::OX, i = p - j * S::OX;
    const int gy = y_org + j, gx = x_org + i;
    if (gy < H && gx < W) dst[gy * W + gx] = res[j * S::OP + i];
  }
}

// ------------------------------------------------------------------------------
// K2: one semi-Lagrangian step (integrator.py:101-110, 193-205)
// ------------------------------------------------------------------------------
template <typename T>
struct StepArgs {
  const T* I;
  const T* z;
  const T* v;
  T* In;
  T* zn;
  const T* phi_in;  // nullable
  T* phi_out;
  T dt, dtmu;
  bool has_mu;
  int32_t* guard_in;   // nullable: guard word of the input step (checked at step 0 only)
  int32_t* guard_out;  // nullable: guard word of the output step
  int guard_stride;
  Grid2 g;
};

// Each thread handles kStepPix pixels of one column (rows kThreads/32 apart):
// all loads of a phase are issued before any is consumed, so enough bytes are
// in flight to cover HBM latency (the one-pixel form stalled on its v load).
constexpr int kStepPix = 2;
constexpr int kStepRows = (kThreads / 32) * kStepPix;  // rows per block

template <typename T>
__global__ void __launch_bounds__(kThreads) k_sl_step2d(StepArgs<T> a) {
  const int H = a.g.H, W = a.g.W;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int yb = blockIdx.y * kStepRows + (threadIdx.x >> 5);
  const int b = blockIdx.z;
  if (x >= W) return;
  const long long N = a.g.N;
  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  const T* __restrict__ v0 = a.v + b * 2 * N;
  const T* __restrict__ v1 = v0 + N;
  int yy[kStepPix];
  bool act[kStepPix];
  long long q[kStepPix];
  T vy[kStepPix], vx[kStepPix], up[kStepPix], dn[kStepPix], lf[kStepPix], rt[kStepPix];
#pragma unroll
  for (int k = 0; k < kStepPix; ++k) {
    yy[k] = yb + k * (kThreads / 32);
    act[k] = yy[k] < H;
    const int y = act[k] ? yy[k] : H - 1;
    q[k] = (long long)y * W + x;
  }
#pragma unroll
  for (int k = 0; k < kStepPix; ++k) {
    const int y = act[k] ? yy[k] : H - 1;
    vy[k] = v0[q[k]];
    vx[k] = v1[q[k]];
    up[k] = v0[y > 0 ? q[k] - W : q[k]];
    dn[k] = v0[y < H - 1 ? q[k] + W : q[k]];
    lf[k] = v1[x > 0 ? q[k] - 1 : q[k]];
    rt[k] = v1[x < W - 1 ? q[k] + 1 : q[k]];
  }
  AxisPlan<T> py[kStepPix], px[kStepPix];
  long long c00[kStepPix];
#pragma unroll
  for (int k = 0; k < kStepPix; ++k) {
    const int y = act[k] ? yy[k] : H - 1;
    py[k] = plan_axis<T>(y, vy[k], a.dt, H);
    px[k] = plan_axis<T>(x, vx[k], a.dt, W);
    c00[k] = (long long)py[k].i0 * W + px[k].i0;
  }
  T ci[kStepPix][4], cz[kStepPix][4], zq[kStepPix];
#pragma unroll
  for (int k = 0; k < kStepPix; ++k) {
    ci[k][0] = I[c00[k]];
    ci[k][1] = I[c00[k] + W];
    ci[k][2] = I[c00[k] + 1];
    ci[k][3] = I[c00[k] + W + 1];
    cz[k][0] = z[c00[k]];
    cz[k][1] = z[c00[k] + W];
    cz[k][2] = z[c00[k] + 1];
    cz[k][3] = z[c00[k] + W + 1];
    zq[k] = (a.has_mu || a.guard_in) ? z[q[k]] : T(0);
  }
  unsigned fin = 0, fout = 0;
#pragma unroll
  for (int k = 0; k < kStepPix; ++k) {
    if (!act[k]) continue;
    const int y = yy[k];
    if (a.guard_in) {  // _guard(0, image, momentum) on the inputs (integrator.py:184)
      fin |= guard_bits(I[q[k]], MR_GUARD_IMAGE_NONFINITE) |
             guard_bits(zq[k], MR_GUARD_MOMENTUM_NONFINITE);
    }
    T bi = bilerp(ci[k][0], ci[k][1], ci[k][2], ci[k][3], py[k].f, px[k].f);
    if (a.has_mu) bi = bi + a.dtmu * zq[k];  // advect_image_sl_arr: + dt*mu*z
    const T bz = bilerp(cz[k][0], cz[k][1], cz[k][2], cz[k][3], py[k].f, px[k].f);
    // divergence_arr (fields.py:169-170)
    const T div = grad1(up[k], vy[k], dn[k], y, H) + grad1(lf[k], vx[k], rt[k], x, W);
    const T zn = bz * (T(1) - a.dt * div);
    a.In[b * N + q[k]] = bi;
    a.zn[b * N + q[k]] = zn;
    fout |= guard_bits(bi, MR_GUARD_IMAGE_NONFINITE) | guard_bits(zn, MR_GUARD_MOMENTUM_NONFINITE);
    if (a.phi_in) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const T* __restrict__ ph = a.phi_in + (b * 2 + c) * N;
        a.phi_out[(b * 2 + c) * N + q[k]] = bilerp(ph[c00[k]], ph[c00[k] + W], ph[c00[k] + 1],
                                                   ph[c00[k] + W + 1], py[k].f, px[k].f);
      }
    }
  }
  // flags are almost always zero: no warp reduction needed
  if (fin && a.guard_in)
    atomicOr(reinterpret_cast<int*>(a.guard_in + (long long)b * a.guard_stride), (int)fin);
  if (fout && a.guard_out)
    atomicOr(reinterpret_cast<int*>(a.guard_out + (long long)b * a.guard_stride), (int)fout);
}

template <typename T>
__global__ void k_identity2d(T* phi, Grid2 g) {
  long long n = (long long)g.B * g.N;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    long long b = p / g.N, q = p - b * g.N;
    int y = (int)(q / g.W), x = (int)(q - (long long)y * g.W);
    phi[(b * 2 + 0) * g.N + q] = T(y);
    phi[(b * 2 + 1) * g.N + q] = T(x);
  }
}

// ------------------------------------------------------------------------------
// K3: adjoint of one SL step (objective.py:118-147, SL branches)
// ------------------------------------------------------------------------------
template <typename T>
struct AdjArgs {
  const T* I;
  const T* z;
  const T* v;
  const T* ibar;  // adjoint of I_{k+1}
  const T* zbar;  // adjoint of z_{k+1}
  T* ib;          // scatter target (zeroed)
  T* zb;          // scatter target (zeroed)
  T* vbar;        // [B][2][N] output
  T dt, dtmu;
  bool has_mu;
  T reg_lam;  // k = 0 only: vbar -= reg_lam * z grad I (regulariser fold)
  Grid2 g;
  // deterministic mode (DET kernels): fixed-point scatter targets, per-pair
  // max |ibar|, |zbar| as double bits, overflow flag
  unsigned long long* qib;
  unsigned long long* qzb;
  const unsigned long long* mbits;
  int* ovf;
};

constexpr int kAdjTX = 32, kAdjTY = kThreads / 32;

// Scatter of the four bilinear-transpose contributions of one pixel
// (bilinear_adjoint_values, fields.py:243-254) with warp-level merging: lanes
// are consecutive x of one row, so where lane l-1's right cells are lane l's
// left cells (same integer offset) lane l adds them and lane l-1 skips its
// own -> ~2 instead of 4 red.global.add per pixel on smooth fields.
template <typename T>
__device__ __forceinline__ void scatter4_merged(T* __restrict__ out, long long cell, bool valid,
                                                long long W, T ca, T cb, T cc, T cd) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long key = valid ? cell : -4;
  const long long prev_key = __shfl_up_sync(full, key, 1);
  const long long next_key = __shfl_down_sync(full, key, 1);
  const T pc = __shfl_up_sync(full, cc, 1);
  const T pd = __shfl_up_sync(full, cd, 1);
  if (!valid) return;
  const bool merge_left = lane > 0 && prev_key >= 0 && prev_key + 1 == key;
  const bool merged_by_next = lane < 31 && next_key >= 0 && key + 1 == next_key;
  if (merge_left) {
    ca += pc;
    cb += pd;
  }
  atomicAdd(out + cell, ca);
  atomicAdd(out + cell + W, cb);
  if (!merged_by_next) {
    atomicAdd(out + cell + 1, cc);
    atomicAdd(out + cell + W + 1, cd);
  }
}

constexpr int kAdjPix = 1;                       // pixels per thread (rows kAdjTY apart)
constexpr int kAdjRows = kAdjTY * kAdjPix;        // tile rows

template <typename T, bool DET = false>
__global__ void __launch_bounds__(kThreads) k_sl_adjoint2d(AdjArgs<T> a) {
  __shared__ T s_div[kAdjRows + 2][kAdjTX + 2];  // s = -dt * zbar * B(z), halo 1
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * kAdjTX, y0 = blockIdx.y * kAdjRows;
  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  const T* __restrict__ v0 = a.v + b * 2 * N;
  const T* __restrict__ v1 = v0 + N;
  const T* __restrict__ ibar = a.ibar + b * N;
  const T* __restrict__ zbar = a.zbar + b * N;
  const T dt = a.dt;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x = x0 + tx;

  int yy[kAdjPix];
  bool own[kAdjPix];
  long long q[kAdjPix];
  T vy[kAdjPix], vx[kAdjPix], up[kAdjPix], dn[kAdjPix], lf[kAdjPix], rt[kAdjPix];
  T ibv[kAdjPix], zbv[kAdjPix];
#pragma unroll
  for (int k = 0; k < kAdjPix; ++k) {
    yy[k] = y0 + ty + k * kAdjTY;
    own[k] = x < W && yy[k] < H;
    const int y = own[k] ? yy[k] : 0;
    const int xc = own[k] ? x : 0;
    q[k] = (long long)y * W + xc;
    vy[k] = v0[q[k]];
    vx[k] = v1[q[k]];
    up[k] = v0[y > 0 ? q[k] - W : q[k]];
    dn[k] = v0[y < H - 1 ? q[k] + W : q[k]];
    lf[k] = v1[xc > 0 ? q[k] - 1 : q[k]];
    rt[k] = v1[xc < W - 1 ? q[k] + 1 : q[k]];
    ibv[k] = ibar[q[k]];
    zbv[k] = zbar[q[k]];
  }
  AxisPlan<T> py[kAdjPix], px[kAdjPix];
  long long c00[kAdjPix];
#pragma unroll
  for (int k = 0; k < kAdjPix; ++k) {
    py[k] = plan_axis<T>(own[k] ? yy[k] : 0, vy[k], dt, H);
    px[k] = plan_axis<T>(own[k] ? x : 0, vx[k], dt, W);
    c00[k] = (long long)py[k].i0 * W + px[k].i0;
  }
  T ci[kAdjPix][4], cz[kAdjPix][4];
#pragma unroll
  for (int k = 0; k < kAdjPix; ++k) {
    ci[k][0] = I[c00[k]];
    ci[k][1] = I[c00[k] + W];
    ci[k][2] = I[c00[k] + 1];
    ci[k][3] = I[c00[k] + W + 1];
    cz[k][0] = z[c00[k]];
    cz[k][1] = z[c00[k] + W];
    cz[k][2] = z[c00[k] + 1];
    cz[k][3] = z[c00[k] + W + 1];
  }
  T wz[kAdjPix];
#pragma unroll
  for (int k = 0; k < kAdjPix; ++k) {
    const int y = own[k] ? yy[k] : 0;
    const T scale = T(1) - dt * (grad1(up[k], vy[k], dn[k], y, H) +
                                 grad1(lf[k], vx[k], rt[k], own[k] ? x : 0, W));
    wz[k] = zbv[k] * scale;
    s_div[ty + k * kAdjTY + 1][tx + 1] =
        own[k] ? -dt * (zbv[k] * bilerp(cz[k][0], cz[k][1], cz[k][2], cz[k][3], py[k].f, px[k].f))
               : T(0);
  }

  // ---- s on the 1-pixel halo ring of the tile ----
  constexpr int NHALO = 2 * (kAdjTX + 2) + 2 * kAdjRows;
  for (int h = threadIdx.x; h < NHALO; h += kThreads) {
    int j, i;
    if (h < kAdjTX + 2) { j = 0; i = h; }
    else if (h < 2 * (kAdjTX + 2)) { j = kAdjRows + 1; i = h - (kAdjTX + 2); }
    else { const int k = h - 2 * (kAdjTX + 2); j = 1 + (k >> 1); i = (k & 1) ? kAdjTX + 1 : 0; }
    const int gy = y0 - 1 + j, gx = x0 - 1 + i;
    T sv = T(0);
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
      const long long qq = (long long)gy * W + gx;
      const AxisPlan<T> hy = plan_axis<T>(gy, v0[qq], dt, H);
      const AxisPlan<T> hx = plan_axis<T>(gx, v1[qq], dt, W);
      const long long h00 = (long long)hy.i0 * W + hx.i0;
      sv = -dt * (zbar[qq] * bilerp(z[h00], z[h00 + W], z[h00 + 1], z[h00 + W + 1], hy.f, hx.f));
    }
    s_div[j][i] = sv;
  }

  // ---- scatters: ib = P^T ibar; zb = P^T (zbar*scale) + dt mu ibar ----
  if constexpr (DET) {
    const double f = fix_factor(a.mbits, b);
    unsigned ovf = 0;
#pragma unroll
    for (int k = 0; k < kAdjPix; ++k) {
      const T fy = py[k].f, fx = px[k].f, wy = T(1) - fy, wx = T(1) - fx;
      const T g = ibv[k], w = wz[k];
      scatter4_merged_fix(a.qib + b * N, c00[k], own[k], (long long)W, f, wy * wx * g,
                          fy * wx * g, wy * fx * g, fy * fx * g, ovf);
      scatter4_merged_fix(a.qzb + b * N, c00[k], own[k], (long long)W, f, wy * wx * w,
                          fy * wx * w, wy * fx * w, fy * fx * w, ovf);
      if (own[k] && a.has_mu) fix_add(a.qzb + b * N + q[k], to_fix(a.dtmu * g, f, ovf));
    }
    if (ovf) atomicOr(a.ovf, 1);
  } else {
    T* __restrict__ ibo = a.ib + b * N;
    T* __restrict__ zbo = a.zb + b * N;
#pragma unroll
    for (int k = 0; k < kAdjPix; ++k) {
      const T fy = py[k].f, fx = px[k].f, wy = T(1) - fy, wx = T(1) - fx;
      const T g = ibv[k], w = wz[k];
      scatter4_merged(ibo, c00[k], own[k], (long long)W, wy * wx * g, fy * wx * g, wy * fx * g,
                      fy * fx * g);
      scatter4_merged(zbo, c00[k], own[k], (long long)W, wy * wx * w, fy * wx * w, wy * fx * w,
                      fy * fx * w);
      if (own[k] && a.has_mu) atomicAdd(zbo + q[k], a.dtmu * g);  // zb = dt*mu*ibar (:133)
    }
  }
  __syncthreads();

  // ---- vbar (objective.py:131-132, 143-147) ----
#pragma unroll
  for (int k = 0; k < kAdjPix; ++k) {
    if (!own[k]) continue;
    const int y = yy[k];
    const T fy = py[k].f, fx = px[k].f, wy = T(1) - fy, wx = T(1) - fx;
    const T ia = ci[k][0], ib2 = ci[k][1], ic = ci[k][2], id = ci[k][3];
    const T za = cz[k][0], zb2 = cz[k][1], zc = cz[k][2], zd = cz[k][3];
    const T ddy = (wx * (ib2 - ia) + fx * (id - ic)) * (py[k].inside ? T(1) : T(0));
    const T ddx = (wy * (ic - ia) + fy * (id - ib2)) * (px[k].inside ? T(1) : T(0));
    T vb0 = -dt * ddy * ibv[k];
    T vb1 = -dt * ddx * ibv[k];
    const T dzy = (wx * (zb2 - za) + fx * (zd - zc)) * (py[k].inside ? T(1) : T(0));
    const T dzx = (wy * (zc - za) + fy * (zd - zb2)) * (px[k].inside ? T(1) : T(0));
    vb0 += -dt * dzy * wz[k];
    vb1 += -dt * dzx * wz[k];
    const int j = ty + k * kAdjTY + 1, i = tx + 1;
    const T sm_ = s_div[j - 1][i], sp_ = s_div[j + 1][i];
    const T s_first_y = (y <= 1) ? s_div[j - y][i] : T(0);
    const T s_last_y = (y >= H - 2) ? s_div[j + (H - 1 - y)][i] : T(0);
    vb0 += diff_adj1(sm_, sp_, s_first_y, s_last_y, y, H);
    const T sl_ = s_div[j][i - 1], sr_ = s_div[j][i + 1];
    const T s_first_x = (x <= 1) ? s_div[j][i - x] : T(0);
    const T s_last_x = (x >= W - 2) ? s_div[j][i + (W - 1 - x)] : T(0);
    vb1 += diff_adj1(sl_, sr_, s_first_x, s_last_x, x, W);
    if (a.reg_lam != T(0)) {
      T g0, g1;
      grad2(I, y, x, H, W, g0, g1);
      const T zz = z[q[k]];
      vb0 = vb0 - a.reg_lam * (zz * g0);
      vb1 = vb1 - a.reg_lam * (zz * g1);
    }
    a.vbar[b * 2 * N + q[k]] = vb0;
    a.vbar[b * 2 * N + N + q[k]] = vb1;
  }
}

// ------------------------------------------------------------------------------
// K4: adjoint of v = -K*(z grad I) (objective.py:157-161); REG adds the
// regulariser gradient at k = 0 (objective.py:165-169).
// ------------------------------------------------------------------------------
template <typename T>
struct VelAdjArgs {
  const T* I;
  const T* z;
  const T* vbar;   // [B][2][N]
  T* ib;           // in/out: ib_acc -> ibar_k (unused when REG)
  T* zb;           // in/out: zb_acc -> zbar_k
  // REG only
  const T* v0;     // forward v at k = 0
  T* zout;         // dH/dz0
  int32_t* flags;  // per pair non-finite flag
  T lam, two_rho;
  int use_tma;
  T* zero_a;       // nullable: buffers zeroed at the owner pixels (the consumed
  T* zero_b;       //   ibar/zbar of step k+1 = next step's scatter targets)
  T* vtmp;         // nullable scratch [B][2][N]: enables the split path (axis-0 pass
                   //   to vtmp, then the axis-1 pass + epilogue), fp32 only
  Grid2 g;
};

// Tensor maps of K4: vbar (dims W,H,2B), then the epilogue operands
// I, z, ib|v0 (W,H,B | W,H,2B), zb, v0 (REG, second component).
struct VelAdjMaps {
  CUtensorMap vbar, I, z, op2, zb;
};

// smem of K4: mbarriers | region rg (padded so that, once pass 1 is done, its
// tail holds the epilogue operands [5][OY][OX] next to the result) | vt.
template <typename T, int R>
struct VelAdjSmem {
  using S = FirSmem<T, R, 2>;
  static constexpr int OXP = S::OX + S::A;  // epilogue box width (room for the shift)
  static constexpr int OXY = round_up(OXP * S::OY, 32);  // operand stride (128-B aligned)
  static constexpr int res = round_up(2 * S::OY * S::OP + S::A, 32);
  static constexpr int rg = S::region > res + 5 * OXY ? S::region : res + 5 * OXY;
  static constexpr size_t head = 128;
  static constexpr size_t bytes = head + sizeof(T) * (size_t)(rg + S::vt);
};

template <typename T, int R, bool REG>
__global__ void __launch_bounds__(kThreads)
    k_velocity_adj2d(VelAdjArgs<T> a, Taps<T> tp, const __grid_constant__ VelAdjMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using S = FirSmem<T, R, 2>;
  using V = VelAdjSmem<T, R>;
  constexpr int OX = S::OX, OY = S::OY, OP = S::OP, RX = S::RX, RY = S::RY, PX = S::PX,
                OXY = V::OXY, OXP = V::OXP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* rg0 = reinterpret_cast<T*>(smem_raw + V::head);
  T* vt = rg0 + V::rg;
  T* tail0 = rg0 + V::res;  // [5][OY][OXP]: I, z, ib|v0_0, zb, -|v0_1
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x_org = blockIdx.x * (OX - 2) - 1, y_org = blockIdx.y * (OY - 2) - 1;
  const int offV = align_shift(x_org - R, S::A), offE = align_shift(x_org, S::A);
  T* rg = rg0 + offV;      // region element (j, i) at rg[j*PX + i]
  T* tail = tail0 + offE;  // operand k element (j, i) at tail[k*OXY + j*OXP + i]
  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  const T* __restrict__ vb0 = a.vbar + b * 2 * N;
  const T* __restrict__ vb1 = vb0 + N;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- stage vbar, zero outside the image ----
  // (at k = 0 the transport adjoint already folded -lam*m0 into vbar, so
  //  -K^T(vbar - lam m0) also yields the +lam K^T m0 regulariser term, A.17)
  if (a.use_tma) {
    if (tid == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      fence_barrier_init();
      mbar_expect_tx(bar, (unsigned)(sizeof(T) * 2 * PX * RY));
      tma_load_3d(rg0, &maps.vbar, x_org - R - offV, y_org - R, 2 * b, bar);
      tma_load_3d(rg0 + S::CS, &maps.vbar, x_org - R - offV, y_org - R, 2 * b + 1, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
  } else {
    for (int j = warp; j < RY; j += kNW) {
      const int gy = y_org - R + j;
      const bool rin = gy >= 0 && gy < H;
      const long long rq = rin ? (long long)gy * W : 0;
      for (int i = lane; i < RX; i += 32) {
        const int gx = x_org - R + i;
        const bool in = rin && gx >= 0 && gx < W;
        const long long q = in ? rq + gx : 0;
        cp_async_elem_zfill(rg + j * PX + i, vb0 + q, in);
        cp_async_elem_zfill(rg + S::CS + j * PX + i, vb1 + q, in);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }

  // prefetch the epilogue operands into rg's tail while pass 2 runs
  auto prefetch = [&]() {
    if (a.use_tma) {
      if (tid == 0) {
        // WAR across proxies: pass 1 read this smem through the generic proxy
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(bar + 1, (unsigned)(sizeof(T) * OXY * (REG ? 5 : 4)));
        const int xa = x_org - offE;
        tma_load_3d(tail0, &maps.I, xa, y_org, b, bar + 1);
        tma_load_3d(tail0 + OXY, &maps.z, xa, y_org, b, bar + 1);
        tma_load_3d(tail0 + 2 * OXY, &maps.op2, xa, y_org, REG ? 2 * b : b, bar + 1);
        tma_load_3d(tail0 + 3 * OXY, &maps.zb, xa, y_org, b, bar + 1);
        if (REG) tma_load_3d(tail0 + 4 * OXY, &maps.op2, xa, y_org, 2 * b + 1, bar + 1);
      }
      return;
    }
    const T* src2 = REG ? a.v0 + b * 2 * N : a.ib + b * N;
    const T* src4 = REG ? a.v0 + b * 2 * N + N : nullptr;
    for (int j = warp; j < OY; j += kNW) {
      const int gy = y_org + j;
      const bool rin = gy >= 0 && gy < H;
      const long long rq = rin ? (long long)gy * W : 0;
      for (int i = lane; i < OX; i += 32) {
        const int gx = x_org + i;
        const bool in = rin && gx >= 0 && gx < W;
        const long long q = in ? rq + gx : 0;
        const int p = j * OXP + i;
        cp_async_elem_zfill(tail + p, I + q, in);
        cp_async_elem_zfill(tail + OXY + p, z + q, in);
        cp_async_elem_zfill(tail + 2 * OXY + p, src2 + q, in);
        cp_async_elem_zfill(tail + 3 * OXY + p, a.zb + b * N + q, in);
        if (REG) cp_async_elem_zfill(tail + 4 * OXY + p, src4 + q, in);
      }
    }
    cp_async_commit();
  };
  const T* res = fir2d_passes<T, R, 2, true>(rg, vt, tp, x_org, y_org, H, W, prefetch);
  if (a.use_tma) {
    mbar_wait(bar + 1, 0);
  } else {
    cp_async_wait_all();
  }
  __syncthreads();

  const T* tI = tail;
  const T* tz = tail + OXY;
  const T* t2 = tail + 2 * OXY;
  const T* tzb = tail + 3 * OXY;
  const T* t4 = tail + 4 * OXY;
  unsigned bad = 0;
  // tile interior: every owner has both neighbours on both axes and no edge
  // terms of the stencil transpose -> branch-free (bitwise-identical) formulas
  const bool interior = !REG && y_org + 1 >= 2 && y_org + OY - 2 <= H - 3 && x_org + 1 >= 2 &&
                        x_org + OX - 2 <= W - 3;
  if (interior) {
    for (int j = 1 + warp; j < OY - 1; j += kNW)
      for (int i = 1 + lane; i < OX - 1; i += 32) {
        const long long q = (long long)(y_org + j) * W + (x_org + i);
        const int e = j * OXP + i;
        const T g0 = (tI[e + OXP] - tI[e - OXP]) / T(2);
        const T g1 = (tI[e + 1] - tI[e - 1]) / T(2);
        const T m0 = -res[j * OP + i];
        const T m1 = -res[(OY + j) * OP + i];
        a.zb[b * N + q] = tzb[e] + (m0 * g0 + m1 * g1);
        if (a.zero_a) {
          a.zero_a[b * N + q] = T(0);
          a.zero_b[b * N + q] = T(0);
        }
        // G^T(mbar z): 0.5 q[j-1] - 0.5 q[j+1] per axis (fields.py:148-158)
        const T gm = -res[(j - 1) * OP + i] * tz[e - OXP];
        const T gp = -res[(j + 1) * OP + i] * tz[e + OXP];
        const T hm = -res[(OY + j) * OP + i - 1] * tz[e - 1];
        const T hp = -res[(OY + j) * OP + i + 1] * tz[e + 1];
        const T t0 = T(0.5) * gm - T(0.5) * gp;
        const T t1 = T(0.5) * hm - T(0.5) * hp;
        a.ib[b * N + q] = t2[e] + (t0 + t1);
      }
  } else
  for (int j = 1 + warp; j < OY - 1; j += kNW)
  for (int i = 1 + lane; i < OX - 1; i += 32) {
    const int gy = y_org + j, gx = x_org + i;
    if (gy >= H || gx >= W) continue;
    long long q = (long long)gy * W + gx;
    const int e = j * OXP + i;
    const T c = tI[e];
    const T g0 = grad1(tI[e - OXP], c, tI[e + OXP], gy, H);
    const T g1 = grad1(tI[e - 1], c, tI[e + 1], gx, W);
    const T m0 = -res[j * OP + i];
    const T m1 = -res[(OY + j) * OP + i];
    T zb_new = tzb[e] + (m0 * g0 + m1 * g1);  // objective.py:159
    if (REG) {
      // + lam*(K m0 . grad I0 + 2 rho z0) with K m0 = -v0 (objective.py:165-169)
      T km = -(t2[e] * g0 + t4[e] * g1);
      zb_new = zb_new + a.lam * (km + a.two_rho * tz[e]);
      a.zout[b * N + q] = zb_new;
      bad |= isfinite(zb_new) ? 0u : 1u;
    } else {
      a.zb[b * N + q] = zb_new;
      if (a.zero_a) {
        a.zero_a[b * N + q] = T(0);
        a.zero_b[b * N + q] = T(0);
      }
      // ib += G^T(mbar z) (objective.py:160-161), gather form on q_c = mbar_c * z
      auto q0 = [&](int jr) { return -res[jr * OP + i] * tz[jr * OXP + i]; };
      auto q1 = [&](int ic) { return -res[(OY + j) * OP + ic] * tz[j * OXP + ic]; };
      const T zc = tz[e];
      const T qc0 = m0 * zc, qc1 = m1 * zc;
      const T gm = (gy > 0) ? q0(j - 1) : T(0);
      const T gp = (gy < H - 1) ? q0(j + 1) : T(0);
      const T gf = (gy == 0) ? qc0 : ((gy == 1) ? gm : T(0));
      const T gl = (gy == H - 1) ? qc0 : ((gy == H - 2) ? gp : T(0));
      const T t0 = diff_adj1(gm, gp, gf, gl, gy, H);
      const T hm = (gx > 0) ? q1(i - 1) : T(0);
      const T hp = (gx < W - 1) ? q1(i + 1) : T(0);
      const T hf = (gx == 0) ? qc1 : ((gx == 1) ? hm : T(0));
      const T hl = (gx == W - 1) ? qc1 : ((gx == W - 2) ? hp : T(0));
      const T t1 = diff_adj1(hm, hp, hf, hl, gx, W);
      a.ib[b * N + q] = t2[e] + (t0 + t1);
    }
  }
  if (REG) {
    unsigned all = __reduce_or_sync(0xffffffffu, bad);
    if (all && (threadIdx.x & 31) == 0) atomicOr(reinterpret_cast<int*>(a.flags + b), 1);
  }
}

// ------------------------------------------------------------------------------
// K4 split path, second kernel (fp32): the axis-0 transposed FIR already ran over
// whole columns (k_fir_axis0_f32, no halo FLOPs) into a.vbar; this kernel stages
// OY rows x (OX + 2R) columns of it by TMA (zero fill = the transpose's zero
// padding along axis 1), copies them to the odd-pitch pass-2 buffer, runs the
// axis-1 transposed FIR (fir2d_pass2) and the same epilogue as k_velocity_adj2d.
// The owner operands zb, ib | v0 come from global memory into registers while
// the FIR runs; I and z tiles (neighbours needed) arrive by TMA.
// ------------------------------------------------------------------------------
template <int R>
struct VelAdjHSmem {
  using S = FirSmem<float, R, 2>;
  static constexpr int CSH = round_up(S::OY * S::PX, 32);    // staged rows per component
  static constexpr int stage = round_up(2 * CSH + S::A, 32);
  static constexpr int OXP = S::OX + S::A;                   // epilogue box width
  static constexpr int OXY = round_up(OXP * S::OY, 32);
  static constexpr int res = round_up(2 * S::OY * S::OP, 32);  // res at the start of rg
  static constexpr int rg = stage > res + 2 * OXY + S::A ? stage : res + 2 * OXY + S::A;
  static constexpr size_t head = 128;
  static constexpr size_t bytes = head + sizeof(float) * (size_t)(rg + S::vt);
};

template <int R, bool REG>
__global__ void __launch_bounds__(kThreads)
    k_velocity_adj2d_h(VelAdjArgs<float> a, Taps<float> tp, const __grid_constant__ VelAdjMaps maps) {
  using T = float;
  using S = FirSmem<T, R, 2>;
  using V = VelAdjHSmem<R>;
  constexpr int OX = S::OX, OY = S::OY, OP = S::OP, RX = S::RX, PX = S::PX, VP = S::VP,
                OXP = V::OXP, OXY = V::OXY, CSH = V::CSH;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* rg0 = reinterpret_cast<T*>(smem_raw + V::head);
  T* vt = rg0 + V::rg;
  T* res = rg0;                 // [2][OY][OP] after the copy
  T* tail0 = rg0 + V::res;      // [2][OY][OXP]: I, z
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x_org = blockIdx.x * (OX - 2) - 1, y_org = blockIdx.y * (OY - 2) - 1;
  const int offV = align_shift(x_org - R, S::A), offE = align_shift(x_org, S::A);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(T) * 2 * PX * OY));
    tma_load_3d(rg0, &maps.vbar, x_org - R - offV, y_org, 2 * b, bar);
    tma_load_3d(rg0 + CSH, &maps.vbar, x_org - R - offV, y_org, 2 * b + 1, bar);
  }
  // owner operands into registers while the tile arrives and the FIR runs
  constexpr int NJ = (OY - 2 + kNW - 1) / kNW, NI = (OX - 2 + 31) / 32;
  T pre_a[NJ][NI], pre_b[NJ][NI], pre_c[NJ][NI];
  const T* __restrict__ zb_p = a.zb + b * N;
  const T* __restrict__ o2_p = REG ? a.v0 + b * 2 * N : a.ib + b * N;
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
    for (int ii = 0; ii < NI; ++ii) {
      const int j = 1 + warp + jj * kNW, i = 1 + lane + ii * 32;
      const int gy = y_org + j, gx = x_org + i;
      const bool ok = j < OY - 1 && i < OX - 1 && gy < H && gx < W;
      const int q = ok ? gy * W + gx : 0;  // < N < 2^31 per pair
      pre_a[jj][ii] = ok ? zb_p[q] : T(0);
      pre_b[jj][ii] = ok ? o2_p[q] : T(0);
      pre_c[jj][ii] = (REG && ok) ? o2_p[N + q] : T(0);
    }
  __syncthreads();
  mbar_wait(bar, 0);
  // staged rows -> odd-pitch pass-2 input vt [2][OY][VP] (consecutive lanes on both
  // sides: conflict-free loads and stores)
  for (int rc = warp; rc < 2 * OY; rc += kNW) {
    const int r = rc >> 1, c = rc & 1;
    const T* srow = rg0 + c * CSH + r * PX + offV;
    T* vrow = vt + (c * OY + r) * VP;
#pragma unroll
    for (int i = lane; i < RX; i += 32) vrow[i] = srow[i];
  }
  __syncthreads();
  if (tid == 0) {  // I and z tiles of the epilogue into the freed staging area
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(bar + 1, (unsigned)(sizeof(T) * OXP * OY * 2));
    const int xa = x_org - offE;
    tma_load_3d(tail0, &maps.I, xa, y_org, b, bar + 1);
    tma_load_3d(tail0 + OXY, &maps.z, xa, y_org, b, bar + 1);
  }
  fir2d_pass2<T, R, 2, true>(vt, res, tp, x_org, W);
  mbar_wait(bar + 1, 0);
  __syncthreads();

  const T* tI = tail0 + offE;
  const T* tz = tI + OXY;
  T* __restrict__ zb_o = a.zb + b * N;
  T* __restrict__ ib_o = a.ib + b * N;
  unsigned bad = 0;
  const bool interior = !REG && y_org + 1 >= 2 && y_org + OY - 2 <= H - 3 && x_org + 1 >= 2 &&
                        x_org + OX - 2 <= W - 3;
  if (interior) {
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
      for (int ii = 0; ii < NI; ++ii) {
        const int j = 1 + warp + jj * kNW, i = 1 + lane + ii * 32;
        if (j >= OY - 1 || i >= OX - 1) continue;
        const int q = (y_org + j) * W + (x_org + i);
        const int e = j * OXP + i;
        const T g0 = (tI[e + OXP] - tI[e - OXP]) / T(2);
        const T g1 = (tI[e + 1] - tI[e - 1]) / T(2);
        const T m0 = -res[j * OP + i];
        const T m1 = -res[(OY + j) * OP + i];
        zb_o[q] = pre_a[jj][ii] + (m0 * g0 + m1 * g1);  // objective.py:159
        if (a.zero_a) {
          a.zero_a[b * N + q] = T(0);
          a.zero_b[b * N + q] = T(0);
        }
        // G^T(mbar z): 0.5 q[j-1] - 0.5 q[j+1] per axis (fields.py:148-158)
        const T gm = -res[(j - 1) * OP + i] * tz[e - OXP];
        const T gp = -res[(j + 1) * OP + i] * tz[e + OXP];
        const T hm = -res[(OY + j) * OP + i - 1] * tz[e - 1];
        const T hp = -res[(OY + j) * OP + i + 1] * tz[e + 1];
        const T t0 = T(0.5) * gm - T(0.5) * gp;
        const T t1 = T(0.5) * hm - T(0.5) * hp;
        ib_o[q] = pre_b[jj][ii] + (t0 + t1);
      }
  } else {
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
      for (int ii = 0; ii < NI; ++ii) {
        const int j = 1 + warp + jj * kNW, i = 1 + lane + ii * 32;
        const int gy = y_org + j, gx = x_org + i;
        if (j >= OY - 1 || i >= OX - 1 || gy >= H || gx >= W) continue;
        const int q = gy * W + gx;
        const int e = j * OXP + i;
        const T c = tI[e];
        const T g0 = grad1(tI[e - OXP], c, tI[e + OXP], gy, H);
        const T g1 = grad1(tI[e - 1], c, tI[e + 1], gx, W);
        const T m0 = -res[j * OP + i];
        const T m1 = -res[(OY + j) * OP + i];
        T zb_new = pre_a[jj][ii] + (m0 * g0 + m1 * g1);  // objective.py:159
        if (REG) {
          // + lam*(K m0 . grad I0 + 2 rho z0) with K m0 = -v0 (objective.py:165-169)
          const T km = -(pre_b[jj][ii] * g0 + pre_c[jj][ii] * g1);
          zb_new = zb_new + a.lam * (km + a.two_rho * tz[e]);
          a.zout[b * N + q] = zb_new;
          bad |= isfinite(zb_new) ? 0u : 1u;
        } else {
          zb_o[q] = zb_new;
          if (a.zero_a) {
            a.zero_a[b * N + q] = T(0);
            a.zero_b[b * N + q] = T(0);
          }
          auto q0 = [&](int jr) { return -res[jr * OP + i] * tz[jr * OXP + i]; };
          auto q1 = [&](int ic) { return -res[(OY + j) * OP + ic] * tz[j * OXP + ic]; };
          const T zc = tz[e];
          const T qc0 = m0 * zc, qc1 = m1 * zc;
          const T gm = (gy > 0) ? q0(j - 1) : T(0);
          const T gp = (gy < H - 1) ? q0(j + 1) : T(0);
          const T gf = (gy == 0) ? qc0 : ((gy == 1) ? gm : T(0));
          const T gl = (gy == H - 1) ? qc0 : ((gy == H - 2) ? gp : T(0));
          const T t0 = diff_adj1(gm, gp, gf, gl, gy, H);
          const T hm = (gx > 0) ? q1(i - 1) : T(0);
          const T hp = (gx < W - 1) ? q1(i + 1) : T(0);
          const T hf = (gx == 0) ? qc1 : ((gx == 1) ? hm : T(0));
          const T hl = (gx == W - 1) ? qc1 : ((gx == W - 2) ? hp : T(0));
          const T t1 = diff_adj1(hm, hp, hf, hl, gx, W);
          ib_o[q] = pre_b[jj][ii] + (t0 + t1);
        }
      }
  }
  if (REG) {
    unsigned all = __reduce_or_sync(0xffffffffu, bad);
    if (all && lane == 0) atomicOr(reinterpret_cast<int*>(a.flags + b), 1);
  }
}

// ------------------------------------------------------------------------------
// K1 split path, first kernel (fp32): m = z grad I (gradient_arr, fields.py:161-162)
// fused with the axis-1 pass of smooth_vec_arr (kernel.py:82-85, axis 1 first).
// TMA stages I (rows y_org-1 .. y_org+OY, cols x_org-R-1 .. x_org+OX+R) and z
// (rows y_org .. y_org+OY-1, cols x_org-R .. x_org+OX+R-1); the product is formed
// at the CLAMPED column (replicate border of conv1d_replicate, kernel.py:43-44),
// whose stencil always lies inside the staged box, straight into the odd-pitch
// pass-2 buffer; fir2d_pass2 filters the rows and the tile goes to `out`
// [B][2][H][W].  k_fir_axis0_f32<R, false, 1> then runs the axis-0 pass over
// whole columns (negate + velocity guard).  FIR work 2(2R+1) FFMA per pixel.
// ------------------------------------------------------------------------------
template <int R>
struct VelHSmem {
  using S = FirSmem<float, R, 2>;
  static constexpr int OY = S::OY, RX = S::RX;
  static constexpr int PXI = round_up(RX + 2 + S::A - 1, S::A);  // I box width
  static constexpr int PXZ = round_up(RX + S::A - 1, S::A);      // z box width
  static constexpr int IS = round_up((OY + 2) * PXI, 32);
  static constexpr int ZS = round_up(OY * PXZ, 32);
  static constexpr int resn = round_up(2 * OY * S::OP, 32);
  static constexpr int rg = IS + ZS > resn ? IS + ZS : resn;
  static constexpr size_t head = 128;
  static constexpr size_t bytes = head + sizeof(float) * (size_t)(rg + S::vt);
};

template <int R>
__global__ void __launch_bounds__(kThreads)
    k_velocity2d_h(VelArgs<float> a, Taps<float> tp, const __grid_constant__ CUtensorMap mI,
                   const __grid_constant__ CUtensorMap mZ, float* __restrict__ out) {
  using T = float;
  using S = FirSmem<T, R, 2>;
  using V = VelHSmem<R>;
  constexpr int OX = S::OX, OY = S::OY, OP = S::OP, RX = S::RX, VP = S::VP, PXI = V::PXI,
                PXZ = V::PXZ;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* rg0 = reinterpret_cast<T*>(smem_raw + V::head);
  T* sI = rg0;
  T* sZ = rg0 + V::IS;
  T* vt = rg0 + V::rg;
  T* res = rg0;  // [2][OY][OP] once the product is formed
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x_org = blockIdx.x * OX, y_org = blockIdx.y * OY;
  const int xi = x_org - R - 1, xz = x_org - R;
  const int xi0 = xi - align_shift(xi, S::A), xz0 = xz - align_shift(xz, S::A);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(T) * (PXI * (OY + 2) + PXZ * OY)));
    tma_load_3d(sI, &mI, xi0, y_org - 1, b, bar);
    tma_load_3d(sZ, &mZ, xz0, y_org, b, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // region column i <-> image column x_org - R + i, evaluated at its clamped column
  // (warp <-> row, lanes <-> consecutive columns: conflict-free smem on both sides)
  const int warp = tid >> 5, lane = tid & 31;
  const bool interior = x_org - R >= 1 && x_org + OX + R <= W - 1 && y_org >= 1 &&
                        y_org + OY <= H - 1;
  if (interior) {  // no clamps, central differences everywhere
#pragma unroll
    for (int r = warp; r < OY; r += kNW) {
      const T* pI = sI + (r + 1) * PXI + (x_org - R - xi0);
      const T* pZ = sZ + r * PXZ + (x_org - R - xz0);
#pragma unroll
      for (int i = lane; i < RX; i += 32) {
        const T g0 = (pI[i + PXI] - pI[i - PXI]) * T(0.5);
        const T g1 = (pI[i + 1] - pI[i - 1]) * T(0.5);
        const T zz = pZ[i];
        vt[r * VP + i] = zz * g0;
        vt[(OY + r) * VP + i] = zz * g1;
      }
    }
  } else {
    for (int r = warp; r < OY; r += kNW) {
      const int gy = y_org + r;
#pragma unroll
      for (int i = lane; i < RX; i += 32) {
        T m0 = T(0), m1 = T(0);
        if (gy < H) {
          const int gx = min(max(x_org - R + i, 0), W - 1);
          const T* pI = sI + (r + 1) * PXI + (gx - xi0);
          const T c = pI[0];
          const T g0 = grad1(pI[-PXI], c, pI[PXI], gy, H);
          const T g1 = grad1(pI[-1], c, pI[1], gx, W);
          const T zz = sZ[r * PXZ + (gx - xz0)];
          m0 = zz * g0;
          m1 = zz * g1;
        }
        vt[r * VP + i] = m0;
        vt[(OY + r) * VP + i] = m1;
      }
    }
  }
  __syncthreads();
  fir2d_pass2<T, R, 2, false>(vt, res, tp, x_org, W);
  __syncthreads();
  T* __restrict__ o = out + (long long)b * 2 * N + (long long)y_org * W + x_org;
  if (interior || (x_org + OX <= W && y_org + OY <= H)) {
#pragma unroll
    for (int rc = warp; rc < 2 * OY; rc += kNW) {
      const int c = rc / OY, r = rc - c * OY;
#pragma unroll
      for (int i = lane; i < OX; i += 32) o[c * N + (long long)r * W + i] = res[rc * OP + i];
    }
  } else {
    for (int rc = warp; rc < 2 * OY; rc += kNW) {
      const int c = rc / OY, r = rc - c * OY;
      if (y_org + r >= H) continue;
#pragma unroll
      for (int i = lane; i < OX; i += 32)
        if (x_org + i < W) o[c * N + (long long)r * W + i] = res[rc * OP + i];
    }
  }
}

// ------------------------------------------------------------------------------
// K5: cost terms (objective.py:64-88, fields.py:291-295, kernel.py:103-108)
// ------------------------------------------------------------------------------
template <typename T>
struct CostArgs {
  const T* I0;
  const T* z0;
  const T* v0;
  const T* IT;
  const T* J;
  T* seed;  // nullable: I_T - J
  double* part;  // [B][gridDim.x][4]: per-block {-, data, v.m, z.z} (reduced by k_finalize_terms)
  Grid2 g;
};

static __device__ __forceinline__ double block_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;  // valid on thread 0
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_cost_terms2d(CostArgs<T> a) {
  __shared__ double red[kThreads / 32];
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.y;
  const T* __restrict__ I0 = a.I0 + b * N;
  const T* __restrict__ z0 = a.z0 + b * N;
  const T* __restrict__ w0 = a.v0 + b * 2 * N;
  const T* __restrict__ IT = a.IT + b * N;
  const T* __restrict__ J = a.J + b * N;
  double data = 0.0, vn = 0.0, zn = 0.0;
  // warp <-> row, lanes <-> consecutive columns (no per-element index division)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fp32 rows whose layout allows it: 4 consecutive pixels per lane, float4 loads, the
  // row's loads issued together (the scalar loop below is latency-bound: one dependent
  // round trip per 32 pixels)
  bool vec = false;
  if constexpr (sizeof(T) == 4) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    vec = (W & 3) == 0 && (N & 3) == 0 && al(a.I0) && al(a.z0) && al(a.v0) && al(a.IT) && al(a.J) &&
          (!a.seed || al(a.seed));
  }
  for (int y = blockIdx.x * kNW + warp; y < H; y += gridDim.x * kNW) {
    if constexpr (sizeof(T) == 4) {
      if (vec) {
        const int row = y * W;
        const int rup = (y > 0 ? y - 1 : y) * W, rdn = (y < H - 1 ? y + 1 : y) * W;
        const float cgy = (y == 0 || y == H - 1) ? 1.f : 0.5f;  // one-sided rows: up / dn == c there
#pragma unroll 4
        for (int x = 4 * lane; x < W; x += 128) {
          const float4 it = *reinterpret_cast<const float4*>(IT + row + x);
          const float4 jj = *reinterpret_cast<const float4*>(J + row + x);
          const float4 c = *reinterpret_cast<const float4*>(I0 + row + x);
          const float4 up = *reinterpret_cast<const float4*>(I0 + rup + x);
          const float4 dn = *reinterpret_cast<const float4*>(I0 + rdn + x);
          const float4 zz = *reinterpret_cast<const float4*>(z0 + row + x);
          const float4 wa = *reinterpret_cast<const float4*>(w0 + row + x);
          const float4 wb = *reinterpret_cast<const float4*>(w0 + N + row + x);
          const float lf = x > 0 ? I0[row + x - 1] : c.x, rt = x + 4 < W ? I0[row + x + 4] : c.w;
          const float d4[4] = {it.x - jj.x, it.y - jj.y, it.z - jj.z, it.w - jj.w};
          if (a.seed)
            *reinterpret_cast<float4*>(a.seed + b * N + row + x) = make_float4(d4[0], d4[1], d4[2], d4[3]);
          const float cv[6] = {lf, c.x, c.y, c.z, c.w, rt};
          const float g0[4] = {(dn.x - up.x) * cgy, (dn.y - up.y) * cgy, (dn.z - up.z) * cgy,
                               (dn.w - up.w) * cgy};
          const float zv[4] = {zz.x, zz.y, zz.z, zz.w};
          const float av[4] = {wa.x, wa.y, wa.z, wa.w}, bv[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int gx = x + p;
            const float g1 = gx == 0 ? cv[p + 2] - cv[p + 1]
                                     : (gx == W - 1 ? cv[p + 1] - cv[p] : (cv[p + 2] - cv[p]) * 0.5f);
            data += (double)d4[p] * (double)d4[p];
            vn += (double)(zv[p] * g0[p]) * (double)av[p] + (double)(zv[p] * g1) * (double)bv[p];
            zn += (double)zv[p] * (double)zv[p];
          }
        }
        continue;
      }
    }
    for (int x = lane; x < W; x += 32) {
      const long long q = (long long)y * W + x;
      T diff = IT[q] - J[q];
      if (a.seed) a.seed[b * N + q] = diff;
      data += (double)diff * (double)diff;
      T g0, g1;
      grad2(I0, y, x, H, W, g0, g1);
      T zz = z0[q];
      vn += (double)(zz * g0) * (double)w0[q] + (double)(zz * g1) * (double)w0[N + q];
      zn += (double)zz * (double)zz;
    }
  }
  // per-block partials, reduced in block order by k_finalize_terms (deterministic:
  // no floating-point atomics, so the cost is the same bits on every run)
  double* out = a.part + ((long long)b * gridDim.x + blockIdx.x) * 4;
  double s;
  s = block_sum(data, red);
  if (threadIdx.x == 0) out[1] = s;
  s = block_sum(vn, red);
  if (threadIdx.x == 0) out[2] = s;
  s = block_sum(zn, red);
  if (threadIdx.x == 0) out[3] = s;
}

// terms[b] = {total, 0.5 sum data, -sum v.m, sum z.z} from nblk partials per pair,
// summed in block order; part may alias terms when nblk == 1.
static __global__ void k_finalize_terms(double* terms, const double* part, int nblk, int B,
                                        double lam, double rho) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    double d = 0.0, vn = 0.0, zn = 0.0;
    for (int k = 0; k < nblk; ++k) {
      const double* p = part + ((long long)b * nblk + k) * 4;
      d += p[1];
      vn += p[2];
      zn += p[3];
    }
    double* t = terms + b * 4;
    t[1] = 0.5 * d;
    t[2] = -vn;
    t[3] = zn;
    t[0] = t[1] + lam * (t[2] + rho * t[3]);  // objective.py:87
  }
}

}  // namespace mr
