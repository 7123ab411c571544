// mr_transport2d.cuh -- TMA-staged semi-Lagrangian transport step (2D), K2.
//
// integrator.py:101-110, 193-205 on a TX x TY tile: the tile plus a HB-pixel
// halo of I and z and a 1-pixel halo of v arrive by TMA (bulk, all in flight),
// then every bilinear gather (fields.py:235-240) whose four corners lie inside
// the staged window reads shared memory; feet outside the window (per-step
// back-trace longer than HB) fall back to global loads.  Same arithmetic as
// k_sl_step2d.
#pragma once

#include "mr_kernels2d.cuh"

namespace mr {

template <typename T>
struct TrCfg {
  static constexpr int TX = 64, TY = 16, HB = 4;  // tile, gather halo
  static constexpr int A = 16 / (int)sizeof(T);
  static constexpr int GX = round_up(TX + 2 * HB + A - 1, A);  // I/z box width
  static constexpr int GY = TY + 2 * HB;
  static constexpr int VX = round_up(TX + 2 + A - 1, A);       // v box width
  static constexpr int VY = TY + 2;
  static constexpr int nG = round_up(GX * GY, 32);
  static constexpr int nV = round_up(VX * VY, 32);
  static constexpr size_t head = 128;
  static constexpr size_t bytes = head + sizeof(T) * (size_t)(2 * nG + 2 * nV);
  static constexpr int PIX = TY * TX / kThreads;  // pixels per thread
};

struct StepMaps {
  CUtensorMap I, z, v;  // v: dims (W, H, 2B)
};

template <typename T>
__global__ void __launch_bounds__(kThreads)
    k_sl_step2d_tma(StepArgs<T> a, const __grid_constant__ StepMaps maps) {
  using C = TrCfg<T>;
  constexpr int TX = C::TX, TY = C::TY, HB = C::HB, GX = C::GX, VX = C::VX;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* sI0 = reinterpret_cast<T*>(smem_raw + C::head);
  T* sz0 = sI0 + C::nG;
  T* sv00 = sz0 + C::nG;
  T* sv10 = sv00 + C::nV;
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int gx0 = x0 - HB, gy0 = y0 - HB;  // window origin (image coords)
  const int offG = align_shift(gx0, C::A), offV = align_shift(x0 - 1, C::A);
  const T* sI = sI0 + offG;  // window element (r, c) at sI[r*GX + c]
  const T* sz = sz0 + offG;
  const T* sv0 = sv00 + offV;  // v element (r, c) of rows y0-1.., cols x0-1..
  const T* sv1 = sv10 + offV;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(T) * (2 * GX * C::GY + 2 * VX * C::VY)));
    tma_load_3d(sI0, &maps.I, gx0 - offG, gy0, b, bar);
    tma_load_3d(sz0, &maps.z, gx0 - offG, gy0, b, bar);
    tma_load_3d(sv00, &maps.v, x0 - 1 - offV, y0 - 1, 2 * b, bar);
    tma_load_3d(sv10, &maps.v, x0 - 1 - offV, y0 - 1, 2 * b + 1, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);

  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  unsigned fin = 0, fout = 0;
  constexpr int CPR = TX / 32;  // column chunks per row
#pragma unroll
  for (int k = 0; k < C::PIX; ++k) {
    const int tx = (threadIdx.x & 31) + 32 * (k % CPR);
    const int ty = (threadIdx.x >> 5) + (k / CPR) * (kThreads / 32);
    const int x = x0 + tx, y = y0 + ty;
    if (x >= W || y >= H) continue;
    const long long q = (long long)y * W + x;
    const int vi = (ty + 1) * VX + tx + 1;
    const T vy = sv0[vi], vx = sv1[vi];
    const AxisPlan<T> py = plan_axis<T>(y, vy, a.dt, H);
    const AxisPlan<T> px = plan_axis<T>(x, vx, a.dt, W);
    const int ry = py.i0 - gy0, rx = px.i0 - gx0;  // window coords of corner 00
    T ia, ib2, ic, id, za, zb2, zc, zd;
    if (ry >= 0 && ry + 1 < C::GY && rx >= 0 && rx + 1 < TX + 2 * HB) {
      const int e = ry * GX + rx;
      ia = sI[e]; ib2 = sI[e + GX]; ic = sI[e + 1]; id = sI[e + GX + 1];
      za = sz[e]; zb2 = sz[e + GX]; zc = sz[e + 1]; zd = sz[e + GX + 1];
    } else {  // long back-trace: outside the staged window
      const long long c00 = (long long)py.i0 * W + px.i0;
      ia = I[c00]; ib2 = I[c00 + W]; ic = I[c00 + 1]; id = I[c00 + W + 1];
      za = z[c00]; zb2 = z[c00 + W]; zc = z[c00 + 1]; zd = z[c00 + W + 1];
    }
    const int ce = (ty + HB) * GX + tx + HB;  // own pixel in the window
    if (a.guard_in) {  // _guard(0, image, momentum) on the inputs (integrator.py:184)
      fin |= guard_bits(sI[ce], MR_GUARD_IMAGE_NONFINITE) |
             guard_bits(sz[ce], MR_GUARD_MOMENTUM_NONFINITE);
    }
    T bi = bilerp(ia, ib2, ic, id, py.f, px.f);
    if (a.has_mu) bi = bi + a.dtmu * sz[ce];  // advect_image_sl_arr: + dt*mu*z
    const T bz = bilerp(za, zb2, zc, zd, py.f, px.f);
    const T up = (y > 0) ? sv0[vi - VX] : vy;
    const T dn = (y < H - 1) ? sv0[vi + VX] : vy;
    const T lf = (x > 0) ? sv1[vi - 1] : vx;
    const T rt = (x < W - 1) ? sv1[vi + 1] : vx;
    const T div = grad1(up, vy, dn, y, H) + grad1(lf, vx, rt, x, W);  // fields.py:169-170
    const T zn = bz * (T(1) - a.dt * div);
    a.In[b * N + q] = bi;
    a.zn[b * N + q] = zn;
    fout |= guard_bits(bi, MR_GUARD_IMAGE_NONFINITE) | guard_bits(zn, MR_GUARD_MOMENTUM_NONFINITE);
    if (a.phi_in) {
      const long long c00 = (long long)py.i0 * W + px.i0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const T* __restrict__ ph = a.phi_in + (b * 2 + c) * N;
        a.phi_out[(b * 2 + c) * N + q] =
            bilerp(ph[c00], ph[c00 + W], ph[c00 + 1], ph[c00 + W + 1], py.f, px.f);
      }
    }
  }
  if (fin && a.guard_in)
    atomicOr(reinterpret_cast<int*>(a.guard_in + (long long)b * a.guard_stride), (int)fin);
  if (fout && a.guard_out)
    atomicOr(reinterpret_cast<int*>(a.guard_out + (long long)b * a.guard_stride), (int)fout);
}

}  // namespace mr
