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

#include <type_traits>

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
  T* __restrict__ In_b = a.In + b * N;  // per-pair bases: 32-bit pixel offsets below (N < 2^31)
  T* __restrict__ zn_b = a.zn + b * N;
  unsigned fin = 0, fout = 0;
  constexpr int CPR = TX / 32;  // column chunks per row
  // every tile pixel inside the image and at least 1 away from its edges: central
  // differences only, no per-pixel border selects (same operations, bitwise equal)
  const bool interior = y0 >= 1 && y0 + TY <= H - 1 && x0 >= 1 && x0 + TX <= W - 1;
  // the pixel loop, specialised at compile time on two block-uniform facts: `interior`
  // and `plain` (no input guard, no deformation grid: every step but the first of a shoot
  // without phi)
  auto sweep = [&](auto interior_tag, auto plain_tag) {
    constexpr bool INT = decltype(interior_tag)::value, PLAIN = decltype(plain_tag)::value;
  #pragma unroll
    for (int k = 0; k < C::PIX; ++k) {
      const int tx = (threadIdx.x & 31) + 32 * (k % CPR);
      const int ty = (threadIdx.x >> 5) + (k / CPR) * (kThreads / 32);
      const int x = x0 + tx, y = y0 + ty;
      if (!INT && (x >= W || y >= H)) continue;
      const int q = y * W + x;
      const int vi = (ty + 1) * VX + tx + 1;
      const T vy = sv0[vi], vx = sv1[vi];
      const AxisPlan<T> py = plan_axis<T>(y, vy, a.dt, H);
      const AxisPlan<T> px = plan_axis<T>(x, vx, a.dt, W);
      const int ry = py.i0 - gy0, rx = px.i0 - gx0;  // window coords of corner 00
      T ia, ib2, ic, id, za, zb2, zc, zd;
      if ((unsigned)ry < (unsigned)(C::GY - 1) && (unsigned)rx < (unsigned)(TX + 2 * HB - 1)) {
        const int e = ry * GX + rx;
        ia = sI[e]; ib2 = sI[e + GX]; ic = sI[e + 1]; id = sI[e + GX + 1];
        za = sz[e]; zb2 = sz[e + GX]; zc = sz[e + 1]; zd = sz[e + GX + 1];
      } else {  // long back-trace: outside the staged window
        const int c00 = py.i0 * W + px.i0;
        ia = I[c00]; ib2 = I[c00 + W]; ic = I[c00 + 1]; id = I[c00 + W + 1];
        za = z[c00]; zb2 = z[c00 + W]; zc = z[c00 + 1]; zd = z[c00 + W + 1];
      }
      const int ce = (ty + HB) * GX + tx + HB;  // own pixel in the window
      if (!PLAIN && a.guard_in) {  // _guard(0, image, momentum) on the inputs (integrator.py:184)
        fin |= guard_bits(sI[ce], MR_GUARD_IMAGE_NONFINITE) |
               guard_bits(sz[ce], MR_GUARD_MOMENTUM_NONFINITE);
      }
      T bi = bilerp(ia, ib2, ic, id, py.f, px.f);
      if (a.has_mu) bi = bi + a.dtmu * sz[ce];  // advect_image_sl_arr: + dt*mu*z
      const T bz = bilerp(za, zb2, zc, zd, py.f, px.f);
      T div;  // fields.py:169-170
      if (INT) {
        div = (sv0[vi + VX] - sv0[vi - VX]) / T(2) + (sv1[vi + 1] - sv1[vi - 1]) / T(2);
      } else {
        const T up = (y > 0) ? sv0[vi - VX] : vy;
        const T dn = (y < H - 1) ? sv0[vi + VX] : vy;
        const T lf = (x > 0) ? sv1[vi - 1] : vx;
        const T rt = (x < W - 1) ? sv1[vi + 1] : vx;
        div = grad1(up, vy, dn, y, H) + grad1(lf, vx, rt, x, W);
      }
      const T zn = bz * (T(1) - a.dt * div);
      In_b[q] = bi;
      zn_b[q] = zn;
      // guard: one comparison per output on the common path (NaN fails it too)
      if (!(fabs(bi) <= T(1e6)) || !(fabs(zn) <= T(1e6)))
        fout |= guard_bits(bi, MR_GUARD_IMAGE_NONFINITE) | guard_bits(zn, MR_GUARD_MOMENTUM_NONFINITE);
      if (!PLAIN && a.phi_in) {
        const long long c00 = (long long)py.i0 * W + px.i0;
  #pragma unroll
        for (int c = 0; c < 2; ++c) {
          const T* __restrict__ ph = a.phi_in + (b * 2 + c) * N;
          a.phi_out[(b * 2 + c) * N + q] =
              bilerp(ph[c00], ph[c00 + W], ph[c00 + 1], ph[c00 + W + 1], py.f, px.f);
        }
      }
    }
  };
  const bool plain = !a.guard_in && !a.phi_in;
  if (interior) {
    if (plain) sweep(std::true_type{}, std::true_type{});
    else sweep(std::true_type{}, std::false_type{});
  } else {
    if (plain) sweep(std::false_type{}, std::true_type{});
    else sweep(std::false_type{}, std::false_type{});
  }
  if (fin && a.guard_in)
    atomicOr(reinterpret_cast<int*>(a.guard_in + (long long)b * a.guard_stride), (int)fin);
  if (fout && a.guard_out)
    atomicOr(reinterpret_cast<int*>(a.guard_out + (long long)b * a.guard_stride), (int)fout);
}

}  // namespace mr

namespace mr {

// ---------------------------------------------------------------------------------
// TMA-staged adjoint of one SL step (objective.py:118-147), K3.  Window of I, z
// (HB halo, for the gathers) and of v, ibar, zbar (1-px halo: divergence, and the
// divergence-adjoint seed s on the tile's ring) staged by TMA; phase 1 computes s
// for owners and ring and issues the warp-merged scatters; phase 2 recomputes the
// (smem-cheap) plans and writes vbar with D^T s from shared memory.
// ---------------------------------------------------------------------------------
struct AdjMaps {
  CUtensorMap I, z, v, ibar, zbar;
};

template <typename T>
struct AdjCfg {
  using C = TrCfg<T>;
  static constexpr int nG = C::nG, nV = C::nV;
  static constexpr int nS = round_up((C::TY + 2) * (C::TX + 2), 32);
  static constexpr size_t bytes = C::head + sizeof(T) * (size_t)(2 * nG + 4 * nV + nS);
};

// Warp-merged scatter (scatter4_merged) with 32-bit keys (cell index within one pair < 2^31).
// Two fields scattered through the same four cells (ibar and the weighted zbar share the
// plan): one pair of key shuffles and one set of merge decisions for both.
template <typename T>
__device__ __forceinline__ void scatter4x2_merged32(T* __restrict__ out0, T* __restrict__ out1, int cell,
                                                    bool valid, int W, T wa, T wb, T wc, T wd, T s0,
                                                    T s1) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int key = valid ? cell : -4;
  const int prev_key = __shfl_up_sync(full, key, 1);
  const int next_key = __shfl_down_sync(full, key, 1);
  T a0 = wa * s0, b0 = wb * s0, a1 = wa * s1, b1 = wb * s1;
  const T c0 = wc * s0, d0 = wd * s0, c1 = wc * s1, d1 = wd * s1;
  const T pc0 = __shfl_up_sync(full, c0, 1), pd0 = __shfl_up_sync(full, d0, 1);
  const T pc1 = __shfl_up_sync(full, c1, 1), pd1 = __shfl_up_sync(full, d1, 1);
  if (!valid) return;
  if (lane > 0 && prev_key >= 0 && prev_key + 1 == key) {
    a0 += pc0;
    b0 += pd0;
    a1 += pc1;
    b1 += pd1;
  }
  atomicAdd(out0 + cell, a0);
  atomicAdd(out0 + cell + W, b0);
  atomicAdd(out1 + cell, a1);
  atomicAdd(out1 + cell + W, b1);
  if (!(lane < 31 && next_key >= 0 && key + 1 == next_key)) {
    atomicAdd(out0 + cell + 1, c0);
    atomicAdd(out0 + cell + W + 1, d0);
    atomicAdd(out1 + cell + 1, c1);
    atomicAdd(out1 + cell + W + 1, d1);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    k_sl_adjoint2d_tma(AdjArgs<T> a, const __grid_constant__ AdjMaps maps) {
  using C = TrCfg<T>;
  using AC = AdjCfg<T>;
  constexpr int TX = C::TX, TY = C::TY, HB = C::HB, GX = C::GX, VX = C::VX, SX = TX + 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* sI0 = reinterpret_cast<T*>(smem_raw + C::head);
  T* sz0 = sI0 + C::nG;
  T* sv00 = sz0 + C::nG;
  T* sv10 = sv00 + C::nV;
  T* sib0 = sv10 + C::nV;
  T* szb0 = sib0 + C::nV;
  T* s_div = szb0 + C::nV;  // [(TY+2)][(TX+2)], s = -dt * zbar * B(z)
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int gx0 = x0 - HB, gy0 = y0 - HB;
  const int offG = align_shift(gx0, C::A), offV = align_shift(x0 - 1, C::A);
  const T* sI = sI0 + offG;
  const T* sz = sz0 + offG;
  const T* sv0 = sv00 + offV;   // (r, c) <-> image (y0-1+r, x0-1+c)
  const T* sv1 = sv10 + offV;
  const T* sib = sib0 + offV;
  const T* szb = szb0 + offV;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_expect_tx(bar, (unsigned)(sizeof(T) * (2 * GX * C::GY + 4 * VX * C::VY)));
    tma_load_3d(sI0, &maps.I, gx0 - offG, gy0, b, bar);
    tma_load_3d(sz0, &maps.z, gx0 - offG, gy0, b, bar);
    tma_load_3d(sv00, &maps.v, x0 - 1 - offV, y0 - 1, 2 * b, bar);
    tma_load_3d(sv10, &maps.v, x0 - 1 - offV, y0 - 1, 2 * b + 1, bar);
    tma_load_3d(sib0, &maps.ibar, x0 - 1 - offV, y0 - 1, b, bar);
    tma_load_3d(szb0, &maps.zbar, x0 - 1 - offV, y0 - 1, b, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);

  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  const T dt = a.dt;
  // every tile pixel at least 2 away from the image edges: central stencils only
  const bool interior = y0 >= 2 && y0 + TY - 1 <= H - 3 && x0 >= 2 && x0 + TX - 1 <= W - 3;

  // corners of I or z at the foot of window pixel (r, c) (v-window coordinates)
  auto corners = [&](const T* sf, const T* __restrict__ gf, const AxisPlan<T>& py,
                     const AxisPlan<T>& px, T& ca, T& cb, T& cc, T& cd) {
    const int ry = py.i0 - gy0, rx = px.i0 - gx0;
    if (ry >= 0 && ry + 1 < C::GY && rx >= 0 && rx + 1 < TX + 2 * HB) {
      const int e = ry * GX + rx;
      ca = sf[e]; cb = sf[e + GX]; cc = sf[e + 1]; cd = sf[e + GX + 1];
    } else {
      const long long c00 = (long long)py.i0 * W + px.i0;
      ca = gf[c00]; cb = gf[c00 + W]; cc = gf[c00 + 1]; cd = gf[c00 + W + 1];
    }
  };

  // ---- s on the ring (1-px halo) ----
  constexpr int NRING = 2 * (TX + 2) + 2 * TY;
  for (int h = threadIdx.x; h < NRING; h += kThreads) {
    int j, i;
    if (h < TX + 2) { j = 0; i = h; }
    else if (h < 2 * (TX + 2)) { j = TY + 1; i = h - (TX + 2); }
    else { const int kk = h - 2 * (TX + 2); j = 1 + (kk >> 1); i = (kk & 1) ? TX + 1 : 0; }
    const int gy = y0 - 1 + j, gx = x0 - 1 + i;
    T sv = T(0);
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
      const int vi = j * VX + i;
      const AxisPlan<T> hy = plan_axis<T>(gy, sv0[vi], dt, H);
      const AxisPlan<T> hx = plan_axis<T>(gx, sv1[vi], dt, W);
      T za, zb2, zc, zd;
      corners(sz, z, hy, hx, za, zb2, zc, zd);
      sv = -dt * (szb[vi] * bilerp(za, zb2, zc, zd, hy.f, hx.f));
    }
    s_div[j * SX + i] = sv;
  }

  // The two sweeps over the tile's pixels, specialised at compile time on `interior`
  // (block-uniform): interior tiles carry no ownership predicates and no border stencils.
  auto sweeps = [&](auto interior_tag) {
    constexpr bool INT = decltype(interior_tag)::value;
    // ---- phase 1: per owner pixel the plans, corners, scatters, s, and the partial
    //      vbar (coordinate-gradient terms) kept in registers for phase 2 ----
    T* __restrict__ ibo = a.ib + b * N;
    T* __restrict__ zbo = a.zb + b * N;
    constexpr int CPR = TX / 32;
    T vbp0[C::PIX], vbp1[C::PIX];
  #pragma unroll
    for (int k = 0; k < C::PIX; ++k) {
      const int tx = (threadIdx.x & 31) + 32 * (k % CPR);
      const int ty = (threadIdx.x >> 5) + (k / CPR) * (kThreads / 32);
      const int x = x0 + tx, y = y0 + ty;
      const bool own = INT || (x < W && y < H);
      const int vi = (ty + 1) * VX + tx + 1;
      const T vy = sv0[vi], vx = sv1[vi];
      const AxisPlan<T> py = plan_axis<T>(own ? y : 0, vy, dt, H);
      const AxisPlan<T> px = plan_axis<T>(own ? x : 0, vx, dt, W);
      T ia = T(0), ib2 = T(0), ic = T(0), id = T(0);
      T za = T(0), zb2 = T(0), zc = T(0), zd = T(0);
      if (own) {  // both fields through one window test (same foot)
        const int ry = py.i0 - gy0, rx = px.i0 - gx0;
        if ((unsigned)ry < (unsigned)(C::GY - 1) && (unsigned)rx < (unsigned)(TX + 2 * HB - 1)) {
          const int e = ry * GX + rx;
          za = sz[e]; zb2 = sz[e + GX]; zc = sz[e + 1]; zd = sz[e + GX + 1];
          ia = sI[e]; ib2 = sI[e + GX]; ic = sI[e + 1]; id = sI[e + GX + 1];
        } else {
          const int c00 = py.i0 * W + px.i0;
          za = z[c00]; zb2 = z[c00 + W]; zc = z[c00 + 1]; zd = z[c00 + W + 1];
          ia = I[c00]; ib2 = I[c00 + W]; ic = I[c00 + 1]; id = I[c00 + W + 1];
        }
      }
      const T ib_ = sib[vi], zb_ = szb[vi];
      T scale = T(1);
      if (INT) {
        scale = T(1) - dt * ((sv0[vi + VX] - sv0[vi - VX]) / T(2) + (sv1[vi + 1] - sv1[vi - 1]) / T(2));
      } else if (own) {
        const T up = (y > 0) ? sv0[vi - VX] : vy;
        const T dn = (y < H - 1) ? sv0[vi + VX] : vy;
        const T lf = (x > 0) ? sv1[vi - 1] : vx;
        const T rt = (x < W - 1) ? sv1[vi + 1] : vx;
        scale = T(1) - dt * (grad1(up, vy, dn, y, H) + grad1(lf, vx, rt, x, W));
      }
      const T fy = py.f, fx = px.f, wy = T(1) - fy, wx = T(1) - fx;
      s_div[(ty + 1) * SX + tx + 1] = own ? -dt * (zb_ * (wy * wx * za + fy * wx * zb2 + wy * fx * zc + fy * fx * zd)) : T(0);
      const T wz = zb_ * scale;
      const int c00 = py.i0 * W + px.i0;
      scatter4x2_merged32(ibo, zbo, c00, own, W, wy * wx, fy * wx, wy * fx, fy * fx, ib_, wz);
      if (own && a.has_mu) atomicAdd(zbo + (long long)y * W + x, a.dtmu * ib_);  // :133
      // vbar = -dt (d/dy, d/dx)[P I] ibar - dt (d/dy, d/dx)[P z] w  (objective.py:131-132,143-145)
      const T ddy = (wx * (ib2 - ia) + fx * (id - ic)) * (py.inside ? T(1) : T(0));
      const T ddx = (wy * (ic - ia) + fy * (id - ib2)) * (px.inside ? T(1) : T(0));
      const T dzy = (wx * (zb2 - za) + fx * (zd - zc)) * (py.inside ? T(1) : T(0));
      const T dzx = (wy * (zc - za) + fy * (zd - zb2)) * (px.inside ? T(1) : T(0));
      vbp0[k] = -dt * ddy * ib_ + -dt * dzy * wz;
      vbp1[k] = -dt * ddx * ib_ + -dt * dzx * wz;
    }
    __syncthreads();

    // ---- phase 2: vbar += D^T s (objective.py:146-147), then the k = 0 fold ----
  #pragma unroll
    for (int k = 0; k < C::PIX; ++k) {
      const int tx = (threadIdx.x & 31) + 32 * (k % CPR);
      const int ty = (threadIdx.x >> 5) + (k / CPR) * (kThreads / 32);
      const int x = x0 + tx, y = y0 + ty;
      if (!INT && (x >= W || y >= H)) continue;
      T vb0 = vbp0[k], vb1 = vbp1[k];
      const int j = ty + 1, i = tx + 1;
      const T sm_ = s_div[(j - 1) * SX + i], sp_ = s_div[(j + 1) * SX + i];
      const T sl_ = s_div[j * SX + i - 1], sr_ = s_div[j * SX + i + 1];
      if (INT) {  // D^T s = 0.5 s[j-1] - 0.5 s[j+1] away from the edges
        vb0 += T(0.5) * sm_ - T(0.5) * sp_;
        vb1 += T(0.5) * sl_ - T(0.5) * sr_;
      } else {
        const T s_first_y = (y <= 1) ? s_div[(j - y) * SX + i] : T(0);
        const T s_last_y = (y >= H - 2) ? s_div[(j + (H - 1 - y)) * SX + i] : T(0);
        vb0 += diff_adj1(sm_, sp_, s_first_y, s_last_y, y, H);
        const T s_first_x = (x <= 1) ? s_div[j * SX + i - x] : T(0);
        const T s_last_x = (x >= W - 2) ? s_div[j * SX + i + (W - 1 - x)] : T(0);
        vb1 += diff_adj1(sl_, sr_, s_first_x, s_last_x, x, W);
      }
      const long long q = (long long)y * W + x;
      if (a.reg_lam != T(0)) {  // k = 0: fold -lam*m0
        const int ce = (ty + HB) * GX + tx + HB;
        const T c = sI[ce];
        const T g0 = grad1(sI[ce - GX], c, sI[ce + GX], y, H);
        const T g1 = grad1(sI[ce - 1], c, sI[ce + 1], x, W);
        const T zz = sz[ce];
        vb0 = vb0 - a.reg_lam * (zz * g0);
        vb1 = vb1 - a.reg_lam * (zz * g1);
      }
      a.vbar[b * 2 * N + q] = vb0;
      a.vbar[b * 2 * N + N + q] = vb1;
    }
  };
  if (interior) sweeps(std::true_type{});
  else sweeps(std::false_type{});
}

}  // namespace mr
