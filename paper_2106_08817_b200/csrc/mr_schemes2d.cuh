// mr_schemes2d.cuh -- Eulerian and Hybrid transport steps and their adjoints (2D),
// the two non-semi-Lagrangian branches of the reference's shooting scheme
// (Scheme, integrator.py:48-51):
//
//   forward  integrator.py:194-201
//     EULERIAN  I' = I + dt (-(grad I . v) + mu z)        advect_image_euler_arr :97-98
//               z' = z - dt div(z v)                      continuity_euler_arr   :105-106
//     HYBRID    I' = B(I) + dt mu z  (bilinear pull-back)  advect_image_sl_arr    :101-102
//               z' = z - dt div(z v)
//     both      phi' = B(phi)                              :202-205
//   adjoint  objective.py:118-155 (image branch :124-132, momentum branch :148-155)
//
// The velocity and its adjoint (K1/K4) are shared with the semi-Lagrangian
// path; these kernels replace K2/K3 only.  Every operand is a stencil or a
// 4-corner gather, so one pixel per thread with L1-cached neighbour loads
// (32 x 8 blocks, lanes along x) is the whole design; the Hybrid image adjoint
// reuses the warp-merged bilinear scatter of K3.
#pragma once

#include "mr_kernels2d.cuh"

namespace mr {

enum : int { kSchemeSL = 0, kSchemeEuler = 1, kSchemeHybrid = 2 };

// Gather form of axis_diff_adjoint (fields.py:148-158) of the field f(.) at index j
// of an axis with stride st and n samples (f evaluated only where it is needed).
template <typename T, class F>
__device__ __forceinline__ T diff_adj_gather(F f, long long q, long long st, int j, int n) {
  const T gm = j > 0 ? f(q - st) : T(0);
  const T gp = j < n - 1 ? f(q + st) : T(0);
  const T gc = (j == 0 || j == n - 1) ? f(q) : T(0);
  const T gf = j == 0 ? gc : (j == 1 ? gm : T(0));
  const T gl = j == n - 1 ? gc : (j == n - 2 ? gp : T(0));
  return diff_adj1(gm, gp, gf, gl, j, n);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_scheme_step2d(StepArgs<T> a, T mu, int scheme) {
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * kNW + (threadIdx.x >> 5);
  if (x >= W || y >= H) return;
  const long long q = (long long)y * W + x;
  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  const T* __restrict__ v0 = a.v + b * 2 * N;
  const T* __restrict__ v1 = v0 + N;
  const long long ym = y > 0 ? -(long long)W : 0, yp = y < H - 1 ? W : 0;
  const long long xm = x > 0 ? -1 : 0, xp = x < W - 1 ? 1 : 0;
  const T vy = v0[q], vx = v1[q], Ic = I[q], zc = z[q];
  const AxisPlan<T> py = plan_axis<T>(y, vy, a.dt, H);
  const AxisPlan<T> px = plan_axis<T>(x, vx, a.dt, W);
  const long long c00 = (long long)py.i0 * W + px.i0;
  T bi;
  if (scheme == kSchemeEuler) {  // i + dt * (-(grad_i * v).sum(-1) + mu * z)
    const T g0 = grad1(I[q + ym], Ic, I[q + yp], y, H);
    const T g1 = grad1(I[q + xm], Ic, I[q + xp], x, W);
    bi = Ic + a.dt * (-(g0 * vy + g1 * vx) + mu * zc);
  } else {  // bilinear_apply(i, plan) + dt * mu * z
    bi = bilerp(I[c00], I[c00 + W], I[c00 + 1], I[c00 + W + 1], py.f, px.f);
    if (a.has_mu) bi = bi + a.dtmu * zc;
  }
  // z - dt * divergence_arr(z[..., None] * v)
  const T d0 = grad1(z[q + ym] * v0[q + ym], zc * vy, z[q + yp] * v0[q + yp], y, H);
  const T d1 = grad1(z[q + xm] * v1[q + xm], zc * vx, z[q + xp] * v1[q + xp], x, W);
  const T zn = zc - a.dt * (d0 + d1);
  a.In[b * N + q] = bi;
  a.zn[b * N + q] = zn;
  if (a.guard_in) {  // _guard(0, image, momentum) on the inputs (integrator.py:184)
    const unsigned fin = guard_bits(Ic, MR_GUARD_IMAGE_NONFINITE) |
                         guard_bits(zc, MR_GUARD_MOMENTUM_NONFINITE);
    if (fin) atomicOr(reinterpret_cast<int*>(a.guard_in + (long long)b * a.guard_stride), (int)fin);
  }
  if (a.guard_out) {
    const unsigned fo = guard_bits(bi, MR_GUARD_IMAGE_NONFINITE) |
                        guard_bits(zn, MR_GUARD_MOMENTUM_NONFINITE);
    if (fo) atomicOr(reinterpret_cast<int*>(a.guard_out + (long long)b * a.guard_stride), (int)fo);
  }
  if (a.phi_in) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const T* __restrict__ ph = a.phi_in + (b * 2 + c) * N;
      a.phi_out[(b * 2 + c) * N + q] =
          bilerp(ph[c00], ph[c00 + W], ph[c00 + 1], ph[c00 + W + 1], py.f, px.f);
    }
  }
}

// Adjoint of one Eulerian / Hybrid step w.r.t. (I, z, v) before the velocity
// adjoint: writes vbar, zb_acc (pointwise) and ib_acc (EULERIAN: pointwise
// ibar + G^T(-dt v ibar); HYBRID: bilinear scatter into the zeroed ib_acc).  K4
// then adds zb += mbar . grad I and ib += G^T(mbar z) -- G^T is linear, so the
// reference's single G^T(grad_ibar) (objective.py:160-161) splits exactly.
template <typename T, bool DET = false>
__global__ void __launch_bounds__(kThreads) k_scheme_adj2d(AdjArgs<T> a, int scheme) {
  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * kNW + (threadIdx.x >> 5);
  const bool own = x < W && y < H;
  const int xo = own ? x : 0, yo = own ? y : 0;
  const long long q = (long long)yo * W + xo;
  const T* __restrict__ I = a.I + b * N;
  const T* __restrict__ z = a.z + b * N;
  const T* __restrict__ v0 = a.v + b * 2 * N;
  const T* __restrict__ v1 = v0 + N;
  const T* __restrict__ ibar = a.ibar + b * N;
  const T* __restrict__ zbar = a.zbar + b * N;
  const T dt = a.dt;
  const T vy = v0[q], vx = v1[q], zc = z[q], ib_ = ibar[q], zb_ = zbar[q];
  T g0, g1;
  grad2(I, yo, xo, H, W, g0, g1);
  T vb0, vb1;
  if (scheme == kSchemeEuler) {  // objective.py:124-127
    auto gb0 = [&](long long r) { return (-dt * v0[r]) * ibar[r]; };
    auto gb1 = [&](long long r) { return (-dt * v1[r]) * ibar[r]; };
    const T t0 = diff_adj_gather<T>(gb0, q, W, yo, H);
    const T t1 = diff_adj_gather<T>(gb1, q, 1, xo, W);
    if (own) a.ib[b * N + q] = ib_ + (t0 + t1);
    vb0 = -dt * g0 * ib_;
    vb1 = -dt * g1 * ib_;
  } else {  // HYBRID image: bilinear_adjoint_values + coordinate gradient (:129-132)
    const AxisPlan<T> py = plan_axis<T>(yo, vy, dt, H);
    const AxisPlan<T> px = plan_axis<T>(xo, vx, dt, W);
    const long long c00 = (long long)py.i0 * W + px.i0;
    const T ia = I[c00], ib2 = I[c00 + W], ic = I[c00 + 1], id = I[c00 + W + 1];
    const T fy = py.f, fx = px.f, wy = T(1) - fy, wx = T(1) - fx;
    if constexpr (DET) {
      unsigned ovf = 0;
      scatter4_merged_fix(a.qib + b * N, c00, own, (long long)W, fix_factor(a.mbits, b),
                          wy * wx * ib_, fy * wx * ib_, wy * fx * ib_, fy * fx * ib_, ovf);
      if (ovf) atomicOr(a.ovf, 1);
    } else {
      scatter4_merged(a.ib + b * N, c00, own, (long long)W, wy * wx * ib_, fy * wx * ib_,
                      wy * fx * ib_, fy * fx * ib_);
    }
    const T ddy = (wx * (ib2 - ia) + fx * (id - ic)) * (py.inside ? T(1) : T(0));
    const T ddx = (wy * (ic - ia) + fy * (id - ib2)) * (px.inside ? T(1) : T(0));
    vb0 = -dt * ddy * ib_;
    vb1 = -dt * ddx * ib_;
  }
  if (!own) return;
  // momentum, non-SL branch (objective.py:148-155): zb = dt mu ibar + zbar + qb . v
  auto sd = [&](long long r) { return -dt * zbar[r]; };
  const T q0b = diff_adj_gather<T>(sd, q, W, y, H);
  const T q1b = diff_adj_gather<T>(sd, q, 1, x, W);
  T zb = a.dtmu * ib_;
  zb = zb + zb_;
  zb = zb + (q0b * vy + q1b * vx);
  vb0 += q0b * zc;
  vb1 += q1b * zc;
  if (a.reg_lam != T(0)) {  // regulariser fold at k = 0
    vb0 = vb0 - a.reg_lam * (zc * g0);
    vb1 = vb1 - a.reg_lam * (zc * g1);
  }
  a.zb[b * N + q] = zb;
  a.vbar[b * 2 * N + q] = vb0;
  a.vbar[b * 2 * N + N + q] = vb1;
}

}  // namespace mr
