// mr_kernels3d.cuh -- 3D kernels of the semi-Lagrangian shooting path.
//
// The reference is 2D only; the 3D operators restate it per axis
// exactly as the N-D oracle does (oracle/morphreg_oracle.py): np.gradient per
// axis, its exact transpose, trilinear interpolation with the reference clamp
// and strict inside masks, separable replicate-border Gaussian over 3 axes.
// Layout: scalar [B][D][H][W], vector [B][3][D][H][W]; axis 0 = D.
//
// Velocity  v = -K*(z grad I):   k_product3d -> per-slice 2D FIR (axes 1, 2;
//                                k_smooth2d tile engine) -> k_fir_axis0 (+negate, guard)
// Transport (trilinear):         k_sl_step3d
// Transport adjoint:             k_divseed3d (s = -dt zbar B(z)) -> k_sl_adjoint3d
// Velocity adjoint:              k_fir_axis0^T -> per-slice 2D FIR^T -> k_veladj_epi3d
// Cost terms:                    k_cost_terms3d
#pragma once

#include "mr_kernels2d.cuh"

namespace mr {

struct Grid3 {
  int B, D, H, W;
  long long N;   // D*H*W
  long long HW;  // H*W
};

// Elementwise 3D kernels run on a 3D grid: blockIdx.x -> 32 columns, blockIdx.y ->
// 8 rows, blockIdx.z -> (pair, slice); threadIdx.x = 32 x 8.  No index divisions.
struct Vox {
  int b, d, y, x;
  int q;        // in-pair linear index (N < 2^31)
  bool ok;
};

__device__ __forceinline__ Vox vox3(const Grid3& g) {
  Vox v;
  v.x = blockIdx.x * 32 + (threadIdx.x & 31);
  v.y = blockIdx.y * 8 + (threadIdx.x >> 5);
  v.b = blockIdx.z / g.D;
  v.d = blockIdx.z - v.b * g.D;
  v.ok = v.x < g.W && v.y < g.H;
  v.q = (v.d * g.H + (v.ok ? v.y : 0)) * g.W + (v.ok ? v.x : 0);
  return v;
}

__device__ __forceinline__ void coords3(long long q, const Grid3& g, int& d, int& y, int& x) {
  d = (int)(q / g.HW);
  long long r = q - (long long)d * g.HW;
  y = (int)(r / g.W);
  x = (int)(r - (long long)y * g.W);
}

// np.gradient of f at (d, y, x) along the three axes.
template <typename T>
__device__ __forceinline__ void grad3(const T* __restrict__ f, long long q, int d, int y, int x,
                                      const Grid3& g, T& g0, T& g1, T& g2) {
  const T c = f[q];
  const int HW = (int)g.HW;
  g0 = grad1(d > 0 ? f[q - HW] : c, c, d < g.D - 1 ? f[q + HW] : c, d, g.D);
  g1 = grad1(y > 0 ? f[q - g.W] : c, c, y < g.H - 1 ? f[q + g.W] : c, y, g.H);
  g2 = grad1(x > 0 ? f[q - 1] : c, c, x < g.W - 1 ? f[q + 1] : c, x, g.W);
}

// ------------------------------------------------------------------------------
// m_c = z * d_c I  (integrator.py:94 per axis) -> out [B][3][N]
// ------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) k_product3d(const T* __restrict__ I,
                                                         const T* __restrict__ z, T* out,
                                                         Grid3 g) {
  const Vox v = vox3(g);
  if (!v.ok) return;
  const long long base = (long long)v.b * g.N;
  T g0, g1, g2;
  grad3(I + base, v.q, v.d, v.y, v.x, g, g0, g1, g2);
  const T zz = z[base + v.q];
  T* o = out + (long long)v.b * 3 * g.N + v.q;
  o[0] = zz * g0;
  o[g.N] = zz * g1;
  o[2 * g.N] = zz * g2;
}

// ------------------------------------------------------------------------------
// Trilinear plan / interpolation (fields.py:207-262 generalised; corner c has
// offset bit ax = (c >> ax) & 1, weights multiplied in axis order).
// ------------------------------------------------------------------------------
template <typename T>
struct Plan3 {
  AxisPlan<T> a[3];
  long long base;  // 64-bit: measured faster than int here (IMAD.WIDE addressing)
};

template <typename T>
__device__ __forceinline__ Plan3<T> plan3(int d, int y, int x, T v0, T v1, T v2, T dt,
                                          const Grid3& g) {
  Plan3<T> p;
  p.a[0] = plan_axis<T>(d, v0, dt, g.D);
  p.a[1] = plan_axis<T>(y, v1, dt, g.H);
  p.a[2] = plan_axis<T>(x, v2, dt, g.W);
  p.base = (long long)p.a[0].i0 * g.HW + (long long)p.a[1].i0 * g.W + p.a[2].i0;
  return p;
}

template <typename T>
__device__ __forceinline__ long long corner_off(int c, const Grid3& g) {
  return ((c & 1) ? g.HW : 0) + ((c & 2) ? g.W : 0) + ((c & 4) ? 1 : 0);
}

template <typename T>
__device__ __forceinline__ T axis_w(const Plan3<T>& p, int c, int ax) {
  return ((c >> ax) & 1) ? p.a[ax].f : T(1) - p.a[ax].f;
}

template <typename T>
__device__ __forceinline__ void corners8(const T* __restrict__ f, const Plan3<T>& p,
                                         const Grid3& g, T v[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = f[p.base + corner_off<T>(c, g)];
}

template <typename T>
__device__ __forceinline__ T trilerp(const T v[8], const Plan3<T>& p) {
  T acc = T(0);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const T w = axis_w(p, c, 0) * axis_w(p, c, 1) * axis_w(p, c, 2);
    acc = (c == 0) ? w * v[c] : acc + w * v[c];
  }
  return acc;
}

// d(value)/d(coord_ax) * strict inside mask (interp_coord_grad of the oracle)
template <typename T>
__device__ __forceinline__ void coord_grad3(const T v[8], const Plan3<T>& p, T out[3]) {
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    T acc = T(0);
    bool first = true;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if ((c >> ax) & 1) continue;
      const int hi = c | (1 << ax);
      T w = T(1);
      bool has = false;
#pragma unroll
      for (int o = 0; o < 3; ++o) {
        if (o == ax) continue;
        w = has ? w * axis_w(p, c, o) : axis_w(p, c, o);
        has = true;
      }
      const T t = w * (v[hi] - v[c]);
      acc = first ? t : acc + t;
      first = false;
    }
    out[ax] = acc * (p.a[ax].inside ? T(1) : T(0));
  }
}

// ------------------------------------------------------------------------------
// K2 (3D): one SL step (integrator.py:101-110, 193-205)
// ------------------------------------------------------------------------------
template <typename T>
struct Step3Args {
  const T* I;
  const T* z;
  const T* v;
  T* In;
  T* zn;
  const T* phi_in;
  T* phi_out;
  T dt, dtmu;
  bool has_mu;
  int32_t* guard_in;
  int32_t* guard_out;
  int guard_stride;
  Grid3 g;
};

template <typename T>
__global__ void __launch_bounds__(kThreads) k_sl_step3d(Step3Args<T> a) {
  const Grid3 g = a.g;
  const Vox vx_ = vox3(g);
  if (!vx_.ok) return;
  const int d = vx_.d, y = vx_.y, x = vx_.x, q = vx_.q;
  const long long b = vx_.b;
  const T* __restrict__ I = a.I + b * g.N;
  const T* __restrict__ z = a.z + b * g.N;
  const T* __restrict__ v0 = a.v + b * 3 * g.N;
  const T* __restrict__ v1 = v0 + g.N;
  const T* __restrict__ v2 = v1 + g.N;
  const T a0 = v0[q], a1 = v1[q], a2 = v2[q];
  const T up = d > 0 ? v0[q - g.HW] : a0, dn = d < g.D - 1 ? v0[q + g.HW] : a0;
  const T nn = y > 0 ? v1[q - g.W] : a1, ss = y < g.H - 1 ? v1[q + g.W] : a1;
  const T lf = x > 0 ? v2[q - 1] : a2, rt = x < g.W - 1 ? v2[q + 1] : a2;
  const Plan3<T> p = plan3<T>(d, y, x, a0, a1, a2, a.dt, g);
  T ci[8], cz[8];
  corners8(I, p, g, ci);
  corners8(z, p, g, cz);
  const T zq = (a.has_mu || a.guard_in) ? z[q] : T(0);
  if (a.guard_in) {
    const unsigned fin = guard_bits(I[q], MR_GUARD_IMAGE_NONFINITE) |
                         guard_bits(zq, MR_GUARD_MOMENTUM_NONFINITE);
    if (fin) atomicOr(reinterpret_cast<int*>(a.guard_in + b * a.guard_stride), (int)fin);
  }
  T bi = trilerp(ci, p);
  if (a.has_mu) bi = bi + a.dtmu * zq;
  const T bz = trilerp(cz, p);
  const T div = grad1(up, a0, dn, d, g.D) + grad1(nn, a1, ss, y, g.H) + grad1(lf, a2, rt, x, g.W);
  const T zn = bz * (T(1) - a.dt * div);
  a.In[b * g.N + q] = bi;
  a.zn[b * g.N + q] = zn;
  if (a.guard_out && (!(fabs(bi) <= T(1e6)) || !(fabs(zn) <= T(1e6)))) {  // NaN fails the test too
    const unsigned fo = guard_bits(bi, MR_GUARD_IMAGE_NONFINITE) |
                        guard_bits(zn, MR_GUARD_MOMENTUM_NONFINITE);
    if (fo) atomicOr(reinterpret_cast<int*>(a.guard_out + b * a.guard_stride), (int)fo);
  }
  if (a.phi_in) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      corners8(a.phi_in + (b * 3 + c) * g.N, p, g, ci);
      a.phi_out[(b * 3 + c) * g.N + q] = trilerp(ci, p);
    }
  }
}

template <typename T>
__global__ void k_identity3d(T* phi, Grid3 g) {
  const long long total = (long long)g.B * g.N;
  for (long long pp = blockIdx.x * (long long)blockDim.x + threadIdx.x; pp < total;
       pp += (long long)gridDim.x * blockDim.x) {
    const long long b = pp / g.N, q = pp - b * g.N;
    int d, y, x;
    coords3(q, g, d, y, x);
    phi[(b * 3 + 0) * g.N + q] = T(d);
    phi[(b * 3 + 1) * g.N + q] = T(y);
    phi[(b * 3 + 2) * g.N + q] = T(x);
  }
}

// ------------------------------------------------------------------------------
// K3 (3D): transport adjoint.  k_divseed3d writes s = -dt * zbar * B(z)
// (objective.py:145); k_sl_adjoint3d does the scatters, the coordinate
// gradients and vbar_c += D_c^T s (objective.py:128-147).
// ------------------------------------------------------------------------------
template <typename T>
struct Adj3Args {
  const T* I;
  const T* z;
  const T* v;
  const T* ibar;
  const T* zbar;
  const T* s;  // divergence-adjoint seed
  T* ib;
  T* zb;
  T* vbar;     // [B][3][N]
  T* s_out;    // k_divseed3d output
  T dt, dtmu;
  bool has_mu;
  T reg_lam;
  Grid3 g;
  unsigned long long* qib;  // deterministic mode: fixed-point scatter targets (mr_common.cuh)
  unsigned long long* qzb;
  const unsigned long long* mbits;
  int* ovf;
};

template <typename T>
__global__ void __launch_bounds__(kThreads) k_divseed3d(Adj3Args<T> a) {
  const Grid3 g = a.g;
  const Vox v = vox3(g);
  if (!v.ok) return;
  const long long b = v.b;
  const T* __restrict__ v0 = a.v + b * 3 * g.N;
  const Plan3<T> p = plan3<T>(v.d, v.y, v.x, v0[v.q], v0[g.N + v.q], v0[2 * g.N + v.q], a.dt, g);
  T cv[8];
  corners8(a.z + b * g.N, p, g, cv);
  a.s_out[b * g.N + v.q] = -a.dt * (a.zbar[b * g.N + v.q] * trilerp(cv, p));
}

// Scatter of the 8 trilinear-transpose contributions with warp-level merging of
// x-adjacent cells (lanes are consecutive x): where lane l-1's +x cells are
// lane l's cells, lane l adds them and lane l-1 skips its own (4 of 8 REDs).
template <typename T>
__device__ __forceinline__ void scatter8_merged(T* __restrict__ out, int base, bool valid,
                                                const Grid3& g, const T w[8]) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int key = valid ? base : -4;
  const int prev_key = __shfl_up_sync(full, key, 1);
  const int next_key = __shfl_down_sync(full, key, 1);
  const bool merge_left = lane > 0 && prev_key >= 0 && prev_key + 1 == key;
  const bool merged_by_next = lane < 31 && next_key >= 0 && key + 1 == next_key;
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // corners c (x bit 0) pair with c | 4 (x bit 1)
    const int off = ((c & 1) ? (int)g.HW : 0) + ((c & 2) ? g.W : 0);
    const T pr = __shfl_up_sync(full, w[c | 4], 1);
    if (valid) {
      atomicAdd(out + base + off, merge_left ? w[c] + pr : w[c]);
      if (!merged_by_next) atomicAdd(out + base + off + 1, w[c | 4]);
    }
  }
}

// scatter8_merged in fixed point (contributions converted before any merge)
template <typename T>
__device__ __forceinline__ void scatter8_merged_fix(unsigned long long* __restrict__ out, int base,
                                                    bool valid, const Grid3& g, const T w[8],
                                                    double f, unsigned& ovf) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int key = valid ? base : -4;
  const int prev_key = __shfl_up_sync(full, key, 1);
  const int next_key = __shfl_down_sync(full, key, 1);
  const bool merge_left = lane > 0 && prev_key >= 0 && prev_key + 1 == key;
  const bool merged_by_next = lane < 31 && next_key >= 0 && key + 1 == next_key;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int off = ((c & 1) ? (int)g.HW : 0) + ((c & 2) ? g.W : 0);
    const long long lo = valid ? to_fix((double)w[c], f, ovf) : 0;
    const long long hi = valid ? to_fix((double)w[c | 4], f, ovf) : 0;
    const long long pr = __shfl_up_sync(full, hi, 1);
    if (valid) {
      fix_add(out + base + off, merge_left ? lo + pr : lo);
      if (!merged_by_next) fix_add(out + base + off + 1, hi);
    }
  }
}

template <typename T, bool DET = false>
__global__ void __launch_bounds__(kThreads) k_sl_adjoint3d(Adj3Args<T> a) {
  // Latency-bound gathers: every load (v and its neighbours, ibar/zbar, the 8+8
  // corners of I and z, the s neighbours) is issued before the first scatter, so
  // they are all in flight together instead of behind the atomics.
  const Grid3 g = a.g;
  const Vox vx_ = vox3(g);
  const bool own = vx_.ok;
  const int d = vx_.d, y = own ? vx_.y : 0, x = own ? vx_.x : 0, q = vx_.q;
  const long long b = vx_.b;
  const T* __restrict__ I = a.I + b * g.N;
  const T* __restrict__ z = a.z + b * g.N;
  const T* __restrict__ v0 = a.v + b * 3 * g.N;
  const T* __restrict__ v1 = v0 + g.N;
  const T* __restrict__ v2 = v1 + g.N;
  const T* __restrict__ s = a.s + b * g.N;
  const T a0 = v0[q], a1 = v1[q], a2 = v2[q];
  const T ib_ = a.ibar[b * g.N + q], zb_ = a.zbar[b * g.N + q];
  const int st[3] = {(int)g.HW, g.W, 1};
  const int pos[3] = {d, y, x};
  const int n[3] = {g.D, g.H, g.W};
  // Interior voxels (2 <= pos <= n-3 on every axis): the np.gradient stencil and
  // the gather form of its transpose have no edge terms, so neighbour loads are
  // unconditional and D^T s is 0.5 s[j-1] - 0.5 s[j+1] -- the same operations
  // diff_adj1 performs there (bitwise equal).  Only the loads and the stencil
  // arithmetic branch; the scatters below stay warp-converged.
  const bool inner = own && d >= 2 && d <= g.D - 3 && y >= 2 && y <= g.H - 3 && x >= 2 &&
                     x <= g.W - 3;
  T vm0, vp0, vm1, vp1, vm2, vp2;
  T sm[3], sp[3];
  const T sc = s[q];
  if (inner) {
    vm0 = v0[q - g.HW];
    vp0 = v0[q + g.HW];
    vm1 = v1[q - g.W];
    vp1 = v1[q + g.W];
    vm2 = v2[q - 1];
    vp2 = v2[q + 1];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sm[c] = s[q - st[c]];
      sp[c] = s[q + st[c]];
    }
  } else {
    vm0 = d > 0 ? v0[q - g.HW] : a0;
    vp0 = d < g.D - 1 ? v0[q + g.HW] : a0;
    vm1 = y > 0 ? v1[q - g.W] : a1;
    vp1 = y < g.H - 1 ? v1[q + g.W] : a1;
    vm2 = x > 0 ? v2[q - 1] : a2;
    vp2 = x < g.W - 1 ? v2[q + 1] : a2;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      sm[c] = pos[c] > 0 ? s[q - st[c]] : T(0);
      sp[c] = pos[c] < n[c] - 1 ? s[q + st[c]] : T(0);
    }
  }
  const Plan3<T> p = plan3<T>(d, y, x, a0, a1, a2, a.dt, g);
  const int base = (int)p.base;
  T cI[8], cz[8];
  corners8(I, p, g, cI);
  corners8(z, p, g, cz);

  T w8[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) w8[c] = axis_w(p, c, 0) * axis_w(p, c, 1) * axis_w(p, c, 2);
  const T div = inner ? (vp0 - vm0) / T(2) + (vp1 - vm1) / T(2) + (vp2 - vm2) / T(2)
                     : grad1(vm0, a0, vp0, d, g.D) + grad1(vm1, a1, vp1, y, g.H) +
                           grad1(vm2, a2, vp2, x, g.W);
  const T wz = zb_ * (T(1) - a.dt * div);
  T dI[3], dz[3];
  coord_grad3(cI, p, dI);
  coord_grad3(cz, p, dz);
  T vb[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) vb[c] = -a.dt * dI[c] * ib_;
#pragma unroll
  for (int c = 0; c < 3; ++c) vb[c] += -a.dt * dz[c] * wz;
  if (inner) {
#pragma unroll
    for (int c = 0; c < 3; ++c) vb[c] += T(0.5) * sm[c] - T(0.5) * sp[c];
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // vbar_c += D_c^T s (gather form along each axis)
      const int j = pos[c];
      const T sf = j == 0 ? sc : (j == 1 ? sm[c] : T(0));
      const T sl = j == n[c] - 1 ? sc : (j == n[c] - 2 ? sp[c] : T(0));
      vb[c] += diff_adj1(sm[c], sp[c], sf, sl, j, n[c]);
    }
  }

  T cw[8];
  if constexpr (DET) {
    const double f = fix_factor(a.mbits, b);
    unsigned ovf = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) cw[c] = w8[c] * ib_;
    scatter8_merged_fix(a.qib + b * g.N, base, own, g, cw, f, ovf);
#pragma unroll
    for (int c = 0; c < 8; ++c) cw[c] = w8[c] * wz;
    scatter8_merged_fix(a.qzb + b * g.N, base, own, g, cw, f, ovf);
    if (own && a.has_mu) fix_add(a.qzb + b * g.N + q, to_fix((double)(a.dtmu * ib_), f, ovf));
    if (ovf) atomicOr(a.ovf, 1);
    if (!own) return;
  } else {
    T* __restrict__ ibo = a.ib + b * g.N;
    T* __restrict__ zbo = a.zb + b * g.N;
#pragma unroll
    for (int c = 0; c < 8; ++c) cw[c] = w8[c] * ib_;
    scatter8_merged(ibo, base, own, g, cw);
#pragma unroll
    for (int c = 0; c < 8; ++c) cw[c] = w8[c] * wz;
    scatter8_merged(zbo, base, own, g, cw);
    if (!own) return;
    if (a.has_mu) atomicAdd(zbo + q, a.dtmu * ib_);
  }
  if (a.reg_lam != T(0)) {
    T g0, g1, g2;
    grad3(I, q, d, y, x, g, g0, g1, g2);
    const T zz = z[q];
    vb[0] = vb[0] - a.reg_lam * (zz * g0);
    vb[1] = vb[1] - a.reg_lam * (zz * g1);
    vb[2] = vb[2] - a.reg_lam * (zz * g2);
  }
  T* vo = a.vbar + b * 3 * g.N + q;
  vo[0] = vb[0];
  vo[g.N] = vb[1];
  vo[2 * g.N] = vb[2];
}

// ------------------------------------------------------------------------------
// K4 epilogue (3D): ktv = K^T vbar (so mbar = -ktv);
//   zb += mbar . grad I;  ib += G^T(mbar z)  (objective.py:157-161)
//   REG (k = 0): zout = zb + mbar.grad I0 + lam (K m0 . grad I0 + 2 rho z0), K m0 = -v0
// ------------------------------------------------------------------------------
template <typename T>
struct VelAdj3Args {
  const T* I;
  const T* z;
  const T* ktv;  // [B][3][N]
  T* ib;
  T* zb;
  const T* v0;
  T* zout;
  int32_t* flags;
  T lam, two_rho;
  Grid3 g;
};

template <typename T, bool REG>
__global__ void __launch_bounds__(kThreads) k_veladj_epi3d(VelAdj3Args<T> a) {
  const Grid3 g = a.g;
  const Vox v = vox3(g);
  if (!v.ok) return;
  const int d = v.d, y = v.y, x = v.x, q = v.q;
  const long long b = v.b;
  const long long pp = b * g.N + q;
  const T* __restrict__ I = a.I + b * g.N;
  const T* __restrict__ z = a.z + b * g.N;
  const T* __restrict__ kt = a.ktv + b * 3 * g.N;
  T gr[3];
  grad3(I, q, d, y, x, g, gr[0], gr[1], gr[2]);
  const T m0 = -kt[q], m1 = -kt[g.N + q], m2 = -kt[2 * g.N + q];
  T zb_new = a.zb[pp] + (m0 * gr[0] + m1 * gr[1] + m2 * gr[2]);
  if (REG) {
    const T* __restrict__ w = a.v0 + b * 3 * g.N;
    const T km = -(w[q] * gr[0] + w[g.N + q] * gr[1] + w[2 * g.N + q] * gr[2]);
    zb_new = zb_new + a.lam * (km + a.two_rho * z[q]);
    a.zout[pp] = zb_new;
    if (!isfinite(zb_new)) atomicOr(reinterpret_cast<int*>(a.flags + b), 1);
  } else {
    a.zb[pp] = zb_new;
    const int st[3] = {(int)g.HW, g.W, 1};
    const int pos[3] = {d, y, x};
    const int n[3] = {g.D, g.H, g.W};
    T acc = T(0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T* kc = kt + c * g.N;
      auto qv = [&](int qq) { return -kc[qq] * z[qq]; };
      const int j = pos[c];
      const T qc = qv(q);
      const T gm = j > 0 ? qv(q - st[c]) : T(0);
      const T gp = j < n[c] - 1 ? qv(q + st[c]) : T(0);
      const T gf = j == 0 ? qc : (j == 1 ? gm : T(0));
      const T gl = j == n[c] - 1 ? qc : (j == n[c] - 2 ? gp : T(0));
      const T t = diff_adj1(gm, gp, gf, gl, j, n[c]);
      acc = (c == 0) ? t : acc + t;
    }
    a.ib[pp] = a.ib[pp] + acc;
  }
}

// ------------------------------------------------------------------------------
// K5 (3D): cost terms
// ------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) k_cost_terms3d(const T* __restrict__ I0,
                                                            const T* __restrict__ z0,
                                                            const T* __restrict__ v0,
                                                            const T* __restrict__ IT,
                                                            const T* __restrict__ J, T* seed,
                                                            double* part, Grid3 g) {
  __shared__ double red[kThreads / 32];
  const int b = blockIdx.y;
  const T* Ib = I0 + b * g.N;
  const T* zb = z0 + b * g.N;
  const T* vb = v0 + b * 3 * g.N;
  double data = 0.0, vn = 0.0, zn = 0.0;
  for (long long q = blockIdx.x * (long long)kThreads + threadIdx.x; q < g.N;
       q += (long long)gridDim.x * kThreads) {
    const T diff = IT[b * g.N + q] - J[b * g.N + q];
    if (seed) seed[b * g.N + q] = diff;
    data += (double)diff * (double)diff;
    int d, y, x;
    coords3(q, g, d, y, x);
    T g0, g1, g2;
    grad3(Ib, q, d, y, x, g, g0, g1, g2);
    const T zz = zb[q];
    vn += (double)(zz * g0) * (double)vb[q] + (double)(zz * g1) * (double)vb[g.N + q] +
          (double)(zz * g2) * (double)vb[2 * g.N + q];
    zn += (double)zz * (double)zz;
  }
  double s;
  double* out = part + ((long long)b * gridDim.x + blockIdx.x) * 4;  // see k_cost_terms2d
  s = block_sum(data, red);
  if (threadIdx.x == 0) out[1] = s;
  s = block_sum(vn, red);
  if (threadIdx.x == 0) out[2] = s;
  s = block_sum(zn, red);
  if (threadIdx.x == 0) out[3] = s;
}

}  // namespace mr
