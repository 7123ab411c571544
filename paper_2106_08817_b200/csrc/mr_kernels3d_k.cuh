// mr_kernels3d_k.cuh -- multi-voxel variants of the 3D elementwise / gather
// kernels (K voxels consecutive along axis 0 per thread).  Same per-voxel
// arithmetic as the single-voxel kernels in mr_kernels3d.cuh; included by
// mr_capi.cu only.
#pragma once

#include "mr_kernels3d.cuh"

namespace mr {

// Multi-voxel product: K voxels consecutive along axis 0 per thread; the axis-0
// column of I (d0-1 .. d0+K) is loaded once and shared.  Same arithmetic as
// k_product3d (bitwise equal).
template <typename T, int K>
__global__ void __launch_bounds__(kThreads) k_product3d_k(const T* __restrict__ I,
                                                           const T* __restrict__ z, T* out,
                                                           Grid3 g) {
  const int DK = (g.D + K - 1) / K;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= g.W || y >= g.H) return;
  const int b = blockIdx.z / DK;
  const int d0 = (blockIdx.z - b * DK) * K;
  const int HW = (int)g.HW;
  const T* __restrict__ f = I + (long long)b * g.N;
  const int q0 = (d0 * g.H + y) * g.W + x;
  T col[K + 2], up[K], dn[K], lf[K], rt[K], zz[K];
#pragma unroll
  for (int j = 0; j < K + 2; ++j) {
    const int dd = min(max(d0 - 1 + j, 0), g.D - 1);
    col[j] = f[q0 + (dd - d0) * HW];
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int dd = min(d0 + j, g.D - 1);
    const int q = q0 + (dd - d0) * HW;
    const T c = col[j + 1];
    up[j] = y > 0 ? f[q - g.W] : c;
    dn[j] = y < g.H - 1 ? f[q + g.W] : c;
    lf[j] = x > 0 ? f[q - 1] : c;
    rt[j] = x < g.W - 1 ? f[q + 1] : c;
    zz[j] = z[(long long)b * g.N + q];
  }
  T* o = out + (long long)b * 3 * g.N;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int d = d0 + j;
    if (d >= g.D) break;
    const int q = q0 + j * HW;
    const T c = col[j + 1];
    const T g0 = grad1(d > 0 ? col[j] : c, c, d < g.D - 1 ? col[j + 2] : c, d, g.D);
    const T g1 = grad1(up[j], c, dn[j], y, g.H);
    const T g2 = grad1(lf[j], c, rt[j], x, g.W);
    o[q] = zz[j] * g0;
    o[g.N + q] = zz[j] * g1;
    o[2 * g.N + q] = zz[j] * g2;
  }
}

// Velocity-adjoint epilogue (non-REG steps), K voxels along axis 0 per thread:
// the axis-0 columns of I, ktv_0 and z (d0-1 .. d0+K) are loaded once and
// shared.  Per-voxel arithmetic is k_veladj_epi3d<T, false>'s.
template <typename T, int K>
__global__ void __launch_bounds__(kThreads) k_veladj_epi3d_k(VelAdj3Args<T> a) {
  const Grid3 g = a.g;
  const int DK = (g.D + K - 1) / K;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= g.W || y >= g.H) return;
  const int b = blockIdx.z / DK;
  const int d0 = (blockIdx.z - b * DK) * K;
  const int HW = (int)g.HW;
  const long long pb = (long long)b * g.N;
  const T* __restrict__ I = a.I + pb;
  const T* __restrict__ z = a.z + pb;
  const T* __restrict__ k0 = a.ktv + 3 * pb;
  const T* __restrict__ k1 = k0 + g.N;
  const T* __restrict__ k2 = k1 + g.N;
  const int q0 = (d0 * g.H + y) * g.W + x;
  T ci[K + 2], ck[K + 2], cz[K + 2];
#pragma unroll
  for (int j = 0; j < K + 2; ++j) {
    const int q = q0 + (min(max(d0 - 1 + j, 0), g.D - 1) - d0) * HW;
    ci[j] = I[q];
    ck[j] = k0[q];
    cz[j] = z[q];
  }
  T iu[K], id[K], il[K], ir[K], m1[K], m2[K], zb[K], ib[K];
  T k1m[K], k1p[K], z1m[K], z1p[K], k2m[K], k2p[K], z2m[K], z2p[K];
  // in-plane interior (2 <= y <= H-3, 2 <= x <= W-3): no edge terms on axes 1, 2
  const bool inner_yx = y >= 2 && y <= g.H - 3 && x >= 2 && x <= g.W - 3;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int q = q0 + (min(d0 + j, g.D - 1) - d0) * HW;
    const T c = ci[j + 1];
    m1[j] = k1[q];
    m2[j] = k2[q];
    zb[j] = a.zb[pb + q];
    ib[j] = a.ib[pb + q];
    if (inner_yx) {
      iu[j] = I[q - g.W];
      id[j] = I[q + g.W];
      il[j] = I[q - 1];
      ir[j] = I[q + 1];
      k1m[j] = k1[q - g.W];
      z1m[j] = z[q - g.W];
      k1p[j] = k1[q + g.W];
      z1p[j] = z[q + g.W];
      k2m[j] = k2[q - 1];
      z2m[j] = z[q - 1];
      k2p[j] = k2[q + 1];
      z2p[j] = z[q + 1];
    } else {
      iu[j] = y > 0 ? I[q - g.W] : c;
      id[j] = y < g.H - 1 ? I[q + g.W] : c;
      il[j] = x > 0 ? I[q - 1] : c;
      ir[j] = x < g.W - 1 ? I[q + 1] : c;
      k1m[j] = y > 0 ? k1[q - g.W] : T(0);
      z1m[j] = y > 0 ? z[q - g.W] : T(0);
      k1p[j] = y < g.H - 1 ? k1[q + g.W] : T(0);
      z1p[j] = y < g.H - 1 ? z[q + g.W] : T(0);
      k2m[j] = x > 0 ? k2[q - 1] : T(0);
      z2m[j] = x > 0 ? z[q - 1] : T(0);
      k2p[j] = x < g.W - 1 ? k2[q + 1] : T(0);
      z2p[j] = x < g.W - 1 ? z[q + 1] : T(0);
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int d = d0 + j;
    if (d >= g.D) break;
    const long long pp = pb + q0 + j * HW;
    const T c = ci[j + 1];
    const T gr0 = grad1(d > 0 ? ci[j] : c, c, d < g.D - 1 ? ci[j + 2] : c, d, g.D);
    const T gr1 = grad1(iu[j], c, id[j], y, g.H);
    const T gr2 = grad1(il[j], c, ir[j], x, g.W);
    const T mm0 = -ck[j + 1], mm1 = -m1[j], mm2 = -m2[j];
    a.zb[pp] = zb[j] + (mm0 * gr0 + mm1 * gr1 + mm2 * gr2);
    // G^T(mbar z): qv = -ktv_c * z at the voxel and its axis-c neighbours
    const T qc0 = -ck[j + 1] * cz[j + 1];
    const T qm0 = d > 0 ? -ck[j] * cz[j] : T(0);
    const T qp0 = d < g.D - 1 ? -ck[j + 2] * cz[j + 2] : T(0);
    const T qc1 = -m1[j] * cz[j + 1], qm1 = -k1m[j] * z1m[j], qp1 = -k1p[j] * z1p[j];
    const T qc2 = -m2[j] * cz[j + 1], qm2 = -k2m[j] * z2m[j], qp2 = -k2p[j] * z2p[j];
    const T qcv[3] = {qc0, qc1, qc2}, qmv[3] = {qm0, qm1, qm2}, qpv[3] = {qp0, qp1, qp2};
    const int pos[3] = {d, y, x};
    const int n[3] = {g.D, g.H, g.W};
    T acc = T(0);
    if (inner_yx && d >= 2 && d <= g.D - 3) {  // diff_adj1 without edge terms
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        const T t = T(0.5) * qmv[cc] - T(0.5) * qpv[cc];
        acc = (cc == 0) ? t : acc + t;
      }
    } else {
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        const int jj = pos[cc];
        const T gf = jj == 0 ? qcv[cc] : (jj == 1 ? qmv[cc] : T(0));
        const T gl = jj == n[cc] - 1 ? qcv[cc] : (jj == n[cc] - 2 ? qpv[cc] : T(0));
        const T t = diff_adj1(qmv[cc], qpv[cc], gf, gl, jj, n[cc]);
        acc = (cc == 0) ? t : acc + t;
      }
    }
    a.ib[pp] = ib[j] + acc;
  }
}

}  // namespace mr
