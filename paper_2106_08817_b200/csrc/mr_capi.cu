// mr_capi.cu -- extern "C" boundary (include/morphreg_sm100.h) and the native
// whole-loop drivers of shoot() / grad().
//
// The drivers replace the Python T-step loops of integrator.shoot
// (integrator.py:163-219) and objective.grad (objective.py:91-174): one ctypes
// call launches the whole forward sweep (2 kernels per step) or the whole
// reverse sweep (memset + 2 kernels per step), stream-ordered, with no host
// synchronisation inside.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mr_launch.cuh"
#include "mr_kernels3d_k.cuh"
#include "mr_tma.h"
#include "mr_schemes2d.cuh"
#include "mr_transport2d.cuh"

namespace mr {

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int set_error(int code, const std::string& msg) { return fail(code, msg); }

static int check_cuda(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MR_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return MR_OK;
}

static int check_rc(int rc, const char* where) {
  if (rc == MR_OK) return MR_OK;
  if (rc < 0) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = g_last_cuda;
    g_last_cuda = cudaSuccess;
    return fail(rc, std::string(where) + ": " + cudaGetErrorString(e));
  }
  return fail(rc, std::string(where) + ": invalid argument");
}

static int validate(int dtype, const mr_grid& g, bool allow3d = true) {
  if (dtype != MR_F32 && dtype != MR_F64) return fail(MR_EINVAL, "dtype must be MR_F32 or MR_F64");
  if (g.ndim != 2 && g.ndim != 3) return fail(MR_EINVAL, "ndim must be 2 or 3");
  if (g.ndim == 3 && !allow3d)
    return fail(MR_EINVAL, "3D: use the whole-loop entry points mr_shoot_forward/mr_shoot_adjoint");
  if (g.batch < 1) return fail(MR_EINVAL, "batch must be >= 1");
  if (g.n[0] < 2 || g.n[1] < 2 || (g.ndim == 3 && g.n[2] < 2)) {
    std::string dims = std::to_string(g.n[0]) + "x" + std::to_string(g.n[1]);
    if (g.ndim == 3) dims += "x" + std::to_string(g.n[2]);
    return fail(MR_EINVAL, "grid must be at least 2x2, got " + dims);
  }
  long long N = (long long)g.n[0] * g.n[1] * (g.ndim == 3 ? g.n[2] : 1);
  if (N > (1LL << 31) - 1) return fail(MR_EINVAL, "grid too large");
  if ((long long)g.batch * 3 * (g.ndim == 3 ? g.n[0] : 1) > 65535)
    return fail(MR_EINVAL, "batch too large for one launch");
  return MR_OK;
}

static Grid2 grid2(const mr_grid& g) {
  Grid2 r;
  r.B = g.batch;
  r.H = g.n[0];
  r.W = g.n[1];
  r.N = (long long)r.H * r.W;
  return r;
}

template <typename T>
static int make_taps(const mr_kernel& k, Taps<T>& tp) {
  if (k.radius < 1 || k.radius > kMaxR)
    return fail(MR_EINVAL, "kernel radius must lie in [1, " + std::to_string(kMaxR) + "], got " +
                               std::to_string(k.radius));
  if (!k.weights) return fail(MR_EINVAL, "kernel weights pointer is NULL");
  const int R = k.radius;
  std::memset(&tp, 0, sizeof(tp));
  // symmetrise (the reference weights are exactly symmetric; this only guards
  // against caller-side asymmetry since the transpose relies on it)
  for (int t = 0; t <= 2 * R; ++t) {
    double w = 0.5 * (k.weights[t] + k.weights[2 * R - t]);
    if (!std::isfinite(w)) return fail(MR_EINVAL, "kernel weights must be finite");
    tp.w[t] = (T)w;
  }
  double acc = 0.0;
  for (int m = 0; m <= R; ++m) {  // W[m] = sum_{k<=m} w_k (kernel.py:48-68 edge rows)
    acc += 0.5 * (k.weights[m] + k.weights[2 * R - m]);
    tp.e[m] = (T)acc;
  }
  return MR_OK;
}

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static Grid3 grid3(const mr_grid& g) {
  Grid3 r;
  r.B = g.batch;
  r.D = g.n[0];
  r.H = g.n[1];
  r.W = g.n[2];
  r.HW = (long long)r.H * r.W;
  r.N = (long long)r.D * r.HW;
  return r;
}

static long long scalars(const mr_grid& g) {
  return (long long)g.batch * g.n[0] * g.n[1] * (g.ndim == 3 ? g.n[2] : 1);
}

static dim3 grid3d(const Grid3& g) {
  return dim3((unsigned)((g.W + 31) / 32), (unsigned)((g.H + 7) / 8), (unsigned)(g.B * g.D));
}

// Multi-voxel 3D kernels: K voxels consecutive along axis 0 per thread.  Measured
// on cfg4 (4 pairs, B200): product 60.5 / 42.8 / 38.9 us at K = 1 / 2 / 4; velocity-
// adjoint epilogue 123 / 105 / 175 us.  The gather kernels (transport step,
// divergence seed, transport adjoint) were slower at K > 1 (register-bound
// occupancy: step 110 -> 124 us, adjoint 250 -> 343 us at K = 2) and stay at K = 1.
constexpr int kProductK = 4, kEpiK = 2;

static dim3 grid3d_k(const Grid3& g, int K) {
  return dim3((unsigned)((g.W + 31) / 32), (unsigned)((g.H + 7) / 8),
              (unsigned)(g.B * ((g.D + K - 1) / K)));
}

static unsigned flat_blocks(long long n) {
  long long b = (n + kThreads - 1) / kThreads;
  return (unsigned)(b < 148LL * 16 ? b : 148LL * 16);
}

// ---- 3D building blocks ----------------------------------------------------------

// v = -K*(z grad I): product -> per-slice FIR (axes 1, 2) -> axis-0 FIR (+negate, guard).
// `v` doubles as the product scratch; `tmp` holds 3 scalars per voxel.
template <typename T>
static int velocity3d(const Grid3& g, int R, const Taps<T>& tp, const T* I, const T* z, T* v,
                      T* tmp, int32_t* guard, int guard_stride, cudaStream_t s) {
  k_product3d_k<T, kProductK><<<grid3d_k(g, kProductK), kThreads, 0, s>>>(I, z, v, g);
  int rc = cuda_status(cudaGetLastError());
  if (rc) return rc;
  Grid2 sl{g.B * 3 * g.D, g.H, g.W, g.HW};  // every (pair, component, slice) as a 2D image
  rc = launch_smooth2d<T>(sl, R, tp, v, tmp, false, s);
  if (rc) return rc;
  return launch_fir_axis0<T>(R, tp, tmp, v, g.B * 3, g.D, g.HW, false, 1, guard, guard_stride, 3, s);
}

template <typename T>
static int sl_step3d(const Grid3& g, double dt, double mu, const T* I, const T* z, const T* v,
                     T* In, T* zn, const T* phi_in, T* phi_out, cudaStream_t s,
                     int32_t* guard_in = nullptr, int32_t* guard_out = nullptr,
                     int guard_stride = 1) {
  Step3Args<T> a{I,       z,      v,        In,          zn,      phi_in,    phi_out,
                 (T)dt,   (T)(dt * mu), mu != 0.0, guard_in, guard_out, guard_stride, g};
  k_sl_step3d<T><<<grid3d(g), kThreads, 0, s>>>(a);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------------------------
template <typename T>
static int launch_sl_step2d(const Grid2& g, double dt, double mu, const T* I, const T* z,
                            const T* v, T* In, T* zn, const T* phi_in, T* phi_out,
                            cudaStream_t s, int32_t* guard_in = nullptr,
                            int32_t* guard_out = nullptr, int guard_stride = 1) {
  StepArgs<T> a{I,     z,       v,      In,        zn,          phi_in,
                phi_out, (T)dt, (T)(dt * mu), mu != 0.0, guard_in, guard_out,
                guard_stride, g};
  {  // TMA-staged tile variant when the layout is TMA-describable
    using C = TrCfg<T>;
    StepMaps m;
    if (make_map3<T>(&m.I, I, g.W, g.H, g.B, C::GX, C::GY) &&
        make_map3<T>(&m.z, z, g.W, g.H, g.B, C::GX, C::GY) &&
        make_map3<T>(&m.v, v, g.W, g.H, 2LL * g.B, C::VX, C::VY)) {
      const cudaError_t attr = ensure_smem<k_sl_step2d_tma<T>>(C::bytes);
      if (attr != cudaSuccess) return cuda_status(attr);
      dim3 grid((g.W + C::TX - 1) / C::TX, (g.H + C::TY - 1) / C::TY, g.B);
      k_sl_step2d_tma<T><<<grid, kThreads, C::bytes, s>>>(a, m);
      return cuda_status(cudaGetLastError());
    }
  }
  dim3 grid((g.W + 31) / 32, (g.H + kStepRows - 1) / kStepRows, g.B);
  k_sl_step2d<T><<<grid, kThreads, 0, s>>>(a);
  return cuda_status(cudaGetLastError());
}

template <typename T>
static int launch_sl_adjoint2d(const Grid2& g, double dt, double mu, const T* I, const T* z,
                               const T* v, const T* ibar, const T* zbar, T* ib, T* zb, T* vbar,
                               cudaStream_t s, double reg_lam = 0.0) {
  AdjArgs<T> a{I, z, v, ibar, zbar, ib, zb, vbar, (T)dt, (T)(dt * mu), mu != 0.0, (T)reg_lam, g};
  {  // TMA-staged tile variant when the layout is TMA-describable
    using C = TrCfg<T>;
    AdjMaps m;
    if (make_map3<T>(&m.I, I, g.W, g.H, g.B, C::GX, C::GY) &&
        make_map3<T>(&m.z, z, g.W, g.H, g.B, C::GX, C::GY) &&
        make_map3<T>(&m.v, v, g.W, g.H, 2LL * g.B, C::VX, C::VY) &&
        make_map3<T>(&m.ibar, ibar, g.W, g.H, g.B, C::VX, C::VY) &&
        make_map3<T>(&m.zbar, zbar, g.W, g.H, g.B, C::VX, C::VY)) {
      constexpr size_t bytes = AdjCfg<T>::bytes;
      const cudaError_t attr = ensure_smem<k_sl_adjoint2d_tma<T>>(bytes);
      if (attr != cudaSuccess) return cuda_status(attr);
      dim3 grid((g.W + C::TX - 1) / C::TX, (g.H + C::TY - 1) / C::TY, g.B);
      k_sl_adjoint2d_tma<T><<<grid, kThreads, bytes, s>>>(a, m);
      return cuda_status(cudaGetLastError());
    }
  }
  dim3 grid((g.W + kAdjTX - 1) / kAdjTX, (g.H + kAdjRows - 1) / kAdjRows, g.B);
  k_sl_adjoint2d<T><<<grid, kThreads, 0, s>>>(a);
  return cuda_status(cudaGetLastError());
}

// Deterministic-mode transport adjoint (2D): the generic kernels with fixed-point
// scatters (SL: k_sl_adjoint2d<T, true>; HYBRID: k_scheme_adj2d<T, true>).
template <typename T, typename Tail>
static int launch_adjoint2d_det(int scheme, const Grid2& g, double dt, double mu, const T* I,
                                const T* z, const T* v, const T* ibar, const T* zbar, T* ib,
                                T* zb, T* vbar, const Tail& tail, cudaStream_t s,
                                double reg_lam) {
  AdjArgs<T> a{I, z, v, ibar, zbar, ib, zb, vbar, (T)dt, (T)(dt * mu), mu != 0.0, (T)reg_lam, g};
  a.qib = tail.q;
  a.qzb = tail.q + (long long)g.B * g.N;
  a.mbits = tail.mbits;
  a.ovf = tail.ovf;
  if (scheme == kSchemeSL) {
    dim3 grid((g.W + kAdjTX - 1) / kAdjTX, (g.H + kAdjRows - 1) / kAdjRows, g.B);
    k_sl_adjoint2d<T, true><<<grid, kThreads, 0, s>>>(a);
  } else {
    dim3 grid((g.W + 31) / 32, (g.H + kNW - 1) / kNW, g.B);
    k_scheme_adj2d<T, true><<<grid, kThreads, 0, s>>>(a, scheme);
  }
  return cuda_status(cudaGetLastError());
}

// Eulerian / Hybrid transport step and its adjoint (mr_schemes2d.cuh).
template <typename T>
static int launch_scheme_step2d(int scheme, const Grid2& g, double dt, double mu, const T* I,
                                const T* z, const T* v, T* In, T* zn, const T* phi_in,
                                T* phi_out, cudaStream_t s, int32_t* guard_in,
                                int32_t* guard_out, int guard_stride) {
  StepArgs<T> a{I,     z,       v,      In,        zn,          phi_in,
                phi_out, (T)dt, (T)(dt * mu), mu != 0.0, guard_in, guard_out,
                guard_stride, g};
  dim3 grid((g.W + 31) / 32, (g.H + kNW - 1) / kNW, g.B);
  k_scheme_step2d<T><<<grid, kThreads, 0, s>>>(a, (T)mu, scheme);
  return cuda_status(cudaGetLastError());
}

template <typename T>
static int launch_scheme_adj2d(int scheme, const Grid2& g, double dt, double mu, const T* I,
                               const T* z, const T* v, const T* ibar, const T* zbar, T* ib, T* zb,
                               T* vbar, cudaStream_t s, double reg_lam) {
  AdjArgs<T> a{I, z, v, ibar, zbar, ib, zb, vbar, (T)dt, (T)(dt * mu), mu != 0.0, (T)reg_lam, g};
  dim3 grid((g.W + 31) / 32, (g.H + kNW - 1) / kNW, g.B);
  k_scheme_adj2d<T><<<grid, kThreads, 0, s>>>(a, scheme);
  return cuda_status(cudaGetLastError());
}

// Cost-term partials: kCostBlocks per pair in the workspace tail (deterministic
// block-order reduction); without a workspace one block per pair writes its sums
// straight into terms (same result bits, slower on large grids).
constexpr int kCostBlocks = 1024;

template <typename T>
static int launch_cost_terms2d(const Grid2& g, double lam, double rho, const T* I0, const T* z0,
                               const T* v0, const T* IT, const T* J, double* terms, T* seed,
                               cudaStream_t s, double* part = nullptr) {
  // one warp per row: blocks of kNW rows
  long long blocks = (g.H + kNW - 1) / kNW;
  if (blocks > kCostBlocks) blocks = kCostBlocks;
  if (!part) {
    part = terms;
    blocks = 1;
  }
  CostArgs<T> a{I0, z0, v0, IT, J, seed, part, g};
  k_cost_terms2d<T><<<dim3((unsigned)blocks, g.B), kThreads, 0, s>>>(a);
  k_finalize_terms<<<(g.B + 127) / 128, 128, 0, s>>>(terms, part, (int)blocks, g.B, lam, rho);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------------------------
template <typename T>
static int shoot_forward3d(const mr_grid& mg, const mr_kernel& k, const Taps<T>& tp, double mu,
                           int T_, T* I, T* z, T* v, void* phi, int32_t* guard, T* tmp,
                           cudaStream_t s) {
  const Grid3 g = grid3(mg);
  const double dt = 1.0 / T_;
  const long long S1 = (long long)g.B * g.N;
  const long long SV = 3 * S1;
  T* ph[2] = {nullptr, nullptr};
  if (phi) {
    T* base = static_cast<T*>(phi);
    ph[0] = (T_ % 2 == 0) ? base : base + SV;
    ph[1] = (T_ % 2 == 0) ? base + SV : base;
    k_identity3d<T><<<592, 256, 0, s>>>(ph[0], g);
  }
  if (guard && cudaMemsetAsync(guard, 0, sizeof(int32_t) * (size_t)g.B * (T_ + 1), s) != cudaSuccess)
    return check_cuda("memset guard");
  int rc;
  for (int step = 0; step < T_; ++step) {
    rc = velocity3d<T>(g, k.radius, tp, I + step * S1, z + step * S1, v + step * SV, tmp,
                       guard ? guard + step : nullptr, T_ + 1, s);
    if (rc) return check_rc(rc, "velocity3d");
    rc = sl_step3d<T>(g, dt, mu, I + step * S1, z + step * S1, v + step * SV, I + (step + 1) * S1,
                      z + (step + 1) * S1, ph[step & 1], ph[(step + 1) & 1], s,
                      (guard && step == 0) ? guard : nullptr, guard ? guard + step + 1 : nullptr,
                      T_ + 1);
    if (rc) return check_rc(rc, "sl_step3d");
  }
  rc = velocity3d<T>(g, k.radius, tp, I + T_ * S1, z + T_ * S1, v + T_ * SV, tmp,
                     guard ? guard + T_ : nullptr, T_ + 1, s);
  if (rc) return check_rc(rc, "velocity3d");
  return MR_OK;
}

template <typename T>
static int shoot_forward(const mr_grid& mg, const mr_kernel& k, int scheme, double mu, int T_, void* trI,
                         void* trz, void* trv, void* phi, int32_t* guard, void* ws,
                         cudaStream_t s) {
  Taps<T> tp;
  int rc = make_taps<T>(k, tp);
  if (rc) return rc;
  if (mg.ndim == 3) {
    if (!ws) return fail(MR_EINVAL, "3D shoot needs a workspace (mr_forward_workspace_bytes)");
    return shoot_forward3d<T>(mg, k, tp, mu, T_, static_cast<T*>(trI), static_cast<T*>(trz),
                              static_cast<T*>(trv), phi, guard, static_cast<T*>(ws), s);
  }
  const Grid2 g = grid2(mg);
  const double dt = 1.0 / T_;  // ShootingConfig.dt (integrator.py:67-69)
  T* I = static_cast<T*>(trI);
  T* z = static_cast<T*>(trz);
  T* v = static_cast<T*>(trv);
  const long long S1 = (long long)g.B * g.N;  // scalar state stride
  const long long SV = 2 * S1;                 // vector state stride
  T* ph[2] = {nullptr, nullptr};
  if (phi) {
    // phi holds 2 x [B][2][N]; the result ends in the first half.
    T* base = static_cast<T*>(phi);
    ph[0] = (T_ % 2 == 0) ? base : base + SV;
    ph[1] = (T_ % 2 == 0) ? base + SV : base;
    k_identity2d<T><<<592, 256, 0, s>>>(ph[0], g);
  }
  if (guard && cudaMemsetAsync(guard, 0, sizeof(int32_t) * (size_t)g.B * (T_ + 1), s) != cudaSuccess)
    return check_cuda("memset guard");
  // split velocity (two kernels, whole-column axis-0 pass) once its 64 x 32 tiles
  // fill the GPU twice; the single-kernel path below that (launch-bound sizes)
  if ((long long)((g.W + 63) / 64) * ((g.H + 31) / 32) * g.B < 2 * 148) ws = nullptr;
  for (int step = 0; step < T_; ++step) {
    rc = launch_velocity2d<T>(g, k.radius, tp, I + step * S1, z + step * S1, v + step * SV,
                              guard ? guard + step : nullptr, T_ + 1, s, static_cast<T*>(ws));
    if (rc) return check_rc(rc, "velocity");
    if (scheme == kSchemeSL)
      rc = launch_sl_step2d<T>(g, dt, mu, I + step * S1, z + step * S1, v + step * SV,
                               I + (step + 1) * S1, z + (step + 1) * S1, ph[step & 1],
                               ph[(step + 1) & 1], s,
                               (guard && step == 0) ? guard : nullptr,
                               guard ? guard + step + 1 : nullptr, T_ + 1);
    else
      rc = launch_scheme_step2d<T>(scheme, g, dt, mu, I + step * S1, z + step * S1,
                                   v + step * SV, I + (step + 1) * S1, z + (step + 1) * S1,
                                   ph[step & 1], ph[(step + 1) & 1], s,
                                   (guard && step == 0) ? guard : nullptr,
                                   guard ? guard + step + 1 : nullptr, T_ + 1);
    if (rc) return check_rc(rc, "sl_step");
  }
  rc = launch_velocity2d<T>(g, k.radius, tp, I + T_ * S1, z + T_ * S1, v + T_ * SV,
                            guard ? guard + T_ : nullptr, T_ + 1, s, static_cast<T*>(ws));
  if (rc) return check_rc(rc, "velocity");
  return MR_OK;
}

template <typename T>
static int cost_terms3d(const Grid3& g, double lam, double rho, const T* I0, const T* z0,
                        const T* v0, const T* IT, const T* J, double* terms, T* seed,
                        cudaStream_t s, double* part = nullptr) {
  long long blocks = (g.N + kThreads * 4 - 1) / (kThreads * 4);
  if (blocks > kCostBlocks) blocks = kCostBlocks;
  if (!part) {
    part = terms;
    blocks = 1;
  }
  k_cost_terms3d<T><<<dim3((unsigned)blocks, g.B), kThreads, 0, s>>>(I0, z0, v0, IT, J, seed,
                                                                      part, g);
  k_finalize_terms<<<(g.B + 127) / 128, 128, 0, s>>>(terms, part, (int)blocks, g.B, lam, rho);
  return cuda_status(cudaGetLastError());
}

// ---- adjoint workspace tail (after the per-voxel scalar buffers) -----------------
// [q accumulators: 2 x B*N u64][mbits: B u64][overflow flag][cost partials: B x kCostBlocks x 4]
struct AdjTail {
  unsigned long long* q;
  unsigned long long* mbits;
  int* ovf;
  double* part;
};

static size_t round256(size_t x) { return (x + 255) / 256 * 256; }

static size_t adjoint_head_bytes(int dtype, const mr_grid& g) {
  return (size_t)(dtype == MR_F32 ? 4 : 8) * (size_t)scalars(g) * (g.ndim == 3 ? 11 : 8);
}

static size_t adjoint_tail_bytes(const mr_grid& g) {
  const size_t S1 = (size_t)scalars(g);
  return round256(16 * S1) + round256(8 * (size_t)g.batch) + 256 +
         round256((size_t)g.batch * kCostBlocks * 4 * 8);
}

static AdjTail adjoint_tail(int dtype, const mr_grid& g, void* ws) {
  const size_t S1 = (size_t)scalars(g);
  char* p = static_cast<char*>(ws) + round256(adjoint_head_bytes(dtype, g));
  AdjTail t;
  t.q = reinterpret_cast<unsigned long long*>(p);
  p += round256(16 * S1);
  t.mbits = reinterpret_cast<unsigned long long*>(p);
  p += round256(8 * (size_t)g.batch);
  t.ovf = reinterpret_cast<int*>(p);
  p += 256;
  t.part = reinterpret_cast<double*>(p);
  return t;
}

static dim3 pair_grid(long long N, int B) {
  long long nb = (N + 255) / 256;
  if (nb > 256) nb = 256;
  return dim3((unsigned)nb, (unsigned)B);
}

// Deterministic mode, once per step before the scatter: per-pair max |ibar|, |zbar|.
template <typename T>
static int det_prepare(const AdjTail& t, const T* ibar, const T* zbar, long long N, int B,
                       cudaStream_t s) {
  if (cudaMemsetAsync(t.mbits, 0, sizeof(unsigned long long) * (size_t)B, s) != cudaSuccess)
    return MR_ECUDA;
  k_absmax_pair<T><<<pair_grid(N, B), 256, 0, s>>>(ibar, zbar, N, t.mbits);
  return cuda_status(cudaGetLastError());
}

// ... and after it: fixed point -> T into the scatter targets (cells reset to 0).
template <typename T>
static int det_finish(const AdjTail& t, T* ib, T* zb, long long N, int B, cudaStream_t s) {
  const long long S1 = N * B;
  k_fix_to_float<T><<<pair_grid(N, B), 256, 0, s>>>(t.q, ib, N, t.mbits);
  if (zb) k_fix_to_float<T><<<pair_grid(N, B), 256, 0, s>>>(t.q + S1, zb, N, t.mbits);
  return cuda_status(cudaGetLastError());
}

static __global__ void k_det_flags(int32_t* flags, const int* ovf, int B) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && *ovf) flags[b] |= 2;
}

template <typename T>
static int shoot_adjoint3d(const mr_grid& mg, const mr_kernel& k, const Taps<T>& tp, double mu,
                           int T_, double lam, double rho, const T* I, const T* z, const T* v,
                           const T* J, T* zbar0, double* terms, int32_t* flags, T* w,
                           cudaStream_t s, bool det) {
  const AdjTail tail = adjoint_tail(sizeof(T) == 4 ? MR_F32 : MR_F64, mg, w);
  const Grid3 g = grid3(mg);
  const double dt = 1.0 / T_;
  const long long S1 = (long long)g.B * g.N;
  const long long SV = 3 * S1;
  T* cur = w;              // ibar | zbar   (2*S1)
  T* acc = w + 2 * S1;     // ib   | zb     (2*S1)
  T* vbar = w + 4 * S1;    // 3*S1
  T* tmp = w + 7 * S1;     // 3*S1
  T* sbuf = w + 10 * S1;   // S1
  Grid2 sl{g.B * 3 * g.D, g.H, g.W, g.HW};
  if (cudaMemsetAsync(flags, 0, sizeof(int32_t) * (size_t)g.B, s) != cudaSuccess)
    return check_cuda("memset flags");
  int rc = cost_terms3d<T>(g, lam, rho, I, z, v, I + T_ * S1, J, terms, cur, s, tail.part);
  if (rc) return check_rc(rc, "cost_terms3d");
  if (cudaMemsetAsync(cur + S1, 0, sizeof(T) * S1, s) != cudaSuccess) return check_cuda("memset");
  if (det && (cudaMemsetAsync(tail.q, 0, 16 * (size_t)S1, s) != cudaSuccess ||
              cudaMemsetAsync(tail.ovf, 0, sizeof(int), s) != cudaSuccess))
    return check_cuda("memset");
  for (int step = T_ - 1; step >= 0; --step) {
    if (det) {
      if ((rc = det_prepare<T>(tail, cur, cur + S1, g.N, g.B, s))) return check_rc(rc, "det");
    } else if (cudaMemsetAsync(acc, 0, sizeof(T) * 2 * S1, s) != cudaSuccess) {
      return check_cuda("memset");
    }
    Adj3Args<T> a{};
    a.I = I + step * S1;
    a.z = z + step * S1;
    a.v = v + step * SV;
    a.ibar = cur;
    a.zbar = cur + S1;
    a.s = sbuf;
    a.ib = acc;
    a.zb = acc + S1;
    a.vbar = vbar;
    a.s_out = sbuf;
    a.dt = (T)dt;
    a.dtmu = (T)(dt * mu);
    a.has_mu = mu != 0.0;
    a.reg_lam = (T)(step == 0 ? lam : 0.0);
    a.g = g;
    a.qib = tail.q;
    a.qzb = tail.q + S1;
    a.mbits = tail.mbits;
    a.ovf = tail.ovf;
    k_divseed3d<T><<<grid3d(g), kThreads, 0, s>>>(a);
    if (det)
      k_sl_adjoint3d<T, true><<<grid3d(g), kThreads, 0, s>>>(a);
    else
      k_sl_adjoint3d<T><<<grid3d(g), kThreads, 0, s>>>(a);
    if ((rc = cuda_status(cudaGetLastError()))) return check_rc(rc, "sl_adjoint3d");
    if (det && (rc = det_finish<T>(tail, acc, acc + S1, g.N, g.B, s))) return check_rc(rc, "det");
    // ktv = K^T vbar: axis 0 first, then axes 1, 2 per slice (kernel.py:76-79 order)
    rc = launch_fir_axis0<T>(k.radius, tp, vbar, tmp, g.B * 3, g.D, g.HW, true, 0, nullptr, 1, 3, s);
    if (rc) return check_rc(rc, "fir_axis0^T");
    rc = launch_smooth2d<T>(sl, k.radius, tp, tmp, vbar, true, s);
    if (rc) return check_rc(rc, "smooth2d^T");
    VelAdj3Args<T> e{};
    e.I = a.I;
    e.z = a.z;
    e.ktv = vbar;
    e.ib = acc;
    e.zb = acc + S1;
    e.lam = (T)lam;
    e.two_rho = (T)(2.0 * rho);
    e.g = g;
    if (step == 0) {
      e.v0 = v;
      e.zout = zbar0;
      e.flags = flags;
      k_veladj_epi3d<T, true><<<grid3d(g), kThreads, 0, s>>>(e);
    } else {
      k_veladj_epi3d_k<T, kEpiK><<<grid3d_k(g, kEpiK), kThreads, 0, s>>>(e);
    }
    if ((rc = cuda_status(cudaGetLastError()))) return check_rc(rc, "veladj_epi3d");
    T* t = cur;
    cur = acc;
    acc = t;
  }
  if (det) {
    k_det_flags<<<(g.B + 127) / 128, 128, 0, s>>>(flags, tail.ovf, g.B);
    if ((rc = cuda_status(cudaGetLastError()))) return check_rc(rc, "det flags");
  }
  return MR_OK;
}

template <typename T>
static int shoot_adjoint(const mr_grid& mg, const mr_kernel& k, int scheme, double mu, int T_, double lam,
                         double rho, const void* trI, const void* trz, const void* trv,
                         const void* Jv, void* zbar0, double* terms, int32_t* flags, void* ws,
                         cudaStream_t s, bool det) {
  Taps<T> tp;
  int rc = make_taps<T>(k, tp);
  if (rc) return rc;
  if (mg.ndim == 3)
    return shoot_adjoint3d<T>(mg, k, tp, mu, T_, lam, rho, static_cast<const T*>(trI),
                              static_cast<const T*>(trz), static_cast<const T*>(trv),
                              static_cast<const T*>(Jv), static_cast<T*>(zbar0), terms, flags,
                              static_cast<T*>(ws), s, det);
  const AdjTail tail = adjoint_tail(sizeof(T) == 4 ? MR_F32 : MR_F64, mg, ws);
  const Grid2 g = grid2(mg);
  const double dt = 1.0 / T_;
  const T* I = static_cast<const T*>(trI);
  const T* z = static_cast<const T*>(trz);
  const T* v = static_cast<const T*>(trv);
  const T* J = static_cast<const T*>(Jv);
  const long long S1 = (long long)g.B * g.N;
  const long long SV = 2 * S1;
  T* w = static_cast<T*>(ws);
  // workspace: [ibar, zbar] [ib_acc, zb_acc] vbar
  T* cur = w;            // ibar | zbar   (2*S1)
  T* acc = w + 2 * S1;   // ib   | zb     (2*S1)
  T* vbar = w + 4 * S1;  // 2*S1
  T* vtmp = w + 6 * S1;  // 2*S1: axis-0 pass of the split velocity adjoint
  if (cudaMemsetAsync(flags, 0, sizeof(int32_t) * (size_t)g.B, s) != cudaSuccess)
    return check_cuda("memset flags");
  rc = launch_cost_terms2d<T>(g, lam, rho, I, z, v, I + T_ * S1, J, terms, cur, s, tail.part);
  if (rc) return check_rc(rc, "cost_terms");
  // zbar_T = 0 and the first scatter targets; afterwards the velocity-adjoint
  // kernel of each step zeroes the buffers the next step scatters into
  if (cudaMemsetAsync(cur + S1, 0, sizeof(T) * S1, s) != cudaSuccess) return check_cuda("memset");
  if (cudaMemsetAsync(acc, 0, sizeof(T) * 2 * S1, s) != cudaSuccess) return check_cuda("memset");
  const bool det_scatter = det && scheme != kSchemeEuler;  // the Eulerian adjoint has no scatter
  if (det_scatter && (cudaMemsetAsync(tail.q, 0, 16 * (size_t)S1, s) != cudaSuccess ||
                      cudaMemsetAsync(tail.ovf, 0, sizeof(int), s) != cudaSuccess))
    return check_cuda("memset");
  for (int step = T_ - 1; step >= 0; --step) {
    if (det_scatter) {
      if ((rc = det_prepare<T>(tail, cur, cur + S1, g.N, g.B, s))) return check_rc(rc, "det");
      rc = launch_adjoint2d_det<T>(scheme, g, dt, mu, I + step * S1, z + step * S1,
                                   v + step * SV, cur, cur + S1, acc, acc + S1, vbar, tail, s,
                                   step == 0 ? lam : 0.0);
      if (rc) return check_rc(rc, "sl_adjoint (deterministic)");
      rc = det_finish<T>(tail, acc, scheme == kSchemeSL ? acc + S1 : nullptr, g.N, g.B, s);
    } else if (scheme == kSchemeSL) {
      rc = launch_sl_adjoint2d<T>(g, dt, mu, I + step * S1, z + step * S1, v + step * SV, cur,
                                  cur + S1, acc, acc + S1, vbar, s, step == 0 ? lam : 0.0);
    } else {
      rc = launch_scheme_adj2d<T>(scheme, g, dt, mu, I + step * S1, z + step * S1,
                                  v + step * SV, cur, cur + S1, acc, acc + S1, vbar, s,
                                  step == 0 ? lam : 0.0);
    }
    if (rc) return check_rc(rc, "sl_adjoint");
    VelAdjArgs<T> a{};
    a.I = I + step * S1;
    a.z = z + step * S1;
    a.vbar = vbar;
    a.vtmp = vtmp;
    a.ib = acc;
    a.zb = acc + S1;
    a.g = g;
    a.lam = (T)lam;
    a.two_rho = (T)(2.0 * rho);
    const bool reg = (step == 0);
    if (!reg) {  // ibar/zbar of step k+1 are consumed: zero them for the next scatter
      a.zero_a = cur;
      a.zero_b = cur + S1;
    }
    if (reg) {
      a.v0 = v;  // v at k = 0
      a.zout = static_cast<T*>(zbar0);
      a.flags = flags;
    }
    rc = launch_velocity_adj2d<T>(g, k.radius, tp, a, reg, s);
    if (rc) return check_rc(rc, "velocity_adjoint");
    T* t = cur;
    cur = acc;
    acc = t;
  }
  if (det_scatter) {
    k_det_flags<<<(g.B + 127) / 128, 128, 0, s>>>(flags, tail.ovf, g.B);
    if ((rc = cuda_status(cudaGetLastError()))) return check_rc(rc, "det flags");
  }
  return MR_OK;
}

}  // namespace mr

using namespace mr;

// ================================ C ABI ===========================================
extern "C" {

int mr_version(void) { return 1; }

const char* mr_last_error(void) { return g_last_error.c_str(); }

const char* mr_strerror(int code) {
  switch (code) {
    case MR_OK: return "ok";
    case MR_EINVAL: return "invalid argument";
    case MR_ECUDA: return "CUDA error";
    default: return "unknown error";
  }
}

#define MR_DISPATCH(dtype, CALL_F32, CALL_F64) ((dtype) == MR_F32 ? (CALL_F32) : (CALL_F64))

int mr_velocity(int dtype, mr_grid g, mr_kernel k, const void* I, const void* z, void* v,
                int32_t* guard, void* workspace, void* stream) {
  int rc = validate(dtype, g, false);
  if (rc) return rc;
  if (!I || !z || !v) return fail(MR_EINVAL, "NULL field pointer");
  Grid2 g2 = grid2(g);
  if (dtype == MR_F32) {
    Taps<float> tp;
    if ((rc = make_taps<float>(k, tp))) return rc;
    rc = launch_velocity2d<float>(g2, k.radius, tp, (const float*)I, (const float*)z, (float*)v,
                                  guard, 1, as_stream(stream), (float*)workspace);
  } else {
    Taps<double> tp;
    if ((rc = make_taps<double>(k, tp))) return rc;
    rc = launch_velocity2d<double>(g2, k.radius, tp, (const double*)I, (const double*)z,
                                   (double*)v, guard, 1, as_stream(stream));
  }
  return check_rc(rc, "mr_velocity");
}

int mr_smooth(int dtype, mr_grid g, mr_kernel k, const void* a, void* out, int32_t adjoint,
              void* stream) {
  int rc = validate(dtype, g, false);
  if (rc) return rc;
  if (!a || !out) return fail(MR_EINVAL, "NULL field pointer");
  Grid2 g2 = grid2(g);
  if (dtype == MR_F32) {
    Taps<float> tp;
    if ((rc = make_taps<float>(k, tp))) return rc;
    rc = launch_smooth2d<float>(g2, k.radius, tp, (const float*)a, (float*)out, adjoint != 0,
                                as_stream(stream));
  } else {
    Taps<double> tp;
    if ((rc = make_taps<double>(k, tp))) return rc;
    rc = launch_smooth2d<double>(g2, k.radius, tp, (const double*)a, (double*)out, adjoint != 0,
                                 as_stream(stream));
  }
  return check_rc(rc, "mr_smooth");
}

int mr_sl_step(int dtype, mr_grid g, double dt, double mu, const void* I, const void* z,
               const void* v, void* I_next, void* z_next, const void* phi_in, void* phi_out,
               void* stream) {
  int rc = validate(dtype, g);
  if (rc) return rc;
  if (!I || !z || !v || !I_next || !z_next) return fail(MR_EINVAL, "NULL field pointer");
  if ((phi_in == nullptr) != (phi_out == nullptr))
    return fail(MR_EINVAL, "phi_in and phi_out must both be set or both be NULL");
  if (g.ndim == 3) {
    Grid3 g3 = grid3(g);
    rc = MR_DISPATCH(dtype,
                     sl_step3d<float>(g3, dt, mu, (const float*)I, (const float*)z,
                                      (const float*)v, (float*)I_next, (float*)z_next,
                                      (const float*)phi_in, (float*)phi_out, as_stream(stream)),
                     sl_step3d<double>(g3, dt, mu, (const double*)I, (const double*)z,
                                       (const double*)v, (double*)I_next, (double*)z_next,
                                       (const double*)phi_in, (double*)phi_out,
                                       as_stream(stream)));
    return check_rc(rc, "mr_sl_step");
  }
  Grid2 g2 = grid2(g);
  rc = MR_DISPATCH(dtype,
                   launch_sl_step2d<float>(g2, dt, mu, (const float*)I, (const float*)z,
                                           (const float*)v, (float*)I_next, (float*)z_next,
                                           (const float*)phi_in, (float*)phi_out,
                                           as_stream(stream)),
                   launch_sl_step2d<double>(g2, dt, mu, (const double*)I, (const double*)z,
                                            (const double*)v, (double*)I_next, (double*)z_next,
                                            (const double*)phi_in, (double*)phi_out,
                                            as_stream(stream)));
  return check_rc(rc, "mr_sl_step");
}

int mr_scheme_step(int dtype, mr_grid g, int32_t scheme, double dt, double mu, const void* I,
                   const void* z, const void* v, void* I_next, void* z_next, const void* phi_in,
                   void* phi_out, void* stream) {
  if (scheme == MR_SCHEME_SEMI_LAGRANGIAN)
    return mr_sl_step(dtype, g, dt, mu, I, z, v, I_next, z_next, phi_in, phi_out, stream);
  if (scheme != MR_SCHEME_EULERIAN && scheme != MR_SCHEME_HYBRID)
    return fail(MR_EINVAL, "unknown scheme");
  int rc = validate(dtype, g, false);
  if (rc) return rc;
  if (!I || !z || !v || !I_next || !z_next) return fail(MR_EINVAL, "NULL field pointer");
  if ((phi_in == nullptr) != (phi_out == nullptr))
    return fail(MR_EINVAL, "phi_in and phi_out must both be set or both be NULL");
  Grid2 g2 = grid2(g);
  rc = MR_DISPATCH(dtype,
                   launch_scheme_step2d<float>(scheme, g2, dt, mu, (const float*)I, (const float*)z,
                                               (const float*)v, (float*)I_next, (float*)z_next,
                                               (const float*)phi_in, (float*)phi_out,
                                               as_stream(stream), nullptr, nullptr, 1),
                   launch_scheme_step2d<double>(scheme, g2, dt, mu, (const double*)I,
                                                (const double*)z, (const double*)v,
                                                (double*)I_next, (double*)z_next,
                                                (const double*)phi_in, (double*)phi_out,
                                                as_stream(stream), nullptr, nullptr, 1));
  return check_rc(rc, "mr_scheme_step");
}

int mr_sl_step_adjoint(int dtype, mr_grid g, double dt, double mu, const void* I, const void* z,
                       const void* v, const void* ibar, const void* zbar, void* ib, void* zb,
                       void* vbar, void* stream) {
  int rc = validate(dtype, g, false);
  if (rc) return rc;
  if (!I || !z || !v || !ibar || !zbar || !ib || !zb || !vbar)
    return fail(MR_EINVAL, "NULL field pointer");
  Grid2 g2 = grid2(g);
  rc = MR_DISPATCH(
      dtype,
      launch_sl_adjoint2d<float>(g2, dt, mu, (const float*)I, (const float*)z, (const float*)v,
                                 (const float*)ibar, (const float*)zbar, (float*)ib, (float*)zb,
                                 (float*)vbar, as_stream(stream)),
      launch_sl_adjoint2d<double>(g2, dt, mu, (const double*)I, (const double*)z,
                                  (const double*)v, (const double*)ibar, (const double*)zbar,
                                  (double*)ib, (double*)zb, (double*)vbar, as_stream(stream)));
  return check_rc(rc, "mr_sl_step_adjoint");
}

int mr_velocity_adjoint(int dtype, mr_grid g, mr_kernel k, const void* I, const void* z,
                        const void* vbar, void* ib, void* zb, void* workspace, void* stream) {
  int rc = validate(dtype, g, false);
  if (rc) return rc;
  if (!I || !z || !vbar || !ib || !zb) return fail(MR_EINVAL, "NULL field pointer");
  Grid2 g2 = grid2(g);
  if (dtype == MR_F32) {
    Taps<float> tp;
    if ((rc = make_taps<float>(k, tp))) return rc;
    VelAdjArgs<float> a{};
    a.I = (const float*)I; a.z = (const float*)z; a.vbar = (const float*)vbar;
    a.ib = (float*)ib; a.zb = (float*)zb; a.g = g2;
    a.vtmp = (float*)workspace;
    rc = launch_velocity_adj2d<float>(g2, k.radius, tp, a, false, as_stream(stream));
  } else {
    Taps<double> tp;
    if ((rc = make_taps<double>(k, tp))) return rc;
    VelAdjArgs<double> a{};
    a.I = (const double*)I; a.z = (const double*)z; a.vbar = (const double*)vbar;
    a.ib = (double*)ib; a.zb = (double*)zb; a.g = g2;
    rc = launch_velocity_adj2d<double>(g2, k.radius, tp, a, false, as_stream(stream));
  }
  return check_rc(rc, "mr_velocity_adjoint");
}

size_t mr_forward_workspace_bytes(int dtype, mr_grid g) {
  if (validate(dtype, g)) return 0;
  // 2D: optional (NULL keeps the single-kernel velocity); 2 scalars per pixel
  // hold the axis-1 pass of the split fp32 velocity.  3D: 3 scalars per voxel.
  return (size_t)(dtype == MR_F32 ? 4 : 8) * (size_t)scalars(g) * (g.ndim == 2 ? 2 : 3);
}

static int validate_scheme(int32_t scheme, const mr_grid& g) {
  if (scheme != MR_SCHEME_SEMI_LAGRANGIAN && scheme != MR_SCHEME_EULERIAN &&
      scheme != MR_SCHEME_HYBRID)
    return fail(MR_EINVAL, "unknown scheme " + std::to_string(scheme));
  if (scheme != MR_SCHEME_SEMI_LAGRANGIAN && g.ndim != 2)
    return fail(MR_EINVAL, "the eulerian and hybrid schemes are 2D (as the reference)");
  return MR_OK;
}

int mr_shoot_forward(int dtype, mr_grid g, mr_kernel k, double mu, int32_t n_steps,
                     void* traj_I, void* traj_z, void* traj_v, void* phi, int32_t* guard,
                     void* workspace, void* stream) {
  return mr_shoot_forward_scheme(dtype, g, k, MR_SCHEME_SEMI_LAGRANGIAN, mu, n_steps, traj_I,
                                 traj_z, traj_v, phi, guard, workspace, stream);
}

int mr_shoot_forward_scheme(int dtype, mr_grid g, mr_kernel k, int32_t scheme, double mu,
                            int32_t n_steps, void* traj_I, void* traj_z, void* traj_v, void* phi,
                            int32_t* guard, void* workspace, void* stream) {
  int rc = validate(dtype, g);
  if (rc) return rc;
  if ((rc = validate_scheme(scheme, g))) return rc;
  if (n_steps < 1) return fail(MR_EINVAL, "n_steps must be >= 1, got " + std::to_string(n_steps));
  if (!(mu >= 0.0)) return fail(MR_EINVAL, "mu must be >= 0");
  if (!traj_I || !traj_z || !traj_v) return fail(MR_EINVAL, "NULL trajectory pointer");
  rc = MR_DISPATCH(dtype,
                   shoot_forward<float>(g, k, scheme, mu, n_steps, traj_I, traj_z, traj_v, phi, guard,
                                        workspace, as_stream(stream)),
                   shoot_forward<double>(g, k, scheme, mu, n_steps, traj_I, traj_z, traj_v, phi, guard,
                                         workspace, as_stream(stream)));
  if (rc) return rc;
  return check_cuda("mr_shoot_forward");
}

size_t mr_adjoint_workspace_bytes(int dtype, mr_grid g) {
  if (validate(dtype, g)) return 0;
  return round256(adjoint_head_bytes(dtype, g)) + adjoint_tail_bytes(g);
}

size_t mr_cost_workspace_bytes(int dtype, mr_grid g) {
  if (validate(dtype, g)) return 0;
  return (size_t)g.batch * kCostBlocks * 4 * sizeof(double);
}

int mr_shoot_adjoint(int dtype, mr_grid g, mr_kernel k, double mu, int32_t n_steps, double lam,
                     double rho, const void* traj_I, const void* traj_z, const void* traj_v,
                     const void* J, void* zbar0, double* terms, int32_t* flags, void* workspace,
                     void* stream) {
  return mr_shoot_adjoint_scheme(dtype, g, k, MR_SCHEME_SEMI_LAGRANGIAN, mu, n_steps, lam, rho,
                                 traj_I, traj_z, traj_v, J, zbar0, terms, flags, workspace,
                                 stream);
}

int mr_shoot_adjoint_scheme(int dtype, mr_grid g, mr_kernel k, int32_t scheme, double mu,
                            int32_t n_steps, double lam, double rho, const void* traj_I,
                            const void* traj_z, const void* traj_v, const void* J, void* zbar0,
                            double* terms, int32_t* flags, void* workspace, void* stream) {
  return mr_shoot_adjoint_ex(dtype, g, k, scheme, mu, n_steps, lam, rho, traj_I, traj_z, traj_v,
                             J, zbar0, terms, flags, workspace, 0, stream);
}

int mr_shoot_adjoint_ex(int dtype, mr_grid g, mr_kernel k, int32_t scheme, double mu,
                        int32_t n_steps, double lam, double rho, const void* traj_I,
                        const void* traj_z, const void* traj_v, const void* J, void* zbar0,
                        double* terms, int32_t* flags, void* workspace, int32_t options,
                        void* stream) {
  if (options & ~MR_OPT_DETERMINISTIC) return fail(MR_EINVAL, "unknown option bits");
  const bool det = (options & MR_OPT_DETERMINISTIC) != 0;
  int rc = validate(dtype, g);
  if (rc) return rc;
  if ((rc = validate_scheme(scheme, g))) return rc;
  if (n_steps < 1) return fail(MR_EINVAL, "n_steps must be >= 1");
  if (!(lam > 0.0)) return fail(MR_EINVAL, "lambda must be positive");
  if (!(rho >= 0.0)) return fail(MR_EINVAL, "rho must be >= 0");
  if (!traj_I || !traj_z || !traj_v || !J || !zbar0 || !terms || !flags || !workspace)
    return fail(MR_EINVAL, "NULL pointer");
  rc = MR_DISPATCH(dtype,
                   shoot_adjoint<float>(g, k, scheme, mu, n_steps, lam, rho, traj_I, traj_z, traj_v, J,
                                        zbar0, terms, flags, workspace, as_stream(stream), det),
                   shoot_adjoint<double>(g, k, scheme, mu, n_steps, lam, rho, traj_I, traj_z, traj_v, J,
                                         zbar0, terms, flags, workspace, as_stream(stream), det));
  if (rc) return rc;
  return check_cuda("mr_shoot_adjoint");
}

int mr_cost_terms(int dtype, mr_grid g, double lam, double rho, const void* I0, const void* z0,
                  const void* v0, const void* IT, const void* J, double* terms, void* ibar_seed,
                  void* workspace, void* stream) {
  double* part = static_cast<double*>(workspace);
  int rc = validate(dtype, g);
  if (rc) return rc;
  if (!I0 || !z0 || !v0 || !IT || !J || !terms) return fail(MR_EINVAL, "NULL pointer");
  if (g.ndim == 3) {
    Grid3 g3 = grid3(g);
    rc = MR_DISPATCH(dtype,
                     cost_terms3d<float>(g3, lam, rho, (const float*)I0, (const float*)z0,
                                         (const float*)v0, (const float*)IT, (const float*)J,
                                         terms, (float*)ibar_seed, as_stream(stream), part),
                     cost_terms3d<double>(g3, lam, rho, (const double*)I0, (const double*)z0,
                                          (const double*)v0, (const double*)IT,
                                          (const double*)J, terms, (double*)ibar_seed,
                                          as_stream(stream), part));
    return check_rc(rc, "mr_cost_terms");
  }
  Grid2 g2 = grid2(g);
  rc = MR_DISPATCH(dtype,
                   launch_cost_terms2d<float>(g2, lam, rho, (const float*)I0, (const float*)z0,
                                              (const float*)v0, (const float*)IT, (const float*)J,
                                              terms, (float*)ibar_seed, as_stream(stream), part),
                   launch_cost_terms2d<double>(g2, lam, rho, (const double*)I0,
                                               (const double*)z0, (const double*)v0,
                                               (const double*)IT, (const double*)J, terms,
                                               (double*)ibar_seed, as_stream(stream), part));
  return check_rc(rc, "mr_cost_terms");
}

}  // extern "C"
