// mr_ops.cu -- array-level operators of the reference API on the device.
//
// These are the building blocks the reference re-exports and its tests call
// directly (morphreg/__init__.py:5-89; fields.py:144-280; kernel.py:36-92):
// np.gradient along one axis and its exact transpose, gradient / divergence,
// the replicate-border 1D FIR and its exact transpose, and multilinear
// interpolation at arbitrary sample coordinates with its value transpose and
// coordinate derivative.  They are not on the shooting hot path (the whole-loop
// kernels fuse all of them); they exist so `paper_2106_08817_b200` is a
// drop-in for code that uses the operators one by one.  Both precisions; the
// fp64 instantiation follows the reference's evaluation order (separate
// multiply and add where numpy rounds them separately), so it reproduces the
// reference to the last bit on the forward operators.
//
// Layout: scalar batch [B][N], vector batch [B][d][N], N = n0*n1(*n2), C order.
#include <cmath>
#include <string>

#include "mr_common.cuh"

namespace mr {
namespace ops {

struct OpGrid {
  int B, d;
  int n[3];
  long long st[3];  // element stride of each axis
  long long N;
};

// ndim 1..3 (the reference's array operators accept any ndarray: 1D lines are
// used by its dense-transpose tests); unused trailing extents are 1.
static OpGrid op_grid(const mr_grid& g) {
  OpGrid o;
  o.B = g.batch;
  o.d = g.ndim;
  for (int i = 0; i < 3; ++i) o.n[i] = i < g.ndim ? g.n[i] : 1;
  o.st[2] = 1;
  o.st[1] = o.n[2];
  o.st[0] = (long long)o.n[1] * o.n[2];
  if (g.ndim == 2) {  // [H][W]: axis 0 stride W, axis 1 stride 1
    o.st[0] = o.n[1];
    o.st[1] = 1;
  } else if (g.ndim == 1) {
    o.st[0] = 1;
  }
  o.N = (long long)o.n[0] * o.n[1] * o.n[2];
  return o;
}

__device__ __forceinline__ int coord(const OpGrid& g, long long q, int ax) {
  return (int)((q / g.st[ax]) % g.n[ax]);
}

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

// np.gradient (unit spacing, edge_order 1) of one line at index j (fields.py:144-145)
template <typename T>
__device__ __forceinline__ T diff_at(const T* __restrict__ a, long long q, long long s, int j, int n) {
  if (j == 0) return a[q + s] - a[q];
  if (j == n - 1) return a[q] - a[q - s];
  return (a[q + s] - a[q - s]) / T(2);
}

// axis_diff_adjoint (fields.py:148-158) in gather form, reference term order
template <typename T>
__device__ __forceinline__ T diff_adj_at(const T* __restrict__ g, long long q, long long s, int j,
                                         int n) {
  const long long q0 = q - (long long)j * s;  // line start
  const T gm = j >= 1 ? g[q - s] : T(0);
  const T gp = j + 1 <= n - 1 ? g[q + s] : T(0);
  return diff_adj1(gm, gp, g[q0], g[q0 + (long long)(n - 1) * s], j, n);
}

template <typename T>
__global__ void k_axis_diff(const T* __restrict__ a, T* __restrict__ out, OpGrid g, int ax,
                            int adjoint) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long q = e % g.N;
    const int j = coord(g, q, ax);
    out[e] = adjoint ? diff_adj_at(a, e, g.st[ax], j, g.n[ax]) : diff_at(a, e, g.st[ax], j, g.n[ax]);
  }
}

// gradient_arr (fields.py:161-162): out [B][d][N]
template <typename T>
__global__ void k_gradient(const T* __restrict__ f, T* __restrict__ out, OpGrid g) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / g.N, q = e - b * g.N;
    for (int ax = 0; ax < g.d; ++ax)
      out[(b * g.d + ax) * g.N + q] = diff_at(f, e, g.st[ax], coord(g, q, ax), g.n[ax]);
  }
}

// gradient_adjoint_arr (fields.py:165-166): gbar [B][d][N] -> [B][N], axis order
template <typename T>
__global__ void k_gradient_adjoint(const T* __restrict__ gb, T* __restrict__ out, OpGrid g) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / g.N, q = e - b * g.N;
    T acc = T(0);
    for (int ax = 0; ax < g.d; ++ax) {
      const T t = diff_adj_at(gb + (b * g.d + ax) * g.N, q, g.st[ax], coord(g, q, ax), g.n[ax]);
      acc = ax == 0 ? t : acc + t;
    }
    out[e] = acc;
  }
}

// divergence_arr (fields.py:169-170): v [B][d][N] -> [B][N], axis order
template <typename T>
__global__ void k_divergence(const T* __restrict__ v, T* __restrict__ out, OpGrid g) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / g.N, q = e - b * g.N;
    T acc = T(0);
    for (int ax = 0; ax < g.d; ++ax) {
      const T t = diff_at(v + (b * g.d + ax) * g.N, q, g.st[ax], coord(g, q, ax), g.n[ax]);
      acc = ax == 0 ? t : acc + t;
    }
    out[e] = acc;
  }
}

template <typename T>
struct OpTaps {
  int r;
  T w[2 * kMaxR + 1];
};

// conv1d_replicate (kernel.py:36-45): out = sum_k w_k a[clamp(j + k - r)], taps
// accumulated in k order with separately rounded products (numpy `out += wk * take`).
// Transpose (kernel.py:48-68): zero-padded correlation, plus at j = 0 / n-1 every
// tap that the forward clamped onto that sample.
template <typename T>
__global__ void k_conv1d(const T* __restrict__ a, T* __restrict__ out, OpGrid g, int ax,
                         OpTaps<T> tp, int adjoint) {
  const long long total = (long long)g.B * g.N;
  const int n = g.n[ax], r = tp.r;
  const long long s = g.st[ax];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long q = e % g.N;
    const int j = coord(g, q, ax);
    const long long line = e - (long long)j * s;
    T acc = T(0);
    if (!adjoint) {
      for (int k = 0; k <= 2 * r; ++k) {
        const int i = min(max(j + k - r, 0), n - 1);
        acc = add_rn(acc, mul_rn(tp.w[k], a[line + (long long)i * s]));
      }
    } else {
      // out[j] = sum over (i, k) with clamp(i + k - r) == j of w_k g[i]
      for (int k = 0; k <= 2 * r; ++k) {
        const int i = j - k + r;  // unclamped source hitting j exactly
        if (j != 0 && j != n - 1) {
          if (i >= 0 && i < n) acc += tp.w[k] * a[line + (long long)i * s];
        } else {
          // every i whose tap k lands at or beyond this edge
          const int lo = j == 0 ? 0 : max(n - 1 - k + r, 0);
          const int hi = j == 0 ? min(r - k, n - 1) : n - 1;
          for (int ii = lo; ii <= hi; ++ii) acc += tp.w[k] * a[line + (long long)ii * s];
        }
      }
    }
    out[e] = acc;
  }
}

// ---- multilinear interpolation at absolute coordinates (fields.py:196-262) ------

template <typename T>
struct Plan {
  int i0[3];
  T f[3];
  bool inside[3];
};

// bilinear_plan per axis (fields.py:214-224): clamp to [0, n-1], i0 = min(floor, n-2),
// strict inside mask.
template <typename T>
__device__ __forceinline__ Plan<T> make_plan(const T* __restrict__ coords, long long b, long long q,
                                             const OpGrid& g, int* bad) {
  Plan<T> p;
  for (int ax = 0; ax < g.d; ++ax) {
    T y = coords[(b * g.d + ax) * g.N + q];
    if (!isfinite(y)) {
      if (bad) atomicOr(bad, 1);
      y = T(0);
    }
    const int n = g.n[ax];
    T yc = y < T(0) ? T(0) : (y > T(n - 1) ? T(n - 1) : y);
    int i0 = min((int)floor(yc), n - 2);
    p.i0[ax] = i0;
    p.f[ax] = yc - (T)i0;
    p.inside[ax] = (y > T(0)) && (y < T(n - 1));
  }
  return p;
}

// corner c has offset bit ax = (c >> ax) & 1; weight = product over axes in order
// (2D: a, b, c, d and wy*wx, fy*wx, wy*fx, fy*fx of fields.py:227-240)
template <typename T>
__device__ __forceinline__ T corner_weight(const Plan<T>& p, int d, int c, int skip) {
  T w = T(1);
  bool first = true;
  for (int ax = 0; ax < d; ++ax) {
    if (ax == skip) continue;
    const T wa = ((c >> ax) & 1) ? p.f[ax] : T(1) - p.f[ax];
    w = first ? wa : mul_rn(w, wa);
    first = false;
  }
  return w;
}

template <typename T>
__device__ __forceinline__ long long corner_index(const Plan<T>& p, const OpGrid& g, int c) {
  long long q = 0;
  for (int ax = 0; ax < g.d; ++ax) q += (long long)(p.i0[ax] + ((c >> ax) & 1)) * g.st[ax];
  return q;
}

// interpolate / interpolate_vec / bilinear_apply: a [B][C][N] -> out [B][C][N]
template <typename T>
__global__ void k_interp(const T* __restrict__ coords, const T* __restrict__ a, T* __restrict__ out,
                         OpGrid g, int C, int* bad) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / g.N, q = e - b * g.N;
    const Plan<T> p = make_plan(coords, b, q, g, bad);
    for (int c = 0; c < C; ++c) {
      const T* src = a + (b * C + c) * g.N;
      T acc = T(0);
      for (int k = 0; k < (1 << g.d); ++k) {
        const T t = mul_rn(corner_weight(p, g.d, k, -1), src[corner_index(p, g, k)]);
        acc = k == 0 ? t : add_rn(acc, t);
      }
      out[(b * C + c) * g.N + q] = acc;
    }
  }
}

// bilinear_adjoint_values (fields.py:243-254): out [B][N] += B^T gbar (scatter)
template <typename T>
__global__ void k_interp_adjoint(const T* __restrict__ coords, const T* __restrict__ gbar,
                                 T* __restrict__ out, OpGrid g, int* bad) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / g.N, q = e - b * g.N;
    const Plan<T> p = make_plan(coords, b, q, g, bad);
    const T gv = gbar[e];
    for (int k = 0; k < (1 << g.d); ++k)
      atomicAdd(out + b * g.N + corner_index(p, g, k), corner_weight(p, g.d, k, -1) * gv);
  }
}

// bilinear_coord_grad (fields.py:257-262): out [B][d][N]
template <typename T>
__global__ void k_interp_coord_grad(const T* __restrict__ coords, const T* __restrict__ a,
                                    T* __restrict__ out, OpGrid g, int* bad) {
  const long long total = (long long)g.B * g.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / g.N, q = e - b * g.N;
    const Plan<T> p = make_plan(coords, b, q, g, bad);
    const T* src = a + b * g.N;
    for (int ax = 0; ax < g.d; ++ax) {
      T acc = T(0);
      bool first = true;
      for (int c = 0; c < (1 << g.d); ++c) {
        if ((c >> ax) & 1) continue;
        const T diff = src[corner_index(p, g, c | (1 << ax))] - src[corner_index(p, g, c)];
        const T t = g.d == 1 ? diff : mul_rn(corner_weight(p, g.d, c, ax), diff);
        acc = first ? t : add_rn(acc, t);
        first = false;
      }
      out[(b * g.d + ax) * g.N + q] = mul_rn(acc, (T)(p.inside[ax] ? 1 : 0));
    }
  }
}

// dot (fields.py:285-288) / ssd (fields.py:291-295) / sum of squares per pair:
// one 1024-thread block per pair, fp64 accumulation, fixed-order tree reduction
// (deterministic: the same inputs give the same bits on every run).
template <typename T>
__global__ void __launch_bounds__(1024) k_reduce(const T* __restrict__ a, const T* __restrict__ b,
                                                 double* __restrict__ out, long long N, int op) {
  __shared__ double red[32];
  const long long base = (long long)blockIdx.x * N;
  double acc = 0.0;
  for (long long q = threadIdx.x; q < N; q += blockDim.x) {
    const double x = (double)a[base + q];
    if (op == 0) {
      acc += x * (double)b[base + q];
    } else if (op == 1) {
      const double d = x - (double)b[base + q];
      acc += d * d;
    } else {
      acc += x * x;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = acc;
  __syncthreads();
  if (w == 0) {
    double s = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) out[blockIdx.x] = op == 1 ? 0.5 * s : s;
  }
}

static inline unsigned blocks_for(long long n) {
  long long b = (n + 255) / 256;
  return (unsigned)(b < 1 ? 1 : (b > 65535 * 8 ? 65535 * 8 : b));
}

}  // namespace ops

// error text shared with mr_capi.cu (mr_last_error)
int set_error(int code, const std::string& msg);

}  // namespace mr

using namespace mr;
using namespace mr::ops;

namespace {

int op_validate(int dtype, const mr_grid& g, bool allow1d = false) {
  if (dtype != MR_F32 && dtype != MR_F64) return set_error(MR_EINVAL, "dtype must be MR_F32 or MR_F64");
  if (g.ndim != 2 && g.ndim != 3 && !(allow1d && g.ndim == 1))
    return set_error(MR_EINVAL, allow1d ? "ndim must be 1, 2 or 3" : "ndim must be 2 or 3");
  if (g.batch < 1) return set_error(MR_EINVAL, "batch must be >= 1");
  for (int i = 0; i < g.ndim; ++i)
    if (g.n[i] < 2) return set_error(MR_EINVAL, "every axis needs at least 2 samples");
  return MR_OK;
}

int op_launched(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(MR_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return MR_OK;
}

template <typename T>
int op_taps(const mr_kernel& k, OpTaps<T>& tp) {
  if (k.radius < 1 || k.radius > kMaxR)
    return set_error(MR_EINVAL, "kernel radius must lie in [1, " + std::to_string(kMaxR) + "]");
  if (!k.weights) return set_error(MR_EINVAL, "kernel weights pointer is NULL");
  tp.r = k.radius;
  for (int t = 0; t <= 2 * k.radius; ++t) {
    if (!std::isfinite(k.weights[t])) return set_error(MR_EINVAL, "kernel weights must be finite");
    tp.w[t] = (T)k.weights[t];
  }
  return MR_OK;
}

}  // namespace

extern "C" {

int mr_axis_diff(int dtype, mr_grid g, int32_t axis, const void* a, void* out, int32_t adjoint,
                 void* stream) {
  int rc = op_validate(dtype, g, true);
  if (rc) return rc;
  if (axis < 0 || axis >= g.ndim) return set_error(MR_EINVAL, "axis out of range");
  if (!a || !out) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (dtype == MR_F32)
    k_axis_diff<float><<<nb, 256, 0, s>>>((const float*)a, (float*)out, o, axis, adjoint);
  else
    k_axis_diff<double><<<nb, 256, 0, s>>>((const double*)a, (double*)out, o, axis, adjoint);
  return op_launched("mr_axis_diff");
}

int mr_gradient(int dtype, mr_grid g, const void* f, void* out, int32_t adjoint, void* stream) {
  int rc = op_validate(dtype, g);
  if (rc) return rc;
  if (!f || !out) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (adjoint) {
    if (dtype == MR_F32)
      k_gradient_adjoint<float><<<nb, 256, 0, s>>>((const float*)f, (float*)out, o);
    else
      k_gradient_adjoint<double><<<nb, 256, 0, s>>>((const double*)f, (double*)out, o);
  } else if (dtype == MR_F32) {
    k_gradient<float><<<nb, 256, 0, s>>>((const float*)f, (float*)out, o);
  } else {
    k_gradient<double><<<nb, 256, 0, s>>>((const double*)f, (double*)out, o);
  }
  return op_launched("mr_gradient");
}

int mr_divergence(int dtype, mr_grid g, const void* v, void* out, void* stream) {
  int rc = op_validate(dtype, g);
  if (rc) return rc;
  if (!v || !out) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (dtype == MR_F32)
    k_divergence<float><<<nb, 256, 0, s>>>((const float*)v, (float*)out, o);
  else
    k_divergence<double><<<nb, 256, 0, s>>>((const double*)v, (double*)out, o);
  return op_launched("mr_divergence");
}

int mr_conv1d(int dtype, mr_grid g, mr_kernel k, int32_t axis, const void* a, void* out,
              int32_t adjoint, void* stream) {
  int rc = op_validate(dtype, g, true);
  if (rc) return rc;
  if (axis < 0 || axis >= g.ndim) return set_error(MR_EINVAL, "axis out of range");
  if (!a || !out) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (dtype == MR_F32) {
    OpTaps<float> tp;
    if ((rc = op_taps(k, tp))) return rc;
    k_conv1d<float><<<nb, 256, 0, s>>>((const float*)a, (float*)out, o, axis, tp, adjoint);
  } else {
    OpTaps<double> tp;
    if ((rc = op_taps(k, tp))) return rc;
    k_conv1d<double><<<nb, 256, 0, s>>>((const double*)a, (double*)out, o, axis, tp, adjoint);
  }
  return op_launched("mr_conv1d");
}

int mr_interpolate(int dtype, mr_grid g, const void* coords, const void* a, void* out,
                   int32_t ncomp, int32_t* bad, void* stream) {
  int rc = op_validate(dtype, g);
  if (rc) return rc;
  if (!coords || !a || !out) return set_error(MR_EINVAL, "NULL field pointer");
  if (ncomp < 1) return set_error(MR_EINVAL, "ncomp must be >= 1");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (dtype == MR_F32)
    k_interp<float><<<nb, 256, 0, s>>>((const float*)coords, (const float*)a, (float*)out, o, ncomp, bad);
  else
    k_interp<double><<<nb, 256, 0, s>>>((const double*)coords, (const double*)a, (double*)out, o,
                                        ncomp, bad);
  return op_launched("mr_interpolate");
}

int mr_interpolate_adjoint(int dtype, mr_grid g, const void* coords, const void* gbar, void* out,
                           int32_t* bad, void* stream) {
  int rc = op_validate(dtype, g);
  if (rc) return rc;
  if (!coords || !gbar || !out) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dtype == MR_F32 ? 4 : 8;
  if (cudaMemsetAsync(out, 0, es * (size_t)o.B * o.N, s) != cudaSuccess)
    return op_launched("mr_interpolate_adjoint memset");
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (dtype == MR_F32)
    k_interp_adjoint<float><<<nb, 256, 0, s>>>((const float*)coords, (const float*)gbar, (float*)out,
                                               o, bad);
  else
    k_interp_adjoint<double><<<nb, 256, 0, s>>>((const double*)coords, (const double*)gbar,
                                                (double*)out, o, bad);
  return op_launched("mr_interpolate_adjoint");
}

int mr_interpolate_coord_grad(int dtype, mr_grid g, const void* coords, const void* a, void* out,
                              int32_t* bad, void* stream) {
  int rc = op_validate(dtype, g);
  if (rc) return rc;
  if (!coords || !a || !out) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = blocks_for((long long)o.B * o.N);
  if (dtype == MR_F32)
    k_interp_coord_grad<float><<<nb, 256, 0, s>>>((const float*)coords, (const float*)a, (float*)out,
                                                  o, bad);
  else
    k_interp_coord_grad<double><<<nb, 256, 0, s>>>((const double*)coords, (const double*)a,
                                                   (double*)out, o, bad);
  return op_launched("mr_interpolate_coord_grad");
}

int mr_reduce(int dtype, mr_grid g, int32_t op, const void* a, const void* b, double* out,
              void* stream) {
  int rc = op_validate(dtype, g, true);
  if (rc) return rc;
  if (op < 0 || op > 2) return set_error(MR_EINVAL, "op must be 0 (dot), 1 (ssd) or 2 (sum of squares)");
  if (!a || !out || (op < 2 && !b)) return set_error(MR_EINVAL, "NULL field pointer");
  const OpGrid o = op_grid(g);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == MR_F32)
    k_reduce<float><<<o.B, 1024, 0, s>>>((const float*)a, (const float*)b, out, o.N, op);
  else
    k_reduce<double><<<o.B, 1024, 0, s>>>((const double*)a, (const double*)b, out, o.N, op);
  return op_launched("mr_reduce");
}

}  // extern "C"
