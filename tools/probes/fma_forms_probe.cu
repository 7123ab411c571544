// Microbenchmark (debug aid): FMA issue forms on sm_100a, in FMA/clk/SM.
//   A  FFMA  x * c[bank] + acc        (weight from the kernel-parameter bank)
//   B  FFMA  x * imm + acc            (weight as an immediate literal)
//   C  FFMA  x * reg + acc            (weight in a register)
//   D  FFMA2 {x,y} * {w,w} + acc2     (packed fp32x2, weight pair in registers)
//   E  FFMA2 with the weight from the parameter bank (uniform register)
// 16 independent accumulators per thread, 8 CTAs x 256 threads per SM.
#include <cstdio>
#include <cstdint>

struct W16 { float w[16]; };

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\n"
      "mov.b64 rc, {%6, %7};\nfma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <int MODE>
__global__ void __launch_bounds__(256) kfma(float* out, W16 wp, const float* wg, int iters,
                                            long long* cyc) {
  float acc[16], x[4];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int i = 0; i < 4; ++i) x[i] = 1.0f + threadIdx.x * 1e-6f * i;
  float wr[16];
  for (int i = 0; i < 16; ++i) wr[i] = wg[(i + threadIdx.x) & 15];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 3 || MODE == 4) {
      float2* a2 = reinterpret_cast<float2*>(acc);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float w = MODE == 3 ? wr[i] : wp.w[i];
        a2[i] = ffma2(make_float2(x[i & 3], x[(i + 1) & 3]), make_float2(w, w), a2[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float w = MODE == 0 ? wp.w[i] : MODE == 1 ? 0.01f * (i + 1) : wr[i];
        acc[i] = fmaf(x[i & 3], w, acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = __int_as_float(__float_as_int(x[i]) ^ (it & 1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int blocks = 148 * 8, threads = 256, iters = 32768;
  float* o; cudaMalloc(&o, blocks * threads * 4);
  float* wg; cudaMalloc(&wg, 64); cudaMemset(wg, 0, 64);
  long long* cyc; cudaMalloc(&cyc, blocks * 8);
  long long* hc = new long long[blocks];
  W16 wp; for (int i = 0; i < 16; ++i) wp.w[i] = 0.01f * (i + 1);
  const char* names[5] = {"FFMA c[bank]", "FFMA imm", "FFMA reg", "FFMA2 reg", "FFMA2 UR"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 5; ++m) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (m == 0) kfma<0><<<blocks, threads>>>(o, wp, wg, iters, cyc);
      if (m == 1) kfma<1><<<blocks, threads>>>(o, wp, wg, iters, cyc);
      if (m == 2) kfma<2><<<blocks, threads>>>(o, wp, wg, iters, cyc);
      if (m == 3) kfma<3><<<blocks, threads>>>(o, wp, wg, iters, cyc);
      if (m == 4) kfma<4><<<blocks, threads>>>(o, wp, wg, iters, cyc);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(hc, cyc, blocks * 8, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < blocks; ++i) mx = hc[i] > mx ? hc[i] : mx;
      const double fma_per_sm = 8.0 * threads * 16.0 * iters;
      printf("%-14s %.3f ms  %.1f FMA/clk/SM (clock64, max block)  %.1f TFMA/s (events)\n",
             names[m], ms, fma_per_sm / mx, fma_per_sm * 148 / (ms * 1e-3) / 1e12);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
