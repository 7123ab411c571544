// Microbenchmark (debug aid): issue rates of FFMA / FFMA2 with register and
// uniform-register (kernel-parameter) multiplicands on sm_100a.
#include <cstdio>
__device__ __forceinline__ float2 f2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\n"
      "mov.b64 rc, {%6, %7};\nfma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
struct W { float w[16]; };
// scalar FFMA, multiplicand in a uniform register (kernel param)
__global__ void k_ffma_u(float* out, W w, int iters) {
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = threadIdx.x * 0.5f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(x, w.w[i], acc[i]);
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// scalar FFMA, all-register operands
__global__ void k_ffma_r(float* out, W w, int iters) {
  float acc[16], wr[16];
  for (int i = 0; i < 16; ++i) { acc[i] = threadIdx.x * 1e-3f + i; wr[i] = w.w[i] + threadIdx.x * 1e-9f; }
  float x = threadIdx.x * 0.5f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(x, wr[i], acc[i]);
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2_u(float* out, W w, int iters) {
  float2 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 x = make_float2(threadIdx.x * 0.5f, 0.25f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = f2(x, make_float2(w.w[i], w.w[i]), acc[i]);
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2_r(float* out, W w, int iters) {
  float2 acc[8], wr[8];
  for (int i = 0; i < 8; ++i) { acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
    float t = w.w[i] + threadIdx.x * 1e-9f; wr[i] = make_float2(t, t); }
  float2 x = make_float2(threadIdx.x * 0.5f, 0.25f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = f2(x, wr[i], acc[i]);
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  W w; for (int i = 0; i < 16; ++i) w.w[i] = 0.999f - 1e-3f * i;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  void (*ks[4])(float*, W, int) = {k_ffma_r, k_ffma_u, k_ffma2_r, k_ffma2_u};
  const char* names[4] = {"FFMA  reg*reg", "FFMA  reg*UR ", "FFMA2 reg*reg", "FFMA2 reg*UR "};
  for (int rep = 0; rep < 2; ++rep)
    for (int k = 0; k < 4; ++k) {
      cudaEventRecord(a); ks[k]<<<148 * 8, 256>>>(o, w, iters); cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fl = 2.0 * 16 * (double)iters * 148 * 8 * 256;
      if (rep) printf("%s: %.3f ms  %.1f TFLOP/s\n", names[k], ms, fl / ms / 1e9);
    }
  return 0;
}
