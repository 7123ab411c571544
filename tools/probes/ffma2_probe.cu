// Microbenchmark (debug aid): FFMA vs FFMA2 throughput on sm_100a.
#include <cstdio>
__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %4};\n"
      "mov.b64 rc, {%5, %6};\nfma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(w), "f"(c.x), "f"(c.y));
  return d;
}
__global__ void k1(float* out, float w, int iters) {
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], w, 0.5f * i);
  float s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, float w, int iters) {
  float2 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 0.001f + i, i + 0.5f);
  const float2 c = make_float2(0.25f, 0.75f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = ffma2(acc[i], w, c);
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k1<<<148 * 8, 256>>>(o, 0.999f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms1; cudaEventElapsedTime(&ms1, a, b);
    cudaEventRecord(a); k2<<<148 * 8, 256>>>(o, 0.999f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    double fl = 2.0 * 16 * (double)iters * 148 * 8 * 256;
    printf("FFMA : %.3f ms  %.1f TFLOP/s\nFFMA2: %.3f ms  %.1f TFLOP/s\n", ms1, fl / ms1 / 1e9, ms2, fl / ms2 / 1e9);
  }
  return 0;
}
