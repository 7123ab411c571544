// TMA probe variants (debug aid)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2106_08817_b200/csrc/mr_common.cuh"
#include "../../paper_2106_08817_b200/csrc/mr_tma.h"
using namespace mr;
__device__ __forceinline__ void tma3_cta(void* dst, const void* map, int x, int y, int z, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)) : "memory");
}
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, float* out, int bx, int by, int x0, int y0) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  float* dst = reinterpret_cast<float*>(sm + 128);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(bar, bx * by * 4);
    if (V == 0) tma_load_3d(dst, &map, x0, y0, 1, bar);
    if (V == 1) tma3_cta(dst, &map, x0, y0, 1, bar);
    if (V == 2) tma_load_3d(dst, gmap, x0, y0, 1, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = dst[i];
}
int main(int argc, char** argv) {
  int V = atoi(argv[1]);
  int W = atoi(argv[2]), H = atoi(argv[3]), B = 2, bx = atoi(argv[4]), by = atoi(argv[5]);
  int x0 = atoi(argv[6]), y0 = atoi(argv[7]);
  std::vector<float> h(W * H * B);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o; CUtensorMap* gm;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, bx * by * 4); cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  bool ok = make_map3<float>(&m, d, W, H, B, bx, by);
  cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  cudaMemset(o, 0xff, bx * by * 4);
  size_t sm = 128 + bx * by * 4;
  if (V == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<0><<<1, 128, sm>>>(m, gm, o, bx, by, x0, y0); }
  if (V == 1) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<1><<<1, 128, sm>>>(m, gm, o, bx, by, x0, y0); }
  if (V == 2) { cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<2><<<1, 128, sm>>>(m, gm, o, bx, by, x0, y0); }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> r(bx * by);
  cudaMemcpy(r.data(), o, bx * by * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int j = 0; j < by; ++j) for (int i = 0; i < bx; ++i) {
    int gx = x0 + i, gy = y0 + j;
    float ex = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? (float)(W * H + gy * W + gx) : 0.f;
    if (r[j * bx + i] != ex) ++bad;
  }
  printf("V%d W%d H%d box %dx%d at (%d,%d): encode=%d %s mismatches=%d\n", V, W, H, bx, by, x0, y0, ok, cudaGetErrorString(e), bad);
  return e ? 1 : 0;
}
