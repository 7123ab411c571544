// Minimal TMA probe (debug aid): load a 3D box with OOB, check values.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2106_08817_b200/csrc/mr_common.cuh"
#include "../../paper_2106_08817_b200/csrc/mr_tma.h"
using namespace mr;
template <int VARIANT>
__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int bx, int by) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  float* dst = reinterpret_cast<float*>(sm + 128);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    if (VARIANT == 0) fence_barrier_init();
    else asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(bar, bx * by * 4);
    tma_load_3d(dst, &map, -3, -2, 1, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = dst[i];
}
int main(int argc, char** argv) {
  int variant0 = atoi(argv[1]);
  int W = atoi(argv[2]), H = atoi(argv[3]), B = 2, bx = atoi(argv[4]), by = atoi(argv[5]);
  std::vector<float> h(W * H * B);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, bx * by * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  bool ok = make_map3<float>(&m, d, W, H, B, bx, by);
  printf("encode ok=%d\n", ok);
  for (int variant = variant0; variant <= variant0; ++variant) {
    cudaMemset(o, 0xff, bx * by * 4);
    if (variant == 0) k<0><<<1, 128, 128 + bx * by * 4>>>(m, o, bx, by);
    else k<1><<<1, 128, 128 + bx * by * 4>>>(m, o, bx, by);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> r(bx * by);
    cudaMemcpy(r.data(), o, bx * by * 4, cudaMemcpyDeviceToHost);
    // element (row 2, col 3) of the box = image (0, 0) of pair 1 = 256
    printf("variant %d: %s  box[2][3]=%g box[0][0]=%g box[3][4]=%g\n", variant, cudaGetErrorString(e), r[2 * bx + 3], r[0], r[3 * bx + 4]);
    if (e) return 1;
  }
  return 0;
}
