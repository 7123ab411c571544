// mr_tma.h -- host-side TMA tensor-map encoding (driver entry point via the runtime,
// no link-time dependency on libcuda).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cstring>

namespace mr {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 3D map over a C-contiguous [D][H][W] array (dims W, H, D) with box (bx, by, 1);
// zero fill out of bounds.  Returns false when the layout is not TMA-describable
// (alignment) -- callers then stage with cp.async.
template <typename T>
inline bool make_map3(CUtensorMap* m, const void* base, int W, int H, long long D, int bx, int by) {
  std::memset(m, 0, sizeof(*m));
  auto enc = tma_encode_fn();
  if (!enc || !base) return false;
  const size_t es = sizeof(T);
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if ((W * es) % 16 != 0) return false;
  if (D < 1 || D > INT_MAX || bx > 256 || by > 256 || (bx * es) % 16 != 0) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)D};
  cuuint64_t strides[2] = {(cuuint64_t)W * es, (cuuint64_t)W * (cuuint64_t)H * es};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMapDataType dt =
      sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace mr
