#include "mr_fir_impl.cuh"
namespace mr {
MR_RADIUS_LIST(MR_VADJ_EXTERN_F64)
}
MR_INSTANTIATE_VELADJ(double)
