#include "mr_fir_impl.cuh"
namespace mr {
MR_RADIUS_LIST(MR_VEL_EXTERN_F64)
}
MR_INSTANTIATE_VELOCITY(double)
