#include "mr_fir_impl.cuh"
namespace mr {
MR_RADIUS_LIST(MR_VEL2_EXTERN)
}
namespace mr {
MR_RADIUS_LIST(MR_VEL_EXTERN_F32)
}
MR_INSTANTIATE_VELOCITY(float)
