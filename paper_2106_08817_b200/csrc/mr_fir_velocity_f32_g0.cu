#include "mr_fir_impl.cuh"
namespace mr {
MR_RADIUS_LIST(MR_VEL2_EXTERN)
}
namespace mr {
MR_RADIUS_GROUP0(MR_VEL_INST_F32)
}
