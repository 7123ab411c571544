#include "mr_fir_impl.cuh"
namespace mr {
MR_RADIUS_GROUP0(MR_VEL_INST_F64)
}
