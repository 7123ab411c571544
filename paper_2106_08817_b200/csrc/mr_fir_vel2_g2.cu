#include "mr_fir_impl.cuh"
#include "mr_vel2d.cuh"
namespace mr {
MR_RADIUS_GROUP2(MR_VEL2_INST)
}
