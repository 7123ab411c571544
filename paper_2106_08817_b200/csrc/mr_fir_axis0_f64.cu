#include "mr_fir_axis0.cuh"
namespace mr {
MR_RADIUS_LIST(MR_AX0_EXTERN_F64)
}
MR_INSTANTIATE_AXIS0(double)
