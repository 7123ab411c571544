#include "mr_fir_axis0.cuh"
namespace mr {
MR_AX0_GROUP2(MR_AX0_INST_F64)
}
