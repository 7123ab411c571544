#include "mr_fir_impl.cuh"
namespace mr {
MR_RADIUS_GROUP3(MR_VADJ_INST_F32)
}
