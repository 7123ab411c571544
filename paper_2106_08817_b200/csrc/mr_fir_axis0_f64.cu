#include "mr_fir_impl.cuh"
MR_INSTANTIATE_AXIS0(double)
