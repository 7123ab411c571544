#include "mr_fir_impl.cuh"
MR_INSTANTIATE_VELADJ(float)
