// fp32 instantiation of the engine kernels (the product path).
#include "uuv_kernels.cuh"
#include "uuv_common_kernels.cuh"

UUV_INSTANTIATE(float)
